// dist.cu — vertex-partitioned multi-GPU PageRank over NCCL.
//
// One process per GPU.  Rank r owns destinations [lo_r, hi_r), balanced by
// in-edge count (RMAT in-degrees are skewed), and runs the PULL+WM gather
// (prpull.cuh) over its rows only.  Every iteration:
//   1. local gather + fused vertex update of owned rows -> contrib_next[lo_r:hi_r]
//   2. in-place allgather of the owned contrib slices (grouped ncclBroadcast,
//      slices have unequal lengths) so every rank holds the full vector
//   3. ncclAllReduce of the two f64 scalars (L1 of this iteration, dangling
//      mass of the next) -- adjacent in the scalar array.
// NCCL is resolved with dlopen at first use (reusing the libnccl.so.2 the
// process already loaded, e.g. torch's), so libgg.so has no hard dependency.
#include <dlfcn.h>
#include <cstring>
#include <nccl.h>
#include "prpull.cuh"
#include "prdist.cuh"

namespace gg {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (api.h) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) fail(GG_ERR_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) fail(GG_ERR_NCCL, std::string("libnccl.so.2 lacks ") + n);
    return p;
  };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
  api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  api.h = h;
  return api;
}

#define GG_NCCL(x)                                                                  \
  do {                                                                              \
    ncclResult_t r__ = (x);                                                         \
    if (r__ != ncclSuccess)                                                         \
      ::gg::fail(GG_ERR_NCCL, ::gg::strf("%s failed: %s", #x, nccl().GetErrorString(r__))); \
  } while (0)

// Destination partition balanced by in-edges: lo_r = first v with
// in_off[v] >= r * E / P (computed identically on every rank).
__global__ void k_partition(const int64_t* in_off, int64_t V, int nranks, int64_t* bounds) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > nranks) return;
  if (r == 0) { bounds[0] = 0; return; }
  if (r == nranks) { bounds[r] = V; return; }
  const int64_t E = in_off[V];
  const int64_t target = (int64_t)((__int128)E * r / nranks);
  int64_t lo = 0, hi = V;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (in_off[mid] < target) lo = mid + 1; else hi = mid;
  }
  bounds[r] = lo;
}

}  // namespace gg

using namespace gg;

struct gg_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, dev = 0;
};

#define GG_API_BEGIN try {
#define GG_API_END                      \
  return GG_OK;                         \
  }                                     \
  catch (const gg::Error& e) {          \
    set_last_error(e.what());           \
    return e.code;                      \
  }                                     \
  catch (const std::exception& e) {     \
    set_last_error(e.what());           \
    return GG_ERR_ENGINE;               \
  }

extern "C" {

int gg_nccl_unique_id(char out[128]) {
  GG_API_BEGIN
  if (!out) fail(GG_ERR_VALUE, "null argument");
  ncclUniqueId id;
  GG_NCCL(nccl().GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  GG_API_END
}

int gg_comm_init(int32_t device, int32_t nranks, int32_t rank, const char id[128], gg_comm** out) {
  GG_API_BEGIN
  if (!out || !id) fail(GG_ERR_VALUE, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(GG_ERR_VALUE, "bad rank/nranks");
  DeviceGuard guard(device);
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  auto c = new gg_comm;
  c->rank = rank;
  c->nranks = nranks;
  c->dev = device;
  ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    fail(GG_ERR_NCCL, strf("ncclCommInitRank failed: %s", nccl().GetErrorString(r)));
  }
  *out = c;
  GG_API_END
}

int gg_comm_destroy(gg_comm* c) {
  GG_API_BEGIN
  if (c) {
    if (c->comm) nccl().CommDestroy(c->comm);
    delete c;
  }
  GG_API_END
}

}

namespace gg {
// NCCL exchange of the partitioned EdgeBlocking run (prdist.cuh): one rank
// per process; the slices have unequal lengths, so the all-gather is a group
// of in-place broadcasts (one per owner).
struct NcclExchange : PrExchange {
  gg_comm* c;
  std::vector<void*> opened;  // IPC-mapped peer buffers (closed by unmap_peers)
  explicit NcclExchange(gg_comm* cc) : c(cc) {}
  // Fused all-gather over NVLink: every rank exports its two contribution
  // buffers (cudaIpcGetMemHandle), the handles are all-gathered over NCCL,
  // and each peer's buffers are mapped (cudaIpcOpenMemHandle).  Enabled by
  // GG_PR_P2P=1 (all peers must report peer access); any failure leaves the
  // NCCL all-gather in place.
  bool map_peers(const std::vector<void*>& c0s, const std::vector<void*>& c1s, size_t bytes,
                 std::vector<std::vector<void*>>& pc0, std::vector<std::vector<void*>>& pc1) override {
    const char* e = getenv("GG_PR_P2P");
    if (!e || atoi(e) == 0 || c->nranks < 2 || c->nranks - 1 > 15) return false;
    // every rank must agree, so the decision itself is all-reduced (min);
    // peer access is checked against the peers' actual device ordinals
    int ok = 1;
    {
      DevBuf<int> devs(c->nranks);
      GG_CUDA(cudaMemset(devs.p, 0xff, c->nranks * sizeof(int)));
      GG_CUDA(cudaMemcpy(devs.p + c->rank, &c->dev, sizeof(int), cudaMemcpyHostToDevice));
      NcclApi& api = nccl();
      GG_NCCL(api.GroupStart());
      for (int r = 0; r < c->nranks; ++r)
        GG_NCCL(api.Broadcast(devs.p + r, devs.p + r, 1, ncclInt32, r, c->comm, 0));
      GG_NCCL(api.GroupEnd());
      std::vector<int> hd(c->nranks);
      GG_CUDA(cudaMemcpy(hd.data(), devs.p, c->nranks * sizeof(int), cudaMemcpyDeviceToHost));
      for (int r = 0; r < c->nranks; ++r) {
        if (r == c->rank) continue;
        int can = 0;
        if (hd[r] == c->dev || cudaDeviceCanAccessPeer(&can, c->dev, hd[r]) != cudaSuccess) can = 0;
        ok &= can;
      }
      cudaGetLastError();
    }
    cudaIpcMemHandle_t mine[2];
    if (ok && (cudaIpcGetMemHandle(&mine[0], c0s[0]) != cudaSuccess ||
               cudaIpcGetMemHandle(&mine[1], c1s[0]) != cudaSuccess)) ok = 0;
    cudaGetLastError();
    DevBuf<int> dok(1);
    GG_CUDA(cudaMemcpy(dok.p, &ok, 4, cudaMemcpyHostToDevice));
    GG_NCCL(nccl().AllReduce(dok.p, dok.p, 1, ncclInt32, ncclMin, c->comm, 0));
    GG_CUDA(cudaMemcpy(&ok, dok.p, 4, cudaMemcpyDeviceToHost));
    if (!ok) return false;
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    DevBuf<uint8_t> all(2 * hb * c->nranks);
    GG_CUDA(cudaMemcpy(all.p + 2 * hb * c->rank, mine, 2 * hb, cudaMemcpyHostToDevice));
    {
      NcclApi& api = nccl();
      GG_NCCL(api.GroupStart());
      for (int r = 0; r < c->nranks; ++r)
        GG_NCCL(api.Broadcast(all.p + 2 * hb * r, all.p + 2 * hb * r, 2 * hb, ncclUint8, r, c->comm, 0));
      GG_NCCL(api.GroupEnd());
    }
    std::vector<uint8_t> h(2 * hb * c->nranks);
    GG_CUDA(cudaMemcpy(h.data(), all.p, h.size(), cudaMemcpyDeviceToHost));
    pc0.assign(1, {});
    pc1.assign(1, {});
    for (int r = 0; r < c->nranks; ++r) {
      if (r == c->rank) continue;
      void* p0 = nullptr;
      void* p1 = nullptr;
      cudaIpcMemHandle_t h0, h1;
      memcpy(&h0, h.data() + 2 * hb * r, hb);
      memcpy(&h1, h.data() + 2 * hb * r + hb, hb);
      GG_CUDA(cudaIpcOpenMemHandle(&p0, h0, cudaIpcMemLazyEnablePeerAccess));
      GG_CUDA(cudaIpcOpenMemHandle(&p1, h1, cudaIpcMemLazyEnablePeerAccess));
      opened.push_back(p0);
      opened.push_back(p1);
      pc0[0].push_back(p0);
      pc1[0].push_back(p1);
    }
    (void)bytes;
    return true;
  }
  void unmap_peers() override {
    for (void* q : opened) cudaIpcCloseMemHandle(q);
    opened.clear();
  }
  void allreduce2(std::vector<double*>& d, cudaStream_t st) override {
    NcclApi& api = nccl();
    GG_NCCL(api.AllReduce(d[0], d[0], 2, ncclFloat64, ncclSum, c->comm, st));
  }
  void allgather(std::vector<void*>& bufs, size_t elt, const std::vector<int64_t>& bounds,
                 cudaStream_t st) override {
    NcclApi& api = nccl();
    GG_NCCL(api.GroupStart());
    for (int r = 0; r < c->nranks; ++r) {
      const size_t cnt = (size_t)(bounds[r + 1] - bounds[r]) * elt;
      char* p = (char*)bufs[0] + (size_t)bounds[r] * elt;
      if (cnt) GG_NCCL(api.Broadcast(p, p, cnt, ncclUint8, r, c->comm, st));
    }
    GG_NCCL(api.GroupEnd());
  }
  // overlap: the rest of the all-gather runs on a non-blocking side stream
  // (it does not serialise with the legacy default stream the kernels use)
  cudaStream_t side = nullptr;
  cudaEvent_t ready = nullptr, done = nullptr;
  bool pending = false;
  void allgather_split(std::vector<void*>& bufs, size_t elt, const std::vector<int64_t>& bounds,
                       int64_t hot_end, cudaStream_t st) override {
    std::vector<int64_t> hb(bounds.size()), cb(bounds.size());
    split_bounds(bounds, hot_end, hb, cb);
    if (!side) {
      GG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      GG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
      GG_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    }
    allgather(bufs, elt, hb, st);
    // the rest starts only after the hot part: collectives on one
    // communicator must run in the same order on every rank, so two of them
    // may never be in flight at once from different streams (the main
    // stream's next collective waits for `done` via wait_rest)
    GG_CUDA(cudaEventRecord(ready, st));
    GG_CUDA(cudaStreamWaitEvent(side, ready, 0));
    allgather(bufs, elt, cb, side);
    GG_CUDA(cudaEventRecord(done, side));
    pending = true;
  }
  void wait_rest(cudaStream_t st) override {
    if (pending) GG_CUDA(cudaStreamWaitEvent(st, done, 0));
    pending = false;
  }
  ~NcclExchange() override {
    unmap_peers();
    if (side) {
      cudaStreamSynchronize(side);
      cudaStreamDestroy(side);
      cudaEventDestroy(ready);
      cudaEventDestroy(done);
    }
  }
};

__global__ void k_or_slices(uint32_t* dst, const uint32_t* stage, int64_t n, int parts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = dst[i];
    for (int k = 0; k < parts; ++k) x |= stage[(int64_t)k * n + i];
    dst[i] = x;
  }
}

struct NcclBfsExchange : BfsExchange {
  gg_comm* c;
  DevBuf<uint32_t> stage;  // the peers' slices of this rank's word range
  explicit NcclBfsExchange(gg_comm* cc) : c(cc) {}
  // grouped send/recv: my slice of every peer's bitmap arrives in `stage`,
  // then one kernel ORs them into my words (V/8 bytes per rank per level)
  void alltoall_or_words(std::vector<uint32_t*>& bufs, const std::vector<int64_t>& wb, cudaStream_t st) override {
    NcclApi& api = nccl();
    const int P = c->nranks, me = c->rank;
    const int64_t mine = wb[me + 1] - wb[me];
    if ((int64_t)stage.n < std::max<int64_t>(mine * (P - 1), 1)) stage.alloc(std::max<int64_t>(mine * (P - 1), 1));
    GG_NCCL(api.GroupStart());
    for (int q = 0, k = 0; q < P; ++q) {
      if (q == me) continue;
      const int64_t nq = wb[q + 1] - wb[q];
      if (nq) GG_NCCL(api.Send(bufs[0] + wb[q], (size_t)nq, ncclUint32, q, c->comm, st));
      if (mine) GG_NCCL(api.Recv(stage.p + (int64_t)k * mine, (size_t)mine, ncclUint32, q, c->comm, st));
      ++k;
    }
    GG_NCCL(api.GroupEnd());
    if (mine && P > 1)
      k_or_slices<<<grid_for(mine, 256, c->dev), 256, 0, st>>>(bufs[0] + wb[me], stage.p, mine, P - 1);
    GG_LAUNCH_CHECK();
    bytes += (uint64_t)(P - 1) * (uint64_t)mine * 4;
  }
  void allgather_bytes(std::vector<void*>& bufs, size_t elt, const std::vector<int64_t>& bounds,
                       cudaStream_t st) override {
    NcclApi& api = nccl();
    GG_NCCL(api.GroupStart());
    for (int r = 0; r < c->nranks; ++r) {
      const size_t cnt = (size_t)(bounds[r + 1] - bounds[r]) * elt;
      char* p = (char*)bufs[0] + (size_t)bounds[r] * elt;
      if (cnt) GG_NCCL(api.Broadcast(p, p, cnt, ncclUint8, r, c->comm, st));
    }
    GG_NCCL(api.GroupEnd());
    bytes += (uint64_t)(bounds.back() - bounds[0] - (bounds[c->rank + 1] - bounds[c->rank])) * elt;
  }
};

int64_t bfs_dist_run(gg_comm* c, const Graph& g, int64_t source, double theta, int32_t* parents_out, Runtime& rt) {
  NcclBfsExchange ex(c);
  return bfs_rank(g, c->nranks, c->rank, ex, source, theta, parents_out, rt);
}

int64_t pagerank_dist_blocked(gg_comm* c, const Graph& g, const gg_schedule& s, bool fp32, int64_t max_iters,
                              double tol, double damping, double* ranks_out, Runtime& rt) {
  NcclExchange ex(c);
  int64_t local = 0;
  if (fp32)
    pagerank_blocked_rank<float>(g, s, c->nranks, c->rank, ex, max_iters, tol, damping, ranks_out, rt, &local);
  else
    pagerank_blocked_rank<double>(g, s, c->nranks, c->rank, ex, max_iters, tol, damping, ranks_out, rt, &local);
  return local;
}
int64_t pagerank_dist_run(gg_comm* c, const Graph& g, int64_t max_iters, double tol, double damping,
                          double* ranks_out, Runtime& rt);
}

int64_t gg::pagerank_dist_run(gg_comm* c, const Graph& g, int64_t max_iters, double tol,
                              double damping, double* ranks_out, Runtime& rt) {
  typedef float CT;
  const ncclDataType_t kCT = ncclFloat32;
  const int64_t V = g.V;
  const int dev = g.dev;
  cudaStream_t st = rt.stream;
  const int P = c->nranks, me = c->rank;
  CsrView in = g.in_view();
  CsrView out = g.out_view();
  DevBuf<int64_t> dbounds(P + 1);
  k_partition<<<1, 64, 0, st>>>(in.off, V, P, dbounds.p);
  GG_LAUNCH_CHECK();
  std::vector<int64_t> bounds(P + 1);
  GG_CUDA(cudaMemcpyAsync(bounds.data(), dbounds.p, (P + 1) * 8, cudaMemcpyDeviceToHost, st));
  GG_CUDA(cudaStreamSynchronize(st));
  const int64_t lo = bounds[me], hi = bounds[me + 1];
  std::shared_ptr<PullPlan> plan_hold = pull_plan_for(g, kPieceEdges, lo, hi);
  PullPlan* plan = plan_hold.get();
  const int64_t iters_cap = max_iters > 0 ? max_iters : 0;
  DevBuf<double> rank(V), scal(2 * (iters_cap + 2)), hubsum(V);
  DevBuf<CT> contrib0(V), contrib1(V);
  DevBuf<int32_t> outdeg(V);
  scal.zero(st);
  hubsum.zero(st);
  k_outdeg<<<grid_for(V, 256, dev), 256, 0, st>>>(out.off, V, outdeg.p);
  // initial rank/contrib/dangling mass over the whole vertex set (identical
  // on every rank, so no exchange is needed before the first iteration)
  k_pr_init_dist<CT><<<grid_for(V, 256, dev), 256, 0, st>>>(out.off, V, rank.p, contrib0.p, scal.p);
  GG_LAUNCH_CHECK();
  count_launch(2);
  PrPullArgs<CT> a{plan->voff.p, plan->vowner.p, plan->nvrows / 32, in.nbr, contrib0.p, contrib1.p,
                   rank.p, outdeg.p, hubsum.p, plan->hubs.p, plan->nhubs, scal.p, V, damping};
  const unsigned grid = (unsigned)sm_count(dev) * 8;
  const unsigned hgrid = grid_for(plan->nhubs, 256, dev);
  int64_t it = 0;
  double l1 = INFINITY;
  NcclApi& api = nccl();
  while (!(it >= max_iters || l1 < tol)) {
    CT* cur = (it & 1) ? contrib1.p : contrib0.p;
    CT* nxt = (it & 1) ? contrib0.p : contrib1.p;
    a.contrib = cur;
    a.contrib_next = nxt;
    rt.edge_begin();
    k_pr_pull<CT><<<grid, 256, 0, st>>>(a, it);
    if (plan->nhubs) k_pr_pull_hubs<CT><<<hgrid, 256, 0, st>>>(a, it);
    GG_LAUNCH_CHECK();
    count_launch(plan->nhubs ? 2 : 1);
    rt.edge_end();
    // allgather of the owned contrib slices + the two scalars
    GG_NCCL(api.GroupStart());
    for (int r = 0; r < P; ++r) {
      size_t cnt = (size_t)(bounds[r + 1] - bounds[r]);
      if (cnt) GG_NCCL(api.Broadcast(nxt + bounds[r], nxt + bounds[r], cnt, kCT, r, c->comm, st));
    }
    GG_NCCL(api.AllReduce(scal.p + 2 * it + 1, scal.p + 2 * it + 1, 2, ncclFloat64, ncclSum, c->comm, st));
    GG_NCCL(api.GroupEnd());
    rt.stats.dispatch_count += 1;
    rt.stats.direction_log.push_back(GG_PULL);
    ++it;
    if (tol > 0.0) {
      GG_CUDA(cudaMemcpyAsync(&l1, scal.p + 2 * (it - 1) + 1, 8, cudaMemcpyDeviceToHost, st));
      GG_CUDA(cudaStreamSynchronize(st));
    }
  }
  // gather the owned rank slices
  GG_NCCL(api.GroupStart());
  for (int r = 0; r < P; ++r) {
    size_t cnt = (size_t)(bounds[r + 1] - bounds[r]);
    if (cnt) GG_NCCL(api.Broadcast(rank.p + bounds[r], rank.p + bounds[r], cnt, ncclFloat64, r, c->comm, st));
  }
  GG_NCCL(api.GroupEnd());
  rt.stats.rounds += it;
  int64_t in_edges = 0, e_lo = 0, e_hi = 0;
  GG_CUDA(cudaMemcpyAsync(&e_lo, in.off + lo, 8, cudaMemcpyDeviceToHost, st));
  GG_CUDA(cudaMemcpyAsync(&e_hi, in.off + hi, 8, cudaMemcpyDeviceToHost, st));
  GG_CUDA(cudaStreamSynchronize(st));
  in_edges = e_hi - e_lo;
  rt.stats.edges_traversed += it * in_edges;
  GG_CUDA(cudaMemcpyAsync(ranks_out, rank.p, V * 8, cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
  return in_edges;
}
