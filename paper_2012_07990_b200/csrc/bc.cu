// bc.cu — algos.bc (reference algos.py:314-395) on the device.
//
// Per source: forward rounds with the BC functor (CAS depth + sigma add in
// push, owner store in pull; hybrid-capable), recording every round's
// frontier members (frontier.members(), algos.py:369) in one device array;
// then backward rounds over the recorded levels len-2 .. 0, push only, with
// f64 atomic adds into delta[u] (algos.py:378-389); scores accumulate
// delta over v != source and are halved at the end.  sigma is f64 (the
// reference uses exact Python ints; f64 is exact up to 2^53 paths).
#include "apply.cuh"
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

namespace gg {

__global__ void k_bc_init(int32_t* depth, double* sigma, double* delta, int64_t V, int64_t s) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    depth[v] = v == s ? 0 : -1;
    sigma[v] = v == s ? 1.0 : 0.0;
    delta[v] = 0.0;
  }
}

__global__ void k_bc_accumulate(const double* delta, double* score, int64_t V, int64_t s) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    if (v != s) score[v] += delta[v];
}

// bc_run's array-of-structs state (ops.cuh BcState): init and accumulate
__global__ void k_bc_init_aos(BcState* st, int64_t V, int64_t s) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    BcState x{};
    x.sigma = v == s ? 1.0 : 0.0;
    x.delta = 0.0;
    x.depth = v == s ? 0 : -1;
    st[v] = x;
  }
}
__global__ void k_bits_set(const int32_t* ids, int64_t n, uint32_t* bm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ids[i];
    atomicOr(bm + (v >> 5), 1u << (v & 31));
  }
}
__global__ void k_bc_accumulate_aos(const BcState* st, double* score, int64_t V, int64_t s) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    if (v != s) score[v] += st[v].delta;
}

__global__ void k_halve(double* score, int64_t V) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    score[v] *= 0.5;
}

struct DenseMember {
  const uint32_t* bits;
  const uint8_t* bools;
  __device__ __forceinline__ bool operator()(int32_t v) const {
    return bits ? ((bits[v >> 5] >> (v & 31)) & 1u) : (bools[v] != 0);
  }
};

// Append a frontier's members to `order` at `pos`; returns the count.
static int64_t snapshot(Runtime& rt, Frontier* f, int32_t* order, int64_t pos, DevBuf<unsigned long long>& n) {
  cudaStream_t st = rt.stream;
  int64_t cnt = frontier_size(&rt, f);
  if (cnt == 0) return 0;
  if (f->repr == GG_SPARSE) {
    GG_CUDA(cudaMemcpyAsync(order + pos, f->ids.p, cnt * 4, cudaMemcpyDeviceToDevice, st));
    return cnt;
  }
  dense_to_sparse(f, order + pos, n.p, st);
  return cnt;
}

// gg_edgeset_apply(GG_UDF_BC_FORWARD): a forward round (algos.py:353-365);
// state arr0 = int32 depth[V], arr1 = double sigma[V], i0 = level.
std::unique_ptr<Frontier> apply_bc_forward(Runtime* rt, const gg_udf_state& st, bool use_filter,
                                           std::unique_ptr<Frontier>* in, const gg_binding& b,
                                           bool reuse, bool collect) {
  if (!st.arr0 || !st.arr1) fail(GG_ERR_VALUE, "bc forward needs depth and sigma arrays");
  return apply_op(rt, OpBcFwd{(int32_t*)st.arr0, (double*)st.arr1, (int32_t)st.i0}, use_filter, in,
                  b, reuse, collect);
}

// gg_edgeset_apply(GG_UDF_BC_BACKWARD): a backward round (algos.py:378-382),
// push only; state arr0 = depth, arr1 = sigma, arr2 = double delta[V].
std::unique_ptr<Frontier> apply_bc_backward(Runtime* rt, const gg_udf_state& st, bool use_filter,
                                            std::unique_ptr<Frontier>* in, const gg_binding& b,
                                            bool reuse, bool collect) {
  if (!st.arr0 || !st.arr1 || !st.arr2) fail(GG_ERR_VALUE, "bc backward needs depth, sigma and delta");
  return apply_op(rt, OpBcBwd{(const int32_t*)st.arr0, (const double*)st.arr1, (double*)st.arr2},
                  use_filter, in, b, reuse, collect);
}

void bc_run(const Graph& g, const int64_t* sources, int64_t nsrc, const gg_binding& b, Runtime& rt,
            double* scores_out) {
  if (nsrc <= 0) fail(GG_ERR_VALUE, "sources must be a non-empty list");
  for (int64_t i = 0; i < nsrc; ++i)
    if (sources[i] < 0 || sources[i] >= g.V)
      fail(GG_ERR_VALUE, strf("invalid source %lld for graph with %lld vertices",
                              (long long)sources[i], (long long)g.V));
  if (!g.symmetric) fail(GG_ERR_VALUE, "bc assumes a symmetric graph; load with symmetrize");
  check_binding(b);
  DeviceGuard guard(g.dev);
  const int64_t V = g.V;
  const int dev = g.dev;
  cudaStream_t st = rt.stream;
  gg_binding bwd{};
  bwd.is_hybrid = 0;
  bwd.s1 = b.s1;  // (bound.s1 if hybrid else bound).copy(), direction PUSH
  bwd.s1.direction = GG_PUSH;
  bwd.s2 = bwd.s1;
  DevBuf<BcState> state(std::max<int64_t>(V, 1));  // depth, sigma, delta per vertex: one sector
  const int64_t W = (V + 31) / 32;
  DevBuf<uint32_t> vis(std::max<int64_t>(W, 1)), nxt(std::max<int64_t>(W, 1));  // level bitmaps
  DevBuf<int32_t> order(V + 1);
  DevBuf<double> score(V);
  DevBuf<unsigned long long> nsel(1);
  score.zero(st);
  for (int64_t si = 0; si < nsrc; ++si) {
    const int64_t s = sources[si];
    k_bc_init_aos<<<grid_for(V, 256, dev), 256, 0, st>>>(state.p, V, s);
    GG_CUDA(cudaMemsetAsync(vis.p, 0, std::max<int64_t>(W, 1) * 4, st));
    GG_LAUNCH_CHECK();
    count_launch();
    int32_t s32 = (int32_t)s;
    std::unique_ptr<Frontier> frontier = rt.new_frontier(&s32, 1);
    std::vector<int64_t> level_start{0};
    int32_t level = 0;
    int64_t pos = 0;
    while (frontier_size(&rt, frontier.get()) > 0) {
      const int64_t lo = pos;
      pos += snapshot(rt, frontier.get(), order.p, pos, nsel);
      level_start.push_back(pos);
      if (pos > lo) {  // this level joins the visited bitmap before its arcs are walked
        k_bits_set<<<grid_for(pos - lo, 256, dev), 256, 0, st>>>(order.p + lo, pos - lo, vis.p);
        GG_LAUNCH_CHECK();
        count_launch();
      }
      OpBcFwdAoS op{state.p, level, vis.p};
      rt.edge_begin();
      std::unique_ptr<Frontier> out = apply_op(&rt, op, true, &frontier, b, true, true);
      rt.edge_end();
      frontier = std::move(out);
      level += 1;
      rt.stats.rounds += 1;
    }
    rt.release(std::move(frontier));
    const int64_t nrounds = (int64_t)level_start.size() - 1;
    OpBcBwdAoS bop{state.p, nxt.p};
    for (int64_t r = nrounds - 2; r >= 0; --r) {
      const int64_t lo = level_start[r], cnt = level_start[r + 1] - lo;
      {  // bitmap of level r + 1
        const int64_t l1 = level_start[r + 1], n1 = level_start[r + 2] - l1;
        GG_CUDA(cudaMemsetAsync(nxt.p, 0, std::max<int64_t>(W, 1) * 4, st));
        if (n1 > 0) k_bits_set<<<grid_for(n1, 256, dev), 256, 0, st>>>(order.p + l1, n1, nxt.p);
        GG_LAUNCH_CHECK();
        count_launch();
      }
      std::unique_ptr<Frontier> wave = rt.acquire(GG_SPARSE);  // new_frontier(n, rounds[r])
      GG_CUDA(cudaMemcpyAsync(wave->ids.p, order.p + lo, cnt * 4, cudaMemcpyDeviceToDevice, st));
      unsigned long long c = (unsigned long long)cnt;
      GG_CUDA(cudaMemcpyAsync(wave->count.p, &c, 8, cudaMemcpyHostToDevice, st));
      wave->size_cache = cnt;
      rt.edge_begin();
      apply_op(&rt, bop, false, &wave, bwd, true, false);
      rt.edge_end();
      rt.stats.rounds += 1;
    }
    k_bc_accumulate_aos<<<grid_for(V, 256, dev), 256, 0, st>>>(state.p, score.p, V, s);
    GG_LAUNCH_CHECK();
    count_launch();
  }
  k_halve<<<grid_for(V, 256, dev), 256, 0, st>>>(score.p, V);
  GG_LAUNCH_CHECK();
  count_launch();
  GG_CUDA(cudaMemcpyAsync(scores_out, score.p, V * sizeof(double), cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gg
