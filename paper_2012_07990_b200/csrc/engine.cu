// engine.cu — edgeset.apply dispatcher, device frontiers and per-query runtime.
//
// Reference anchors (all in /root/reference/pkg/src/schedge/):
//   edgeset_apply                  engine.py:418-460
//   _apply_push/_apply_pull/_apply_edge_only   engine.py:463-608
//   _OutputBuilder                 engine.py:279-397
//   _sparse_view/_dense_view       engine.py:404-415
//   hybrid_apply                   engine.py:622-636 (strictly greater)
//   FrontierPool                   runtime.py:124-157
//   VertexSubset.convert/members   frontier.py:186-265
#include "apply.cuh"
#include <cstdio>
#include <map>
#include <mutex>
#include <cub/device/device_select.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

namespace gg {

// ---------------------------------------------------------------------------
// Frontier storage and conversions
// ---------------------------------------------------------------------------
std::unique_ptr<Frontier> frontier_alloc(int dev, int64_t universe, int repr, int64_t sparse_cap) {
  auto f = std::make_unique<Frontier>();
  f->dev = dev;
  f->universe = universe;
  f->repr = repr;
  f->count.alloc(1);
  f->count.zero();
  if (repr == GG_SPARSE) {
    f->ids.alloc(sparse_cap > 0 ? sparse_cap : 1);
  } else if (repr == GG_BITMAP) {
    f->bits.alloc((universe + 31) / 32 + 1);
    f->bits.zero();
  } else {
    f->bools.alloc(((universe + 3) & ~int64_t(3)) + 4);
    f->bools.zero();
  }
  f->size_cache = 0;
  return f;
}

void frontier_clear(Frontier* f, cudaStream_t s) {
  GG_CUDA(cudaMemsetAsync(f->count.p, 0, sizeof(unsigned long long), s));
  if (f->repr == GG_BITMAP) f->bits.zero(s);
  if (f->repr == GG_BOOLMAP) f->bools.zero(s);
  f->size_cache = 0;
}

__global__ void k_popcount_bits(const uint32_t* w, int64_t nwords, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nwords;
       i += (int64_t)gridDim.x * blockDim.x)
    c += __popc(w[i]);
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}
__global__ void k_popcount_bytes(const uint8_t* b, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += b[i] != 0;
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

// dense size into f->count (the unfused "separate materialisation pass")
void dense_size_on_device(Frontier* f, cudaStream_t s) {
  GG_CUDA(cudaMemsetAsync(f->count.p, 0, sizeof(unsigned long long), s));
  if (f->repr == GG_BITMAP) {
    int64_t nw = (f->universe + 31) / 32;
    k_popcount_bits<<<grid_for(nw, 256, f->dev), 256, 0, s>>>(f->bits.p, nw, f->count.p);
  } else {
    k_popcount_bytes<<<grid_for(f->universe, 256, f->dev), 256, 0, s>>>(f->bools.p, f->universe,
                                                                         f->count.p);
  }
  GG_LAUNCH_CHECK();
  count_launch();
  f->size_cache = -1;
}

// the per-round frontier-size read-backs (hybrid direction choice, loop
// end) go through a pinned per-thread word: a copy into pageable memory is
// staged by the driver and costs several microseconds more per round
static unsigned long long* pinned_word() {
  static thread_local unsigned long long* w = nullptr;
  if (!w) GG_CUDA(cudaMallocHost(&w, sizeof(unsigned long long)));
  return w;
}

int64_t frontier_size_raw(Frontier* f, cudaStream_t s) {
  if (f->size_cache >= 0) return f->size_cache;
  unsigned long long* h = pinned_word();
  GG_CUDA(cudaMemcpyAsync(h, f->count.p, sizeof(*h), cudaMemcpyDeviceToHost, s));
  GG_CUDA(cudaStreamSynchronize(s));
  f->size_cache = (int64_t)*h;
  return f->size_cache;
}

int64_t frontier_size(Runtime* rt, Frontier* f) { return frontier_size_raw(f, rt->stream); }

struct MemberPred {
  const uint32_t* bits;
  const uint8_t* bools;
  __device__ __forceinline__ bool operator()(int32_t v) const {
    return bits ? ((bits[v >> 5] >> (v & 31)) & 1u) : (bools[v] != 0);
  }
};

__global__ void k_sparse_to_bits(const int32_t* ids, const unsigned long long* n, uint32_t* bits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = ids[i];
    atomicOr(bits + (v >> 5), 1u << (v & 31));
  }
}
__global__ void k_sparse_to_bytes(const int32_t* ids, const unsigned long long* n, uint8_t* b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[ids[i]] = 1;
}
__global__ void k_bits_to_bytes(const uint32_t* bits, int64_t V, uint8_t* b) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    b[v] = (bits[v >> 5] >> (v & 31)) & 1u;
}
__global__ void k_bytes_to_bits(const uint8_t* b, int64_t V, uint32_t* bits) {
  // one warp builds one word: ballot over 32 consecutive bytes
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); base < V;
       base += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = base + lane_id();
    unsigned m = __ballot_sync(0xffffffffu, v < V && b[v] != 0);
    if (lane_id() == 0) bits[base >> 5] = m;
  }
}

// Dense -> SPARSE in ascending id order (frontier.py:186-201) in two passes
// over 32-vertex masks: per-block member counts, then each block sums the
// counts before it, scans its threads' counts and writes its members.  Each
// thread owns 4 consecutive masks (128 vertices); a block covers 32768.
// (Replaces a cub::DeviceSelect over a V-long counting iterator: ~60 us at
// V = 2^24 for what is a 2 MB bitmap.)
constexpr int kD2sWords = 4;
constexpr int64_t kD2sPerBlock = 256 * kD2sWords * 32;
__device__ __forceinline__ uint32_t dense_mask(const uint32_t* bits, const uint8_t* bools, int64_t V,
                                               int64_t w) {
  const int64_t v0 = w * 32;
  if (v0 >= V) return 0u;
  uint32_t m = 0;
  if (bits) {
    m = bits[w];
  } else if (v0 + 32 <= V) {
    const uint4* q = reinterpret_cast<const uint4*>(bools + v0);  // bools are 4-byte padded; v0 % 32 == 0
    const uint4 x = q[0], y = q[1];
    const uint32_t words[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if ((words[k] >> (8 * b)) & 0xffu) m |= 1u << (4 * k + b);
  } else {
    for (int64_t v = v0; v < V; ++v)
      if (bools[v]) m |= 1u << (v - v0);
  }
  const int64_t tail = V - v0;
  return tail >= 32 ? m : (m & ((1u << tail) - 1u));
}
__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long x, unsigned long long* s_w) {
  x = warp_sum(x);
  if (lane_id() == 0) s_w[threadIdx.x >> 5] = x;
  __syncthreads();
  unsigned long long t = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += s_w[k];
  __syncthreads();
  return t;
}
__global__ void __launch_bounds__(256) k_d2s_count(const uint32_t* bits, const uint8_t* bools, int64_t V,
                                                   unsigned long long* block_counts) {
  __shared__ unsigned long long s_w[8];
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kD2sWords;
  unsigned long long c = 0;
#pragma unroll
  for (int k = 0; k < kD2sWords; ++k) c += __popc(dense_mask(bits, bools, V, w0 + k));
  c = block_sum_u64(c, s_w);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = c;
}
__global__ void __launch_bounds__(256) k_d2s_write(const uint32_t* bits, const uint8_t* bools, int64_t V,
                                                   const unsigned long long* block_counts, int32_t* out,
                                                   unsigned long long* count) {
  __shared__ unsigned long long s_w[8];
  __shared__ unsigned long long s_scan[8];
  // members of the blocks before this one
  unsigned long long before = 0;
  for (int64_t b = threadIdx.x; b < blockIdx.x; b += blockDim.x) before += block_counts[b];
  before = block_sum_u64(before, s_w);
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kD2sWords;
  uint32_t m[kD2sWords];
  unsigned c = 0;
#pragma unroll
  for (int k = 0; k < kD2sWords; ++k) {
    m[k] = dense_mask(bits, bools, V, w0 + k);
    c += __popc(m[k]);
  }
  // block exclusive scan of c
  const int lane = lane_id(), wid = threadIdx.x >> 5;
  unsigned x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_scan[wid] = x;
  __syncthreads();
  unsigned long long pos = before + (x - c);
  for (int k = 0; k < wid; ++k) pos += s_scan[k];
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) *count = pos + c;
#pragma unroll
  for (int k = 0; k < kD2sWords; ++k) {
    uint32_t r = m[k];
    const int32_t base = (int32_t)((w0 + k) * 32);
    while (r) {
      const int b = __ffs(r) - 1;
      out[pos++] = base + b;
      r &= r - 1;
    }
  }
}

void dense_to_sparse(const Frontier* src, int32_t* out, unsigned long long* count, cudaStream_t s) {
  const int64_t V = src->universe;
  const int64_t nb = std::max<int64_t>(1, (V + kD2sPerBlock - 1) / kD2sPerBlock);
  DevBuf<unsigned long long> bc(nb);
  const uint32_t* bits = src->repr == GG_BITMAP ? src->bits.p : nullptr;
  const uint8_t* bools = src->repr == GG_BOOLMAP ? src->bools.p : nullptr;
  k_d2s_count<<<(unsigned)nb, 256, 0, s>>>(bits, bools, V, bc.p);
  GG_LAUNCH_CHECK();
  k_d2s_write<<<(unsigned)nb, 256, 0, s>>>(bits, bools, V, bc.p, out, count);
  GG_LAUNCH_CHECK();
  count_launch(2);
}

void frontier_convert_into(Runtime* rt, Frontier* src, Frontier* dst) {
  cudaStream_t s = rt->stream;
  const int dev = rt->dev;
  frontier_clear(dst, s);
  const int64_t V = src->universe;
  if (src->repr == dst->repr) {
    if (src->repr == GG_SPARSE) {
      int64_t n = frontier_size_raw(src, s);
      if (n) GG_CUDA(cudaMemcpyAsync(dst->ids.p, src->ids.p, n * 4, cudaMemcpyDeviceToDevice, s));
    } else if (src->repr == GG_BITMAP) {
      GG_CUDA(cudaMemcpyAsync(dst->bits.p, src->bits.p, src->bits.bytes(), cudaMemcpyDeviceToDevice, s));
    } else {
      GG_CUDA(cudaMemcpyAsync(dst->bools.p, src->bools.p, src->bools.bytes(), cudaMemcpyDeviceToDevice, s));
    }
    GG_CUDA(cudaMemcpyAsync(dst->count.p, src->count.p, 8, cudaMemcpyDeviceToDevice, s));
    dst->size_cache = src->size_cache;
    return;
  }
  if (dst->repr == GG_SPARSE) {
    // dense -> SPARSE in ascending id order (frontier.py:186-201)
    dense_to_sparse(src, dst->ids.p, dst->count.p, s);
    dst->size_cache = -1;
    return;
  }
  if (src->repr == GG_SPARSE) {
    // sparse -> dense deduplicates by construction
    if (dst->repr == GG_BITMAP)
      k_sparse_to_bits<<<grid_for(V, 256, dev), 256, 0, s>>>(src->ids.p, src->count.p, dst->bits.p);
    else
      k_sparse_to_bytes<<<grid_for(V, 256, dev), 256, 0, s>>>(src->ids.p, src->count.p, dst->bools.p);
  } else if (dst->repr == GG_BOOLMAP) {
    k_bits_to_bytes<<<grid_for(V, 256, dev), 256, 0, s>>>(src->bits.p, V, dst->bools.p);
  } else {
    k_bytes_to_bits<<<grid_for(V, 256, dev), 256, 0, s>>>(src->bools.p, V, dst->bits.p);
  }
  GG_LAUNCH_CHECK();
  count_launch();
  dense_size_on_device(dst, s);
}

void frontier_members(Frontier* f, int32_t* out, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  if (f->repr == GG_SPARSE) {
    GG_CUDA(cudaMemcpyAsync(out, f->ids.p, n * 4, cudaMemcpyDefault, s));
    GG_CUDA(cudaStreamSynchronize(s));
    return;
  }
  Frontier tmp;
  tmp.dev = f->dev;
  tmp.universe = f->universe;
  tmp.repr = GG_SPARSE;
  tmp.ids.alloc(f->universe);
  tmp.count.alloc(1);
  dense_to_sparse(f, tmp.ids.p, tmp.count.p, s);
  GG_CUDA(cudaMemcpyAsync(out, tmp.ids.p, n * 4, cudaMemcpyDefault, s));
  GG_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// Runtime
// ---------------------------------------------------------------------------
Runtime::Runtime(const Graph* graph, const gg_exec* c) : g(graph), dev(graph->dev) {
  if (c) cfg = *c;
  if (cfg.num_workers < 1) fail(GG_ERR_ENGINE, "num_workers must be >= 1");
  if (cfg.warp_size < 1 || cfg.cta_size < 1) fail(GG_ERR_ENGINE, "warp_size and cta_size must be >= 1");
  if (cfg.cta_size % cfg.warp_size) fail(GG_ERR_ENGINE, "warp_size must divide cta_size");
  scanned.alloc(1);
  scanned.zero();
}

Runtime::~Runtime() {
  for (auto& p : edge_events) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  if (edge_open) cudaEventDestroy(edge_open);
  for (auto& p : top_events) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
}

void Runtime::edge_begin() {
  GG_CUDA(cudaEventCreate(&edge_open));
  GG_CUDA(cudaEventRecord(edge_open, stream));
}

void Runtime::edge_end() {
  cudaEvent_t e;
  GG_CUDA(cudaEventCreate(&e));
  GG_CUDA(cudaEventRecord(e, stream));
  edge_events.emplace_back(edge_open, e);
  edge_open = nullptr;
}

double Runtime::edge_ms(int64_t* launches) {
  double total = 0;
  for (auto& p : edge_events) {
    GG_CUDA(cudaEventSynchronize(p.second));
    float ms = 0;
    GG_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
    total += ms;
  }
  if (launches) *launches = (int64_t)edge_events.size();
  return total;
}

double Runtime::top_ms(int64_t* launches) {
  double total = 0;
  for (auto& p : top_events) {
    GG_CUDA(cudaEventSynchronize(p.second));
    float ms = 0;
    GG_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
    total += ms;
  }
  if (launches) *launches = (int64_t)top_events.size();
  return total;
}

int64_t Runtime::edges_traversed() {
  unsigned long long h = 0;
  GG_CUDA(cudaMemcpyAsync(&h, scanned.p, sizeof(h), cudaMemcpyDeviceToHost, stream));
  GG_CUDA(cudaStreamSynchronize(stream));
  return stats.edges_traversed + (int64_t)h;
}

static int64_t sparse_capacity(const Graph* g) {
  // A SPARSE frontier with dedup off may hold one entry per scanned arc.
  return std::max<int64_t>(g->V, g->E) + 1;
}

std::unique_ptr<Frontier> Runtime::acquire(int repr) {
  if (spare[repr]) {
    auto f = std::move(spare[repr]);
    f->retired = false;
    return f;
  }
  stats.frontier_allocations += 1;
  return frontier_alloc(dev, g->V, repr, repr == GG_SPARSE ? sparse_capacity(g) : 0);
}

void Runtime::release(std::unique_ptr<Frontier> f) {
  if (!f) return;
  frontier_clear(f.get(), stream);
  f->retired = true;
  if (!spare[f->repr]) spare[f->repr] = std::move(f);
}

__global__ void k_check_ids(const int32_t* ids, int64_t n, int64_t V, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (ids[i] < 0 || ids[i] >= V) *bad = 1;
}

std::unique_ptr<Frontier> Runtime::new_frontier(const int32_t* ids, int64_t n) {
  auto f = acquire(GG_SPARSE);
  // a user multiset may be longer than max(V, E) + 1 (frontier.py accepts any)
  if (n > (int64_t)f->ids.n) f->ids.alloc(n);
  cudaPointerAttributes at{};
  bool host = true;
  if (cudaPointerGetAttributes(&at, ids) == cudaSuccess) host = at.type == cudaMemoryTypeUnregistered || at.type == cudaMemoryTypeHost;
  else cudaGetLastError();
  if (host && n <= 4096) {
    // small host list (a BFS / BC source): check on the host, no round trip;
    // pageable copies are staged before cudaMemcpyAsync returns
    for (int64_t i = 0; i < n; ++i)
      if (ids[i] < 0 || ids[i] >= g->V) fail(GG_ERR_ENGINE, "vertex id out of range");
    if (n) GG_CUDA(cudaMemcpyAsync(f->ids.p, ids, n * 4, cudaMemcpyHostToDevice, stream));
    unsigned long long hn = (unsigned long long)n;
    GG_CUDA(cudaMemcpyAsync(f->count.p, &hn, 8, cudaMemcpyHostToDevice, stream));
    f->size_cache = n;
    return f;
  }
  if (n) {
    GG_CUDA(cudaMemcpyAsync(f->ids.p, ids, n * 4, cudaMemcpyDefault, stream));
    DevBuf<int> bad(1);
    bad.zero(stream);
    k_check_ids<<<grid_for(n, 256, dev), 256, 0, stream>>>(f->ids.p, n, g->V, bad.p);
    GG_LAUNCH_CHECK();
    int hb = 0;
    GG_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, stream));
    GG_CUDA(cudaStreamSynchronize(stream));
    if (hb) fail(GG_ERR_ENGINE, "vertex id out of range");
  }
  unsigned long long hn = (unsigned long long)n;
  GG_CUDA(cudaMemcpyAsync(f->count.p, &hn, 8, cudaMemcpyHostToDevice, stream));
  GG_CUDA(cudaStreamSynchronize(stream));
  f->size_cache = n;
  return f;
}

// ---------------------------------------------------------------------------
// Schedule validation (sched.py:123-153)
// ---------------------------------------------------------------------------
void check_schedule(const gg_schedule& s) {
  std::string p;
  auto add = [&](const char* m) { p += p.empty() ? m : (std::string("; ") + m); };
  if (s.direction != GG_PUSH && s.direction != GG_PULL) add("unknown direction");
  if (s.pull_repr != GG_BOOLMAP && s.pull_repr != GG_BITMAP) add("unknown pull frontier representation");
  if (s.load_balance < 0 || s.load_balance > 6) add("unknown load balance");
  if (s.frontier_creation < 0 || s.frontier_creation > 2) add("unknown frontier creation");
  if (s.dedup_strategy < 0 || s.dedup_strategy > 2) add("unknown dedup strategy");
  if (s.blocking && s.load_balance != GG_LB_EDGE_ONLY) add("blocking requires EDGE_ONLY load balancing");
  if (s.blocking_size < 0) add("blocking_size must be >= 1");
  if (s.delta < 1) add("delta must be >= 1");
  if (!p.empty()) fail(GG_ERR_SCHEDULE, "invalid schedule: " + p);
}

void check_binding(const gg_binding& b) {
  check_schedule(b.s1);
  if (b.is_hybrid) {
    check_schedule(b.s2);
    if (!(b.threshold > 0.0 && b.threshold < 1.0)) fail(GG_ERR_SCHEDULE, "threshold must lie in (0, 1)");
  }
}

// ---------------------------------------------------------------------------
// Dispatch
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Caching device allocator (see common.cuh)
// ---------------------------------------------------------------------------
namespace {
struct DevicePool {
  std::mutex mu;
  std::map<std::pair<int, size_t>, std::vector<void*>> free_blocks;
  size_t cached = 0;                  // all devices (gg_pool_stats)
  std::map<int, size_t> dev_cached;   // per device: compared against that device's cap
  int64_t mallocs = 0, frees = 0;
};
DevicePool& pool() {
  static DevicePool* p = new DevicePool;  // never destroyed: frees at exit are unordered
  return *p;
}
size_t size_class(size_t bytes) {
  if (bytes <= (1u << 20)) {
    size_t c = 256;
    while (c < bytes) c <<= 1;
    return c;
  }
  const size_t g = 2u << 20;
  return (bytes + g - 1) / g * g;
}
// Cache at most this many bytes (beyond it, frees go to the driver):
// GG_POOL_MAX_GB, read on every free so a process can lower it between
// queries, else 60% of the device's HBM.  The cap must hold a whole query's
// working set: RMAT-27 PageRank end to end (COO, CSR, sort buffers, layout)
// frees ~74 GB per call, and at a 48 GB cap every call paid 16 cudaMalloc +
// 16 synchronising cudaFree (0.63-1.19 s per call instead of 0.61 s).
// (per device: each device's cache is held against its own HBM size)
size_t pool_limit(int dev) {
  const char* e = getenv("GG_POOL_MAX_GB");
  if (e) {
    const double gb = atof(e);
    return gb > 0 ? (size_t)(gb * (double)(size_t(1) << 30)) : 0;
  }
  static std::mutex mu;
  static std::map<int, size_t> dflt;
  std::lock_guard<std::mutex> lk(mu);
  auto it = dflt.find(dev);
  if (it != dflt.end()) return it->second;
  size_t total = size_t(80) << 30;
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess) total = prop.totalGlobalMem;  // once per device
  else cudaGetLastError();
  return dflt[dev] = (size_t)(0.6 * (double)total);
}
}  // namespace

void pool_trim() {
  DevicePool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : P.free_blocks) {
    cudaSetDevice(kv.first.first);
    for (void* q : kv.second) cudaFree(q);
    P.frees += (int64_t)kv.second.size();
  }
  cudaSetDevice(cur);
  P.free_blocks.clear();
  P.cached = 0;
  P.dev_cached.clear();
}

void pool_counters(int64_t* mallocs, int64_t* frees, int64_t* cached) {
  DevicePool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  *mallocs = P.mallocs;
  *frees = P.frees;
  *cached = (int64_t)P.cached;
}

void* pool_alloc(size_t bytes, size_t* granted) {
  const size_t c = size_class(bytes);
  int dev = 0;
  GG_CUDA(cudaGetDevice(&dev));
  DevicePool& P = pool();
  {
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.free_blocks.find({dev, c});
    if (it != P.free_blocks.end() && !it->second.empty()) {
      void* q = it->second.back();
      it->second.pop_back();
      P.cached -= c;
      P.dev_cached[dev] -= c;
      *granted = c;
      return q;
    }
  }
  void* q = nullptr;
  static const bool trace = getenv("GG_POOL_TRACE") != nullptr;
  double t0 = trace ? now_ms() : 0.0;
  cudaError_t e = cudaMalloc(&q, c);
  if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and retry once
    cudaGetLastError();
    if (trace) fprintf(stderr, "gg pool: out of memory at %zu bytes, trimming\n", c);
    pool_trim();
    e = cudaMalloc(&q, c);
  }
  if (trace) fprintf(stderr, "gg pool: cudaMalloc %zu bytes %.2f ms\n", c, now_ms() - t0);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(P.mu);
    P.mallocs += 1;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(GG_ERR_CUDA, strf("cudaMalloc(%zu) failed: %s", c, cudaGetErrorString(e)));
  }
  *granted = c;
  return q;
}

void pool_free(void* q, size_t granted) {
  if (!q) return;
  int dev = 0;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, q) == cudaSuccess) dev = at.device;
  else if (cudaGetDevice(&dev) != cudaSuccess) return;
  DevicePool& P = pool();
  std::vector<std::pair<int, void*>> evict;
  {
    std::lock_guard<std::mutex> lk(P.mu);
    const size_t lim = pool_limit(dev);
    size_t& dc = P.dev_cached[dev];
    if (granted > lim) {
      evict.push_back({dev, q});
    } else {
      // Make room by returning the largest cached blocks of OTHER size
      // classes: one-off temporaries (graph build sort buffers) go, while a
      // block that is freed and re-requested every call stays cached
      // (otherwise every call pays a synchronising cudaFree + cudaMalloc).
      for (auto it = P.free_blocks.rbegin(); dc + granted > lim && it != P.free_blocks.rend(); ++it) {
        if (it->first.first != dev || it->first.second == granted) continue;  // this device, other sizes
        while (!it->second.empty() && dc + granted > lim) {
          evict.push_back({it->first.first, it->second.back()});
          it->second.pop_back();
          P.cached -= it->first.second;
          dc -= it->first.second;
        }
      }
      if (dc + granted <= lim) {
        P.free_blocks[{dev, granted}].push_back(q);
        P.cached += granted;
        dc += granted;
      } else {
        evict.push_back({dev, q});
      }
    }
    P.frees += (int64_t)evict.size();
  }
  if (evict.empty()) return;
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& e : evict) {
    cudaSetDevice(e.first);
    cudaFree(e.second);
  }
  cudaSetDevice(cur);
}

void etwc_huge(Runtime* rt, EtwcEntry** q, unsigned long long** n, int64_t small_frontier,
               int64_t entries) {
  rt->g->ensure_out();
  // no hub and a frontier that fills the grid: no grid pass (no extra barriers)
  if (rt->g->max_out_degree < kEtwcHuge && (small_frontier == 0 || rt->g->max_out_degree < kWarp)) {
    *q = nullptr;
    *n = nullptr;
    return;
  }
  // one entry per active-list entry at most (a multiset frontier -- dedup
  // off -- repeats a hub once per occurrence), per kEtwcHuge arcs otherwise;
  // a small frontier queues each vertex's CTA- and warp-stage ranges (two)
  const int64_t cap = std::max({rt->g->E / kEtwcHuge, 2 * small_frontier, 2 * entries}) + 1;
  if (rt->etwc_q.n < (size_t)cap) rt->etwc_q.alloc(cap);
  if (!rt->etwc_n.p) rt->etwc_n.alloc(1);
  GG_CUDA(cudaMemsetAsync(rt->etwc_n.p, 0, sizeof(unsigned long long), rt->stream));
  *q = rt->etwc_q.p;
  *n = rt->etwc_n.p;
}

int max_coop_blocks(const void* fn, int block, int dev, size_t smem, int cap_per_sm) {
  int per_sm = 0;
  GG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem));
  if (per_sm < 1) fail(GG_ERR_CUDA, "kernel cannot be co-resident");
  // a grid barrier costs ~1.2 us at 1-2 CTAs/SM and ~2.5 us at 8 (measured,
  // profiles/r01/microbench_gridsync.txt): latency-bound fused loops cap the
  // resident CTAs per SM; GG_COOP_PER_SM overrides every cooperative launch
  if (cap_per_sm >= 1 && cap_per_sm < per_sm) per_sm = cap_per_sm;
  if (const char* e = getenv("GG_COOP_PER_SM")) {
    int cap = atoi(e);
    if (cap >= 1 && cap < per_sm) per_sm = cap;
  }
  return per_sm * sm_count(dev);
}

__global__ void k_degrees_of(const InView in, const int64_t* off, int64_t n, int64_t* deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { deg[i] = 0; continue; }
    int32_t u = active_at(in, i);
    deg[i] = off[u + 1] - off[u];
  }
}

__global__ void k_strict_spans(const int64_t* off, int64_t V, int64_t nspans, int64_t* span) {
  const int64_t total = off[V];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= nspans;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t == nspans) { span[t] = V; continue; }
    // edge target of span t, snapped to the first vertex whose range starts
    // at or after it (bisect_left over offsets, engine.py:216-225)
    int64_t target = (int64_t)((__int128)total * t / nspans);
    int64_t lo = 0, hi = V;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (off[mid] < target) lo = mid + 1; else hi = mid;
    }
    span[t] = t == 0 ? 0 : lo;
  }
}

__global__ void k_clear_marks(const int32_t* ids, const unsigned long long* n, uint32_t* bits,
                              uint8_t* bytes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = ids[i];
    if (bits) atomicAnd(bits + (v >> 5), ~(1u << (v & 31)));
    if (bytes) bytes[v] = 0;
  }
}


__global__ void k_degree_sum(const InView in, const int64_t* off, int64_t n,
                             unsigned long long* sum) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t u = active_at(in, i);
    s += (unsigned long long)(off[u + 1] - off[u]);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(sum, s);
}

int64_t degree_sum(Runtime* rt, const InView& in, int64_t n) {
  DevBuf<unsigned long long> d(1);
  d.zero(rt->stream);
  k_degree_sum<<<grid_for(n, 256, rt->dev), 256, 0, rt->stream>>>(in, rt->g->out_view().off, n, d.p);
  GG_LAUNCH_CHECK();
  count_launch();
  unsigned long long h = 0;
  GG_CUDA(cudaMemcpyAsync(&h, d.p, sizeof(h), cudaMemcpyDeviceToHost, rt->stream));
  GG_CUDA(cudaStreamSynchronize(rt->stream));
  return (int64_t)h;
}

__global__ void k_split_dump(const InView in, const int64_t* off, int64_t n, int lb, int cta,
                             int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = active_at(in, i);
    const int64_t size = off[u + 1] - off[u];
    if (lb == GG_LB_ETWC) {
      const EtwcSizes s = etwc_sizes(size, cta);
      out[3 * i] = s.e0;
      out[3 * i + 1] = s.e1;
      out[3 * i + 2] = s.e2;
    } else {
      out[i] = twc_bin_of(size, cta);
    }
  }
}

void strict_prefix(Runtime* rt, const InView& in, int64_t n);

int64_t partition_dump(Runtime* rt, Frontier* active, int lb, int64_t* out, int64_t cap) {
  if (active->repr != GG_SPARSE) fail(GG_ERR_FRONTIER, "partition dump takes a SPARSE active list");
  rt->g->ensure_out();
  const int64_t n = frontier_size_raw(active, rt->stream);
  const InView in = active->view();
  int64_t len = 0;
  if (lb == GG_LB_STRICT) {
    len = n + 1;
    if (len > cap) fail(GG_ERR_VALUE, "output buffer too small");
    strict_prefix(rt, in, n);
    GG_CUDA(cudaMemcpy(out, rt->prefix.p, len * 8, cudaMemcpyDefault));
    return len;
  }
  if (lb != GG_LB_ETWC && lb != GG_LB_TWC) fail(GG_ERR_VALUE, "partition dump covers ETWC, TWC, STRICT");
  len = lb == GG_LB_ETWC ? 3 * n : n;
  if (len > cap) fail(GG_ERR_VALUE, "output buffer too small");
  if (!n) return 0;
  DevBuf<int64_t> d(len);
  k_split_dump<<<grid_for(n, 256, rt->dev), 256, 0, rt->stream>>>(in, rt->g->out_view().off, n, lb,
                                                                  rt->cfg.cta_size, d.p);
  GG_LAUNCH_CHECK();
  GG_CUDA(cudaMemcpyAsync(out, d.p, len * 8, cudaMemcpyDefault, rt->stream));
  GG_CUDA(cudaStreamSynchronize(rt->stream));
  return len;
}

void strict_prefix(Runtime* rt, const InView& in, int64_t n) {
  cudaStream_t st = rt->stream;
  rt->prefix.alloc(n + 1);
  DevBuf<int64_t> deg(n + 1);
  k_degrees_of<<<grid_for(n + 1, 256, rt->dev), 256, 0, st>>>(in, rt->g->out_view().off, n, deg.p);
  GG_LAUNCH_CHECK();
  size_t temp = 0;
  GG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, deg.p, rt->prefix.p, n + 1, st));
  GG_CUDA(cub::DeviceScan::ExclusiveSum(rt->cub_tmp.get(temp), temp, deg.p, rt->prefix.p, n + 1, st));
  count_launch(2);
  GG_CUDA(cudaStreamSynchronize(st));
}

void strict_spans(Runtime* rt, int64_t nspans) {
  if (rt->spans_n == nspans) return;
  rt->spans.alloc(nspans + 1);
  k_strict_spans<<<grid_for(nspans + 1, 256, rt->dev), 256, 0, rt->stream>>>(
      rt->g->in_view().off, rt->g->V, nspans, rt->spans.p);
  GG_LAUNCH_CHECK();
  count_launch();
  rt->spans_n = nspans;
}

void clear_marks(Runtime* rt, Frontier* out, const OutBuilder& ob) {
  k_clear_marks<<<grid_for(rt->g->V, 256, rt->dev), 256, 0, rt->stream>>>(
      out->ids.p, out->count.p, ob.mark_bits, ob.mark_bytes);
  GG_LAUNCH_CHECK();
  count_launch();
}

Frontier* converted_view(Runtime* rt, Frontier* in, int repr) {
  rt->stats.frontier_conversions += 1;
  if (!rt->conv || rt->conv->repr != repr)
    rt->conv = frontier_alloc(rt->dev, rt->g->V, repr, repr == GG_SPARSE ? sparse_capacity(rt->g) : 0);
  frontier_convert_into(rt, in, rt->conv.get());
  return rt->conv.get();
}

void twc_queues(Runtime* rt, TwcQueues* q, int64_t entries) {
  // every active-list entry lands in one bin: a bin holds up to max(V,
  // entries) ids (entries > V for a multiset SPARSE input, dedup off)
  const int64_t cap = std::max(rt->g->V, entries) + 1;
  if (rt->twc_q.n < (size_t)(3 * cap)) rt->twc_q.alloc(3 * cap);
  if (!rt->twc_cnt.p) rt->twc_cnt.alloc(3);
  GG_CUDA(cudaMemsetAsync(rt->twc_cnt.p, 0, 3 * 8, rt->stream));
  *q = TwcQueues{{rt->twc_q.p, rt->twc_q.p + cap, rt->twc_q.p + 2 * cap}, rt->twc_cnt.p};
}

OutBuilder make_builder(Runtime* rt, const gg_schedule& s, Frontier* out) {
  OutBuilder ob{};
  ob.mode = out ? s.frontier_creation : OUT_NONE;
  ob.dedup = DEDUP_NONE;
  if (!out) return ob;
  ob.queue = out->ids.p;
  ob.qcount = out->count.p;
  ob.bits = out->bits.p;
  ob.bools = out->bools.p;
  const int64_t V = rt->g->V;
  if (s.dedup) {
    if (s.dedup_strategy == GG_DEDUP_MONOTONIC_COUNTERS) {
      if (!rt->stamps.p) {
        rt->stamps.alloc(V + 1);
        GG_CUDA(cudaMemsetAsync(rt->stamps.p, 0xff, rt->stamps.bytes(), rt->stream));
      }
      rt->round += 1;  // counters.next_round()
      ob.dedup = DEDUP_COUNTERS;
      ob.stamps = rt->stamps.p;
      ob.round = rt->round;
    } else if (s.frontier_creation == GG_CREATE_FUSED) {
      if (s.dedup_strategy == GG_DEDUP_BITMAP) {
        if (!rt->mark_bits.p) { rt->mark_bits.alloc((V + 31) / 32 + 1); rt->mark_bits.zero(rt->stream); }
        ob.dedup = DEDUP_MARK_BITS;
        ob.mark_bits = rt->mark_bits.p;
      } else {
        if (!rt->mark_bytes.p) { rt->mark_bytes.alloc(((V + 3) & ~int64_t(3)) + 4); rt->mark_bytes.zero(rt->stream); }
        ob.dedup = DEDUP_MARK_BYTES;
        ob.mark_bytes = rt->mark_bytes.p;
      }
    } else {
      ob.dedup = DEDUP_SLOT;
    }
  }
  return ob;
}


std::unique_ptr<Frontier> edgeset_apply(Runtime* rt, int udf, const gg_udf_state& st, bool use_filter,
                                        std::unique_ptr<Frontier>* input, const gg_binding& b,
                                        bool reuse, bool collect_output) {
  DeviceGuard guard(rt->dev);
  switch (udf) {
    case UDF_BFS:
      return apply_op(rt, OpBfs{(int32_t*)st.arr0}, use_filter, input, b, reuse, collect_output);
    case UDF_COUNT:
      return apply_op(rt, OpCount{(unsigned long long*)st.arr0}, use_filter, input, b, reuse,
                      collect_output);
    case UDF_ENQUEUE:
      return apply_op(rt, OpEnqueue{}, use_filter, input, b, reuse, collect_output);
    case UDF_PR:
      return apply_op(rt, OpPr<double>{(double*)st.arr0, (const double*)st.arr1}, use_filter, input,
                      b, reuse, collect_output);
    case UDF_PR32:
      return apply_op(rt, OpPr<float>{(double*)st.arr0, (const float*)st.arr1}, use_filter, input, b,
                      reuse, collect_output);
    case UDF_CC_HOOK:
      return apply_cc_hook(rt, st, use_filter, input, b, reuse, collect_output);
    case UDF_BC_FORWARD:
      return apply_bc_forward(rt, st, use_filter, input, b, reuse, collect_output);
    case UDF_BC_BACKWARD:
      return apply_bc_backward(rt, st, use_filter, input, b, reuse, collect_output);
    case UDF_SSSP_RELAX:
      return apply_sssp_relax(rt, st, use_filter, input, b, reuse, collect_output);
    default:
      fail(GG_ERR_VALUE, "unknown udf id");
  }
}

}  // namespace gg
