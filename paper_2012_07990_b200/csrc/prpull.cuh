// prpull.cuh — PageRank PULL+WM gather kernels shared by the single-GPU driver
// (pagerank.cu) and the vertex-partitioned multi-GPU driver (dist.cu).
#pragma once
#include "engine.cuh"
#include <cub/device/device_scan.cuh>

namespace gg {

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double s[32];
  v = warp_sum(v);
  __syncthreads();
  if (lane_id() == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? s[threadIdx.x] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

// ---------------------------------------------------------------------------
// PULL + WM fast path: warp-mapped gather over CSR-in with the vertex update
// fused into the same kernel (one launch per iteration + a tiny hub pass).
//
// Pull plan (cached per graph): destinations are "virtual rows"; a row with
// in-degree > hub_t is split into ceil(deg/hub_t) pieces so no warp owns an
// unbounded range.  Each warp takes 32 consecutive virtual rows, streams
// their concatenated in-edges 32 at a time (coalesced int32 loads), gathers
// contrib[src], reduces per row with a shuffle segmented scan, and finishes
// whole rows in registers: rank' = base + d*sum, L1, dangling mass, next
// contrib.  Hub pieces add their partial sums into hubsum[row] (f64 atomic)
// and the hub pass finishes those rows.  No per-edge atomics.
// ---------------------------------------------------------------------------
// Longest virtual row: a warp owns 32 consecutive virtual rows, so a chunk
// carries at most 32 * kPieceEdges edges (bounded warp work -> no stragglers).
constexpr int64_t kPieceEdges = 64;

struct PullPlan {
  int64_t hub_t = 0, nvrows = 0, nhubs = 0, lo = 0, hi = 0;
  DevBuf<int64_t> voff;    // nvrows + 1
  DevBuf<int32_t> vowner;  // row, or ~row for a hub piece, or INT32_MIN padding
  DevBuf<int32_t> hubs;    // hub rows
};

static __global__ void k_plan_pieces(const int64_t* off, int64_t V, int64_t hub_t, int64_t* pieces) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = off[v + 1] - off[v];  // off is shifted to the first row of the range
    pieces[v] = d > hub_t ? (d + hub_t - 1) / hub_t : 1;
  }
}
static __global__ void k_plan_fill(const int64_t* off, int64_t V, int64_t hub_t, const int64_t* vstart,
                            int64_t nvrows, int64_t* voff, int32_t* vowner, int32_t* hubs,
                            unsigned long long* nhubs, int64_t row0) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = off[v], d = off[v + 1] - lo, s = vstart[v];
    if (d > hub_t) {
      int64_t np = (d + hub_t - 1) / hub_t;
      for (int64_t k = 0; k < np; ++k) {
        voff[s + k] = lo + k * hub_t;
        vowner[s + k] = ~(int32_t)(row0 + v);
      }
      hubs[atomicAdd(nhubs, 1ULL)] = (int32_t)(row0 + v);
    } else {
      voff[s] = lo;
      vowner[s] = (int32_t)(row0 + v);
    }
  }
}
static __global__ void k_plan_pad(int64_t first, int64_t nvrows, int64_t E, int64_t* voff, int32_t* vowner) {
  for (int64_t i = first + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nvrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    voff[i] = E;
    if (i < nvrows) vowner[i] = INT32_MIN;
  }
}

// Plan over destination rows [lo, hi) (a rank's partition, or all rows).
// Callers hold the returned shared_ptr for the query (a concurrent query may
// replace the cache entry; the plan it uses stays alive).
inline std::shared_ptr<PullPlan> pull_plan_for(const Graph& gc, int64_t hub_t, int64_t lo = 0,
                                               int64_t hi = -1) {
  Graph& g = const_cast<Graph&>(gc);
  if (hi < 0) hi = g.V;
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.pull_plan && g.pull_plan->hub_t == hub_t && g.pull_plan->lo == lo && g.pull_plan->hi == hi)
    return g.pull_plan;
  CsrView in = g.in_view();
  in.off += lo;
  const int dev = g.dev;
  const int64_t V = hi - lo;
  auto p = std::make_shared<PullPlan>();
  p->hub_t = hub_t;
  p->lo = lo;
  p->hi = hi;
  DevBuf<int64_t> pieces(V + 1), vstart(V + 1);
  k_plan_pieces<<<grid_for(V, 256, dev), 256>>>(in.off, V, hub_t, pieces.p);
  GG_LAUNCH_CHECK();
  size_t temp = 0;
  GG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, pieces.p, vstart.p, V));
  DevBuf<uint8_t> tb(temp);
  GG_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, temp, pieces.p, vstart.p, V));
  int64_t last_start = 0, last_pieces = 0;
  GG_CUDA(cudaMemcpy(&last_start, vstart.p + V - 1, 8, cudaMemcpyDeviceToHost));
  GG_CUDA(cudaMemcpy(&last_pieces, pieces.p + V - 1, 8, cudaMemcpyDeviceToHost));
  const int64_t real = last_start + last_pieces;
  p->nvrows = (real + 31) / 32 * 32;
  p->voff.alloc(p->nvrows + 1);
  p->vowner.alloc(p->nvrows);
  p->hubs.alloc(V);
  DevBuf<unsigned long long> nh(1);
  nh.zero();
  k_plan_fill<<<grid_for(V, 256, dev), 256>>>(in.off, V, hub_t, vstart.p, p->nvrows, p->voff.p,
                                              p->vowner.p, p->hubs.p, nh.p, lo);
  int64_t end_edge = 0;
  GG_CUDA(cudaMemcpy(&end_edge, in.off + V, 8, cudaMemcpyDeviceToHost));
  k_plan_pad<<<grid_for(p->nvrows - real + 1, 256, dev), 256>>>(real, p->nvrows, end_edge, p->voff.p,
                                                                p->vowner.p);
  GG_LAUNCH_CHECK();
  unsigned long long h = 0;
  GG_CUDA(cudaMemcpy(&h, nh.p, 8, cudaMemcpyDeviceToHost));
  p->nhubs = (int64_t)h;
  g.pull_plan = p;
  return p;
}

static __global__ void k_outdeg(const int64_t* off, int64_t V, int32_t* deg) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    deg[v] = (int32_t)(off[v + 1] - off[v]);
}

template <class CT>
struct PrPullArgs {
  const int64_t* voff;
  const int32_t* vowner;
  int64_t nchunks;
  const int32_t* nbr;
  const CT* contrib;
  CT* contrib_next;
  double* rank;
  const int32_t* outdeg;
  double* hubsum;
  const int32_t* hubs;
  int64_t nhubs;
  double* scal;
  int64_t V;
  double damping;
  int coherent = 0;  // fused loops re-read contrib written earlier in the same launch
};

// finish one destination: fused vertex pass (algos.py:192-198 + :184-189)
template <class CT>
__device__ __forceinline__ void pr_finish(const PrPullArgs<CT>& a, int32_t v, double sum,
                                          double base, double& l1, double& dm) {
  double nv = base + a.damping * sum;
  l1 += fabs(nv - a.rank[v]);
  a.rank[v] = nv;
  int32_t od = __ldg(a.outdeg + v);
  if (od) a.contrib_next[v] = (CT)(nv / (double)od);
  else dm += nv;
}

// MODE 0: whole rows, finish in place.  MODE 1 (cold EdgeBlocking segment):
// add row sums into acc (== hubsum).  MODE 2 (hot, final segment): finish
// with sum + acc and reset acc.  Hub pieces always add into hubsum.
template <class CT, int MODE = 0>
__device__ __forceinline__ void pr_pull_chunks(const PrPullArgs<CT>& a, int64_t it, double* s_acc_all,
                                               int64_t c_begin = 0, int64_t c_end = -1) {
  if (c_end < 0) c_end = a.nchunks;
  const int lane = lane_id();
  const int wib = threadIdx.x >> 5;
  double* s_acc = s_acc_all + wib * 32;
  const double n = (double)a.V;
  const double base = (1.0 - a.damping) / n + a.damping * a.scal[2 * it] / n;
  double l1 = 0, dm = 0;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = c_begin + warp; c < c_end; c += nwarps) {
    const int64_t vr = c * 32 + lane;
    const int64_t lo = __ldg(a.voff + vr);
    const int64_t deg = __ldg(a.voff + vr + 1) - lo;
    const int32_t owner = __ldg(a.vowner + vr);
    int64_t incl = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int64_t excl = incl - deg;
    const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
    s_acc[lane] = 0.0;
    __syncwarp();
    // kU strides of 32 edges per step: all index loads, then all gathers,
    // then the reductions -- kU*32 independent gathers in flight per warp.
    constexpr int kU = 4;
    for (int64_t k0 = 0; k0 < total; k0 += 32 * kU) {
      int jv[kU];
      int32_t uv[kU];
      double val[kU];
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const int64_t k = k0 + q * 32 + lane;
        int j = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          int64_t em = __shfl_sync(0xffffffffu, excl, j + step);
          if (em <= k) j += step;
        }
        const int64_t loj = __shfl_sync(0xffffffffu, lo, j);
        const int64_t exj = __shfl_sync(0xffffffffu, excl, j);
        jv[q] = j;
        uv[q] = k < total ? __ldg(a.nbr + loj + (k - exj)) : -1;
      }
#pragma unroll
      for (int q = 0; q < kU; ++q)
        val[q] = uv[q] >= 0 ? (double)(a.coherent ? ld_fresh(a.contrib + uv[q]) : __ldg(a.contrib + uv[q]))
                            : 0.0;
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const int64_t k = k0 + q * 32 + lane;
        const int j = jv[q];
        double v = val[q];
        // segmented inclusive scan over runs of equal owner lane j
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          double t = __shfl_up_sync(0xffffffffu, v, o);
          int jj = __shfl_up_sync(0xffffffffu, j, o);
          if (lane >= o && jj == j) v += t;
        }
        const int jn = __shfl_down_sync(0xffffffffu, j, 1);
        const bool tail = k < total && (lane == 31 || jn != j || k + 1 >= total);
        if (tail) s_acc[j] += v;
        __syncwarp();
      }
    }
    const double sum = s_acc[lane];
    __syncwarp();
    if (owner >= 0) {
      if (MODE == 1) {
        if (sum != 0.0) a.hubsum[owner] += sum;
      } else {
        double s = sum;
        if (MODE == 2) {
          s += a.hubsum[owner];
          a.hubsum[owner] = 0.0;
        }
        pr_finish(a, owner, s, base, l1, dm);
      }
    } else if (owner != INT32_MIN && sum != 0.0) {
      atomicAdd(a.hubsum + ~owner, sum);
    }
  }
  if (MODE != 1) {
    l1 = block_sum(l1);
    dm = block_sum(dm);
    if (threadIdx.x == 0) {
      if (l1 != 0.0) atomicAdd(a.scal + 2 * it + 1, l1);
      if (dm != 0.0) atomicAdd(a.scal + 2 * (it + 1), dm);
    }
  }
}

template <class CT>
__device__ __forceinline__ void pr_pull_hubs(const PrPullArgs<CT>& a, int64_t it) {
  const double n = (double)a.V;
  const double base = (1.0 - a.damping) / n + a.damping * a.scal[2 * it] / n;
  double l1 = 0, dm = 0;
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < a.nhubs;
       h += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = a.hubs[h];
    double sum = a.hubsum[v];
    a.hubsum[v] = 0.0;
    pr_finish(a, v, sum, base, l1, dm);
  }
  l1 = block_sum(l1);
  dm = block_sum(dm);
  if (threadIdx.x == 0) {
    if (l1 != 0.0) atomicAdd(a.scal + 2 * it + 1, l1);
    if (dm != 0.0) atomicAdd(a.scal + 2 * (it + 1), dm);
  }
}

template <class CT>
__global__ void __launch_bounds__(256) k_pr_pull(PrPullArgs<CT> a, int64_t it) {
  __shared__ double s_acc[8 * 32];
  pr_pull_chunks(a, it, s_acc);
}

template <class CT, int MODE>
__global__ void __launch_bounds__(256) k_pr_seg(PrPullArgs<CT> a, int64_t it, int64_t c_begin,
                                                int64_t c_end) {
  __shared__ double s_acc[8 * 32];
  pr_pull_chunks<CT, MODE>(a, it, s_acc, c_begin, c_end);
}

template <class CT>
__global__ void __launch_bounds__(256) k_pr_pull_hubs(PrPullArgs<CT> a, int64_t it) {
  pr_pull_hubs(a, it);
}

// whole loop in one cooperative launch (kernel fusion)
template <class CT>
__global__ void __launch_bounds__(256) k_pr_pull_fused(PrPullArgs<CT> a, CT* c0, CT* c1,
                                                       int64_t max_iters, double tol,
                                                       int64_t* iters_out) {
  __shared__ double s_acc[8 * 32];
  cg::grid_group grid = cg::this_grid();
  a.coherent = 1;
  int64_t it = 0;
  double l1 = INFINITY;
  while (!(it >= max_iters || l1 < tol)) {
    a.contrib = (it & 1) ? c1 : c0;
    a.contrib_next = (it & 1) ? c0 : c1;
    pr_pull_chunks(a, it, s_acc);
    grid.sync();
    pr_pull_hubs(a, it);
    grid.sync();
    l1 = *((volatile double*)a.scal + 2 * it + 1);
    ++it;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *iters_out = it;
}


template <class CT>
static __global__ void __launch_bounds__(256) k_pr_init_dist(const int64_t* off, int64_t V, double* rank,
                                                             CT* contrib, double* dm0) {
  const double r0 = 1.0 / (double)V;
  double dm = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = off[v + 1] - off[v];
    rank[v] = r0;
    contrib[v] = d ? (CT)(r0 / (double)d) : (CT)0;
    if (!d) dm += r0;
  }
  dm = block_sum(dm);
  if (threadIdx.x == 0 && dm != 0.0) atomicAdd(dm0, dm);
}

}  // namespace gg
