// prtile.cuh — merge-path tiled PageRank gather (no per-edge atomics).
//
// A "row set" is a list of destination rows with CSR offsets into an edge
// array of source ids: row r owns edges [roff[r], roff[r+1]).  The merge of
// rows and edges (each row = its edges followed by an END item) is cut into
// tiles of kTile items (Merrill & Garland merge-based SpMV); one CTA per tile:
//   1. stage the tile's relative row ends in smem;
//   2. load the tile's source ids (coalesced) and gather contrib[src] --
//      kTile/256 independent gathers per thread in flight -- into smem;
//   3. each thread walks kIpt merge items, adding edge values and emitting
//      row totals at END items (smem f64 adds combine rows split between
//      threads);
//   4. rows whose END is in the tile are finished in registers: MODE 0/2
//      fused vertex update (rank', L1, dangling mass, next contrib), MODE 1
//      accumulate into acc.  A row cut by a tile boundary ("crossing" row)
//      adds its partial into hubsum and is finished by the crossing-row pass.
#pragma once
#include "prpull.cuh"

namespace gg {

constexpr int kTile = 2048;
constexpr int kTileThreads = 256;
constexpr int kIpt = kTile / kTileThreads;  // merge items per thread

template <class CT>
struct TileArgs {
  const int64_t* roff;      // rows + 1
  const int32_t* owner;     // null: owner(r) = r - row_base
  int64_t row_base;         // first row of the row set in roff/owner numbering
  const int32_t* src;       // edge source ids
  const int64_t* tile_row;  // ntiles + 1 tile start coordinates (global row index)
  const int64_t* tile_edge; // (global edge index)
  int64_t ntiles;
  const CT* contrib;
  CT* contrib_next;
  double* rank;
  const int32_t* outdeg;
  double* acc;      // per-destination accumulator (MODE 1/2)
  double* hubsum;   // crossing-row partials (== acc in blocked mode)
  double* scal;
  int64_t V;
  double damping;
  int coherent;
};

__device__ __forceinline__ void smem_add(double* p, double v) { atomicAdd(p, v); }

template <class CT, int MODE>
__device__ __forceinline__ void pr_tiles(const TileArgs<CT>& a, int64_t it, double* s_val,
                                         int32_t* s_rend, double* s_rowsum) {
  const double n = (double)a.V;
  const double base = (1.0 - a.damping) / n + a.damping * a.scal[2 * it] / n;
  double l1 = 0, dm = 0;
  const int tid = threadIdx.x;
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const int64_t rb = a.tile_row[t], eb = a.tile_edge[t];
    const int64_t re = a.tile_row[t + 1], ee = a.tile_edge[t + 1];
    const int nr = (int)(re - rb), ne = (int)(ee - eb);
    // 1-2. row ends and gathered edge values into smem
    for (int i = tid; i < nr; i += kTileThreads) {
      s_rend[i] = (int32_t)(__ldg(a.roff + rb + i + 1) - eb);
      s_rowsum[i] = 0.0;
    }
    int32_t us[kIpt];
#pragma unroll
    for (int q = 0; q < kIpt; ++q) {
      const int j = tid + q * kTileThreads;
      us[q] = j < ne ? __ldcs(a.src + eb + j) : -1;
    }
#pragma unroll
    for (int q = 0; q < kIpt; ++q) {
      const int j = tid + q * kTileThreads;
      if (us[q] >= 0)
        s_val[j] = (double)(a.coherent ? ld_fresh(a.contrib + us[q]) : __ldg(a.contrib + us[q]));
    }
    __syncthreads();
    // 3. merge walk: start coordinate by binary search on the diagonal
    const int d0 = tid * kIpt;
    int lo = 0, hi = nr;  // rows consumed before d0: first i with s_rend[i] + i >= d0
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (s_rend[mid] + mid < d0) lo = mid + 1; else hi = mid;
    }
    int i = lo, j = d0 - lo;
    double sum = 0.0;
    const int total_items = nr + ne;
    // rows started and ended inside this thread's items are stored directly;
    // the first row's partial (head) and the open last row (tail) are
    // combined across threads by a segmented scan -- no shared atomics.
    int head_row = -1;
    double head_val = 0.0;
#pragma unroll
    for (int q = 0; q < kIpt; ++q) {
      if (d0 + q < total_items) {
        if (i < nr && j == s_rend[i]) {
          if (head_row < 0) {
            head_row = i;
            head_val = sum;
          } else {
            s_rowsum[i] = sum;
          }
          sum = 0.0;
          ++i;
        } else {
          sum += s_val[j];
          ++j;
        }
      }
    }
    // segmented inclusive scan of the tails (rows are nondecreasing in tid)
    int trow = i;
    double tval = sum;
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double v = __shfl_up_sync(0xffffffffu, tval, o);
      int r = __shfl_up_sync(0xffffffffu, trow, o);
      if (lane >= o && r == trow) tval += v;
    }
    __shared__ int s_wrow_first[kTileThreads / 32], s_wrow_last[kTileThreads / 32];
    __shared__ double s_wval[kTileThreads / 32];
    __shared__ int s_win_row[kTileThreads / 32];
    __shared__ double s_win_val[kTileThreads / 32];
    if (lane == 0) s_wrow_first[w] = trow;
    if (lane == 31) {
      s_wrow_last[w] = trow;
      s_wval[w] = tval;
    }
    __syncthreads();
    if (tid == 0) {
      int crow = -2;
      double cval = 0.0;
      for (int k = 0; k < kTileThreads / 32; ++k) {
        s_win_row[k] = crow;
        s_win_val[k] = cval;
        if (s_wrow_first[k] == s_wrow_last[k] && s_wrow_last[k] == crow) {
          cval += s_wval[k];
        } else {
          crow = s_wrow_last[k];
          cval = s_wval[k];
        }
      }
    }
    __syncthreads();
    if (trow == s_win_row[w]) tval += s_win_val[w];
    // publish each thread's scanned tail for its successor; the tile's last
    // open row (row `re`, continuing into the next tile) is a crossing row
    double* s_tval = s_val;  // edge values are no longer needed
    int32_t* s_trow = reinterpret_cast<int32_t*>(s_val + kTileThreads);
    __syncthreads();
    s_tval[tid] = tval;
    s_trow[tid] = trow;
    __syncthreads();
    if (head_row >= 0) {
      double tot = head_val;
      if (tid > 0 && s_trow[tid - 1] == head_row) tot += s_tval[tid - 1];
      s_rowsum[head_row] = tot;
    }
    if (tid == kTileThreads - 1 && trow >= nr && tval != 0.0) {
      const int64_t r = re;
      const int32_t o = a.owner ? a.owner[r - a.row_base] : (int32_t)(r - a.row_base);
      atomicAdd(a.hubsum + o, tval);
    }
    __syncthreads();
    // 4. finish the rows whose END is in this tile
    const bool first_cut = nr > 0 && __ldg(a.roff + rb) < eb;
    for (int k = tid; k < nr; k += kTileThreads) {
      const int64_t r = rb + k;
      const int32_t o = a.owner ? __ldg(a.owner + (r - a.row_base)) : (int32_t)(r - a.row_base);
      const double tot = s_rowsum[k];
      if (MODE == 1) {
        if (tot != 0.0) {
          if (k == 0 && first_cut) atomicAdd(a.acc + o, tot);
          else a.acc[o] += tot;
        }
        continue;
      }
      if (k == 0 && first_cut) {  // crossing row: finished by the crossing pass
        if (tot != 0.0) atomicAdd(a.hubsum + o, tot);
        continue;
      }
      double s = tot;
      if (MODE == 2) {
        s += a.acc[o];
        a.acc[o] = 0.0;
      }
      pr_finish_tile(a, o, s, base, l1, dm);
    }
    __syncthreads();
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
__device__ __forceinline__ void pr_finish_tile(const TileArgs<CT>& a, int32_t v, double sum,
                                               double base, double& l1, double& dm);

template <class CT>
__device__ __forceinline__ void pr_finish_tile(const TileArgs<CT>& a, int32_t v, double sum,
                                               double base, double& l1, double& dm) {
  double nv = base + a.damping * sum;
  l1 += fabs(nv - a.rank[v]);
  a.rank[v] = nv;
  int32_t od = __ldg(a.outdeg + v);
  if (od) a.contrib_next[v] = (CT)(nv / (double)od);
  else dm += nv;
}

// crossing rows: rows cut by a tile boundary, finished after all tiles
template <class CT>
__device__ __forceinline__ void pr_crossing(const TileArgs<CT>& a, int64_t it, const int32_t* rows,
                                            int64_t nrows) {
  const double n = (double)a.V;
  const double base = (1.0 - a.damping) / n + a.damping * a.scal[2 * it] / n;
  double l1 = 0, dm = 0;
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nrows;
       h += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = rows[h];
    double s = a.hubsum[v];
    a.hubsum[v] = 0.0;
    pr_finish_tile(a, v, s, base, l1, dm);
  }
  l1 = block_sum(l1);
  dm = block_sum(dm);
  if (threadIdx.x == 0) {
    if (l1 != 0.0) atomicAdd(a.scal + 2 * it + 1, l1);
    if (dm != 0.0) atomicAdd(a.scal + 2 * (it + 1), dm);
  }
}

template <class CT, int MODE>
__global__ void __launch_bounds__(kTileThreads) k_pr_tiles(TileArgs<CT> a, int64_t it) {
  __shared__ double s_val[kTile];
  __shared__ int32_t s_rend[kTile + 1];
  __shared__ double s_rowsum[kTile + 1];
  pr_tiles<CT, MODE>(a, it, s_val, s_rend, s_rowsum);
}

template <class CT>
__global__ void __launch_bounds__(256) k_pr_crossing(TileArgs<CT> a, int64_t it, const int32_t* rows,
                                                     int64_t nrows) {
  pr_crossing(a, it, rows, nrows);
}

// ---------------------------------------------------------------------------
// Host: merge-path tile partition of a row set and its crossing rows.
// ---------------------------------------------------------------------------
struct TilePlan {
  int64_t nrows = 0, ntiles = 0, ncross = 0;
  DevBuf<int64_t> tile_row, tile_edge;
  DevBuf<int32_t> cross;
};

// tile t starts at merge diagonal d = t*kTile: rows consumed = first r with
// (roff[r+1]-e0) + r >= d  (r relative), edges consumed = d - rows.
static __global__ void k_tile_starts(const int64_t* roff, int64_t nrows, int64_t row0, int64_t ntiles,
                                     int64_t* trow, int64_t* tedge) {
  const int64_t e0 = roff[row0], ne = roff[row0 + nrows] - e0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = t * (int64_t)kTile;
    if (d > nrows + ne) d = nrows + ne;
    int64_t lo = 0, hi = nrows;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if ((roff[row0 + mid + 1] - e0) + mid < d) lo = mid + 1; else hi = mid;
    }
    trow[t] = row0 + lo;
    tedge[t] = e0 + (d - lo);
  }
}
// rows cut by an inner tile boundary (their edges start before the boundary)
static __global__ void k_mark_cross(const int64_t* roff, const int64_t* trow, const int64_t* tedge,
                                    int64_t ntiles, int64_t row0, int64_t nrows, uint8_t* mark) {
  for (int64_t t = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = trow[t];
    if (r < row0 + nrows && roff[r] < tedge[t]) mark[r - row0] = 1;
  }
}

}  // namespace gg
