// traverse.cuh — device side of edgeset.apply (reference engine.py:418-608).
//
// One template family per load-balancing strategy (engine.py:32-256), for
// both directions, plus the flat / blocked COO paths (engine.py:558-608,
// blocking.py:116-186).  A traversal is parameterised by an Op functor (the
// named device UDF, see ops.cuh) and an OutBuilder (output frontier creation
// with dedup, engine.py:279-397).
//
// Graph layout in HBM (built once, graph.cu):
//   CSR-out  out_off int64[V+1], out_nbr int32[E], out_w uint32[E]
//   CSR-in   in_off  int64[V+1], in_nbr  int32[E], in_w  uint32[E]
//   COO      src int32[E], dst int32[E], w uint32[E]   (load order)
// Frontiers: SPARSE int32 queue + u64 device count; BITMAP u32 words (same
// byte/bit order as the reference's bytearray, frontier.py:184); BOOLMAP u8.
#pragma once
#include <type_traits>
#include "common.cuh"
#include <cooperative_groups.h>

namespace gg {
namespace cg = cooperative_groups;

constexpr int kWarp = 32;

// ETWC split of one vertex's edge range (engine.py:62-85): a cta multiple
// (stage 2), then a warp multiple (stage 1), then the remainder (stage 0).
struct EtwcSizes {
  int64_t e2, e1, e0;
};
__host__ __device__ __forceinline__ EtwcSizes etwc_sizes(int64_t size, int cta) {
  const int64_t e2 = (size / cta) * cta;
  const int64_t e1 = ((size - e2) / kWarp) * kWarp;
  return {e2, e1, size - e2 - e1};
}
// TWC bin (engine.py:131-142): promotion is strictly greater.
__host__ __device__ __forceinline__ int twc_bin_of(int64_t deg, int cta) {
  return deg > cta ? 2 : (deg > kWarp ? 1 : 0);
}

// ---------------------------------------------------------------------------
// Read-only views
// ---------------------------------------------------------------------------
struct CsrView {
  const int64_t* off;
  const int32_t* nbr;
  const uint32_t* w;  // may be null
  int64_t V;
};

struct CooView {
  const int32_t* src;
  const int32_t* dst;
  const uint32_t* w;
  int64_t E;
};

// Input frontier view. repr -1 = every vertex active (input None).
struct InView {
  int repr;
  const int32_t* ids;
  const unsigned long long* count;
  const uint32_t* bits;
  const uint8_t* bools;
  int coherent = 0;  // fused loops: membership written earlier in the same launch
  int64_t n_fixed = -1;  // SPARSE size known to every thread (fused loops): *count unread

  __device__ __forceinline__ int64_t size() const { return n_fixed >= 0 ? n_fixed : (int64_t)*count; }
  __device__ __forceinline__ bool member(int32_t u) const {
    if (repr == GG_BITMAP)
      return ((coherent ? ld_fresh(bits + (u >> 5)) : __ldg(bits + (u >> 5))) >> (u & 31)) & 1u;
    if (repr == GG_BOOLMAP) return (coherent ? ld_fresh(bools + u) : __ldg(bools + u)) != 0;
    return true;  // all active
  }
};

// ---------------------------------------------------------------------------
// Output frontier builder (engine.py:279-397 + frontier.py:34-118).
// ---------------------------------------------------------------------------
enum { OUT_NONE = -1 };
enum { DEDUP_NONE = 0, DEDUP_COUNTERS = 1, DEDUP_MARK_BITS = 2, DEDUP_MARK_BYTES = 3,
       DEDUP_SLOT = 4 };

__device__ __forceinline__ bool test_and_set_bit(uint32_t* words, int32_t v) {
  uint32_t m = 1u << (v & 31);
  return (atomicOr(words + (v >> 5), m) & m) != 0;
}
__device__ __forceinline__ bool test_and_set_byte(uint8_t* bytes, int32_t v) {
  // byte test-and-set through the aligned 32-bit word holding it
  uint32_t* w = reinterpret_cast<uint32_t*>(bytes + (v & ~3));
  uint32_t m = 1u << ((v & 3) * 8);
  return (atomicOr(w, m) & m) != 0;
}

struct OutBuilder {
  int mode;   // OUT_NONE or GG_CREATE_*
  int dedup;  // DEDUP_*
  int32_t* queue;
  unsigned long long* qcount;
  uint32_t* bits;
  uint8_t* bools;
  int32_t* stamps;
  int32_t round;
  uint32_t* mark_bits;
  uint8_t* mark_bytes;

  __device__ __forceinline__ bool accept(int32_t v) const {
    switch (dedup) {
      case DEDUP_COUNTERS:
        if (*((volatile int32_t*)stamps + v) == round) return false;
        return atomicExch(stamps + v, round) != round;
      case DEDUP_MARK_BITS: return !test_and_set_bit(mark_bits, v);
      case DEDUP_MARK_BYTES: return !test_and_set_byte(mark_bytes, v);
      default: return true;
    }
  }

  // ctx.enqueue(v) (runtime.py:319-323): returns the dedup decision.
  __device__ __forceinline__ bool emit(int32_t v) const {
    if (mode == GG_CREATE_FUSED) {
      bool ok = accept(v);
      // warp-aggregated append: one atomic per converged group of lanes
      cg::coalesced_group g = cg::coalesced_threads();
      unsigned ballot = g.ballot(ok);
      unsigned long long base = 0;
      if (g.thread_rank() == 0 && ballot) base = atomicAdd(qcount, (unsigned long long)__popc(ballot));
      base = g.shfl(base, 0);
      if (ok) queue[base + __popc(ballot & ((1u << g.thread_rank()) - 1))] = v;
      return ok;
    }
    if (mode == GG_CREATE_UNFUSED_BOOLMAP) {
      if (dedup == DEDUP_SLOT) return !test_and_set_byte(bools, v);
      if (dedup != DEDUP_NONE && !accept(v)) return false;
      bools[v] = 1;
      return true;
    }
    if (mode == GG_CREATE_UNFUSED_BITMAP) {
      if (dedup != DEDUP_SLOT && dedup != DEDUP_NONE && !accept(v)) return false;
      // warp-aggregated bit set: lanes whose vertices share an output word
      // OR their bits together and one of them issues the atomic (a pull
      // level sets 32 consecutive vertices' bits from one warp); with slot
      // dedup the first lane holding a vertex takes it iff its bit was clear
      const unsigned act = __activemask();
      const unsigned lane = lane_id();
      const unsigned same_v = __match_any_sync(act, v);
      const bool first_v = lane == (unsigned)(__ffs(same_v) - 1);
      const uint32_t w = (uint32_t)v >> 5, bit = 1u << (v & 31);
      const unsigned same_w = __match_any_sync(act, w);
      const uint32_t m = __reduce_or_sync(same_w, first_v ? bit : 0u);
      const int leader = __ffs(same_w) - 1;
      uint32_t old = 0;
      if ((int)lane == leader) old = atomicOr(bits + w, m);
      old = __shfl_sync(same_w, old, leader);
      if (dedup == DEDUP_SLOT) return first_v && !(old & bit);
      return true;
    }
    return false;
  }
};

// Edges scanned (RunStats.edges_traversed): one atomic per warp.
__device__ __forceinline__ void add_scanned(unsigned long long* ctr, int64_t n) {
  unsigned long long s = (unsigned long long)n;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane_id() == 0 && s) atomicAdd(ctr, s);
}

// Active id at position i of the input (input None => identity).
__device__ __forceinline__ int32_t active_at(const InView& in, int64_t i) {
  return in.repr == -1 ? (int32_t)i : __ldg(in.ids + i);
}
__device__ __forceinline__ int64_t active_count(const InView& in, int64_t V) {
  return in.repr == -1 ? V : in.size();
}

// Largest j in [0, n) with key(j) <= x over a sorted array (binary search).
template <class F>
__device__ __forceinline__ int upper_idx(F key, int n, int64_t x) {
  int lo = 0, hi = n;  // invariant: answer in [lo, hi)
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (key(mid) <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// ===========================================================================
// PUSH (engine.py:463-503): per active source, scan out-edges, filter dst,
// udf with atomic helpers.
// ===========================================================================
struct EtwcEntry;
// a queued arc range [lo, lo + len) of source u (ETWC / hub grid pass)
struct EtwcEntry {
  int64_t lo;
  int32_t len;
  int32_t u;
  __device__ __forceinline__ int64_t hi() const { return lo + len; }
};
template <class Op>
struct PushArgs {
  CsrView g;
  InView in;
  Op op;
  OutBuilder out;
  int use_filter;
  unsigned long long* scanned;
  // ETWC: CTA-stage ranges of at least kEtwcHuge edges go to this global
  // queue and are processed by the whole grid afterwards (null: in-CTA)
  EtwcEntry* huge = nullptr;
  unsigned long long* huge_n = nullptr;
  int64_t huge_min = 16384;  // kEtwcHuge; the CTA size for small frontiers (run_push)
};

template <class Op>
__device__ __forceinline__ void push_edge(const PushArgs<Op>& a, int32_t u, int64_t e) {
  int32_t v = __ldg(a.g.nbr + e);
  if (a.use_filter && !a.op.filter(v)) return;
  uint32_t w = a.g.w ? __ldg(a.g.w + e) : 0u;
  a.op.push(u, v, w, a.out);
}

// cooperative range walk (defined with the ETWC stages below); ops may pin
// the traversal kernels' residency (kMinBlocks CTAs of 256 per SM: a
// register cap, the *_mb kernel twins) when their chains are latency-bound.
// Ops that do not declare it launch the plain kernels: an explicit minimum
// of 1 would lift the compiler's own register budget (BC kernels went from
// 32-48 to 58-70 registers and ~12% slower, measured)
template <class Op>
__device__ __forceinline__ void push_range_strided(const PushArgs<Op>& a, int32_t u, int64_t lo, int64_t hi,
                                                   int64_t first, int64_t stride, bool warp_uniform = true);
template <class, class = void>
struct MinBlocks : std::integral_constant<int, 1> {};
template <class T>
struct MinBlocks<T, std::void_t<decltype(T::kMinBlocks)>> : std::integral_constant<int, T::kMinBlocks> {};

// VERTEX_BASED (engine.py:179-183): one thread per active vertex.
template <class Op>
__device__ __forceinline__ void b_push_vb(PushArgs<Op> a) {
  const int64_t n = active_count(a.in, a.g.V);
  int64_t sc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t u = active_at(a.in, i);
    int64_t lo = __ldg(a.g.off + u), hi = __ldg(a.g.off + u + 1);
    sc += hi - lo;
    for (int64_t e = lo; e < hi; ++e) push_edge(a, u, e);
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_push_vb(PushArgs<Op> a) {
  b_push_vb<Op>(a);
}

// WM (engine.py:167-176): each warp takes 32 contiguous active vertices and
// processes their concatenated edge lists lane-cyclically (warp prefix sum +
// shuffle binary search to find each edge's owner).
template <class Op>
__device__ __forceinline__ void b_push_wm(PushArgs<Op> a) {
  const int64_t n = active_count(a.in, a.g.V);
  const int lane = lane_id();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // even contiguous split of the active list over warps, earlier warps take
  // the extra (engine.py:167-176, partition_even_chunks :32-44): a small
  // frontier spreads its edges over many warps (one edge per lane) instead
  // of queueing them behind one another
  const int64_t per = n / nwarps, extra = n % nwarps;
  const int64_t wstart = warp * per + min(warp, extra);
  const int64_t wend = wstart + per + (warp < extra ? 1 : 0);
  int64_t sc = 0;
  for (int64_t base = wstart; base < wend; base += kWarp) {
    int64_t i = base + lane;
    int32_t u = -1;
    int64_t lo = 0, deg = 0;
    if (i < wend) {
      u = active_at(a.in, i);
      lo = __ldg(a.g.off + u);
      deg = __ldg(a.g.off + u + 1) - lo;
    }
    // inclusive warp scan of degrees
    int64_t incl = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int64_t excl = incl - deg;
    int64_t total = __shfl_sync(0xffffffffu, incl, 31);
    sc += deg;
    for (int64_t k0 = 0; k0 < total; k0 += kWarp) {
      const int64_t k = k0 + lane;
      // owner = largest lane j with excl_j <= k (never a zero-degree lane
      // when k < total); all lanes take part in every shuffle.
      int j = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        int64_t em = __shfl_sync(0xffffffffu, excl, j + step);
        if (em <= k) j += step;
      }
      int32_t uj = __shfl_sync(0xffffffffu, u, j);
      int64_t loj = __shfl_sync(0xffffffffu, lo, j);
      int64_t exj = __shfl_sync(0xffffffffu, excl, j);
      if (k < total) push_edge(a, uj, loj + (k - exj));
    }
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_push_wm(PushArgs<Op> a) {
  b_push_wm<Op>(a);
}

// CM (engine.py:160-164): each CTA takes blockDim contiguous active vertices
// and processes their concatenated edges cooperatively (CTA prefix sum in
// shared memory + binary search).
template <class Op>
__device__ __forceinline__ void b_push_cm(PushArgs<Op> a) {
  __shared__ int64_t s_excl[257];
  __shared__ int64_t s_lo[256];
  __shared__ int32_t s_u[256];
  const int64_t n = active_count(a.in, a.g.V);
  int64_t sc = 0;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t deg = 0;
    if (i < n) {
      int32_t u = active_at(a.in, i);
      s_u[threadIdx.x] = u;
      s_lo[threadIdx.x] = __ldg(a.g.off + u);
      deg = __ldg(a.g.off + u + 1) - s_lo[threadIdx.x];
    } else {
      s_u[threadIdx.x] = -1;
      s_lo[threadIdx.x] = 0;
    }
    sc += deg;
    s_excl[threadIdx.x + 1] = deg;
    if (threadIdx.x == 0) s_excl[0] = 0;
    __syncthreads();
    // simple Hillis-Steele scan over 256 entries (shared memory)
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
      int64_t t = (threadIdx.x + 1 > (unsigned)o) ? s_excl[threadIdx.x + 1 - o] : 0;
      __syncthreads();
      s_excl[threadIdx.x + 1] += t;
      __syncthreads();
    }
    const int64_t total = s_excl[blockDim.x];
    const int cnt = (int)blockDim.x;
    for (int64_t k = threadIdx.x; k < total; k += blockDim.x) {
      int j = upper_idx([&](int m) { return s_excl[m]; }, cnt, k);
      // skip zero-degree owners that share the same prefix
      while (j + 1 < cnt && s_excl[j + 1] <= k) ++j;
      push_edge(a, s_u[j], s_lo[j] + (k - s_excl[j]));
    }
    __syncthreads();
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_push_cm(PushArgs<Op> a) {
  b_push_cm<Op>(a);
}

// STRICT (engine.py:97-122): exact edge balance.  `prefix` is the exclusive
// degree prefix over the active list (length n+1, computed by a device scan);
// each thread takes a contiguous run of `per` edges and locates its first
// owner by binary search.
template <class Op>
__device__ __forceinline__ void b_push_strict(PushArgs<Op> a, const int64_t* prefix,
                                                      int64_t per) {
  const int64_t n = active_count(a.in, a.g.V);
  const int64_t total = prefix[n];
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t elo = t * per; elo < total; elo += (int64_t)gridDim.x * blockDim.x * per) {
    int64_t ehi = min(total, elo + per);
    // largest i with prefix[i] <= elo
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (__ldg(prefix + mid) <= elo) lo = mid; else hi = mid;
    }
    for (int64_t i = lo; i < n; ++i) {
      int64_t p0 = __ldg(prefix + i), p1 = __ldg(prefix + i + 1);
      if (p0 >= ehi) break;
      int64_t a0 = max(elo, p0), a1 = min(ehi, p1);
      if (a0 >= a1) continue;
      int32_t u = active_at(a.in, i);
      int64_t off = __ldg(a.g.off + u);
      for (int64_t k = a0; k < a1; ++k) push_edge(a, u, off + (k - p0));
    }
  }
  if (t == 0) atomicAdd(a.scanned, (unsigned long long)total);
}
template <class Op>
__global__ void __launch_bounds__(256) k_push_strict(PushArgs<Op> a, const int64_t* prefix,
                                                      int64_t per) {
  b_push_strict<Op>(a, prefix, per);
}

// TWC (engine.py:125-157): global buckets by degree (> cta: CTA queue,
// > warp: warp queue, else thread queue; strictly greater promotion).
struct TwcQueues {
  int32_t* q[3];               // 0 thread, 1 warp, 2 cta
  unsigned long long* cnt;     // [3]
};

template <class Op>
__device__ __forceinline__ void b_twc_bin(PushArgs<Op> a, TwcQueues q, int cta) {
  const int64_t n = active_count(a.in, a.g.V);
  int64_t sc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t u = active_at(a.in, i);
    const int64_t lo = __ldg(a.g.off + u);
    int64_t deg = __ldg(a.g.off + u + 1) - lo;
    sc += deg;
    if (a.huge && deg >= a.huge_min) {  // hub: the chunked grid pass (run_push)
      a.huge[atomicAdd(a.huge_n, 1ULL)] = EtwcEntry{lo, (int32_t)deg, u};
      continue;
    }
    int b = twc_bin_of(deg, cta);
    cg::coalesced_group g = cg::coalesced_threads();
    cg::coalesced_group gb = cg::labeled_partition(g, b);
    unsigned long long base = 0;
    if (gb.thread_rank() == 0) base = atomicAdd(q.cnt + b, (unsigned long long)gb.size());
    base = gb.shfl(base, 0);
    q.q[b][base + gb.thread_rank()] = u;
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_twc_bin(PushArgs<Op> a, TwcQueues q, int cta) {
  b_twc_bin<Op>(a, q, cta);
}

template <class Op>
__device__ __forceinline__ void b_twc_thread(PushArgs<Op> a, const int32_t* qu,
                                                    const unsigned long long* cnt) {
  const int64_t n = (int64_t)*cnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t u = qu[i];
    int64_t lo = __ldg(a.g.off + u), hi = __ldg(a.g.off + u + 1);
    push_range_strided(a, u, lo, hi, 0, 1, false);
  }
}
template <class Op>
__global__ void __launch_bounds__(256) k_twc_thread(PushArgs<Op> a, const int32_t* qu,
                                                    const unsigned long long* cnt) {
  b_twc_thread<Op>(a, qu, cnt);
}
template <class Op, int kMinB>
__global__ void __launch_bounds__(256, kMinB) k_twc_thread_mb(PushArgs<Op> a, const int32_t* qu,
                                                             const unsigned long long* cnt) {
  b_twc_thread<Op>(a, qu, cnt);
}

template <class Op>
__device__ __forceinline__ void b_twc_warp(PushArgs<Op> a, const int32_t* qu,
                                                  const unsigned long long* cnt) {
  const int64_t n = (int64_t)*cnt;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    int32_t u = qu[i];
    int64_t lo = __ldg(a.g.off + u), hi = __ldg(a.g.off + u + 1);
    push_range_strided(a, u, lo, hi, lane_id(), kWarp);
  }
}
template <class Op>
__global__ void __launch_bounds__(256) k_twc_warp(PushArgs<Op> a, const int32_t* qu,
                                                  const unsigned long long* cnt) {
  b_twc_warp<Op>(a, qu, cnt);
}
template <class Op, int kMinB>
__global__ void __launch_bounds__(256, kMinB) k_twc_warp_mb(PushArgs<Op> a, const int32_t* qu,
                                                           const unsigned long long* cnt) {
  b_twc_warp<Op>(a, qu, cnt);
}

// (Dealing the whole CTA bin over the grid in chunks, like the ETWC grid
// pass, measured slower for CC on Kronecker-25 -- 66 vs 85 GTEPS: the bin
// holds ~10^6 ranges and every CTA walks the whole bin to number the chunks;
// only hubs of >= kEtwcHuge arcs take that pass, queued by b_twc_bin.)
template <class Op>
__device__ __forceinline__ void b_twc_cta(PushArgs<Op> a, const int32_t* qu,
                                                 const unsigned long long* cnt) {
  const int64_t n = (int64_t)*cnt;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    int32_t u = qu[i];
    int64_t lo = __ldg(a.g.off + u), hi = __ldg(a.g.off + u + 1);
    push_range_strided(a, u, lo, hi, threadIdx.x, blockDim.x);
  }
}
template <class Op>
__global__ void __launch_bounds__(256) k_twc_cta(PushArgs<Op> a, const int32_t* qu,
                                                 const unsigned long long* cnt) {
  b_twc_cta<Op>(a, qu, cnt);
}
template <class Op, int kMinB>
__global__ void __launch_bounds__(256, kMinB) k_twc_cta_mb(PushArgs<Op> a, const int32_t* qu,
                                                          const unsigned long long* cnt) {
  b_twc_cta<Op>(a, qu, cnt);
}


// ETWC (engine.py:51-85, 186-193; paper Alg. 3).  Each CTA takes blockDim
// contiguous active vertices; every vertex's range is split into a
// CTA-multiple (Q2), warp-multiple (Q1) and remainder (Q0) chunk, queued in
// shared memory (warp ballot + CTA prefix for slots), then the stages run in
// order 0, 1, 2 with thread / warp / CTA cooperative processing.
// A single CTA walking a hub's whole CTA-stage range serialises on the hub
// (RMAT/Kronecker hubs have 10^5-10^6 arcs, several can land in one CTA's
// slice of the active list): such ranges are handed to the whole grid.
constexpr int64_t kEtwcHuge = 16384;
// active lists shorter than kEtwcSmallPerSm x SMs (< 1 CTA per 4 SMs) send
// every CTA-stage range to the grid pass (run_push, fused loops)
constexpr int64_t kEtwcSmallPerSm = 64;

// Ops whose push is "accumulate into the SOURCE" (BC backward: delta[u] +=
// f(v)) declare kPushReduce and provide push_val / push_commit: a range walk
// sums its arcs per thread, reduces over the warp and issues one atomic per
// warp instead of one per arc on the same address.
template <class, class = void>
struct PushReduce : std::false_type {};
template <class T>
struct PushReduce<T, std::void_t<decltype(T::kPushReduce)>> : std::integral_constant<bool, T::kPushReduce> {};
// Ops whose per-arc work is a chain of dependent loads (CC hook: label[v],
// then label[max], then the atomic) declare kPush4 and provide push4(u, v[4],
// live mask): a range walk hands them 4 arcs at once so the 4 chains' loads
// are in flight together (the hook round was latency-bound: long_scoreboard
// 68%, one chain per thread); push4 applies the op's filter (when the apply
// has one) to the batch itself.  Unweighted ops only.
template <class, class = void>
struct PushBatch : std::false_type {};
template <class T>
struct PushBatch<T, std::void_t<decltype(T::kPush4)>> : std::integral_constant<bool, T::kPush4> {};

// Cooperative range walk with 4 independent arcs in flight per thread.
// `warp_uniform`: every lane of the warp walks the same source u.
template <class Op>
__device__ __forceinline__ void push_range_strided(const PushArgs<Op>& a, int32_t u, int64_t lo, int64_t hi,
                                                   int64_t first, int64_t stride, bool warp_uniform) {
  int64_t e = lo + first;
  if constexpr (PushReduce<Op>::value) {
    // 4 arcs in flight: their (dependent) id -> filter -> state chains are
    // independent of each other (BC backward was latency-bound, one chain
    // per thread: long_scoreboard 75%)
    double acc = 0.0;
    for (; e + 3 * stride < hi; e += 4 * stride) {
      int32_t v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __ldg(a.g.nbr + e + k * stride);
      double x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) x[k] = (a.use_filter && !a.op.filter(v[k])) ? 0.0 : a.op.push_val(u, v[k]);
      acc += (x[0] + x[1]) + (x[2] + x[3]);
    }
    for (; e < hi; e += stride) {
      const int32_t v = __ldg(a.g.nbr + e);
      if (a.use_filter && !a.op.filter(v)) continue;
      acc += a.op.push_val(u, v);
    }
    if (warp_uniform) {
      acc = warp_sum(acc);
      if (lane_id() == 0 && acc != 0.0) a.op.push_commit(u, acc);
    } else if (acc != 0.0) {
      a.op.push_commit(u, acc);
    }
    return;
  }
  if constexpr (PushBatch<Op>::value) {
    for (; e < hi; e += 4 * stride) {
      int32_t v[4];
      unsigned live = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool in = e + k * stride < hi;
        v[k] = in ? __ldg(a.g.nbr + e + k * stride) : 0;
        if (in) live |= 1u << k;
      }
      a.op.push4(u, v, live, a.use_filter, a.out);  // applies the filter itself, batched
    }
  } else {
    for (; e + 3 * stride < hi; e += 4 * stride) {
      int32_t v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __ldg(a.g.nbr + e + k * stride);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (a.use_filter && !a.op.filter(v[k])) continue;
        uint32_t w = a.g.w ? __ldg(a.g.w + e + k * stride) : 0u;
        a.op.push(u, v[k], w, a.out);
      }
    }
    for (; e < hi; e += stride) push_edge(a, u, e);
  }
}

// Grid-wide pass over the CTA-stage ranges queued by b_push_etwc.  The
// ranges are cut into chunks of kHugeChunk arcs, numbered in queue order, and
// chunk j goes to CTA j mod gridDim (each CTA walks its chunks with all its
// threads), so the work is balanced over the whole grid however the arcs are
// spread over the ranges.  The queue is read 256 entries at a time: a block
// scan of the per-entry chunk counts, then a binary search per chunk.
constexpr int64_t kHugeChunk = 2048;
// A FUSED output is staged per chunk in shared memory (a push arc emits at
// most once) and appended with one global atomic per chunk: with one atomic
// per converged lane group on the queue counter, a 7072-vertex RMAT-24 BFS
// level that discovers 4 M vertices spent most of its 1.4 ms waiting on
// that single address.
// (kStage = false inside the fused cooperative kernels: their static shared
// memory is at the 48 KB limit.)
struct ChunkStage {
  int32_t q[kHugeChunk];
  unsigned long long n, base;
};
template <class Op, bool kStage, class Src>
__device__ __forceinline__ void push_ranges_chunked(const PushArgs<Op>& a, int64_t n, Src src) {
  __shared__ EtwcEntry s_e[256];
  __shared__ int64_t s_end[256];  // inclusive prefix of chunk counts in the batch
  __shared__ int64_t s_w[8];
  ChunkStage* st = nullptr;
  if constexpr (kStage) {
    __shared__ ChunkStage s_stage;
    st = &s_stage;
  }
  const bool stage = kStage && a.out.mode == GG_CREATE_FUSED;
  PushArgs<Op> b = a;
  if (stage) {
    b.out.queue = st->q;
    b.out.qcount = &st->n;
    if (threadIdx.x == 0) st->n = 0;  // published by the batch loop's first barrier
  }
  const int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t G = gridDim.x;
  int64_t gchunk = 0;  // chunks of the batches before this one
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    int64_t x = 0;
    if (i < n) {
      const EtwcEntry c = src(i);
      s_e[threadIdx.x] = c;
      x = (c.len + kHugeChunk - 1) / kHugeChunk;
    }
#pragma unroll
    for (int o = 1; o < kWarp; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == kWarp - 1) s_w[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int64_t t = lane < nw ? s_w[lane] : 0;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      if (lane < nw) s_w[lane] = t;
    }
    __syncthreads();
    if (wid > 0) x += s_w[wid - 1];
    s_end[threadIdx.x] = x;
    __syncthreads();
    const int64_t total = s_end[blockDim.x - 1];
    const int last = (int)min((int64_t)blockDim.x, n - base) - 1;
    for (int64_t j = ((int64_t)blockIdx.x - gchunk % G + G) % G; j < total; j += G) {
      int lo = 0, hi = last;  // first entry whose prefix end exceeds j
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_end[mid] > j) hi = mid; else lo = mid + 1;
      }
      const EtwcEntry c = s_e[lo];
      const int64_t first = s_end[lo] - (c.len + kHugeChunk - 1) / kHugeChunk;
      const int64_t clo = c.lo + (j - first) * kHugeChunk;
      push_range_strided(b, c.u, clo, min(clo + kHugeChunk, c.hi()), threadIdx.x, blockDim.x);
      if (stage) {  // CTA-uniform: j depends on blockIdx only
        __syncthreads();
        const unsigned long long m = st->n;
        if (m) {
          if (threadIdx.x == 0) st->base = atomicAdd(a.out.qcount, m);
          __syncthreads();
          for (unsigned long long i = threadIdx.x; i < m; i += blockDim.x) a.out.queue[st->base + i] = st->q[i];
          __syncthreads();
          if (threadIdx.x == 0) st->n = 0;
        }
        __syncthreads();
      }
    }
    gchunk += total;
    __syncthreads();
  }
}
template <class Op, bool kStage = true>
__device__ __forceinline__ void b_push_huge(PushArgs<Op> a) {
  const int64_t n = (int64_t)*((volatile unsigned long long*)a.huge_n);
  push_ranges_chunked<Op, kStage>(a, n, [&](int64_t i) { return a.huge[i]; });
}
template <class Op>
__global__ void __launch_bounds__(256) k_push_huge(PushArgs<Op> a) {
  b_push_huge<Op>(a);
}
template <class Op, int kMinB>
__global__ void __launch_bounds__(256, kMinB) k_push_huge_mb(PushArgs<Op> a) {
  b_push_huge<Op>(a);
}

// Thread stage of ETWC for batched ops (CC hook, BC forward): the Q0 ranges
// (each < 32 arcs, one per vertex) are concatenated and every thread takes an
// equal contiguous share of their arcs, 4 at a time (push4u: one source per
// arc), instead of one range per thread -- a thread with a 31-arc remainder
// no longer holds its CTA at the chunk barrier (barrier stalls were 21% of
// the CC hook round).  Which thread walks which arc is not observable.
#ifndef GG_ETWC_BALANCED_T0
#define GG_ETWC_BALANCED_T0 1
#endif
constexpr bool kEtwcBalancedT0 = GG_ETWC_BALANCED_T0 != 0;
template <class Op>
__device__ __forceinline__ void etwc_stage0_balanced(const PushArgs<Op>& a, const EtwcEntry* q, int n) {
  __shared__ int32_t s_ex[257];  // exclusive prefix of the ranges' lengths; s_ex[n] = total
  __shared__ int32_t s_wsum[32];
  const int t = threadIdx.x, lane = lane_id(), wid = t >> 5;
  int32_t len = t < n ? q[t].len : 0;
  int32_t x = len;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[wid] = x;
  __syncthreads();
  int32_t off = 0;
  for (int w = 0; w < wid; ++w) off += s_wsum[w];
  if (t < n) s_ex[t] = off + x - len;
  if (t == n - 1) s_ex[n] = off + x;
  if (n == 0 && t == 0) s_ex[0] = 0;
  __syncthreads();
  const int32_t T = s_ex[n];
  const int32_t j0 = (int32_t)((int64_t)T * t / blockDim.x), j1 = (int32_t)((int64_t)T * (t + 1) / blockDim.x);
  if (j0 >= j1) return;
  int lo = 0, hi = n;  // entry holding arc j0: last k with s_ex[k] <= j0
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_ex[mid] <= j0) lo = mid; else hi = mid;
  }
  int k = lo;
  int32_t kend = s_ex[k + 1];
  for (int32_t j = j0; j < j1; j += 4) {
    int32_t u[4], v[4];
    unsigned live = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int32_t jj = j + b;
      u[b] = 0;
      v[b] = 0;
      if (jj < j1) {
        while (jj >= kend) {
          ++k;
          kend = s_ex[k + 1];
        }
        const EtwcEntry& c = q[k];
        u[b] = c.u;
        v[b] = __ldg(a.g.nbr + c.lo + (jj - (kend - c.len)));
        live |= 1u << b;
      }
    }
    a.op.push4u(u, v, live, a.use_filter, a.out);
  }
}

template <class Op>
__device__ __forceinline__ void b_push_etwc(PushArgs<Op> a, int cta) {
  __shared__ EtwcEntry s_q[3][256];
  __shared__ int s_n[3];
  const int64_t n = active_count(a.in, a.g.V);
  const int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t sc = 0;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < 3) s_n[threadIdx.x] = 0;
    __syncthreads();
    int64_t i = base + threadIdx.x;
    int64_t start = 0, end = 0;
    int32_t u = -1;
    if (i < n) {
      u = active_at(a.in, i);
      start = __ldg(a.g.off + u);
      end = __ldg(a.g.off + u + 1);
    }
    int64_t size = end - start;
    sc += size;
    const EtwcSizes sz = etwc_sizes(size, cta);
    int64_t e2 = sz.e2, e1 = sz.e1, e0 = sz.e0;
    EtwcEntry c2{start, (int32_t)e2, u}, c1{start + e2, (int32_t)e1, u},
        c0{start + e2 + e1, (int32_t)e0, u};
    if (a.huge && e2 >= a.huge_min) {  // whole-grid pass after this kernel / phase
      a.huge[atomicAdd(a.huge_n, 1ULL)] = c2;
      e2 = 0;
    }
    // small frontier (huge_min lowered to the CTA size): the warp-stage
    // ranges go to the grid pass as well -- a few hundred frontier vertices
    // fill one CTA, whose 8 warps otherwise walk every vertex's warp stage
    // (a 246-vertex RMAT-24 BFS level: 328 us in that one CTA)
    if (a.huge && a.huge_min <= cta && e1 > 0) {
      a.huge[atomicAdd(a.huge_n, 1ULL)] = c1;
      e1 = 0;
    }
    bool has[3] = {e0 > 0, e1 > 0, e2 > 0};
    const EtwcEntry* ent[3] = {&c0, &c1, &c2};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      unsigned b = __ballot_sync(0xffffffffu, has[q]);
      int slot = 0;
      if (lane == 0 && b) slot = atomicAdd(&s_n[q], __popc(b));
      slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(b & ((1u << lane) - 1));
      if (has[q]) s_q[q][slot] = *ent[q];
    }
    __syncthreads();
    // stage 0: individual threads
    if constexpr (PushBatch<Op>::value) {
      if (kEtwcBalancedT0) {
        etwc_stage0_balanced(a, s_q[0], s_n[0]);
      } else {
        for (int k = threadIdx.x; k < s_n[0]; k += blockDim.x) {
          EtwcEntry c = s_q[0][k];
          push_range_strided(a, c.u, c.lo, c.hi(), 0, 1, false);
        }
      }
    } else {
      for (int k = threadIdx.x; k < s_n[0]; k += blockDim.x) {
        EtwcEntry c = s_q[0][k];
        push_range_strided(a, c.u, c.lo, c.hi(), 0, 1, false);
      }
    }
    // stage 1: warps
    for (int k = wid; k < s_n[1]; k += nw) {
      EtwcEntry c = s_q[1][k];
      push_range_strided(a, c.u, c.lo, c.hi(), lane, kWarp);
    }
    // stage 2: whole CTA
    for (int k = 0; k < s_n[2]; ++k) {
      EtwcEntry c = s_q[2][k];
      push_range_strided(a, c.u, c.lo, c.hi(), threadIdx.x, blockDim.x);
    }
    __syncthreads();
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_push_etwc(PushArgs<Op> a, int cta) {
  b_push_etwc<Op>(a, cta);
}
template <class Op, int kMinB>
__global__ void __launch_bounds__(256, kMinB) k_push_etwc_mb(PushArgs<Op> a, int cta) {
  b_push_etwc<Op>(a, cta);
}

// ===========================================================================
// PULL (engine.py:506-555): per destination passing the filter, scan in-edges,
// test source membership, udf with owner-write rights.  The op reduces over a
// destination's in-edges into an accumulator (register/shuffle/shared), and
// finishes with one owner write.
// ===========================================================================
template <class Op>
struct PullArgs {
  CsrView g;  // CSR-in
  InView in;  // membership (dense) or all
  Op op;
  OutBuilder out;
  int use_filter;
  unsigned long long* scanned;
};

template <class Op>
__device__ __forceinline__ bool pull_visit(const PullArgs<Op>& a, typename Op::Acc& acc,
                                           int32_t v, int64_t e) {
  int32_t u = __ldg(a.g.nbr + e);
  if (!a.in.member(u)) return false;
  uint32_t w = a.g.w ? __ldg(a.g.w + e) : 0u;
  return a.op.visit(acc, v, u, w);
}

// VERTEX_BASED: thread per destination (early exit when the op says so).
// (A two-phase variant -- per-thread probe of the first two in-arcs, then
// warp-cooperative scans of the unsettled destinations -- measured 3x slower
// on the first RMAT-24 bottom-up level: 1.52 vs 0.52 ms.)
#ifndef GG_PULL_K
#define GG_PULL_K 2
#endif
constexpr int kPullK = GG_PULL_K;  // bottom-up destinations per thread in lock step
template <class Op>
__device__ __forceinline__ void b_pull_vb(PullArgs<Op> a) {
  if constexpr (Op::kEarlyExit) {
    // early-exit ops: kPullK destinations per thread, probed in lock step, so
    // each thread keeps kPullK independent in-list walks (neighbour id, then
    // frontier bit) in flight -- the kernel is latency-bound
    int64_t sc = 0;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < a.g.V; v0 += kPullK * nth) {
      bool act[kPullK], done[kPullK];
      int64_t e[kPullK], h[kPullK];
      typename Op::Acc acc[kPullK];
#pragma unroll
      for (int k = 0; k < kPullK; ++k) {
        const int64_t v = v0 + k * nth;
        act[k] = v < a.g.V && (!a.use_filter || a.op.filter((int32_t)v));
        e[k] = 0;
        h[k] = 0;
        if (act[k]) {
          e[k] = __ldg(a.g.off + v);
          h[k] = __ldg(a.g.off + v + 1);
          sc += h[k] - e[k];
        }
        acc[k] = a.op.init();
        done[k] = e[k] >= h[k];
      }
      while (true) {
        bool any = false;
#pragma unroll
        for (int k = 0; k < kPullK; ++k) any |= !done[k];
        if (!any) break;
        int32_t u[kPullK];
#pragma unroll
        for (int k = 0; k < kPullK; ++k) u[k] = done[k] ? 0 : __ldg(a.g.nbr + e[k]);
        bool m[kPullK];
#pragma unroll
        for (int k = 0; k < kPullK; ++k) m[k] = !done[k] && a.in.member(u[k]);
#pragma unroll
        for (int k = 0; k < kPullK; ++k) {
          if (done[k]) continue;
          const uint32_t w = a.g.w ? __ldg(a.g.w + e[k]) : 0u;
          if ((m[k] && a.op.visit(acc[k], (int32_t)(v0 + k * nth), u[k], w)) || ++e[k] >= h[k]) done[k] = true;
        }
      }
#pragma unroll
      for (int k = 0; k < kPullK; ++k)
        if (act[k]) a.op.finish((int32_t)(v0 + k * nth), acc[k], a.out);
    }
    add_scanned(a.scanned, sc);
    return;
  }
  int64_t sc = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < a.g.V;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (a.use_filter && !a.op.filter((int32_t)v)) continue;
    int64_t lo = __ldg(a.g.off + v), hi = __ldg(a.g.off + v + 1);
    sc += hi - lo;
    typename Op::Acc acc = a.op.init();
    for (int64_t e = lo; e < hi; ++e)
      if (pull_visit(a, acc, (int32_t)v, e)) break;
    a.op.finish((int32_t)v, acc, a.out);
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_pull_vb(PullArgs<Op> a) {
  b_pull_vb<Op>(a);
}

// Warp-cooperative reduction of one destination's in-range [lo, hi).
template <class Op>
__device__ __forceinline__ typename Op::Acc pull_warp_range(const PullArgs<Op>& a, int32_t v,
                                                            int64_t lo, int64_t hi) {
  typename Op::Acc acc = a.op.init();
  for (int64_t e0 = lo; e0 < hi; e0 += kWarp) {
    bool stop = false;
    if (e0 + lane_id() < hi) stop = pull_visit(a, acc, v, e0 + lane_id());
    if (Op::kEarlyExit && __any_sync(0xffffffffu, stop)) break;
  }
  return Op::warp_reduce(acc);
}

// WM: warps take contiguous destination chunks; each destination's in-list
// is reduced by the whole warp.
template <class Op>
__device__ __forceinline__ void b_pull_wm(PullArgs<Op> a) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t chunk = (a.g.V + nwarps - 1) / nwarps;
  int64_t sc = 0;
  for (int64_t v = warp * chunk; v < min(a.g.V, (warp + 1) * chunk); ++v) {
    if (a.use_filter && !a.op.filter((int32_t)v)) continue;
    int64_t lo = __ldg(a.g.off + v), hi = __ldg(a.g.off + v + 1);
    if (lane_id() == 0) sc += hi - lo;
    typename Op::Acc acc = pull_warp_range(a, (int32_t)v, lo, hi);
    if (lane_id() == 0) a.op.finish((int32_t)v, acc, a.out);
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_pull_wm(PullArgs<Op> a) {
  b_pull_wm<Op>(a);
}

// Block-wide reduction helper (accumulators are tiny PODs).
template <class Op>
__device__ __forceinline__ typename Op::Acc block_reduce(typename Op::Acc acc) {
  __shared__ typename Op::Acc s_part[32];
  acc = Op::warp_reduce(acc);
  const int wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane_id() == 0) s_part[wid] = acc;
  __syncthreads();
  typename Op::Acc r = s_part[0];
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = Op::combine(r, s_part[k]);
  return r;
}

// CM: CTAs take contiguous destination chunks (engine.py:160-164, even
// split, earlier chunks take the extra); inside its chunk a CTA's threads own
// destinations cyclically, each reducing its in-list with early exit.
template <class Op>
__device__ __forceinline__ void b_pull_cm(PullArgs<Op> a) {
  const int64_t V = a.g.V;
  const int64_t base = V / gridDim.x, extra = V % gridDim.x;
  const int64_t b = blockIdx.x;
  const int64_t start = b * base + min(b, extra);
  const int64_t end = start + base + (b < extra ? 1 : 0);
  int64_t sc = 0;
  for (int64_t v = start + threadIdx.x; v < end; v += blockDim.x) {
    if (a.use_filter && !a.op.filter((int32_t)v)) continue;
    int64_t lo = __ldg(a.g.off + v), hi = __ldg(a.g.off + v + 1);
    sc += hi - lo;
    typename Op::Acc acc = a.op.init();
    for (int64_t e = lo; e < hi; ++e)
      if (pull_visit(a, acc, (int32_t)v, e)) break;
    a.op.finish((int32_t)v, acc, a.out);
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_pull_cm(PullArgs<Op> a) {
  b_pull_cm<Op>(a);
}

// STRICT (engine.py:216-225): edge-balanced destination spans snapped to
// vertex boundaries (each destination keeps one owner).  `span_start[t]` is
// the first destination of span t (length nspans+1), computed on the device.
template <class Op>
__device__ __forceinline__ void b_pull_strict(PullArgs<Op> a, const int64_t* span_start,
                                                     int64_t nspans) {
  // one warp per span; its lanes own the span's destinations cyclically
  int64_t sc = 0;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < nspans; t += nw) {
    for (int64_t v = span_start[t] + lane_id(); v < span_start[t + 1]; v += kWarp) {
      if (a.use_filter && !a.op.filter((int32_t)v)) continue;
      int64_t lo = __ldg(a.g.off + v), hi = __ldg(a.g.off + v + 1);
      sc += hi - lo;
      typename Op::Acc acc = a.op.init();
      for (int64_t e = lo; e < hi; ++e)
        if (pull_visit(a, acc, (int32_t)v, e)) break;
      a.op.finish((int32_t)v, acc, a.out);
    }
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_pull_strict(PullArgs<Op> a, const int64_t* span_start,
                                                     int64_t nspans) {
  b_pull_strict<Op>(a, span_start, nspans);
}

// TWC pull (engine.py:249-251): destinations binned by in-degree; the three
// consumers reuse thread / warp / CTA reduction.
template <class Op>
__device__ __forceinline__ void b_pull_twc_bin(PullArgs<Op> a, TwcQueues q, int cta) {
  int64_t sc = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < a.g.V;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (a.use_filter && !a.op.filter((int32_t)v)) continue;
    int64_t deg = __ldg(a.g.off + v + 1) - __ldg(a.g.off + v);
    sc += deg;
    int b = twc_bin_of(deg, cta);
    cg::coalesced_group g = cg::coalesced_threads();
    cg::coalesced_group gb = cg::labeled_partition(g, b);
    unsigned long long base = 0;
    if (gb.thread_rank() == 0) base = atomicAdd(q.cnt + b, (unsigned long long)gb.size());
    base = gb.shfl(base, 0);
    q.q[b][base + gb.thread_rank()] = (int32_t)v;
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_pull_twc_bin(PullArgs<Op> a, TwcQueues q, int cta) {
  b_pull_twc_bin<Op>(a, q, cta);
}

template <class Op>
__device__ __forceinline__ void b_pull_twc_thread(PullArgs<Op> a, const int32_t* qv,
                                                         const unsigned long long* cnt) {
  const int64_t n = (int64_t)*cnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = qv[i];
    int64_t lo = __ldg(a.g.off + v), hi = __ldg(a.g.off + v + 1);
    typename Op::Acc acc = a.op.init();
    for (int64_t e = lo; e < hi; ++e)
      if (pull_visit(a, acc, v, e)) break;
    a.op.finish(v, acc, a.out);
  }
}
template <class Op>
__global__ void __launch_bounds__(256) k_pull_twc_thread(PullArgs<Op> a, const int32_t* qv,
                                                         const unsigned long long* cnt) {
  b_pull_twc_thread<Op>(a, qv, cnt);
}

template <class Op>
__device__ __forceinline__ void b_pull_twc_warp(PullArgs<Op> a, const int32_t* qv,
                                                       const unsigned long long* cnt) {
  const int64_t n = (int64_t)*cnt;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    int32_t v = qv[i];
    typename Op::Acc acc = pull_warp_range(a, v, __ldg(a.g.off + v), __ldg(a.g.off + v + 1));
    if (lane_id() == 0) a.op.finish(v, acc, a.out);
  }
}
template <class Op>
__global__ void __launch_bounds__(256) k_pull_twc_warp(PullArgs<Op> a, const int32_t* qv,
                                                       const unsigned long long* cnt) {
  b_pull_twc_warp<Op>(a, qv, cnt);
}

template <class Op>
__device__ __forceinline__ void b_pull_twc_cta(PullArgs<Op> a, const int32_t* qv,
                                                      const unsigned long long* cnt) {
  const int64_t n = (int64_t)*cnt;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    int32_t v = qv[i];
    int64_t lo = __ldg(a.g.off + v), hi = __ldg(a.g.off + v + 1);
    typename Op::Acc acc = a.op.init();
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) pull_visit(a, acc, v, e);
    acc = block_reduce<Op>(acc);
    if (threadIdx.x == 0) a.op.finish(v, acc, a.out);
  }
}
template <class Op>
__global__ void __launch_bounds__(256) k_pull_twc_cta(PullArgs<Op> a, const int32_t* qv,
                                                      const unsigned long long* cnt) {
  b_pull_twc_cta<Op>(a, qv, cnt);
}

// ETWC pull (engine.py:252-255): chunked in-ranges stay inside one CTA.  Each
// destination contributes at most one entry per stage; stage partials are
// kept per destination slot in shared memory and combined by the owner
// thread, which then performs the single owner write.
template <class Op>
__device__ __forceinline__ void b_pull_etwc(PullArgs<Op> a, int cta) {
  __shared__ EtwcEntry s_q[3][256];
  __shared__ int s_slot[3][256];  // queue entry -> destination slot
  __shared__ typename Op::Acc s_part[3][256];
  __shared__ int s_n[3];
  const int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t sc = 0;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < a.g.V;
       base += (int64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < 3) s_n[threadIdx.x] = 0;
    const typename Op::Acc zero = a.op.init();
    for (int q = 0; q < 3; ++q) s_part[q][threadIdx.x] = zero;
    __syncthreads();
    int64_t v = base + threadIdx.x;
    bool keep = v < a.g.V && (!a.use_filter || a.op.filter((int32_t)v));
    int64_t start = 0, end = 0;
    if (keep) {
      start = __ldg(a.g.off + v);
      end = __ldg(a.g.off + v + 1);
    }
    int64_t size = end - start;
    sc += size;
    const EtwcSizes sz = etwc_sizes(size, cta);
    int64_t e2 = sz.e2, e1 = sz.e1, e0 = sz.e0;
    EtwcEntry c[3] = {{start + e2 + e1, (int32_t)e0, (int32_t)v}, {start + e2, (int32_t)e1, (int32_t)v},
                      {start, (int32_t)e2, (int32_t)v}};
    bool has[3] = {e0 > 0, e1 > 0, e2 > 0};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      unsigned b = __ballot_sync(0xffffffffu, has[q]);
      int slot = 0;
      if (lane == 0 && b) slot = atomicAdd(&s_n[q], __popc(b));
      slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(b & ((1u << lane) - 1));
      if (has[q]) {
        s_q[q][slot] = c[q];
        s_slot[q][slot] = threadIdx.x;
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < s_n[0]; k += blockDim.x) {
      EtwcEntry ce = s_q[0][k];
      typename Op::Acc acc = a.op.init();
      for (int64_t e = ce.lo; e < ce.hi(); ++e)
        if (pull_visit(a, acc, ce.u, e)) break;
      s_part[0][s_slot[0][k]] = acc;
    }
    for (int k = wid; k < s_n[1]; k += nw) {
      EtwcEntry ce = s_q[1][k];
      typename Op::Acc acc = pull_warp_range(a, ce.u, ce.lo, ce.hi());
      if (lane == 0) s_part[1][s_slot[1][k]] = acc;
    }
    for (int k = 0; k < s_n[2]; ++k) {
      EtwcEntry ce = s_q[2][k];
      typename Op::Acc acc = a.op.init();
      for (int64_t e = ce.lo + threadIdx.x; e < ce.hi(); e += blockDim.x) pull_visit(a, acc, ce.u, e);
      acc = block_reduce<Op>(acc);
      if (threadIdx.x == 0) s_part[2][s_slot[2][k]] = acc;
    }
    __syncthreads();
    if (keep) {
      typename Op::Acc acc =
          Op::combine(Op::combine(s_part[0][threadIdx.x], s_part[1][threadIdx.x]), s_part[2][threadIdx.x]);
      a.op.finish((int32_t)v, acc, a.out);
    }
    __syncthreads();
  }
  add_scanned(a.scanned, sc);
}
template <class Op>
__global__ void __launch_bounds__(256) k_pull_etwc(PullArgs<Op> a, int cta) {
  b_pull_etwc<Op>(a, cta);
}

// ===========================================================================
// EDGE_ONLY (engine.py:558-608): flat COO, source membership + dst filter per
// arc, always the atomic interface.  Vectorised 16-byte loads of src/dst.
// ===========================================================================
template <class Op>
struct EdgeArgs {
  CooView coo;
  InView in;  // dense membership or all
  Op op;
  OutBuilder out;
  int use_filter;
};

template <class Op>
__device__ __forceinline__ void edge_one(const EdgeArgs<Op>& a, int32_t u, int32_t v, int64_t e) {
  if (!a.in.member(u)) return;
  if (a.use_filter && !a.op.filter(v)) return;
  uint32_t w = a.coo.w ? __ldg(a.coo.w + e) : 0u;
  a.op.push(u, v, w, a.out);
}

template <class Op>
__device__ __forceinline__ void edge_range(const EdgeArgs<Op>& a, int64_t lo, int64_t hi,
                                           int64_t tid, int64_t nthreads) {
  // scalar head until 16-byte alignment of both arrays, vector body, tail
  int64_t head = lo;
  while (head < hi && (((uintptr_t)(a.coo.src + head)) & 15)) ++head;
  if (((uintptr_t)(a.coo.dst + head) & 15) != 0) head = hi;  // misaligned pair: scalar
  for (int64_t e = lo + tid; e < head; e += nthreads)
    edge_one(a, __ldg(a.coo.src + e), __ldg(a.coo.dst + e), e);
  int64_t nvec = (hi - head) >> 2;
  const int4* s4 = reinterpret_cast<const int4*>(a.coo.src + head);
  const int4* d4 = reinterpret_cast<const int4*>(a.coo.dst + head);
  for (int64_t k = tid; k < nvec; k += nthreads) {
    int4 s = ld_stream4(s4 + k), d = ld_stream4(d4 + k);
    int64_t e = head + 4 * k;
    if constexpr (PushBatch<Op>::value) {  // the 4 arcs' chains in flight together
      const int32_t uu[4] = {s.x, s.y, s.z, s.w}, vv[4] = {d.x, d.y, d.z, d.w};
      unsigned live = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (a.in.member(uu[q])) live |= 1u << q;
      a.op.push4u(uu, vv, live, a.use_filter, a.out);
    } else {
      edge_one(a, s.x, d.x, e);
      edge_one(a, s.y, d.y, e + 1);
      edge_one(a, s.z, d.z, e + 2);
      edge_one(a, s.w, d.w, e + 3);
    }
  }
  for (int64_t e = head + 4 * nvec + tid; e < hi; e += nthreads)
    edge_one(a, __ldg(a.coo.src + e), __ldg(a.coo.dst + e), e);
}

template <class Op>
__device__ __forceinline__ void b_edge_only(EdgeArgs<Op> a) {
  edge_range(a, 0, a.coo.E, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
             (int64_t)gridDim.x * blockDim.x);
}
template <class Op>
__global__ void __launch_bounds__(256) k_edge_only(EdgeArgs<Op> a) {
  b_edge_only<Op>(a);
}
template <class Op, int kMinB>
__global__ void __launch_bounds__(256, kMinB) k_edge_only_mb(EdgeArgs<Op> a) {
  b_edge_only<Op>(a);
}

// EdgeBlocking Alg. 2 (blocking.py:116-186): segments in order, the whole
// grid cooperates on one segment, grid barrier between segments.  Launched
// cooperatively (one dispatch).
template <class Op>
__device__ __forceinline__ void b_edge_blocked(EdgeArgs<Op> a, const int64_t* seg_end,
                                                      int64_t nseg) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  int64_t lo = 0;
  for (int64_t s = 0; s < nseg; ++s) {
    int64_t hi = seg_end[s];
    edge_range(a, lo, hi, tid, nthreads);
    lo = hi;
    grid.sync();
  }
}
template <class Op>
__global__ void __launch_bounds__(256) k_edge_blocked(EdgeArgs<Op> a, const int64_t* seg_end,
                                                      int64_t nseg) {
  b_edge_blocked<Op>(a, seg_end, nseg);
}
template <class Op, int kMinB>
__global__ void __launch_bounds__(256, kMinB) k_edge_blocked_mb(EdgeArgs<Op> a, const int64_t* seg_end,
                                                                int64_t nseg) {
  b_edge_blocked<Op>(a, seg_end, nseg);
}

}  // namespace gg
