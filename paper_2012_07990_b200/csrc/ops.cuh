// ops.cuh — named device UDFs.  The reference runs an arbitrary Python
// callable per edge through EdgeContext (runtime.py:299-362); a GPU cannot,
// so every UDF the reference's algorithms and tests use is a functor here
// (SURVEY §7 hard part 1).  Each functor provides
//   filter(v)                       to_filter of the algorithm
//   push(u, v, w, out)              atomic interface (PUSH / EDGE_ONLY)
//   Acc init / visit / combine / finish   owner-write interface (PULL)
#pragma once
#include "traverse.cuh"

namespace gg {

// Ops whose push emits a destination only on winning a CAS on its state
// (at most once per vertex per apply): their SPARSE output never exceeds V,
// whatever the input multiplicity.  Every other op may emit once per scanned
// arc, so a multiset input can need more than max(V, E) + 1 output slots.
template <class Op>
struct EmitsOncePerVertex { static constexpr bool value = false; };

template <class T>
__device__ __forceinline__ T shfl_xor_any(T v, int o) {
  return __shfl_xor_sync(0xffffffffu, v, o);
}

// BFS (algos.py:114-125): parent CAS in push; plain owner store in pull.
struct OpBfs {
  int32_t* parent;
  using Acc = int32_t;
  static constexpr bool kEarlyExit = true;
  __device__ __forceinline__ bool filter(int32_t v) const {
    return *((volatile int32_t*)parent + v) == -1;
  }
  __device__ __forceinline__ void push(int32_t u, int32_t v, uint32_t, const OutBuilder& out) const {
    if (atomicCAS(parent + v, -1, u) == -1) out.emit(v);
  }
  __device__ __forceinline__ Acc init() const { return -1; }
  __device__ __forceinline__ bool visit(Acc& acc, int32_t, int32_t u, uint32_t) const {
    if (acc == -1) acc = u;
    return true;  // the first frontier in-neighbour settles v (algos.py:121-125)
  }
  static __device__ __forceinline__ Acc combine(Acc a, Acc b) { return a != -1 ? a : b; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = combine(a, shfl_xor_any(a, o));
    return a;
  }
  __device__ __forceinline__ void finish(int32_t v, const Acc& acc, const OutBuilder& out) const {
    if (acc != -1 && parent[v] == -1) {
      parent[v] = acc;
      out.emit(v);
    }
  }
};

template <>
struct EmitsOncePerVertex<OpBfs> { static constexpr bool value = true; };

// Test UDF: in-degree counting from the active set (test_engine.py:246-264).
struct OpCount {
  unsigned long long* counts;
  using Acc = unsigned long long;
  static constexpr bool kEarlyExit = false;
  __device__ __forceinline__ bool filter(int32_t) const { return true; }
  __device__ __forceinline__ void push(int32_t, int32_t v, uint32_t, const OutBuilder&) const {
    atomicAdd(counts + v, 1ULL);
  }
  __device__ __forceinline__ Acc init() const { return 0; }
  __device__ __forceinline__ bool visit(Acc& acc, int32_t, int32_t, uint32_t) const { ++acc; return false; }
  static __device__ __forceinline__ Acc combine(Acc a, Acc b) { return a + b; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) { return warp_sum(a); }
  __device__ __forceinline__ void finish(int32_t v, const Acc& acc, const OutBuilder&) const {
    if (acc) counts[v] += acc;
  }
};

// Test UDF: ctx.enqueue(ctx.dst) with no guard (test_engine.py:384-399);
// pull enqueues once per member in-edge, like the reference's owner loop.
struct OpEnqueue {
  using Acc = unsigned long long;
  static constexpr bool kEarlyExit = false;
  __device__ __forceinline__ bool filter(int32_t) const { return true; }
  __device__ __forceinline__ void push(int32_t, int32_t v, uint32_t, const OutBuilder& out) const {
    out.emit(v);
  }
  __device__ __forceinline__ Acc init() const { return 0; }
  __device__ __forceinline__ bool visit(Acc& acc, int32_t, int32_t, uint32_t) const { ++acc; return false; }
  static __device__ __forceinline__ Acc combine(Acc a, Acc b) { return a + b; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) { return warp_sum(a); }
  __device__ __forceinline__ void finish(int32_t v, const Acc& acc, const OutBuilder& out) const {
    for (unsigned long long k = 0; k < acc; ++k) out.emit(v);
  }
};

// PageRank gather (algos.py:180-181): acc[dst] += contrib[src].
template <class CT>
struct OpPr {
  double* acc;
  const CT* contrib;
  using Acc = double;
  static constexpr bool kEarlyExit = false;
  __device__ __forceinline__ bool filter(int32_t) const { return true; }
  __device__ __forceinline__ void push(int32_t u, int32_t v, uint32_t, const OutBuilder&) const {
    atomicAdd(acc + v, (double)__ldg(contrib + u));
  }
  __device__ __forceinline__ Acc init() const { return 0.0; }
  __device__ __forceinline__ bool visit(Acc& a, int32_t, int32_t u, uint32_t) const {
    a += (double)__ldg(contrib + u);
    return false;
  }
  static __device__ __forceinline__ Acc combine(Acc a, Acc b) { return a + b; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) { return warp_sum(a); }
  __device__ __forceinline__ void finish(int32_t v, const Acc& a, const OutBuilder&) const {
    if (a != 0.0) acc[v] += a;
  }
};

// Connected-components hook (algos.py:283-293): atomic_min(label, hi, lo) on
// the larger *label* (not the vertex); any direction uses the atomic form.
struct OpHook {
  int32_t* label;
  int* changed;
  // optional (cc_run): bit v set iff label[v] was the giant component's root
  // label when the round started; an arc between two such vertices joins
  // one tree to itself, so its two random label reads are skipped (an
  // L2-resident bit test instead: most arcs after the first round)
  const uint32_t* giant = nullptr;
  // root shortcut: when the larger label is the random endpoint v's own id
  // (label[v] == v, just read), label[hi] is known to be hi > lo, so the
  // re-read before the atomic is skipped (one L2 request per arc less in
  // the first round, where most vertices are still roots).  Not applied to
  // u: lanes of a warp share u, so its re-read is one coalesced request,
  // while one atomic per lane on a hub's label would serialise.
  bool root_skip = false;
  static constexpr bool kPush4 = true;
  static constexpr int kMinBlocks = 8;  // 32 registers: full residency (latency-bound chains)
  using Acc = int;
  static constexpr bool kEarlyExit = false;
  __device__ __forceinline__ bool filter(int32_t) const { return true; }
  __device__ __forceinline__ void hook(int32_t u, int32_t v) const {
    if (giant && ((__ldg(giant + (u >> 5)) >> (u & 31)) & (__ldg(giant + (v >> 5)) >> (v & 31)) & 1u)) return;
    int32_t la = *((volatile int32_t*)label + u), lb = *((volatile int32_t*)label + v);
    if (la == lb) return;
    int32_t lo = la < lb ? la : lb, hi = la < lb ? lb : la;
    // skip hooks that cannot lower label[hi] (hub roots receive one hook per
    // incident arc; only the smaller ones need the atomic)
    if (!(root_skip && hi == v && lb == v) && lo >= *((volatile int32_t*)label + hi)) return;
    // read before write: one hot flag line, written once per round instead of
    // once per successful hook (which serialises at its L2 slice)
    if (atomicMin(label + hi, lo) > lo && !*((volatile int*)changed)) *changed = 1;
  }
  __device__ __forceinline__ void push(int32_t u, int32_t v, uint32_t, const OutBuilder&) const {
    hook(u, v);
  }
  // hook() for 4 arcs of one source: the same tests and atomic per arc, with
  // each step's 4 loads issued together (label[u] read once per batch)
  __device__ __forceinline__ void push4(int32_t u, const int32_t (&v)[4], unsigned live, int,
                                        const OutBuilder&) const {  // filter(): always true
    if (giant && ((__ldg(giant + (u >> 5)) >> (u & 31)) & 1u)) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (((live >> k) & 1u) && ((__ldg(giant + (v[k] >> 5)) >> (v[k] & 31)) & 1u)) live &= ~(1u << k);
    }
    if (!live) return;
    const int32_t la = *((volatile int32_t*)label + u);
    int32_t lb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) lb[k] = ((live >> k) & 1u) ? *((volatile int32_t*)label + v[k]) : la;
    int32_t lo[4], hi[4], cur[4];
    unsigned need = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      lo[k] = la < lb[k] ? la : lb[k];
      hi[k] = la < lb[k] ? lb[k] : la;
      if (lb[k] != la) need |= 1u << k;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool known_root = root_skip && hi[k] == v[k] && lb[k] == v[k];
      cur[k] = ((need >> k) & 1u) && !known_root ? *((volatile int32_t*)label + hi[k]) : INT32_MAX;
    }
    bool any = false;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((need >> k) & 1u) && lo[k] < cur[k]) any |= atomicMin(label + hi[k], lo[k]) > lo[k];
    if (any && !*((volatile int*)changed)) *changed = 1;
  }
  // the same for 4 arcs with their own sources (ETWC's balanced thread stage)
  __device__ __forceinline__ void push4u(const int32_t (&u)[4], const int32_t (&v)[4], unsigned live, int,
                                         const OutBuilder&) const {
    if (giant) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (((live >> k) & 1u) && ((__ldg(giant + (u[k] >> 5)) >> (u[k] & 31)) & 1u) &&
            ((__ldg(giant + (v[k] >> 5)) >> (v[k] & 31)) & 1u))
          live &= ~(1u << k);
    }
    if (!live) return;
    int32_t la[4], lb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool l = (live >> k) & 1u;
      la[k] = l ? *((volatile int32_t*)label + u[k]) : 0;
      lb[k] = l ? *((volatile int32_t*)label + v[k]) : 0;
    }
    int32_t lo[4], hi[4], cur[4];
    unsigned need = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      lo[k] = la[k] < lb[k] ? la[k] : lb[k];
      hi[k] = la[k] < lb[k] ? lb[k] : la[k];
      if (((live >> k) & 1u) && lb[k] != la[k]) need |= 1u << k;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool known_root = root_skip && hi[k] == v[k] && lb[k] == v[k];
      cur[k] = ((need >> k) & 1u) && !known_root ? *((volatile int32_t*)label + hi[k]) : INT32_MAX;
    }
    bool any = false;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((need >> k) & 1u) && lo[k] < cur[k]) any |= atomicMin(label + hi[k], lo[k]) > lo[k];
    if (any && !*((volatile int*)changed)) *changed = 1;
  }
  __device__ __forceinline__ Acc init() const { return 0; }
  __device__ __forceinline__ bool visit(Acc&, int32_t v, int32_t u, uint32_t) const {
    hook(u, v);
    return false;
  }
  static __device__ __forceinline__ Acc combine(Acc a, Acc) { return a; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) { return a; }
  __device__ __forceinline__ void finish(int32_t, const Acc&, const OutBuilder&) const {}
};

// Delta-stepping relaxation (algos.py:233-234 -> BucketQueue.update_priority_min,
// priority.py:59-83): atomic min on the 64-bit priority; on improvement the
// vertex is enqueued (deduplicated) into the current bucket when its bucket
// equals the active index, else into far.  PUSH only (algos.py:226-227).
struct OpRelax {
  unsigned long long* dist;
  unsigned long long delta;
  unsigned long long index;
  OutBuilder cur;  // FUSED sparse + boolmap marks (per-round dedup)
  OutBuilder far;  // FUSED sparse + boolmap marks (persistent until advance)
  using Acc = int;
  static constexpr bool kEarlyExit = false;
  __device__ __forceinline__ bool filter(int32_t) const { return true; }
  __device__ __forceinline__ void push(int32_t u, int32_t v, uint32_t w, const OutBuilder&) const {
    unsigned long long du = *((volatile unsigned long long*)dist + u);
    unsigned long long cand = du + (unsigned long long)w;
    unsigned long long old = atomicMin(dist + v, cand);
    if (cand < old) {
      if (cand / delta == index) cur.emit(v);
      else far.emit(v);
    }
  }
  __device__ __forceinline__ Acc init() const { return 0; }
  __device__ __forceinline__ bool visit(Acc&, int32_t v, int32_t u, uint32_t w) const {
    push(u, v, w, cur);
    return false;
  }
  static __device__ __forceinline__ Acc combine(Acc a, Acc) { return a; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) { return a; }
  __device__ __forceinline__ void finish(int32_t, const Acc&, const OutBuilder&) const {}
};

// Betweenness forward round (algos.py:347-365).  depth int32, sigma f64
// (path counts; exact up to 2^53, the reference uses Python ints).
struct BcAcc {
  double s;
  int found;
};
struct OpBcFwd {
  int32_t* depth;
  double* sigma;
  int32_t level;
  using Acc = BcAcc;
  static constexpr bool kEarlyExit = false;
  __device__ __forceinline__ bool filter(int32_t v) const {
    int32_t d = *((volatile int32_t*)depth + v);
    return d == -1 || d == level + 1;
  }
  __device__ __forceinline__ void push(int32_t u, int32_t v, uint32_t, const OutBuilder& out) const {
    const int32_t nl = level + 1;
    // the CAS only when v looked unvisited (the filter admitted -1 or nl)
    if (*((volatile int32_t*)depth + v) == -1 && atomicCAS(depth + v, -1, nl) == -1) out.emit(v);
    if (*((volatile int32_t*)depth + v) == nl) atomicAdd(sigma + v, sigma[u]);
  }
  __device__ __forceinline__ Acc init() const { return {0.0, 0}; }
  __device__ __forceinline__ bool visit(Acc& a, int32_t, int32_t u, uint32_t) const {
    a.s += sigma[u];
    a.found = 1;
    return false;
  }
  static __device__ __forceinline__ Acc combine(Acc a, Acc b) { return {a.s + b.s, a.found | b.found}; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a.s += __shfl_xor_sync(0xffffffffu, a.s, o);
      a.found |= __shfl_xor_sync(0xffffffffu, a.found, o);
    }
    return a;
  }
  __device__ __forceinline__ void finish(int32_t v, const Acc& a, const OutBuilder& out) const {
    if (!a.found) return;
    if (depth[v] == -1) {
      depth[v] = level + 1;
      out.emit(v);
    }
    sigma[v] += a.s;
  }
};

// Betweenness backward round (algos.py:378-389), push only:
// delta[u] += sigma[u]/sigma[v] * (1 + delta[v]) when depth[v] == depth[u]+1.
struct OpBcBwd {
  const int32_t* depth;
  const double* sigma;
  double* delta;
  using Acc = int;
  static constexpr bool kEarlyExit = false;
  __device__ __forceinline__ bool filter(int32_t) const { return true; }
  __device__ __forceinline__ void push(int32_t u, int32_t v, uint32_t, const OutBuilder&) const {
    if (__ldg(depth + v) == __ldg(depth + u) + 1)
      atomicAdd(delta + u, __ldg(sigma + u) / __ldg(sigma + v) * (1.0 + delta[v]));
  }
  // range walks accumulate per source and commit once per warp (traverse.cuh)
  static constexpr bool kPushReduce = true;
  __device__ __forceinline__ double push_val(int32_t u, int32_t v) const {
    return __ldg(depth + v) == __ldg(depth + u) + 1 ? __ldg(sigma + u) / __ldg(sigma + v) * (1.0 + delta[v]) : 0.0;
  }
  __device__ __forceinline__ void push_commit(int32_t u, double x) const { atomicAdd(delta + u, x); }
  __device__ __forceinline__ Acc init() const { return 0; }
  __device__ __forceinline__ bool visit(Acc&, int32_t v, int32_t u, uint32_t w) const {
    push(u, v, w, OutBuilder{});
    return false;
  }
  static __device__ __forceinline__ Acc combine(Acc a, Acc) { return a; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) { return a; }
  __device__ __forceinline__ void finish(int32_t, const Acc&, const OutBuilder&) const {}
};

// The same two rounds over an array-of-structs state (bc_run's own layout):
// depth, sigma and delta of a vertex share one 32-byte sector, so the
// backward round's three random gathers per arc (depth[v], sigma[v],
// delta[v]) are one sector, and the forward round's depth test, CAS and
// sigma add hit one line.  The UDF boundary (gg_edgeset_apply) keeps the
// reference's separate arrays (OpBcFwd / OpBcBwd above).
struct __align__(32) BcState {
  double sigma;
  double delta;
  int32_t depth;
  int32_t pad[3];
};
// `vis`: bitmap of the vertices of levels 0..level (set between rounds); an
// arc into one of them is dropped with an L2-resident bit test instead of a
// random 32-byte state gather (the frontier's arcs mostly lead back).
__device__ __forceinline__ bool bm_has(const uint32_t* bm, int32_t v) {
  return (__ldg(bm + (v >> 5)) >> (v & 31)) & 1u;
}
struct OpBcFwdAoS {
  BcState* st;
  int32_t level;
  const uint32_t* vis;
  using Acc = BcAcc;
  static constexpr bool kEarlyExit = false;
  __device__ __forceinline__ bool filter(int32_t v) const {
    if (bm_has(vis, v)) return false;  // depth <= level: neither -1 nor level + 1
    const int32_t d = *((volatile int32_t*)&st[v].depth);
    return d == -1 || d == level + 1;
  }
  __device__ __forceinline__ void push(int32_t u, int32_t v, uint32_t, const OutBuilder& out) const {
    const int32_t nl = level + 1;
    if (*((volatile int32_t*)&st[v].depth) == -1 && atomicCAS(&st[v].depth, -1, nl) == -1) out.emit(v);
    if (*((volatile int32_t*)&st[v].depth) == nl) atomicAdd(&st[v].sigma, st[u].sigma);
  }
  // filter + push for 4 arcs of one source with each step's memory
  // operations issued together (bit tests, depth reads, CAS, sigma adds).
  // Only this round writes depths, all to level + 1, so after a CAS the
  // depth is level + 1 whoever won: the re-read of push() is not needed.
  static constexpr bool kPush4 = true;
  static constexpr int kMinBlocks = 8;  // 32 registers (6 CTAs at 40: measured equal or slower)
  __device__ __forceinline__ void push4(int32_t u, const int32_t (&v)[4], unsigned live, int use_filter,
                                        const OutBuilder& out) const {
    const int32_t nl = level + 1;
    if (use_filter) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (((live >> k) & 1u) && bm_has(vis, v[k])) live &= ~(1u << k);
    }
    if (!live) return;
    int32_t d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = ((live >> k) & 1u) ? *((volatile int32_t*)&st[v[k]].depth) : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((live >> k) & 1u) && use_filter && d[k] != -1 && d[k] != nl) live &= ~(1u << k);
    int32_t old[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) old[k] = ((live >> k) & 1u) && d[k] == -1 ? atomicCAS(&st[v[k]].depth, -1, nl) : d[k];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((live >> k) & 1u) && d[k] == -1 && old[k] == -1) out.emit(v[k]);
    const double su = st[u].sigma;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((live >> k) & 1u) && (d[k] == -1 || d[k] == nl) && (old[k] == -1 || old[k] == nl))
        atomicAdd(&st[v[k]].sigma, su);
  }
  __device__ __forceinline__ void push4u(const int32_t (&u)[4], const int32_t (&v)[4], unsigned live,
                                         int use_filter, const OutBuilder& out) const {
    const int32_t nl = level + 1;
    if (use_filter) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (((live >> k) & 1u) && bm_has(vis, v[k])) live &= ~(1u << k);
    }
    if (!live) return;
    int32_t d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = ((live >> k) & 1u) ? *((volatile int32_t*)&st[v[k]].depth) : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((live >> k) & 1u) && use_filter && d[k] != -1 && d[k] != nl) live &= ~(1u << k);
    int32_t old[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) old[k] = ((live >> k) & 1u) && d[k] == -1 ? atomicCAS(&st[v[k]].depth, -1, nl) : d[k];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((live >> k) & 1u) && d[k] == -1 && old[k] == -1) out.emit(v[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((live >> k) & 1u) && (d[k] == -1 || d[k] == nl) && (old[k] == -1 || old[k] == nl))
        atomicAdd(&st[v[k]].sigma, st[u[k]].sigma);
  }
  __device__ __forceinline__ Acc init() const { return {0.0, 0}; }
  __device__ __forceinline__ bool visit(Acc& a, int32_t, int32_t u, uint32_t) const {
    a.s += st[u].sigma;
    a.found = 1;
    return false;
  }
  static __device__ __forceinline__ Acc combine(Acc a, Acc b) { return {a.s + b.s, a.found | b.found}; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) { return OpBcFwd::warp_reduce(a); }
  __device__ __forceinline__ void finish(int32_t v, const Acc& a, const OutBuilder& out) const {
    if (!a.found) return;
    if (st[v].depth == -1) {
      st[v].depth = level + 1;
      out.emit(v);
    }
    st[v].sigma += a.s;
  }
};
// `next`: bitmap of the level after the frontier's; only arcs into it carry
// a dependency (depth[v] == depth[u] + 1), the rest skip the state gather.
struct OpBcBwdAoS {
  BcState* st;
  const uint32_t* next;
  using Acc = int;
  static constexpr bool kEarlyExit = false;
  __device__ __forceinline__ bool filter(int32_t) const { return true; }
  __device__ __forceinline__ double contrib(int32_t u, int32_t v) const {
    if (!bm_has(next, v)) return 0.0;
    // one 32-byte load of v's state (depth, sigma, delta); u's is per range
    const double2 sd = __ldg(reinterpret_cast<const double2*>(&st[v]));  // v's state is final
    const int32_t dv = __ldg(&st[v].depth);                               // (same sector: L1 hit)
    return dv == __ldg(&st[u].depth) + 1 ? __ldg(&st[u].sigma) / sd.x * (1.0 + sd.y) : 0.0;
  }
  __device__ __forceinline__ void push(int32_t u, int32_t v, uint32_t, const OutBuilder&) const {
    const double x = contrib(u, v);
    if (x != 0.0) atomicAdd(&st[u].delta, x);
  }
  static constexpr bool kPushReduce = true;
  __device__ __forceinline__ double push_val(int32_t u, int32_t v) const { return contrib(u, v); }
  __device__ __forceinline__ void push_commit(int32_t u, double x) const { atomicAdd(&st[u].delta, x); }
  __device__ __forceinline__ Acc init() const { return 0; }
  __device__ __forceinline__ bool visit(Acc&, int32_t v, int32_t u, uint32_t w) const {
    push(u, v, w, OutBuilder{});
    return false;
  }
  static __device__ __forceinline__ Acc combine(Acc a, Acc) { return a; }
  static __device__ __forceinline__ Acc warp_reduce(Acc a) { return a; }
  __device__ __forceinline__ void finish(int32_t, const Acc&, const OutBuilder&) const {}
};

}  // namespace gg
