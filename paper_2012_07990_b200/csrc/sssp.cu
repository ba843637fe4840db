// sssp.cu — algos.sssp_delta (reference algos.py:215-247) with the two-bucket
// queue of priority.BucketQueue (priority.py:17-118) kept on the device.
//
// Device state: dist u64[V] (UNREACHED = 2^64-1), bucket queues as SPARSE
// id lists: current, far (+ a spare for advance), per-round dedup marks for
// current and persistent marks for far (DenseMarks BOOLMAP, priority.py:33-35).
// Round (fused_loop body, algos.py:236-243):
//   current empty -> advance(): drop stale far entries (bucket <= index), pick
//                    the minimum far bucket, split far into current / far;
//   else          -> take current, relax its out-edges with the schedule's
//                    load balancer (PUSH forced), re-bucketing improvements.
// Unfused: one kernel sequence per round with host-side control.
// Fused (s0 kernel fusion): the whole loop, including advance(), is ONE
// cooperative launch with per-bucket frontiers and grid barriers.
#include "fused.cuh"
#include <cstdio>

namespace gg {

static constexpr unsigned long long kUnreached = ~0ULL;

__global__ void k_adv_min(const int32_t* far, const unsigned long long* nfar,
                          const unsigned long long* dist, unsigned long long delta,
                          unsigned long long index, uint8_t* fmark, unsigned long long* best) {
  unsigned long long b_min = kUnreached;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*nfar;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = far[i];
    fmark[v] = 0;
    unsigned long long b = dist[v] / delta;
    if (b > index && b < b_min) b_min = b;
  }
  if (b_min != kUnreached) atomicMin(best, b_min);
}

__global__ void k_adv_split(const int32_t* far, const unsigned long long* nfar,
                            const unsigned long long* dist, unsigned long long delta,
                            unsigned long long index, const unsigned long long* bestp,
                            OutBuilder cur, OutBuilder far2) {
  const unsigned long long best = *bestp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*nfar;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = far[i];
    unsigned long long b = dist[v] / delta;
    if (b <= index) continue;  // stale: handled in an earlier bucket (priority.py:101-105)
    if (b == best) cur.emit(v);
    else far2.emit(v);
  }
}

__global__ void k_clear_byte_marks(const int32_t* ids, const unsigned long long* n, uint8_t* m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*n;
       i += (int64_t)gridDim.x * blockDim.x)
    m[ids[i]] = 0;
}

static OutBuilder queue_builder(Frontier* q, uint8_t* marks) {
  OutBuilder ob{};
  ob.mode = GG_CREATE_FUSED;
  ob.dedup = DEDUP_MARK_BYTES;
  ob.queue = q->ids.p;
  ob.qcount = q->count.p;
  ob.mark_bytes = marks;
  return ob;
}

// ---------------------------------------------------------------------------
// Fused delta-stepping: one cooperative launch for the whole loop.
// ---------------------------------------------------------------------------
struct SsspFusedArgs {
  gg_schedule s;
  CsrView out;
  CooView coo;
  FusedScratch sc;
  unsigned long long* dist;
  unsigned long long delta;
  int32_t* q[5];                  // current-bucket ring [0..2], far pair [3..4]
  unsigned long long* qn;         // counts [5]
  uint8_t* cmark;
  uint8_t* fmark;
  int32_t* stamps;                // fused relax rounds: current-bucket dedup by round stamp
  uint8_t* member;                // EDGE_ONLY input membership (boolmap)
  unsigned long long* best;       // advance scratch
  unsigned long long* scanned;
  long long* counters;            // [0] rounds [1] relax rounds
  int cta;
  unsigned long long* prof;       // GG_SSSP_PROFILE: [0] top-barrier wait [1] prep+barrier
                                  // [2] max edge-phase time of any thread per round (summed) (ns)
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) k_sssp_fused(SsspFusedArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  // Queues: a ring of three for the current bucket (q[0..2]) and a pair for
  // far (q[3], q[4]).  One grid barrier per relax round: every thread reads
  // the counts right after the barrier; a relax round reads ring slot `ci`
  // (its size stays in a register), appends to slot ci+1, and thread 0
  // zeroes slot ci+2 -- the previous round's input, which nobody reads or
  // writes in this round and which becomes the next round's output.  The
  // output's per-round dedup is a round stamp (no marks to clear).  An
  // advance refills the (empty) current slot behind its own barrier.
  int ci = 0, far = 3, far2 = 4;
  unsigned long long index = 0;
  long long rounds = 0, relax = 0, advances = 0;
  unsigned long long t0 = a.prof ? gtime() : 0;
  while (true) {
    grid.sync();
    unsigned long long t1 = 0;
    if (a.prof && tid == 0) {
      t1 = gtime();
      a.prof[0] += t1 - t0;
    }
    const unsigned long long ncur = *((volatile unsigned long long*)a.qn + ci);
    const unsigned long long nfar = *((volatile unsigned long long*)a.qn + far);
    if (ncur == 0 && nfar == 0) break;  // BucketQueue.done()
    ++rounds;
    if (ncur == 0) {
      // advance(): minimum live far bucket, then split far
      unsigned long long* bestp = a.best + (advances & 1);
      unsigned long long b_min = kUnreached;
      for (int64_t i = tid; i < (int64_t)nfar; i += nth) {
        int32_t v = a.q[far][i];
        a.fmark[v] = 0;
        unsigned long long b = a.dist[v] / a.delta;
        if (b > index && b < b_min) b_min = b;
      }
      if (b_min != kUnreached) atomicMin(bestp, b_min);
      grid.sync();
      const unsigned long long best = *((volatile unsigned long long*)bestp);
      if (best != kUnreached) {
        OutBuilder oc{}, of{};
        oc.mode = of.mode = GG_CREATE_FUSED;
        oc.dedup = DEDUP_NONE;  // far holds each vertex once (fmark), so the split does too
        of.dedup = DEDUP_MARK_BYTES;
        oc.queue = a.q[ci]; oc.qcount = a.qn + ci;
        of.queue = a.q[far2]; of.qcount = a.qn + far2; of.mark_bytes = a.fmark;
        for (int64_t i = tid; i < (int64_t)nfar; i += nth) {
          int32_t v = a.q[far][i];
          unsigned long long b = a.dist[v] / a.delta;
          if (b <= index) continue;
          if (b == best) oc.emit(v);
          else of.emit(v);
        }
        index = best;
      }
      if (tid == 0) {
        a.qn[far] = 0;                            // read into registers before the barrier
        a.best[(advances + 1) & 1] = kUnreached;  // next advance's slot
      }
      ++advances;
      int t = far; far = far2; far2 = t;
      if (a.prof) t0 = gtime();
      continue;
    }
    const int in = ci, out = ci == 2 ? 0 : ci + 1, spare = ci == 0 ? 2 : ci - 1;
    if (tid == 0) a.qn[spare] = 0;
    InView iv{};
    iv.coherent = 1;
    if (a.s.load_balance == GG_LB_EDGE_ONLY) {
      for (int64_t i = tid; i < (int64_t)ncur; i += nth) a.member[a.q[in][i]] = 1;
      iv.repr = GG_BOOLMAP;
      iv.bools = a.member;
      grid.sync();
    } else {
      iv.repr = GG_SPARSE;
      iv.ids = a.q[in];
      iv.count = a.qn + in;
      iv.n_fixed = (int64_t)ncur;
    }
    unsigned long long t2 = a.prof ? gtime() : 0;
    if (a.prof && tid == 0) a.prof[1] += t2 - t1;
    OpRelax op{a.dist, a.delta, index, OutBuilder{}, OutBuilder{}};
    op.cur.mode = op.far.mode = GG_CREATE_FUSED;
    op.cur.dedup = DEDUP_COUNTERS;
    op.cur.stamps = a.stamps;
    op.cur.round = (int32_t)(relax + 1);
    op.far.dedup = DEDUP_MARK_BYTES;
    op.cur.queue = a.q[out]; op.cur.qcount = a.qn + out;
    op.far.queue = a.q[far]; op.far.qcount = a.qn + far; op.far.mark_bytes = a.fmark;
    OutBuilder none{};
    none.mode = OUT_NONE;
    fused_edge_phase(a.s, a.out, a.out, a.coo, iv, op, none, false, a.scanned, a.sc, a.cta, grid);
    if (a.prof) {
      const unsigned long long t3 = gtime();
      if (relax < 1024) atomicMax(a.prof + 3 + relax, t3 - t2);  // slowest thread of the round
      t0 = t3;
    }
    if (a.s.load_balance == GG_LB_EDGE_ONLY) {
      grid.sync();  // membership is read by the edge phase
      for (int64_t i = tid; i < (int64_t)ncur; i += nth) a.member[a.q[in][i]] = 0;
    }
    ci = out;
    ++relax;
  }
  if (tid == 0) {
    a.counters[0] = rounds;
    a.counters[1] = relax;
  }
}

// ---------------------------------------------------------------------------
// Fused delta-stepping, VERTEX_BASED: asynchronous bucket phases over
// CTA-local work lists.
//
// The round-synchronous loop above pays one grid barrier plus the load
// balancer's machinery per relax round, and its round count is bounded by
// the graph's hop diameter (~10^4 rounds of ~10 us on the 4096^2 grid).
// Here a bucket is ONE phase with no grid barrier inside it.  Each CTA owns a
// shared-memory work list and runs sub-rounds separated only by
// __syncthreads: every thread takes one entry (vertex, candidate distance,
// arc range), relaxes the vertex's out-arcs unless dist[v] has dropped below
// the candidate (a later entry holds the better value -- the stale check
// replaces per-vertex queue flags), and pushes every improvement that stays
// in the current bucket back to the CTA's own list (graph-local work stays on
// the CTA that found it).  The arc range of a pushed vertex is loaded while
// the atomicMin that decides the push is in flight, so one hop costs two
// dependent memory round trips (arcs, then atomicMin + offsets).
// Improvements past the bucket go to `far` as (vertex, candidate) pairs
// (priority.py:59-77): an entry is live iff dist[v] still equals its
// candidate, which keeps exactly one live copy per vertex without the
// per-vertex marks (and their atomic round trip).  A list past its spill
// mark pushes to a global ring; a CTA with an empty list pulls a share of the
// ring.  `pending` counts pushed entries not yet relaxed: ring pushes add
// before publishing, each CTA adds its sub-round's (local pushes -
// completions) at the sub-round's end, so the sum never reaches 0 while an
// entry exists; a CTA with nothing local and nothing to pull leaves the phase
// once it reads 0.  Then advance() (priority.py:79-115): the minimum live far
// bucket, and a split that seeds the next bucket into the ring, which the
// CTAs divide statically at the next phase's start.
// Results are the exact shortest distances for any relaxation order
// (label-correcting inside a bucket, like the reference's in-bucket rounds);
// the round count is one relax round per bucket plus the advances (equal to
// the reference's whenever no in-bucket re-enqueue happens, e.g. delta = 1).
// ---------------------------------------------------------------------------
constexpr int kLq = 1024;             // CTA work-list capacity (power of two)
constexpr unsigned kFarChunk = 1024;  // far-list slots a CTA reserves at once
constexpr unsigned kFarRoom = 256;    // refill when fewer are left

struct SsspAsyncArgs {
  CsrView g;
  unsigned long long* dist;
  unsigned long long delta;
  int32_t* gv;                // global ring ids, -1 = empty slot
  unsigned long long* gd;     // global ring candidate distances
  unsigned long long mask;    // ring slots - 1 (power of two)
  unsigned long long* ctl;    // [0] head, [16] tail, [32] pending (separate 128-B lines)
  int32_t* q[2];              // far pair: ids (-1 = unused chunk slot) ...
  unsigned long long* qd[2];  // ... and candidate distances
  unsigned long long* qn;     // far counts [2]
  unsigned long long far_cap; // far list capacity (each list)
  unsigned long long* best;   // advance scratch: [0..1] minimum bucket, [2..3] far-has-entries flag
  unsigned long long* scanned;
  long long* counters;        // [0] rounds [1] relax rounds (bucket phases) [2] ring overflow
  int pull_max;               // ring entries per pull (GG_SSSP_PULL)
  int spill;                  // work-list occupancy past which pushes go to the ring (GG_SSSP_SPILL)
  unsigned long long* prof;   // GG_SSSP_PROFILE: [0] phase ns [1] advance ns [2] sub-rounds
                              // [3] idle polls [4] pulls [5] entries [6] stale skips
                              // [7..10] CTA 0: working ns, idle ns, working count, idle count
};

// A load the compiler cannot sink behind a branch (ptxas moves plain loads
// whose results are only used on one side; volatile ones stay put).
__device__ __forceinline__ int64_t ld_pinned_s64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.volatile.global.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void ring_store(const SsspAsyncArgs& a, unsigned long long p, int32_t v,
                                           unsigned long long d) {
  const unsigned long long s = p & a.mask;
  a.gd[s] = d;
  __threadfence();
  *((volatile int32_t*)a.gv + s) = v;  // publishes the slot
}
// Warp-convergent push of (v, d) (where `want`) into the global ring.
__device__ __forceinline__ void ring_push_warp(const SsspAsyncArgs& a, bool want, int32_t v, unsigned long long d) {
  const unsigned b = __ballot_sync(0xffffffffu, want);
  if (!b) return;
  const int leader = __ffs(b) - 1;
  unsigned long long base = 0;
  if ((int)lane_id() == leader) {
    atomicAdd(a.ctl + 32, (unsigned long long)__popc(b));  // pending before publishing
    base = atomicAdd(a.ctl + 16, (unsigned long long)__popc(b));
    if (base + __popc(b) - *((volatile unsigned long long*)a.ctl) > a.mask) a.counters[2] = 1;
  }
  base = __shfl_sync(0xffffffffu, base, leader);
  if (want) ring_store(a, base + __popc(b & lanemask_lt()), v, d);
}
// Push from divergent code (work-list spill): one atomic pair per converged group.
__device__ __forceinline__ void ring_push_one(const SsspAsyncArgs& a, int32_t v, unsigned long long d) {
  cg::coalesced_group grp = cg::coalesced_threads();
  unsigned long long p = 0;
  if (grp.thread_rank() == 0) {
    atomicAdd(a.ctl + 32, (unsigned long long)grp.size());
    p = atomicAdd(a.ctl + 16, (unsigned long long)grp.size());
    if (p + grp.size() - *((volatile unsigned long long*)a.ctl) > a.mask) a.counters[2] = 1;
  }
  ring_store(a, grp.shfl(p, 0) + grp.thread_rank(), v, d);
}
// Far append from divergent code, past a CTA's chunk.
__device__ __forceinline__ void far_push_one(const SsspAsyncArgs& a, int f, int32_t v, unsigned long long d) {
  cg::coalesced_group grp = cg::coalesced_threads();
  unsigned long long p = 0;
  if (grp.thread_rank() == 0) {
    p = atomicAdd(a.qn + f, (unsigned long long)grp.size());
    if (p + grp.size() > a.far_cap) a.counters[2] = 2;
  }
  p = grp.shfl(p, 0) + grp.thread_rank();
  if (p >= a.far_cap) return;
  a.q[f][p] = v;
  a.qd[f][p] = d;
}

__global__ void __launch_bounds__(1024) k_sssp_async(SsspAsyncArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int lane = (int)lane_id();
  const int64_t warp_base = tid - lane;
  volatile unsigned long long* head = a.ctl;
  volatile unsigned long long* tail = a.ctl + 16;
  volatile unsigned long long* pending = a.ctl + 32;
  // work list: vertex, degree, first arc, candidate distance
  __shared__ int32_t s_v[kLq], s_deg[kLq];
  __shared__ int64_t s_lo[kLq];
  __shared__ unsigned long long s_d[kLq];
  __shared__ unsigned s_head, s_tail, s_cnt, s_fn;
  __shared__ int s_net, s_state;
  __shared__ unsigned long long s_ph, s_pn, s_slo, s_shi, s_fbase;
  const bool prof0 = a.prof && blockIdx.x == 0 && threadIdx.x == 0;
  int far = 0, far2 = 1;
  unsigned long long index = 0;
  long long rounds = 0, relax = 0, advances = 0;
  unsigned long long sc = 0;
  while (true) {
    grid.sync();
    // Loop control and the ring's extent are read between two barriers: a
    // CTA that starts the phase early changes pending, head and tail, and a
    // late reader must not see that (it would take another branch).
    const unsigned long long npend = *pending;
    const unsigned long long nfar = *((volatile unsigned long long*)a.qn + far);
    const unsigned long long r_t = *tail;
    const unsigned long long r_h = *head;
    grid.sync();
    if (npend == 0 && nfar == 0) break;  // BucketQueue.done()
    ++rounds;
    const unsigned long long tp0 = a.prof && tid == 0 ? gtime() : 0;
    if (npend == 0) {
      // advance(): every ring entry is consumed, so the head moves to the
      // tail, where the split's entries -- the next phase's seeds -- begin.
      if (tid == 0) *head = r_t;
      unsigned long long* bestp = a.best + (advances & 1);
      unsigned long long* anyp = a.best + 2 + (advances & 1);  // far holds a real entry
      unsigned long long b_min = kUnreached;
      bool any = false;
      for (int64_t i = tid; i < (int64_t)nfar; i += nth) {
        const int32_t v = a.q[far][i];
        if (v < 0) continue;  // unused slot of a CTA's chunk
        any = true;
        const unsigned long long d = a.qd[far][i];
        if (a.dist[v] != d) continue;  // stale copy
        const unsigned long long b = d / a.delta;
        if (b > index && b < b_min) b_min = b;
      }
      if (b_min != kUnreached) atomicMin(bestp, b_min);
      if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(anyp, 1ULL);
      grid.sync();
      const unsigned long long best = *((volatile unsigned long long*)bestp);
      if (*((volatile unsigned long long*)anyp) == 0) {  // only unused chunk slots:
        --rounds;                                         // far was empty (done)
        break;
      }
      if (best != kUnreached) {
        for (int64_t base = warp_base; base < (int64_t)nfar; base += nth) {  // warp-uniform bounds
          const int64_t i = base + lane;
          int32_t v = -1;
          unsigned long long d = 0;
          if (i < (int64_t)nfar) v = a.q[far][i];
          if (v >= 0) d = a.qd[far][i];
          // live copies only (priority.py:101-105 drops stale far entries)
          const bool live = v >= 0 && a.dist[v] == d && d / a.delta > index;
          ring_push_warp(a, live && d / a.delta == best, v, d);
          const bool keep = live && d / a.delta != best;
          const unsigned kb = __ballot_sync(0xffffffffu, keep);
          if (kb) {
            const int leader = __ffs(kb) - 1;
            unsigned long long p = 0;
            if (lane == leader) p = atomicAdd(a.qn + far2, (unsigned long long)__popc(kb));
            p = __shfl_sync(0xffffffffu, p, leader) + __popc(kb & lanemask_lt());
            if (keep && p < a.far_cap) {
              a.q[far2][p] = v;
              a.qd[far2][p] = d;
            }
          }
        }
        index = best;
      }
      if (tid == 0) {
        a.qn[far] = 0;
        a.best[(advances + 1) & 1] = kUnreached;
        a.best[2 + ((advances + 1) & 1)] = 0;
      }
      ++advances;
      const int t = far; far = far2; far2 = t;
      if (a.prof && tid == 0) a.prof[1] += gtime() - tp0;
      continue;
    }
    // ---- one bucket phase: CTA sub-rounds, no grid barrier ----
    // every candidate is >= index * delta, so "in this bucket" is one compare
    const unsigned long long bucket_end =
        index >= ~0ULL / a.delta ? ~0ULL : (index + 1) * a.delta;
    if (threadIdx.x == 0) {
      // this CTA's static share of the bucket's seed entries [r_h, r_t);
      // the ring head is only ever claimed past r_t (pull below)
      const unsigned long long n0 = r_t - r_h;
      s_slo = r_h + n0 * blockIdx.x / gridDim.x;
      s_shi = r_h + n0 * (blockIdx.x + 1) / gridDim.x;
      s_head = s_tail = s_cnt = 0;
      s_fbase = 0;
      s_fn = kFarChunk;  // no far chunk yet
      s_net = 0;
    }
    int idle = 0;
    unsigned long long tw = 0;
    __syncthreads();
    // Two barriers per working sub-round: after thread 0's decisions, and
    // after the relax (thread 0 then folds the sub-round in and decides the
    // next one).  The entries read and the slots pushed never overlap: the
    // list holds at most kLq / 2 entries and a sub-round pushes into
    // [t0, hn + spill) only.
    while (true) {
      if (prof0) tw = clock64();
      if (threadIdx.x == 0) {
        s_state = 0;
        s_pn = 0;
        if (s_tail == s_head && s_slo < s_shi) {  // the static share first
          const unsigned long long take = min(s_shi - s_slo, (unsigned long long)(kLq / 2));
          s_ph = s_slo;
          s_pn = take;
          s_slo += take;
        } else if (s_tail == s_head) {  // nothing local: pull a share of the ring
          unsigned long long hv = *head, t = *tail;
          while (true) {
            const unsigned long long h = hv > r_t ? hv : r_t;  // seeds are static shares
            if (h >= t) break;
            const unsigned long long left = t - h;
            unsigned long long take = left / gridDim.x + 1;
            if (take > (unsigned long long)a.pull_max) take = a.pull_max;  // <= kLq / 2
            if (take > left) take = left;
            const unsigned long long old = atomicCAS(a.ctl, hv, h + take);
            if (old == hv) {
              s_ph = h;
              s_pn = take;
              break;
            }
            hv = old;
            t = *tail;
          }
          if (s_pn == 0) s_state = *pending == 0 ? 1 : 2;
        }
        // far appends of a working sub-round go to this CTA's chunk of the
        // far list (refilled while fewer than kFarRoom slots are left)
        if (s_state == 0 && s_fn + kFarRoom > kFarChunk) {
          for (unsigned i = s_fn; i < kFarChunk; ++i) a.q[far][s_fbase + i] = -1;
          s_fbase = atomicAdd(a.qn + far, (unsigned long long)kFarChunk);
          s_fn = 0;
          if (s_fbase + kFarChunk > a.far_cap) {  // never expected: fail loudly, stay in bounds
            a.counters[2] = 2;
            s_fn = kFarChunk;
            s_fbase = 0;
          }
        }
      }
      __syncthreads();
      if (s_state == 1) {  // phase over: mark this CTA's unused far slots
        for (unsigned i = s_fn + threadIdx.x; i < kFarChunk; i += blockDim.x) a.q[far][s_fbase + i] = -1;
        break;
      }
      if (s_state == 2) {
        if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 3, 1ULL);
        if (prof0) {
          a.prof[8] += clock64() - tw;
          a.prof[10] += 1;
        }
        __nanosleep(++idle < 8 ? 64 : 512);
        __syncthreads();  // everyone has read s_state before thread 0 rewrites it
        continue;
      }
      idle = 0;
      unsigned long long tA = prof0 ? clock64() : 0;
      if (a.prof && threadIdx.x == 0) {
        atomicAdd(a.prof + 2, 1ULL);
        if (s_pn) atomicAdd(a.prof + 4, 1ULL);
      }
      if (s_pn) {  // copy pulled / seed entries into the list (each slot is published)
        for (unsigned k = threadIdx.x; k < (unsigned)s_pn; k += blockDim.x) {
          volatile int32_t* slot = (volatile int32_t*)a.gv + ((s_ph + k) & a.mask);
          int32_t v;
          while ((v = *slot) < 0) __nanosleep(32);
          const unsigned long long d = *((volatile unsigned long long*)a.gd + ((s_ph + k) & a.mask));
          *slot = -1;
          const int64_t lo = __ldg(a.g.off + v), hi = __ldg(a.g.off + v + 1);
          const unsigned j = (s_tail + k) & (kLq - 1);
          s_v[j] = v;
          s_d[j] = d;
          s_lo[j] = lo;
          s_deg[j] = (int32_t)(hi - lo);
        }
        __syncthreads();
        if (threadIdx.x == 0) s_tail += (unsigned)s_pn;
        __syncthreads();
      }
      // lanes per entry: 4 when the sub-round takes <= 64 entries (one arc
      // per lane: a short dependent instruction chain per hop), fewer when
      // the list is long
      const unsigned h0 = s_head, t0 = s_tail;
      const unsigned avail = t0 - h0;
      const int lpe = avail <= blockDim.x / 4 ? 4 : avail <= blockDim.x / 2 ? 2 : 1;
      const unsigned n = min(avail, (unsigned)blockDim.x / lpe);
      const unsigned my = threadIdx.x / lpe;
      const int r = (int)(threadIdx.x % lpe);
      int32_t v = -1, deg = 0;
      int64_t lo = 0;
      unsigned long long d = 0;
      if (my < n) {
        const unsigned j = (h0 + my) & (kLq - 1);
        v = s_v[j];
        d = s_d[j];
        lo = s_lo[j];
        deg = s_deg[j];
      }
      unsigned long long tB = prof0 ? clock64() : 0;
      const unsigned hn = h0 + n;
      // local slots this sub-round may fill: [t0, hn + spill)
      const unsigned room = t0 - hn < (unsigned)a.spill ? (unsigned)a.spill - (t0 - hn) : 0u;
      int net = 0;
      if (v >= 0) {
        if (r == 0) --net;  // this entry completes in this sub-round
        if (a.prof && r == 0) atomicAdd(a.prof + 5, 1ULL);
        // lane r relaxes arcs r, r + lpe, ...; the stale check rides with the
        // first arc's loads, and a pushed vertex's arc range is loaded
        // alongside the atomicMin that decides the push
        for (int e = r; e < deg; e += lpe) {
          const int32_t u = __ldg(a.g.nbr + lo + e);
          const unsigned long long c = d + (unsigned long long)__ldg(a.g.w + lo + e);
          if (e == r && *((volatile unsigned long long*)a.dist + v) < d) {
            if (a.prof && r == 0) atomicAdd(a.prof + 6, 1ULL);
            break;  // stale: a later entry holds the better value
          }
          if (e == 0) sc += (unsigned long long)deg;
          // the target's arc range is loaded together with the atomicMin, not
          // behind its result (a third round trip per hop otherwise): all
          // three as volatile asm, so ptxas keeps them ahead of the compare
          const int64_t ulo = ld_pinned_s64(a.g.off + u), uhi = ld_pinned_s64(a.g.off + u + 1);
          unsigned long long old;
          asm volatile("atom.global.min.u64 %0, [%1], %2;" : "=l"(old) : "l"(a.dist + u), "l"(c) : "memory");
          if (c >= old) continue;
          if (c >= bucket_end) {  // past the bucket: far copy (v, candidate)
            const unsigned fp = atomicAdd(&s_fn, 1u);
            if (fp < kFarChunk) {
              a.q[far][s_fbase + fp] = u;
              a.qd[far][s_fbase + fp] = c;
            } else {
              far_push_one(a, far, u, c);
            }
            continue;
          }
          const unsigned kk = atomicAdd(&s_cnt, 1u);
          if (kk < room) {
            const unsigned j = (t0 + kk) & (kLq - 1);
            s_v[j] = u;
            s_d[j] = c;
            s_lo[j] = ulo;
            s_deg[j] = (int32_t)(uhi - ulo);
            ++net;
          } else {
            ring_push_one(a, u, c);  // the list is full: idle CTAs pull it
          }
        }
      }
      if (net) atomicAdd(&s_net, net);
      unsigned long long tC = prof0 ? clock64() : 0;
      __syncthreads();
      if (prof0) {
        const unsigned long long tD = clock64();
        a.prof[11] += tA - tw;
        a.prof[12] += tB - tA;
        a.prof[13] += tC - tB;
        a.prof[14] += tD - tC;
      }
      if (threadIdx.x == 0) {
        s_head = hn;
        s_tail = t0 + min(s_cnt, room);
        s_cnt = 0;
        if (s_net) atomicAdd(a.ctl + 32, (unsigned long long)(long long)s_net);
        s_net = 0;
        if (prof0) {
          a.prof[7] += clock64() - tw;
          a.prof[9] += 1;
        }
      }
    }
    ++relax;
    if (a.prof && tid == 0) a.prof[0] += gtime() - tp0;
  }
  sc = warp_sum(sc);
  if (lane == 0 && sc) atomicAdd(a.scanned, sc);
  if (tid == 0) {
    a.counters[0] = rounds;
    a.counters[1] = relax;
  }
}

// ---------------------------------------------------------------------------
// BucketQueue as a device object (priority.py:17-118) for custom loops:
// priorities u64[V] (UNREACHED = 2^64-1), current / far SPARSE queues with
// byte-mark dedup (per round for current, until advance for far), a spare
// for recycle().  Host calls order on the legacy stream like every driver.
// ---------------------------------------------------------------------------
struct BucketQueueDev {
  int dev = 0;
  int64_t V = 0;
  unsigned long long delta = 1;
  unsigned long long index = 0;
  DevBuf<unsigned long long> prio, best;
  DevBuf<uint8_t> cmark, fmark;
  DevBuf<int> flag;
  std::unique_ptr<Frontier> cur, far, far2, spare;
};

__global__ void k_bq_update(unsigned long long* prio, int64_t v, unsigned long long cand,
                            unsigned long long delta, unsigned long long index, OutBuilder cur,
                            OutBuilder far, int* improved, int seed) {
  if (seed) {  // seed(): the priority is set, the vertex enters current (priority.py:35-39)
    prio[v] = cand;
    cur.emit((int32_t)v);
    *improved = 1;
    return;
  }
  unsigned long long old = atomicMin(prio + v, cand);
  *improved = cand < old;
  if (cand < old) {
    if (cand / delta == index) cur.emit((int32_t)v);
    else far.emit((int32_t)v);
  }
}

BucketQueueDev* bq_create(int dev, int64_t V, uint64_t delta) {
  if (delta < 1) fail(GG_ERR_VALUE, "delta must be >= 1");
  if (V < 0) fail(GG_ERR_VALUE, "universe must be >= 0");
  DeviceGuard guard(dev);
  auto q = std::make_unique<BucketQueueDev>();
  q->dev = dev;
  q->V = V;
  q->delta = delta;
  q->prio.alloc(V);
  GG_CUDA(cudaMemsetAsync(q->prio.p, 0xff, std::max<int64_t>(V, 1) * 8, 0));
  const int64_t mb = ((V + 3) & ~int64_t(3)) + 4;
  q->cmark.alloc(mb);
  q->fmark.alloc(mb);
  q->cmark.zero();
  q->fmark.zero();
  q->best.alloc(1);
  q->flag.alloc(1);
  q->cur = frontier_alloc(dev, V, GG_SPARSE, V + 1);
  q->far = frontier_alloc(dev, V, GG_SPARSE, V + 1);
  q->far2 = frontier_alloc(dev, V, GG_SPARSE, V + 1);
  return q.release();
}

void bq_destroy(BucketQueueDev* q) {
  if (!q) return;
  DeviceGuard guard(q->dev);
  GG_CUDA(cudaStreamSynchronize(0));
  delete q;
}

static void bq_check_vertex(const BucketQueueDev* q, int64_t v) {
  if (v < 0 || v >= q->V)
    fail(GG_ERR_VALUE, strf("vertex %lld out of range [0, %lld)", (long long)v, (long long)q->V));
}

static bool bq_point_update(BucketQueueDev* q, int64_t v, uint64_t cand, int seed) {
  DeviceGuard guard(q->dev);
  k_bq_update<<<1, 1>>>(q->prio.p, v, cand, q->delta, q->index, queue_builder(q->cur.get(), q->cmark.p),
                        queue_builder(q->far.get(), q->fmark.p), q->flag.p, seed);
  GG_LAUNCH_CHECK();
  count_launch();
  q->cur->size_cache = -1;
  q->far->size_cache = -1;
  int h = 0;
  GG_CUDA(cudaMemcpy(&h, q->flag.p, sizeof(int), cudaMemcpyDeviceToHost));
  return h != 0;
}

void bq_seed(BucketQueueDev* q, int64_t v, uint64_t priority) {
  bq_check_vertex(q, v);
  q->index = priority / q->delta;  // the bucket index snaps to the seed's bucket
  bq_point_update(q, v, priority, 1);
}

bool bq_update_min(BucketQueueDev* q, int64_t v, uint64_t candidate) {
  bq_check_vertex(q, v);
  return bq_point_update(q, v, candidate, 0);
}

std::unique_ptr<Frontier> bq_take_current(BucketQueueDev* q) {
  DeviceGuard guard(q->dev);
  std::unique_ptr<Frontier> taken = std::move(q->cur);
  // clear the per-round marks of the taken ids (priority.py:47)
  k_clear_byte_marks<<<grid_for(std::max<int64_t>(q->V, 1), 256, q->dev), 256>>>(
      taken->ids.p, taken->count.p, q->cmark.p);
  GG_LAUNCH_CHECK();
  count_launch();
  if (q->spare) {
    q->cur = std::move(q->spare);
    q->cur->retired = false;
  } else {
    q->cur = frontier_alloc(q->dev, q->V, GG_SPARSE, q->V + 1);
  }
  frontier_clear(q->cur.get(), 0);
  taken->size_cache = -1;
  return taken;
}

void bq_recycle(BucketQueueDev* q, std::unique_ptr<Frontier> taken) {
  if (!taken) return;
  if (taken->universe != q->V || taken->repr != GG_SPARSE || (int64_t)taken->ids.n < q->V + 1)
    fail(GG_ERR_FRONTIER, "recycle takes a bucket handed out by take_current");
  frontier_clear(taken.get(), 0);
  if (!q->spare) q->spare = std::move(taken);
}

bool bq_advance(BucketQueueDev* q) {
  DeviceGuard guard(q->dev);
  if (frontier_size_raw(q->cur.get(), 0) != 0)
    fail(GG_ERR_ENGINE, "advance with a non-empty current bucket");
  const unsigned grid = (unsigned)sm_count(q->dev) * 8;
  GG_CUDA(cudaMemsetAsync(q->best.p, 0xff, 8, 0));
  k_adv_min<<<grid, 256>>>(q->far->ids.p, q->far->count.p, q->prio.p, q->delta, q->index, q->fmark.p,
                           q->best.p);
  GG_LAUNCH_CHECK();
  unsigned long long hb = 0;
  GG_CUDA(cudaMemcpy(&hb, q->best.p, 8, cudaMemcpyDeviceToHost));
  frontier_clear(q->far2.get(), 0);
  if (hb != kUnreached) {
    k_adv_split<<<grid, 256>>>(q->far->ids.p, q->far->count.p, q->prio.p, q->delta, q->index, q->best.p,
                               queue_builder(q->cur.get(), q->cmark.p),
                               queue_builder(q->far2.get(), q->fmark.p));
    GG_LAUNCH_CHECK();
    q->index = hb;
  }
  count_launch(hb != kUnreached ? 2 : 1);
  frontier_clear(q->far.get(), 0);
  std::swap(q->far, q->far2);
  q->cur->size_cache = -1;
  q->far->size_cache = -1;
  return hb != kUnreached;
}

void bq_info(BucketQueueDev* q, uint64_t* index, int64_t* ncur, int64_t* nfar) {
  DeviceGuard guard(q->dev);
  if (index) *index = q->index;
  if (ncur) *ncur = frontier_size_raw(q->cur.get(), 0);
  if (nfar) *nfar = frontier_size_raw(q->far.get(), 0);
}

void bq_copy_priorities(BucketQueueDev* q, uint64_t* dst) {
  DeviceGuard guard(q->dev);
  if (q->V) GG_CUDA(cudaMemcpy(dst, q->prio.p, q->V * 8, cudaMemcpyDefault));
}

Frontier* bq_queue(BucketQueueDev* q, int which) { return which ? q->far.get() : q->cur.get(); }
int64_t bq_universe(const BucketQueueDev* q) { return q->V; }

// gg_edgeset_apply(GG_UDF_SSSP_RELAX): update_priority_min(dst, prio[src] + w)
// for every arc of the input (algos.py:233-234); state arr0 = the queue.
std::unique_ptr<Frontier> apply_sssp_relax(Runtime* rt, const gg_udf_state& st, bool use_filter,
                                           std::unique_ptr<Frontier>* in, const gg_binding& b,
                                           bool reuse, bool collect) {
  auto* q = static_cast<BucketQueueDev*>(st.arr0);
  if (!q) fail(GG_ERR_VALUE, "sssp relax needs a bucket queue");
  if (q->V != rt->g->V)
    fail(GG_ERR_ENGINE, strf("bucket queue universe %lld does not match graph (%lld vertices)",
                             (long long)q->V, (long long)rt->g->V));
  if (!rt->g->weighted) fail(GG_ERR_VALUE, "sssp relax needs edge weights");
  OpRelax op{q->prio.p, q->delta, q->index, queue_builder(q->cur.get(), q->cmark.p),
             queue_builder(q->far.get(), q->fmark.p)};
  auto out = apply_op(rt, op, use_filter, in, b, reuse, collect);
  q->cur->size_cache = -1;
  q->far->size_cache = -1;
  return out;
}

void sssp_run(const Graph& g, int64_t source, const gg_binding& b, bool fusion, Runtime& rt,
              uint64_t* dist_out) {
  if (source < 0 || source >= g.V)
    fail(GG_ERR_VALUE, strf("invalid source %lld for graph with %lld vertices", (long long)source,
                            (long long)g.V));
  if (!g.weighted) fail(GG_ERR_VALUE, "sssp needs edge weights (load weighted or inject random weights)");
  if (b.is_hybrid)
    fail(GG_ERR_SCHEDULE, "label 's0:s1' of sssp takes a SimpleGPUSchedule (hybrid direction "
                          "switching applies to bfs/bc)");
  check_binding(b);
  DeviceGuard guard(g.dev);
  const int64_t V = g.V;
  const int dev = g.dev;
  cudaStream_t st = rt.stream;
  gg_binding pb = b;
  pb.s1.direction = GG_PUSH;  // relaxation is source-driven (algos.py:226-227)
  const gg_schedule& s = pb.s1;
  const unsigned long long delta = (unsigned long long)s.delta;
  DevBuf<unsigned long long> dist(V);
  GG_CUDA(cudaMemsetAsync(dist.p, 0xff, V * 8, st));
  unsigned long long zero = 0;
  GG_CUDA(cudaMemcpyAsync(dist.p + source, &zero, 8, cudaMemcpyHostToDevice, st));
  const int64_t mb = ((V + 3) & ~int64_t(3)) + 4;
  DevBuf<uint8_t> cmark(mb), fmark(mb);
  cmark.zero(st);
  fmark.zero(st);
  const uint8_t one = 1;
  GG_CUDA(cudaMemcpyAsync(cmark.p + source, &one, 1, cudaMemcpyHostToDevice, st));
  int32_t src32 = (int32_t)source;

  if (fusion && s.load_balance == GG_LB_VERTEX_BASED) {
    // asynchronous bucket phases over CTA work lists (k_sssp_async)
    int per_sm = 2;
    if (const char* e = getenv("GG_SSSP_ASYNC_PER_SM")) per_sm = std::max(1, atoi(e));
    // CTA size x CTAs per SM (GG_SSSP_BLOCK, GG_SSSP_ASYNC_PER_SM), measured
    // on the C3 grid: 128 x 4..8 41-44 ms, 256 x 1/2/3 38/35/31-34 ms,
    // 512 x 2 28.6-30 ms, 1024 x 1 29.8-31 ms -- bigger CTA work lists keep
    // more of the wavefront local (less ring traffic, fewer idle CTAs)
    int block = 512;
    if (const char* e = getenv("GG_SSSP_BLOCK")) block = atoi(e) == 128 ? 128 : atoi(e) == 512 ? 512 : atoi(e) == 1024 ? 1024 : 256;
    const int blocks = max_coop_blocks((const void*)k_sssp_async, block, dev, 0, per_sm);
    uint64_t R = 1 << 20;
    while (R < (uint64_t)(4 * V + 4096)) R <<= 1;
    // far lists: live copies (one per vertex) plus stale copies and the CTAs'
    // unused chunk tails; overflow is detected and reported, never expected
    const uint64_t far_cap = 2 * (uint64_t)V + 2 * (uint64_t)blocks * kFarChunk + 4096;
    DevBuf<int32_t> gv(R), q0(far_cap), q1(far_cap);
    DevBuf<unsigned long long> gd(R), qd0(far_cap), qd1(far_cap), ctl(48), qn(2), best(4);
    DevBuf<long long> counters(3);
    GG_CUDA(cudaMemsetAsync(gv.p, 0xff, R * sizeof(int32_t), st));
    ctl.zero(st);
    qn.zero(st);
    counters.zero(st);
    GG_CUDA(cudaMemsetAsync(best.p, 0xff, 2 * sizeof(unsigned long long), st));
    GG_CUDA(cudaMemsetAsync(best.p + 2, 0, 2 * sizeof(unsigned long long), st));
    const unsigned long long n1 = 1, z = 0;
    GG_CUDA(cudaMemcpyAsync(gv.p, &src32, 4, cudaMemcpyHostToDevice, st));
    GG_CUDA(cudaMemcpyAsync(gd.p, &z, 8, cudaMemcpyHostToDevice, st));
    GG_CUDA(cudaMemcpyAsync(ctl.p + 16, &n1, 8, cudaMemcpyHostToDevice, st));  // tail
    GG_CUDA(cudaMemcpyAsync(ctl.p + 32, &n1, 8, cudaMemcpyHostToDevice, st));  // pending
    SsspAsyncArgs a{};
    a.g = g.out_view();
    a.g.V = V;
    a.dist = dist.p;
    a.delta = delta;
    a.gv = gv.p;
    a.gd = gd.p;
    a.mask = R - 1;
    a.ctl = ctl.p;
    a.q[0] = q0.p;
    a.q[1] = q1.p;
    a.qd[0] = qd0.p;
    a.qd[1] = qd1.p;
    a.qn = qn.p;
    a.far_cap = far_cap;
    a.best = best.p;
    a.scanned = rt.scanned.p;
    a.counters = counters.p;
    a.pull_max = 256;
    if (const char* e = getenv("GG_SSSP_PULL")) a.pull_max = std::max(1, std::min(kLq / 2, atoi(e)));
    DevBuf<unsigned long long> prof;
    if (getenv("GG_SSSP_PROFILE")) {
      prof.alloc(16);
      prof.zero(st);
      a.prof = prof.p;
    }
    // past one sub-round of local work the rest goes to the ring, where idle
    // CTAs pull it (a bigger local list leaves CTAs idle behind a busy one)
    a.spill = 256;
    if (const char* e = getenv("GG_SSSP_SPILL")) a.spill = std::max(32, std::min(kLq / 4, atoi(e)));
    void* args[] = {&a};
    rt.edge_begin();
    GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_sssp_async, blocks, block, args, 0, st));
    rt.edge_end();
    count_launch();
    long long h[3];
    GG_CUDA(cudaMemcpyAsync(h, counters.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    GG_CUDA(cudaStreamSynchronize(st));
    if (h[2] == 1) fail(GG_ERR_CUDA, "fused SSSP: global work ring overflow");
    if (h[2] == 2) fail(GG_ERR_CUDA, "fused SSSP: far list overflow");
    if (a.prof) {
      unsigned long long hp[16];
      GG_CUDA(cudaMemcpy(hp, a.prof, sizeof(hp), cudaMemcpyDeviceToHost));
      fprintf(stderr, "sssp async profile: rounds %lld phases %lld | phases %.3f ms, advances %.3f ms | "
              "sub-rounds %llu (%.1f per CTA per phase), idle polls %llu, pulls %llu, entries %llu, stale %llu\n",
              h[0], h[1], hp[0] / 1e6, hp[1] / 1e6, hp[2], h[1] ? (double)hp[2] / blocks / h[1] : 0.0, hp[3],
              hp[4], hp[5], hp[6]);
      fprintf(stderr, "sssp async profile CTA 0 (SM cycles): %llu working sub-rounds, %.0f cycles each; %llu idle "
              "polls, %.0f cycles each\n", hp[9], hp[9] ? (double)hp[7] / hp[9] : 0.0, hp[10],
              hp[10] ? (double)hp[8] / hp[10] : 0.0);
      if (hp[9])
        fprintf(stderr, "sssp async profile CTA 0 per working sub-round (cycles): head %.0f, list+read %.0f, "
                "thread-0 relax %.0f, end barrier wait %.0f\n", (double)hp[11] / hp[9], (double)hp[12] / hp[9],
                (double)hp[13] / hp[9], (double)hp[14] / hp[9]);
    }
    rt.stats.dispatch_count += 1;
    rt.stats.rounds += h[0];
    for (long long k = 0; k < h[1]; ++k) rt.stats.direction_log.push_back(GG_PUSH);
  } else if (fusion) {
    SsspFusedArgs a{};
    a.s = s;
    if (s.load_balance == GG_LB_EDGE_ONLY) {
      if (!s.blocking) a.coo = g.coo_view();
    } else {
      a.out = g.out_view();
    }
    a.out.V = V;
    a.dist = dist.p;
    a.delta = delta;
    DevBuf<int32_t> q[5];
    DevBuf<unsigned long long> qn(5), best(2);
    qn.zero(st);
    GG_CUDA(cudaMemsetAsync(best.p, 0xff, 2 * sizeof(unsigned long long), st));
    for (int k = 0; k < 5; ++k) {
      q[k].alloc(V + 1);
      a.q[k] = q[k].p;
    }
    GG_CUDA(cudaMemcpyAsync(q[0].p, &src32, 4, cudaMemcpyHostToDevice, st));
    unsigned long long n1 = 1;
    GG_CUDA(cudaMemcpyAsync(qn.p, &n1, 8, cudaMemcpyHostToDevice, st));
    DevBuf<uint8_t> member(mb);
    member.zero(st);
    DevBuf<int32_t> stamps(V);
    stamps.zero(st);
    a.stamps = stamps.p;
    DevBuf<long long> counters(2);
    a.qn = qn.p;
    a.cmark = cmark.p;
    a.fmark = fmark.p;
    a.member = member.p;
    a.best = best.p;
    a.scanned = rt.scanned.p;
    a.counters = counters.p;
    a.cta = rt.cfg.cta_size;
    DevBuf<unsigned long long> prof;
    if (getenv("GG_SSSP_PROFILE")) {
      prof.alloc(3 + 1024);
      prof.zero(st);
      a.prof = prof.p;
    }
    int blocks = max_coop_blocks((const void*)k_sssp_fused, 256, dev, 0, 1);  // barrier-bound
    FusedHost fh;
    const gg_schedule* ss[1] = {&s};
    fh.prepare(rt, ss, 1, blocks);
    a.sc = fh.sc;
    void* args[] = {&a};
    rt.edge_begin();
    GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_sssp_fused, blocks, 256, args, 0, st));
    rt.edge_end();
    count_launch();
    long long h[2];
    GG_CUDA(cudaMemcpyAsync(h, counters.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    GG_CUDA(cudaStreamSynchronize(st));
    if (a.prof) {  // diagnostic: where a fused round's time goes (stderr)
      std::vector<unsigned long long> hp(3 + 1024);
      GG_CUDA(cudaMemcpy(hp.data(), prof.p, hp.size() * 8, cudaMemcpyDeviceToHost));
      unsigned long long mx = 0;
      for (int k = 0; k < 1024; ++k) mx += hp[3 + k];
      const long long nr = h[1] < 1024 ? h[1] : 1024;
      fprintf(stderr, "sssp fused profile: rounds %lld relax %lld | thread0: top-barrier wait %.3f ms, "
              "prep+barrier %.3f ms | slowest-thread edge phase, mean of first %lld rounds: %.3f us\n",
              h[0], h[1], hp[0] / 1e6, hp[1] / 1e6, nr, nr ? mx / 1e3 / nr : 0.0);
    }
    rt.stats.dispatch_count += 1;
    rt.stats.rounds += h[0];
    for (long long k = 0; k < h[1]; ++k) rt.stats.direction_log.push_back(GG_PUSH);
    if (s.load_balance == GG_LB_EDGE_ONLY) rt.stats.frontier_conversions += h[1];
  } else {
    std::unique_ptr<Frontier> cur = frontier_alloc(dev, V, GG_SPARSE, V + 1);
    std::unique_ptr<Frontier> take = frontier_alloc(dev, V, GG_SPARSE, V + 1);
    std::unique_ptr<Frontier> far = frontier_alloc(dev, V, GG_SPARSE, V + 1);
    std::unique_ptr<Frontier> far2 = frontier_alloc(dev, V, GG_SPARSE, V + 1);
    GG_CUDA(cudaMemcpyAsync(cur->ids.p, &src32, 4, cudaMemcpyHostToDevice, st));
    unsigned long long n1 = 1;
    GG_CUDA(cudaMemcpyAsync(cur->count.p, &n1, 8, cudaMemcpyHostToDevice, st));
    DevBuf<unsigned long long> best(1);
    unsigned long long index = 0;
    const unsigned grid = (unsigned)sm_count(dev) * 8;
    while (true) {
      unsigned long long n[2];
      GG_CUDA(cudaMemcpyAsync(&n[0], cur->count.p, 8, cudaMemcpyDeviceToHost, st));
      GG_CUDA(cudaMemcpyAsync(&n[1], far->count.p, 8, cudaMemcpyDeviceToHost, st));
      GG_CUDA(cudaStreamSynchronize(st));
      if (n[0] == 0 && n[1] == 0) break;
      rt.stats.rounds += 1;
      if (n[0] == 0) {  // advance()
        GG_CUDA(cudaMemsetAsync(best.p, 0xff, 8, st));
        k_adv_min<<<grid, 256, 0, st>>>(far->ids.p, far->count.p, dist.p, delta, index, fmark.p, best.p);
        GG_LAUNCH_CHECK();
        unsigned long long hb = 0;
        GG_CUDA(cudaMemcpyAsync(&hb, best.p, 8, cudaMemcpyDeviceToHost, st));
        GG_CUDA(cudaStreamSynchronize(st));
        if (hb != kUnreached) {
          OutBuilder oc = queue_builder(cur.get(), cmark.p);
          OutBuilder of = queue_builder(far2.get(), fmark.p);
          k_adv_split<<<grid, 256, 0, st>>>(far->ids.p, far->count.p, dist.p, delta, index, best.p,
                                            oc, of);
          GG_LAUNCH_CHECK();
          index = hb;
        }
        count_launch(hb != kUnreached ? 2 : 1);
        GG_CUDA(cudaMemsetAsync(far->count.p, 0, 8, st));
        std::swap(far, far2);
        continue;
      }
      std::swap(cur, take);  // take_current()
      GG_CUDA(cudaMemsetAsync(cur->count.p, 0, 8, st));
      k_clear_byte_marks<<<grid, 256, 0, st>>>(take->ids.p, take->count.p, cmark.p);
      GG_LAUNCH_CHECK();
      count_launch();
      take->size_cache = (int64_t)n[0];
      OpRelax op{dist.p, delta, index, queue_builder(cur.get(), cmark.p), queue_builder(far.get(), fmark.p)};
      rt.edge_begin();
      apply_op(&rt, op, false, &take, pb, false, false);
      rt.edge_end();
      take->size_cache = -1;
    }
  }
  GG_CUDA(cudaMemcpyAsync(dist_out, dist.p, V * 8, cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gg
