// fused.cuh — kernel fusion (engine.fused_loop with fusion=True,
// engine.py:639-662; runtime.fused_dispatch, runtime.py:194-209).
//
// A fused loop is ONE cooperative launch (one dispatch): every round runs the
// same load-balancer bodies as the unfused kernels (traverse.cuh b_*), with
// grid barriers where the unfused path would end a kernel, and the loop
// condition, hybrid direction choice, frontier conversions and bucket
// advances evaluated on the device.
#pragma once
#include "apply.cuh"

namespace gg {

// Scratch the phases need (allocated by the host driver).
struct FusedScratch {
  TwcQueues twc;
  int64_t* prefix;      // STRICT push: exclusive degree prefix (cap V+1)
  int64_t* block_sums;  // STRICT push: per-block partial sums (cap gridDim+1)
  const int64_t* spans; // STRICT pull: destination spans (static per graph)
  int64_t nspans;
  const int64_t* seg_end;  // EdgeBlocking segments (EDGE_ONLY + BLOCKED)
  int64_t nseg;
  CooView blocked;
  EtwcEntry* etwc_q;             // ETWC huge CTA-stage ranges (grid pass)
  unsigned long long* etwc_n;    // kept 0 between phases
  int64_t etwc_small;            // active lists shorter than this send every CTA-stage range to the grid pass
};

// Grid-wide exclusive prefix of active out-degrees (STRICT push in a fused
// loop): block partials -> block 0 scans them -> blocks rescan with offsets.
__device__ __forceinline__ void grid_degree_prefix(const InView& in, const int64_t* off, int64_t n,
                                                   int64_t* prefix, int64_t* block_sums,
                                                   cg::grid_group& grid) {
  __shared__ int64_t s_tot;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = min(n, (int64_t)blockIdx.x * per), hi = min(n, lo + per);
  int64_t part = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    int32_t u = active_at(in, i);
    part += off[u + 1] - off[u];
  }
  part = warp_sum(part);
  if (threadIdx.x == 0) s_tot = 0;
  __syncthreads();
  if (lane_id() == 0) atomicAdd((unsigned long long*)&s_tot, (unsigned long long)part);
  __syncthreads();
  if (threadIdx.x == 0) block_sums[blockIdx.x] = s_tot;
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t run = 0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      int64_t t = block_sums[b];
      block_sums[b] = run;
      run += t;
    }
    prefix[n] = run;
  }
  grid.sync();
  if (threadIdx.x == 0) {
    int64_t run = block_sums[blockIdx.x];
    for (int64_t i = lo; i < hi; ++i) {
      prefix[i] = run;
      int32_t u = active_at(in, i);
      run += off[u + 1] - off[u];
    }
  }
  grid.sync();
}

// One edgeset.apply phase inside a cooperative kernel.  The caller provides
// the input view in the representation the direction needs (sparse ids for
// PUSH, dense membership for PULL / EDGE_ONLY, or ALL).
template <class Op>
__device__ __forceinline__ void fused_edge_phase(const gg_schedule& s, const CsrView& out_csr,
                                                 const CsrView& in_csr, const CooView& coo,
                                                 const InView& in, const Op& op,
                                                 const OutBuilder& ob, bool use_filter,
                                                 unsigned long long* scanned, const FusedScratch& sc,
                                                 int cta, cg::grid_group& grid) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  if (s.load_balance == GG_LB_EDGE_ONLY) {
    if (s.blocking) {
      EdgeArgs<Op> a{sc.blocked, in, op, ob, use_filter ? 1 : 0};
      int64_t lo = 0;
      for (int64_t k = 0; k < sc.nseg; ++k) {
        edge_range(a, lo, sc.seg_end[k], tid, nth);
        lo = sc.seg_end[k];
        grid.sync();
      }
    } else {
      EdgeArgs<Op> a{coo, in, op, ob, use_filter ? 1 : 0};
      edge_range(a, 0, coo.E, tid, nth);
    }
    if (tid == 0) atomicAdd(scanned, (unsigned long long)(s.blocking ? sc.blocked.E : coo.E));
    return;
  }
  if (s.direction == GG_PUSH) {
    PushArgs<Op> a{out_csr, in, op, ob, use_filter ? 1 : 0, scanned};
    switch (s.load_balance) {
      case GG_LB_VERTEX_BASED: b_push_vb<Op>(a); break;
      case GG_LB_WM: b_push_wm<Op>(a); break;
      case GG_LB_CM: b_push_cm<Op>(a); break;
      case GG_LB_ETWC:
        a.huge = sc.etwc_q;
        a.huge_n = sc.etwc_n;
        if (a.huge && active_count(in, out_csr.V) < sc.etwc_small) a.huge_min = cta;  // as run_push
        b_push_etwc<Op>(a, cta);
        if (a.huge) {
          grid.sync();
          b_push_huge<Op, false>(a);
          grid.sync();
          if (tid == 0) *sc.etwc_n = 0;  // next append is behind the caller's barrier
        }
        break;
      case GG_LB_STRICT: {
        const int64_t n = active_count(in, out_csr.V);
        grid_degree_prefix(in, out_csr.off, n, sc.prefix, sc.block_sums, grid);
        b_push_strict<Op>(a, sc.prefix, 32);
        break;
      }
      case GG_LB_TWC: {
        if (tid < 3) sc.twc.cnt[tid] = 0;
        grid.sync();
        b_twc_bin<Op>(a, sc.twc, cta);
        grid.sync();
        b_twc_thread<Op>(a, sc.twc.q[0], sc.twc.cnt);
        b_twc_warp<Op>(a, sc.twc.q[1], sc.twc.cnt + 1);
        b_twc_cta<Op>(a, sc.twc.q[2], sc.twc.cnt + 2);
        break;
      }
    }
  } else {
    PullArgs<Op> a{in_csr, in, op, ob, use_filter ? 1 : 0, scanned};
    switch (s.load_balance) {
      case GG_LB_VERTEX_BASED: b_pull_vb<Op>(a); break;
      case GG_LB_WM: b_pull_wm<Op>(a); break;
      case GG_LB_CM: b_pull_cm<Op>(a); break;
      case GG_LB_ETWC: b_pull_etwc<Op>(a, cta); break;
      case GG_LB_STRICT: b_pull_strict<Op>(a, sc.spans, sc.nspans); break;
      case GG_LB_TWC: {
        if (tid < 3) sc.twc.cnt[tid] = 0;
        grid.sync();
        b_pull_twc_bin<Op>(a, sc.twc, cta);
        grid.sync();
        b_pull_twc_thread<Op>(a, sc.twc.q[0], sc.twc.cnt);
        b_pull_twc_warp<Op>(a, sc.twc.q[1], sc.twc.cnt + 1);
        b_pull_twc_cta<Op>(a, sc.twc.q[2], sc.twc.cnt + 2);
        break;
      }
    }
  }
}

// Host: scratch for a fused loop whose rounds may use schedules s1/s2.
struct FusedHost {
  FusedScratch sc{};
  DevBuf<int64_t> prefix, block_sums;
  int grid = 0;
  void prepare(Runtime& rt, const gg_schedule* const* scheds, int nsched, int coop_blocks) {
    const Graph& g = *rt.g;
    grid = coop_blocks;
    for (int k = 0; k < nsched; ++k) {
      const gg_schedule& s = *scheds[k];
      if (s.load_balance == GG_LB_TWC) twc_queues(&rt, &sc.twc);
      if (s.load_balance == GG_LB_ETWC && s.direction == GG_PUSH) {
        sc.etwc_small = kEtwcSmallPerSm * sm_count(rt.dev);
        etwc_huge(&rt, &sc.etwc_q, &sc.etwc_n, sc.etwc_small);
      }
      if (s.load_balance == GG_LB_STRICT && s.direction == GG_PUSH) {
        prefix.alloc(g.V + 2);
        block_sums.alloc(coop_blocks + 1);
        sc.prefix = prefix.p;
        sc.block_sums = block_sums.p;
      }
      if (s.load_balance == GG_LB_STRICT && s.direction == GG_PULL && s.load_balance != GG_LB_EDGE_ONLY) {
        int64_t nspans = std::min<int64_t>(g.V > 0 ? g.V : 1, (int64_t)sm_count(rt.dev) * 2048);
        strict_spans(&rt, nspans);
        sc.spans = rt.spans.p;
        sc.nspans = nspans;
      }
      if (s.load_balance == GG_LB_EDGE_ONLY && s.blocking) {
        int64_t n = s.blocking_size > 0 ? s.blocking_size : default_blocking_size(g);
        Blocked* b = blocked_for(const_cast<Graph&>(g), n);
        sc.seg_end = b->seg_end.p;
        sc.nseg = b->nseg;
        sc.blocked = CooView{b->src.p, b->dst.p, g.weighted ? b->w.p : nullptr, b->E};
      }
    }
  }
};

void cc_fused(Runtime& rt, const gg_schedule& s, int32_t* label, int* flags);

}  // namespace gg
