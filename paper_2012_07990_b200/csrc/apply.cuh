// apply.cuh — the edgeset.apply dispatcher templates (engine.py:418-608),
// shared by every driver translation unit (BFS, PR, SSSP, CC, BC).
#pragma once
#include "engine.cuh"

namespace gg {

template <class Op>
inline void launch_push_huge(const PushArgs<Op>& a, int dev, cudaStream_t st) {
  if constexpr (MinBlocks<Op>::value > 1)
    k_push_huge_mb<Op, MinBlocks<Op>::value><<<(unsigned)sm_count(dev) * 8, 256, 0, st>>>(a);
  else
    k_push_huge<Op><<<(unsigned)sm_count(dev) * 8, 256, 0, st>>>(a);
}

int max_coop_blocks(const void* fn, int block, int dev, size_t smem = 0, int cap_per_sm = 0);
void strict_prefix(Runtime* rt, const InView& in, int64_t n);
void strict_spans(Runtime* rt, int64_t nspans);
void clear_marks(Runtime* rt, Frontier* out, const OutBuilder& ob);
Frontier* converted_view(Runtime* rt, Frontier* in, int repr);
// TWC bins sized for `entries` active-list entries (>= V; a multiset input may exceed V)
void twc_queues(Runtime* rt, TwcQueues* q, int64_t entries = 0);
// ETWC huge-range queue (capacity max(E / kEtwcHuge, small_frontier, entries) + 1),
// count zeroed on the stream
void etwc_huge(Runtime* rt, EtwcEntry** q, unsigned long long** n, int64_t small_frontier = 0,
               int64_t entries = 0);
OutBuilder make_builder(Runtime* rt, const gg_schedule& s, Frontier* out);
void dense_size_on_device(Frontier* f, cudaStream_t s);
// Named UDFs of the algorithm drivers, routed through gg_edgeset_apply
// (each defined beside its driver so the apply_op instantiations are shared).
std::unique_ptr<Frontier> apply_cc_hook(Runtime* rt, const gg_udf_state& st, bool use_filter,
                                        std::unique_ptr<Frontier>* in, const gg_binding& b,
                                        bool reuse, bool collect);
std::unique_ptr<Frontier> apply_bc_forward(Runtime* rt, const gg_udf_state& st, bool use_filter,
                                           std::unique_ptr<Frontier>* in, const gg_binding& b,
                                           bool reuse, bool collect);
std::unique_ptr<Frontier> apply_bc_backward(Runtime* rt, const gg_udf_state& st, bool use_filter,
                                            std::unique_ptr<Frontier>* in, const gg_binding& b,
                                            bool reuse, bool collect);
std::unique_ptr<Frontier> apply_sssp_relax(Runtime* rt, const gg_udf_state& st, bool use_filter,
                                           std::unique_ptr<Frontier>* in, const gg_binding& b,
                                           bool reuse, bool collect);

// sum of the out-degrees of the n entries of a SPARSE input (one round trip)
int64_t degree_sum(Runtime* rt, const InView& in, int64_t n);

template <class Op>
void run_push(Runtime* rt, const gg_schedule& s, const Op& op, bool use_filter, InView in,
                     int64_t n_host, const OutBuilder& out) {
  const Graph* g = rt->g;
  cudaStream_t st = rt->stream;
  PushArgs<Op> a{g->out_view(), in, op, out, use_filter ? 1 : 0, rt->scanned.p};
  const int dev = rt->dev;
  const int64_t work = n_host >= 0 ? n_host : g->V;
  const int cta = rt->cfg.cta_size;
  switch (s.load_balance) {
    case GG_LB_VERTEX_BASED:
      k_push_vb<Op><<<grid_for(work, 256, dev), 256, 0, st>>>(a);
      break;
    case GG_LB_WM:
      k_push_wm<Op><<<grid_for(work * 8, 256, dev), 256, 0, st>>>(a);
      break;
    case GG_LB_CM:
      k_push_cm<Op><<<grid_for(work, 256, dev), 256, 0, st>>>(a);
      break;
    case GG_LB_ETWC: {
      // A frontier that fills only a few CTAs (one per 256 vertices) would
      // leave every CTA-stage range (>= cta arcs) on a handful of SMs (a
      // 744-vertex BFS level of RMAT-24 with hub neighbours: 3.1 ms on 3
      // CTAs): all of them go to the chunk-balanced grid pass instead.  The
      // bound keeps the pass's per-CTA walk of the queue short.
      const bool small = work < kEtwcSmallPerSm * sm_count(dev);
      etwc_huge(rt, &a.huge, &a.huge_n, small ? work : 0, work);
      if (small && a.huge) a.huge_min = cta;
      if constexpr (MinBlocks<Op>::value > 1)
        k_push_etwc_mb<Op, MinBlocks<Op>::value><<<grid_for(work, 256, dev), 256, 0, st>>>(a, cta);
      else
        k_push_etwc<Op><<<grid_for(work, 256, dev), 256, 0, st>>>(a, cta);
      if (a.huge) {
        launch_push_huge<Op>(a, dev, st);
        count_launch();
      }
      break;
    }
    case GG_LB_STRICT: {
      const int64_t n = n_host >= 0 ? n_host : g->V;
      strict_prefix(rt, in, n);
      k_push_strict<Op><<<grid_for(g->E / 32 + 1, 256, dev), 256, 0, st>>>(a, rt->prefix.p, 32);
      break;
    }
    case GG_LB_TWC: {
      TwcQueues q;
      twc_queues(rt, &q, work);
      etwc_huge(rt, &a.huge, &a.huge_n, 0, work);  // hubs skip the bins (b_twc_bin)
      k_twc_bin<Op><<<grid_for(work, 256, dev), 256, 0, st>>>(a, q, cta);
      a.scanned = rt->scanned.p;
      if constexpr (MinBlocks<Op>::value > 1) {
        constexpr int mb = MinBlocks<Op>::value;
        k_twc_thread_mb<Op, mb><<<grid_for(work, 256, dev), 256, 0, st>>>(a, q.q[0], q.cnt);
        k_twc_warp_mb<Op, mb><<<grid_for(work * 32, 256, dev), 256, 0, st>>>(a, q.q[1], q.cnt + 1);
        k_twc_cta_mb<Op, mb><<<grid_for(work * 256, 256, dev), 256, 0, st>>>(a, q.q[2], q.cnt + 2);
      } else {
        k_twc_thread<Op><<<grid_for(work, 256, dev), 256, 0, st>>>(a, q.q[0], q.cnt);
        k_twc_warp<Op><<<grid_for(work * 32, 256, dev), 256, 0, st>>>(a, q.q[1], q.cnt + 1);
        k_twc_cta<Op><<<grid_for(work * 256, 256, dev), 256, 0, st>>>(a, q.q[2], q.cnt + 2);
      }
      count_launch(3);
      if (a.huge) {
        launch_push_huge<Op>(a, dev, st);
        count_launch();
      }
      break;
    }
    default:
      fail(GG_ERR_ENGINE, "no chunker for this load balance");
  }
  GG_LAUNCH_CHECK();
  count_launch();
}

template <class Op>
void run_pull(Runtime* rt, const gg_schedule& s, const Op& op, bool use_filter, InView in,
                     const OutBuilder& out) {
  const Graph* g = rt->g;
  cudaStream_t st = rt->stream;
  PullArgs<Op> a{g->in_view(), in, op, out, use_filter ? 1 : 0, rt->scanned.p};
  const int dev = rt->dev;
  const int64_t V = g->V;
  const int cta = rt->cfg.cta_size;
  switch (s.load_balance) {
    case GG_LB_VERTEX_BASED:
      k_pull_vb<Op><<<grid_for(V, 256, dev), 256, 0, st>>>(a);
      break;
    case GG_LB_WM:
      k_pull_wm<Op><<<grid_for(V * 32, 256, dev), 256, 0, st>>>(a);
      break;
    case GG_LB_CM:
      k_pull_cm<Op><<<grid_for(V * 256, 256, dev), 256, 0, st>>>(a);
      break;
    case GG_LB_ETWC:
      k_pull_etwc<Op><<<grid_for(V, 256, dev), 256, 0, st>>>(a, cta);
      break;
    case GG_LB_STRICT: {
      const int64_t nspans = std::min<int64_t>(V > 0 ? V : 1, (int64_t)sm_count(dev) * 2048);
      strict_spans(rt, nspans);
      k_pull_strict<Op><<<grid_for(nspans * 32, 256, dev), 256, 0, st>>>(a, rt->spans.p, nspans);
      break;
    }
    case GG_LB_TWC: {
      TwcQueues q;
      twc_queues(rt, &q);
      k_pull_twc_bin<Op><<<grid_for(V, 256, dev), 256, 0, st>>>(a, q, cta);
      k_pull_twc_thread<Op><<<grid_for(V, 256, dev), 256, 0, st>>>(a, q.q[0], q.cnt);
      k_pull_twc_warp<Op><<<grid_for(V * 32, 256, dev), 256, 0, st>>>(a, q.q[1], q.cnt + 1);
      k_pull_twc_cta<Op><<<grid_for(V * 256, 256, dev), 256, 0, st>>>(a, q.q[2], q.cnt + 2);
      count_launch(3);
      break;
    }
    default:
      fail(GG_ERR_ENGINE, "no pull partitioner for this load balance");
  }
  GG_LAUNCH_CHECK();
  count_launch();
}

template <class Op>
void run_edge_only(Runtime* rt, const gg_schedule& s, const Op& op, bool use_filter, InView in,
                          const OutBuilder& out) {
  const Graph* g = rt->g;
  cudaStream_t st = rt->stream;
  const int dev = rt->dev;
  if (!g->has_coo) fail(GG_ERR_ENGINE, "graph COO view was dropped");
  EdgeArgs<Op> a{g->coo_view(), in, op, out, use_filter ? 1 : 0};
  if (s.blocking) {
    int64_t n = s.blocking_size > 0 ? s.blocking_size : default_blocking_size(*g);
    Blocked* b = blocked_for(*const_cast<Graph*>(g), n);
    a.coo = CooView{b->src.p, b->dst.p, g->weighted ? b->w.p : nullptr, b->E};
    const int64_t* seg = b->seg_end.p;
    int64_t nseg = b->nseg;
    void* args[] = {&a, &seg, &nseg};
    const void* fn = (const void*)k_edge_blocked<Op>;
    if constexpr (MinBlocks<Op>::value > 1) fn = (const void*)k_edge_blocked_mb<Op, MinBlocks<Op>::value>;
    int blocks = max_coop_blocks(fn, 256, dev);
    GG_CUDA(cudaLaunchCooperativeKernel(fn, blocks, 256, args, 0, st));
  } else {
    if constexpr (MinBlocks<Op>::value > 1)
      k_edge_only_mb<Op, MinBlocks<Op>::value><<<grid_for(g->E / 4 + 1, 256, dev, 16), 256, 0, st>>>(a);
    else
      k_edge_only<Op><<<grid_for(g->E / 4 + 1, 256, dev, 16), 256, 0, st>>>(a);
    GG_LAUNCH_CHECK();
  }
  count_launch();
  rt->stats.edges_traversed += g->E;
}

// The output builder configuration of _OutputBuilder.__init__ (engine.py:288-309).
template <class Op>
std::unique_ptr<Frontier> apply_op(Runtime* rt, const Op& op, bool use_filter,
                                          std::unique_ptr<Frontier>* input, const gg_binding& b,
                                          bool reuse, bool collect_output) {
  NvtxRange nvtx("gg.edgeset_apply");
  check_binding(b);
  const Graph* g = rt->g;
  Frontier* in = input ? input->get() : nullptr;
  if (in && in->universe != g->V)
    fail(GG_ERR_ENGINE, strf("frontier universe %lld does not match graph (%lld vertices)",
                             (long long)in->universe, (long long)g->V));
  if (in && in->retired) fail(GG_ERR_FRONTIER, "frontier was retired");
  // hybrid_apply: s2 iff |input| > threshold * |V| (engine.py:631-632)
  const gg_schedule* sp = &b.s1;
  if (b.is_hybrid) {
    int64_t size = in ? frontier_size(rt, in) : 0;
    sp = ((double)size > b.threshold * (double)g->V) ? &b.s2 : &b.s1;
  }
  const gg_schedule& s = *sp;
  rt->stats.direction_log.push_back(s.direction);

  std::unique_ptr<Frontier> out;
  if (collect_output) {
    int repr = s.frontier_creation == GG_CREATE_FUSED
                   ? GG_SPARSE
                   : (s.frontier_creation == GG_CREATE_UNFUSED_BOOLMAP ? GG_BOOLMAP : GG_BITMAP);
    out = rt->acquire(repr);
    frontier_clear(out.get(), rt->stream);
  }
  OutBuilder ob = make_builder(rt, s, out.get());

  // input views (engine.py:404-415, 559-565)
  auto converted = [&](int repr) -> Frontier* { return converted_view(rt, in, repr); };
  InView iv{};
  iv.repr = -1;
  if (s.load_balance == GG_LB_EDGE_ONLY) {
    if (in) iv = (in->repr == GG_SPARSE ? converted(GG_BOOLMAP) : in)->view();
    run_edge_only(rt, s, op, use_filter, iv, ob);
  } else if (s.direction == GG_PUSH) {
    int64_t n_host = g->V;
    if (in) {
      Frontier* sv = in->repr == GG_SPARSE ? in : converted(GG_SPARSE);
      iv = sv->view();
      n_host = frontier_size_raw(sv, rt->stream);
      // a multiset input (dedup off upstream) may emit more than the output
      // queue's max(V, E) + 1 slots: size it exactly when the bound allows it
      if (out && ob.mode == GG_CREATE_FUSED && ob.dedup == DEDUP_NONE &&
          !EmitsOncePerVertex<Op>::value && n_host > 1) {
        const_cast<Graph*>(g)->ensure_out();
        const int64_t cap = (int64_t)out->ids.n;
        if ((double)n_host * (double)g->max_out_degree >= (double)cap) {
          const int64_t need = degree_sum(rt, iv, n_host) + 1;
          if (need > cap) {
            out->ids.alloc(need);
            ob.queue = out->ids.p;
          }
        }
      }
    }
    if (n_host > 0) run_push(rt, s, op, use_filter, iv, n_host, ob);
  } else {
    if (in) iv = (in->repr == s.pull_repr ? in : converted(s.pull_repr))->view();
    run_pull(rt, s, op, use_filter, iv, ob);
  }
  if (rt->fused_depth == 0) rt->stats.dispatch_count += 1;

  // finalize (engine.py:383-397)
  if (out) {
    if (s.frontier_creation == GG_CREATE_FUSED) {
      if (ob.dedup == DEDUP_MARK_BITS || ob.dedup == DEDUP_MARK_BYTES) {
        clear_marks(rt, out.get(), ob);
      }
      out->size_cache = -1;
    } else {
      dense_size_on_device(out.get(), rt->stream);
      rt->stats.creation_passes += 1;
    }
  }
  if (reuse && input && *input) {
    rt->release(std::move(*input));
    rt->stats.reused_frontiers += 1;
  }
  return out;
}

}  // namespace gg
