// fused.cu — fused (single cooperative launch) loops for CC and BFS.
// See fused.cuh.  Reference: engine.fused_loop (engine.py:639-662),
// runtime.fused_dispatch (runtime.py:194-209), algos.bfs / cc_soman.
#include "fused.cuh"

namespace gg {

// ---------------------------------------------------------------------------
// CC: hook phase + pointer jumping + change test, all on the device.
// ---------------------------------------------------------------------------
struct CcFusedArgs {
  gg_schedule s;
  CsrView out, in;
  CooView coo;
  FusedScratch sc;
  int32_t* label;
  int* flags;  // [0] changed, [1] moved, [2] rounds
  unsigned long long* scanned;
  int cta;
};

__global__ void __launch_bounds__(256) k_cc_fused(CcFusedArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t V = a.out.V;
  OpHook op{a.label, a.flags};
  OutBuilder none{};
  none.mode = OUT_NONE;
  InView all{};
  all.repr = -1;
  int rounds = 0;
  while (true) {
    if (tid == 0) a.flags[0] = 0;
    grid.sync();
    fused_edge_phase(a.s, a.out, a.in, a.coo, all, op, none, false, a.scanned, a.sc, a.cta, grid);
    grid.sync();
    while (true) {  // pointer jumping to a fixpoint
      if (tid == 0) a.flags[1] = 0;
      grid.sync();
      int any = 0;
      for (int64_t v = tid; v < V; v += nth) {
        int32_t l = a.label[v], ll = a.label[l];
        if (ll != l) { a.label[v] = ll; any = 1; }
      }
      if (__any_sync(0xffffffffu, any) && lane_id() == 0 && !*((volatile int*)a.flags + 1)) atomicOr(a.flags + 1, 1);
      grid.sync();
      const int moved = *((volatile int*)a.flags + 1);
      grid.sync();  // every thread has read the flag before thread 0 resets it
      if (!moved) break;
    }
    ++rounds;
    const int changed = *((volatile int*)a.flags);
    grid.sync();
    if (!changed) break;
  }
  if (tid == 0) a.flags[2] = rounds;
}

void cc_fused(Runtime& rt, const gg_schedule& s, int32_t* label, int* flags_unused) {
  const Graph& g = *rt.g;
  DevBuf<int> flags(3);
  flags.zero(rt.stream);
  CcFusedArgs a{};
  a.s = s;
  a.out = s.load_balance != GG_LB_EDGE_ONLY && s.direction == GG_PUSH ? g.out_view() : CsrView{};
  a.out.V = g.V;
  if (s.load_balance != GG_LB_EDGE_ONLY && s.direction == GG_PULL) a.in = g.in_view();
  a.in.V = g.V;
  if (s.load_balance == GG_LB_EDGE_ONLY && !s.blocking) a.coo = g.coo_view();
  a.label = label;
  a.flags = flags.p;
  a.scanned = rt.scanned.p;
  a.cta = rt.cfg.cta_size;
  int blocks = max_coop_blocks((const void*)k_cc_fused, 256, rt.dev);
  FusedHost fh;
  const gg_schedule* ss[1] = {&s};
  fh.prepare(rt, ss, 1, blocks);
  a.sc = fh.sc;
  void* args[] = {&a};
  rt.edge_begin();
  GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_cc_fused, blocks, 256, args, 0, rt.stream));
  rt.edge_end();
  count_launch();
  int h[3];
  GG_CUDA(cudaMemcpyAsync(h, flags.p, sizeof(h), cudaMemcpyDeviceToHost, rt.stream));
  GG_CUDA(cudaStreamSynchronize(rt.stream));
  rt.stats.dispatch_count += 1;
  rt.stats.rounds += h[2];
  for (int k = 0; k < h[2]; ++k) rt.stats.direction_log.push_back(s.direction);
  (void)flags_unused;
}

// ---------------------------------------------------------------------------
// BFS: frontier slots, hybrid choice, conversions and output finalisation on
// the device.  Slot buffers hold a frontier in any representation.
// ---------------------------------------------------------------------------
struct Slot {
  int32_t* ids;
  unsigned long long* count;
  uint32_t* bits;
  uint8_t* bools;
};

struct BfsFusedArgs {
  gg_binding b;
  CsrView out, in;
  CooView coo;
  FusedScratch sc;
  int32_t* parent;
  Slot slot[2];
  Slot conv;              // conversion target (ids / bits / bools)
  int32_t* stamps;        // MonotonicCounters
  uint32_t* mark_bits;    // DenseMarks sidecars
  uint8_t* mark_bytes;
  unsigned long long* scanned;
  int* log;               // per round: chosen schedule index (1 or 2)
  int64_t log_cap;
  long long* counters;    // [0] rounds [1] conversions [2] creation passes
  int cta;
};

__device__ __forceinline__ int repr_of_creation(int c) {
  return c == GG_CREATE_FUSED ? GG_SPARSE : (c == GG_CREATE_UNFUSED_BOOLMAP ? GG_BOOLMAP : GG_BITMAP);
}

__device__ void slot_clear(const Slot& s, int64_t V, int64_t tid, int64_t nth) {
  for (int64_t i = tid; i < (V + 31) / 32; i += nth) s.bits[i] = 0;
  for (int64_t i = tid; i < (V + 3) / 4; i += nth) reinterpret_cast<uint32_t*>(s.bools)[i] = 0;
  if (tid == 0) *s.count = 0;
}

__device__ void popcount_into(const Slot& s, int repr, int64_t V, int64_t tid, int64_t nth) {
  unsigned long long c = 0;
  if (repr == GG_BITMAP)
    for (int64_t i = tid; i < (V + 31) / 32; i += nth) c += __popc(s.bits[i]);
  else
    for (int64_t i = tid; i < V; i += nth) c += s.bools[i] != 0;
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(s.count, c);
}

__global__ void __launch_bounds__(256) k_bfs_fused(BfsFusedArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t V = a.out.V;
  OpBfs op{a.parent};
  int cur = 0, cur_repr = GG_SPARSE;
  int32_t round = 0;
  long long rounds = 0, convs = 0, passes = 0;
  while (true) {
    grid.sync();
    const unsigned long long size = *((volatile unsigned long long*)a.slot[cur].count);
    if (size == 0) break;
    const bool second = a.b.is_hybrid && (double)size > a.b.threshold * (double)V;
    const gg_schedule& s = second ? a.b.s2 : a.b.s1;
    if (tid == 0 && rounds < a.log_cap) a.log[rounds] = second ? 2 : 1;
    const Slot& in = a.slot[cur];
    const Slot& out = a.slot[cur ^ 1];
    // ---- input view in the representation the traversal needs
    int need;
    if (s.load_balance == GG_LB_EDGE_ONLY) need = cur_repr == GG_SPARSE ? GG_BOOLMAP : cur_repr;
    else if (s.direction == GG_PUSH) need = GG_SPARSE;
    else need = s.pull_repr;
    InView iv{};
    iv.repr = need;
    iv.coherent = 1;
    if (need == cur_repr) {
      iv.ids = in.ids; iv.count = in.count; iv.bits = in.bits; iv.bools = in.bools;
    } else {
      ++convs;
      slot_clear(a.conv, V, tid, nth);
      grid.sync();
      if (need == GG_SPARSE) {  // dense -> sparse (compaction, warp-aggregated)
        for (int64_t base = (tid & ~int64_t(31)); base < V; base += nth) {
          int64_t v = base + lane_id();
          bool m = v < V && (cur_repr == GG_BITMAP ? ((in.bits[v >> 5] >> (v & 31)) & 1u)
                                                   : in.bools[v] != 0);
          unsigned bal = __ballot_sync(0xffffffffu, m);
          unsigned long long b0 = 0;
          if (lane_id() == 0 && bal) b0 = atomicAdd(a.conv.count, (unsigned long long)__popc(bal));
          b0 = __shfl_sync(0xffffffffu, b0, 0);
          if (m) a.conv.ids[b0 + __popc(bal & ((1u << lane_id()) - 1))] = (int32_t)v;
        }
      } else {
        for (int64_t v = tid; v < V; v += nth) {
          bool m;
          if (cur_repr == GG_SPARSE) continue;
          m = cur_repr == GG_BITMAP ? ((in.bits[v >> 5] >> (v & 31)) & 1u) : in.bools[v] != 0;
          if (!m) continue;
          if (need == GG_BITMAP) atomicOr(a.conv.bits + (v >> 5), 1u << (v & 31));
          else a.conv.bools[v] = 1;
        }
        if (cur_repr == GG_SPARSE) {
          for (int64_t i = tid; i < (int64_t)size; i += nth) {
            int32_t v = in.ids[i];
            if (need == GG_BITMAP) atomicOr(a.conv.bits + (v >> 5), 1u << (v & 31));
            else a.conv.bools[v] = 1;
          }
        }
      }
      grid.sync();
      iv.ids = a.conv.ids; iv.count = a.conv.count; iv.bits = a.conv.bits; iv.bools = a.conv.bools;
    }
    // ---- output builder (engine.py:288-309)
    ++round;
    OutBuilder ob{};
    ob.mode = s.frontier_creation;
    ob.queue = out.ids;
    ob.qcount = out.count;
    ob.bits = out.bits;
    ob.bools = out.bools;
    ob.dedup = DEDUP_NONE;
    if (s.dedup) {
      if (s.dedup_strategy == GG_DEDUP_MONOTONIC_COUNTERS) {
        ob.dedup = DEDUP_COUNTERS;
        ob.stamps = a.stamps;
        ob.round = round;
      } else if (s.frontier_creation == GG_CREATE_FUSED) {
        ob.dedup = s.dedup_strategy == GG_DEDUP_BITMAP ? DEDUP_MARK_BITS : DEDUP_MARK_BYTES;
        ob.mark_bits = a.mark_bits;
        ob.mark_bytes = a.mark_bytes;
      } else {
        ob.dedup = DEDUP_SLOT;
      }
    }
    fused_edge_phase(s, a.out, a.in, a.coo, iv, op, ob, true, a.scanned, a.sc, a.cta, grid);
    grid.sync();
    // ---- finalize (engine.py:383-397)
    const int out_repr = repr_of_creation(s.frontier_creation);
    if (out_repr == GG_SPARSE) {
      if (ob.dedup == DEDUP_MARK_BITS || ob.dedup == DEDUP_MARK_BYTES) {
        const unsigned long long n = *((volatile unsigned long long*)out.count);
        for (int64_t i = tid; i < (int64_t)n; i += nth) {
          int32_t v = out.ids[i];
          if (ob.dedup == DEDUP_MARK_BITS) atomicAnd(a.mark_bits + (v >> 5), ~(1u << (v & 31)));
          else a.mark_bytes[v] = 0;
        }
      }
    } else {
      ++passes;
      popcount_into(out, out_repr, V, tid, nth);
    }
    // retire the input slot for reuse as the next output (FrontierPool.release)
    slot_clear(in, V, tid, nth);
    cur ^= 1;
    cur_repr = out_repr;
    ++rounds;
  }
  if (tid == 0) {
    a.counters[0] = rounds;
    a.counters[1] = convs;
    a.counters[2] = passes;
  }
}

void bfs_fused(Runtime& rt, const gg_binding& b, int32_t* parent, int32_t source) {
  const Graph& g = *rt.g;
  const int64_t V = g.V;
  cudaStream_t st = rt.stream;
  BfsFusedArgs a{};
  a.b = b;
  const gg_schedule* ss[2] = {&b.s1, &b.s2};
  const int ns = b.is_hybrid ? 2 : 1;
  bool need_out = false, need_in = false, need_coo = false;
  for (int k = 0; k < ns; ++k) {
    const gg_schedule& s = *ss[k];
    if (s.load_balance == GG_LB_EDGE_ONLY) need_coo = !s.blocking;
    else if (s.direction == GG_PUSH) need_out = true;
    else need_in = true;
  }
  if (need_out) a.out = g.out_view();
  if (need_in) a.in = g.in_view();
  if (need_coo) a.coo = g.coo_view();
  a.out.V = V;
  a.in.V = V;
  a.parent = parent;
  DevBuf<int32_t> ids[3];
  DevBuf<unsigned long long> counts(3);
  DevBuf<uint32_t> bits[3];
  DevBuf<uint8_t> bools[3];
  counts.zero(st);
  Slot* slots[3] = {&a.slot[0], &a.slot[1], &a.conv};
  for (int k = 0; k < 3; ++k) {
    ids[k].alloc(V + 1);
    bits[k].alloc((V + 31) / 32 + 1);
    bits[k].zero(st);
    bools[k].alloc(((V + 3) & ~int64_t(3)) + 4);
    bools[k].zero(st);
    *slots[k] = Slot{ids[k].p, counts.p + k, bits[k].p, bools[k].p};
  }
  // seed frontier: [source] (FrontierPool.new_frontier)
  GG_CUDA(cudaMemcpyAsync(ids[0].p, &source, 4, cudaMemcpyHostToDevice, st));
  unsigned long long one = 1;
  GG_CUDA(cudaMemcpyAsync(counts.p, &one, 8, cudaMemcpyHostToDevice, st));
  DevBuf<int32_t> stamps(V + 1);
  GG_CUDA(cudaMemsetAsync(stamps.p, 0xff, stamps.bytes(), st));
  DevBuf<uint32_t> mbits((V + 31) / 32 + 1);
  mbits.zero(st);
  DevBuf<uint8_t> mbytes(((V + 3) & ~int64_t(3)) + 4);
  mbytes.zero(st);
  a.stamps = stamps.p;
  a.mark_bits = mbits.p;
  a.mark_bytes = mbytes.p;
  a.scanned = rt.scanned.p;
  const int64_t log_cap = V + 2;
  DevBuf<int> log(log_cap);
  DevBuf<long long> counters(3);
  a.log = log.p;
  a.log_cap = log_cap;
  a.counters = counters.p;
  a.cta = rt.cfg.cta_size;
  int blocks = max_coop_blocks((const void*)k_bfs_fused, 256, rt.dev, 0, 2);
  FusedHost fh;
  fh.prepare(rt, ss, ns, blocks);
  a.sc = fh.sc;
  void* args[] = {&a};
  rt.edge_begin();
  GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_bfs_fused, blocks, 256, args, 0, st));
  rt.edge_end();
  count_launch();
  long long h[3];
  GG_CUDA(cudaMemcpyAsync(h, counters.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  GG_CUDA(cudaStreamSynchronize(st));
  std::vector<int> lg((size_t)std::min<long long>(h[0], log_cap));
  if (!lg.empty())
    GG_CUDA(cudaMemcpy(lg.data(), log.p, lg.size() * sizeof(int), cudaMemcpyDeviceToHost));
  // RunStats with the reference's FrontierPool accounting replayed on the
  // host: one spare buffer per representation (runtime.py:124-157).
  rt.stats.dispatch_count += 1;
  rt.stats.rounds += h[0];
  rt.stats.frontier_conversions += h[1];
  rt.stats.creation_passes += h[2];
  bool spare[3] = {false, false, false};
  int in_repr = GG_SPARSE;
  rt.stats.frontier_allocations += 1;  // new_frontier([source])
  for (int r : lg) {
    const gg_schedule& s = r == 2 ? b.s2 : b.s1;
    rt.stats.direction_log.push_back(s.direction);
    int out_repr = s.frontier_creation == GG_CREATE_FUSED
                       ? GG_SPARSE
                       : (s.frontier_creation == GG_CREATE_UNFUSED_BOOLMAP ? GG_BOOLMAP : GG_BITMAP);
    if (spare[out_repr]) spare[out_repr] = false;
    else rt.stats.frontier_allocations += 1;
    spare[in_repr] = true;
    rt.stats.reused_frontiers += 1;
    in_repr = out_repr;
  }
}

}  // namespace gg
