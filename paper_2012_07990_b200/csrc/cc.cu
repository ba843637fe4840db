// cc.cu — algos.cc_soman (reference algos.py:267-307) on the device.
//
// Round: changed = 0; edgeset.apply over all vertices with the hook functor
// (atomic_min on label[max(la,lb)]); full pointer jumping to a fixpoint
// (_pointer_jump, algos.py:254-264); repeat while a hook changed a label.
// Output canonicalised to each component's minimum vertex id.
// Fused (s0 kernel fusion): the whole loop is one cooperative launch
// (fused.cuh).
#include "apply.cuh"
#include "fused.cuh"

namespace gg {

__global__ void k_iota_i32(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

__global__ void k_pointer_jump(int32_t* label, int64_t V, int* moved) {
  int any = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t l = label[v], ll = label[l];
    if (ll != l) {
      label[v] = ll;
      any = 1;
    }
  }
  if (__any_sync(0xffffffffu, any) && lane_id() == 0 && !*((volatile int*)moved)) *moved = 1;
}

// the highest-degree vertex (its component is the giant one on the power-law
// inputs): packed (degree, -id) max
__global__ void k_argmax_degree(const int64_t* off, int64_t V, unsigned long long* best) {
  unsigned long long m = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = (unsigned long long)(off[v + 1] - off[v]);
    const unsigned long long key = (d << 32) | (unsigned long long)(0xffffffffu - (uint32_t)v);
    if (key > m) m = key;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
    if (x > m) m = x;
  }
  if (lane_id() == 0 && m) atomicMax(best, m);
}
// giant bitmap: label[v] == label[hub] (after pointer jumping: a root label)
__global__ void k_giant_bits(const int32_t* label, int64_t V, const unsigned long long* best, uint32_t* bits) {
  const int32_t hub = (int32_t)(0xffffffffu - (uint32_t)(*best & 0xffffffffu));
  const int32_t g = label[hub];
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); base < V;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = base + lane_id();
    const unsigned w = __ballot_sync(0xffffffffu, v < V && label[v] == g);
    if (lane_id() == 0) bits[base >> 5] = w;
  }
}

// first member (minimum id) of every label class, then relabel
__global__ void k_cc_first(const int32_t* label, int64_t V, int32_t* first) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
  {
    // read before the atomic: a giant component's members all share one
    // label, and an unconditional atomicMin per member serialises on it
    const int32_t l = label[v];
    if ((int32_t)v < *((volatile int32_t*)first + l)) atomicMin(first + l, (int32_t)v);
  }
}
__global__ void k_cc_canon(const int32_t* label, const int32_t* first, int64_t V, int32_t* out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    out[v] = first[label[v]];
}

// gg_edgeset_apply(GG_UDF_CC_HOOK): one hooking apply of cc_soman's body
// (algos.py:283-297); state arr0 = int32 label[V], arr1 = int changed flag.
std::unique_ptr<Frontier> apply_cc_hook(Runtime* rt, const gg_udf_state& st, bool use_filter,
                                        std::unique_ptr<Frontier>* in, const gg_binding& b,
                                        bool reuse, bool collect) {
  if (!st.arr0 || !st.arr1) fail(GG_ERR_VALUE, "cc hook needs label and changed-flag arrays");
  return apply_op(rt, OpHook{(int32_t*)st.arr0, (int*)st.arr1}, use_filter, in, b, reuse, collect);
}

void cc_run(const Graph& g, const gg_binding& b, bool fusion, Runtime& rt, int32_t* labels_out) {
  if (b.is_hybrid)
    fail(GG_ERR_SCHEDULE, "label 's0:s1' of cc takes a SimpleGPUSchedule (hybrid direction "
                          "switching applies to bfs/bc)");
  check_binding(b);
  DeviceGuard guard(g.dev);
  const int64_t V = g.V;
  const int dev = g.dev;
  cudaStream_t st = rt.stream;
  DevBuf<int32_t> label(V), first(V);
  DevBuf<int> flags(2);  // [0] changed, [1] moved
  k_iota_i32<<<grid_for(V, 256, dev), 256, 0, st>>>(label.p, V);
  GG_LAUNCH_CHECK();
  count_launch();
  if (fusion) {
    cc_fused(rt, b.s1, label.p, flags.p);
  } else {
    OpHook op{label.p, flags.p};
    {
      const char* rs = getenv("GG_CC_ROOT_SKIP");
      op.root_skip = !(rs && atoi(rs) == 0);
    }
    // giant-component filter (OpHook::giant), rebuilt after every round's
    // pointer jumping; none before the first round (labels are the ids)
    const int64_t W = (V + 31) / 32;
    DevBuf<uint32_t> giant(std::max<int64_t>(W, 1));
    DevBuf<unsigned long long> best(1);
    const char* ng = getenv("GG_CC_NO_GIANT");
    const bool use_giant = V > 0 && !(ng && atoi(ng) != 0);
    if (use_giant) {
      g.ensure_out();
      best.zero(st);
      k_argmax_degree<<<grid_for(V, 256, dev), 256, 0, st>>>(g.out_off.p, V, best.p);
      GG_LAUNCH_CHECK();
      count_launch();
    }
    int h[2] = {1, 0};
    while (h[0]) {
      GG_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), st));
      rt.edge_begin();
      apply_op(&rt, op, false, nullptr, b, false, false);
      rt.edge_end();
      do {  // pointer jumping to a fixpoint (host loop, not a dispatch)
        GG_CUDA(cudaMemsetAsync(flags.p + 1, 0, sizeof(int), st));
        k_pointer_jump<<<grid_for(V, 256, dev), 256, 0, st>>>(label.p, V, flags.p + 1);
        GG_LAUNCH_CHECK();
        count_launch();
        GG_CUDA(cudaMemcpyAsync(h, flags.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        GG_CUDA(cudaStreamSynchronize(st));
      } while (h[1]);
      rt.stats.rounds += 1;
      if (use_giant && h[0]) {
        k_giant_bits<<<grid_for(V, 256, dev), 256, 0, st>>>(label.p, V, best.p, giant.p);
        GG_LAUNCH_CHECK();
        count_launch();
        op.giant = giant.p;
      }
    }
  }
  GG_CUDA(cudaMemsetAsync(first.p, 0x7f, V * sizeof(int32_t), st));
  k_cc_first<<<grid_for(V, 256, dev), 256, 0, st>>>(label.p, V, first.p);
  k_cc_canon<<<grid_for(V, 256, dev), 256, 0, st>>>(label.p, first.p, V, label.p);
  GG_LAUNCH_CHECK();
  count_launch(2);
  GG_CUDA(cudaMemcpyAsync(labels_out, label.p, V * sizeof(int32_t), cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gg
