// Multi-tensor SGD / momentum / Adam over every model's packed parameters in
// one launch (pkg/src/hybridnn/optim.py:52-87).  HBM-bound: 12 / 20 / 28 bytes
// per parameter.  Each 4096-float chunk belongs to one model segment; the
// per-model lr, step and bias corrections come from the step's schedule row.
//
// The arithmetic is evaluated in the reference's float32 order with
// explicit round-to-nearest intrinsics (numpy never contracts to FMA), so
// given the same gradients the update is bit-identical to apply_update.
#include "common.cuh"

namespace hnn {

constexpr int OPT_THREADS = 256, OPT_CHUNK = 4096;  // 4 float4 per thread

struct Update {
  int kind;
  float lr, mom, bias1, bias2;
  bool first;
};

__device__ __forceinline__ void update_one(const Update& u, float& p, float g, float& m, float& v) {
  if (u.kind == HNN_OPT_SGD) {
    p = __fsub_rn(p, __fmul_rn(u.lr, g));
  } else if (u.kind == HNN_OPT_SGD_MOMENTUM) {
    m = u.first ? g : __fadd_rn(__fmul_rn(u.mom, m), g);
    p = __fsub_rn(p, __fmul_rn(u.lr, m));
  } else {
    const float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
    const float c1 = __fsub_rn(1.0f, b1), c2 = __fsub_rn(1.0f, b2);
    m = u.first ? __fmul_rn(c1, g) : __fadd_rn(__fmul_rn(b1, m), __fmul_rn(c1, g));
    v = u.first ? __fmul_rn(__fmul_rn(c2, g), g) : __fadd_rn(__fmul_rn(b2, v), __fmul_rn(__fmul_rn(c2, g), g));
    const float mhat = __fdiv_rn(m, u.bias1);
    const float vhat = __fdiv_rn(v, u.bias2);
    p = __fsub_rn(p, __fdiv_rn(__fmul_rn(u.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), eps)));
  }
}

__global__ void __launch_bounds__(OPT_THREADS) multi_tensor_kernel(const hnn_opt_segment* __restrict__ segs, int nseg,
                                                                   const hnn_step_row* __restrict__ cur,
                                                                   const hnn_model_status* __restrict__ status) {
  const int si = find_problem(segs, nseg, blockIdx.x, [](const hnn_opt_segment& q) { return q.chunk_base; });
  const hnn_opt_segment sg = segs[si];
  if (!live(cur, status, sg.model)) return;
  const hnn_step_row row = cur[sg.model];
  Update u{sg.kind, row.lr, sg.momentum, row.bias1, row.bias2, row.opt_step == 1};
  const long long base = (long long)(blockIdx.x - sg.chunk_base) * OPT_CHUNK;
  float4* p4 = reinterpret_cast<float4*>(sg.param + base);
  const float4* g4 = reinterpret_cast<const float4*>(sg.grad + base);
  float4* m4 = sg.m ? reinterpret_cast<float4*>(sg.m + base) : nullptr;
  float4* v4 = sg.v ? reinterpret_cast<float4*>(sg.v + base) : nullptr;
  const int n4 = int(min((long long)OPT_CHUNK, sg.count - base) / 4);
  float4 P[4], G[4], M[4], V[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = threadIdx.x + q * OPT_THREADS;
    if (i < n4) {
      // explicit global-space accesses (the segment pointers come from memory, so a plain
      // dereference compiles to generic LD/ST); gradients are read once -> evict-first
      P[q] = __ldcg(p4 + i);
      G[q] = __ldcs(g4 + i);
      if (u.kind != HNN_OPT_SGD) M[q] = __ldcg(m4 + i);
      if (u.kind == HNN_OPT_ADAM) V[q] = __ldcg(v4 + i);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = threadIdx.x + q * OPT_THREADS;
    if (i >= n4) continue;
    update_one(u, P[q].x, G[q].x, M[q].x, V[q].x);
    update_one(u, P[q].y, G[q].y, M[q].y, V[q].y);
    update_one(u, P[q].z, G[q].z, M[q].z, V[q].z);
    update_one(u, P[q].w, G[q].w, M[q].w, V[q].w);
    __stcg(p4 + i, P[q]);
    if (u.kind != HNN_OPT_SGD) __stcg(m4 + i, M[q]);
    if (u.kind == HNN_OPT_ADAM) __stcg(v4 + i, V[q]);
  }
}

int launch_multi_tensor(const char* who, const hnn_opt_segment* segs, int nseg, int total_chunks,
                        const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(segs && cur && nseg > 0 && total_chunks > 0, who, "bad arguments");
  multi_tensor_kernel<<<total_chunks, OPT_THREADS, 0, as_stream(stream)>>>(segs, nseg, cur, status);
  return check_launch(who);
}

}  // namespace hnn

// Both entry points run the same kernel; each segment carries its own kind, so
// one launch can update SGD and Adam models together.  The two names mirror
// the two branches of apply_update for callers that bind them separately.
extern "C" int hnn_multi_tensor_sgd(const hnn_opt_segment* segs, int nseg, int total_chunks, const hnn_step_row* cur,
                                    const hnn_model_status* status, void* stream) {
  return hnn::launch_multi_tensor("hnn_multi_tensor_sgd", segs, nseg, total_chunks, cur, status, stream);
}

extern "C" int hnn_multi_tensor_adam(const hnn_opt_segment* segs, int nseg, int total_chunks, const hnn_step_row* cur,
                                     const hnn_model_status* status, void* stream) {
  return hnn::launch_multi_tensor("hnn_multi_tensor_adam", segs, nseg, total_chunks, cur, status, stream);
}
