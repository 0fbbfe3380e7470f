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

// weak, non-coherent 16-byte loads (every element is read then written by the same thread, and
// nothing else touches the arenas during the launch) and evict-first streaming stores
__device__ __forceinline__ float4 ld_nc4(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_cs4(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

constexpr int OPT_THREADS = 256, OPT_CHUNK = 4096;  // 4 float4 per thread

// Persistent grid-stride walk over the 4096-float chunks of all segments (chunk ids are
// a flat index; each chunk belongs to exactly one segment).
__global__ void __launch_bounds__(OPT_THREADS) multi_tensor_kernel(const hnn_opt_segment* __restrict__ segs, int nseg,
                                                                   int total_chunks,
                                                                   const hnn_step_row* __restrict__ cur,
                                                                   const hnn_model_status* __restrict__ status) {
  for (int chunk = blockIdx.x; chunk < total_chunks; chunk += gridDim.x) {
    const int si = find_problem(segs, nseg, chunk, [](const hnn_opt_segment& q) { return q.chunk_base; });
    const hnn_opt_segment& sg = segs[si];
    if (!live(cur, status, sg.model)) continue;
    const hnn_step_row& row = cur[sg.model];
    const Update u{sg.kind, row.lr, sg.momentum, row.bias1, row.bias2, row.opt_step == 1};
    const long long base = (long long)(chunk - sg.chunk_base) * OPT_CHUNK;
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
        // dereference would compile to generic LD/ST)
        P[q] = ld_nc4(p4 + i);
        G[q] = ld_nc4(g4 + i);
        if (u.kind != HNN_OPT_SGD) M[q] = ld_nc4(m4 + i);
        if (u.kind == HNN_OPT_ADAM) V[q] = ld_nc4(v4 + i);
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
      st_cs4(p4 + i, P[q]);
      if (u.kind != HNN_OPT_SGD) st_cs4(m4 + i, M[q]);
      if (u.kind == HNN_OPT_ADAM) st_cs4(v4 + i, V[q]);
    }
  }
}

int launch_multi_tensor(const char* who, const hnn_opt_segment* segs, int nseg, int total_chunks,
                        const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(segs && cur && nseg > 0 && total_chunks > 0, who, "bad arguments");
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = total_chunks < 4 * sms ? total_chunks : 4 * sms;  // 2 resident CTAs/SM x 2 waves
  multi_tensor_kernel<<<grid, OPT_THREADS, 0, as_stream(stream)>>>(segs, nseg, total_chunks, cur, status);
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
