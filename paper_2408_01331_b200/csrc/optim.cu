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

constexpr int OPT_THREADS = 256, OPT_CHUNK = 4096;  // 4 float4 per thread per chunk
// Measured on C3 (76.7M Adam params, tools/opt_variants.py), launched alone: 5 CTAs/SM x 1 float4
// per arena per thread 0.399 ms (5.39 TB/s, 82% of the copy peak; a pure-traffic kernel with the
// same access pattern 0.375 ms); 4 CTAs 0.404; 6 / 8 CTAs (register-capped, spilling) 0.44 /
// 0.51; 2 float4 per thread 0.49; 4 float4 at 2 CTAs 0.61.  Inside the step (after the weight-
// gradient GEMMs, profiles/r01) 4 CTAs win: 0.419 ms against 0.443 (5) and 0.461 (3).
#ifndef HNN_OPT_MIN_CTAS
#define HNN_OPT_MIN_CTAS 4
#endif
#ifndef HNN_OPT_UNROLL
#define HNN_OPT_UNROLL 1
#endif
constexpr int OPT_MIN_CTAS = HNN_OPT_MIN_CTAS, OPT_UNROLL = HNN_OPT_UNROLL;

// Persistent grid-stride walk over the 4096-float chunks of all segments (chunk ids are
// a flat index; each chunk belongs to exactly one segment).  A thread handles one float4 of
// each arena at a time: full occupancy (2048 threads x 64 B in flight per SM) hides both the
// HBM latency and the dependent division / sqrt chains of Adam, which at 2 CTAs/SM with
// 16 elements per thread made the launch latency-bound.
__global__ void __launch_bounds__(OPT_THREADS, OPT_MIN_CTAS)
    multi_tensor_kernel(const hnn_opt_segment* __restrict__ segs, int nseg, int total_chunks,
                        const hnn_step_row* __restrict__ cur, const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
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
#pragma unroll 1
    for (int i0 = threadIdx.x; i0 < n4; i0 += OPT_THREADS * OPT_UNROLL) {
      // explicit global-space accesses (the segment pointers come from memory, so a plain
      // dereference would compile to generic LD/ST); all loads of the group issue first
      float4 P[OPT_UNROLL], G[OPT_UNROLL], M[OPT_UNROLL], V[OPT_UNROLL];
#pragma unroll
      for (int q = 0; q < OPT_UNROLL; ++q) {
        const int i = i0 + q * OPT_THREADS;
        if (i < n4) {
          P[q] = ld_nc4(p4 + i);
          G[q] = ld_nc4(g4 + i);
          if (u.kind != HNN_OPT_SGD) M[q] = ld_nc4(m4 + i);
          if (u.kind == HNN_OPT_ADAM) V[q] = ld_nc4(v4 + i);
        }
      }
#pragma unroll
      for (int q = 0; q < OPT_UNROLL; ++q) {
        const int i = i0 + q * OPT_THREADS;
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
  const int grid = total_chunks < OPT_MIN_CTAS * sms ? total_chunks : OPT_MIN_CTAS * sms;  // one wave
  hnn::launch_pdl(multi_tensor_kernel, dim3(grid), dim3(OPT_THREADS), 0, as_stream(stream), segs, nseg, total_chunks, cur, status);
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

namespace hnn {
__global__ void selftest_div_sqrt_kernel(const float* a, const float* b, float* q, float* r, int64_t n) {
  hnn::pdl_wait();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    q[i] = div_rn_exact(a[i], b[i]);
    r[i] = sqrt_rn_exact(a[i]);
  }
}
}  // namespace hnn

extern "C" int hnn_selftest_div_sqrt(const float* a, const float* b, float* q, float* r, int64_t n, void* stream) {
  HNN_REQUIRE(a && b && q && r && n >= 0, "hnn_selftest_div_sqrt", "bad arguments");
  if (n == 0) return HNN_OK;
  hnn::launch_pdl(hnn::selftest_div_sqrt_kernel, dim3(1184), dim3(256), 0, hnn::as_stream(stream), a, b, q, r, n);
  return hnn::check_launch("hnn_selftest_div_sqrt");
}
