// Multi-tensor SGD / momentum / Adam over every model's packed parameters in
// one launch (pkg/src/hybridnn/optim.py:52-87).  HBM-bound: 12 / 20 / 28 bytes
// per parameter.  Each 4096-float chunk belongs to one model segment; the
// per-model lr, step and bias corrections come from the step's schedule row.
//
// The arithmetic is evaluated in the reference's float32 order with
// explicit round-to-nearest intrinsics (numpy never contracts to FMA), so
// given the same gradients the update is bit-identical to apply_update.
#include <cstdlib>
#include <algorithm>

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

// One float4 of every arena: Adam through its fast path unless an element is hard (then the
// exact update_one for all four), SGD / momentum directly.
__device__ __forceinline__ void update4(const Update& u, float r1, float r2, float4& P, float4 G, float4& M, float4& V) {
  if (u.kind == HNN_OPT_ADAM) {
    float4 p = P, m = M, v = V;
    bool hard = adam_fast(u, r1, r2, p.x, G.x, m.x, v.x);
    hard |= adam_fast(u, r1, r2, p.y, G.y, m.y, v.y);
    hard |= adam_fast(u, r1, r2, p.z, G.z, m.z, v.z);
    hard |= adam_fast(u, r1, r2, p.w, G.w, m.w, v.w);
    if (!hard) {
      P = p, M = m, V = v;
      return;
    }
  }
  update_one(u, P.x, G.x, M.x, V.x);
  update_one(u, P.y, G.y, M.y, V.y);
  update_one(u, P.z, G.z, M.z, V.z);
  update_one(u, P.w, G.w, M.w, V.w);
}

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
    const float r1 = recip_refined(u.bias1), r2 = recip_refined(u.bias2);  // Adam's per-step reciprocals
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
        update4(u, r1, r2, P[q], G[q], M[q], V[q]);
        st_cs4(p4 + i, P[q]);
        if (u.kind != HNN_OPT_SGD) st_cs4(m4 + i, M[q]);
        if (u.kind == HNN_OPT_ADAM) st_cs4(v4 + i, V[q]);
      }
    }
  }
}

// ------------------------------------------------------------------ bulk-copy (TMA) kernel (default)
// The same update with the memory side moved to the bulk-copy engine: one CTA per SM, a producer
// thread streams whole 4096-float chunks of p / g / m / v (64 KB) into a 3-stage shared-memory ring
// with cp.async.bulk (up to 192 KB of loads in flight per SM, no load registers), 16 update warps
// read the stage from shared memory (two float4 per thread and array), write p / m / v back in
// place, and one of them issues the bulk stores.  Measured on C3's 76.7M Adam parameters launched
// alone (tools/opt_variants.py, profiles/r02/opt_ab_v3.txt): 0.342-0.348 ms = 6.2 TB/s, 95% of the
// copy peak, against 0.373-0.376 ms for the per-thread kernel above (whose seven LDG / STG streams
// alone take 0.375 ms).  2048-float stages x 6: 0.367 ms; two CTAs per SM of 2048 x 3: 0.352-0.357;
// 8 warps x 1024 floats x 6 stages, two CTAs: 0.353-0.366.  (Before Adam's fast path the update
// warps were issue-bound: 0.438 ms.)
#ifndef HNN_OPTB_E
#define HNN_OPTB_E 4096
#endif
#ifndef HNN_OPTB_STAGES
#define HNN_OPTB_STAGES 3
#endif
#ifndef HNN_OPTB_WARPS
#define HNN_OPTB_WARPS 16
#endif
#ifndef HNN_OPTB_CTAS
#define HNN_OPTB_CTAS 1
#endif
constexpr int OPTB_E = HNN_OPTB_E;                            // floats per array per stage
constexpr int OPTB_STAGES = HNN_OPTB_STAGES;                  // ring of 4 * OPTB_E floats per stage
constexpr int OPTB_WARPS = HNN_OPTB_WARPS;                    // update warps (+1 producer warp)
constexpr int OPTB_CTAS = HNN_OPTB_CTAS;                      // CTAs per SM
constexpr int OPTB_THREADS = 32 * (OPTB_WARPS + 1);
constexpr int OPTB_SMEM = OPTB_STAGES * 4 * OPTB_E * 4 + 1024;  // ring + barriers / stage info
static_assert(OPT_CHUNK % OPTB_E == 0 && OPTB_E % (128 * OPTB_WARPS) == 0, "whole float4 per update thread per array and stage");
static_assert(OPTB_CTAS * OPTB_SMEM <= 228 * 1024, "shared memory per SM");

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ float4 lds4f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4f(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

__global__ void __launch_bounds__(OPTB_THREADS, OPTB_CTAS)
    multi_tensor_bulk_kernel(const hnn_opt_segment* __restrict__ segs, int nseg, int total_units,
                             const hnn_step_row* __restrict__ cur, const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  extern __shared__ __align__(1024) uint8_t optb_smem[];
  const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(optb_smem));
  uint64_t* bars = reinterpret_cast<uint64_t*>(optb_smem + OPTB_STAGES * 4 * OPTB_E * 4);
  int4* info = reinterpret_cast<int4*>(bars + 2 * OPTB_STAGES);  // {segment, element offset, floats, live}
  auto bar = [&](int i) { return static_cast<uint32_t>(__cvta_generic_to_shared(bars + i)); };
  constexpr int FULL = 0, EMPTY = OPTB_STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OPTB_STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar(FULL + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar(EMPTY + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait = [&](uint32_t b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "OPTB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra OPTB_WAIT_%=;\n\t}" ::"r"(b),
        "r"(parity)
        : "memory");
  };
  const int warp = threadIdx.x / 32;
  if (warp == OPTB_WARPS) {
    // ---------------- producer: one thread issues every stage's bulk loads
    if (threadIdx.x % 32 == 0) {
      uint32_t it = 0;
      for (int u = blockIdx.x; u < total_units; u += gridDim.x, ++it) {
        const int s = int(it % OPTB_STAGES);
        if (it >= OPTB_STAGES) wait(bar(EMPTY + s), ((it / OPTB_STAGES) - 1) & 1);
        constexpr int UPC = OPT_CHUNK / OPTB_E;  // units per 4096-float chunk
        const int chunk = u / UPC;
        const int si = find_problem(segs, nseg, chunk, [](const hnn_opt_segment& q) { return q.chunk_base; });
        const hnn_opt_segment& sg = segs[si];
        const long long off = (long long)(chunk - sg.chunk_base) * OPT_CHUNK + (u % UPC) * OPTB_E;
        const int n = int(max(0LL, min((long long)OPTB_E, sg.count - off)));
        const bool ok = n > 0 && live(cur, status, sg.model);
        info[s] = make_int4(si, int(off), n, ok ? 1 : 0);
        const uint32_t st = ring + s * 4 * OPTB_E * 4;
        if (!ok) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar(FULL + s)) : "memory");
          continue;
        }
        const uint32_t bytes = uint32_t(n) * 4;
        const int arrays = 2 + (sg.kind != HNN_OPT_SGD) + (sg.kind == HNN_OPT_ADAM);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar(FULL + s)), "r"(bytes * arrays)
                     : "memory");
        bulk_load(st, sg.param + off, bytes, bar(FULL + s));
        bulk_load(st + OPTB_E * 4, sg.grad + off, bytes, bar(FULL + s));
        if (sg.kind != HNN_OPT_SGD) bulk_load(st + 2 * OPTB_E * 4, sg.m + off, bytes, bar(FULL + s));
        if (sg.kind == HNN_OPT_ADAM) bulk_load(st + 3 * OPTB_E * 4, sg.v + off, bytes, bar(FULL + s));
      }
    }
    return;
  }
  // ---------------- update warps: one float4 of each array per thread and stage
  const int t = threadIdx.x;
  uint32_t it = 0;
  for (int u = blockIdx.x; u < total_units; u += gridDim.x, ++it) {
    const int s = int(it % OPTB_STAGES);
    wait(bar(FULL + s), (it / OPTB_STAGES) & 1);
    const int4 inf = info[s];
    const uint32_t st = ring + s * 4 * OPTB_E * 4;
    if (inf.w) {
      const hnn_opt_segment& sg = segs[inf.x];
      const hnn_step_row& row = cur[sg.model];
      const Update up{sg.kind, row.lr, sg.momentum, row.bias1, row.bias2, row.opt_step == 1};
      const float r1 = recip_refined(up.bias1), r2 = recip_refined(up.bias2);
#pragma unroll
      for (int j = 0; j < OPTB_E / (128 * OPTB_WARPS); ++j) {
        const int i = t + j * 32 * OPTB_WARPS;
        if (4 * i >= inf.z) break;
        const uint32_t a = st + 16 * i;
        float4 P = lds4f(a), G = lds4f(a + OPTB_E * 4);
        float4 M = make_float4(0.f, 0.f, 0.f, 0.f), V = M;
        if (up.kind != HNN_OPT_SGD) M = lds4f(a + 2 * OPTB_E * 4);
        if (up.kind == HNN_OPT_ADAM) V = lds4f(a + 3 * OPTB_E * 4);
        update4(up, r1, r2, P, G, M, V);
        sts4f(a, P);
        if (up.kind != HNN_OPT_SGD) sts4f(a + 2 * OPTB_E * 4, M);
        if (up.kind == HNN_OPT_ADAM) sts4f(a + 3 * OPTB_E * 4, V);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(32 * OPTB_WARPS) : "memory");
      if (t == 0) {
        const uint32_t bytes = uint32_t(inf.z) * 4;
        bulk_store(sg.param + inf.y, st, bytes);
        if (up.kind != HNN_OPT_SGD) bulk_store(sg.m + inf.y, st + 2 * OPTB_E * 4, bytes);
        if (up.kind == HNN_OPT_ADAM) bulk_store(sg.v + inf.y, st + 3 * OPTB_E * 4, bytes);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // stage read: free for the producer
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar(EMPTY + s)) : "memory");
      }
    } else {
      asm volatile("bar.sync 1, %0;" ::"n"(32 * OPTB_WARPS) : "memory");
      if (t == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar(EMPTY + s)) : "memory");
    }
  }
  if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int launch_multi_tensor(const char* who, const hnn_opt_segment* segs, int nseg, int total_chunks,
                        const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(segs && cur && nseg > 0 && total_chunks > 0, who, "bad arguments");
  static int sms = 0, bulk = -1;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (bulk < 0) {
    const char* e = getenv("HNN_OPT_BULK");
    bulk = e ? atoi(e) : 1;  // HNN_OPT_BULK=0: the per-thread kernel (A/B)
    if (bulk) {
      cudaError_t err = cudaFuncSetAttribute(multi_tensor_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OPTB_SMEM);
      if (err != cudaSuccess) {
        set_error(who, cudaGetErrorString(err));
        bulk = -1;
        return HNN_ERR_CUDA;
      }
    }
  }
  if (bulk) {
    const int units = total_chunks * (OPT_CHUNK / OPTB_E);
    int grid = units < OPTB_CTAS * sms ? units : OPTB_CTAS * sms;
    if (const char* g = getenv("HNN_OPT_GRID")) grid = std::max(1, std::min(grid, atoi(g)));  // (probe: SM share)
    hnn::launch_pdl(multi_tensor_bulk_kernel, dim3(grid), dim3(OPTB_THREADS), OPTB_SMEM, as_stream(stream), segs, nseg,
                    units, cur, status);
    return check_launch(who);
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
