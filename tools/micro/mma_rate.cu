// Micro-benchmark: tcgen05.mma issue-to-completion throughput per SM for the shapes the GEMM
// kernels use (tf32 cta_group::1 128xN, tf32 cta_group::2 256xN, f16/bf16 for reference).
// Operands are whatever sits in shared memory (throughput only).  Build + run (debug tool):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o /tmp/mma_rate tools/micro/mma_rate.cu -lcuda
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2408_01331_b200/csrc/tc_common.cuh"

using namespace hnn;

__host__ __device__ constexpr uint32_t f16_idesc(int m, int n, int a_mn, int b_mn) {
  // kind::f16: D fp32 (bits 4-5 = 1), A/B bf16 (bits 7-9 = 1, 10-12 = 1), majorness, N>>3, M>>4
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

template <int PAIR, int KIND, int N>
__global__ void __cluster_dims__(PAIR ? 2 : 1, 1, 1) mma_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  const uint32_t base = smem_u32(sm);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if (PAIR)
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    else
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  const bool issuer = threadIdx.x == 0 && (!PAIR || cluster_rank() == 0);
  unsigned long long t0 = clock64();
  if (issuer) {
    const uint64_t da = smem_desc(base, 16, 1024, 2), db = smem_desc(base + 65536, 16, 1024, 2);
    const uint32_t M = PAIR ? 256 : 128;
    for (int i = 0; i < iters; ++i) {
      if (KIND == 0) {
        const uint32_t idesc = tf32_idesc(M, N, 0, 0);
        if (PAIR) mma_tf32_pair(tmem, da, db, idesc, 1u);
        else mma_tf32(tmem, da, db, idesc, 1u);
      } else {
        const uint32_t idesc = f16_idesc(M, N, 0, 0);
        if (PAIR)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(da), "l"(db), "r"(idesc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(da), "l"(db), "r"(idesc));
      }
    }
    if (PAIR) mma_commit_pair(smem_u32(&bar));
    else mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int PAIR, int KIND, int N>
void run(const char* name) {
  const int iters = 4096, grid = 148;
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  auto k = mma_kernel<PAIR, KIND, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<grid, 128, 200 * 1024>>>(iters, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<grid, 128, 200 * 1024>>>(iters, d);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const int M = PAIR ? 256 : 128, K = KIND == 0 ? 8 : 16;
  const double flops = 2.0 * M * N * K * iters * (grid / (PAIR ? 2 : 1));
  printf("%-28s %s  %.3f ms  %.1f TFLOP/s  clk/MMA %.1f\n", name, cudaGetErrorString(e), ms, flops / ms / 1e9,
         double(h[0]) / iters);
  cudaFree(d);
}

int main() {
  run<0, 0, 128>("tf32 cta1 128x128x8");
  run<0, 0, 256>("tf32 cta1 128x256x8");
  run<1, 0, 128>("tf32 cta2 256x128x8");
  run<1, 0, 256>("tf32 cta2 256x256x8");
  run<0, 1, 256>("bf16 cta1 128x256x16");
  run<1, 1, 256>("bf16 cta2 256x256x16");
  return 0;
}
