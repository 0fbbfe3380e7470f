// Grouped embedding-lookup (pkg/src/hybridnn/ops.py:258-278) for every model of a wave.
//   FWD  y[b, l, :] = table[x[b, l], :]          one warp per (b, l) row, rows past the batch zeroed
//   BWD  dtable[v, :] = sum over positions p of x == v, in ascending p, of dy[p, :]
//        = np.add.at(dt, idx, dy) in its accumulation order: one warp per table row scans the
//          positions 32 at a time (ballot) and adds the matching dy rows in order; no atomics,
//          so the bits are those of the reference's sequential scatter given the same dy.
// Token ids arrive as float32 (the dataset's sample values); the host validated them once on
// upload (integral, in [0, vocab): check_class_indices, src/ops.py:203-211).
#include "common.cuh"

namespace hnn {

constexpr int EM_WARPS = 8;

__device__ __forceinline__ const hnn_embed_problem& em_problem(const hnn_embed_problem* probs, int nprob, int block) {
  return probs[find_problem(probs, nprob, block, [](const hnn_embed_problem& q) { return q.block_base; })];
}

__global__ void __launch_bounds__(32 * EM_WARPS) embed_fwd_kernel(const hnn_embed_problem* __restrict__ probs, int nprob,
                                                                 const hnn_step_row* __restrict__ cur,
                                                                 const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const hnn_embed_problem& p = em_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int lane = threadIdx.x % 32;
  const long long r = (long long)(blockIdx.x - p.block_base) * EM_WARPS + threadIdx.x / 32;  // (b, l) row
  if (r >= (long long)p.cap * p.len) return;
  const int b = int(r / p.len);
  float* dst = p.y + size_t(r) * p.dim;
  if (b >= rows) {
    for (int c = lane; c < p.dim; c += 32) dst[c] = 0.0f;
    return;
  }
  const int v = int(p.x[size_t(b) * p.ldx + (r - (long long)b * p.len)]);
  const float* src = p.table + size_t(v) * p.dim;
  for (int c = lane; c < p.dim; c += 32) dst[c] = __ldg(src + c);
}

__global__ void __launch_bounds__(32 * EM_WARPS) embed_bwd_kernel(const hnn_embed_problem* __restrict__ probs, int nprob,
                                                                 const hnn_step_row* __restrict__ cur,
                                                                 const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const hnn_embed_problem& p = em_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int lane = threadIdx.x % 32;
  const int v = (blockIdx.x - p.block_base) * EM_WARPS + threadIdx.x / 32;  // table row
  if (v >= p.vocab) return;
  const long long npos = (long long)rows * p.len;
  float* out = p.dtable + size_t(v) * p.dim;
  for (int c0 = 0; c0 < p.dim; c0 += 32 * 8) {  // up to 8 columns per lane in registers
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
    for (long long q0 = 0; q0 < npos; q0 += 32) {
      const long long q = q0 + lane;
      bool hit = false;
      if (q < npos) {
        const int b = int(q / p.len);
        hit = int(p.x[size_t(b) * p.ldx + (q - (long long)b * p.len)]) == v;
      }
      unsigned m = __ballot_sync(0xffffffffu, hit);
      while (m) {  // matching positions in ascending order
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const float* d = p.dy + size_t(q0 + j) * p.dim;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int c = c0 + k * 32 + lane;
          if (c < p.dim) acc[k] = __fadd_rn(acc[k], __ldg(d + c));
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = c0 + k * 32 + lane;
      if (c < p.dim) out[c] = acc[k];
    }
  }
}

}  // namespace hnn

extern "C" int hnn_embedding(int op, const hnn_embed_problem* probs, int nprob, int total_blocks,
                             const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_blocks > 0, "hnn_embedding", "bad arguments");
  HNN_REQUIRE(op == HNN_FWD || op == HNN_WGRAD, "hnn_embedding", "op must be HNN_FWD or HNN_WGRAD");
  cudaStream_t s = hnn::as_stream(stream);
  if (op == HNN_FWD)
    hnn::launch_pdl(hnn::embed_fwd_kernel, dim3(total_blocks), dim3(32 * hnn::EM_WARPS), 0, s, probs, nprob, cur, status);
  else
    hnn::launch_pdl(hnn::embed_bwd_kernel, dim3(total_blocks), dim3(32 * hnn::EM_WARPS), 0, s, probs, nprob, cur, status);
  return hnn::check_launch("hnn_embedding");
}
