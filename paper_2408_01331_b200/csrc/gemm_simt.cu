// Grouped fp32 GEMM on CUDA cores for the dense layers (HNN_PREC_F32_SIMT).
//
// One CTA = one 64x64 output tile of one problem; the tile list of a launch
// is the concatenation of every problem's own tiles, so a problem's tiling
// (and therefore its bits) never depends on its neighbours.  K is walked in
// 16-wide slabs staged in shared memory; each thread owns a 4x4 micro-tile.
// Used for every shape the tcgen05 path does not take (small N/K, odd strides)
// and as the reference-precision path.
#include "common.cuh"

namespace hnn {

constexpr int SBM = 64, SBN = 64, SBK = 16, STHREADS = 256;

template <int OP>
__global__ void __launch_bounds__(STHREADS) gemm_simt_kernel(const hnn_gemm_problem* __restrict__ probs, int nprob,
                                                             const hnn_step_row* __restrict__ cur,
                                                             const hnn_model_status* __restrict__ status) {
  __shared__ float As[SBK][SBM + 4];
  __shared__ float Bs[SBK][SBN + 4];
  const int tile = blockIdx.x;
  const int pi = find_problem(probs, nprob, tile, [](const hnn_gemm_problem& q) { return q.tile_base; });
  const hnn_gemm_problem p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int t = tile - p.tile_base;
  const int m0 = (t / p.tiles_n) * SBM, n0 = (t % p.tiles_n) * SBN;
  // FWD/DGRAD: M = cap rows, only the first `rows` are real; WGRAD: K = rows.
  const int m_lim = (OP == HNN_WGRAD) ? p.m : min(p.m, rows);
  const int k_lim = (OP == HNN_WGRAD) ? rows : p.k;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  float bsum = -0.0f;  // bias-gradient column sum (WGRAD, tiles with n0 == 0), row order like numpy

  if (m0 < m_lim) {
    for (int k0 = 0; k0 < k_lim; k0 += SBK) {
      // ---- stage A[m0:+64, k0:+16] as As[k][m]
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int kk, mm;
        if (OP == HNN_WGRAD) { mm = tid & 63; kk = (tid >> 6) + 4 * r; }   // A(m,k) = a[k*lda + m]
        else { kk = tid & 15; mm = (tid >> 4) + 16 * r; }                 // A(m,k) = a[m*lda + k]
        const int gm = m0 + mm, gk = k0 + kk;
        float v = 0.0f;
        if (gm < m_lim && gk < k_lim)
          v = (OP == HNN_WGRAD) ? __ldg(p.a + size_t(gk) * p.lda + gm) : __ldg(p.a + size_t(gm) * p.lda + gk);
        As[kk][mm] = v;
      }
      // ---- stage B[k0:+16, n0:+64] as Bs[k][n]
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int kk, nn;
        if (OP == HNN_FWD) { kk = tid & 15; nn = (tid >> 4) + 16 * r; }   // B(k,n) = b[n*ldb + k]
        else { nn = tid & 63; kk = (tid >> 6) + 4 * r; }                 // B(k,n) = b[k*ldb + n]
        const int gn = n0 + nn, gk = k0 + kk;
        float v = 0.0f;
        if (gn < p.n && gk < k_lim)
          v = (OP == HNN_FWD) ? __ldg(p.b + size_t(gn) * p.ldb + gk) : __ldg(p.b + size_t(gk) * p.ldb + gn);
        Bs[kk][nn] = v;
      }
      __syncthreads();
      if (OP == HNN_WGRAD && p.dbias != nullptr && n0 == 0 && tid < SBM) {
        const int kmax = min(SBK, k_lim - k0);
        for (int kk = 0; kk < kmax; ++kk) bsum = __fadd_rn(bsum, As[kk][tid]);
      }
#pragma unroll
      for (int kk = 0; kk < SBK; ++kk) {
        const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
        const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }

  if (OP == HNN_WGRAD && p.dbias != nullptr && n0 == 0 && tid < SBM && m0 + tid < p.m) p.dbias[m0 + tid] = bsum;

  // ---- epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= p.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= p.n) continue;
      float v = acc[i][j];
      if (OP == HNN_FWD) {
        if (gm >= rows) v = 0.0f;
        else {
          v = __fadd_rn(v, p.bias[gn]);
          if (p.relu) v = np_relu(v);
        }
      } else if (OP == HNN_DGRAD) {
        if (gm >= rows) v = 0.0f;
        else if (p.mask) v = np_mask(v, p.mask[size_t(gm) * p.ldc + gn]);
      }
      p.c[size_t(gm) * p.ldc + gn] = v;
    }
  }
}

int grouped_gemm_simt(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                      const hnn_model_status* status, cudaStream_t s) {
  if (op == HNN_FWD) gemm_simt_kernel<HNN_FWD><<<total_tiles, STHREADS, 0, s>>>(probs, nprob, cur, status);
  else if (op == HNN_DGRAD) gemm_simt_kernel<HNN_DGRAD><<<total_tiles, STHREADS, 0, s>>>(probs, nprob, cur, status);
  else gemm_simt_kernel<HNN_WGRAD><<<total_tiles, STHREADS, 0, s>>>(probs, nprob, cur, status);
  return check_launch("hnn_grouped_gemm(simt)");
}

// Defined in gemm_tc.cu when the tcgen05 path is built.
int grouped_gemm_tc(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                    const hnn_model_status* status, cudaStream_t s);
int gemm_tc_tile_shape(int op, int32_t* tm, int32_t* tn);

}  // namespace hnn

extern "C" int hnn_gemm_tile_shape(int op, int prec, int32_t* tile_m, int32_t* tile_n) {
  HNN_REQUIRE(tile_m && tile_n && op >= HNN_FWD && op <= HNN_WGRAD, "hnn_gemm_tile_shape", "bad arguments");
  if (prec == HNN_PREC_F32_SIMT) {
    *tile_m = hnn::SBM;
    *tile_n = hnn::SBN;
    return HNN_OK;
  }
  if (prec == HNN_PREC_F32_3XTF32) return hnn::gemm_tc_tile_shape(op, tile_m, tile_n);
  hnn::set_error("hnn_gemm_tile_shape", "unknown precision");
  return HNN_ERR_INVALID;
}

extern "C" int hnn_grouped_gemm(int op, int prec, const hnn_gemm_problem* probs, int nprob, int total_tiles,
                                const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_tiles > 0, "hnn_grouped_gemm", "bad arguments");
  HNN_REQUIRE(op >= HNN_FWD && op <= HNN_WGRAD, "hnn_grouped_gemm", "unknown op");
  if (prec == HNN_PREC_F32_SIMT) return hnn::grouped_gemm_simt(op, probs, nprob, total_tiles, cur, status, hnn::as_stream(stream));
  if (prec == HNN_PREC_F32_3XTF32) return hnn::grouped_gemm_tc(op, probs, nprob, total_tiles, cur, status, hnn::as_stream(stream));
  hnn::set_error("hnn_grouped_gemm", "unknown precision");
  return HNN_ERR_INVALID;
}
