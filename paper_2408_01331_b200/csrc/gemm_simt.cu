// Grouped fp32 GEMM on CUDA cores for the dense layers (HNN_PREC_F32_SIMT).
//
// One CTA = one BM x BN output tile of one problem; the tile list of a launch is
// the concatenation of every problem's own tiles, so a problem's tiling (and
// therefore its bits) never depends on its neighbours.  K is walked in BK-wide
// slabs staged in shared memory, double-buffered through registers (the next
// slab's global loads are in flight while the current one is multiplied).
// 64x64 tiles; used for every shape the tcgen05 path and the small-dimension kernels
// (gemm_skinny.cu) do not take, and as the reference-precision path.
#include "common.cuh"

namespace hnn {

constexpr int STHREADS = 256;

template <int BM, int BN>
struct SimtTile {
  static constexpr int BK = 16;
  static constexpr int TM = BM / 16;          // rows per thread  (16 x 16 thread grid)
  static constexpr int TN = BN / 16;          // cols per thread
  static constexpr int A_LD = (BM * BK) / STHREADS;  // A elements each thread stages per slab
  static constexpr int B_LD = (BN * BK) / STHREADS;
};

template <int OP, int BM, int BN>
__global__ void __launch_bounds__(STHREADS) gemm_simt_kernel(const hnn_gemm_problem* __restrict__ probs, int nprob,
                                                             const hnn_step_row* __restrict__ cur,
                                                             const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  using T = SimtTile<BM, BN>;
  constexpr int BK = T::BK, TM = T::TM, TN = T::TN;
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int tile = blockIdx.x;
  const int pi = find_problem(probs, nprob, tile, [](const hnn_gemm_problem& q) { return q.tile_base; });
  const hnn_gemm_problem p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int t = tile - p.tile_base;
  const int m0 = (t / p.tiles_n) * BM, n0 = (t % p.tiles_n) * BN;
  // FWD/DGRAD: M = cap rows, only the first `rows` are real; WGRAD: K = rows.
  const int m_lim = (OP == HNN_WGRAD) ? p.m : min(p.m, rows);
  const int k_lim = (OP == HNN_WGRAD) ? rows : p.k;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

  // staging coordinates: each thread owns A_LD (resp. B_LD) slab elements
  auto a_coord = [&](int r, int& mm, int& kk) {
    const int e = tid + r * STHREADS;
    if (OP == HNN_WGRAD) { mm = e % BM; kk = e / BM; }   // A(m,k) = a[k*lda + m]: threads along m
    else { kk = e % BK; mm = e / BK; }                  // A(m,k) = a[m*lda + k]: threads along k
  };
  auto b_coord = [&](int r, int& kk, int& nn) {
    const int e = tid + r * STHREADS;
    if (OP == HNN_FWD) { kk = e % BK; nn = e / BK; }    // B(k,n) = b[n*ldb + k]
    else { nn = e % BN; kk = e / BN; }                  // B(k,n) = b[k*ldb + n]
  };
  float ra[T::A_LD], rb[T::B_LD];
  auto load_slab = [&](int k0) {
#pragma unroll
    for (int r = 0; r < T::A_LD; ++r) {
      int mm, kk;
      a_coord(r, mm, kk);
      const int gm = m0 + mm, gk = k0 + kk;
      ra[r] = (gm < m_lim && gk < k_lim)
                  ? ((OP == HNN_WGRAD) ? __ldg(p.a + size_t(gk) * p.lda + gm) : __ldg(p.a + size_t(gm) * p.lda + gk))
                  : 0.0f;
    }
#pragma unroll
    for (int r = 0; r < T::B_LD; ++r) {
      int kk, nn;
      b_coord(r, kk, nn);
      const int gn = n0 + nn, gk = k0 + kk;
      rb[r] = (gn < p.n && gk < k_lim)
                  ? ((OP == HNN_FWD) ? __ldg(p.b + size_t(gn) * p.ldb + gk) : __ldg(p.b + size_t(gk) * p.ldb + gn))
                  : 0.0f;
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;
  float bsum = -0.0f;  // bias-gradient column sum (WGRAD, tiles with n0 == 0), row order like numpy

  if (m0 < m_lim) {
    load_slab(0);
    for (int k0 = 0; k0 < k_lim; k0 += BK) {
#pragma unroll
      for (int r = 0; r < T::A_LD; ++r) {
        int mm, kk;
        a_coord(r, mm, kk);
        As[kk][mm] = ra[r];
      }
#pragma unroll
      for (int r = 0; r < T::B_LD; ++r) {
        int kk, nn;
        b_coord(r, kk, nn);
        Bs[kk][nn] = rb[r];
      }
      __syncthreads();
      if (k0 + BK < k_lim) load_slab(k0 + BK);  // next slab in flight during the FMAs
      if (OP == HNN_WGRAD && (p.dbias != nullptr || p.opt_b != nullptr) && n0 == 0 && tid < BM) {
        const int kmax = min(BK, k_lim - k0);
        for (int kk = 0; kk < kmax; ++kk) bsum = __fadd_rn(bsum, As[kk][tid]);
      }
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
        for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }

  if (OP == HNN_WGRAD && (p.dbias != nullptr || p.opt_b != nullptr) && n0 == 0 && tid < BM && m0 + tid < p.m) {
    if (p.dbias) p.dbias[m0 + tid] = bsum;
    if (p.opt_b) {
      const Update u = make_update(cur[p.model], p.opt_kind, p.opt_momentum);
      const int i = m0 + tid;
      float w = p.opt_b[i], m = p.opt_bm ? p.opt_bm[i] : 0.0f, v = p.opt_bv ? p.opt_bv[i] : 0.0f;
      update_sgd(u, w, bsum, m);
      p.opt_b[i] = w;
      if (p.opt_bm) p.opt_bm[i] = m;
      if (p.opt_bv) p.opt_bv[i] = v;
    }
  }
  if (OP == HNN_WGRAD && p.opt_w != nullptr) {
    // fused optimizer: update W (and its moments) with the finished gradient tile
    const Update u = make_update(cur[p.model], p.opt_kind, p.opt_momentum);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int gm = m0 + ty * TM + i;
      if (gm >= p.m) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int gn = n0 + tx * TN + j;
        if (gn >= p.n) continue;
        const size_t off = size_t(gm) * p.ldc + gn;
        float w = p.opt_w[off], m = p.opt_wm ? p.opt_wm[off] : 0.0f, v = p.opt_wv ? p.opt_wv[off] : 0.0f;
        update_sgd(u, w, acc[i][j], m);
        p.opt_w[off] = w;
        if (p.opt_wm) p.opt_wm[off] = m;
        if (p.opt_wv) p.opt_wv[off] = v;
      }
    }
    if (p.c == nullptr) return;
  }

  // ---- epilogue (float4 stores when the row segment is aligned and in range)
  const bool vec = (TN == 4) && ((p.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(p.c) & 15) == 0) &&
                   (!p.mask || (reinterpret_cast<uintptr_t>(p.mask) & 15) == 0);
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty * TM + i;
    if (gm >= p.m) continue;
    const int gn0 = n0 + tx * TN;
    float v[TN];
#pragma unroll
    for (int j = 0; j < TN; ++j) v[j] = acc[i][j];
    if (vec && gn0 + 3 < p.n) {
      if (OP == HNN_FWD) {
        const float4 b4 = *reinterpret_cast<const float4*>(p.bias + gn0);
        const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[j] = (gm >= rows) ? 0.0f : __fadd_rn(v[j], bb[j]);
          if (p.relu && gm < rows) v[j] = np_relu(v[j]);
        }
      } else if (OP == HNN_DGRAD) {
        if (gm >= rows) {
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = 0.0f;
        } else if (p.mask) {
          const float4 m4 = *reinterpret_cast<const float4*>(p.mask + size_t(gm) * p.ldc + gn0);
          v[0] = np_mask(v[0], m4.x);
          v[1] = np_mask(v[1], m4.y);
          v[2] = np_mask(v[2], m4.z);
          v[3] = np_mask(v[3], m4.w);
        }
      }
      *reinterpret_cast<float4*>(p.c + size_t(gm) * p.ldc + gn0) = make_float4(v[0], v[1], v[2], v[3]);
      continue;
    }
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gn = gn0 + j;
      if (gn >= p.n) continue;
      float x = v[j];
      if (OP == HNN_FWD) {
        if (gm >= rows) x = 0.0f;
        else {
          x = __fadd_rn(x, p.bias[gn]);
          if (p.relu) x = np_relu(x);
        }
      } else if (OP == HNN_DGRAD) {
        if (gm >= rows) x = 0.0f;
        else if (p.mask) x = np_mask(x, p.mask[size_t(gm) * p.ldc + gn]);
      }
      p.c[size_t(gm) * p.ldc + gn] = x;
    }
  }
}

// Defined in gemm_skinny.cu: the small-dimension (<= 16) streaming kernels.
int grouped_gemm_skinny(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                        const hnn_model_status* status, cudaStream_t s);
int skinny_tile_shape(int op, int32_t* tm, int32_t* tn);

int grouped_gemm_simt(int op, int skinny, const hnn_gemm_problem* probs, int nprob, int total_tiles,
                      const hnn_step_row* cur, const hnn_model_status* status, cudaStream_t s) {
  if (skinny) return grouped_gemm_skinny(op, probs, nprob, total_tiles, cur, status, s);
  if (op == HNN_FWD) hnn::launch_pdl(gemm_simt_kernel<HNN_FWD, 64, 64>, dim3(total_tiles), dim3(STHREADS), 0, s, probs, nprob, cur, status);
  else if (op == HNN_DGRAD) hnn::launch_pdl(gemm_simt_kernel<HNN_DGRAD, 64, 64>, dim3(total_tiles), dim3(STHREADS), 0, s, probs, nprob, cur, status);
  else hnn::launch_pdl(gemm_simt_kernel<HNN_WGRAD, 64, 64>, dim3(total_tiles), dim3(STHREADS), 0, s, probs, nprob, cur, status);
  return check_launch("hnn_grouped_gemm(simt)");
}

// Defined in gemm_tc.cu.
int grouped_gemm_tc(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                    const hnn_model_status* status, cudaStream_t s);
int gemm_tc_tile_shape(int op, int32_t* tm, int32_t* tn);
// Defined in gemm_tc2.cu (CTA-pair tcgen05 kernel).
int grouped_gemm_tc2(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                     const hnn_model_status* status, cudaStream_t s);
int gemm_tc2_tile_shape(int op, int32_t* tm, int32_t* tn);
int gemm_tc2_chunk_terms();
int grouped_gemm_bf16(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                      const hnn_model_status* status, cudaStream_t s);

}  // namespace hnn

extern "C" int hnn_gemm_tile_shape(int op, int prec, int32_t* tile_m, int32_t* tile_n) {
  HNN_REQUIRE(tile_m && tile_n && op >= HNN_FWD && op <= HNN_WGRAD, "hnn_gemm_tile_shape", "bad arguments");
  if (prec == HNN_PREC_F32_SIMT) {
    *tile_m = 64;
    *tile_n = 64;
    return HNN_OK;
  }
  if (prec == HNN_PREC_F32_SIMT_SKINNY) return hnn::skinny_tile_shape(op, tile_m, tile_n);
  if (prec == HNN_PREC_F32_3XTF32) return hnn::gemm_tc_tile_shape(op, tile_m, tile_n);
  if (prec == HNN_PREC_F32_3XTF32_PAIR || prec == HNN_PREC_BF16_PAIR) return hnn::gemm_tc2_tile_shape(op, tile_m, tile_n);
  hnn::set_error("hnn_gemm_tile_shape", "unknown precision");
  return HNN_ERR_INVALID;
}

extern "C" int hnn_gemm_chunk_terms(int prec, int32_t* terms) {
  HNN_REQUIRE(terms && prec == HNN_PREC_F32_3XTF32_PAIR, "hnn_gemm_chunk_terms", "bad arguments");
  *terms = hnn::gemm_tc2_chunk_terms();
  return HNN_OK;
}

extern "C" int hnn_grouped_gemm(int op, int prec, const hnn_gemm_problem* probs, int nprob, int total_tiles,
                                const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_tiles > 0, "hnn_grouped_gemm", "bad arguments");
  HNN_REQUIRE(op >= HNN_FWD && op <= HNN_WGRAD, "hnn_grouped_gemm", "unknown op");
  cudaStream_t s = hnn::as_stream(stream);
  if (prec == HNN_PREC_F32_SIMT || prec == HNN_PREC_F32_SIMT_SKINNY)
    return hnn::grouped_gemm_simt(op, prec == HNN_PREC_F32_SIMT_SKINNY, probs, nprob, total_tiles, cur, status, s);
  if (prec == HNN_PREC_F32_3XTF32) return hnn::grouped_gemm_tc(op, probs, nprob, total_tiles, cur, status, s);
  if (prec == HNN_PREC_F32_3XTF32_PAIR) return hnn::grouped_gemm_tc2(op, probs, nprob, total_tiles, cur, status, s);
  if (prec == HNN_PREC_BF16_PAIR) return hnn::grouped_gemm_bf16(op, probs, nprob, total_tiles, cur, status, s);
  hnn::set_error("hnn_grouped_gemm", "unknown precision");
  return HNN_ERR_INVALID;
}
