// Grouped implicit-GEMM convolution, NCHW, fp32 (replaces im2col + matmul/einsum,
// pkg/src/hybridnn/ops.py:91-130).  No im2col buffer is ever materialised:
// the A/B slabs are gathered straight from the activations into shared memory.
//
//   FWD   M = cap*OH*OW (output pixels)  N = F  K = C*k*k
//   DGRAD M = cap*H*W   (input pixels)   N = C  K = F*k*k   (transposed conv, gather form, no atomics)
//   WGRAD M = F                          N = C*k*k + 1 (last column = bias grad)
//         K = rows*OH*OW cut into fixed `split_len` chunks -> partials, then a fixed-order reduce.
#include "common.cuh"

namespace hnn {

constexpr int CBM = 64, CBN = 32, CBK = 16, CTHREADS = 128;

struct ConvGeom {
  int c, h, w, f, k, s, pad, oh, ow, kk2, ckk, fkk, ohw, hw;
  __device__ ConvGeom(const hnn_conv_problem& p)
      : c(p.c), h(p.h), w(p.w), f(p.f), k(p.k), s(p.stride), pad(p.pad), oh(p.oh), ow(p.ow) {
    kk2 = k * k;
    ckk = c * kk2;
    fkk = f * kk2;
    ohw = oh * ow;
    hw = h * w;
  }
};

// x value at im2col(row m of output pixels, column kk), zero outside the padded image.
__device__ __forceinline__ float im2col_at(const float* __restrict__ x, const ConvGeom& g, int b, int opix, int kk) {
  const int oy = opix / g.ow, ox = opix - oy * g.ow;
  const int ci = kk / g.kk2, r = kk - ci * g.kk2;
  const int i = r / g.k, j = r - i * g.k;
  const int iy = oy * g.s + i - g.pad, ix = ox * g.s + j - g.pad;
  if (iy < 0 || iy >= g.h || ix < 0 || ix >= g.w) return 0.0f;
  return __ldg(x + ((size_t(b) * g.c + ci) * g.h + iy) * g.w + ix);
}

template <int OP>
__global__ void __launch_bounds__(CTHREADS) conv_kernel(const hnn_conv_problem* __restrict__ probs, int nprob,
                                                        const hnn_step_row* __restrict__ cur,
                                                        const hnn_model_status* __restrict__ status) {
  __shared__ float As[CBK][CBM + 4];
  __shared__ float Bs[CBK][CBN + 4];
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_conv_problem& q) { return q.tile_base; });
  const hnn_conv_problem p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const ConvGeom g(p);
  const int rows = cur[p.model].rows;
  int t = blockIdx.x - p.tile_base;
  int split = 0;
  int M, N, K, m_real;
  if (OP == HNN_FWD) { M = p.cap * g.ohw; N = g.f; K = g.ckk; m_real = rows * g.ohw; }
  else if (OP == HNN_DGRAD) { M = p.cap * g.hw; N = g.c; K = g.fkk; m_real = rows * g.hw; }
  else {
    M = g.f; N = g.ckk + 1; m_real = M;
    const int per_split = ((M + CBM - 1) / CBM) * p.tiles_n;
    split = t / per_split;
    t -= split * per_split;
    K = p.split_len;
  }
  const int m0 = (t / p.tiles_n) * CBM, n0 = (t % p.tiles_n) * CBN;
  const int kbeg = (OP == HNN_WGRAD) ? split * p.split_len : 0;
  const int kend = (OP == HNN_WGRAD) ? min(kbeg + p.split_len, rows * g.ohw) : K;
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;  // 8 x 16 threads, 4x4 micro-tiles (32 x 64)

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  if (m0 < m_real) {
    for (int k0 = kbeg; k0 < kend; k0 += CBK) {
      // ---- A slab As[k][m]
#pragma unroll
      for (int r = 0; r < (CBM * CBK) / CTHREADS; ++r) {
        const int e = tid + r * CTHREADS;
        const int mm = e & (CBM - 1), kk = e >> 6;
        const int gm = m0 + mm, gk = k0 + kk;
        float v = 0.0f;
        if (gm < m_real && gk < kend) {
          if (OP == HNN_FWD) {
            const int b = gm / g.ohw;
            v = im2col_at(p.x, g, b, gm - b * g.ohw, gk);
          } else if (OP == HNN_DGRAD) {
            // A(m = input pixel (b,y,x), kk = (f,i,j)) = dy[b,f,oy,ox] with y = oy*s + i - pad
            const int b = gm / g.hw, pix = gm - b * g.hw;
            const int y = pix / g.w, xx = pix - y * g.w;
            const int fi = gk / g.kk2, r2 = gk - fi * g.kk2;
            const int i = r2 / g.k, j = r2 - i * g.k;
            const int ny = y + g.pad - i, nx = xx + g.pad - j;
            if (ny >= 0 && nx >= 0 && ny % g.s == 0 && nx % g.s == 0) {
              const int oy = ny / g.s, ox = nx / g.s;
              if (oy < g.oh && ox < g.ow) v = __ldg(p.dy + ((size_t(b) * g.f + fi) * g.oh + oy) * g.ow + ox);
            }
          } else {
            // A(m = f, k = (b, opix)) = dy[b, f, opix]
            const int b = gk / g.ohw, opix = gk - b * g.ohw;
            v = __ldg(p.dy + (size_t(b) * g.f + gm) * g.ohw + opix);
          }
        }
        As[kk][mm] = v;
      }
      // ---- B slab Bs[k][n]
#pragma unroll
      for (int r = 0; r < (CBN * CBK) / CTHREADS; ++r) {
        const int e = tid + r * CTHREADS;
        const int nn = e & (CBN - 1), kk = e >> 5;
        const int gn = n0 + nn, gk = k0 + kk;
        float v = 0.0f;
        if (gn < N && gk < kend) {
          if (OP == HNN_FWD) v = __ldg(p.weight + size_t(gn) * g.ckk + gk);                 // w[f, kk]
          else if (OP == HNN_DGRAD) {
            const int fi = gk / g.kk2, r2 = gk - fi * g.kk2;                        // w[f, c, i, j]
            v = __ldg(p.weight + (size_t(fi) * g.c + gn) * g.kk2 + r2);
          } else {
            const int b = gk / g.ohw, opix = gk - b * g.ohw;
            v = (gn == g.ckk) ? 1.0f : im2col_at(p.x, g, b, opix, gn);
          }
        }
        Bs[kk][nn] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < CBK; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if (OP == HNN_FWD) {
        const int b = gm / g.ohw, opix = gm - b * g.ohw;
        if (gm >= m_real) v = 0.0f;
        else {
          v = __fadd_rn(v, p.bias[gn]);
          if (p.relu) v = np_relu(v);
        }
        p.y[(size_t(b) * g.f + gn) * g.ohw + opix] = v;
      } else if (OP == HNN_DGRAD) {
        const int b = gm / g.hw, pix = gm - b * g.hw;
        const size_t off = (size_t(b) * g.c + gn) * g.hw + pix;
        if (gm >= m_real) v = 0.0f;
        else if (p.mask) v = np_mask(v, p.mask[off]);
        p.dx[off] = v;
      } else {
        p.partial[(size_t(split) * g.f + gm) * (g.ckk + 1) + gn] = v;
      }
    }
  }
}

// dw / db = ordered sum over the splits of the partials; one thread per output element.
__global__ void conv_wgrad_reduce_kernel(const hnn_conv_problem* __restrict__ probs, int nprob,
                                         const hnn_step_row* __restrict__ cur,
                                         const hnn_model_status* __restrict__ status) {
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_conv_problem& q) { return q.tile_base; });
  const hnn_conv_problem p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int ckk = p.c * p.k * p.k, cols = ckk + 1;
  const int e = (blockIdx.x - p.tile_base) * blockDim.x + threadIdx.x;
  if (e >= p.f * cols) return;
  const int fi = e / cols, col = e - fi * cols;
  float acc = p.partial[size_t(fi) * cols + col];
  for (int s = 1; s < p.splits; ++s) acc = __fadd_rn(acc, p.partial[(size_t(s) * p.f + fi) * cols + col]);
  if (col == ckk) p.db[fi] = acc;
  else p.dw[size_t(fi) * ckk + col] = acc;
}

}  // namespace hnn

extern "C" int hnn_conv_tile_shape(int op, int32_t* tile_m, int32_t* tile_n) {
  HNN_REQUIRE(tile_m && tile_n, "hnn_conv_tile_shape", "null pointer");
  *tile_m = hnn::CBM;
  *tile_n = hnn::CBN;
  return HNN_OK;
}

extern "C" int hnn_grouped_conv(int op, const hnn_conv_problem* probs, int nprob, int total_tiles,
                                const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_tiles > 0, "hnn_grouped_conv", "bad arguments");
  cudaStream_t s = hnn::as_stream(stream);
  if (op == HNN_FWD) hnn::conv_kernel<HNN_FWD><<<total_tiles, hnn::CTHREADS, 0, s>>>(probs, nprob, cur, status);
  else if (op == HNN_DGRAD) hnn::conv_kernel<HNN_DGRAD><<<total_tiles, hnn::CTHREADS, 0, s>>>(probs, nprob, cur, status);
  else if (op == HNN_WGRAD) hnn::conv_kernel<HNN_WGRAD><<<total_tiles, hnn::CTHREADS, 0, s>>>(probs, nprob, cur, status);
  else {
    hnn::set_error("hnn_grouped_conv", "unknown op");
    return HNN_ERR_INVALID;
  }
  return hnn::check_launch("hnn_grouped_conv");
}

// For the reduce, probs[i].tile_base indexes 256-thread blocks over F*(C*k*k+1) outputs.
extern "C" int hnn_conv_wgrad_reduce(const hnn_conv_problem* probs, int nprob, int total_blocks,
                                     const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_blocks > 0, "hnn_conv_wgrad_reduce", "bad arguments");
  hnn::conv_wgrad_reduce_kernel<<<total_blocks, 256, 0, hnn::as_stream(stream)>>>(probs, nprob, cur, status);
  return hnn::check_launch("hnn_conv_wgrad_reduce");
}
