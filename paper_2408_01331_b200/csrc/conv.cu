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
  hnn::pdl_wait();
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
  hnn::pdl_wait();
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_conv_problem& q) { return q.tile_base; });
  const hnn_conv_problem p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int ckk = p.c * p.k * p.k, cols = ckk + 1;
  const int e = (blockIdx.x - p.tile_base) * blockDim.x + threadIdx.x;
  if (e >= p.f * cols) return;
  const int fi = e / cols, col = e - fi * cols;
  // splits added in order; 16 partials' loads are in flight before their (sequential) adds (one
  // load per dependent add left the LeNet reduce latency-bound: 27 us for 12 MB)
  const float* src = p.partial + size_t(fi) * cols + col;
  const size_t stride = size_t(p.f) * cols;
  float acc = __ldg(src);
  int s = 1;
  for (; s + 16 <= p.splits; s += 16) {
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldg(src + (s + u) * stride);
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, v[u]);
  }
  for (; s < p.splits; ++s) acc = __fadd_rn(acc, __ldg(src + s * stride));
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
  if (op == HNN_FWD) hnn::launch_pdl(hnn::conv_kernel<HNN_FWD>, dim3(total_tiles), dim3(hnn::CTHREADS), 0, s, probs, nprob, cur, status);
  else if (op == HNN_DGRAD) hnn::launch_pdl(hnn::conv_kernel<HNN_DGRAD>, dim3(total_tiles), dim3(hnn::CTHREADS), 0, s, probs, nprob, cur, status);
  else if (op == HNN_WGRAD) hnn::launch_pdl(hnn::conv_kernel<HNN_WGRAD>, dim3(total_tiles), dim3(hnn::CTHREADS), 0, s, probs, nprob, cur, status);
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
  hnn::launch_pdl(hnn::conv_wgrad_reduce_kernel, dim3(total_blocks), dim3(256), 0, hnn::as_stream(stream), probs, nprob, cur, status);
  return hnn::check_launch("hnn_conv_wgrad_reduce");
}

// ---------------------------------------------------------------------------------------------
// Direct convolution for small layers (LeNet-class: one sample's activations plus the whole
// filter bank fit in shared memory), where a 64x32 implicit-GEMM tile would be mostly padding.
// One CTA per (problem, sample) for FWD / DGRAD and per (problem, batch chunk of
// HNN_CONV_DIRECT_BCHUNK samples) for WGRAD; the sample's input (or output gradient) and the
// filters are staged in shared memory and every thread sweeps outputs with fixed-order FMAs.
// WGRAD writes per-chunk partials that hnn_conv_wgrad_reduce sums in chunk order (no atomics).
// probs[i].tile_base counts CTAs.
namespace hnn {

constexpr int DTHREADS = 256;

// Shared-memory layouts of the direct kernels, chosen so that the addresses one warp instruction
// touches fall into distinct banks (ncu, profiles/r02/ncu_direct_c2_v4.txt: 70% of the LeNet conv1
// forward's shared wavefronts and 61% of its weight gradient's were bank conflicts):
//  * x rows at a stride of 1 mod 32 words: the forward's lanes (output row, 4-column block) then
//    read banks oy + 4 * block (at most 2-way for 28-wide rows);
//  * x channels at a stride of K mod 32: the weight gradient's lanes, which own filter rows
//    (f, c, i), read input row (c, i) at bank c * K + i (+ f-independent), distinct for C * K <= 32;
//  * dy planes at a stride of 1 mod 32: lanes of different filters f read distinct banks.
__host__ __device__ inline int up_to_residue(int x, int r) { return x + ((r - x) % 32 + 32) % 32; }
struct DirectLayout {
  int rs, cs, ps;  // x row stride, x channel stride, dy plane stride (floats)
  __host__ __device__ DirectLayout(int c, int h, int w, int k, int oh, int ow) {
    rs = up_to_residue(w, 1);
    cs = up_to_residue(h * rs, k % 32);
    ps = up_to_residue(oh * ow, 1);
  }
};

__device__ __forceinline__ void stage(float* dst, const float* __restrict__ src, int n) {
  // eight loads in flight per thread before their shared-memory stores
  const int step = blockDim.x;
  int i = threadIdx.x;
  for (; i + 7 * step < n; i += 8 * step) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(src + i + u * step);
#pragma unroll
    for (int u = 0; u < 8; ++u) dst[i + u * step] = v[u];
  }
  for (; i < n; i += step) dst[i] = __ldg(src + i);
}

// rows of `w` floats (n rows, planes of `h` rows) into a padded layout: row stride rs, plane stride cs
__device__ __forceinline__ void stage_rows(float* dst, const float* __restrict__ src, int n, int w, int h, int rs,
                                           int cs) {
  const int total = n * w;
  for (int e0 = threadIdx.x; e0 < total; e0 += 8 * blockDim.x) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      v[u] = e < total ? __ldg(src + e) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e >= total) break;
      const int r = e / w, x = e - r * w, pl = r / h;
      dst[pl * cs + (r - pl * h) * rs + x] = v[u];
    }
  }
}

// dy of nplanes (sample, filter) planes starting at plane pl0 of a layer whose 2 x 2 / stride-2
// max-pool backward is folded into the staging (hnn_conv_problem.pool_*): one unit per pool window
// (its gradient, argmax and the relu mask's two row pairs loaded together, every unit's loads issued
// before the first store), maxpool2_bwd's arithmetic (pool_relu.cu), so the staged values are
// bit-identical to the pool launch's dx.  Element (plane, oy, ox) goes to dst[plane * PS + oy * RS + ox].
__device__ __forceinline__ void stage_dy_pooled(float* dst, const hnn_conv_problem& p, size_t pl0, int nplanes,
                                                int PS, int RS) {
  const int pw = p.ow >> 1, pohw = (p.oh >> 1) * pw, ohw = p.oh * p.ow;
  const int total = nplanes * pohw;
  constexpr int U = 4;
  for (int e0 = threadIdx.x; e0 < total; e0 += U * blockDim.x) {
    float d[U];
    int ix[U];
    float2 m0[U], m1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * blockDim.x;
      d[u] = 0.0f;
      ix[u] = -1;
      m0[u] = m1[u] = make_float2(1.0f, 1.0f);
      if (e < total) {
        const int pl = e / pohw, t = e - pl * pohw, wy = t / pw, wx = t - wy * pw;
        const size_t o = pl0 * pohw + e;
        d[u] = __ldg(p.pool_dy + o);
        ix[u] = __ldg(p.pool_idx + o);
        if (p.pool_mask) {
          const float* mk = p.pool_mask + (pl0 + pl) * ohw + (2 * wy) * p.ow + 2 * wx;
          m0[u] = __ldg(reinterpret_cast<const float2*>(mk));
          m1[u] = __ldg(reinterpret_cast<const float2*>(mk + p.ow));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e >= total) break;
      const int pl = e / pohw, t = e - pl * pohw, wy = t / pw, wx = t - wy * pw;
      float g[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) g[k] = __fadd_rn(0.0f, ix[u] == k ? d[u] : 0.0f);  // np.add.at into zeros
      if (p.pool_mask) {
        g[0] = np_mask(g[0], m0[u].x);
        g[1] = np_mask(g[1], m0[u].y);
        g[2] = np_mask(g[2], m1[u].x);
        g[3] = np_mask(g[3], m1[u].y);
      }
      float* o = dst + pl * PS + (2 * wy) * RS + 2 * wx;
      o[0] = g[0];
      o[1] = g[1];
      o[RS] = g[2];
      o[RS + 1] = g[3];
    }
  }
}

// pooled elements per thread per round (loads in flight) and the pooled forward's CTAs-per-SM bound:
// 1 unit at 3 CTAs per SM (80 registers, no spills) measured C2 0.4245 ms against 0.4264 for 2, 4
// or 8 units at 2 CTAs per SM (4 units at 3 CTAs spilled 700 bytes), profiles/r02/pool_fold_ab_v15.txt
#ifndef HNN_POOLX_UNITS
#define HNN_POOLX_UNITS 1
#endif
#ifndef HNN_POOLX_MINB
#define HNN_POOLX_MINB 3
#endif
constexpr int PXU = HNN_POOLX_UNITS;
// Forward staging of sample b's input when x is a folded 2 x 2 / stride-2 max-pool of p.pool_x:
// every pooled element is computed once (maxpool2_fwd's numpy-argmax scan, pool_relu.cu), staged,
// and written out as the pool's y (= p.x) and argmax (p.pool_idx) for the backward.
__device__ __forceinline__ void stage_pooled_x(float* dst, const hnn_conv_problem& p, int b, int c, int h, int w,
                                               int rs, int cs) {
  const int hw = h * w, total = c * hw, w2 = 2 * w;
  const float* src = p.pool_x + size_t(b) * c * 4 * hw;
  float* y = const_cast<float*>(p.x) + size_t(b) * total;
  uint8_t* idx = p.pool_idx + size_t(b) * total;
  for (int e0 = threadIdx.x; e0 < total; e0 += PXU * blockDim.x) {
    float2 r0[PXU], r1[PXU];
#pragma unroll
    for (int u = 0; u < PXU; ++u) {
      const int e = e0 + u * blockDim.x;
      r0[u] = r1[u] = make_float2(0.0f, 0.0f);
      if (e < total) {
        const int pl = e / hw, t = e - pl * hw, oy = t / w, ox = t - oy * w;
        const float* s0 = src + size_t(pl) * 4 * hw + (2 * oy) * w2 + 2 * ox;
        r0[u] = __ldg(reinterpret_cast<const float2*>(s0));
        r1[u] = __ldg(reinterpret_cast<const float2*>(s0 + w2));
      }
    }
#pragma unroll
    for (int u = 0; u < PXU; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e >= total) break;
      // numpy argmax over (0,0) (0,1) (1,0) (1,1): first max wins, first NaN wins outright
      float best = r0[u].x;
      int best_i = 0;
      bool stop = best != best;
      const auto scan = [&](float v, int k) {
        if (!stop && !(v <= best)) {
          best = v;
          best_i = k;
          stop = v != v;
        }
      };
      scan(r0[u].y, 1);
      scan(r1[u].x, 2);
      scan(r1[u].y, 3);
      const int pl = e / hw, t = e - pl * hw, oy = t / w, ox = t - oy * w;
      dst[pl * cs + oy * rs + ox] = best;
      y[e] = best;
      idx[e] = (uint8_t)best_i;
    }
  }
}

// Register-blocked stride-1 paths (LeNet-class layers): a thread computes 4 consecutive outputs of
// one row, so each staged input row segment (4 + K - 1 values) and each weight are loaded from
// shared memory once for 4 * K FMAs (the one-output-per-thread loop issued 2 shared loads per
// FMA and was bound by the 1-wavefront/clock shared-memory pipe).
constexpr int RB = 4;

// Forward, stride 1: a thread computes FG filters x RB consecutive outputs of one row, so per
// (channel, filter row) it loads one RB + K - 1 input segment and, per tap, the FG filters'
// weights as float4 (weights staged tap-major, filters innermost: wt[(c*K + i)*K + j][f], FP = F
// rounded up to 4) for FG * RB FMAs; a thread-per-filter form loaded a weight per RB FMAs and
// was bound by the shared-memory pipe (ncu: issue 73%, FMA pipe 36% on LeNet conv1).
template <int K, int FG, bool PAD0>
__device__ __forceinline__ void direct_fwd_blocked(const hnn_conv_problem& p, const ConvGeom& g, const float* xs,
                                                   int rs, int cs, const float* wt, int fp, float* yb) {
  const int qblocks = (g.ow + RB - 1) / RB;
  const int groups = (g.f + FG - 1) / FG;
  for (int e = threadIdx.x; e < groups * g.oh * qblocks; e += blockDim.x) {
    const int fg = e / (g.oh * qblocks), rq = e - fg * g.oh * qblocks, oy = rq / qblocks, ox0 = (rq - oy * qblocks) * RB;
    const int f0 = fg * FG;
    float acc[FG][RB];
#pragma unroll
    for (int ff = 0; ff < FG; ++ff)
#pragma unroll
      for (int q = 0; q < RB; ++q) acc[ff][q] = 0.0f;
    for (int c = 0; c < g.c; ++c) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int y = oy - g.pad + i;
        if (!PAD0 && (y < 0 || y >= g.h)) continue;
        const float* xr = xs + c * cs + y * rs;
        float seg[RB + K - 1];
#pragma unroll
        for (int t = 0; t < RB + K - 1; ++t) {
          // (no padding: columns past w are the padded row's tail, used only by outputs >= ow)
          const int x = ox0 - g.pad + t;
          seg[t] = (PAD0 || (x >= 0 && x < g.w)) ? xr[x] : 0.0f;
        }
        const float* wr = wt + size_t((c * K + i) * K) * fp + f0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
#pragma unroll
          for (int f4 = 0; f4 < FG / 4; ++f4) {
            const float4 w = *reinterpret_cast<const float4*>(wr + j * fp + 4 * f4);
#pragma unroll
            for (int q = 0; q < RB; ++q) {
              acc[4 * f4 + 0][q] = fmaf(seg[q + j], w.x, acc[4 * f4 + 0][q]);
              acc[4 * f4 + 1][q] = fmaf(seg[q + j], w.y, acc[4 * f4 + 1][q]);
              acc[4 * f4 + 2][q] = fmaf(seg[q + j], w.z, acc[4 * f4 + 2][q]);
              acc[4 * f4 + 3][q] = fmaf(seg[q + j], w.w, acc[4 * f4 + 3][q]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int ff = 0; ff < FG; ++ff) {
      const int f = f0 + ff;
      if (f >= g.f) break;
      const float bias = __ldg(p.bias + f);
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const int ox = ox0 + q;
        if (ox >= g.ow) break;
        float v = __fadd_rn(acc[ff][q], bias);
        if (p.relu) v = np_relu(v);
        yb[(f * g.oh + oy) * g.ow + ox] = v;
      }
    }
  }
}

// FG for the blocked forward: 8 filters per thread when that still gives the CTA >= 128 work items
__device__ __forceinline__ int fwd_fg(const ConvGeom& g) {
  const int q = (g.ow + RB - 1) / RB;
  return ((g.f + 7) / 8) * g.oh * q >= 128 ? 8 : 4;
}

// Input gradient, stride 1 (the transposed convolution in gather form): a thread computes CG
// channels x RB consecutive inputs of one row from a zero-padded copy of dy (K - 1 zeros around
// every plane: no bounds tests in the loop) and tap-major float4 weights (wt[(f*K + i)*K + j][c],
// channels innermost, CP = C rounded up to 8), CG * RB FMAs per weight load.
struct DgradLayout {
  int pd, rows, rs, plane, cp;  // pad, padded rows, row stride, plane stride, padded channels
  __host__ __device__ DgradLayout(int c, int h, int w, int k, int pad, int oh, int ow) {
    pd = k - 1;
    rows = oh + 2 * pd;
    const int need = ((w + RB - 1) / RB) * RB + pad + k - 1;  // last quad's segment end
    rs = max(ow + 2 * pd, need) | 1;                          // odd: rows spread over banks
    plane = rows * rs;
    cp = (c + 7) & ~7;
  }
};

template <int K, int CG>
__device__ __forceinline__ void direct_dgrad_blocked(const hnn_conv_problem& p, const ConvGeom& g, const DgradLayout& L,
                                                     const float* dp, const float* wt, float* dxb, const float* mb) {
  const int qblocks = (g.w + RB - 1) / RB;
  const int groups = (g.c + CG - 1) / CG;
  for (int e = threadIdx.x; e < groups * g.h * qblocks; e += blockDim.x) {
    const int cg = e / (g.h * qblocks), rq = e - cg * g.h * qblocks, y = rq / qblocks, x0 = (rq - y * qblocks) * RB;
    const int c0 = cg * CG;
    float acc[CG][RB];
#pragma unroll
    for (int cc = 0; cc < CG; ++cc)
#pragma unroll
      for (int q = 0; q < RB; ++q) acc[cc][q] = 0.0f;
    for (int f = 0; f < g.f; ++f) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        // dx[x] gets dy[x + pad - j] * w[j]: seg[t] = dy[y + pad - i][x0 + pad - (K - 1) + t], padded
        const float* dr = dp + f * L.plane + (y + g.pad - i + L.pd) * L.rs + x0 + g.pad;
        float seg[RB + K - 1];
#pragma unroll
        for (int t = 0; t < RB + K - 1; ++t) seg[t] = dr[t];
        const float* wr = wt + size_t((f * K + i) * K) * L.cp + c0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
#pragma unroll
          for (int c4 = 0; c4 < CG / 4; ++c4) {
            const float4 w = *reinterpret_cast<const float4*>(wr + j * L.cp + 4 * c4);
#pragma unroll
            for (int q = 0; q < RB; ++q) {
              const float d = seg[q + K - 1 - j];
              acc[4 * c4 + 0][q] = fmaf(d, w.x, acc[4 * c4 + 0][q]);
              acc[4 * c4 + 1][q] = fmaf(d, w.y, acc[4 * c4 + 1][q]);
              acc[4 * c4 + 2][q] = fmaf(d, w.z, acc[4 * c4 + 2][q]);
              acc[4 * c4 + 3][q] = fmaf(d, w.w, acc[4 * c4 + 3][q]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int cc = 0; cc < CG; ++cc) {
      const int c = c0 + cc;
      if (c >= g.c) break;
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const int x = x0 + q;
        if (x >= g.w) break;
        const int o = (c * g.h + y) * g.w + x;
        dxb[o] = mb ? np_mask(acc[cc][q], mb[o]) : acc[cc][q];
      }
    }
  }
}

// Weight gradient of one staged sample, stride 1: a thread owns FG filters x one input row (c, i)
// and the K taps j of those filter rows, sweeping the output rows of its row group; per 4 outputs it
// loads one 4 + K - 1 input segment and 4 dy values per filter for FG * 4 * K FMAs (one filter per
// thread loaded the segment once per 4 * K FMAs: issue-bound, FMA pipe 27%, profiles/r02).  G row
// groups (fixed) are combined in order.
template <int K, int FG>
__device__ __forceinline__ void direct_wgrad_blocked(const hnn_conv_problem& p, const ConvGeom& g, const float* xs,
                                                     int cs, int rs, const float* ds, int ps, int nb, float* red,
                                                     float* out) {
  const int fgroups = (g.f + FG - 1) / FG;
  const int nrow = fgroups * g.c * K;  // (filter group, c, i) work rows
  const int G = max(1, min(8, int(blockDim.x) / nrow));
  const int cols = g.ckk + 1;
  const int frow = g.f * g.c * K;      // (f, c, i) filter rows of the partial layout
  const int qblocks = (g.ow + RB - 1) / RB;
  for (int t = threadIdx.x; t < nrow * G; t += blockDim.x) {
    const int grp = t / nrow, rrow = t - grp * nrow;
    const int fg = rrow / (g.c * K), ci = rrow - fg * g.c * K, c = ci / K, i = ci - c * K;
    const int f0 = fg * FG;
    float acc[FG][K];
#pragma unroll
    for (int ff = 0; ff < FG; ++ff)
#pragma unroll
      for (int j = 0; j < K; ++j) acc[ff][j] = 0.0f;
    for (int sb = 0; sb < nb; ++sb) {
      const float* xc = xs + (sb * g.c + c) * cs;
      for (int oy = grp; oy < g.oh; oy += G) {
        const int y = oy - g.pad + i;
        if (y < 0 || y >= g.h) continue;
        const float* xr = xc + y * rs;
        for (int qb = 0; qb < qblocks; ++qb) {
          const int ox0 = qb * RB;
          float seg[RB + K - 1];
#pragma unroll
          for (int u = 0; u < RB + K - 1; ++u) {
            const int x = ox0 - g.pad + u;
            seg[u] = (x >= 0 && x < g.w) ? xr[x] : 0.0f;
          }
#pragma unroll
          for (int ff = 0; ff < FG; ++ff) {
            const int f = min(f0 + ff, g.f - 1);  // (a padded filter recomputes the last: discarded)
            const float* dr = ds + (sb * g.f + f) * ps + oy * g.ow;
            float d[RB];
#pragma unroll
            for (int q = 0; q < RB; ++q) d[q] = ox0 + q < g.ow ? dr[ox0 + q] : 0.0f;
#pragma unroll
            for (int j = 0; j < K; ++j)
#pragma unroll
              for (int q = 0; q < RB; ++q) acc[ff][j] = fmaf(d[q], seg[q + j], acc[ff][j]);
          }
        }
      }
    }
    // group 0 -> slot G-1, group g > 0 -> slot g-1 (combined in group order after the barrier)
    const int slot = grp > 0 ? grp - 1 : G - 1;
#pragma unroll
    for (int ff = 0; ff < FG; ++ff) {
      const int f = f0 + ff;
      if (f >= g.f) break;
      const int fr = (f * g.c + c) * K + i;
#pragma unroll
      for (int j = 0; j < K; ++j) red[(slot * frow + fr) * K + j] = acc[ff][j];
    }
  }
  __syncthreads();
  for (int fr = threadIdx.x; fr < frow; fr += blockDim.x) {
    const int f = fr / (g.c * K), ci = fr - f * g.c * K, c = ci / K, i = ci - c * K;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      float a = red[((G - 1) * frow + fr) * K + j];  // group 0
      for (int grp = 1; grp < G; ++grp) a = __fadd_rn(a, red[((grp - 1) * frow + fr) * K + j]);
      out[f * cols + c * K * K + i * K + j] = a;
    }
  }
  // bias gradient: sequential sum of the staged samples' dy per filter
  for (int f = threadIdx.x; f < g.f; f += blockDim.x) {
    float a = 0.0f;
    for (int sb = 0; sb < nb; ++sb) {
      const float* df = ds + (sb * g.f + f) * ps;
      for (int u = 0; u < g.ohw; ++u) a = __fadd_rn(a, df[u]);
    }
    out[f * cols + g.ckk] = a;
  }
}

// FG for the blocked weight gradient: as many filters per thread (<= 4) as keep >= 2 row groups
__device__ __forceinline__ int wgrad_fg(const ConvGeom& g, int threads) {
  for (int fg = 4; fg > 1; --fg)
    if (((g.f + fg - 1) / fg) * g.c * g.k * 2 <= threads) return fg;
  return 1;
}

// POOLX (FWD only): problems may carry a folded max-pool of their input (hnn_conv_problem.pool_x); a
// separate instantiation because the staging branch alone made ptxas spill in the compute paths.
template <int OP, bool POOLX = false>
__global__ void __launch_bounds__(DTHREADS, POOLX ? HNN_POOLX_MINB : 3) conv_direct_kernel(const hnn_conv_problem* __restrict__ probs, int nprob,
                                                               const hnn_step_row* __restrict__ cur,
                                                               const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  extern __shared__ float sm[];
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_conv_problem& q) { return q.tile_base; });
  const hnn_conv_problem& p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const ConvGeom g(p);
  const int rows = cur[p.model].rows;
  const int unit = blockIdx.x - p.tile_base;  // sample (FWD/DGRAD) or batch chunk (WGRAD)
  if (OP == HNN_FWD) {
    const int b = unit;
    float* yb = p.y + size_t(b) * g.f * g.ohw;
    if (b >= rows) {
      for (int e = threadIdx.x; e < g.f * g.ohw; e += blockDim.x) yb[e] = 0.0f;
      if (POOLX && p.pool_x)  // (the folded pool's outputs for rows past the batch: zeros, like its own launch)
        for (int e = threadIdx.x; e < g.c * g.hw; e += blockDim.x) {
          const_cast<float*>(p.x)[size_t(b) * g.c * g.hw + e] = 0.0f;
          p.pool_idx[size_t(b) * g.c * g.hw + e] = 0;
        }
      return;
    }
    const DirectLayout lay(g.c, g.h, g.w, g.k, g.oh, g.ow);
    float* xs = sm;                 // [C][H][rs], channel stride cs
    float* ws = sm + ((g.c * lay.cs + 3) & ~3);  // [F][C*k*k] (generic) / [C*k*k][fp] (blocked; float4 rows)
    if (POOLX && p.pool_x) stage_pooled_x(xs, p, b, g.c, g.h, g.w, lay.rs, lay.cs);
    else stage_rows(xs, p.x + size_t(b) * g.c * g.hw, g.c * g.h, g.w, g.h, lay.rs, lay.cs);
    if (g.s == 1 && (g.k == 5 || g.k == 3)) {
      const int fp = (g.f + 3) & ~3;
      for (int e = threadIdx.x; e < g.ckk * fp; e += blockDim.x) {  // tap-major, filters innermost
        const int t = e / fp, f = e - t * fp;
        ws[e] = f < g.f ? __ldg(p.weight + size_t(f) * g.ckk + t) : 0.0f;
      }
      __syncthreads();
      const bool fg8 = fwd_fg(g) == 8;
      // padding 0: every tap is in the image (the row tail past w feeds only outputs >= ow, which
      // the row stride rs >= ow + K - 1 + (RB - 1) keeps inside the staged row)
      const bool pad0 = g.pad == 0 && lay.rs >= ((g.ow + RB - 1) / RB) * RB + g.k - 1;
      if (g.k == 5) {
        if (pad0) return fg8 ? direct_fwd_blocked<5, 8, true>(p, g, xs, lay.rs, lay.cs, ws, fp, yb)
                             : direct_fwd_blocked<5, 4, true>(p, g, xs, lay.rs, lay.cs, ws, fp, yb);
        return fg8 ? direct_fwd_blocked<5, 8, false>(p, g, xs, lay.rs, lay.cs, ws, fp, yb)
                   : direct_fwd_blocked<5, 4, false>(p, g, xs, lay.rs, lay.cs, ws, fp, yb);
      }
      return fg8 ? direct_fwd_blocked<3, 8, false>(p, g, xs, lay.rs, lay.cs, ws, fp, yb)
                 : direct_fwd_blocked<3, 4, false>(p, g, xs, lay.rs, lay.cs, ws, fp, yb);
    }
    stage(ws, p.weight, g.f * g.ckk);
    __syncthreads();
    for (int e = threadIdx.x; e < g.f * g.ohw; e += blockDim.x) {
      const int f = e / g.ohw, opix = e - f * g.ohw;
      const int oy = opix / g.ow, ox = opix - oy * g.ow;
      const int y0 = oy * g.s - g.pad, x0 = ox * g.s - g.pad;
      const int i0 = max(0, -y0), i1 = min(g.k, g.h - y0), j0 = max(0, -x0), j1 = min(g.k, g.w - x0);
      const float* wf = ws + f * g.ckk;
      float acc = 0.0f;
      for (int c = 0; c < g.c; ++c) {
        const float* xc = xs + c * lay.cs + y0 * lay.rs + x0;
        const float* wc = wf + c * g.kk2;
        for (int i = i0; i < i1; ++i)
          for (int j = j0; j < j1; ++j) acc = fmaf(xc[i * lay.rs + j], wc[i * g.k + j], acc);
      }
      float v = __fadd_rn(acc, __ldg(p.bias + f));
      if (p.relu) v = np_relu(v);
      yb[e] = v;
    }
  } else if (OP == HNN_DGRAD) {
    const int b = unit;
    float* dxb = p.dx + size_t(b) * g.c * g.hw;
    if (b >= rows) {
      for (int e = threadIdx.x; e < g.c * g.hw; e += blockDim.x) dxb[e] = 0.0f;
      return;
    }
    const float* mb = p.mask ? p.mask + size_t(b) * g.c * g.hw : nullptr;
    if (g.s == 1 && (g.k == 5 || g.k == 3) && g.pad <= g.k - 1) {
      const DgradLayout L(g.c, g.h, g.w, g.k, g.pad, g.oh, g.ow);
      float* dp = sm;                                    // [F][rows][rs] zero-padded dy planes
      float* wt = sm + ((g.f * L.plane + 3) & ~3);       // [F*k*k][cp] tap-major weights
      for (int e = threadIdx.x; e < g.f * L.plane; e += blockDim.x) dp[e] = 0.0f;
      for (int e = threadIdx.x; e < g.f * g.k * g.k * L.cp; e += blockDim.x) {
        const int t = e / L.cp, c = e - t * L.cp, f = t / (g.k * g.k), ij = t - f * g.k * g.k;
        wt[e] = c < g.c ? __ldg(p.weight + (size_t(f) * g.c + c) * g.k * g.k + ij) : 0.0f;
      }
      __syncthreads();
      if (p.pool_idx) stage_dy_pooled(dp + L.pd * L.rs + L.pd, p, size_t(b) * g.f, g.f, L.plane, L.rs);
      else stage_rows(dp + L.pd * L.rs + L.pd, p.dy + size_t(b) * g.f * g.ohw, g.f * g.oh, g.ow, g.oh, L.rs, L.plane);
      __syncthreads();
      const int groups8 = (g.c + 7) / 8, qb = (g.w + RB - 1) / RB;
      const bool cg8 = groups8 * g.h * qb >= 128;
      if (g.k == 5) return cg8 ? direct_dgrad_blocked<5, 8>(p, g, L, dp, wt, dxb, mb)
                               : direct_dgrad_blocked<5, 4>(p, g, L, dp, wt, dxb, mb);
      return cg8 ? direct_dgrad_blocked<3, 8>(p, g, L, dp, wt, dxb, mb)
                 : direct_dgrad_blocked<3, 4>(p, g, L, dp, wt, dxb, mb);
    }
    float* ds = sm;                  // [F][OH][OW]
    float* ws = sm + g.f * g.ohw;    // [F][C][k][k]
    if (p.pool_idx) stage_dy_pooled(ds, p, size_t(b) * g.f, g.f, g.ohw, g.ow);
    else stage(ds, p.dy + size_t(b) * g.f * g.ohw, g.f * g.ohw);
    stage(ws, p.weight, g.f * g.ckk);
    __syncthreads();
    for (int e = threadIdx.x; e < g.c * g.hw; e += blockDim.x) {
      const int c = e / g.hw, pix = e - c * g.hw;
      const int y = pix / g.w, x = pix - y * g.w;
      // taps i with (y + pad - i) divisible by s and 0 <= (y + pad - i)/s < OH, ascending i;
      // oy steps down by one per tap (no division in the loop)
      const int ry = (y + g.pad) % g.s, rx = (x + g.pad) % g.s;
      const int oy_first = (y + g.pad - ry) / g.s, ox_first = (x + g.pad - rx) / g.s;
      float acc = 0.0f;
      for (int f = 0; f < g.f; ++f) {
        const float* df = ds + f * g.ohw;
        const float* wfc = ws + (f * g.c + c) * g.kk2;
        for (int i = ry, oy = oy_first; i < g.k && oy >= 0; i += g.s, --oy) {
          if (oy >= g.oh) continue;
          const float* drow = df + oy * g.ow;
          const float* wrow = wfc + i * g.k;
          for (int j = rx, ox = ox_first; j < g.k && ox >= 0; j += g.s, --ox) {
            if (ox >= g.ow) continue;
            acc = fmaf(drow[ox], wrow[j], acc);
          }
        }
      }
      dxb[e] = mb ? np_mask(acc, mb[e]) : acc;
    }
  } else {
    // WGRAD: the CTA stages its chunk of samples (inputs with a padded, bank-conflict-free
    // layout: row stride W+1, channel stride H*(W+1)+1); thread t owns weights t, t+256, ...
    // and sweeps the valid output window of each staged sample in order.
    constexpr int MAXW = 16;
    const int cols = g.ckk + 1, nw = g.f * cols;
    const DirectLayout lay(g.c, g.h, g.w, g.k, g.oh, g.ow);
    const int rs = lay.rs, cs = lay.cs, ps = lay.ps;
    const int b0 = unit * HNN_CONV_DIRECT_BCHUNK, nb = max(0, min(HNN_CONV_DIRECT_BCHUNK, rows - b0));
    float* xs = sm;                                            // [nb][C] x (H x rs), channel stride cs
    float* ds = sm + HNN_CONV_DIRECT_BCHUNK * g.c * cs;        // [nb][F] dy planes (OH x OW), stride ps
    stage_rows(xs, p.x + size_t(b0) * g.c * g.hw, nb * g.c * g.h, g.w, g.h, rs, cs);
    if (p.pool_idx) stage_dy_pooled(ds, p, size_t(b0) * g.f, nb * g.f, ps, g.ow);
    else stage_rows(ds, p.dy + size_t(b0) * g.f * g.ohw, nb * g.f, g.ohw, 1, g.ohw, ps);
    __syncthreads();
    if (g.s == 1 && (g.k == 5 || g.k == 3)) {
      float* red = ds + HNN_CONV_DIRECT_BCHUNK * g.f * ps;  // [G][f*c*k][k] group partials
      float* out = p.partial + size_t(unit) * nw;
      const int fg = wgrad_fg(g, blockDim.x);
      if (g.k == 5) {
        if (fg == 4) direct_wgrad_blocked<5, 4>(p, g, xs, cs, rs, ds, ps, nb, red, out);
        else if (fg == 3) direct_wgrad_blocked<5, 3>(p, g, xs, cs, rs, ds, ps, nb, red, out);
        else if (fg == 2) direct_wgrad_blocked<5, 2>(p, g, xs, cs, rs, ds, ps, nb, red, out);
        else direct_wgrad_blocked<5, 1>(p, g, xs, cs, rs, ds, ps, nb, red, out);
      } else {
        if (fg == 4) direct_wgrad_blocked<3, 4>(p, g, xs, cs, rs, ds, ps, nb, red, out);
        else if (fg == 3) direct_wgrad_blocked<3, 3>(p, g, xs, cs, rs, ds, ps, nb, red, out);
        else if (fg == 2) direct_wgrad_blocked<3, 2>(p, g, xs, cs, rs, ds, ps, nb, red, out);
        else direct_wgrad_blocked<3, 1>(p, g, xs, cs, rs, ds, ps, nb, red, out);
      }
      return;
    }
    float acc[MAXW];
#pragma unroll
    for (int q = 0; q < MAXW; ++q) acc[q] = 0.0f;
#pragma unroll
    for (int q = 0; q < MAXW; ++q) {
      const int wi = threadIdx.x + q * DTHREADS;
      if (wi >= nw) break;
      const int f = wi / cols, col = wi - f * cols;
      float a = 0.0f;
      if (col == g.ckk) {
        for (int sb = 0; sb < nb; ++sb) {
          const float* df = ds + (sb * g.f + f) * ps;
          for (int t = 0; t < g.ohw; ++t) a = __fadd_rn(a, df[t]);
        }
      } else {
        const int c = col / g.kk2, r = col - c * g.kk2, i = r / g.k, j = r - i * g.k;
        const int ny = g.h - 1 + g.pad - i, nx = g.w - 1 + g.pad - j;
        const int oy0 = max(0, (g.pad - i + g.s - 1) / g.s), oy1 = ny < 0 ? 0 : min(g.oh, ny / g.s + 1);
        const int ox0 = max(0, (g.pad - j + g.s - 1) / g.s), ox1 = nx < 0 ? 0 : min(g.ow, nx / g.s + 1);
        // four interleaved partial sums (ox residues mod 4) hide the shared-memory latency of
        // the dependent FMA chain; they are combined in a fixed order, so results stay deterministic
        float a4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int sb = 0; sb < nb; ++sb) {
          const float* df = ds + (sb * g.f + f) * ps;
          const float* xc = xs + (sb * g.c + c) * cs + (i - g.pad) * rs + (j - g.pad);
          for (int oy = oy0; oy < oy1; ++oy) {
            const float* xr = xc + oy * g.s * rs;
            const float* dr = df + oy * g.ow;
            int ox = ox0;
            for (; ox + 3 < ox1; ox += 4) {
              a4[0] = fmaf(dr[ox], xr[ox * g.s], a4[0]);
              a4[1] = fmaf(dr[ox + 1], xr[(ox + 1) * g.s], a4[1]);
              a4[2] = fmaf(dr[ox + 2], xr[(ox + 2) * g.s], a4[2]);
              a4[3] = fmaf(dr[ox + 3], xr[(ox + 3) * g.s], a4[3]);
            }
            for (; ox < ox1; ++ox) a4[ox & 3] = fmaf(dr[ox], xr[ox * g.s], a4[ox & 3]);
          }
        }
        a = __fadd_rn(__fadd_rn(a4[0], a4[1]), __fadd_rn(a4[2], a4[3]));
      }
      acc[q] = a;
    }
#pragma unroll
    for (int q = 0; q < MAXW; ++q) {
      const int wi = threadIdx.x + q * DTHREADS;
      if (wi >= nw) break;
      p.partial[size_t(unit) * nw + wi] = acc[q];  // == partial[(split * F + f) * cols + col]
    }
  }
}

// Shared-memory bytes a problem needs on the direct path (host and device agree on this).
__host__ __device__ inline int conv_direct_smem(int op, int c, int h, int w, int f, int k, int oh, int ow) {
  const int ckk = c * k * k;
  const DirectLayout lay(c, h, w, k, oh, ow);
  if (op == HNN_FWD) return 4 * (((c * lay.cs + 3) & ~3) + ((f + 7) & ~7) * ckk);  // (filters padded: blocked path)
  if (op == HNN_DGRAD) {
    const int pad = (h - oh + k - 1) / 2;  // stride 1: h = oh + k - 1 - 2 * pad
    if (k == 5 || k == 3) {  // (the blocked path needs the padded layout; otherwise the plain one fits)
      const DgradLayout L(c, h, w, k, pad, oh, ow);
      return 4 * max(((f * L.plane + 3) & ~3) + f * k * k * L.cp, f * oh * ow + f * ckk);
    }
    return 4 * (f * oh * ow + f * ckk);
  }
  // staged samples + the blocked stride-1 path's row-group partials (G <= 8 groups of f*c*k*k)
  return 4 * HNN_CONV_DIRECT_BCHUNK * (c * lay.cs + f * lay.ps) + 4 * 8 * f * c * k * k;
}

}  // namespace hnn

extern "C" int hnn_conv_direct_smem(int op, int c, int h, int w, int f, int k, int oh, int ow) {
  return hnn::conv_direct_smem(op, c, h, w, f, k, oh, ow);
}

// Threads per CTA the direct kernel wants for a layer: 128 when the register-blocked stride-1 forward /
// input gradient has at most 128 work items per sample (LeNet conv2: 120 / 112), so that twice as
// many samples share an SM; 256 otherwise.
extern "C" int hnn_conv_direct_threads(int op, int c, int h, int w, int f, int k, int oh, int ow) {
  const int pad2 = oh - h + k - 1;  // 2 * padding of a stride-1 layer (the blocked paths)
  const bool blocked = (k == 5 || k == 3) && pad2 >= 0 && pad2 % 2 == 0 && pad2 / 2 <= k - 1;
  if (!blocked || op == HNN_WGRAD) return hnn::DTHREADS;
  const int rows = op == HNN_FWD ? oh : h, qb = ((op == HNN_FWD ? ow : w) + hnn::RB - 1) / hnn::RB;
  const int ch = op == HNN_FWD ? f : c;  // filters (forward) / channels (input gradient) per thread block
  const int g8 = ((ch + 7) / 8) * rows * qb;
  const int items = g8 >= 128 ? g8 : ((ch + 3) / 4) * rows * qb;
  return items <= 128 ? 128 : hnn::DTHREADS;
}

extern "C" int hnn_grouped_conv_direct_ex(int op, const hnn_conv_problem* probs, int nprob, int total_blocks, int smem,
                                          int threads, const hnn_step_row* cur, const hnn_model_status* status,
                                          void* stream);

extern "C" int hnn_grouped_conv_direct(int op, const hnn_conv_problem* probs, int nprob, int total_blocks, int smem,
                                       const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  return hnn_grouped_conv_direct_ex(op, probs, nprob, total_blocks, smem, hnn::DTHREADS, cur, status, stream);
}

extern "C" int hnn_grouped_conv_direct_ex(int op, const hnn_conv_problem* probs, int nprob, int total_blocks, int smem,
                                          int threads, const hnn_step_row* cur, const hnn_model_status* status,
                                          void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_blocks > 0, "hnn_grouped_conv_direct", "bad arguments");
  HNN_REQUIRE(threads >= 32 && threads <= hnn::DTHREADS && threads % 32 == 0, "hnn_grouped_conv_direct", "bad block size");
  HNN_REQUIRE(smem > 0 && smem <= 200 * 1024, "hnn_grouped_conv_direct", "layer too large for the direct path");
  cudaStream_t s = hnn::as_stream(stream);
  static int configured[4] = {0, 0, 0, 0};
  if (op == HNN_CONV_DIRECT_FWD_POOLED) {
    if (smem > configured[3]) {
      cudaFuncSetAttribute(hnn::conv_direct_kernel<HNN_FWD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      configured[3] = 200 * 1024;
    }
    hnn::launch_pdl(hnn::conv_direct_kernel<HNN_FWD, true>, dim3(total_blocks), dim3(threads), smem, s, probs, nprob, cur, status);
  } else if (op == HNN_FWD) {
    if (smem > configured[0]) {
      cudaFuncSetAttribute(hnn::conv_direct_kernel<HNN_FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      configured[0] = 200 * 1024;
    }
    hnn::launch_pdl(hnn::conv_direct_kernel<HNN_FWD>, dim3(total_blocks), dim3(threads), smem, s, probs, nprob, cur, status);
  } else if (op == HNN_DGRAD) {
    if (smem > configured[1]) {
      cudaFuncSetAttribute(hnn::conv_direct_kernel<HNN_DGRAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      configured[1] = 200 * 1024;
    }
    hnn::launch_pdl(hnn::conv_direct_kernel<HNN_DGRAD>, dim3(total_blocks), dim3(threads), smem, s, probs, nprob, cur, status);
  } else if (op == HNN_WGRAD) {
    if (smem > configured[2]) {
      cudaFuncSetAttribute(hnn::conv_direct_kernel<HNN_WGRAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      configured[2] = 200 * 1024;
    }
    hnn::launch_pdl(hnn::conv_direct_kernel<HNN_WGRAD>, dim3(total_blocks), dim3(threads), smem, s, probs, nprob, cur, status);
  } else {
    hnn::set_error("hnn_grouped_conv_direct", "unknown op");
    return HNN_ERR_INVALID;
  }
  return hnn::check_launch("hnn_grouped_conv_direct");
}
