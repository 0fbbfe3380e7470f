// Data-movement kernels around the tensor-core convolution path (pkg/src/hybridnn/ops.py:91-130).
//
// A conv2d layer big enough for the tensor cores (C*k*k and F >= 64) is lowered onto the CTA-pair
// 3xTF32 GEMM (gemm_tc2.cu) with NCHW activations kept in the reference layout:
//   FWD    cols[m, kk] = im2col(x)  (m = (b, oh, ow), kk = (c, r, s): the reference's K order)
//          y = cols x W^T + bias (+relu)      GEMM epilogue stores NCHW directly (c_mode 1)
//   DGRAD  dyT[m, f] = dy (NCHW -> rows)      transpose
//          dcols = dyT x W                    GEMM (row-major [m, kk])
//          dx = col2im(dcols) * (x > 0)       gather form, taps in (r, s) order, no atomics
//   WGRAD  partial[s] = dyT^T x cols          GEMM, fixed K splits over output pixels
//          dW = sum_s partial[s] (in order); db = sum_b sum_hw dy (in order)
// Every kernel is a fixed function of the problem's shape (bit-exact isolation, no atomics).
#include <cuda_bf16.h>

#include "common.cuh"

namespace hnn {

constexpr int CT_THREADS = 256;

__device__ __forceinline__ const hnn_convtc_problem& ct_problem(const hnn_convtc_problem* probs, int nprob,
                                                                int block) {
  return probs[find_problem(probs, nprob, block, [](const hnn_convtc_problem& q) { return q.block_base; })];
}

// cols[m, kk] for m < cap*OH*OW, kk < K (row stride kkp): zeros outside the image (padding) and for
// samples beyond this step's batch rows.  One CTA = 32 consecutive output pixels x 32 channels:
// the x reads (lane = pixel) and the cols writes (a pixel's 32*k*k contiguous floats, lane-strided)
// are both coalesced, through a shared-memory tile of 32 x (32*k*k) floats.
constexpr int IC_PIX = 32, IC_CH = 32;

__global__ void __launch_bounds__(CT_THREADS) im2col_kernel(const hnn_convtc_problem* __restrict__ probs, int nprob,
                                                           const hnn_step_row* __restrict__ cur,
                                                           const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  extern __shared__ float ic_tile[];  // [IC_PIX][IC_CH * k * k + 1]
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int kk2 = p.k * p.k, seg = IC_CH * kk2, ld = seg + 1;
  if (p.bf16 && p.c * kk2 <= 32) {
    // a network's first layer (C = 3): one thread per output pixel, its C*k*k taps straight from x
    // (consecutive threads = consecutive pixels: coalesced reads and colst writes), the cols row
    // (<= 32 bf16 = 64 bytes incl. zero padding) as four 16-byte stores.  256 pixels per CTA.
    const int m = (blockIdx.x - p.block_base) * CT_THREADS + threadIdx.x;
    const int ohw = p.oh * p.ow;
    if (m >= p.cap * ohw) return;
    const int b = m / ohw, o = m - b * ohw, oy = o / p.ow, ox = o - oy * p.ow;
    const bool valid = b < cur[p.model].rows;
    __nv_bfloat16 v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __float2bfloat16_rn(0.0f);
    if (p.k == 3) {  // (C <= 3): every tap index is a compile-time register slot
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const int h = oy * p.stride - p.pad + r;
#pragma unroll
          for (int sx = 0; sx < 3; ++sx) {
            const int w = ox * p.stride - p.pad + sx;
            float x = 0.0f;
            if (c < p.c && valid && h >= 0 && h < p.h && w >= 0 && w < p.w)
              x = __ldg(p.x + ((size_t(b) * p.c + c) * p.h + h) * p.w + w);
            v[c * 9 + r * 3 + sx] = __float2bfloat16_rn(x);
          }
        }
    } else {
      for (int c = 0; c < p.c; ++c)
        for (int r = 0; r < p.k; ++r) {
          const int h = oy * p.stride - p.pad + r;
          for (int sx = 0; sx < p.k; ++sx) {
            const int w = ox * p.stride - p.pad + sx, j = (c * p.k + r) * p.k + sx;
            float x = 0.0f;
            if (valid && h >= 0 && h < p.h && w >= 0 && w < p.w)
              x = __ldg(p.x + ((size_t(b) * p.c + c) * p.h + h) * p.w + w);
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (q == j) v[q] = __float2bfloat16_rn(x);
          }
        }
    }
    if (p.cols) {
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.cols) + size_t(m) * p.kkp);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q * 8 < p.kkp) dst[q] = *reinterpret_cast<const uint4*>(&v[q * 8]);
    }
    if (p.colst) {
      __nv_bfloat16* ct = reinterpret_cast<__nv_bfloat16*>(p.colst);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < p.kk) ct[size_t(j) * p.pix_ld + m] = v[j];
    }
    return;
  }
  const int ohw = p.oh * p.ow;
  const int cblocks = (p.c + IC_CH - 1) / IC_CH;
  const int t = blockIdx.x - p.block_base;
  const int pb = t / cblocks, cb = t - pb * cblocks;
  const int m0 = pb * IC_PIX, c0 = cb * IC_CH;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m = m0 + lane;
  const int b = m / ohw, o = m - b * ohw, oh = o / p.ow, ow = o - oh * p.ow;
  const bool valid = m < p.cap * ohw && b < rows;
  if (p.bf16 && !p.cols && !p.colst) {
    // only the NHWC copy (implicit-GEMM forward and weight gradient of a "same" layer): one tap,
    // through a 32 x 33 transpose tile; zeros past the batch
    float* t = ic_tile;
    for (int ci = warp; ci < IC_CH; ci += CT_THREADS / 32) {
      const int c = c0 + ci;
      t[lane * 33 + ci] = (valid && c < p.c) ? __ldg(p.x + (size_t(b) * p.c + c) * ohw + o) : 0.0f;
    }
    __syncthreads();
    __nv_bfloat16* xh = reinterpret_cast<__nv_bfloat16*>(p.dyt);
    for (int pi = warp; pi < IC_PIX; pi += CT_THREADS / 32) {
      const int mm = m0 + pi;
      if (mm < p.cap * ohw && c0 + lane < p.c) xh[size_t(mm) * p.c + c0 + lane] = __float2bfloat16_rn(t[pi * 33 + lane]);
    }
    return;
  }
  if (p.k == 3) {  // the common 3 x 3 case: a channel's 9 taps load together (independent requests)
    for (int ci = warp; ci < IC_CH; ci += CT_THREADS / 32) {
      const int c = c0 + ci;
      const float* xc = p.x + (size_t(b) * p.c + c) * p.h * p.w;
      float v[9];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int h = oh * p.stride - p.pad + r;
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          const int w = ow * p.stride - p.pad + s;
          v[r * 3 + s] = (valid && c < p.c && h >= 0 && h < p.h && w >= 0 && w < p.w) ? __ldg(xc + h * p.w + w) : 0.0f;
        }
      }
#pragma unroll
      for (int j = 0; j < 9; ++j) ic_tile[lane * ld + ci * 9 + j] = v[j];
    }
  } else {
    for (int ci = warp; ci < IC_CH; ci += CT_THREADS / 32) {
      const int c = c0 + ci;
      const float* xc = p.x + (size_t(b) * p.c + c) * p.h * p.w;
      for (int r = 0; r < p.k; ++r) {
        const int h = oh * p.stride - p.pad + r;
        for (int s = 0; s < p.k; ++s) {
          const int w = ow * p.stride - p.pad + s;
          float v = 0.0f;
          if (valid && c < p.c && h >= 0 && h < p.h && w >= 0 && w < p.w) v = __ldg(xc + h * p.w + w);
          ic_tile[lane * ld + ci * kk2 + r * p.k + s] = v;
        }
      }
    }
  }
  __syncthreads();
  const int width = min(seg, (p.c - c0) * kk2);
  if (p.bf16 && p.dyt) {
    // the implicit-GEMM forward's NHWC bf16 copy of x, from the centre taps of this tile ("same"
    // stride-1 layers only: output pixel = input pixel): 32 channels of a pixel per warp store
    const int centre = p.pad * p.k + p.pad;
    __nv_bfloat16* xh = reinterpret_cast<__nv_bfloat16*>(p.dyt);
    for (int pi = warp; pi < IC_PIX; pi += CT_THREADS / 32) {
      const int mm = m0 + pi;
      if (mm < p.cap * ohw && c0 + lane < p.c)
        xh[size_t(mm) * p.c + c0 + lane] = __float2bfloat16_rn(ic_tile[pi * ld + lane * kk2 + centre]);
    }
  }
  if (p.bf16) {
    __nv_bfloat16* cb16 = reinterpret_cast<__nv_bfloat16*>(p.cols);
    for (int pi = warp; pi < IC_PIX && cb16; pi += CT_THREADS / 32) {  // (no cols: implicit-GEMM forward)
      const int mm = m0 + pi;
      if (mm >= p.cap * ohw) break;
      __nv_bfloat16* dst = cb16 + size_t(mm) * p.kkp + c0 * kk2;
      for (int j = lane; j < width; j += 32) dst[j] = __float2bfloat16_rn(ic_tile[pi * ld + j]);
      if (cb == 0)
        for (int j = p.kk + lane; j < p.kkp; j += 32) cb16[size_t(mm) * p.kkp + j] = __float2bfloat16_rn(0.0f);
    }
    if (p.colst) {  // pixel-contiguous copy [kkp, pix_ld] for the weight-gradient GEMM
      __nv_bfloat16* ct = reinterpret_cast<__nv_bfloat16*>(p.colst);
      const int mm = m0 + lane;
      if (mm < p.cap * ohw)
        for (int j = warp; j < width; j += CT_THREADS / 32)
          ct[size_t(c0 * kk2 + j) * p.pix_ld + mm] = __float2bfloat16_rn(ic_tile[lane * ld + j]);
    }
    return;
  }
  for (int pi = warp; pi < IC_PIX; pi += CT_THREADS / 32) {
    const int mm = m0 + pi;
    if (mm >= p.cap * ohw) break;
    float* dst = p.cols + size_t(mm) * p.kkp + c0 * kk2;
    for (int j = lane; j < width; j += 32) dst[j] = ic_tile[pi * ld + j];
    if (cb == 0)  // zero pad columns kk..kkp-1 (TMA needs 16-byte rows)
      for (int j = p.kk + lane; j < p.kkp; j += 32) p.cols[size_t(mm) * p.kkp + j] = 0.0f;
  }
}

int im2col_smem_bytes(int k) { return IC_PIX * (IC_CH * k * k + 1) * 4; }

// dyT[m, f] = dy[b, f, hw] (m = b*HW + hw) through 32 x 32 shared-memory tiles; one CTA = 32
// channels x TR_TILES consecutive (sample, 32-pixel run) units, every thread's 4 * TR_TILES loads issued
// before the first store (one 32 x 32 tile per CTA: a few dependent round trips per 4 KB, 1.4-2 TB/s
// on C4); bpart[b, th, f] = sum over pixel run th of dy[b, f, hw] (bias gradient partials).
constexpr int TR_TILES = HNN_CONVTC_TRANSPOSE_HW_TILES;
__global__ void __launch_bounds__(CT_THREADS) transpose_dy_kernel(const hnn_convtc_problem* __restrict__ probs,
                                                                 int nprob, const hnn_step_row* __restrict__ cur,
                                                                 const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  __shared__ float tile[TR_TILES][32][33];
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int hw_n = p.oh * p.ow;
  const int tiles_hw = (hw_n + 31) / 32, tiles_f = (p.f + 31) / 32;
  const int t = blockIdx.x - p.block_base;
  // units q = (sample, pixel run) in row-major order, TR_TILES consecutive units per CTA (several
  // samples per CTA when a plane has fewer than TR_TILES runs)
  const int q0 = (t / tiles_f) * TR_TILES, tf = t - (t / tiles_f) * tiles_f, nq = rows * tiles_hw;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  int ub[TR_TILES], uh[TR_TILES];  // unit's sample and first pixel (ub = -1: past the batch)
#pragma unroll
  for (int u = 0; u < TR_TILES; ++u) {
    const int q = q0 + u, b = q / tiles_hw;
    ub[u] = q < nq ? b : -1;  // rows beyond the batch are never read by the GEMMs
    uh[u] = (q - b * tiles_hw) * 32;
  }
  if (ub[0] < 0) return;
  float v[TR_TILES][4];
#pragma unroll
  for (int u = 0; u < TR_TILES; ++u)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int f = tf * 32 + ty + 8 * i, hw = uh[u] + tx;
      v[u][i] = (ub[u] >= 0 && f < p.f && hw < hw_n) ? __ldg(p.dy + (size_t(ub[u]) * p.f + f) * hw_n + hw) : 0.0f;
    }
#pragma unroll
  for (int u = 0; u < TR_TILES; ++u)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = ty + 8 * i, f = tf * 32 + j, hw = uh[u] + tx;
      tile[u][j][tx] = v[u][i];
      if (p.bf16 && p.dyk && ub[u] >= 0 && f < p.f && hw < hw_n)  // dyk[f, b*HW + hw]: filter-major, pixel-contiguous
        reinterpret_cast<__nv_bfloat16*>(p.dyk)[size_t(f) * p.pix_ld + size_t(ub[u]) * hw_n + hw] =
            __float2bfloat16_rn(v[u][i]);
    }
  __syncthreads();
  const int fld = p.bf16 ? (p.f + 7) & ~7 : (p.f + 3) & ~3;  // dyt rows padded to 16 bytes (TMA)
  if (p.dyt) {
    const int f = tf * 32 + tx;
#pragma unroll
    for (int u = 0; u < TR_TILES; ++u)
      for (int j = ty; j < 32; j += 8) {
        const int hw = uh[u] + j;
        if (ub[u] >= 0 && hw < hw_n && f < p.f) {
          const size_t o = (size_t(ub[u]) * hw_n + hw) * fld + f;
          if (p.bf16) reinterpret_cast<__nv_bfloat16*>(p.dyt)[o] = __float2bfloat16_rn(tile[u][tx][j]);
          else p.dyt[o] = tile[u][tx][j];
        }
      }
  }
  // bias partial of each pixel run: bpart[b, th, f] = sum over its 32 pixels of dy[b, f, hw]
  // (fixed order; the reduce adds the runs in (b, th) order).  A per-(b, f) sequential sum over all
  // HW pixels was a 1024-long dependent chain per thread (0.1-0.16 ms per C4 layer).
  if (ty < TR_TILES && p.bpart) {
    const int f = tf * 32 + tx, q = q0 + ty;
    if (f < p.f && q < nq) {
      float acc = 0.0f;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) acc = __fadd_rn(acc, tile[ty][tx][j]);  // pixels th*32 + j (0 past HW)
      p.bpart[size_t(q) * p.f + f] = acc;  // (q = b * tiles_hw + th)
    }
  }
}

// dx[b, c, h, w] = (x > 0 if masked) * sum over taps (r, s) in order of dcols[m(oh, ow), (c, r, s)]
// with h = oh*stride - pad + r, w = ow*stride - pad + s; zeros for samples beyond the batch.
// One CTA = one input row segment (b, h, 32 columns) x 16 channels: the dcols rows it needs
// (valid oh, an ow window) are staged in shared memory with coalesced row reads, then each thread
// (column, channel) gathers its taps from the tile.
constexpr int CI_W = 32, CI_CH = 16, CI_OWMAX = 40;

// STRIDE / K as template parameters: the tap arithmetic is shifts and compares (runtime integer
// divisions made this kernel issue-bound: ~900 instructions per output element, ncu IPC 2.5).
template <int STRIDE, int K>
__device__ __forceinline__ void col2im_tile(const hnn_convtc_problem& p, int rows, float* ci_tile) {
  constexpr int KK2 = K * K, SEG = CI_CH * KK2, SLD = SEG + 1;
  const int wblocks = (p.w + CI_W - 1) / CI_W, cblocks = (p.c + CI_CH - 1) / CI_CH;
  int t = blockIdx.x - p.block_base;
  const int cb = t % cblocks;
  t /= cblocks;
  const int wb = t % wblocks;
  t /= wblocks;
  const int h = t % p.h, b = t / p.h;
  const int c0 = cb * CI_CH, w0 = wb * CI_W;
  const int w1 = min(p.w, w0 + CI_W) - 1;
  // output-column window touched by input columns w0..w1 (any tap): ow in [ow_lo, ow_hi]
  const int ow_lo = max(0, (w0 + p.pad - (K - 1) + STRIDE - 1) / STRIDE);
  const int ow_hi = min(p.ow - 1, (w1 + p.pad) / STRIDE);
  const int nw = ow_hi - ow_lo + 1;
  const bool live_rows = b < rows;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // staged rows: (valid tap row r, output column ow_lo + i); their source / destination offsets
  // go to a small table so that every thread then issues all its 16-byte loads back to back
  // (a row-at-a-time copy loop serialised ~13 L2 round trips per warp)
  __shared__ int row_src[K * CI_OWMAX], row_dst[K * CI_OWMAX];
  __shared__ int nrows_s;
  // valid tap rows r (compile-time K: a handful of compares), then one table entry per thread
  // (a single thread filling the table serially was most of this kernel's time)
  int vr[K], nvr = 0;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int hh = h + p.pad - r;
    vr[r] = 0;
    if (live_rows && nw > 0 && hh >= 0 && !(STRIDE > 1 && hh % STRIDE) && hh / STRIDE < p.oh) vr[nvr++] = r;
  }
  for (int e = threadIdx.x; e < nvr * nw; e += CT_THREADS) {
    const int k = e / nw, i = e - k * nw;
    int r = 0;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j == k) r = vr[j];
    const int hh = h + p.pad - r;
    row_src[e] = int(((size_t(b) * p.oh + hh / STRIDE) * p.ow + ow_lo + i) * p.kkp / 4);
    row_dst[e] = (r * CI_OWMAX + i) * SLD;
  }
  if (threadIdx.x == 0) nrows_s = nvr * nw;
  __syncthreads();
  {
    const int width = min(SEG, (p.c - c0) * KK2);
    const bool vec = (width & 3) == 0 && (p.kkp & 3) == 0 && ((c0 * KK2) & 3) == 0;
    const int w4 = vec ? width / 4 : 0;
    const int total = nrows_s * w4;
    const float4* base4 = reinterpret_cast<const float4*>(p.dcols) + (c0 * KK2) / 4;
    constexpr int PER = (3 * CI_OWMAX * SEG / 4 + CT_THREADS - 1) / CT_THREADS;  // max loads per thread
    float4 v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + u * CT_THREADS;
      if (e < total) {
        const int q = e / (SEG / 4), j = e - q * (SEG / 4);  // constant divisor
        v[u] = j < w4 ? __ldg(base4 + row_src[q] + j) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + u * CT_THREADS;
      if (e < total) {
        const int q = e / (SEG / 4), j = e - q * (SEG / 4);
        float* dst = ci_tile + row_dst[q] + 4 * j;
        dst[0] = v[u].x;
        dst[1] = v[u].y;
        dst[2] = v[u].z;
        dst[3] = v[u].w;
      }
    }
    if (!vec && live_rows) {  // unaligned channel segments (not produced by the planner)
      for (int e = threadIdx.x; e < nrows_s * width; e += CT_THREADS) {
        const int q = e / width, j = e - q * width;
        ci_tile[row_dst[q] + j] = __ldg(p.dcols + size_t(row_src[q]) * 4 + c0 * KK2 + j);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < CI_W * CI_CH; e += CT_THREADS) {
    const int ci = e / CI_W, w = w0 + e % CI_W, c = c0 + ci;
    if (w >= p.w || c >= p.c) continue;
    float acc = 0.0f;
    if (live_rows) {
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const int hh = h + p.pad - r;
        if (hh < 0 || (STRIDE > 1 && hh % STRIDE) || hh / STRIDE >= p.oh) continue;
#pragma unroll
        for (int s = 0; s < K; ++s) {
          const int ww = w + p.pad - s;
          if (ww < 0 || (STRIDE > 1 && ww % STRIDE)) continue;
          const int ow = ww / STRIDE;
          if (ow >= p.ow) continue;
          acc = __fadd_rn(acc, ci_tile[(r * CI_OWMAX + ow - ow_lo) * SLD + ci * KK2 + r * K + s]);
        }
      }
    }
    const size_t off = ((size_t(b) * p.c + c) * p.h + h) * p.w + w;
    if (live_rows && p.mask) acc = np_mask(acc, __ldg(p.mask + off));
    p.dx[off] = acc;
  }
}

__global__ void __launch_bounds__(CT_THREADS) col2im_kernel(const hnn_convtc_problem* __restrict__ probs, int nprob,
                                                           const hnn_step_row* __restrict__ cur,
                                                           const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  extern __shared__ float ci_tile[];  // [k][CI_OWMAX][CI_CH * k * k + 1]
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  if (p.k == 3 && p.stride == 1) col2im_tile<1, 3>(p, rows, ci_tile);
  else if (p.k == 3 && p.stride == 2) col2im_tile<2, 3>(p, rows, ci_tile);
  else if (p.k == 2 && p.stride == 1) col2im_tile<1, 2>(p, rows, ci_tile);
  else if (p.k == 2 && p.stride == 2) col2im_tile<2, 2>(p, rows, ci_tile);
  else if (p.k == 1 && p.stride == 1) col2im_tile<1, 1>(p, rows, ci_tile);
  else if (p.k == 1 && p.stride == 2) col2im_tile<2, 1>(p, rows, ci_tile);
  // other (kernel, stride) pairs are not routed to this path (runtime.py)
}

int col2im_smem_bytes(int k) { return k * CI_OWMAX * (CI_CH * k * k + 1) * 4; }

constexpr int RED_ROW_MAX = 512 * 9;  // floats of one staged weight-gradient row (C <= 512, k <= 3)
// dW[f, kk] = sum over the valid splits (in order) of partial[s*F + f, kk];
// db[f] = sum over (batch row, pixel tile) in order of bpart[b, tile, f].
__global__ void __launch_bounds__(CT_THREADS) wgrad_reduce_kernel(const hnn_convtc_problem* __restrict__ probs,
                                                                 int nprob, const hnn_step_row* __restrict__ cur,
                                                                 const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const long long kmax = (long long)rows * p.oh * p.ow;
  const int splits = int(min((long long)p.ksplit, (kmax + p.ksplit_len - 1) / p.ksplit_len));
  // split s occupies rows [s * fp, s * fp + f) of the partial buffer, fp = f rounded up to 32
  // (32-bit element indices: a weight tensor is far below 2^31 elements; 64-bit divisions per
  // element made this launch issue-bound)
  const int total = p.f * p.kk;
  const size_t ptotal = size_t((p.f + 31) & ~31) * p.kkp;
  const long long tid = (long long)(blockIdx.x - p.block_base) * CT_THREADS + threadIdx.x;
  const int kk2 = p.k * p.k;
  if (p.rsc && (p.kk & 3) == 0 && (p.kkp & 3) == 0 && p.kk <= RED_ROW_MAX) {
    // (r, s, c)-ordered partial columns: one filter row per CTA pass, its columns summed four at a
    // time (8 splits in flight) into shared memory at their reference (c, r, s) position, then
    // the row stored contiguously (element-wise stores at the permuted position were 36-byte strided:
    // 2.4 TB/s, 0.16 ms per C4 step)
    __shared__ float rowbuf[RED_ROW_MAX];
    for (int f = blockIdx.x - p.block_base; f < p.f; f += p.blocks) {
      const size_t pe0 = size_t(f) * p.kkp;
      for (int c4 = threadIdx.x; c4 < p.kk / 4; c4 += CT_THREADS) {
        const size_t pe = pe0 + 4 * c4;
        float4 v[8];
        const int s8 = min(splits, 8);
#pragma unroll
        for (int s = 0; s < 8; ++s)
          v[s] = s < s8 ? __ldg(reinterpret_cast<const float4*>(p.partial + s * ptotal + pe)) : make_float4(0, 0, 0, 0);
        float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < s8) {
            acc.x = __fadd_rn(acc.x, v[s].x);
            acc.y = __fadd_rn(acc.y, v[s].y);
            acc.z = __fadd_rn(acc.z, v[s].z);
            acc.w = __fadd_rn(acc.w, v[s].w);
          }
        for (int s = 8; s < splits; ++s) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(p.partial + s * ptotal + pe));
          acc.x = __fadd_rn(acc.x, t.x);
          acc.y = __fadd_rn(acc.y, t.y);
          acc.z = __fadd_rn(acc.z, t.z);
          acc.w = __fadd_rn(acc.w, t.w);
        }
        const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int col = 4 * c4 + q, rs = col / p.c;
          rowbuf[(col - rs * p.c) * kk2 + rs] = a4[q];  // (stride k*k words: conflict-free for k = 3)
        }
      }
      __syncthreads();
      for (int j = threadIdx.x; j < p.kk; j += CT_THREADS) p.dw[size_t(f) * p.kk + j] = rowbuf[j];
      __syncthreads();
    }
  } else if ((p.kk & 3) == 0 && (p.kkp & 3) == 0) {
    // four consecutive partial columns per thread: 16-byte loads, 8 splits x 16 bytes in flight
    for (int e4 = int(tid); e4 < total / 4; e4 += p.blocks * CT_THREADS) {
      const int e = 4 * e4, f = e / p.kk, col = e - f * p.kk;
      const size_t pe = size_t(f) * p.kkp + col;
      float4 v[8];
      const int s8 = min(splits, 8);
#pragma unroll
      for (int s = 0; s < 8; ++s)
        v[s] = s < s8 ? __ldg(reinterpret_cast<const float4*>(p.partial + s * ptotal + pe)) : make_float4(0, 0, 0, 0);
      float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < s8) {
          acc.x = __fadd_rn(acc.x, v[s].x);
          acc.y = __fadd_rn(acc.y, v[s].y);
          acc.z = __fadd_rn(acc.z, v[s].z);
          acc.w = __fadd_rn(acc.w, v[s].w);
        }
      for (int s = 8; s < splits; ++s) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p.partial + s * ptotal + pe));
        acc.x = __fadd_rn(acc.x, t.x);
        acc.y = __fadd_rn(acc.y, t.y);
        acc.z = __fadd_rn(acc.z, t.z);
        acc.w = __fadd_rn(acc.w, t.w);
      }
      const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int kr = col + q;
        if (p.rsc) {
          const int rs = (col + q) / p.c;
          kr = (col + q - rs * p.c) * kk2 + rs;
        }
        p.dw[size_t(f) * p.kk + kr] = a4[q];
      }
    }
  } else
  for (int e = int(tid); e < total; e += p.blocks * CT_THREADS) {
    // e walks the partial columns (coalesced reads of every split); rsc: partial column (r, s, c)
    // goes to reference column (c, r, s)
    const int f = e / p.kk, col = e - f * p.kk;
    int kr = col;
    if (p.rsc) {
      const int rs = col / p.c;
      kr = (col - rs * p.c) * kk2 + rs;
    }
    const size_t pe = size_t(f) * p.kkp + col;  // partial rows are kkp wide
    float v[8];
    const int s8 = min(splits, 8);
#pragma unroll
    for (int s = 0; s < 8; ++s) v[s] = s < s8 ? __ldg(p.partial + s * ptotal + pe) : 0.0f;  // loads together
    float acc = 0.0f;
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (s < s8) acc = __fadd_rn(acc, v[s]);
    for (int s = 8; s < splits; ++s) acc = __fadd_rn(acc, __ldg(p.partial + s * ptotal + pe));
    p.dw[size_t(f) * p.kk + kr] = acc;
  }
  // bias: one warp per filter; lane l sums the (batch row, pixel tile) partials l, l+32, ... in
  // order, then a fixed xor tree combines the lanes
  const int lane = threadIdx.x % 32;
  const long long warp = tid / 32, nwarps = (long long)p.blocks * CT_THREADS / 32;
  const int nq = rows * ((p.oh * p.ow + 31) / 32);
  for (long long f = warp; f < p.f; f += nwarps) {
    float acc = 0.0f;
    int q = lane;
    for (; q + 7 * 32 < nq; q += 8 * 32) {  // eight partials in flight, added in the same order
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(p.bpart + size_t(q + u * 32) * p.f + f);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, v[u]);
    }
    for (; q < nq; q += 32) acc = __fadd_rn(acc, __ldg(p.bpart + size_t(q) * p.f + f));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) p.db[f] = acc;
  }
}


// wpad[f, kk'] = w[f, kk] for kk < K, 0 for the pad columns (GEMM B operand with 16-byte rows).
__global__ void __launch_bounds__(CT_THREADS) pad_weights_kernel(const hnn_convtc_problem* __restrict__ probs, int nprob,
                                                                const hnn_step_row* __restrict__ cur,
                                                                const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const long long total = (long long)p.f * p.kkp;
  for (long long e = (long long)(blockIdx.x - p.block_base) * CT_THREADS + threadIdx.x; e < total;
       e += (long long)p.blocks * CT_THREADS) {
    const long long f = e / p.kkp, j = e - f * p.kkp;
    const float v = j < p.kk ? __ldg(p.weight + f * p.kk + j) : 0.0f;
    if (p.bf16) reinterpret_cast<__nv_bfloat16*>(p.wpad)[e] = __float2bfloat16_rn(v);
    else p.wpad[e] = v;
  }
}

// Flipped, transposed weights for the stride-1 input gradient computed as a forward conv of dy:
// wflip[c, (f, r', s')] = w[f, c, k-1-r', k-1-s'] (row length f*k*k; written to p.wpad).
__global__ void __launch_bounds__(CT_THREADS) flip_weights_kernel(const hnn_convtc_problem* __restrict__ probs,
                                                                 int nprob, const hnn_step_row* __restrict__ cur,
                                                                 const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const int kk2 = p.k * p.k, row = p.f * kk2;
  const long long total = (long long)p.c * row;
  for (long long e = (long long)(blockIdx.x - p.block_base) * CT_THREADS + threadIdx.x; e < total;
       e += (long long)p.blocks * CT_THREADS) {
    const int c = int(e / row), j = int(e - (long long)c * row);
    const int f = j / kk2, rs = j - f * kk2, r = rs / p.k, s = rs - r * p.k;
    const float v = __ldg(p.weight + ((size_t(f) * p.c + c) * p.k + (p.k - 1 - r)) * p.k + (p.k - 1 - s));
    if (p.bf16) reinterpret_cast<__nv_bfloat16*>(p.wpad)[e] = __float2bfloat16_rn(v);
    else p.wpad[e] = v;
  }
}

// Implicit-GEMM B operands, K in (r, s, channel) order (the NHWC A tile of a K block is one tap's
// 64 channels):  RSC   wpad[f, (r, s, c)] = w[f, c, r, s]
//                FLIP  wpad[c, (r, s, f)] = w[f, c, k-1-r, k-1-s]   (input gradient as a forward conv)
// One CTA per output row (a filter f, or a channel c for FLIP): its k*k*inner source values are
// read coalesced into shared memory (RSC: w[f] is contiguous; FLIP: w[:, c] is one k*k run per
// filter) and written back permuted, coalesced.  (An element-per-thread gather read 36-byte-strided
// words: 0.1 ms per launch on C4.)
constexpr int RSC_MAX = 512 * 9;  // k*k*inner floats staged per CTA (k <= 3, <= 512 channels)
template <bool FLIP>
__global__ void __launch_bounds__(CT_THREADS) rsc_weights_kernel(const hnn_convtc_problem* __restrict__ probs, int nprob,
                                                                const hnn_step_row* __restrict__ cur,
                                                                const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  __shared__ float stage[RSC_MAX];
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const int kk2 = p.k * p.k;
  const int inner = FLIP ? p.f : p.c;  // contiguous channel of the K index
  const int row = kk2 * inner;         // K
  const int nrow = FLIP ? p.c : p.f;
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.wpad);
  for (int o = blockIdx.x - p.block_base; o < nrow; o += p.blocks) {
    __syncthreads();
    if (FLIP) {  // stage[f * kk2 + t] = w[f, c=o, t]
      for (int e = threadIdx.x; e < row; e += CT_THREADS) {
        const int f = e / kk2, t = e - f * kk2;
        stage[e] = __ldg(p.weight + (size_t(f) * p.c + o) * kk2 + t);
      }
    } else {  // stage[c * kk2 + t] = w[f=o, c, t]
      for (int e = threadIdx.x; e < row; e += CT_THREADS) stage[e] = __ldg(p.weight + size_t(o) * row + e);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < row; j += CT_THREADS) {  // j = (r, s, ch)
      const int rs = j / inner, ch = j - rs * inner;
      const int t = FLIP ? (kk2 - 1 - rs) : rs;  // flipped tap: (k-1-r, k-1-s)
      out[size_t(o) * row + j] = __float2bfloat16_rn(stage[ch * kk2 + t]);
    }
  }
}

// Parity-class weights of a 3x3 / stride-2 / pad-1 input gradient (HNN_CONVTC_PARITY_WEIGHTS): dx at
// (2i + ph, 2j + pw) = sum over rr < 1 + ph, ss < 1 + pw of dy[i + rr][j + ss] . w[., ., ph+1-2rr, pw+1-2ss]
__global__ void __launch_bounds__(CT_THREADS) parity_weights_kernel(const hnn_convtc_problem* __restrict__ probs,
                                                                   int nprob, const hnn_step_row* __restrict__ cur,
                                                                   const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const int ph = p.ksplit >> 1, pw = p.ksplit & 1, kh = 1 + ph, kw = 1 + pw;
  const long long row = (long long)kh * kw * p.f, total = (long long)p.c * row;
  for (long long e = (long long)(blockIdx.x - p.block_base) * CT_THREADS + threadIdx.x; e < total;
       e += (long long)p.blocks * CT_THREADS) {
    const int c = int(e / row), j = int(e - (long long)c * row);
    const int rs = j / p.f, f = j - rs * p.f, rr = rs / kw, ss = rs - rr * kw;
    const int r = ph + 1 - 2 * rr, sx = pw + 1 - 2 * ss;
    reinterpret_cast<__nv_bfloat16*>(p.wpad)[e] =
        __float2bfloat16_rn(__ldg(p.weight + ((size_t(f) * p.c + c) * 3 + r) * 3 + sx));
  }
}

// bf16 wpad[kk, f] = w[f, kk] (kk < kkp; pad rows zero): the stride-2 dcols GEMM's K-major B.
__global__ void __launch_bounds__(CT_THREADS) wt_weights_kernel(const hnn_convtc_problem* __restrict__ probs, int nprob,
                                                               const hnn_step_row* __restrict__ cur,
                                                               const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  const long long total = (long long)p.kkp * p.f;
  for (long long e = (long long)(blockIdx.x - p.block_base) * CT_THREADS + threadIdx.x; e < total;
       e += (long long)p.blocks * CT_THREADS) {
    const long long j = e / p.f, f = e - j * p.f;
    const float v = j < p.kk ? __ldg(p.weight + f * p.kk + j) : 0.0f;
    reinterpret_cast<__nv_bfloat16*>(p.wpad)[e] = __float2bfloat16_rn(v);
  }
}

// K-split forward-type conv GEMM finish (HNN_CONVTC_SPLITK_FWD): the splits' raw sums, in order,
// + bias, relu; written NCHW (and the NHWC bf16 copy for an implicit next layer) exactly like the
// unsplit GEMM epilogue (gemm_tc2.cu, c_mode 1).  Phase 1 reads the partials along n (coalesced),
// phase 2 writes NCHW along the pixels through a padded shared tile.
constexpr int SK_BATCH = 4;  // partial loads in flight per element

__global__ void __launch_bounds__(CT_THREADS) splitk_fwd_kernel(const hnn_convtc_problem* __restrict__ probs,
                                                                int nprob, const hnn_step_row* __restrict__ cur,
                                                                const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const hnn_convtc_problem& p = ct_problem(probs, nprob, blockIdx.x);
  if (!live(cur, status, p.model)) return;
  __shared__ float tile[32][33];
  const int t = blockIdx.x - p.block_base, nblk = (p.f + 31) / 32;
  const int m0 = (t / nblk) * 32, n0 = (t % nblk) * 32;
  const int hw = p.oh * p.ow, M = p.cap * hw, R = cur[p.model].rows * hw;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int n = n0 + tx;
  const float bias = (p.db && n < p.f) ? __ldg(p.db + n) : 0.0f;
  const size_t split = size_t(p.pix_ld) * p.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty + 8 * i, m = m0 + r;
    float v = 0.0f;
    if (m < R && n < p.f) {
      const float* src = p.partial + size_t(m) * p.f + n;
      v = __ldg(src);
      for (int s0 = 1; s0 < p.ksplit; s0 += SK_BATCH) {
        float q[SK_BATCH];
#pragma unroll
        for (int j = 0; j < SK_BATCH; ++j) q[j] = s0 + j < p.ksplit ? __ldg(src + (s0 + j) * split) : 0.0f;
#pragma unroll
        for (int j = 0; j < SK_BATCH; ++j)
          if (s0 + j < p.ksplit) v = __fadd_rn(v, q[j]);
      }
      v = __fadd_rn(v, bias);
      if (p.rsc) v = np_relu(v);
    }
    tile[r][tx] = v;
    if (p.dyt && m < M && n < p.f) reinterpret_cast<__nv_bfloat16*>(p.dyt)[size_t(m) * p.f + n] = __float2bfloat16_rn(v);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = ty + 8 * i, no = n0 + c, m = m0 + tx;
    if (m >= M || no >= p.f) continue;
    const int b = m / hw, pix = m - b * hw;
    const size_t o = (size_t(b) * p.f + no) * hw + pix;
    float v = tile[tx][c];
    if (p.mask) v = m < R ? np_mask(v, __ldg(p.mask + o)) : 0.0f;
    p.dx[o] = v;
  }
}

}  // namespace hnn

extern "C" int hnn_conv_tc_aux(int op, const hnn_convtc_problem* probs, int nprob, int total_blocks, int max_k,
                               const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_blocks > 0, "hnn_conv_tc_aux", "bad arguments");
  cudaStream_t s = hnn::as_stream(stream);
  switch (op) {
    case HNN_CONVTC_IM2COL:
      HNN_REQUIRE(max_k > 0 && max_k <= 5, "hnn_conv_tc_aux", "kernel size above 5");
      cudaFuncSetAttribute(hnn::im2col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, hnn::im2col_smem_bytes(5));
      hnn::launch_pdl(hnn::im2col_kernel, dim3(total_blocks), dim3(hnn::CT_THREADS), hnn::im2col_smem_bytes(max_k), s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_TRANSPOSE_DY:
      hnn::launch_pdl(hnn::transpose_dy_kernel, dim3(total_blocks), dim3(hnn::CT_THREADS), 0, s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_COL2IM:
      HNN_REQUIRE(max_k > 0 && max_k <= 3, "hnn_conv_tc_aux", "kernel size above 3");
      cudaFuncSetAttribute(hnn::col2im_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, hnn::col2im_smem_bytes(3));
      hnn::launch_pdl(hnn::col2im_kernel, dim3(total_blocks), dim3(hnn::CT_THREADS), hnn::col2im_smem_bytes(max_k), s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_PAD_WEIGHTS:
      hnn::launch_pdl(hnn::pad_weights_kernel, dim3(total_blocks), dim3(hnn::CT_THREADS), 0, s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_FLIP_WEIGHTS:
      hnn::launch_pdl(hnn::flip_weights_kernel, dim3(total_blocks), dim3(hnn::CT_THREADS), 0, s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_PAD_WEIGHTS_RSC:
      hnn::launch_pdl(hnn::rsc_weights_kernel<false>, dim3(total_blocks), dim3(hnn::CT_THREADS), 0, s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_FLIP_WEIGHTS_RSC:
      hnn::launch_pdl(hnn::rsc_weights_kernel<true>, dim3(total_blocks), dim3(hnn::CT_THREADS), 0, s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_PARITY_WEIGHTS:
      hnn::launch_pdl(hnn::parity_weights_kernel, dim3(total_blocks), dim3(hnn::CT_THREADS), 0, s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_WT_WEIGHTS:
      hnn::launch_pdl(hnn::wt_weights_kernel, dim3(total_blocks), dim3(hnn::CT_THREADS), 0, s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_SPLITK_FWD:
      hnn::launch_pdl(hnn::splitk_fwd_kernel, dim3(total_blocks), dim3(hnn::CT_THREADS), 0, s, probs, nprob, cur, status);
      break;
    case HNN_CONVTC_WGRAD_REDUCE:
      hnn::launch_pdl(hnn::wgrad_reduce_kernel, dim3(total_blocks), dim3(hnn::CT_THREADS), 0, s, probs, nprob, cur, status);
      break;
    default:
      hnn::set_error("hnn_conv_tc_aux", "unknown op");
      return HNN_ERR_INVALID;
  }
  return hnn::check_launch("hnn_conv_tc_aux");
}
