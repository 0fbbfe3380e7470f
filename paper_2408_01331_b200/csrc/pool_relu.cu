// Grouped max-pool (fwd/bwd, relu mask fused into bwd) and stand-alone relu
// (pkg/src/hybridnn/ops.py:62-67, 149-174).  HBM-bound elementwise kernels.  Per problem
// (hnn_pool_problem.mode): 2 x 2 / stride 2 pools on even planes run one thread per four windows
// (both directions); other windows one thread per output (fwd) or per input element (bwd,
// gather form, so the reference's np.add.at scatter becomes a fixed-order sum with no atomics).
#include <cuda_bf16.h>

#include "common.cuh"

namespace hnn {

constexpr int PTHREADS = 256;

// ------------------------------------------------------------- 2 x 2 windows (HNN_POOL_WINDOWS_2X2)
// One unit per window for both directions, PW windows per thread with every load issued before
// the first compare: the elementwise form (one 256-element CTA per block, ~5 dependent round trips
// per CTA: problem search, problem, batch rows, data, store) ran 16 waves of latency-bound CTAs
// per SM (C2's first pool gradient: 46 us for 45 MB).  h and w are even, so a window's two row
// pairs are aligned float2 and (DGRAD) every input element lies in exactly one window.
constexpr int PW = HNN_POOL_WINDOWS_PER_BLOCK / PTHREADS;
static_assert(PW * PTHREADS == HNN_POOL_WINDOWS_PER_BLOCK, "whole windows per thread");

struct WinPos {
  int plane, b, pix;  // pix: the window's top-left input element within its plane
};

__device__ __forceinline__ WinPos win_pos(const hnn_pool_problem& p, int e) {
  const int ohw = p.oh * p.ow;
  WinPos r;
  r.plane = e / ohw;
  const int o = e - r.plane * ohw, oy = o / p.ow, ox = o - oy * p.ow;
  r.b = r.plane / p.c;
  r.pix = (2 * oy) * p.w + 2 * ox;
  return r;
}

__device__ __forceinline__ void maxpool2_fwd(const hnn_pool_problem& p, int rows) {
  const int total = p.cap * p.c * p.oh * p.ow, hw = p.h * p.w;
  const int e0 = (blockIdx.x - p.block_base) * HNN_POOL_WINDOWS_PER_BLOCK + threadIdx.x;
  float2 r0[PW], r1[PW];
#pragma unroll
  for (int u = 0; u < PW; ++u) {
    const int e = e0 + u * PTHREADS;
    r0[u] = r1[u] = make_float2(0.0f, 0.0f);
    if (e < total) {
      const WinPos q = win_pos(p, e);
      if (q.b < rows) {
        const float* s0 = p.x + size_t(q.plane) * hw + q.pix;
        r0[u] = *reinterpret_cast<const float2*>(s0);
        r1[u] = *reinterpret_cast<const float2*>(s0 + p.w);
      }
    }
  }
  __nv_bfloat16* xh = reinterpret_cast<__nv_bfloat16*>(p.xh);  // NHWC bf16 copy: [(b, o), c]
#pragma unroll
  for (int u = 0; u < PW; ++u) {
    const int e = e0 + u * PTHREADS;
    if (e >= total) break;
    const WinPos q = win_pos(p, e);
    // numpy argmax over (0,0) (0,1) (1,0) (1,1): first max wins, first NaN wins outright
    float best = r0[u].x;
    int best_i = 0;
    if (best == best) {
      const float vs[3] = {r0[u].y, r1[u].x, r1[u].y};
#pragma unroll
      for (int k = 1; k < 4; ++k) {
        const float v = vs[k - 1];
        if (!(v <= best)) {
          best = v;
          best_i = k;
          if (v != v) break;
        }
      }
    }
    if (q.b >= rows) best = 0.0f, best_i = 0;  // rows past the batch: zeros (loads skipped)
    p.y[e] = best;
    p.idx[e] = (uint8_t)best_i;
    if (xh) {
      const int ohw = p.oh * p.ow, o = e - q.plane * ohw;
      xh[(size_t(q.b) * ohw + o) * p.c + (q.plane - q.b * p.c)] = __float2bfloat16_rn(best);
    }
  }
}

__device__ __forceinline__ void maxpool2_bwd(const hnn_pool_problem& p, int rows) {
  const int total = p.cap * p.c * p.oh * p.ow, hw = p.h * p.w;
  const int e0 = (blockIdx.x - p.block_base) * HNN_POOL_WINDOWS_PER_BLOCK + threadIdx.x;
  float d[PW];
  int ix[PW];
  float2 m0[PW], m1[PW];
#pragma unroll
  for (int u = 0; u < PW; ++u) {
    const int e = e0 + u * PTHREADS;
    d[u] = 0.0f;
    ix[u] = -1;  // (no window element selected: rows past the batch)
    m0[u] = m1[u] = make_float2(1.0f, 1.0f);
    if (e < total) {
      const WinPos q = win_pos(p, e);
      if (q.b < rows) {
        d[u] = p.dy[e];
        ix[u] = p.idx[e];
        if (p.mask) {
          const float* mk = p.mask + size_t(q.plane) * hw + q.pix;
          m0[u] = *reinterpret_cast<const float2*>(mk);
          m1[u] = *reinterpret_cast<const float2*>(mk + p.w);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < PW; ++u) {
    const int e = e0 + u * PTHREADS;
    if (e >= total) break;
    const WinPos q = win_pos(p, e);
    float g[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) g[k] = __fadd_rn(0.0f, ix[u] == k ? d[u] : 0.0f);  // np.add.at into zeros
    if (p.mask && ix[u] >= 0) {
      g[0] = np_mask(g[0], m0[u].x);
      g[1] = np_mask(g[1], m0[u].y);
      g[2] = np_mask(g[2], m1[u].x);
      g[3] = np_mask(g[3], m1[u].y);
    }
    float* dx = p.dx + size_t(q.plane) * hw + q.pix;
    *reinterpret_cast<float2*>(dx) = make_float2(g[0], g[1]);
    *reinterpret_cast<float2*>(dx + p.w) = make_float2(g[2], g[3]);
  }
}

__global__ void __launch_bounds__(PTHREADS) maxpool_fwd_kernel(const hnn_pool_problem* __restrict__ probs, int nprob,
                                                               const hnn_step_row* __restrict__ cur,
                                                               const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_pool_problem& q) { return q.block_base; });
  const hnn_pool_problem p = probs[pi];
  if (!live(cur, status, p.model)) return;
  if (p.mode == HNN_POOL_WINDOWS_2X2) return maxpool2_fwd(p, cur[p.model].rows);
  // 32-bit index arithmetic (the host keeps cap*c*h*w < 2^31): 64-bit divisions made these
  // elementwise kernels issue-bound (0.12 ms for a 33 MB pool gradient)
  const int e = (blockIdx.x - p.block_base) * PTHREADS + threadIdx.x;
  const int total = p.cap * p.c * p.oh * p.ow;
  if (e >= total) return;
  const int ohw = p.oh * p.ow;
  const int plane = e / ohw;  // b*C + c
  const int o = e - plane * ohw, oy = o / p.ow, ox = o - oy * p.ow;
  const int b = plane / p.c;
  __nv_bfloat16* xh = reinterpret_cast<__nv_bfloat16*>(p.xh);  // NHWC bf16 copy: [(b, o), c]
  const size_t xo = (size_t(b) * ohw + o) * p.c + (plane - b * p.c);
  if (b >= cur[p.model].rows) {
    p.y[e] = 0.0f;
    p.idx[e] = 0;
    if (xh) xh[xo] = __float2bfloat16_rn(0.0f);
    return;
  }
  const float* src = p.x + size_t(plane) * p.h * p.w;
  // numpy argmax over the window flattened (i, j): first max wins, first NaN wins outright
  float best;
  int best_i = 0;
  if (p.k == 2 && p.stride == 2 && 2 * oy + 1 < p.h && 2 * ox + 1 < p.w) {
    // the common 2 x 2 window: its four values requested together, then the same scan
    const float* s0 = src + (2 * oy) * p.w + 2 * ox;
    const float v0 = s0[0], v1 = s0[1], v2 = s0[p.w], v3 = s0[p.w + 1];
    best = v0;
    if (best == best) {
      const float vs[3] = {v1, v2, v3};
#pragma unroll
      for (int q = 1; q < 4; ++q) {
        const float v = vs[q - 1];
        if (!(v <= best)) {
          best = v;
          best_i = q;
          if (v != v) break;
        }
      }
    }
  } else if ((best = src[(oy * p.stride) * p.w + ox * p.stride]) == best) {
    for (int q = 1; q < p.k * p.k; ++q) {
      const int i = q / p.k, j = q - i * p.k;
      const float v = src[(oy * p.stride + i) * p.w + ox * p.stride + j];
      if (!(v <= best)) {
        best = v;
        best_i = q;
        if (v != v) break;
      }
    }
  }
  p.y[e] = best;
  p.idx[e] = (uint8_t)best_i;
  if (xh) xh[xo] = __float2bfloat16_rn(best);
}

__global__ void __launch_bounds__(PTHREADS) maxpool_bwd_kernel(const hnn_pool_problem* __restrict__ probs, int nprob,
                                                               const hnn_step_row* __restrict__ cur,
                                                               const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_pool_problem& q) { return q.block_base; });
  const hnn_pool_problem p = probs[pi];
  if (!live(cur, status, p.model)) return;
  if (p.mode == HNN_POOL_WINDOWS_2X2) return maxpool2_bwd(p, cur[p.model].rows);
  const int e = (blockIdx.x - p.block_base) * PTHREADS + threadIdx.x;
  const int total = p.cap * p.c * p.h * p.w;
  if (e >= total) return;
  const int hw = p.h * p.w;
  const int plane = e / hw, yx = e - plane * hw, y = yx / p.w, x = yx - y * p.w;
  const int b = plane / p.c;
  float acc = 0.0f;
  if (b < cur[p.model].rows && p.k == 2 && p.stride == 2) {
    // the common non-overlapping 2 x 2 window: exactly one window covers (y, x)
    const int oy = y >> 1, ox = x >> 1;
    // the window's argmax, its gradient and the relu mask are requested together (a gradient
    // load issued only after the argmax compare cost a second round trip)
    const float mk = p.mask ? p.mask[e] : 1.0f;
    if (oy < p.oh && ox < p.ow) {
      const size_t o = size_t(plane) * p.oh * p.ow + size_t(oy) * p.ow + ox;
      const float d = p.dy[o];
      const int ix = p.idx[o];
      if (ix == ((y & 1) << 1 | (x & 1))) acc = d;
      acc = __fadd_rn(0.0f, acc);  // (the general path's 0 + dy: -0 -> +0)
    }
    if (p.mask) acc = np_mask(acc, mk);
  } else if (b < cur[p.model].rows) {
    // windows (oy, ox) covering (y, x), visited in ascending (oy, ox) like np.add.at's index order
    const int oy_lo = max(0, (y - p.k + p.stride) / p.stride), oy_hi = min(p.oh - 1, y / p.stride);
    const int ox_lo = max(0, (x - p.k + p.stride) / p.stride), ox_hi = min(p.ow - 1, x / p.stride);
    const size_t obase = size_t(plane) * p.oh * p.ow;
    for (int oy = oy_lo; oy <= oy_hi; ++oy) {
      const int i = y - oy * p.stride;
      if (i < 0 || i >= p.k) continue;
      for (int ox = ox_lo; ox <= ox_hi; ++ox) {
        const int j = x - ox * p.stride;
        if (j < 0 || j >= p.k) continue;
        const size_t o = obase + size_t(oy) * p.ow + ox;
        if (p.idx[o] == i * p.k + j) acc = __fadd_rn(acc, p.dy[o]);
      }
    }
    if (p.mask) acc = np_mask(acc, p.mask[e]);
  }
  p.dx[e] = acc;
}

__global__ void __launch_bounds__(PTHREADS) relu_kernel(int op, const hnn_relu_problem* __restrict__ probs, int nprob,
                                                        const hnn_step_row* __restrict__ cur,
                                                        const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_relu_problem& q) { return q.block_base; });
  const hnn_relu_problem p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int e = (blockIdx.x - p.block_base) * PTHREADS + threadIdx.x;
  if (e >= p.cap * p.row) return;
  const bool real = (e / p.row) < cur[p.model].rows;
  if (op == HNN_FWD) p.y[e] = real ? np_relu(p.x[e]) : 0.0f;
  else p.dx[e] = real ? np_mask(p.dy[e], p.x[e]) : 0.0f;
}

}  // namespace hnn

extern "C" int hnn_grouped_maxpool(int op, const hnn_pool_problem* probs, int nprob, int total_blocks,
                                   const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_blocks > 0, "hnn_grouped_maxpool", "bad arguments");
  cudaStream_t s = hnn::as_stream(stream);
  if (op == HNN_FWD) hnn::launch_pdl(hnn::maxpool_fwd_kernel, dim3(total_blocks), dim3(hnn::PTHREADS), 0, s, probs, nprob, cur, status);
  else if (op == HNN_DGRAD) hnn::launch_pdl(hnn::maxpool_bwd_kernel, dim3(total_blocks), dim3(hnn::PTHREADS), 0, s, probs, nprob, cur, status);
  else {
    hnn::set_error("hnn_grouped_maxpool", "op must be HNN_FWD or HNN_DGRAD");
    return HNN_ERR_INVALID;
  }
  return hnn::check_launch("hnn_grouped_maxpool");
}

extern "C" int hnn_grouped_relu(int op, const hnn_relu_problem* probs, int nprob, int total_blocks,
                                const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_blocks > 0, "hnn_grouped_relu", "bad arguments");
  HNN_REQUIRE(op == HNN_FWD || op == HNN_DGRAD, "hnn_grouped_relu", "op must be HNN_FWD or HNN_DGRAD");
  hnn::launch_pdl(hnn::relu_kernel, dim3(total_blocks), dim3(hnn::PTHREADS), 0, hnn::as_stream(stream), op, probs, nprob, cur, status);
  return hnn::check_launch("hnn_grouped_relu");
}
