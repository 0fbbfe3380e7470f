// Fused logits tail of small models: the last dense layer's forward, softmax-cross-entropy +
// accuracy + abort flag, and the layer's input and weight gradients (+ the fused SGD / momentum
// update) in ONE launch, one CTA per model (pkg/src/hybridnn/ops.py:46-55 dense fwd / bwd,
// ops.py:220-251 SCE, train.py:239-256 abort-before-update).
//
// For the batch-64 / 128 configs (C1, C2, C4, C5) the four launches it replaces (skinny forward,
// SCE, skinny input gradient, skinny weight gradient) were each a ~10-25 us latency chain on a
// handful of CTAs (profiles/r02/step_breakdown_c5_v9.txt: 47 of C5's 111 us).  Here the layer's
// input rows stay in L2 / L1 between the phases and W lives in shared memory, so the SGD update of
// W (after the input gradient read it) needs no ordering across CTAs.
//
// Arithmetic: the SCE rows and the batch loss follow sce.cu exactly (numpy max / argmax NaN rules,
// pairwise float32 sums); the dot products are plain FMA chains in a fixed order (the GEMM of the
// reference is BLAS: compared with the oracle at tolerance); the bias gradient is numpy's axis-0
// order.  A non-finite loss aborts the model before any gradient or update.
#include "sce_common.cuh"

namespace hnn {

constexpr int TAIL_THREADS = 512, TAIL_WARPS = TAIL_THREADS / 32, TAIL_CMAX = 16;

template <int MJ>
__device__ __forceinline__ void tail_backward(const hnn_tail_problem& p, int R, const float* ws, const float* D,
                                              float* red, const Update& u) {
  // thread = (column quad qd, row group g): dX rows and the weight-gradient partials of its quad
  const int Q = p.k / 4, G = max(1, TAIL_THREADS / Q);
  const int g = threadIdx.x / Q, qd = threadIdx.x - g * Q;
  const bool active = g < G && qd < Q;
  float part[MJ][4];
#pragma unroll
  for (int j = 0; j < MJ; ++j) part[j][0] = part[j][1] = part[j][2] = part[j][3] = 0.0f;
  if (active) {
    float4 w[MJ];
#pragma unroll
    for (int j = 0; j < MJ; ++j) w[j] = j < p.classes ? reinterpret_cast<const float4*>(ws + j * p.k)[qd] : make_float4(0, 0, 0, 0);
    const int r_lo = (R * g) / G, r_hi = (R * (g + 1)) / G;
#pragma unroll 4
    for (int r = r_lo; r < r_hi; ++r) {
      const float4 xv = __ldg(reinterpret_cast<const float4*>(p.x + size_t(r) * p.ldx) + qd);
      const float* dr = D + r * TAIL_CMAX;
      float4 o = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int j = 0; j < MJ; ++j) {
        const float dj = j < p.classes ? dr[j] : 0.0f;  // (columns past the classes are not written)
        part[j][0] = fmaf(dj, xv.x, part[j][0]);
        part[j][1] = fmaf(dj, xv.y, part[j][1]);
        part[j][2] = fmaf(dj, xv.z, part[j][2]);
        part[j][3] = fmaf(dj, xv.w, part[j][3]);
        o.x = fmaf(dj, w[j].x, o.x);
        o.y = fmaf(dj, w[j].y, o.y);
        o.z = fmaf(dj, w[j].z, o.z);
        o.w = fmaf(dj, w[j].w, o.w);
      }
      if (p.dx) {
        if (p.mask) {
          const float4 mk = p.mask == p.x ? xv : __ldg(reinterpret_cast<const float4*>(p.mask + size_t(r) * p.ldx) + qd);
          o.x = np_mask(o.x, mk.x);
          o.y = np_mask(o.y, mk.y);
          o.z = np_mask(o.z, mk.z);
          o.w = np_mask(o.w, mk.w);
        }
        reinterpret_cast<float4*>(p.dx + size_t(r) * p.ld_dx)[qd] = o;
      }
    }
    if (p.dx)  // rows past this step's batch: exact zeros
      for (int r = R + g; r < p.cap; r += G)
        reinterpret_cast<float4*>(p.dx + size_t(r) * p.ld_dx)[qd] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (g > 0) {
      float* dst = red + (size_t(g - 1) * Q + qd) * (TAIL_CMAX * 4);
#pragma unroll
      for (int j = 0; j < MJ; ++j)
        *reinterpret_cast<float4*>(dst + j * 4) = make_float4(part[j][0], part[j][1], part[j][2], part[j][3]);
    }
  }
  __syncthreads();
  if (active && g == 0) {
    for (int gg = 1; gg < G; ++gg) {  // row groups in fixed order
      const float* src = red + (size_t(gg - 1) * Q + qd) * (TAIL_CMAX * 4);
#pragma unroll
      for (int j = 0; j < MJ; ++j) {
        const float4 v = *reinterpret_cast<const float4*>(src + j * 4);
        part[j][0] += v.x;
        part[j][1] += v.y;
        part[j][2] += v.z;
        part[j][3] += v.w;
      }
    }
#pragma unroll
    for (int j = 0; j < MJ; ++j) {
      if (j >= p.classes) break;
      const size_t off = size_t(j) * p.k + size_t(qd) * 4;
      if (p.dw) *reinterpret_cast<float4*>(p.dw + off) = make_float4(part[j][0], part[j][1], part[j][2], part[j][3]);
      if (p.opt_w) {
        float4 w = *reinterpret_cast<const float4*>(ws + off);
        float4 m = p.opt_wm ? *reinterpret_cast<const float4*>(p.opt_wm + off) : make_float4(0, 0, 0, 0);
        update_sgd(u, w.x, part[j][0], m.x);
        update_sgd(u, w.y, part[j][1], m.y);
        update_sgd(u, w.z, part[j][2], m.z);
        update_sgd(u, w.w, part[j][3], m.w);
        *reinterpret_cast<float4*>(p.opt_w + off) = w;
        if (p.opt_wm) *reinterpret_cast<float4*>(p.opt_wm + off) = m;
      }
    }
  }
}

__global__ void __launch_bounds__(TAIL_THREADS) logits_tail_kernel(const hnn_tail_problem* __restrict__ probs,
                                                                   const hnn_step_row* __restrict__ cur,
                                                                   hnn_model_status* __restrict__ status,
                                                                   float* __restrict__ loss_out,
                                                                   int32_t* __restrict__ correct_out) {
  hnn::pdl_wait();
  extern __shared__ __align__(16) float tsm[];
  const hnn_tail_problem p = probs[blockIdx.x];
  if (!cur[p.model].active) return;
  if (status && !status[p.model].alive) return;
  const hnn_step_row s = cur[p.model];
  const int R = s.rows, C = p.classes, K = p.k;
  float* ws = tsm;                                   // [C][K] the layer's weights
  float* L = ws + C * K;                             // [cap][16] logits of the batch
  float* D = L + p.cap * TAIL_CMAX;                  // [cap][16] dlogits
  float* logp = D + p.cap * TAIL_CMAX;               // [cap]
  float* red = logp + ((p.cap + 3) & ~3);            // row-group partials of the weight gradient
  __shared__ int warp_hits[TAIL_WARPS];
  __shared__ int s_finite;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int e = threadIdx.x; e < C * K / 4; e += TAIL_THREADS)
    reinterpret_cast<float4*>(ws)[e] = __ldg(reinterpret_cast<const float4*>(p.w) + e);
  __syncthreads();
  // ---- forward: a warp per row, lanes stride K by float4, a fixed xor tree per column
  for (int r = warp; r < p.cap; r += TAIL_WARPS) {
    float acc[TAIL_CMAX];
#pragma unroll
    for (int j = 0; j < TAIL_CMAX; ++j) acc[j] = 0.0f;
    if (r < R) {
      const float4* xr = reinterpret_cast<const float4*>(p.x + size_t(r) * p.ldx);
      for (int k4 = lane; k4 < K / 4; k4 += 32) {
        const float4 xv = __ldg(xr + k4);
#pragma unroll
        for (int j = 0; j < TAIL_CMAX; ++j)
          if (j < C) {
            const float4 wv = reinterpret_cast<const float4*>(ws + j * K)[k4];
            acc[j] = fmaf(xv.x, wv.x, fmaf(xv.y, wv.y, fmaf(xv.z, wv.z, fmaf(xv.w, wv.w, acc[j]))));
          }
      }
    }
#pragma unroll
    for (int j = 0; j < TAIL_CMAX; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    float v = 0.0f;
#pragma unroll
    for (int j = 0; j < TAIL_CMAX; ++j)
      if (j == lane) v = acc[j];
    if (lane < C) {
      float y = 0.0f;
      if (r < R) y = __fadd_rn(v, __ldg(p.b + lane));  // rows past the batch: exact zeros
      L[r * TAIL_CMAX + lane] = y;
      if (p.logits) p.logits[size_t(r) * p.ld_logits + lane] = y;
    }
  }
  __syncthreads();
  // ---- softmax-cross-entropy, one row per thread (sce.cu's arithmetic)
  int hits = 0;
  const float inv_n = __fdiv_rn(1.0f, (float)R);
  for (int r = threadIdx.x; r < R; r += TAIL_THREADS) {
    float lp;
    int hit;
    sce_row_thread<TAIL_CMAX>(L + r * TAIL_CMAX, D + r * TAIL_CMAX, C, p.labels[r], inv_n, lp, hit);
    logp[r] = lp;
    hits += hit;
  }
  hits = __reduce_add_sync(0xffffffffu, hits);
  if (lane == 0) warp_hits[warp] = hits;
  __syncthreads();
  if (threadIdx.x == 0) {
    int correct = 0;
    for (int w = 0; w < TAIL_WARPS; ++w) correct += warp_hits[w];
    const float loss = -__fdiv_rn(np_pairwise_sum(logp, R), (float)R);
    const bool finite = isfinite(loss);
    if (!finite) correct = 0;
    if (loss_out) loss_out[p.model] = loss;
    if (correct_out) correct_out[p.model] = correct;
    if (status) {
      hnn_model_status& st = status[p.model];
      st.last_loss = loss;
      st.last_correct = correct;
      if (!finite) {
        st.alive = 0;
        st.abort_epoch = s.epoch;
        st.abort_batch = s.batch;
      } else {
        st.loss_sum += (double)loss * (double)R;
        st.correct_sum += correct;
        st.seen += R;
      }
    }
    s_finite = finite;
  }
  __syncthreads();
  if (!s_finite) return;  // abort before any gradient or update (train.py:239-243)
  // ---- bias gradient (numpy's axis-0 order) and its fused update
  const Update u = make_update(s, p.opt_kind, p.opt_momentum);
  if (threadIdx.x < C) {
    const int j = threadIdx.x;
    float bsum = -0.0f;
    for (int r = 0; r < R; ++r) bsum = __fadd_rn(bsum, D[r * TAIL_CMAX + j]);
    if (p.db) p.db[j] = bsum;
    if (p.opt_b) {
      float w = p.opt_b[j], m = p.opt_bm ? p.opt_bm[j] : 0.0f;
      update_sgd(u, w, bsum, m);
      p.opt_b[j] = w;
      if (p.opt_bm) p.opt_bm[j] = m;
    }
  }
  // ---- input gradient + weight gradient in one pass over the layer input
  if (C <= 4) tail_backward<4>(p, R, ws, D, red, u);
  else if (C <= 8) tail_backward<8>(p, R, ws, D, red, u);
  else if (C <= 10) tail_backward<10>(p, R, ws, D, red, u);
  else tail_backward<16>(p, R, ws, D, red, u);
}

}  // namespace hnn

extern "C" int hnn_tail_smem(int cap, int k, int classes) {
  const int Q = k / 4, G = Q > 0 ? (hnn::TAIL_THREADS / Q > 1 ? hnn::TAIL_THREADS / Q : 1) : 1;
  return 4 * (classes * k + 2 * cap * hnn::TAIL_CMAX + ((cap + 3) & ~3) + (G - 1) * Q * hnn::TAIL_CMAX * 4);
}

extern "C" int hnn_logits_tail(const hnn_tail_problem* probs, int nprob, int smem, const hnn_step_row* cur,
                               hnn_model_status* status, float* loss_out, int32_t* correct_out, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && smem > 0 && smem <= 200 * 1024, "hnn_logits_tail", "bad arguments");
  static int configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(hnn::logits_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = 200 * 1024;
  }
  hnn::launch_pdl(hnn::logits_tail_kernel, dim3(nprob), dim3(hnn::TAIL_THREADS), smem, hnn::as_stream(stream), probs,
                  cur, status, loss_out, correct_out);
  return hnn::check_launch("hnn_logits_tail");
}
