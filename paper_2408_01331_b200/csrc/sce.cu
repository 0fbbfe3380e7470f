// Fused softmax-cross-entropy + accuracy + abort flag, one CTA per model
// (pkg/src/hybridnn/ops.py:220-251, train.py:239-243, 252-255, 274-276).
//
// Reductions follow numpy's float32 order exactly: row sums and the batch
// mean use numpy's pairwise summation (8 accumulators, blocks of 128,
// recursive halving on multiples of 8), the row max / argmax are sequential
// scans with numpy's NaN rules.  Given identical logits the loss, dlogits and
// correct count therefore match the reference up to expf/logf rounding.
#include "sce_common.cuh"

namespace hnn {

constexpr int SCE_THREADS = 1024, SCE_WARPS = SCE_THREADS / 32;

__global__ void __launch_bounds__(SCE_THREADS) sce_kernel(const hnn_sce_problem* __restrict__ probs,
                                                          const hnn_step_row* __restrict__ cur,
                                                          hnn_model_status* __restrict__ status, int train,
                                                          float* __restrict__ loss_out,
                                                          int32_t* __restrict__ correct_out, int max_classes) {
  hnn::pdl_wait();
  extern __shared__ float smem[];
  const hnn_sce_problem p = probs[blockIdx.x];
  if (!cur[p.model].active) return;
  if (train && status && !status[p.model].alive) return;
  const hnn_step_row s = cur[p.model];
  const int R = s.rows, C = p.classes;
  float* logp = smem;                                    // [cap]
  float* rowbuf = smem + p.cap + (threadIdx.x / 32) * max_classes;  // per-warp [C]
  __shared__ int warp_hits[SCE_WARPS];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int hits = 0;
  const float inv_n = __fdiv_rn(1.0f, (float)R);
  if (C <= 16) {
    for (int r = threadIdx.x; r < p.cap; r += SCE_THREADS) {
      float* drow = p.dlogits ? p.dlogits + size_t(r) * p.ld : nullptr;
      if (r >= R) {
        if (drow)
          for (int j = 0; j < C; ++j) drow[j] = 0.0f;
        continue;
      }
      float lp;
      int hit;
      sce_row_thread<16>(p.logits + size_t(r) * p.ld, drow, C, p.labels[r], inv_n, lp, hit);
      logp[r] = lp;
      hits += hit;
    }
    hits = __reduce_add_sync(0xffffffffu, hits);
  } else
  for (int r = warp; r < p.cap; r += SCE_WARPS) {
    float* drow = p.dlogits ? p.dlogits + size_t(r) * p.ld : nullptr;
    if (r >= R) {
      if (drow)
        for (int j = lane; j < C; j += 32) drow[j] = 0.0f;
      continue;
    }
    const float* lrow = p.logits + size_t(r) * p.ld;
    for (int j = lane; j < C; j += 32) rowbuf[j] = lrow[j];
    __syncwarp();
    float mx = 0.0f;
    int arg = 0;
    if (lane == 0) {
      // np.max (NaN propagates) and np.argmax (first max, first NaN stops)
      mx = rowbuf[0];
      float best = rowbuf[0];
      bool nan_seen = (best != best);
      for (int j = 1; j < C; ++j) {
        const float v = rowbuf[j];
        if (!nan_seen && !(v <= best)) {
          best = v;
          arg = j;
          if (v != v) nan_seen = true;
        }
        mx = (mx >= v || mx != mx) ? mx : v;
      }
      if (nan_seen) mx = __int_as_float(0x7fc00000);
    }
    mx = __shfl_sync(0xffffffffu, mx, 0);
    arg = __shfl_sync(0xffffffffu, arg, 0);
    const int t = p.labels[r];
    __syncwarp();
    float sh_t = 0.0f;
    for (int j = lane; j < C; j += 32) {
      const float sh = __fsub_rn(rowbuf[j], mx);
      if (j == t) sh_t = sh;
      rowbuf[j] = expf(sh);
    }
    // the lane that owns column t broadcasts shifted[t]
    sh_t = __shfl_sync(0xffffffffu, sh_t, t % 32);
    __syncwarp();
    float lse = 0.0f;
    if (lane == 0) lse = logf(np_pairwise_sum(rowbuf, C));
    lse = __shfl_sync(0xffffffffu, lse, 0);
    if (lane == 0) {
      logp[r] = __fsub_rn(sh_t, lse);
      hits += (arg == t);
    }
    if (drow) {
      for (int j = lane; j < C; j += 32) {
        float pr = expf(__fsub_rn(__fsub_rn(lrow[j], mx), lse));
        if (j == t) pr = __fsub_rn(pr, 1.0f);
        drow[j] = __fmul_rn(pr, inv_n);
      }
    }
    __syncwarp();
  }
  if (lane == 0) warp_hits[warp] = hits;
  __syncthreads();
  if (threadIdx.x == 0) {
    int correct = 0;
    for (int w = 0; w < SCE_WARPS; ++w) correct += warp_hits[w];
    const float mean = __fdiv_rn(np_pairwise_sum(logp, R), (float)R);
    const float loss = -mean;
    const bool finite = isfinite(loss);
    if (train && !finite) correct = 0;
    if (loss_out) loss_out[p.model] = loss;
    if (correct_out) correct_out[p.model] = correct;
    if (status) {
      hnn_model_status& st = status[p.model];
      st.last_loss = loss;
      st.last_correct = correct;
      if (train && !finite) {
        st.alive = 0;
        st.abort_epoch = s.epoch;
        st.abort_batch = s.batch;
      } else {
        st.loss_sum += (double)loss * (double)R;
        st.correct_sum += correct;
        st.seen += R;
      }
    }
  }
}

}  // namespace hnn

extern "C" int hnn_sce_fused(const hnn_sce_problem* probs, int nprob, int max_cap, int max_classes,
                             const hnn_step_row* cur, hnn_model_status* status, int train, float* loss_out,
                             int32_t* correct_out, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && max_cap > 0 && max_classes > 0, "hnn_sce_fused", "bad arguments");
  const size_t smem = (size_t(max_cap) + size_t(hnn::SCE_WARPS) * max_classes) * sizeof(float);
  HNN_REQUIRE(smem <= 200 * 1024, "hnn_sce_fused", "batch capacity / class count too large for one CTA");
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(hnn::sce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  hnn::launch_pdl(hnn::sce_kernel, dim3(nprob), dim3(hnn::SCE_THREADS), smem, hnn::as_stream(stream), probs, cur, status, train, loss_out,
                                                                              correct_out, max_classes);
  return hnn::check_launch("hnn_sce_fused");
}
