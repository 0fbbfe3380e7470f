// numpy-exact softmax-cross-entropy row arithmetic shared by sce.cu and tail.cu
// (pkg/src/hybridnn/ops.py:220-251).
#pragma once

#include "common.cuh"

namespace hnn {

// numpy @TYPE@_pairwise_sum for float32, contiguous (reduce starts from +0.0).
__device__ inline float np_pairwise_sum(const float* a, int n) {
  if (n < 8) {
    float res = 0.0f;
    for (int i = 0; i < n; ++i) res = __fadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], a[i + j]);
    float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                          __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __fadd_rn(res, a[i]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __fadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
}

// One row per thread for C <= 16 classes (every config: 10): the warp-per-row path below spends
// its time in lane-0 serial sections (34 us for C3's 32 x 256 rows).  Same arithmetic, in
// registers: numpy max / argmax NaN rules, expf of shifted logits, numpy's pairwise float32 sum.
template <int CM>
__device__ __forceinline__ void sce_row_thread(const float* lrow, float* drow, int C, int t, float inv_n,
                                               float& logp, int& hit) {
  float v[CM], e[CM];
#pragma unroll
  for (int j = 0; j < CM; ++j) v[j] = j < C ? lrow[j] : 0.0f;
  float mx = v[0], best = v[0];
  int arg = 0;
  bool nan_seen = (best != best);
#pragma unroll
  for (int j = 1; j < CM; ++j) {
    if (j >= C) break;
    const float x = v[j];
    if (!nan_seen && !(x <= best)) {
      best = x;
      arg = j;
      if (x != x) nan_seen = true;
    }
    mx = (mx >= x || mx != mx) ? mx : x;
  }
  if (nan_seen) mx = __int_as_float(0x7fc00000);
  float sh_t = 0.0f;
#pragma unroll
  for (int j = 0; j < CM; ++j) {
    if (j >= C) break;
    const float sh = __fsub_rn(v[j], mx);
    if (j == t) sh_t = sh;
    e[j] = expf(sh);
  }
  float sum;
  if (C < 8) {
    sum = 0.0f;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < C) sum = __fadd_rn(sum, e[j]);
  } else {
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = e[j];
    const int full = C - (C % 8);
#pragma unroll
    for (int i = 8; i < CM; i += 8)
      if (i < full)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], e[i + j]);
    sum = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                    __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
#pragma unroll
    for (int j = 8; j < CM; ++j)
      if (j >= full && j < C) sum = __fadd_rn(sum, e[j]);
  }
  const float lse = logf(sum);
  logp = __fsub_rn(sh_t, lse);
  hit = (arg == t);
  if (drow) {
#pragma unroll
    for (int j = 0; j < CM; ++j) {
      if (j >= C) break;
      float pr = expf(__fsub_rn(__fsub_rn(v[j], mx), lse));
      if (j == t) pr = __fsub_rn(pr, 1.0f);
      drow[j] = __fmul_rn(pr, inv_n);
    }
  }
}

}  // namespace hnn
