/*
 * hnn_b200.h — C-ABI of the B200 hybrid-training hot path.
 *
 * Replaces, for all N merged models at once, the per-model numpy work the
 * reference does inside train.run_batch (pkg/src/hybridnn/train.py:223-256):
 *
 *   entry point                 replaces (reference file:line)
 *   --------------------------  -------------------------------------------------------
 *   hnn_step_begin              per-batch schedule: store.batches / lr_at_epoch / opt step
 *                               (store.py:68-81, optim.py:22-30, optim.py:57,73-76)
 *   hnn_gather_rows             Batch(x=train_x[idx], y=train_y[idx])   (store.py:77-80)
 *   hnn_host_gather_rows        the same gather on the host (data loader of the host-fed step)
 *   hnn_host_gather_batch       one step's host gather for all models, split over host threads
 *   hnn_hostfed_step            the host-fed step's copies + graph launch as one native call
 *   hnn_grouped_gemm            dense fwd / bwd  _dense_fwd, _dense_bwd (ops.py:46-55) with
 *                               relu fwd/bwd fused (ops.py:62-67); fp32 SIMT or tcgen05 3xTF32
 *   hnn_gemm_tc_encode          host-side TMA descriptors for the tcgen05 path
 *   hnn_grouped_conv            conv2d fwd / bwd _conv2d_fwd, _conv2d_bwd (ops.py:100-130): a SIMT
 *                               implicit-GEMM fallback (64x32 tiles); the planner routes LeNet-class
 *                               layers to hnn_grouped_conv_direct[_ex] and wide ones to hnn_conv_tc_aux
 *                               + the tcgen05 GEMMs, so the default routes never launch it
 *   hnn_grouped_conv_direct     the same for small channel counts, direct (register-blocked over
 *                               filters / channels x 4 outputs; _ex takes the block size)
 *   hnn_conv_tc_aux             im2col / NHWC copies / dy transposes / weight layouts / split reduce
 *                               around the tensor-core conv GEMMs (ops.py:100-130)
 *   hnn_conv_wgrad_reduce       the fixed-order finish of the conv weight/bias gradient
 *   hnn_skinny_backward         the <= 10-unit logits layer's input + weight gradient in one pass
 *   hnn_grouped_maxpool         maxpool2d fwd / bwd (ops.py:149-174), relu mask fused
 *   hnn_grouped_relu            stand-alone relu fwd / bwd (ops.py:62-67)
 *   hnn_logits_tail             a small model's logits layer fwd + SCE + bwd (+ fused SGD) in one launch
 *   hnn_sce_fused               softmax_cross_entropy + argmax accuracy + non-finite abort
 *                               (ops.py:220-251, train.py:239-243,252-255)
 *   hnn_multi_tensor_sgd        optim.apply_update, SGD / momentum branch (optim.py:59-71)
 *   hnn_multi_tensor_adam       optim.apply_update, Adam branch (optim.py:73-87); both run the bulk-
 *                               copy multi-tensor kernel (HNN_OPT_BULK=0: the per-thread one)
 *   hnn_last_error              error text for the last nonzero status on this thread
 *
 * Conventions (every entry point):
 *   - all pointers are caller-owned DEVICE memory except where noted; the
 *     problem tables themselves live in device memory;
 *   - every call is asynchronous and stream-ordered on `stream`
 *     (a cudaStream_t passed as void*); no allocation, no host sync;
 *   - return 0 on success, a nonzero HNN_ERR_* otherwise (no C++ exception
 *     crosses the ABI); hnn_last_error() describes the failure;
 *   - a model takes part in a launch only if its current schedule row has
 *     active != 0 and (when a status array is passed) its status.alive != 0;
 *   - results per model never depend on which other models share a launch:
 *     tiling is a fixed function of each problem's own shape, there are no
 *     atomics and no data-dependent split-K, so isolation is bit-exact.
 */
#ifndef HNN_B200_H
#define HNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HNN_OK 0
#define HNN_ERR_INVALID 1     /* bad argument / unsupported shape */
#define HNN_ERR_CUDA 2        /* a CUDA runtime call failed */
#define HNN_ERR_UNSUPPORTED 3 /* feature not built into this library */

/* hnn_grouped_gemm / hnn_grouped_conv `op` */
#define HNN_FWD 0
#define HNN_DGRAD 1
#define HNN_WGRAD 2

/* hnn_grouped_gemm `prec` */
#define HNN_PREC_F32_SIMT 0   /* fp32 FFMA, CUDA cores */
#define HNN_PREC_F32_3XTF32 1 /* tcgen05 kind::tf32, hi/lo split, fp32 accumulate in TMEM */
#define HNN_PREC_F32_3XTF32_PAIR 3 /* as HNN_PREC_F32_3XTF32 on CTA pairs (tcgen05 cta_group::2), 256 x 256
                                      tiles; same TMA maps (hnn_gemm_tc_encode).  The problem table MUST be
                                      followed by a tile schedule: int32 npairs, offsets[npairs + 1], tile
                                      ids[total_tiles]; when npairs != min(total_tiles, SMs/2) (or npairs is
                                      0) the pairs take tiles round-robin instead */
#define HNN_PREC_BF16_PAIR 4 /* CTA-pair tcgen05 kind::f16: a / b point to bf16 data, BOTH K-major for every op
                                (A [m, k], B [n, k], lda / ldb in elements; maps from hnn_gemm_bf16_encode),
                                fp32 accumulation, promotion and outputs as HNN_PREC_F32_3XTF32_PAIR */
#define HNN_PREC_F32_SIMT_SKINNY 2 /* fp32 FFMA streaming kernels for one dimension <= 16 (logits layers):
                                      FWD n <= 16, DGRAD k <= 16, WGRAD m <= 16; rows/columns multiple of 4 */

/* optimizer segment kinds */
#define HNN_OPT_SGD 0
#define HNN_OPT_SGD_MOMENTUM 1
#define HNN_OPT_ADAM 2

/* One model's schedule for the current step (device array, one row per model). */
typedef struct hnn_step_row {
  int32_t active;    /* model trains (or evaluates) at this step */
  int32_t rows;      /* real rows in this batch (<= the model's batch capacity) */
  int32_t perm_base; /* index into the model's permutation of the batch's first row */
  int32_t epoch;     /* zero-based epoch of this batch */
  int32_t batch;     /* zero-based batch index within the epoch */
  int32_t opt_step;  /* optimizer step count t after this update (1-based) */
  float lr;          /* F32(lr_at_epoch(...)) */
  float bias1;       /* F32(1 - 0.9^t)   (Adam) */
  float bias2;       /* F32(1 - 0.999^t) (Adam) */
  int32_t reserved[3];
} hnn_step_row; /* 48 bytes */

/* Persistent per-model device status, updated by hnn_sce_fused. */
typedef struct hnn_model_status {
  int32_t alive;       /* 0 once a non-finite loss was seen (the job aborts) */
  int32_t abort_epoch; /* epoch / batch of the first non-finite loss, -1 if none */
  int32_t abort_batch;
  int32_t last_correct;
  float last_loss;
  int32_t reserved;
  double loss_sum;     /* sum of F64(loss) * rows since the host last reset it */
  int64_t correct_sum; /* argmax hits since the last reset */
  int64_t seen;        /* rows since the last reset */
} hnn_model_status; /* 48 bytes */

/* Copy sched[*counter] (n_models rows) into cur and advance *counter. 1 block. */
int hnn_step_begin(const hnn_step_row* sched, int32_t* counter, hnn_step_row* cur, int n_models, void* stream);

typedef struct hnn_gather_problem {
  const float* src_x;     /* dataset samples [n, sample] */
  const int32_t* src_y;   /* dataset labels as int32 class ids [n] */
  const int32_t* perm;    /* this model's epoch permutation [n] (identity for evaluation) */
  float* dst_x;           /* batch [cap, ld_dst]; rows >= rows are zero-filled */
  int32_t* dst_y;         /* batch labels [cap]; rows >= rows get 0 */
  int32_t sample;         /* floats per sample */
  int32_t ld_dst;         /* row stride of dst_x in floats */
  int32_t cap;            /* batch capacity (the job's batch_size) */
  int32_t model;
} hnn_gather_problem;

int hnn_gather_rows(const hnn_gather_problem* probs, int nprob, int max_cap, const hnn_step_row* cur,
                    void* stream);

/* Host-side batch gather for the host-fed step (the same Batch(x=train_x[idx], y=train_y[idx]) as
 * store.py:77-80, done by the host data loader into pinned memory): for r < n,
 * dst_x[r*ld_dst .. + cols) = src_x[idx[r]*ld_src .. + cols) and dst_y[r] = (int32) src_y[idx[r]].
 * Plain host code (no CUDA calls); reentrant, so loader threads run it in parallel. */
int hnn_host_gather_rows(float* dst_x, int64_t ld_dst, int32_t* dst_y, const float* src_x, int64_t ld_src,
                         const float* src_y, const int64_t* idx, int64_t n, int64_t cols);

/* One step's host gather for every model at once (the loader's per-step call): item i gathers
 * rows idx[0..n) exactly as hnn_host_gather_rows and zeroes rows [n, cap) of its destination (a
 * short final batch, as the device gather writes).  The rows of all items are split evenly over
 * `threads` host threads (<= 64); the result does not depend on the thread count. */
typedef struct hnn_host_gather_item {
  float* dst_x;
  int32_t* dst_y;
  const float* src_x;
  const float* src_y;
  const int64_t* idx;
  int64_t ld_dst, ld_src, cols, n, cap;
} hnn_host_gather_item;

int hnn_host_gather_batch(const hnn_host_gather_item* items, int n_items, int threads);

/* The host-fed step (train.HostFedStepper) as one native call: on `copy_stream`, wait until staging
 * slot `slot` (0 / 1) is free (its previous batch moved out), H2D host_x / host_y (pinned) into it,
 * record the slot's ready event; on `compute_stream`, wait for it, copy the staged batch into the
 * arenas, record the slot's free event, launch `graph_exec` (the captured host-fed step graph, a
 * cudaGraphExec_t), then D2H out_dev[i] -> out_host[i] (per-model loss / correct).  *copied_event =
 * the ready event: once it completes the host buffers may be refilled (hnn_event_synchronize). */
typedef struct hnn_hostfed_io {
  const void* host_x;
  void* stage_x;
  void* arena_x;
  int64_t x_bytes;
  const void* host_y;
  void* stage_y;
  void* arena_y;
  int64_t y_bytes;
  const void* out_dev[2];
  void* out_host[2];
  int64_t out_bytes[2];
} hnn_hostfed_io;

int hnn_hostfed_create(void** ctx_out);
int hnn_hostfed_destroy(void* ctx);
int hnn_hostfed_step(void* ctx, int slot, const hnn_hostfed_io* io, void* graph_exec, void* compute_stream,
                     void* copy_stream, void** copied_event);
int hnn_event_synchronize(void* event);

/*
 * Row-major grouped GEMM problem.  Let R = cur[model].rows.
 *  FWD:   C[i,j] = sum_k A[i*lda+k] * B[j*ldb+k] + bias[j]; relu if `relu`;   i < m (= cap), rows >= R -> 0
 *  DGRAD: C[i,j] = sum_k A[i*lda+k] * B[k*ldb+j]; times (mask[i*ldc+j] > 0) if mask; rows >= R -> 0
 *  WGRAD: C[i,j] = sum_{r<R} A[r*lda+i] * B[r*ldb+j]; dbias[i] = sum_{r<R} A[r*lda+i] (row order)
 * tile_base / tiles_n are filled by the planner (tiles of the chosen kernel, see hnn_gemm_tiles).
 */
typedef struct hnn_gemm_problem {
  const float* a;
  const float* b;
  float* c;
  const float* bias;
  const float* mask;
  float* dbias;
  int32_t m, n, k;
  int32_t lda, ldb, ldc;
  int32_t model;
  int32_t relu;
  int32_t tile_base;
  int32_t tiles_n;
  const void* tmap_a; /* HNN_PREC_F32_3XTF32: device copies of the problem's TMA maps (hnn_gemm_tc_encode) */
  const void* tmap_b;
  const void* tmap_c;
  /* WGRAD optimizer fusion: when opt_w != NULL the epilogue applies the model's SGD / momentum
   * update (arithmetic of hnn_multi_tensor_*) to the weight with the tile's finished gradient,
   * and to the bias with dbias; c / dbias may then be NULL (gradient not stored).  The pair
   * kernels (HNN_PREC_*_PAIR) trap on a fused Adam problem: Adam runs in hnn_multi_tensor_adam. */
  float* opt_w;
  float* opt_wm;
  float* opt_wv;
  float* opt_b;
  float* opt_bm;
  float* opt_bv;
  int32_t opt_kind; /* HNN_OPT_* */
  float opt_momentum;
  /* Convolution lowering (HNN_PREC_F32_3XTF32_PAIR; 1 / 0 for dense layers):
   *   row_mult    GEMM rows (FWD/DGRAD M, WGRAD K) per batch sample (OH*OW for a conv): this
   *               step's valid rows are cur.rows * row_mult;
   *   c_mode      FWD output layout: 0 row-major [m, ldc]; 1 NCHW, element (m, n) at
   *               c[((m / row_mult) * n_total + n) * row_mult + m % row_mult], n_total = n; with
   *               c_mode 1 a non-NULL mask (same NCHW layout) multiplies by (mask > 0) and a NULL
   *               bias adds nothing (a conv input gradient computed as a forward conv of dy);
   *               2 + (ph * 2 + pw): NCHW into one parity class of a grid twice as large in each
   *               direction, element (m, n) with hw = m % row_mult = i * im_ow + j at
   *               c[((m / row_mult) * n_total + n) * 4 * row_mult + (2i + ph) * 2 * im_ow + 2j + pw]
   *               (a stride-2 conv's input gradient as four stride-1 convs of dy);
   *   ksplit      WGRAD fixed K split count (>= 1): split s covers K rows [s*ksplit_len,
   *               (s+1)*ksplit_len) and writes rows [s*mp, s*mp + m) of c, mp = m rounded up
   *               to 32 (the TMA map covers ksplit*mp rows); the splits are summed in order by
   *               hnn_conv_tc_aux(HNN_CONVTC_WGRAD_REDUCE). */
  int32_t row_mult;
  int32_t c_mode;
  int32_t ksplit;
  int32_t ksplit_len;
  /* HNN_PREC_F32_3XTF32_PAIR: tile columns 64, 128 or 256 (0 = 256); the K-major B TMA box is
   * tile_n / 2 rows (each CTA of the pair stages half of the tile's B columns). */
  int32_t tile_n;
  int32_t im_kw;  /* implicit convolution: taps per row (0 = im_k, i.e. square) */
  /* HNN_PREC_BF16_PAIR FWD, implicit convolution (im_c > 0): A is not a [m, k] matrix but NHWC
   * bf16 activations a[n][h][w][c] (im_n x im_h x im_w x im_c, c contiguous, im_c % 64 == 0); GEMM
   * row m = (b, oh, ow) of a stride-1 conv's im_oh x im_ow output (row_mult = im_oh * im_ow) and
   * K = (r, s, c) over the im_k x im_kw taps with padding im_pad (taps outside the image read as
   * zeros, by the TMA), so the B rows are in (r, s, c) order (HNN_CONVTC_PAD_WEIGHTS_RSC /
   * FLIP_WEIGHTS_RSC).  Each 128-row CTA tile must be whole output rows of whole or one image:
   * 128 % im_ow == 0 and (im_oh * im_ow) % 128 == 0 or 128 % (im_oh * im_ow) == 0.
   * WGRAD with im_c > 0: B (the weight-gradient GEMM's N = (r, s, c) x K = output pixels operand)
   * is read implicitly from the same NHWC activations as an MN-major operand, 64 pixels x 64
   * channels of one tap per CTA (tile_n must be 128; 64-pixel K blocks of whole rows / images);
   * A (dy, [f, pixels]) stays an ordinary K-major matrix. */
  int32_t im_c, im_k, im_pad, im_h, im_w, im_oh, im_ow, im_n;
  /* HNN_PREC_BF16_PAIR FWD with c_mode 1 (row_mult % 32 == 0): when xh_out != NULL the epilogue
   * also writes the output as NHWC bf16 rows [m, n] (after bias / relu; zero rows past the batch):
   * the next layer's implicit-GEMM input, so that layer needs no separate NHWC copy.  tmap_xh: its
   * TMA map (hnn_gemm_bf16_encode, the problem's fourth map). */
  void* xh_out;
  const void* tmap_xh;
} hnn_gemm_problem;

/* Tile edge (m, n) used by (op, prec); lets the host lay out tile_base / tiles_n. */
int hnn_gemm_tile_shape(int op, int prec, int32_t* tile_m, int32_t* tile_n);

/* K terms the tensor core sums into one TMEM chunk before the accumulator warps add the chunk into
 * their fp32 running sums (HNN_PREC_F32_3XTF32_PAIR).  A split-K forward must split K into ranges
 * of exactly this length to reproduce the unsplit promotion order bit for bit. */
int hnn_gemm_chunk_terms(int prec, int32_t* terms);

int hnn_grouped_gemm(int op, int prec, const hnn_gemm_problem* probs, int nprob, int total_tiles,
                     const hnn_step_row* cur, const hnn_model_status* status, void* stream);

/*
 * Host-side: encode the TMA tensor maps (A, B, C, and the bf16 path's NHWC copy X2; 128 bytes each)
 * of every problem for the tcgen05 path into host_maps[4*nprob]; the caller copies them to device
 * memory and stores their device addresses in tmap_a / tmap_b / tmap_c / tmap_xh.  Requirements:
 * 16-byte aligned bases and row strides.
 * Tiles are 128 x 128 (hnn_gemm_tile_shape); WGRAD problems need m <= 4096.
 */
int hnn_gemm_tc_encode(int op, const hnn_gemm_problem* host_probs, int nprob, void* host_maps);
/*
 * Split-K forward (HNN_PREC_F32_3XTF32_PAIR FWD problems with ksplit > 1 write raw partial sums
 * of K range [s*ksplit_len, ...) to rows s*mp + r of c, mp = m rounded up to 32; bias / relu 0):
 * y[r, j] = relu?(sum_s partial + bias[j]) for r < the step's rows, 0 beyond (_dense_fwd,
 * ops.py:46-48).  Table fields: a = partials (lda = partial row stride), c = y (ldc), bias, relu,
 * m, n, ksplit, model; tile_base / tiles_n = the problem's first block and block count.
 */
/* The logits layer's input and weight gradients in one pass over its input X (gemm_skinny.cu):
 * wgrad_probs[i] / dgrad_probs[i] are the HNN_WGRAD / HNN_DGRAD problems of the same dense layer
 * (tile_base / tiles_n in wgrad_probs: 128-column tiles), m <= 10 output units, no fused optimizer
 * (W is read by every tile).  Results equal hnn_grouped_gemm's two skinny launches bit for bit. */
int hnn_skinny_backward(const hnn_gemm_problem* wgrad_probs, const hnn_gemm_problem* dgrad_probs, int nprob,
                        int total_tiles, const hnn_step_row* cur, const hnn_model_status* status, void* stream);

int hnn_splitk_epilogue(const hnn_gemm_problem* probs, int nprob, int total_blocks, const hnn_step_row* cur,
                        const hnn_model_status* status, void* stream);
int hnn_gemm_bf16_encode(int op, const hnn_gemm_problem* host_probs, int nprob, void* host_maps);

/*
 * Implicit-GEMM convolution on NCHW, zero padding `pad`, square kernel k.
 *  FWD:   y = conv(x, w) + bias (relu if `relu`), rows >= R zero        GEMM M=cap*OH*OW, N=F, K=C*k*k
 *  DGRAD: dx = conv_transpose(dy, w), times (mask > 0) if mask          GEMM M=cap*H*W,   N=C, K=F*k*k
 *  WGRAD: partial[s] = sum over the s-th fixed chunk of (rows x OH x OW) of dy (x) im2col(x),
 *         column C*k*k of each partial holding the bias-gradient chunk; then hnn_conv_wgrad_reduce.
 */
typedef struct hnn_conv_problem {
  const float* x;
  const float* weight; /* [F, C, k, k] */
  const float* bias;
  float* y;
  const float* dy;
  float* dx;
  const float* mask;
  float* partial; /* WGRAD workspace [splits, F, C*k*k + 1] */
  float* dw;      /* [F, C, k, k] */
  float* db;      /* [F] */
  int32_t cap, c, h, w, f, k, stride, pad, oh, ow;
  int32_t model;
  int32_t relu;
  int32_t tile_base;
  int32_t tiles_n;
  int32_t splits;     /* WGRAD: number of fixed K chunks */
  int32_t split_len;  /* WGRAD: GEMM-K elements per chunk (multiple of OH*OW not required) */
  /* Direct path only, may be NULL (max-pools folded into a direct conv instead of their own launch):
   * DGRAD / WGRAD: the layer's output feeds a 2 x 2 / stride-2 max-pool (OH, OW even) whose backward
   *   is folded into this layer's dy staging: dy[b, f, oy, ox] = np_mask(0 + (pool_idx[w] == (oy&1)*2
   *   + (ox&1) ? pool_dy[w] : 0), pool_mask[b, f, oy, ox]) with w = (b, f, oy/2, ox/2) -- exactly
   *   hnn_grouped_maxpool's DGRAD (pool_mask NULL: no relu mask); `dy` is never written or read.
   * FWD: the layer's input x is the output of a 2 x 2 / stride-2 max-pool of pool_x [cap, C, 2H, 2W]
   *   computed while staging (hnn_grouped_maxpool's FWD arithmetic), which also writes the pool's
   *   outputs x (= pool_y) and pool_idx, zeros for rows past the batch. */
  const float* pool_dy;   /* DGRAD / WGRAD: [cap, F, OH/2, OW/2] */
  uint8_t* pool_idx;      /* [cap, F, OH/2, OW/2] (DGRAD / WGRAD, read) / [cap, C, H, W] (FWD, written) */
  const float* pool_mask; /* DGRAD / WGRAD: [cap, F, OH, OW] or NULL */
  const float* pool_x;    /* FWD: the pool's input [cap, C, 2H, 2W] */
} hnn_conv_problem;

int hnn_conv_tile_shape(int op, int32_t* tile_m, int32_t* tile_n);

int hnn_grouped_conv(int op, const hnn_conv_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                     const hnn_model_status* status, void* stream);

/*
 * Direct (non-GEMM) convolution for small layers (LeNet-class: one sample's activations and the
 * filters fit in shared memory; at most 16*256 weights): one CTA per sample (FWD, DGRAD) or per
 * chunk of HNN_CONV_DIRECT_BCHUNK samples (WGRAD partials, splits = ceil(cap / chunk), reduced by
 * hnn_conv_wgrad_reduce).  tile_base counts CTAs; `smem` = max over the launch's problems of
 * hnn_conv_direct_smem(op, ...).
 */
#define HNN_CONV_DIRECT_BCHUNK 1
int hnn_conv_direct_smem(int op, int c, int h, int w, int f, int k, int oh, int ow);
int hnn_grouped_conv_direct(int op, const hnn_conv_problem* probs, int nprob, int total_blocks, int smem,
                            const hnn_step_row* cur, const hnn_model_status* status, void* stream);
/* Threads per CTA the direct kernels want for a layer (128 when a stride-1 forward / input gradient
 * has at most 128 register-blocked work items per sample, else 256), and the launch taking it
 * (`threads` = max over the launch's problems; hnn_grouped_conv_direct launches 256). */
int hnn_conv_direct_threads(int op, int c, int h, int w, int f, int k, int oh, int ow);
/* hnn_grouped_conv_direct_ex op for a forward whose problems may carry pool_x (folded max-pools). */
#define HNN_CONV_DIRECT_FWD_POOLED 16
int hnn_grouped_conv_direct_ex(int op, const hnn_conv_problem* probs, int nprob, int total_blocks, int smem,
                               int threads, const hnn_step_row* cur, const hnn_model_status* status, void* stream);

/* dw[f,:] = sum_s partial[s,f,:C*k*k] and db[f] = sum_s partial[s,f,C*k*k] in split order. */
int hnn_conv_wgrad_reduce(const hnn_conv_problem* probs, int nprob, int total_blocks, const hnn_step_row* cur,
                          const hnn_model_status* status, void* stream);

typedef struct hnn_pool_problem {
  const float* x;
  float* y;
  uint8_t* idx;       /* argmax within each k*k window, first max wins (numpy argmax) */
  const float* dy;
  float* dx;
  const float* mask;  /* BWD: multiply by (mask > 0) (fused relu backward), may be NULL */
  int32_t cap, c, h, w, k, stride, oh, ow;
  int32_t model;
  int32_t block_base;
  int32_t blocks;
  /* HNN_POOL_ELEMENTWISE: one thread per output (FWD) / input element (DGRAD), 256 per block.
   * HNN_POOL_WINDOWS_2X2 (k = stride = 2, h and w even): one unit per 2 x 2 window for both ops,
   * HNN_POOL_WINDOWS_PER_BLOCK windows per block, row pairs moved as float2 */
  int32_t mode;
  /* FWD: when non-NULL, the output is also written as NHWC bf16 rows [cap * oh * ow, c] (zeros
   * past the batch): the next layer's implicit-GEMM input */
  void* xh;
} hnn_pool_problem;
#define HNN_POOL_ELEMENTWISE 0
#define HNN_POOL_WINDOWS_2X2 1
#ifndef HNN_POOL_WINDOWS_PER_BLOCK
#define HNN_POOL_WINDOWS_PER_BLOCK 1024
#endif

int hnn_grouped_maxpool(int op, const hnn_pool_problem* probs, int nprob, int total_blocks,
                        const hnn_step_row* cur, const hnn_model_status* status, void* stream);

typedef struct hnn_relu_problem {
  const float* x; /* relu input */
  float* y;
  const float* dy;
  float* dx;
  int32_t cap, row; /* row = floats per sample */
  int32_t model;
  int32_t block_base;
  int32_t blocks;
  int32_t reserved;
} hnn_relu_problem;

int hnn_grouped_relu(int op, const hnn_relu_problem* probs, int nprob, int total_blocks, const hnn_step_row* cur,
                     const hnn_model_status* status, void* stream);

typedef struct hnn_sce_problem {
  const float* logits; /* [cap, ld] */
  const int32_t* labels;
  float* dlogits;      /* [cap, ld]; NULL for evaluation */
  int32_t ld;
  int32_t classes;
  int32_t cap;
  int32_t model;
} hnn_sce_problem;

/*
 * One block per problem (max_cap / max_classes size its shared memory).  train != 0: non-finite loss -> status.alive = 0 and abort_epoch/batch
 * recorded, nothing accumulated; otherwise loss_sum += F64(loss)*R, correct_sum, seen updated.
 * train == 0 (evaluation): always accumulates (train.py:274-276), never aborts.
 * loss_out[model] / correct_out[model] receive the step's loss and hit count when not NULL.
 */
int hnn_sce_fused(const hnn_sce_problem* probs, int nprob, int max_cap, int max_classes, const hnn_step_row* cur,
                  hnn_model_status* status, int train, float* loss_out, int32_t* correct_out, void* stream);

/* The fused logits tail of a small model (tail.cu, one CTA per model): the last dense layer's
 * forward y = x W^T + b (W [classes, k], classes <= 16), softmax-CE + accuracy + abort exactly as
 * hnn_sce_fused (train mode), then — unless the loss is non-finite — dx = (dlogits W) * (mask > 0)
 * (rows >= R zero), dW = dlogits^T x and db (numpy axis-0 order) into dw / db and / or the fused
 * SGD / momentum update of opt_w / opt_b (opt_kind, opt_momentum; never Adam).  x rows 16-byte
 * aligned (ldx % 4 == 0, k % 4 == 0); `smem` = max over problems of hnn_tail_smem(cap, k, classes). */
typedef struct hnn_tail_problem {
  const float* x;
  const float* w;
  const float* b;
  float* logits;      /* [cap, ld_logits] (optional) */
  const int32_t* labels;
  float* dx;          /* [cap, ld_dx] (NULL: no input gradient) */
  const float* mask;  /* relu mask source (x itself or NULL) */
  float* dw;
  float* db;
  float* opt_w;
  float* opt_wm;
  float* opt_b;
  float* opt_bm;
  int32_t ldx, ld_logits, ld_dx, cap, k, classes, model, opt_kind;
  float opt_momentum;
  int32_t reserved;
} hnn_tail_problem;

int hnn_tail_smem(int cap, int k, int classes);
int hnn_logits_tail(const hnn_tail_problem* probs, int nprob, int smem, const hnn_step_row* cur,
                    hnn_model_status* status, float* loss_out, int32_t* correct_out, void* stream);

typedef struct hnn_opt_segment {
  float* param;
  const float* grad;
  float* m;           /* Adam first moment / SGD velocity */
  float* v;           /* Adam second moment */
  int64_t count;      /* floats in the segment (param/grad/m/v are 16-byte aligned) */
  int32_t model;
  int32_t kind;       /* HNN_OPT_* */
  float momentum;
  int32_t chunk_base; /* first 4096-float chunk of this segment in the launch */
  int32_t chunks;
  int32_t reserved;
} hnn_opt_segment;

int hnn_multi_tensor_sgd(const hnn_opt_segment* segs, int nseg, int total_chunks, const hnn_step_row* cur,
                         const hnn_model_status* status, void* stream);
int hnn_multi_tensor_adam(const hnn_opt_segment* segs, int nseg, int total_chunks, const hnn_step_row* cur,
                          const hnn_model_status* status, void* stream);

/*
 * Tensor-core convolution path (conv_tc.cu): a conv2d layer lowered onto the CTA-pair GEMM
 * (HNN_PREC_F32_3XTF32_PAIR) with explicit im2col buffers; NCHW activations.  Replaces the same
 * reference functions as hnn_grouped_conv (ops.py:91-130) for layers with C*k*k, F >= 64.
 *   HNN_CONVTC_IM2COL        cols[m, kk] = x[b, c, oh*s-p+r, ow*s-p+s'], m = (b, oh, ow), kk = (c, r, s');
 *                            rows are kkp wide (pad columns zero)
 *   HNN_CONVTC_TRANSPOSE_DY  dyt[m, f] = dy[b, f, oh, ow] (rows padded to 16 bytes); bpart[b, t, f] = sum of dy[b, f, hw]
 *                            over pixel tile t (32 pixels) when bpart != NULL.  Also the NCHW -> NHWC bf16
 *                            copy of a conv input for the implicit GEMM (dy = x, f = c, oh/ow = h/w).
 *   im2col in bf16 mode skips cols when cols == NULL (only colst, the weight-gradient operand), and
 *   for a "same" stride-1 layer with dyt != NULL also writes the NHWC bf16 copy of x to dyt.
 *   HNN_CONVTC_COL2IM        dx[b, c, h, w] = (mask > 0) * sum_(r, s') dcols[m, kk] (gather, tap order)
 *   HNN_CONVTC_WGRAD_REDUCE  dw[f, kk] = sum_s partial[s][f][kk] (splits in order); db[f] = sum over (b, t) of bpart[b, t, f]
 * Each problem covers `blocks` CTAs starting at block_base: im2col one per (32 output pixels, 32
 * channels), transpose one per (sample, 32 pixels, 32 filters), col2im one per (sample, input row,
 * 32 columns, 16 channels), reduce any count (grid-stride).  max_k = largest kernel size (<= 5;
 * col2im <= 3).
 */
#define HNN_CONVTC_IM2COL 0
#define HNN_CONVTC_TRANSPOSE_DY 1
/* HNN_CONVTC_TRANSPOSE_DY blocks: ceil(cap * ceil(oh*ow / 32) / HNN_CONVTC_TRANSPOSE_HW_TILES) * ceil(f / 32)
 * (one block = 32 channels x HNN_CONVTC_TRANSPOSE_HW_TILES consecutive (sample, 32-pixel run) units) */
#define HNN_CONVTC_TRANSPOSE_HW_TILES 4
#define HNN_CONVTC_COL2IM 2
#define HNN_CONVTC_WGRAD_REDUCE 3
#define HNN_CONVTC_PAD_WEIGHTS 4  /* wpad[f, kk'] = w[f, kk] (kk' < kkp, zero pad): when C*k*k % 4 != 0 */
#define HNN_CONVTC_WT_WEIGHTS 6   /* bf16 wpad[kk, f] = w[f, kk] */
#define HNN_CONVTC_FLIP_WEIGHTS 5 /* wpad[c, (f, r, s)] = w[f, c, k-1-r, k-1-s]: stride-1 input gradient as a
                                     forward conv of dy (im2col of dy with pad k-1-pad, then a GEMM) */
#define HNN_CONVTC_PAD_WEIGHTS_RSC 7  /* bf16 wpad[f, (r, s, c)] = w[f, c, r, s]: implicit-GEMM forward B */
#define HNN_CONVTC_FLIP_WEIGHTS_RSC 8 /* bf16 wpad[c, (r, s, f)] = w[f, c, k-1-r, k-1-s]: implicit-GEMM input
                                         gradient (forward conv of NHWC dy) B */
#define HNN_CONVTC_PARITY_WEIGHTS 9   /* 3x3 / stride 2 / pad 1 input gradient as four stride-1 convs of dy:
                                         class q = ksplit (ph = q >> 1, pw = q & 1), taps rr < 1 + ph,
                                         ss < 1 + pw: bf16 wpad[c, (rr, ss, f)] = w[f, c, ph+1-2rr, pw+1-2ss] */
#define HNN_CONVTC_SPLITK_FWD 10      /* finish a K-split forward-type conv GEMM (bf16 layers whose output tiles
                                         fill few CTA pairs): for m = (b, hw) < cap*oh*ow, n < f:
                                         v = sum_s partial[s*pix_ld + m][n] (splits in order) + db[n],
                                         relu if rsc; dx[b, n, hw] = v, times (mask[b, n, hw] > 0) if mask;
                                         rows past the step's batch are 0; dyt (bf16 [m, f]) = v if dyt.
                                         One CTA per 32 pixels x 32 columns. */

typedef struct hnn_convtc_problem {
  const float* x;    /* [cap, c, h, w] */
  float* cols;       /* [cap*oh*ow, kk] */
  const float* dy;   /* [cap, f, oh, ow] */
  float* dyt;        /* [cap*oh*ow, f] */
  const float* dcols;/* [cap*oh*ow, kk] */
  float* dx;         /* [cap, c, h, w] */
  const float* mask; /* [cap, c, h, w] or NULL */
  const float* partial; /* [ksplit, round_up(f, 32), kkp] */
  float* dw;         /* [f, kk] */
  float* db;         /* [f] */
  float* bpart;      /* [cap, ceil(oh*ow/32), f] */
  const float* weight; /* [f, kk] (HNN_CONVTC_PAD_WEIGHTS) */
  float* wpad;       /* [f, kkp] */
  int32_t cap, c, h, w, f, k, stride, pad, oh, ow, kk;
  int32_t kkp;       /* cols / partial / wpad row length: kk rounded up to a multiple of 4 */
  int32_t ksplit, ksplit_len;
  int32_t model, block_base, blocks;
  /* bf16 mode (HNN_PREC_BF16_PAIR GEMMs): cols, dyt, wpad hold bf16; im2col also writes colst
   * [kkp, pix_ld] and the transpose dyk [f, pix_ld] (pixel-contiguous K-major weight-gradient
   * operands); HNN_CONVTC_WT_WEIGHTS writes wpad = w^T [kkp, f] (stride-2 dcols GEMM operand). */
  void* colst;
  void* dyk;
  int32_t bf16;
  int32_t pix_ld;
  /* HNN_CONVTC_WGRAD_REDUCE: the partial columns are in (r, s, c) order (implicit-GEMM weight
   * gradient); dw is still written in the reference [f, c, r, s] layout */
  int32_t rsc;
  int32_t reserved;
} hnn_convtc_problem;

int hnn_conv_tc_aux(int op, const hnn_convtc_problem* probs, int nprob, int total_blocks, int max_k,
                    const hnn_step_row* cur, const hnn_model_status* status, void* stream);

/*
 * Grouped embedding-lookup (ops.py:258-278; embed.cu).  op HNN_FWD: y[b, l, :] = table[x[b, l], :]
 * (rows past the batch zeroed), one warp per (b, l) row, blocks = ceil(cap * len / 8);
 * op HNN_WGRAD: dtable[v, :] = sum over positions with x == v, in ascending position order, of
 * dy[p, :] (np.add.at's order; no atomics), one warp per table row, blocks = ceil(vocab / 8).
 * Token ids are float32 sample values, validated by the host (integral, in [0, vocab)).
 */
typedef struct hnn_embed_problem {
  const float* x;     /* [cap, ldx] token ids */
  const float* table; /* [vocab, dim] */
  float* y;           /* [cap, len * dim] */
  const float* dy;    /* [cap, len * dim] */
  float* dtable;      /* [vocab, dim] */
  int32_t cap, len, ldx, dim, vocab;
  int32_t model, block_base, blocks;
} hnn_embed_problem;

int hnn_embedding(int op, const hnn_embed_problem* probs, int nprob, int total_blocks, const hnn_step_row* cur,
                  const hnn_model_status* status, void* stream);

/* Self-test of the optimizer's exact float32 arithmetic (no reference counterpart): for i < n,
 * q[i] = a[i] / b[i] and r[i] = sqrt(a[i]) with the same round-to-nearest-even routines the
 * Adam update uses (optim.py:84-87: m / bias1, v / bias2, np.sqrt, the final quotient). */
int hnn_selftest_div_sqrt(const float* a, const float* b, float* q, float* r, int64_t n, void* stream);

/* Sizes of the ABI structs, so bindings can assert their layouts. */
int hnn_struct_size(const char* name);

const char* hnn_last_error(void);
const char* hnn_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HNN_B200_H */
