// Dense-layer GEMMs with one tiny dimension (<= 16): the 10-class logits layer of every model
// (pkg/src/hybridnn/ops.py:46-55).  They move far more bytes than they compute, so each is a
// vectorised, coalesced streaming kernel instead of a tiled GEMM (a 64x64 or 128x16 tile
// wastes most of its lanes on a 10-wide edge):
//   FWD   y[B, n<=16]  = x[B, K] W[n, K]^T + b   one warp per 4 rows, lanes stride K by float4,
//                                                 W rows loaded once per k-step for all 4 rows
//   DGRAD dx[B, N]     = dy[B, k<=16] W[k, N]    one float4 column quad per thread, 4 rows,
//                      (* (x > 0) relu mask)       W quads held in registers across the rows
//   WGRAD dW[m<=16, N] = dy[R, m]^T x[R, N]      one float4 column quad per thread over a fixed
//                                                 quarter of the rows, quarters reduced in order;
//                                                 bias gradient and the fused optimizer included
// Tiling is a fixed function of each problem's shape (bit-exact isolation); no atomics.
#include <cstdlib>

#include "common.cuh"

namespace hnn {

constexpr int KTHREADS = 256;
#ifndef HNN_SKINNY_FWD_ROWS
#define HNN_SKINNY_FWD_ROWS 2
#endif
constexpr int FWD_ROWS = HNN_SKINNY_FWD_ROWS;  // rows per warp; tile = 8 warps x 2 rows = 16 rows
#ifndef HNN_SKINNY_DG_ROWS
#define HNN_SKINNY_DG_ROWS 8
#endif
constexpr int DG_ROWS = HNN_SKINNY_DG_ROWS;  // DGRAD rows per thread; tile = 8 row groups x 8 rows x 128 columns
constexpr int WG_QUADS = 32; // WGRAD column quads per CTA; tile = 128 columns, 8 row groups
#ifndef HNN_SKBWD_UNROLL
#define HNN_SKBWD_UNROLL 4
#endif
#ifndef HNN_SKBWD_WSMEM
#define HNN_SKBWD_WSMEM 0
#endif
constexpr int SKBWD_UNROLL = HNN_SKBWD_UNROLL;

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

__device__ __forceinline__ float dot4(float4 a, float4 b, float acc) {
  return fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, acc))));
}

// ------------------------------------------------------------------------------------------ FWD
template <int NJ>
__device__ __forceinline__ void rowdot_rows(const hnn_gemm_problem& p, int r0, int rows, int lane) {
  float acc[FWD_ROWS][NJ];
#pragma unroll
  for (int i = 0; i < FWD_ROWS; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j] = 0.0f;
  const float* x[FWD_ROWS];
#pragma unroll
  for (int i = 0; i < FWD_ROWS; ++i) x[i] = p.a + size_t(min(r0 + i, max(rows - 1, 0))) * p.lda;
  const float* w[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) w[j] = p.b + size_t(min(j, p.n - 1)) * p.ldb;  // clamped: no branch
  const bool vec = ((p.lda & 3) == 0) && ((p.ldb & 3) == 0) && ((reinterpret_cast<uintptr_t>(p.a) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(p.b) & 15) == 0);
  int k = 0;
  if (vec) {
    for (; k + 128 <= p.k; k += 128) {
      const int kk = k + lane * 4;
      float4 u[FWD_ROWS], v[NJ];
#pragma unroll
      for (int i = 0; i < FWD_ROWS; ++i) u[i] = ldg4(x[i] + kk);
#pragma unroll
      for (int j = 0; j < NJ; ++j) v[j] = ldg4(w[j] + kk);
#pragma unroll
      for (int i = 0; i < FWD_ROWS; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j] = dot4(u[i], v[j], acc[i][j]);
    }
  }
  for (int kk = k + lane; kk < p.k; kk += 32) {
    float u[FWD_ROWS];
#pragma unroll
    for (int i = 0; i < FWD_ROWS; ++i) u[i] = __ldg(x[i] + kk);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const float v = __ldg(w[j] + kk);
#pragma unroll
      for (int i = 0; i < FWD_ROWS; ++i) acc[i][j] = fmaf(u[i], v, acc[i][j]);
    }
  }
  // fixed xor-shuffle tree per dot product (deterministic)
#pragma unroll
  for (int i = 0; i < FWD_ROWS; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[i][j] += __shfl_xor_sync(0xffffffffu, acc[i][j], o);
  if (lane < p.n) {
    const float b = __ldg(p.bias + lane);
#pragma unroll
    for (int i = 0; i < FWD_ROWS; ++i) {
      const int r = r0 + i;
      if (r >= p.m) break;
      float y = 0.0f;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (j == lane) y = acc[i][j];
      if (r < rows) {
        y = __fadd_rn(y, b);
        if (p.relu) y = np_relu(y);
      } else {
        y = 0.0f;  // rows past this step's batch are exact zeros
      }
      p.c[size_t(r) * p.ldc + lane] = y;
    }
  }
}

__global__ void __launch_bounds__(KTHREADS) skinny_fwd_kernel(const hnn_gemm_problem* __restrict__ probs, int nprob,
                                                              const hnn_step_row* __restrict__ cur,
                                                              const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_gemm_problem& q) { return q.tile_base; });
  const hnn_gemm_problem& p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r0 = (blockIdx.x - p.tile_base) * (8 * FWD_ROWS) + warp * FWD_ROWS;
  if (r0 >= p.m) return;
  // CTA-uniform dispatch on the column count: loads and FMAs carry no per-column branches
  if (p.n <= 4) rowdot_rows<4>(p, r0, rows, lane);
  else if (p.n <= 8) rowdot_rows<8>(p, r0, rows, lane);
  else if (p.n <= 10) rowdot_rows<10>(p, r0, rows, lane);
  else if (p.n <= 12) rowdot_rows<12>(p, r0, rows, lane);
  else rowdot_rows<16>(p, r0, rows, lane);
}

// FWD, bulk-copy form (problems with 16-byte rows and K % 128 == 0: the C1 / C3 / C5 logits
// layers): the same 16-row tile, its x rows and the n <= 16 W rows streamed through a 4-stage
// shared-memory ring in 128-float K chunks by a producer warp (cp.async.bulk, one row per lane), 8
// update warps = 2 rows each x 32 K-slices (float4 each), slices combined by a fixed xor tree.  The
// per-warp streaming form walked each row's whole K as a chain of dependent L2 / HBM round trips
// at 24 warps per SM (C3: 39 us for 35.6 MB, ncu long-scoreboard bound).  Other problems take the
// per-warp form inside the same launch (the tile shape is shared).
#ifndef HNN_FB_KC
#define HNN_FB_KC 128
#endif
#ifndef HNN_FB_STAGES
#define HNN_FB_STAGES 4
#endif
constexpr int FB_KC = HNN_FB_KC, FB_STAGES = HNN_FB_STAGES, FB_THREADS = KTHREADS + 32;
constexpr int FB_STAGE_BYTES = 2 * 16 * FB_KC * 4;  // 16 x rows + 16 W rows
constexpr int FB_SMEM = FB_STAGES * FB_STAGE_BYTES + 256;
static_assert(FB_KC % 128 == 0 && 8 * FWD_ROWS == 16, "lane = float4 slice of each 128-wide K block; 16-row tiles");

__device__ __forceinline__ bool fwd_bulk_ok(const hnn_gemm_problem& p) {
  return p.n <= 16 && (p.k % FB_KC) == 0 && (p.lda & 3) == 0 && (p.ldb & 3) == 0 &&
         (reinterpret_cast<uintptr_t>(p.a) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.b) & 15) == 0;
}

template <int NJ>
__device__ __forceinline__ void fwd_bulk_tile(const hnn_gemm_problem& p, int r0, int rows, uint8_t* smem) {
  const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FB_STAGES * FB_STAGE_BYTES);
  auto bar = [&](int i) { return static_cast<uint32_t>(__cvta_generic_to_shared(bars + i)); };
  auto wait = [&](uint32_t b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "FB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra FB_WAIT_%=;\n\t}" ::"r"(b),
        "r"(parity)
        : "memory");
  };
  const int nchunks = p.k / FB_KC;
  const int xrows = min(16, p.m - r0);  // rows of this tile inside the buffer (cap)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == KTHREADS / 32) {
    // ---------------- producer warp: lanes 0..15 copy x rows, lanes 16..31 W rows
    const uint32_t bytes = uint32_t(xrows + p.n) * FB_KC * 4;
    for (int c = 0; c < nchunks; ++c) {
      const int st = c % FB_STAGES;
      if (c >= FB_STAGES) wait(bar(FB_STAGES + st), ((c / FB_STAGES) - 1) & 1);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar(st)), "r"(bytes) : "memory");
      __syncwarp();
      const uint32_t dst = ring + st * FB_STAGE_BYTES;
      const float* src = nullptr;
      uint32_t d = 0;
      if (lane < 16 && lane < xrows) {
        src = p.a + size_t(r0 + lane) * p.lda + c * FB_KC;
        d = dst + lane * FB_KC * 4;
      } else if (lane >= 16 && lane - 16 < p.n) {
        src = p.b + size_t(lane - 16) * p.ldb + c * FB_KC;
        d = dst + (16 + lane - 16) * FB_KC * 4;
      }
      if (src)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                     "l"(src), "r"(FB_KC * 4), "r"(bar(st))
                     : "memory");
    }
    return;
  }
  // ---------------- 8 warps x FWD_ROWS rows, lane = K-slice: lane l holds float4 l of every 128
  // K-wide block, exactly the per-warp form's assignment (rowdot_rows), so both forms add every dot
  // product in the same order (and the same 32-lane xor tree); each W float4 read from shared
  // memory serves the warp's FWD_ROWS rows (16 K-slices x 16 rows re-read the W rows once per row:
  // shared-memory bound, 31 us on C3)
  float acc[FWD_ROWS][NJ];
#pragma unroll
  for (int i = 0; i < FWD_ROWS; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j] = 0.0f;
  for (int c = 0; c < nchunks; ++c) {
    const int st = c % FB_STAGES;
    wait(bar(st), (c / FB_STAGES) & 1);
    const float* xs = reinterpret_cast<const float*>(smem + st * FB_STAGE_BYTES) + warp * FWD_ROWS * FB_KC;
    const float* ws = reinterpret_cast<const float*>(smem + st * FB_STAGE_BYTES) + 16 * FB_KC;
#pragma unroll
    for (int h = 0; h < FB_KC / 128; ++h) {
      const int k = (lane + 32 * h) * 4;
      float4 u[FWD_ROWS];
#pragma unroll
      for (int i = 0; i < FWD_ROWS; ++i) u[i] = *reinterpret_cast<const float4*>(xs + i * FB_KC + k);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const float4 w = *reinterpret_cast<const float4*>(ws + j * FB_KC + k);
#pragma unroll
        for (int i = 0; i < FWD_ROWS; ++i) acc[i][j] = dot4(u[i], w, acc[i][j]);
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(KTHREADS) : "memory");  // every warp has read stage st
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar(FB_STAGES + st)) : "memory");
  }
#pragma unroll
  for (int i = 0; i < FWD_ROWS; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[i][j] += __shfl_xor_sync(0xffffffffu, acc[i][j], o);
  if (lane >= p.n) return;
  const float b = __ldg(p.bias + lane);
#pragma unroll
  for (int i = 0; i < FWD_ROWS; ++i) {
    const int row = r0 + warp * FWD_ROWS + i;
    if (row >= p.m) break;
    float v = 0.0f;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
      if (j == lane) v = acc[i][j];
    float y = 0.0f;
    if (row < rows) {
      y = __fadd_rn(v, b);
      if (p.relu) y = np_relu(y);
    }
    p.c[size_t(row) * p.ldc + lane] = y;
  }
}

__global__ void __launch_bounds__(FB_THREADS) skinny_fwd_bulk_kernel(const hnn_gemm_problem* __restrict__ probs,
                                                                     int nprob, const hnn_step_row* __restrict__ cur,
                                                                     const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  extern __shared__ __align__(128) uint8_t fb_smem[];
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_gemm_problem& q) { return q.tile_base; });
  const hnn_gemm_problem& p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t0 = (blockIdx.x - p.tile_base) * (8 * FWD_ROWS);
  if (t0 >= p.m) return;
  if (fwd_bulk_ok(p)) {
    if (threadIdx.x == 0) {
      uint64_t* bars = reinterpret_cast<uint64_t*>(fb_smem + FB_STAGES * FB_STAGE_BYTES);
      for (int i = 0; i < 2 * FB_STAGES; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bars + i))));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (p.n <= 4) fwd_bulk_tile<4>(p, t0, rows, fb_smem);
    else if (p.n <= 8) fwd_bulk_tile<8>(p, t0, rows, fb_smem);
    else if (p.n <= 10) fwd_bulk_tile<10>(p, t0, rows, fb_smem);
    else if (p.n <= 12) fwd_bulk_tile<12>(p, t0, rows, fb_smem);
    else fwd_bulk_tile<16>(p, t0, rows, fb_smem);
    return;
  }
  if (warp >= KTHREADS / 32) return;  // (the per-warp form: 8 warps x FWD_ROWS rows)
  const int r0 = t0 + warp * FWD_ROWS;
  if (r0 >= p.m) return;
  if (p.n <= 4) rowdot_rows<4>(p, r0, rows, lane);
  else if (p.n <= 8) rowdot_rows<8>(p, r0, rows, lane);
  else if (p.n <= 10) rowdot_rows<10>(p, r0, rows, lane);
  else if (p.n <= 12) rowdot_rows<12>(p, r0, rows, lane);
  else rowdot_rows<16>(p, r0, rows, lane);
}

// ---------------------------------------------------------------------------------------- DGRAD
template <int KJ>
__device__ __forceinline__ void outer_rows(const hnn_gemm_problem& p, int r0, int col, int rows, const float* dys) {
  float4 w[KJ];
#pragma unroll
  for (int j = 0; j < KJ; ++j) w[j] = j < p.k ? ldg4(p.b + size_t(j) * p.ldb + col) : make_float4(0, 0, 0, 0);
  // the relu-mask quads of MK rows are requested together (one round trip per MK rows); four for
  // the 16-row W, whose quads already hold 64 registers
  constexpr int MK = KJ > 12 ? 4 : DG_ROWS;
#pragma unroll
  for (int h = 0; h < DG_ROWS; h += MK) {
    float4 mk[MK];
#pragma unroll
    for (int i = 0; i < MK; ++i) {
      const int r = r0 + h + i;
      mk[i] = (p.mask && r < rows && r < p.m) ? ldg4(p.mask + size_t(r) * p.ldc + col) : make_float4(1, 1, 1, 1);
    }
#pragma unroll
    for (int i = 0; i < MK; ++i) {
      const int r = r0 + h + i;
      if (r >= p.m) break;
      float4 o = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (r < rows) {
        const float* dy = dys + (threadIdx.x >> 5) * DG_ROWS * 16 + (h + i) * 16;  // staged dy row (shared)
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
          const float d = dy[j];
          o.x = fmaf(d, w[j].x, o.x);
          o.y = fmaf(d, w[j].y, o.y);
          o.z = fmaf(d, w[j].z, o.z);
          o.w = fmaf(d, w[j].w, o.w);
        }
        if (p.mask) {
          o.x = np_mask(o.x, mk[i].x);
          o.y = np_mask(o.y, mk[i].y);
          o.z = np_mask(o.z, mk[i].z);
          o.w = np_mask(o.w, mk[i].w);
        }
      }
      *reinterpret_cast<float4*>(p.c + size_t(r) * p.ldc + col) = o;
    }
  }
}

__global__ void __launch_bounds__(KTHREADS) skinny_dgrad_kernel(const hnn_gemm_problem* __restrict__ probs, int nprob,
                                                                const hnn_step_row* __restrict__ cur,
                                                                const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  __shared__ float dys[8 * DG_ROWS * 16];  // the CTA's 64 dy rows, 16 columns (zero padded)
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_gemm_problem& q) { return q.tile_base; });
  const hnn_gemm_problem& p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int t = blockIdx.x - p.tile_base;
  const int m0 = (t / p.tiles_n) * (8 * DG_ROWS), n0 = (t % p.tiles_n) * 128;
  {  // the CTA's dy rows: every thread's loads issued before its shared-memory stores
    constexpr int PER = 8 * DG_ROWS * 16 / KTHREADS;
    float v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + u * KTHREADS, r = m0 + e / 16, j = e % 16;
      v[u] = (j < p.k && r < rows && r < p.m) ? __ldg(p.a + size_t(r) * p.lda + j) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) dys[threadIdx.x + u * KTHREADS] = v[u];
  }
  __syncthreads();
  const int col = n0 + (threadIdx.x & 31) * 4, r0 = m0 + (threadIdx.x >> 5) * DG_ROWS;
  if (col >= p.n || r0 >= p.m) return;  // n is a multiple of 4 (host routing)
  if (p.k <= 4) outer_rows<4>(p, r0, col, rows, dys);
  else if (p.k <= 8) outer_rows<8>(p, r0, col, rows, dys);
  else if (p.k <= 10) outer_rows<10>(p, r0, col, rows, dys);
  else if (p.k <= 12) outer_rows<12>(p, r0, col, rows, dys);
  else outer_rows<16>(p, r0, col, rows, dys);
}

// ---------------------------------------------------------------------------------------- WGRAD
// CTA = WG_QUADS column quads x WG_GROUPS row groups (256 threads); each thread accumulates its
// quad over its group's rows (8 x rows in flight), the groups are summed in fixed order through
// shared memory.  128-column tiles and 8 groups (272 CTAs on C3, 3 per SM) instead of 256 columns
// x 4 groups (144 CTAs at one per SM: ncu 10% occupancy, L1TEX-latency bound).
constexpr int WG_CHUNK = 256;  // dy rows staged in shared memory per pass ([256][16] floats)
constexpr int WG_GROUPS = KTHREADS / WG_QUADS;

// dy rows [base, base + n) x 16 columns (zero padded) into shared memory: every thread's 16 loads
// are issued before its stores (a load -> store per element serialised 16 round trips per thread:
// most of the tiny-batch weight-gradient launches' time)
__device__ __forceinline__ void stage_dy(const hnn_gemm_problem& p, int base, int n, float* dys) {
  constexpr int PER = WG_CHUNK * 16 / KTHREADS;
  float v[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = threadIdx.x + u * KTHREADS, r = e >> 4, j = e & 15;
    v[u] = (j < p.m && r < n) ? __ldg(p.a + size_t(base + r) * p.lda + j) : 0.0f;
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) dys[threadIdx.x + u * KTHREADS] = v[u];
}

// numpy's axis-0 sum of column j of the staged dy rows: sequential in row order, eight rows' shared
// loads issued ahead of their dependent adds
__device__ __forceinline__ float colsum_rows(const float* dys, int n, int j, float acc) {
  int r = 0;
  for (; r + 8 <= n; r += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = dys[(r + u) * 16 + j];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, v[u]);
  }
  for (; r < n; ++r) acc = __fadd_rn(acc, dys[r * 16 + j]);
  return acc;
}

template <int MJ>
__device__ __forceinline__ void colacc(const hnn_gemm_problem& p, int col, int r_lo, int r_hi, int base,
                                       float (&part)[MJ][4], const float* dys) {
  const float* x = p.b + col;
#pragma unroll 8  // (eight rows of x in flight per thread)
  for (int r = r_lo; r < r_hi; ++r) {
    const float4 xv = ldg4(x + size_t(r) * p.ldb);
    const float* d = dys + (r - base) * 16;
#pragma unroll
    for (int j = 0; j < MJ; ++j) {
      part[j][0] = fmaf(d[j], xv.x, part[j][0]);
      part[j][1] = fmaf(d[j], xv.y, part[j][1]);
      part[j][2] = fmaf(d[j], xv.z, part[j][2]);
      part[j][3] = fmaf(d[j], xv.w, part[j][3]);
    }
  }
}

template <int MJ>
__device__ __forceinline__ void wgrad_tile(const hnn_gemm_problem& p, const hnn_step_row& row, int col, bool active,
                                           int q, int qd, float* dys, float* red, bool bias_thread) {
  const int rows = row.rows;
  float part[MJ][4];
#pragma unroll
  for (int j = 0; j < MJ; ++j) part[j][0] = part[j][1] = part[j][2] = part[j][3] = 0.0f;
  float bsum = -0.0f;
  // fixed decomposition: 256-row chunks in order; inside a chunk, row group q of each thread
  for (int base = 0; base < rows; base += WG_CHUNK) {
    const int n = min(WG_CHUNK, rows - base);
    __syncthreads();
    stage_dy(p, base, n, dys);
    __syncthreads();
    if (bias_thread) bsum = colsum_rows(dys, n, threadIdx.x, bsum);  // numpy's axis-0 order
    if (active) colacc<MJ>(p, col, base + (n * q) / WG_GROUPS, base + (n * (q + 1)) / WG_GROUPS, base, part, dys);
  }
  if (bias_thread) {
    if (p.dbias) p.dbias[threadIdx.x] = bsum;
    if (p.opt_b) {
      const Update u = make_update(row, p.opt_kind, p.opt_momentum);
      const int i = threadIdx.x;
      float w = p.opt_b[i], m = p.opt_bm ? p.opt_bm[i] : 0.0f, v = p.opt_bv ? p.opt_bv[i] : 0.0f;
      update_sgd(u, w, bsum, m);
      p.opt_b[i] = w;
      if (p.opt_bm) p.opt_bm[i] = m;
      if (p.opt_bv) p.opt_bv[i] = v;
    }
  }
  if (q > 0) {
    float* dst = red + (size_t(q - 1) * WG_QUADS + qd) * 64;
#pragma unroll
    for (int j = 0; j < MJ; ++j)
      *reinterpret_cast<float4*>(dst + j * 4) = make_float4(part[j][0], part[j][1], part[j][2], part[j][3]);
  }
  __syncthreads();
  if (q != 0 || !active) return;
  // row groups summed in fixed order 0 + 1 + ... + WG_GROUPS-1
  for (int g = 0; g < WG_GROUPS - 1; ++g) {
    const float* src = red + (size_t(g) * WG_QUADS + qd) * 64;
#pragma unroll
    for (int j = 0; j < MJ; ++j) {
      const float4 v = *reinterpret_cast<const float4*>(src + j * 4);
      part[j][0] += v.x;
      part[j][1] += v.y;
      part[j][2] += v.z;
      part[j][3] += v.w;
    }
  }
  const Update u = make_update(row, p.opt_kind, p.opt_momentum);
#pragma unroll
  for (int j = 0; j < MJ; ++j) {
    if (j >= p.m) break;
    const size_t off = size_t(j) * p.ldc + col;
    if (p.c) *reinterpret_cast<float4*>(p.c + off) = make_float4(part[j][0], part[j][1], part[j][2], part[j][3]);
    if (p.opt_w) {
      float4 w = *reinterpret_cast<float4*>(p.opt_w + off);
      float4 m = p.opt_wm ? *reinterpret_cast<float4*>(p.opt_wm + off) : make_float4(0, 0, 0, 0);
      float4 v = p.opt_wv ? *reinterpret_cast<float4*>(p.opt_wv + off) : make_float4(0, 0, 0, 0);
      update_sgd(u, w.x, part[j][0], m.x);
      update_sgd(u, w.y, part[j][1], m.y);
      update_sgd(u, w.z, part[j][2], m.z);
      update_sgd(u, w.w, part[j][3], m.w);
      *reinterpret_cast<float4*>(p.opt_w + off) = w;
      if (p.opt_wm) *reinterpret_cast<float4*>(p.opt_wm + off) = m;
      if (p.opt_wv) *reinterpret_cast<float4*>(p.opt_wv + off) = v;
    }
  }
}

__global__ void __launch_bounds__(KTHREADS) skinny_wgrad_kernel(const hnn_gemm_problem* __restrict__ probs, int nprob,
                                                                const hnn_step_row* __restrict__ cur,
                                                                const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  extern __shared__ __align__(16) float wg_smem[];
  float* dys = wg_smem;                   // [WG_CHUNK][16] staged dy rows (zero padded)
  float* red = wg_smem + WG_CHUNK * 16;   // [WG_GROUPS - 1][WG_QUADS][16][4] partials of groups 1..
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_gemm_problem& q) { return q.tile_base; });
  const hnn_gemm_problem& p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int n0 = (blockIdx.x - p.tile_base) * (4 * WG_QUADS);
  const int qd = threadIdx.x % WG_QUADS, q = threadIdx.x / WG_QUADS;
  const int col = n0 + qd * 4;
  const bool active = col < p.n;  // n is a multiple of 4 (host routing)
  const bool bias_thread = n0 == 0 && threadIdx.x < p.m && (p.dbias || p.opt_b);
  if (p.m <= 4) wgrad_tile<4>(p, cur[p.model], col, active, q, qd, dys, red, bias_thread);
  else if (p.m <= 8) wgrad_tile<8>(p, cur[p.model], col, active, q, qd, dys, red, bias_thread);
  else if (p.m <= 10) wgrad_tile<10>(p, cur[p.model], col, active, q, qd, dys, red, bias_thread);
  else if (p.m <= 12) wgrad_tile<12>(p, cur[p.model], col, active, q, qd, dys, red, bias_thread);
  else wgrad_tile<16>(p, cur[p.model], col, active, q, qd, dys, red, bias_thread);
}

// ------------------------------------------------------------------------ fused DGRAD + WGRAD
// The logits layer's backward in one pass over its input X (the WGRAD operand and the DGRAD relu
// mask are the same tensor): CTA = the WGRAD tile above (128 columns x 8 row groups); per row a
// thread loads its X quad once, adds dY[r, :]^T x into its weight-gradient partial, and writes
// dX[r, quad] = (dY[r, :] W[:, quad]) * (X > 0) with the DGRAD kernel's FMA order (bit-identical
// to the two separate launches).  Only for problems without a fused optimizer: W must not change
// while any CTA still reads it.  wp / dp: the WGRAD and DGRAD problems of the same layers, in the
// same order (tile_base in wp); at most 10 output units (the host routes wider layers to the two
// separate launches: 16 units' W quads and partials would not fit two CTAs' registers).
template <int MJ>
__device__ __forceinline__ void bwd_tile(const hnn_gemm_problem& p, const hnn_gemm_problem& d, const hnn_step_row& row,
                                         int col, bool active, int q, int qd, float* dys, float* red, bool bias_thread) {
  const int rows = row.rows;
  float part[MJ][4];
#pragma unroll
  for (int j = 0; j < MJ; ++j) part[j][0] = part[j][1] = part[j][2] = part[j][3] = 0.0f;
#if HNN_SKBWD_WSMEM
  // W quads of the CTA's 128 columns in shared memory (the registers hold the partials and more rows
  // of X in flight instead)
  float4* wq = reinterpret_cast<float4*>(red + (WG_GROUPS - 1) * WG_QUADS * 64);  // [MJ][WG_QUADS]
  if (q == 0)
    for (int j = 0; j < MJ; ++j)
      wq[j * WG_QUADS + qd] = (active && j < d.k) ? ldg4(d.b + size_t(j) * d.ldb + col) : make_float4(0, 0, 0, 0);
#define SKBWD_W(j) wq[(j) * WG_QUADS + qd]
#else
  float4 w[MJ];
#pragma unroll
  for (int j = 0; j < MJ; ++j) w[j] = (active && j < d.k) ? ldg4(d.b + size_t(j) * d.ldb + col) : make_float4(0, 0, 0, 0);
#define SKBWD_W(j) w[j]
#endif
  const bool own_mask = d.mask != nullptr && d.mask != p.b;  // (a mask other than X: loaded separately)
  float bsum = -0.0f;
  for (int base = 0; base < rows; base += WG_CHUNK) {
    const int n = min(WG_CHUNK, rows - base);
    __syncthreads();
    stage_dy(p, base, n, dys);
    __syncthreads();
    if (bias_thread) bsum = colsum_rows(dys, n, threadIdx.x, bsum);  // numpy's axis-0 order
    if (active) {
      const int r_lo = base + (n * q) / WG_GROUPS, r_hi = base + (n * (q + 1)) / WG_GROUPS;
      const float* x = p.b + col;
#pragma unroll SKBWD_UNROLL
      for (int r = r_lo; r < r_hi; ++r) {
        const float4 xv = ldg4(x + size_t(r) * p.ldb);
        const float* dr = dys + (r - base) * 16;
        float4 o = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
        for (int j = 0; j < MJ; ++j) {
          const float dj = dr[j];
          const float4 wj = SKBWD_W(j);
          part[j][0] = fmaf(dj, xv.x, part[j][0]);
          part[j][1] = fmaf(dj, xv.y, part[j][1]);
          part[j][2] = fmaf(dj, xv.z, part[j][2]);
          part[j][3] = fmaf(dj, xv.w, part[j][3]);
          o.x = fmaf(dj, wj.x, o.x);
          o.y = fmaf(dj, wj.y, o.y);
          o.z = fmaf(dj, wj.z, o.z);
          o.w = fmaf(dj, wj.w, o.w);
        }
        if (d.mask) {
          const float4 mk = own_mask ? ldg4(d.mask + size_t(r) * d.ldc + col) : xv;
          o.x = np_mask(o.x, mk.x);
          o.y = np_mask(o.y, mk.y);
          o.z = np_mask(o.z, mk.z);
          o.w = np_mask(o.w, mk.w);
        }
        *reinterpret_cast<float4*>(d.c + size_t(r) * d.ldc + col) = o;
      }
    }
  }
  if (active)  // rows past this step's batch: exact zeros (as the DGRAD kernel writes them)
    for (int r = rows + q; r < d.m; r += WG_GROUPS)
      *reinterpret_cast<float4*>(d.c + size_t(r) * d.ldc + col) = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (bias_thread && p.dbias) p.dbias[threadIdx.x] = bsum;
  if (q > 0) {
    float* dst = red + (size_t(q - 1) * WG_QUADS + qd) * 64;
#pragma unroll
    for (int j = 0; j < MJ; ++j)
      *reinterpret_cast<float4*>(dst + j * 4) = make_float4(part[j][0], part[j][1], part[j][2], part[j][3]);
  }
  __syncthreads();
  if (q != 0 || !active) return;
  for (int g = 0; g < WG_GROUPS - 1; ++g) {  // row groups summed in fixed order 0 + 1 + ... + 7
    const float* src = red + (size_t(g) * WG_QUADS + qd) * 64;
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
    if (j >= p.m) break;
    if (p.c) *reinterpret_cast<float4*>(p.c + size_t(j) * p.ldc + col) = make_float4(part[j][0], part[j][1], part[j][2], part[j][3]);
  }
}

#undef SKBWD_W

__global__ void __launch_bounds__(KTHREADS, 2) skinny_bwd_kernel(const hnn_gemm_problem* __restrict__ wprobs,
                                                                 const hnn_gemm_problem* __restrict__ dprobs, int nprob,
                                                                 const hnn_step_row* __restrict__ cur,
                                                                 const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  extern __shared__ __align__(16) float wg_smem[];
  float* dys = wg_smem;
  float* red = wg_smem + WG_CHUNK * 16;
  const int pi = find_problem(wprobs, nprob, blockIdx.x, [](const hnn_gemm_problem& q) { return q.tile_base; });
  const hnn_gemm_problem& p = wprobs[pi];
  const hnn_gemm_problem& d = dprobs[pi];
  if (!live(cur, status, p.model)) return;
  const int n0 = (blockIdx.x - p.tile_base) * (4 * WG_QUADS);
  const int qd = threadIdx.x % WG_QUADS, q = threadIdx.x / WG_QUADS;
  const int col = n0 + qd * 4;
  const bool active = col < p.n;
  const bool bias_thread = n0 == 0 && threadIdx.x < p.m && p.dbias;
  if (p.m <= 4) bwd_tile<4>(p, d, cur[p.model], col, active, q, qd, dys, red, bias_thread);
  else if (p.m <= 8) bwd_tile<8>(p, d, cur[p.model], col, active, q, qd, dys, red, bias_thread);
  else bwd_tile<10>(p, d, cur[p.model], col, active, q, qd, dys, red, bias_thread);  // (host: m <= 10)
}

int skinny_tile_shape(int op, int32_t* tm, int32_t* tn) {
  if (op == HNN_FWD) { *tm = 8 * FWD_ROWS; *tn = 16; }
  else if (op == HNN_DGRAD) { *tm = 8 * DG_ROWS; *tn = 128; }
  else { *tm = 16; *tn = 4 * WG_QUADS; }
  return HNN_OK;
}

int grouped_gemm_skinny(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                        const hnn_model_status* status, cudaStream_t s) {
  if (op == HNN_FWD) {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(skinny_fwd_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FB_SMEM);
      configured = true;
    }
    const char* e = getenv("HNN_SKINNY_FWD_BULK");  // (0: the per-warp form, A/B and the bit-identity test)
    const bool bulk = e ? atoi(e) != 0 : true;
    if (bulk)
      hnn::launch_pdl(skinny_fwd_bulk_kernel, dim3(total_tiles), dim3(FB_THREADS), FB_SMEM, s, probs, nprob, cur, status);
    else
      hnn::launch_pdl(skinny_fwd_kernel, dim3(total_tiles), dim3(KTHREADS), 0, s, probs, nprob, cur, status);
  } else if (op == HNN_DGRAD) {
    hnn::launch_pdl(skinny_dgrad_kernel, dim3(total_tiles), dim3(KTHREADS), 0, s, probs, nprob, cur, status);
  } else {
    constexpr int smem = (WG_CHUNK * 16 + (WG_GROUPS - 1) * WG_QUADS * 64) * 4;  // 72 KB
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(skinny_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      configured = true;
    }
    hnn::launch_pdl(skinny_wgrad_kernel, dim3(total_tiles), dim3(KTHREADS), smem, s, probs, nprob, cur, status);
  }
  return check_launch("hnn_grouped_gemm(skinny)");
}

}  // namespace hnn

extern "C" int hnn_skinny_backward(const hnn_gemm_problem* wgrad_probs, const hnn_gemm_problem* dgrad_probs, int nprob,
                                   int total_tiles, const hnn_step_row* cur, const hnn_model_status* status,
                                   void* stream) {
  HNN_REQUIRE(wgrad_probs && dgrad_probs && cur && nprob > 0 && total_tiles > 0, "hnn_skinny_backward", "bad arguments");
  constexpr int smem = (hnn::WG_CHUNK * 16 + (hnn::WG_GROUPS - 1) * hnn::WG_QUADS * 64 + 10 * hnn::WG_QUADS * 4) * 4;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(hnn::skinny_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  hnn::launch_pdl(hnn::skinny_bwd_kernel, dim3(total_tiles), dim3(hnn::KTHREADS), smem, hnn::as_stream(stream),
                  wgrad_probs, dgrad_probs, nprob, cur, status);
  return hnn::check_launch("hnn_skinny_backward");
}
