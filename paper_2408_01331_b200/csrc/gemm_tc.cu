// Grouped fp32 GEMM on the 5th-gen tensor cores: tcgen05.mma kind::tf32, 3xTF32.
//
// fp32 parity forbids plain TF32 (SURVEY finding 4: relu-mask flips give 1e-1
// gradient errors), so every operand x is split into hi = trunc_tf32(x) and
// lo = rna_tf32(x - hi) and the tile accumulates  A_hi*B_hi + A_hi*B_lo + A_lo*B_hi.
// The tensor core itself truncates fp32 operands to tf32 (measured: feeding raw fp32 as
// "hi" gives the same 6e-7 GEMM error as an explicit split, a rounding unit would give
// ~1e-4), so the raw TMA tile IS the hi operand and converters only write lo.
//
// Per CTA: one 128 x BN output tile of one problem (tile list = concatenation of
// every problem's tiles, ordered heaviest first by the host; a tile's arithmetic
// never depends on its neighbours -> bit-exact isolation).
//   warp 0       TMA producer: raw fp32 tiles, 128-byte swizzle, into a STAGES-deep ring
//   warp 1       TMEM allocator + single-thread MMA issuer (12 MMAs per 32-wide K block)
//   warps 2..5   converters: lo = rna_tf32(x - trunc(x)) into a separate lo ring, fence.proxy.async
//   warps 6..13  accumulators (two per TMEM lane quarter, 64 columns each): promote each
//                128-term TMEM chunk into fp32 registers (RN adds),
//                then the epilogue (bias / relu / relu-mask / zero pad rows) into 128B-swizzled
//                smem staging blocks written out by TMA stores
// Operand majorness per op (row-major fp32 tensors in HBM):
//   FWD    A = X  [cap, K]  K-major      B = W  [N, K]     K-major
//   DGRAD  A = dY [cap, U]  K-major      B = W  [U, N]     N-major
//   WGRAD  A = dY [rows, M] M-major      B = X  [rows, N]  N-major
#include "tc_common.cuh"

namespace hnn {

constexpr int TC_BM = 128, TC_BN = 128, TC_BK = 32;
constexpr int TC_RAW_STAGES = 4;  // TMA ring of raw fp32 tiles (= the hi operands)
constexpr int TC_LO_STAGES = 2;   // converter ring of lo operands
constexpr int TC_THREADS = 448;   // TMA, MMA, 4 converter warps, 8 accumulator warps (2 per lane quarter)
constexpr int TC_CONV_THREADS = 128;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 4;              // 16 KB
constexpr int TC_B_BYTES = TC_BN * TC_BK * 4;              // 16 KB
constexpr int TC_HI_BYTES = TC_A_BYTES + TC_B_BYTES;       // one raw (or lo) stage
constexpr int TC_EPI_BYTES = 8 * 32 * 32 * 4;              // per accumulator warp: one 32x32 fp32 staging block
constexpr int TC_SMEM_BYTES = (TC_RAW_STAGES + TC_LO_STAGES) * TC_HI_BYTES + TC_EPI_BYTES + 1024 + 256;
constexpr int TC_CHUNK_KB = 4;  // k-blocks per TMEM chunk before promotion to fp32 registers

// ---------------------------------------------------------------- the kernel
//
// Persistent: grid = min(tiles, SMs); CTA c walks tiles c, c+grid, ... (the host orders tiles
// heaviest first).  Pipeline counters run across tiles, so a CTA's TMA / converter / MMA /
// accumulator roles overlap the tail of one tile with the head of the next.
//
// Accumulation precision: the tensor core accumulates one chunk (TC_CHUNK_KB k-blocks = 64
// terms) into one of two TMEM buffers; the accumulator warps add each finished chunk into fp32
// registers with round-to-nearest adds ("promotion") and release the buffer.  Long-K sums thus
// see the tensor core's internal accumulation only inside 64-term chunks, keeping errors at
// fp32-FFMA level — needed by Adam, whose first steps amplify absolute gradient errors near
// |g| ~ eps (measured: single-accumulator 3xTF32 gave 8e-6 relative gradient error, enough to
// move Adam weights by up to lr).


template <int OP>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const hnn_gemm_problem* __restrict__ probs, int nprob, int total_tiles,
                   const hnn_step_row* __restrict__ cur, const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  constexpr int A_MN = (OP == HNN_WGRAD) ? 1 : 0;
  constexpr int B_MN = (OP == HNN_FWD) ? 0 : 1;
  constexpr int SR = TC_RAW_STAGES, SL = TC_LO_STAGES;
  extern __shared__ uint8_t smem_raw[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t raw_base = smem_u32(base);                       // [SR][A | B]
  const uint32_t lo_base = raw_base + SR * TC_HI_BYTES;            // [SL][A | B], same layout
  const uint32_t epi_base = raw_base + (SR + SL) * TC_HI_BYTES;  // [8 warps][32 x 128 B], 1024-aligned
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + (SR + SL) * TC_HI_BYTES + TC_EPI_BYTES);
  // barriers
  constexpr int RAW_FULL = 0, RAW_EMPTY = SR, LO_FULL = 2 * SR, LO_EMPTY = 2 * SR + SL;
  constexpr int ACC_FULL = 2 * SR + 2 * SL, ACC_EMPTY = ACC_FULL + 2, NBARS = ACC_EMPTY + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBARS);
  auto bar = [&](int i) { return smem_u32(bars + i); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < SR; ++s) {
      mbar_init(bar(RAW_FULL + s), 1);                 // producer's expect_tx arrival + TMA bytes
      mbar_init(bar(RAW_EMPTY + s), 1);                // MMA commit
    }
    for (int s = 0; s < SL; ++s) {
      mbar_init(bar(LO_FULL + s), TC_CONV_THREADS);    // every converter thread
      mbar_init(bar(LO_EMPTY + s), 1);                 // MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(ACC_FULL + b), 1);                 // MMA commit
      mbar_init(bar(ACC_EMPTY + b), 256);              // every accumulator thread
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    // columns: two chunk buffers [0,128) and [128,256)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * TC_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // every role walks the same tile sequence; tiles of inactive models are skipped by all roles
  auto tile_info = [&](int tile, const hnn_gemm_problem*& p, int& m0, int& n0, int& nkb, int& rows) -> bool {
    p = &probs[find_problem(probs, nprob, tile, [](const hnn_gemm_problem& q) { return q.tile_base; })];
    if (!live(cur, status, p->model)) return false;
    rows = cur[p->model].rows;
    const int t = tile - p->tile_base;
    m0 = (t / p->tiles_n) * TC_BM;
    n0 = (t % p->tiles_n) * TC_BN;
    const int ktot = (OP == HNN_WGRAD) ? rows : p->k;
    nkb = (ktot + TC_BK - 1) / TC_BK;
    return nkb > 0;
  };

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      uint32_t kg = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const hnn_gemm_problem* p;
        int m0, n0, nkb, rows;
        if (!tile_info(tile, p, m0, n0, nkb, rows)) continue;
        for (int kb = 0; kb < nkb; ++kb, ++kg) {
          const int s = kg % SR;
          if (kg >= SR) mbar_wait(bar(RAW_EMPTY + s), ((kg / SR) - 1) & 1);
          const uint32_t st = raw_base + s * TC_HI_BYTES;
          mbar_expect_tx(bar(RAW_FULL + s), TC_HI_BYTES);
          const int k0 = kb * TC_BK;
          if (A_MN) {
#pragma unroll
            for (int b = 0; b < TC_BM / 32; ++b)
              tma_load_2d(st + b * 4096, p->tmap_a, bar(RAW_FULL + s), m0 + 32 * b, k0);
          } else {
            tma_load_2d(st, p->tmap_a, bar(RAW_FULL + s), k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int b = 0; b < TC_BN / 32; ++b)
              tma_load_2d(st + TC_A_BYTES + b * 4096, p->tmap_b, bar(RAW_FULL + s), n0 + 32 * b, k0);
          } else {
            tma_load_2d(st + TC_A_BYTES, p->tmap_b, bar(RAW_FULL + s), k0, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread): hi*hi as soon as the raw tile lands,
    // then the two correction products once the converters have written lo
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(TC_BM, TC_BN, A_MN, B_MN);
      constexpr uint32_t alb = A_MN ? 4096 : 16, asb = A_MN ? 512 : 1024, alt = A_MN ? 1 : 2;
      constexpr uint32_t blb = B_MN ? 4096 : 16, bsb = B_MN ? 512 : 1024, blt = B_MN ? 1 : 2;
      uint32_t kg = 0, cg = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const hnn_gemm_problem* p;
        int m0, n0, nkb, rows;
        if (!tile_info(tile, p, m0, n0, nkb, rows)) continue;
        for (int kb = 0; kb < nkb; ++kb, ++kg) {
          const int in_chunk = kb % TC_CHUNK_KB;
          const uint32_t buf = cg & 1;
          if (in_chunk == 0 && cg >= 2) {
            mbar_wait(bar(ACC_EMPTY + buf), ((cg >> 1) - 1) & 1);  // promoted and released
            tc_fence_after();
          }
          const int s = kg % SR, l = kg % SL;
          const uint32_t a_hi = raw_base + s * TC_HI_BYTES, b_hi = a_hi + TC_A_BYTES;
          const uint32_t a_lo = lo_base + l * TC_HI_BYTES, b_lo = a_lo + TC_A_BYTES;
          const uint32_t acc = tmem + buf * TC_BN;
          mbar_wait(bar(RAW_FULL + s), (kg / SR) & 1);
          tc_fence_after();
#pragma unroll
          for (int j = 0; j < TC_BK / 8; ++j) {
            // K step j = 8 tf32: +32 B inside a K-major row, +1024 B (two 4-row atoms) in MN-major
            const uint32_t ao = A_MN ? j * 1024 : j * 32, bo = B_MN ? j * 1024 : j * 32;
            mma_tf32(acc, smem_desc(a_hi + ao, alb, asb, alt), smem_desc(b_hi + bo, blb, bsb, blt), idesc,
                     (in_chunk | j) != 0);
          }
          mbar_wait(bar(LO_FULL + l), (kg / SL) & 1);
          tc_fence_after();
#pragma unroll
          for (int j = 0; j < TC_BK / 8; ++j) {
            const uint32_t ao = A_MN ? j * 1024 : j * 32, bo = B_MN ? j * 1024 : j * 32;
            const uint64_t dah = smem_desc(a_hi + ao, alb, asb, alt), dal = smem_desc(a_lo + ao, alb, asb, alt);
            const uint64_t dbh = smem_desc(b_hi + bo, blb, bsb, blt), dbl = smem_desc(b_lo + bo, blb, bsb, blt);
            mma_tf32(acc, dal, dbh, idesc, 1);
            mma_tf32(acc, dah, dbl, idesc, 1);
          }
          mma_commit(bar(RAW_EMPTY + s));  // raw and lo slots free once these MMAs have read them
          mma_commit(bar(LO_EMPTY + l));
          if (in_chunk == TC_CHUNK_KB - 1 || kb == nkb - 1) {
            mma_commit(bar(ACC_FULL + buf));  // chunk partial ready for promotion
            ++cg;
          }
        }
      }
    }
  } else if (warp < 6) {
    // ---------------- converters: lo = rna_tf32(x - trunc_tf32(x)); the raw tile stays as hi
    const int ct = threadIdx.x - 64;  // 0..127
    constexpr int PER = TC_HI_BYTES / 16 / TC_CONV_THREADS;
    uint32_t kg = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const hnn_gemm_problem* p;
      int m0, n0, nkb, rows;
      if (!tile_info(tile, p, m0, n0, nkb, rows)) continue;
      for (int kb = 0; kb < nkb; ++kb, ++kg) {
        const int s = kg % SR, l = kg % SL;
        mbar_wait(bar(RAW_FULL + s), (kg / SR) & 1);
        const uint32_t hi = raw_base + s * TC_HI_BYTES, lo = lo_base + l * TC_HI_BYTES;
        uint4 v[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) v[u] = lds128(hi + 16 * (ct + u * TC_CONV_THREADS));
        if (kg >= SL) mbar_wait(bar(LO_EMPTY + l), ((kg / SL) - 1) & 1);
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          uint4 o;
          o.x = tf32_bits(__float_as_uint(__uint_as_float(v[u].x) - __uint_as_float(v[u].x & 0xFFFFE000u)));
          o.y = tf32_bits(__float_as_uint(__uint_as_float(v[u].y) - __uint_as_float(v[u].y & 0xFFFFE000u)));
          o.z = tf32_bits(__float_as_uint(__uint_as_float(v[u].z) - __uint_as_float(v[u].z & 0xFFFFE000u)));
          o.w = tf32_bits(__float_as_uint(__uint_as_float(v[u].w) - __uint_as_float(v[u].w & 0xFFFFE000u)));
          sts128(lo + 16 * (ct + u * TC_CONV_THREADS), o);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(bar(LO_FULL + l));
      }
    }
  } else {
    // ---------------- accumulators + epilogue (warps 6..13: lane quarter warp % 4, column half)
    constexpr int HALF = TC_BN / 2;
    const int q = warp & 3, half = (warp - 6) >> 2;
    const uint32_t lane_base = tmem + (uint32_t(q * 32) << 16) + half * HALF;
    const uint32_t stg = epi_base + (warp - 6) * 4096;
    uint32_t cg = 0, nstore = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const hnn_gemm_problem* p;
      int m0, n0, nkb, rows;
      if (!tile_info(tile, p, m0, n0, nkb, rows)) continue;
      const int nchunks = (nkb + TC_CHUNK_KB - 1) / TC_CHUNK_KB;
      const int row0 = m0 + q * 32, row = row0 + lane;
      const int nh = n0 + half * HALF;
      float sum[HALF];
      for (int c = 0; c < nchunks; ++c, ++cg) {
        const uint32_t buf = cg & 1;
        mbar_wait(bar(ACC_FULL + buf), (cg >> 1) & 1);
        tc_fence_after();
        // promotion: fp32 running total += chunk (round-to-nearest adds)
#pragma unroll
        for (int cb = 0; cb < HALF; cb += 32) {
          uint32_t r0[32];
          tmem_ld32(lane_base + buf * TC_BN + cb, r0);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            sum[cb + j] = (c == 0) ? __uint_as_float(r0[j]) : __fadd_rn(sum[cb + j], __uint_as_float(r0[j]));
        }
        tc_fence_before();
        mbar_arrive(bar(ACC_EMPTY + buf));
      }
      // epilogue: per 32x32 block, registers -> 128B-swizzled staging (16-byte chunk j of row r
      // lives at chunk j ^ (r & 7): conflict-free STS.128) -> one TMA store per block
      const bool zero_row = (OP != HNN_WGRAD) && row >= rows;
      const float* mrow = (OP == HNN_DGRAD && p->mask && row < p->m) ? p->mask + size_t(row) * p->ldc : nullptr;
#pragma unroll
      for (int cb = 0; cb < HALF; cb += 32) {
        if (lane == 0 && nstore > 0) tma_store_wait_read();  // previous store done reading staging
        __syncwarp();
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          float v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int jj = j4 * 4 + e, n = nh + cb + jj;
            float x = sum[cb + jj];
            if (OP == HNN_FWD) {
              if (zero_row) x = 0.0f;
              else {
                if (n < p->n) x = __fadd_rn(x, __ldg(p->bias + n));
                if (p->relu & 1) x = np_relu(x);
              }
            } else if (OP == HNN_DGRAD) {
              if (zero_row) x = 0.0f;
              else if (mrow && n < p->n) x = np_mask(x, __ldg(mrow + n));
            }
            v[e] = x;
          }
          sts128(stg + lane * 128 + ((j4 ^ (lane & 7)) << 4),
                 make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3])));
        }
        __syncwarp();
        if (OP == HNN_WGRAD && p->opt_w != nullptr) {
          // fused optimizer: lane = column, so W / moment accesses of a row are one coalesced
          // 128-byte transaction; the gradient comes back out of the swizzled staging block
          const Update u = make_update(cur[p->model], p->opt_kind, p->opt_momentum);
          const int n = nh + cb + lane;
          if (n < p->n) {
            for (int rr = 0; rr < 32; ++rr) {
              const int r = row0 + rr;
              if (r >= p->m) break;
              const float g = lds32(stg + rr * 128 + ((((lane >> 2) ^ (rr & 7))) << 4) + ((lane & 3) << 2));
              const size_t off = size_t(r) * p->ldc + n;
              float w = p->opt_w[off], mm = p->opt_wm ? p->opt_wm[off] : 0.0f, vv = p->opt_wv ? p->opt_wv[off] : 0.0f;
              update_sgd(u, w, g, mm);
              p->opt_w[off] = w;
              if (p->opt_wm) p->opt_wm[off] = mm;
              if (p->opt_wv) p->opt_wv[off] = vv;
            }
          }
          __syncwarp();
        }
        if (p->c != nullptr) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) tma_store_2d(p->tmap_c, stg, nh + cb, row0);
          ++nstore;
        }
      }
    }
    if (lane == 0) tma_store_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_BN));
  }
}

// dbias[i] = sum_{r<R} A[r*lda + i], sequential row order (numpy's axis-0 sum), one thread per
// column; with optimizer fusion the bias is updated here too.
// WGRAD bias gradient: db[i] = sum over rows r < R of dY[r, i] in numpy's axis-0 order (sequential
// from -0.0, row by row), + the fused bias update.  One CTA per 32 columns of a problem: the four
// warps stage COLSUM_CHUNK rows x 32 columns of dY in shared memory with all their float4 loads in
// flight (8 per thread), then warp 0 (lane = column) adds the rows in order.  One thread per
// column streaming its own column (the previous form) kept too few bytes in flight per SM: 22 us
// per C3 launch at 1.6 TB/s (profiles/r02/ncu_step_c3_v2.txt).
constexpr int COLSUM_CHUNK = 128, COLSUM_THREADS = 128;

__global__ void __launch_bounds__(COLSUM_THREADS) colsum_kernel(const hnn_gemm_problem* __restrict__ probs, int nprob,
                                                               const hnn_step_row* __restrict__ cur,
                                                               const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  __shared__ __align__(16) float tile[COLSUM_CHUNK][32];
  const hnn_gemm_problem& p = probs[blockIdx.y];
  if ((!p.dbias && !p.opt_b) || !live(cur, status, p.model)) return;
  const int c0 = blockIdx.x * 32;
  if (c0 >= p.m) return;
  const int R = cur[p.model].rows * p.row_mult;
  const int t = threadIdx.x, lane = t & 31;
  const bool vec = (p.lda & 3) == 0 && (reinterpret_cast<uintptr_t>(p.a) & 15) == 0 && c0 + 32 <= p.m;
  const int q = t & 7, r_in = t >> 3;  // float4 column quad, row within a 16-row slab
  float acc = -0.0f;
  for (int base = 0; base < R; base += COLSUM_CHUNK) {
    const int n = min(COLSUM_CHUNK, R - base);
    if (vec) {
      float4 v[COLSUM_CHUNK / 16];
#pragma unroll
      for (int j = 0; j < COLSUM_CHUNK / 16; ++j) {
        const int r = r_in + 16 * j;
        v[j] = r < n ? __ldg(reinterpret_cast<const float4*>(p.a + size_t(base + r) * p.lda + c0) + q)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < COLSUM_CHUNK / 16; ++j) *reinterpret_cast<float4*>(&tile[r_in + 16 * j][4 * q]) = v[j];
    } else {
      for (int e = t; e < n * 32; e += COLSUM_THREADS) {
        const int r = e >> 5, c = e & 31;
        tile[r][c] = c0 + c < p.m ? __ldg(p.a + size_t(base + r) * p.lda + c0 + c) : 0.0f;
      }
    }
    __syncthreads();
    if (t < 32) {
      int r = 0;
      for (; r + 8 <= n; r += 8) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = tile[r + j][lane];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc = __fadd_rn(acc, v[j]);
      }
      for (; r < n; ++r) acc = __fadd_rn(acc, tile[r][lane]);
    }
    __syncthreads();
  }
  const int i = c0 + lane;
  if (t >= 32 || i >= p.m) return;
  if (p.dbias) p.dbias[i] = acc;
  if (p.opt_b) {
    const Update u = make_update(cur[p.model], p.opt_kind, p.opt_momentum);
    float w = p.opt_b[i], m = p.opt_bm ? p.opt_bm[i] : 0.0f, v = p.opt_bv ? p.opt_bv[i] : 0.0f;
    update_sgd(u, w, acc, m);
    p.opt_b[i] = w;
    if (p.opt_bm) p.opt_bm[i] = m;
    if (p.opt_bv) p.opt_bv[i] = v;
  }
}

// Split-K forward epilogue (HNN_PREC_F32_3XTF32_PAIR problems with ksplit > 1 wrote raw partial
// sums): y[r, j] = relu?(sum over splits in order of partial[s*mp + r, j] + bias[j]) for r < rows,
// 0 beyond the batch.  Problem fields: a = partials (row stride lda, split stride mp = m rounded up
// to 32 rows), c = y (row stride ldc), bias, relu, m, n, ksplit, model; tile_base / tiles_n = this
// problem's first block and block count.
__global__ void __launch_bounds__(256) splitk_epilogue_kernel(const hnn_gemm_problem* __restrict__ probs, int nprob,
                                                             const hnn_step_row* __restrict__ cur,
                                                             const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  const int pi = find_problem(probs, nprob, blockIdx.x, [](const hnn_gemm_problem& q) { return q.tile_base; });
  const hnn_gemm_problem& p = probs[pi];
  if (!live(cur, status, p.model)) return;
  const int rows = cur[p.model].rows;
  const int S = p.ksplit, total = p.m * p.n;
  const size_t split_stride = size_t((p.m + 31) & ~31) * p.lda;
  for (int e = (blockIdx.x - p.tile_base) * 256 + threadIdx.x; e < total; e += p.tiles_n * 256) {
    const int r = e / p.n, j = e - r * p.n;
    float v[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) v[s] = s < S ? __ldg(p.a + s * split_stride + size_t(r) * p.lda + j) : 0.0f;
    // in order, the first split taken as is: the unsplit kernel's promotion sequence when every
    // split is one 128-term chunk (then the result is bit-identical to not splitting)
    float acc = 0.0f;
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (s < S) acc = s == 0 ? v[0] : __fadd_rn(acc, v[s]);
    for (int s = 8; s < S; ++s) acc = __fadd_rn(acc, __ldg(p.a + s * split_stride + size_t(r) * p.lda + j));
    float y = 0.0f;
    if (r < rows) {
      y = __fadd_rn(acc, p.bias ? __ldg(p.bias + j) : 0.0f);
      if (p.relu & 1) y = np_relu(y);
    }
    p.c[size_t(r) * p.ldc + j] = y;
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

// 2D fp32 map: inner extent `inner` (contiguous), `outer` rows of `stride_floats`, box {32, box_outer}.
int encode_2d(CUtensorMap* map, const float* ptr, uint64_t inner, uint64_t outer, uint64_t stride_floats,
                     uint32_t box_outer, bool mn_major) {
  EncodeTiled enc = encoder();
  if (!enc) return HNN_ERR_CUDA;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride_floats * 4};
  cuuint32_t box[2] = {32, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? HNN_OK : HNN_ERR_CUDA;
}

// 2D bf16 map, K-major operand: inner extent `inner` (contiguous K), `outer` rows, box {64, box_outer}
// (64 bf16 = one 128-byte swizzled row).
int encode_2d_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t stride_elems,
                   uint32_t box_outer) {
  EncodeTiled enc = encoder();
  if (!enc) return HNN_ERR_CUDA;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride_elems * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? HNN_OK : HNN_ERR_CUDA;
}

// 4D bf16 map over NHWC activations for the implicit-GEMM convolution: dims {c, w, h, n}, box
// {64, ow, box_h, box_n} = one 128-row K-major tile (rows (n, h, w), 128-byte swizzled rows).
int encode_nhwc_bf16(CUtensorMap* map, const void* ptr, const hnn_gemm_problem& p, int pixels) {
  EncodeTiled enc = encoder();
  if (!enc) return HNN_ERR_CUDA;
  const int hw = p.im_oh * p.im_ow;
  const uint32_t box_h = uint32_t(hw >= pixels ? pixels / p.im_ow : p.im_oh),
                 box_n = uint32_t(hw >= pixels ? 1 : pixels / hw);
  cuuint64_t dims[4] = {uint64_t(p.im_c), uint64_t(p.im_w), uint64_t(p.im_h), uint64_t(p.im_n)};
  cuuint64_t strides[3] = {uint64_t(p.im_c) * 2, uint64_t(p.im_w) * p.im_c * 2, uint64_t(p.im_h) * p.im_w * p.im_c * 2};
  cuuint32_t box[4] = {64, uint32_t(p.im_ow), box_h, box_n};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? HNN_OK : HNN_ERR_CUDA;
}

// 3D fp32 map over an NCHW conv output [cap][c][hw] (c_mode 1 with hw % 32 == 0): box {32 pixels,
// 32 channels, 1 image}, unswizzled (the epilogue stages [channel][pixel] blocks)
int encode_nchw_f32(CUtensorMap* map, const float* ptr, uint64_t hw, uint64_t c, uint64_t cap) {
  EncodeTiled enc = encoder();
  if (!enc) return HNN_ERR_CUDA;
  cuuint64_t dims[3] = {hw, c, cap};
  cuuint64_t strides[2] = {hw * 4, c * hw * 4};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? HNN_OK : HNN_ERR_CUDA;
}

// 2D bf16 map over NHWC rows [m, n] (the epilogue's second output), box {32 channels, 32 pixels},
// unswizzled (staged as [pixel][channel])
int encode_rows_bf16(CUtensorMap* map, const void* ptr, uint64_t n, uint64_t m) {
  EncodeTiled enc = encoder();
  if (!enc) return HNN_ERR_CUDA;
  cuuint64_t dims[2] = {n, m};
  cuuint64_t strides[1] = {n * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? HNN_OK : HNN_ERR_CUDA;
}

int gemm_tc_tile_shape(int op, int32_t* tm, int32_t* tn) {
  *tm = TC_BM;
  *tn = TC_BN;
  return HNN_OK;
}

int launch_colsum(const hnn_gemm_problem* probs, int nprob, const hnn_step_row* cur, const hnn_model_status* status,
                  cudaStream_t s);

int grouped_gemm_tc(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                    const hnn_model_status* status, cudaStream_t s) {
  static bool configured[3] = {false, false, false};
  if (!configured[op]) {
    cudaError_t e;
    if (op == HNN_FWD) e = cudaFuncSetAttribute(gemm_tc_kernel<HNN_FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_BYTES);
    else if (op == HNN_DGRAD) e = cudaFuncSetAttribute(gemm_tc_kernel<HNN_DGRAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_BYTES);
    else e = cudaFuncSetAttribute(gemm_tc_kernel<HNN_WGRAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_BYTES);
    if (e != cudaSuccess) {
      set_error("hnn_grouped_gemm(tc)", cudaGetErrorString(e));
      return HNN_ERR_CUDA;
    }
    configured[op] = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = total_tiles < sms ? total_tiles : sms;
  if (op == HNN_FWD)
    hnn::launch_pdl(gemm_tc_kernel<HNN_FWD>, dim3(grid), dim3(TC_THREADS), TC_SMEM_BYTES, s, probs, nprob, total_tiles, cur, status);
  else if (op == HNN_DGRAD)
    hnn::launch_pdl(gemm_tc_kernel<HNN_DGRAD>, dim3(grid), dim3(TC_THREADS), TC_SMEM_BYTES, s, probs, nprob, total_tiles, cur, status);
  else {
    hnn::launch_pdl(gemm_tc_kernel<HNN_WGRAD>, dim3(grid), dim3(TC_THREADS), TC_SMEM_BYTES, s, probs, nprob, total_tiles, cur, status);
    int rc = check_launch("hnn_grouped_gemm(tc)");
    if (rc) return rc;
    return launch_colsum(probs, nprob, cur, status, s);
  }
  return check_launch("hnn_grouped_gemm(tc)");
}

// WGRAD bias gradient (+ fused bias update) for every problem of a tensor-core launch.
int launch_colsum(const hnn_gemm_problem* probs, int nprob, const hnn_step_row* cur, const hnn_model_status* status,
                  cudaStream_t s) {
  dim3 grid2(128, nprob);  // columns up to 128*32 = 4096 per problem (planner guarantees m <= 4096)
  hnn::launch_pdl(colsum_kernel, dim3(grid2), dim3(COLSUM_THREADS), 0, s, probs, nprob, cur, status);
  return check_launch("hnn_grouped_gemm(colsum)");
}

}  // namespace hnn

// Encode the three TMA maps of every problem (host memory, 128 bytes each: A, B, C per problem).
extern "C" int hnn_gemm_tc_encode(int op, const hnn_gemm_problem* host_probs, int nprob, void* host_maps) {
  HNN_REQUIRE(host_probs && host_maps && nprob > 0, "hnn_gemm_tc_encode", "bad arguments");
  CUtensorMap* maps = reinterpret_cast<CUtensorMap*>(host_maps);
  for (int i = 0; i < nprob; ++i) {
    const hnn_gemm_problem& p = host_probs[i];
    int rc;
    if (op == HNN_FWD) {          // A = X[cap, K] (K-major), B = W[N, K] (K-major)
      const uint32_t brows = p.tile_n > 0 ? uint32_t(p.tile_n / 2) : uint32_t(hnn::TC_BN);
      rc = hnn::encode_2d(&maps[4 * i], p.a, p.k, p.m, p.lda, hnn::TC_BM, false);
      if (!rc) rc = hnn::encode_2d(&maps[4 * i + 1], p.b, p.k, p.n, p.ldb, brows, false);
    } else if (op == HNN_DGRAD) { // A = dY[cap, U] (K-major), B = W[U, N] (N-major)
      rc = hnn::encode_2d(&maps[4 * i], p.a, p.k, p.m, p.lda, hnn::TC_BM, false);
      if (!rc) rc = hnn::encode_2d(&maps[4 * i + 1], p.b, p.n, p.k, p.ldb, 32, true);
    } else {                      // A = dY[cap, M] (M-major), B = X[cap, N] (N-major)
      rc = hnn::encode_2d(&maps[4 * i], p.a, p.m, p.k, p.lda, 32, true);
      if (!rc) rc = hnn::encode_2d(&maps[4 * i + 1], p.b, p.n, p.k, p.ldb, 32, true);
    }
    // C (all ops): row-major [m, n] with row stride ldc; 32x32 boxes, 128-byte swizzle
    // (a K-split WGRAD writes ksplit stacked [m, n] partials)
    const uint64_t crows = ((op == HNN_WGRAD || op == HNN_FWD) && p.ksplit > 1) ? uint64_t((p.m + 31) & ~31) * uint64_t(p.ksplit)
                                                             : uint64_t(p.m);
    if (!rc && p.c && p.c_mode == 1 && p.row_mult % 32 == 0)  // NCHW via 3D TMA stores
      rc = hnn::encode_nchw_f32(&maps[4 * i + 2], p.c, uint64_t(p.row_mult), uint64_t(p.n),
                                uint64_t(p.m / p.row_mult));
    else if (!rc && p.c && p.c_mode == 0)  // (other c_modes store NCHW directly, no map)
      rc = hnn::encode_2d(&maps[4 * i + 2], p.c, p.n, crows, p.ldc, 32, false);
    if (rc) {
      hnn::set_error("hnn_gemm_tc_encode", "cuTensorMapEncodeTiled failed (alignment / stride / driver)");
      return rc;
    }
  }
  return HNN_OK;
}

// HNN_PREC_BF16_PAIR: A [m, k] and B [n, k] are K-major bf16 (lda / ldb in elements); C fp32 as above.
extern "C" int hnn_splitk_epilogue(const hnn_gemm_problem* probs, int nprob, int total_blocks,
                                   const hnn_step_row* cur, const hnn_model_status* status, void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && total_blocks > 0, "hnn_splitk_epilogue", "bad arguments");
  hnn::launch_pdl(hnn::splitk_epilogue_kernel, dim3(total_blocks), dim3(256), 0, hnn::as_stream(stream), probs, nprob,
                  cur, status);
  return hnn::check_launch("hnn_splitk_epilogue");
}

extern "C" int hnn_gemm_bf16_encode(int op, const hnn_gemm_problem* host_probs, int nprob, void* host_maps) {
  HNN_REQUIRE(host_probs && host_maps && nprob > 0, "hnn_gemm_bf16_encode", "bad arguments");
  CUtensorMap* maps = reinterpret_cast<CUtensorMap*>(host_maps);
  for (int i = 0; i < nprob; ++i) {
    const hnn_gemm_problem& p = host_probs[i];
    const uint32_t brows = p.tile_n > 0 ? uint32_t(p.tile_n / 2) : 128u;
    int rc;
    const int hw = p.im_oh * p.im_ow;
    const int taps = p.im_k * (p.im_kw > 0 ? p.im_kw : p.im_k);
    if (p.im_c > 0 && op == HNN_FWD) {  // implicit-GEMM convolution: A = NHWC activations
      HNN_REQUIRE(p.im_c % 64 == 0 && p.im_ow > 0 && 128 % p.im_ow == 0 && (hw % 128 == 0 || 128 % hw == 0) &&
                      p.k == taps * p.im_c,
                  "hnn_gemm_bf16_encode", "implicit convolution geometry not supported");
      rc = hnn::encode_nhwc_bf16(&maps[4 * i], p.a, p, 128);
    } else {
      rc = hnn::encode_2d_bf16(&maps[4 * i], p.a, p.k, p.m, p.lda, hnn::TC_BM);
    }
    if (rc) {
    } else if (p.im_c > 0 && op == HNN_WGRAD) {  // implicit weight gradient: B = NHWC activations, MN-major
      HNN_REQUIRE(p.im_c % 64 == 0 && p.tile_n == 128 && p.im_ow > 0 && 64 % p.im_ow == 0 &&
                      (hw % 64 == 0 || 64 % hw == 0) && p.n == taps * p.im_c,
                  "hnn_gemm_bf16_encode", "implicit weight-gradient geometry not supported");
      rc = hnn::encode_nhwc_bf16(&maps[4 * i + 1], p.b, p, 64);
    } else {
      rc = hnn::encode_2d_bf16(&maps[4 * i + 1], p.b, p.k, p.n, p.ldb, brows);
    }
    const uint64_t crows = ((op == HNN_WGRAD || op == HNN_FWD) && p.ksplit > 1) ? uint64_t((p.m + 31) & ~31) * uint64_t(p.ksplit)
                                                             : uint64_t(p.m);
    if (!rc && p.c && p.c_mode == 1 && p.row_mult % 32 == 0)  // NCHW via 3D TMA stores
      rc = hnn::encode_nchw_f32(&maps[4 * i + 2], p.c, uint64_t(p.row_mult), uint64_t(p.n),
                                uint64_t(p.m / p.row_mult));
    else if (!rc && p.c && p.c_mode == 0)  // (other c_modes store NCHW directly, no map)
      rc = hnn::encode_2d(&maps[4 * i + 2], p.c, p.n, crows, p.ldc, 32, false);
    if (!rc && p.xh_out) {
      HNN_REQUIRE(op == HNN_FWD && p.c_mode == 1 && p.row_mult % 32 == 0 && p.n % 8 == 0, "hnn_gemm_bf16_encode",
                  "xh_out needs a bf16 NCHW forward with 32-pixel runs and 16-byte rows");
      rc = hnn::encode_rows_bf16(&maps[4 * i + 3], p.xh_out, uint64_t(p.n), uint64_t(p.m));
    }
    if (rc) {
      hnn::set_error("hnn_gemm_bf16_encode", "cuTensorMapEncodeTiled failed (alignment / stride / driver)");
      return rc;
    }
  }
  return HNN_OK;
}
