// Grouped fp32 GEMM on CTA pairs: tcgen05.mma.cta_group::2 kind::tf32, 3xTF32, 256 x 256 tiles.
//
// Why pairs: the single-CTA kernel (gemm_tc.cu, 128 x 128 tiles) is shared-memory-bandwidth
// bound — per 32-wide K block its 12 tf32 MMAs read 96 KB of operands out of smem and TMA +
// the lo converters move another 96 KB, ~250 B/clk against ~128 B/clk (ncu: tensor pipe 24-35%,
// profiles/r01/ncu_c3_v4.txt).  With cta_group::2 one MMA covers a 256 x 256 tile across the
// two SMs of a TPC: each CTA stages half of A (its 128 rows) and half of B (128 of the 256
// columns), the tensor cores exchange the B halves, and per CTA the operand reads drop to
// 64 B/clk with the converter traffic at 62 B/clk.
//
// Arithmetic is the single-CTA kernel's: every operand x is used as hi = x (the tensor core
// truncates fp32 to tf32) and lo = rna_tf32(x - trunc_tf32(x)); the tile accumulates
// A_lo*B_hi + A_hi*B_lo + A_hi*B_hi.  Accumulation precision ("promotion"): the tensor core
// sums one chunk of TC2_CHUNK_KB K blocks into one of two 256-column TMEM buffers; the
// accumulator warps add each finished chunk into fp32 registers (IEEE adds) and release the
// buffer, so the MMAs of the next chunk never wait for a promotion (double buffering).
// The split itself is fp32-exact to ~2^-24 (emulated with exact sums: 3.9e-7 GEMM error at
// K = 256, the same as an fp32 BLAS); what costs accuracy is the tensor core's accumulation,
// which aligns each MMA's addends to the largest and drops the bits below.  So a chunk is TWO
// 32-term K blocks, and the small correction products of both go first, while the accumulator is
// still small (measured, tools/adam_probe2.py, C3 h = 2048: gradient error against float64 3.8e-6
// with 4-block chunks and hi*hi first; 4.0-5.6e-7 with one-block chunks, lo first; 5.1-7.0e-7 with
// two-block chunks, both blocks' corrections first; the reference's own fp32 BLAS 3.0-5.4e-7,
// profiles/r02/chunk_accuracy_v4.txt).  One-block chunks promote once per K block, and every
// promotion reads the tile's whole 128 x 256 fp32 accumulator out of TMEM (128 KB per CTA at
// ~64-128 B/clk): the MMA thread waited for promoted buffers 20-43% of its time; two-block chunks
// cut the C3 GEMMs 0.652 -> 0.622 ms.  Each
// CTA's 128 x 256 running sum lives in registers: 8 accumulator warps x 128 columns (384
// threads per CTA leave 168 registers per thread).
//
// Roles (384 threads per CTA, 1 CTA per SM, persistent over a heaviest-first tile list; both
// CTAs of a pair walk the same tiles):
//   warp 0       TMA producer: this CTA's A half and B half, raw fp32, into a 3-stage ring
//   warp 1       TMEM allocator (pair) + single-thread MMA issuer (leader CTA only)
//   warps 2,3    converters: lo ring from the raw ring, then arrive on the leader
//   warps 4..11  accumulators: promotion + epilogue (bias / relu / relu-mask / zero rows) of
//                this CTA's 128 rows, TMA stores; WGRAD optimizer fusion as in gemm_tc.cu
// The raw ring (TC2_RAW K blocks) and the lo ring (TC2_LO) are separate: TMA refills a raw slot
// when the MMAs reading it complete; a converter writes a lo slot once its raw tiles have landed
// and the lo slot's previous MMAs are done (up to TC2_LO - 1 K blocks ahead of the MMAs).
// Barriers: raw full/empty, acc full: per CTA (the leader's commits multicast to both);
// lo full and acc empty: in the leader, arrived on by both CTAs.
#include <algorithm>
#include <cstdlib>
#include <cuda_bf16.h>

#include "tc_common.cuh"

namespace hnn {

constexpr int TC2_BM = 128;                // rows per CTA (pair tile: 256)
constexpr int TC2_BN = 256;                // pair tile columns (each CTA stages 128 of B)
constexpr int TC2_BK = 32;
constexpr int TC2_STAGES = 3;  // ring bytes = 2 * TC2_STAGES * 32 KB (raw A | raw B and lo A | lo B halves)
// fp32: the raw tiles (TMA) and their lo tiles (converters) live in separate rings, deeper for raw:
// a raw slot is refilled as soon as the MMAs that read it complete, so TMA runs TC2_RAW K blocks
// ahead of the tensor core instead of the two a shared raw+lo stage allowed
#ifndef HNN_TC2_RAW_STAGES
#define HNN_TC2_RAW_STAGES 4
#endif
constexpr int TC2_RAW = HNN_TC2_RAW_STAGES, TC2_LO = 2 * TC2_STAGES - TC2_RAW;
static_assert(TC2_RAW >= 2 && TC2_LO >= 2, "raw / lo ring depths");
constexpr int TC2_CONV_WARPS = 2;  // (a fourth warpgroup with two more converter warps measured no gain:
                                   //  profiles/r02/wg3_converters_ab_v9.txt)
constexpr int TC2_THREADS = 384;
#ifndef HNN_TC2_CHUNK_KB
#define HNN_TC2_CHUNK_KB 2
#endif
#ifndef HNN_TC2_LO_FIRST
#define HNN_TC2_LO_FIRST 1
#endif
constexpr int TC2_CHUNK_KB = HNN_TC2_CHUNK_KB;
#ifndef HNN_TC2_PROMO_COLS
#define HNN_TC2_PROMO_COLS 16
#endif
constexpr int TC2_PROMO_COLS = HNN_TC2_PROMO_COLS;
#ifndef HNN_TC2_REGS_ACC
#define HNN_TC2_REGS_ACC 216  // 0: no setmaxnreg split
#endif
#ifndef HNN_TC2_REGS_LO
#define HNN_TC2_REGS_LO 72
#endif  // accumulator columns per TMEM load in the promotion
// K blocks per TMEM accumulation chunk of one tile: a fused-SGD weight-gradient tile whose whole K
// fits 4 blocks keeps one chunk (its epilogue reads the finished sums straight from TMEM)
template <int OP>
static __device__ __forceinline__ int tc2_chunk_kb(const hnn_gemm_problem* p, int nkb) {
  return (OP == HNN_WGRAD && p->opt_w != nullptr && p->opt_wm == nullptr && nkb <= 4) ? 4 : TC2_CHUNK_KB;
}
#ifndef HNN_TC2_NARROW_LAST
#define HNN_TC2_NARROW_LAST 1
#endif
constexpr int TC2_A_BYTES = TC2_BM * TC2_BK * 4;        // 16 KB
constexpr int TC2_B_BYTES = (TC2_BN / 2) * TC2_BK * 4;  // 16 KB (this CTA's half)
constexpr int TC2_STAGE = TC2_A_BYTES + TC2_B_BYTES;
constexpr int TC2_EPI_BYTES = 8 * 32 * 32 * 4;
constexpr int TC2_INFO_RING = 8;  // tile-info entries the producer publishes ahead of the other roles
constexpr int TC2_SMEM_BYTES = TC2_STAGES * 2 * TC2_STAGE + TC2_EPI_BYTES + 1024 + 1024;  // + barriers, tile info

#ifdef HNN_TC2_TRACE  // debug build only (tools/tc2_trace.py): per-CTA wait-cycle counters
__device__ unsigned long long g_tc2_trace[296 * 16];
#define TC2_T0(v) const long long v = clock64()
#define TC2_T1(v, slot) tr[slot] += clock64() - (v)
#else
#define TC2_T0(v)
#define TC2_T1(v, slot)
#endif

// Fused plain SGD over a single-chunk weight-gradient tile (K <= 128: the C1 / C2 / C5 dense
// layers): nothing to promote, so the accumulators are read from TMEM block by block and the
// registers a running sum would hold carry the weights instead, loaded ahead (block 0's before
// the MMAs finish).  Returns the updated TMA-store count.  (Every register array here and in the
// promoting epilogue is defined on all paths: a conditionally-written array is live across the
// tile loop in ptxas's eyes, and that alone spilled 1-2 KB per thread.)
static __device__ __forceinline__ uint32_t tc2_sgd_direct(uint32_t lane_base, uint32_t buf, uint32_t acc_full, uint32_t parity,
                                                       uint32_t acc_empty, uint32_t stg, int row0, int nh, int hn,
                                                       int pm, int pn, int ldc, float* ow, float* cptr,
                                                       const void* tmap_c, float lr, int sp, uint32_t nstore) {
  const int lane = threadIdx.x % 32;
  const int rmax = min(32, pm - row0);
  const int nblk = rmax > 0 ? (min(hn, pn - nh) + 31) / 32 : 0;  // live 32 x 32 blocks
  // lane = row here (the TMEM layout): each lane streams its own row's 32 weights of a block
  // as 8 float4 (the sibling float4 fills the other half of each 32-byte sector) and updates
  // them straight from the accumulator registers; block cb + 1's weights load during block cb
  const bool row_ok = lane < rmax;
  float* const wrow = ow + size_t(row0 + (row_ok ? lane : 0)) * ldc + nh;
  const bool vec = (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(ow) & 15) == 0;
  float4 wA[8], wB[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) wA[j] = wB[j] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#define TC2_LOADW(WV, cb)                                                                          \
  if (row_ok) {                                                                                   \
    if (vec && nh + (cb) + 32 <= pn) {                                                            \
      _Pragma("unroll") for (int j = 0; j < 8; ++j) WV[j] = *reinterpret_cast<const float4*>(wrow + (cb) + 4 * j); \
    } else {                                                                                      \
      _Pragma("unroll") for (int j = 0; j < 8; ++j) {                                             \
  const int c = nh + (cb) + 4 * j;                                                          \
  WV[j].x = c < pn ? wrow[(cb) + 4 * j] : 0.0f;                                              \
  WV[j].y = c + 1 < pn ? wrow[(cb) + 4 * j + 1] : 0.0f;                                      \
  WV[j].z = c + 2 < pn ? wrow[(cb) + 4 * j + 2] : 0.0f;                                      \
  WV[j].w = c + 3 < pn ? wrow[(cb) + 4 * j + 3] : 0.0f;                                      \
      }                                                                                           \
    }                                                                                             \
  }
// one 32 x 32 block: accumulators out of TMEM, the next block's weights into `wn`, optional
// gradient store, SGD on `w` (optim.py: p - lr * g)
#define G32(k) ((k) < 16 ? g0[(k) & 15] : g1[(k) & 15])
#define TC2_SGD_BLOCK(WV, WN, cb)                                                                  \
  if ((cb) < 32 * nblk) {                                                                         \
    uint32_t g0[16], g1[16];                                                                      \
    tmem_ld16(lane_base + buf * TC2_BN + (cb), g0);                                               \
    tmem_ld16(lane_base + buf * TC2_BN + (cb) + 16, g1);                                          \
    if ((cb) + 32 < 32 * nblk) { TC2_LOADW(WN, (cb) + 32) }                                       \
    if (cptr != nullptr) {                                                                        \
      if (lane == 0 && nstore > 0) tma_store_wait_read();                                         \
      __syncwarp();                                                                               \
      _Pragma("unroll") for (int j4 = 0; j4 < 8; ++j4)                                            \
  sts128(stg + lane * 128 + ((j4 ^ (lane & 7)) << 4), make_uint4(G32(4 * j4), G32(4 * j4 + 1), G32(4 * j4 + 2), G32(4 * j4 + 3))); \
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");                                \
      __syncwarp();                                                                               \
      if (lane == 0) tma_store_2d(tmap_c, stg, nh + (cb), row0 + sp * ((pm + 31) & ~31));         \
      ++nstore;                                                                                   \
    }                                                                                             \
    if (row_ok) {                                                                                 \
      _Pragma("unroll") for (int j = 0; j < 8; ++j) {                                             \
  WV[j].x = __fsub_rn(WV[j].x, __fmul_rn(lr, __uint_as_float(G32(4 * j))));                    \
  WV[j].y = __fsub_rn(WV[j].y, __fmul_rn(lr, __uint_as_float(G32(4 * j + 1))));                \
  WV[j].z = __fsub_rn(WV[j].z, __fmul_rn(lr, __uint_as_float(G32(4 * j + 2))));                \
  WV[j].w = __fsub_rn(WV[j].w, __fmul_rn(lr, __uint_as_float(G32(4 * j + 3))));                \
      }                                                                                           \
      if (vec && nh + (cb) + 32 <= pn) {                                                          \
  _Pragma("unroll") for (int j = 0; j < 8; ++j) *reinterpret_cast<float4*>(wrow + (cb) + 4 * j) = WV[j]; \
      } else {                                                                                    \
  _Pragma("unroll") for (int j = 0; j < 8; ++j) {                                           \
    const int c = nh + (cb) + 4 * j;                                                        \
    if (c < pn) wrow[(cb) + 4 * j] = WV[j].x;                                                \
    if (c + 1 < pn) wrow[(cb) + 4 * j + 1] = WV[j].y;                                        \
    if (c + 2 < pn) wrow[(cb) + 4 * j + 2] = WV[j].z;                                        \
    if (c + 3 < pn) wrow[(cb) + 4 * j + 3] = WV[j].w;                                        \
  }                                                                                         \
      }                                                                                           \
    }                                                                                             \
  }
  if (nblk > 0) { TC2_LOADW(wA, 0) }
  mbar_wait(acc_full, parity);
  tc_fence_after();
  static_assert(TC2_BN / 2 == 128, "four 32-column blocks per warp");
  TC2_SGD_BLOCK(wA, wB, 0)
  TC2_SGD_BLOCK(wB, wA, 32)
  TC2_SGD_BLOCK(wA, wB, 64)
  TC2_SGD_BLOCK(wB, wA, 96)
#undef TC2_SGD_BLOCK
#undef G32
#undef TC2_LOADW
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive_cluster(acc_empty + 8 * buf);
  return nstore;
}

// KIND: 0 = fp32 operands, 3xTF32 (kind::tf32, converters write lo); 1 = bf16 operands, one
// kind::f16 MMA per K step (HNN_PREC_BF16_PAIR: every operand K-major, 64-element K blocks; the
// converter warps only relay "stage landed" to the leader).
template <int OP, int KIND = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC2_THREADS, 1)
    gemm_tc2_kernel(const hnn_gemm_problem* __restrict__ probs, int nprob, int total_tiles,
                    const hnn_step_row* __restrict__ cur, const hnn_model_status* __restrict__ status) {
  hnn::pdl_wait();
  constexpr bool BF16 = KIND == 1;
  constexpr int A_MN = (!BF16 && OP == HNN_WGRAD) ? 1 : 0;
  constexpr int B_MN = (!BF16 && OP != HNN_FWD) ? 1 : 0;
  constexpr int KBE = BF16 ? 64 : TC2_BK;  // K elements per 128-byte stage row
  // bf16 stages carry no lo half: twice as many of them in the same shared memory, i.e. twice the
  // bytes in flight for the HBM-streaming conv GEMMs (a 64-filter layer's MMA needs 20 KB per
  // 128 clocks per CTA, so these launches are bound by the TMA pipeline depth)
  constexpr int SR = BF16 ? 2 * TC2_STAGES : TC2_RAW;  // raw ring depth
  constexpr int SL = BF16 ? SR : TC2_LO;               // lo ring (bf16: the converters' per-stage relay)
  extern __shared__ uint8_t smem_raw[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
#ifdef HNN_TC2_TRACE
  const long long t_start = clock64();
  long long tr[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif

  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t raw_base = smem_u32(base);
  // raw slot s at raw_base + s * TC2_STAGE; (fp32) lo slot l at raw_base + (SR + l) * TC2_STAGE
  const uint32_t epi_base = raw_base + 2 * TC2_STAGES * TC2_STAGE;
  uint8_t* tail = base + 2 * TC2_STAGES * TC2_STAGE + TC2_EPI_BYTES;  // 1 KB: barriers, TMEM address, tile-info ring
  uint64_t* bars = reinterpret_cast<uint64_t*>(tail);
  constexpr int RAW_FULL = 0, RAW_EMPTY = SR, LO_FULL = 2 * SR, LO_EMPTY = 2 * SR + SL;
  constexpr int ACC_FULL = 2 * SR + 2 * SL, ACC_EMPTY = ACC_FULL + 2, INFO_FULL = ACC_EMPTY + 2,
                INFO_EMPTY = INFO_FULL + TC2_INFO_RING, NBARS = INFO_EMPTY + TC2_INFO_RING;
  static_assert(NBARS * 8 <= 512, "barrier area");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tail + 512);
  int4* info = reinterpret_cast<int4*>(tail + 528);  // entry i: info[2i] = {problem | -1, m0, n0, nkb},
                                                     //          info[2i+1] = {rows, kofs, split, tile_n}
  auto bar = [&](int i) { return smem_u32(bars + i); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < SR; ++s) {
      mbar_init(bar(RAW_FULL + s), 1);                  // local TMA expect_tx arrival + bytes
      mbar_init(bar(RAW_EMPTY + s), 1);                 // leader MMA commit (multicast): raw slot free
    }
    for (int l = 0; l < SL; ++l) {
      mbar_init(bar(LO_FULL + l), 2 * TC2_CONV_WARPS);  // converter warps of both CTAs (leader's copy)
      mbar_init(bar(LO_EMPTY + l), 1);                  // (fp32) leader MMA commit (multicast): lo slot free
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(ACC_FULL + b), 1);    // leader MMA commit (multicast)
      mbar_init(bar(ACC_EMPTY + b), 16);  // 8 accumulator warps x 2 CTAs (leader's copy)
    }
    for (int i = 0; i < TC2_INFO_RING; ++i) {
      mbar_init(bar(INFO_FULL + i), 1);  // the producer thread
      // readers: MMA thread (leader CTA only), converter warps, accumulator warps
      mbar_init(bar(INFO_EMPTY + i), (leader ? 1 : 0) + TC2_CONV_WARPS + 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive / multicast commit
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // tile -> (problem, m0, n0, K blocks, valid rows, K offset, split); rows = this step's valid
  // GEMM rows (batch rows x row_mult: output pixels of a conv).  WGRAD tiles are split along K
  // into ksplit fixed ranges (t = (mt * tiles_n + nt) * ksplit + split).
  auto tile_info = [&](int tile, const hnn_gemm_problem*& p, int& m0, int& n0, int& nkb, int& rows, int& kofs,
                       int& sp, int& tn) -> bool {
    p = &probs[find_problem(probs, nprob, tile, [](const hnn_gemm_problem& q) { return q.tile_base; })];
    if (!live(cur, status, p->model)) return false;
    rows = cur[p->model].rows * p->row_mult;
    int t = tile - p->tile_base;
    sp = 0;
    kofs = 0;
    int ktot = p->k;
    if (OP == HNN_WGRAD) {
      ktot = rows;
      const int S = p->ksplit;
      if (S > 1) {
        sp = t % S;
        t /= S;
        kofs = sp * p->ksplit_len;
        ktot = min(rows, kofs + p->ksplit_len) - kofs;
      }
    } else if (OP == HNN_FWD && p->ksplit > 1) {  // split-K forward: raw partial sums per K range
      const int S = p->ksplit;
      sp = t % S;
      t /= S;
      kofs = sp * p->ksplit_len;
      ktot = min(p->k, kofs + p->ksplit_len) - kofs;
    }
    tn = p->tile_n > 0 ? p->tile_n : TC2_BN;  // pair tile columns: 64, 128 or 256
    m0 = (t / p->tiles_n) * (2 * TC2_BM);
    n0 = (t % p->tiles_n) * tn;
    if (HNN_TC2_NARROW_LAST && !BF16 && B_MN) {
      // the last column tile of a ragged n takes the narrowest width covering the rest (n = 784:
      // 3 x 256 + one 64-wide tile instead of a fourth 256-wide one with 16 useful columns); each
      // output column's sum is independent of the MMA's N, so results are unchanged.  (fp32
      // input / weight gradients only: their B tiles load in 32-column boxes, so the TMA bytes
      // follow tn; the K-major forward B box is fixed per problem by its tensor map.)
      const int rem = p->n - n0;
      if (rem < tn) tn = rem <= 64 ? 64 : (rem <= 128 ? 128 : tn);
    }
    nkb = ktot > 0 ? (ktot + KBE - 1) / KBE : 0;
    return nkb > 0;
  };
  // bf16: the producer thread computes every tile's info once (the problem search and the
  // live-model / row-count loads are a chain of dependent global loads) and publishes it in a small
  // shared ring; the MMA thread, converters and accumulator warps read it from there (C4 -1%).
  auto read_info = [&](uint32_t seq, bool warp_wide, const hnn_gemm_problem*& p, int& m0, int& n0, int& nkb,
                       int& rows, int& kofs, int& sp, int& tn) -> bool {
    const int slot = int(seq % TC2_INFO_RING);
    mbar_wait(bar(INFO_FULL + slot), (seq / TC2_INFO_RING) & 1);
    const int4 e0 = info[2 * slot], e1 = info[2 * slot + 1];
    if (warp_wide) __syncwarp();
    if (!warp_wide || (threadIdx.x & 31) == 0) mbar_arrive(bar(INFO_EMPTY + slot));
    if (e0.x < 0) return false;
    p = probs + e0.x;
    m0 = e0.y, n0 = e0.z, nkb = e0.w, rows = e1.x, kofs = e1.y, sp = e1.z, tn = e1.w;
    return true;
  };
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  // tile schedule (host LPT, trailing the problem table): this pair's tiles are
  // sched_ids[sched_off[pair] .. sched_off[pair + 1]); round-robin if absent / mismatched
  const int* sched = reinterpret_cast<const int*>(probs + nprob);
  const bool use_sched = sched[0] == npairs;
  const int t_begin = use_sched ? sched[1 + pair] : pair;
  const int t_end = use_sched ? sched[2 + pair] : total_tiles;
  const int t_step = use_sched ? 1 : npairs;
  const int* sched_ids = sched + 2 + npairs;
  auto tile_id = [&](int i) { return use_sched ? __ldg(sched_ids + i) : i; };

#if HNN_TC2_REGS_ACC
  // register split: the TMA / MMA / converter warpgroup needs few registers, the accumulator warps
  // hold a 128-column running sum plus a TMEM load in flight (384 x 168 = 128 x LO + 256 x HI)
  static_assert((TC2_THREADS - 256) * HNN_TC2_REGS_LO + 256 * HNN_TC2_REGS_ACC <= TC2_THREADS * ((65536 / TC2_THREADS) & ~7),
                "register split");
#endif
  if (warp < 4) {
#if HNN_TC2_REGS_ACC
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(HNN_TC2_REGS_LO));
#endif
  if (warp == 0) {
    // ---------------- TMA producer (both CTAs): rows m0 + rank*128.., columns n0 + rank*128..
    if (lane == 0) {
      uint32_t kg = 0, iseq = 0;
      for (int ti = t_begin; ti < t_end; ti += t_step) {
        const int tile = tile_id(ti);
        const hnn_gemm_problem* p;
        int m0, n0, nkb, rows, kofs, sp, tn;
        const bool ok = tile_info(tile, p, m0, n0, nkb, rows, kofs, sp, tn);
        if (BF16) {  // (fp32: the extra live registers of the ring spilled the running sum; not used)
          const int slot = int(iseq % TC2_INFO_RING);
          if (iseq >= TC2_INFO_RING) mbar_wait(bar(INFO_EMPTY + slot), ((iseq / TC2_INFO_RING) - 1) & 1);
          info[2 * slot] = make_int4(ok ? int(p - probs) : -1, m0, n0, nkb);
          info[2 * slot + 1] = make_int4(rows, kofs, sp, tn);
          mbar_arrive(bar(INFO_FULL + slot));  // (release: the entry is visible to the waiting readers)
          ++iseq;
        }
        if (!ok) continue;
        const int am = m0 + int(rank) * TC2_BM, bn = n0 + int(rank) * (tn / 2);
        const uint32_t stage_bytes = TC2_A_BYTES + (tn / 2) * TC2_BK * 4;
        for (int kb = 0; kb < nkb; ++kb, ++kg) {
          const int s = kg % SR;
          TC2_T0(t3);
          if (kg >= SR) mbar_wait(bar(RAW_EMPTY + s), ((kg / SR) - 1) & 1);
          TC2_T1(t3, 3);
          const uint32_t st = raw_base + s * TC2_STAGE;
          mbar_expect_tx(bar(RAW_FULL + s), stage_bytes);
          const int k0 = kofs + kb * KBE;
          if (A_MN) {
#pragma unroll
            for (int b = 0; b < TC2_BM / 32; ++b) tma_load_2d(st + b * 4096, p->tmap_a, bar(RAW_FULL + s), am + 32 * b, k0);
          } else if (BF16 && OP == HNN_FWD && p->im_c > 0) {
            // implicit-GEMM convolution: K block kb = tap (r, s) x 64 channels of the NHWC input,
            // this CTA's 128 output pixels = whole output rows (or images) starting at (b0, oh0)
            // (a split-K tile starts at K block kofs / 64 of the whole problem)
            const int kw = p->im_kw > 0 ? p->im_kw : p->im_k;
            const int kbg = kb + kofs / 64, cbk = p->im_c / 64, tap = kbg / cbk, r = tap / kw, sx = tap - r * kw;
            const int hw = p->im_oh * p->im_ow, b0 = am / hw, oh0 = (am - b0 * hw) / p->im_ow;
            tma_load_4d(st, p->tmap_a, bar(RAW_FULL + s), (kbg - tap * cbk) * 64, sx - p->im_pad, oh0 + r - p->im_pad, b0);
          } else {
            tma_load_2d(st, p->tmap_a, bar(RAW_FULL + s), k0, am);
          }
          if (B_MN) {
            for (int b = 0; b < tn / 64; ++b)
              tma_load_2d(st + TC2_A_BYTES + b * 4096, p->tmap_b, bar(RAW_FULL + s), bn + 32 * b, k0);
          } else if (BF16 && OP == HNN_WGRAD && p->im_c > 0) {
            // implicit weight gradient: this CTA's 64 columns = 64 channels of one tap (r, s) of
            // the NHWC input; the K block = 64 output pixels (whole rows / images) -> MN-major tile
            const int kw = p->im_kw > 0 ? p->im_kw : p->im_k;
            const int tap = bn / p->im_c, c0 = bn - tap * p->im_c, r = tap / kw, sx = tap - r * kw;
            const int hw = p->im_oh * p->im_ow, b0 = k0 / hw, oh0 = (k0 - b0 * hw) / p->im_ow;
            // columns past the last tap (n not a multiple of 128) read an image past the end: zeros
            tma_load_4d(st + TC2_A_BYTES, p->tmap_b, bar(RAW_FULL + s), c0, sx - p->im_pad, oh0 + r - p->im_pad,
                        tap < p->im_k * kw ? b0 : p->im_n);
          } else {
            tma_load_2d(st + TC2_A_BYTES, p->tmap_b, bar(RAW_FULL + s), k0, bn);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: leader CTA, one thread
    if (leader && lane == 0) {
      constexpr uint32_t alb = A_MN ? 4096 : 16, asb = A_MN ? 512 : 1024, alt = A_MN ? 1 : 2;
      constexpr uint32_t blb = B_MN ? 4096 : 16, bsb = B_MN ? 512 : 1024, blt = B_MN ? 1 : 2;
      uint32_t kg = 0, cg = 0, iseq = 0;
      for (int ti = t_begin; ti < t_end; ti += t_step) {
        const int tile = tile_id(ti);
        const hnn_gemm_problem* p;
        int m0, n0, nkb, rows, kofs, sp, tn;
        if (BF16 ? !read_info(iseq++, false, p, m0, n0, nkb, rows, kofs, sp, tn)
               : !tile_info(tile, p, m0, n0, nkb, rows, kofs, sp, tn))
          continue;
        // (bf16 implicit weight gradient: B is MN-major, bit 16)
        const bool b_imp = BF16 && OP == HNN_WGRAD && p->im_c > 0;
        const int ckb = tc2_chunk_kb<OP>(p, nkb);
        const uint32_t idesc =
            BF16 ? (bf16_idesc(2 * TC2_BM, tn) | (b_imp ? (1u << 16) : 0u)) : tf32_idesc(2 * TC2_BM, tn, A_MN, B_MN);
        if (!BF16 && HNN_TC2_LO_FIRST && ckb == 2) {
          // two-block chunks, correction products of BOTH blocks first (the accumulator is still
          // small while they add), then both hi x hi blocks: half the promotions of one-block
          // chunks — each promotion reads the whole 128 x 256 fp32 accumulator out of TMEM, and at
          // one per K block those reads paced the MMAs (tools/tc2_trace.py: MMA thread waiting
          // for a promoted buffer 20-43% of its time, profiles/r02)
          for (int kb = 0; kb < nkb; kb += 2) {
            const int cn = min(2, nkb - kb);
            const uint32_t buf = cg & 1;
            TC2_T0(t1);
            if (cg >= 2) mbar_wait(bar(ACC_EMPTY + buf), ((cg >> 1) - 1) & 1);  // promoted
            TC2_T1(t1, 1);
            const uint32_t acc = tmem + buf * TC2_BN;
            for (int i = 0; i < cn; ++i) {
              const uint32_t kgi = kg + i;
              const int s = kgi % SR, l = kgi % SL;
              const uint32_t a_hi = raw_base + s * TC2_STAGE, b_hi = a_hi + TC2_A_BYTES;
              const uint32_t a_lo = raw_base + (SR + l) * TC2_STAGE, b_lo = a_lo + TC2_A_BYTES;
              TC2_T0(t0);
              mbar_wait(bar(LO_FULL + l), (kgi / SL) & 1);  // both CTAs: raw landed, lo written
              TC2_T1(t0, 0);
              tc_fence_after();
#pragma unroll
              for (int j = 0; j < TC2_BK / 8; ++j) {
                const uint32_t ao = A_MN ? j * 1024 : j * 32, bo = B_MN ? j * 1024 : j * 32;
                mma_tf32_pair(acc, smem_desc(a_lo + ao, alb, asb, alt), smem_desc(b_hi + bo, blb, bsb, blt), idesc,
                              (i | j) != 0);
                mma_tf32_pair(acc, smem_desc(a_hi + ao, alb, asb, alt), smem_desc(b_lo + bo, blb, bsb, blt), idesc, 1u);
              }
              mma_commit_pair(bar(LO_EMPTY + l));  // lo slot l consumed
            }
            for (int i = 0; i < cn; ++i) {
              const int s = (kg + i) % SR;
              const uint32_t a_hi = raw_base + s * TC2_STAGE, b_hi = a_hi + TC2_A_BYTES;
#pragma unroll
              for (int j = 0; j < TC2_BK / 8; ++j) {
                const uint32_t ao = A_MN ? j * 1024 : j * 32, bo = B_MN ? j * 1024 : j * 32;
                mma_tf32_pair(acc, smem_desc(a_hi + ao, alb, asb, alt), smem_desc(b_hi + bo, blb, bsb, blt), idesc, 1u);
              }
              mma_commit_pair(bar(RAW_EMPTY + s));  // raw slot s consumed
            }
            mma_commit_pair(bar(ACC_FULL + buf));
            ++cg;
            kg += cn;
          }
          continue;
        }
        for (int kb = 0; kb < nkb; ++kb, ++kg) {
          const int in_chunk = BF16 ? kb : kb % ckb;  // bf16: one chunk per tile (no promotion)
          const uint32_t buf = cg & 1;
          TC2_T0(t1);
          if (in_chunk == 0 && cg >= 2) mbar_wait(bar(ACC_EMPTY + buf), ((cg >> 1) - 1) & 1);  // promoted
          TC2_T1(t1, 1);
          const int s = kg % SR, l = kg % SL;
          const uint32_t a_hi = raw_base + s * TC2_STAGE, b_hi = a_hi + TC2_A_BYTES;
          const uint32_t a_lo = raw_base + (SR + l) * TC2_STAGE, b_lo = a_lo + TC2_A_BYTES;
          const uint32_t acc = tmem + buf * TC2_BN;
          TC2_T0(t0);
          mbar_wait(bar(LO_FULL + l), (kg / SL) & 1);  // both CTAs: raw landed, lo written
          TC2_T1(t0, 0);
          tc_fence_after();
          if (BF16) {
#pragma unroll
            for (int j = 0; j < 4; ++j)  // K step 16 bf16 = +32 B inside the K-major rows
              mma_f16_pair(acc, smem_desc(a_hi + j * 32, 16, 1024, 2),
                           b_imp ? smem_desc(b_hi + j * 2048, 8192, 1024, 2)  // MN-major: 16 K rows = 2 KB
                                 : smem_desc(b_hi + j * 32, 16, 1024, 2),
                           idesc, (in_chunk | j) != 0);
          } else {
#if HNN_TC2_LO_FIRST
            // correction products first, while the accumulator is still small (the tensor core
            // aligns each MMA's addends to the largest and drops the bits below)
#pragma unroll
            for (int j = 0; j < TC2_BK / 8; ++j) {
              const uint32_t ao = A_MN ? j * 1024 : j * 32, bo = B_MN ? j * 1024 : j * 32;
              mma_tf32_pair(acc, smem_desc(a_lo + ao, alb, asb, alt), smem_desc(b_hi + bo, blb, bsb, blt), idesc,
                            (in_chunk | j) != 0);
              mma_tf32_pair(acc, smem_desc(a_hi + ao, alb, asb, alt), smem_desc(b_lo + bo, blb, bsb, blt), idesc, 1u);
            }
#pragma unroll
            for (int j = 0; j < TC2_BK / 8; ++j) {
              const uint32_t ao = A_MN ? j * 1024 : j * 32, bo = B_MN ? j * 1024 : j * 32;
              mma_tf32_pair(acc, smem_desc(a_hi + ao, alb, asb, alt), smem_desc(b_hi + bo, blb, bsb, blt), idesc, 1u);
            }
#else
#pragma unroll
            for (int j = 0; j < TC2_BK / 8; ++j) {
              const uint32_t ao = A_MN ? j * 1024 : j * 32, bo = B_MN ? j * 1024 : j * 32;
              const uint64_t dah = smem_desc(a_hi + ao, alb, asb, alt), dal = smem_desc(a_lo + ao, alb, asb, alt);
              const uint64_t dbh = smem_desc(b_hi + bo, blb, bsb, blt), dbl = smem_desc(b_lo + bo, blb, bsb, blt);
              mma_tf32_pair(acc, dah, dbh, idesc, (in_chunk | j) != 0);
              mma_tf32_pair(acc, dal, dbh, idesc, 1u);
              mma_tf32_pair(acc, dah, dbl, idesc, 1u);
            }
#endif
          }
          mma_commit_pair(bar(RAW_EMPTY + s));  // raw slot s consumed
          if (!BF16) mma_commit_pair(bar(LO_EMPTY + l));  // lo slot l consumed
          TC2_T1(t0, 5);
          if ((!BF16 && in_chunk == ckb - 1) || kb == nkb - 1) {
            mma_commit_pair(bar(ACC_FULL + buf));
            ++cg;
          }
        }
      }
    }
  } else {
    // ---------------- converters (both CTAs): lo = rna_tf32(x - trunc_tf32(x)); raw stays as hi
    const int ct = threadIdx.x - 64;
    constexpr int CT = 32 * TC2_CONV_WARPS, PER = TC2_STAGE / 16 / CT, NPART = 4, PART = PER / NPART;
    const uint32_t lo_full_leader = map_cluster(bar(LO_FULL), 0);
    uint32_t kg = 0, iseq = 0;
    for (int ti = t_begin; ti < t_end; ti += t_step) {
        const int tile = tile_id(ti);
      const hnn_gemm_problem* p;
      int m0, n0, nkb, rows, kofs, sp, tn;
      if (BF16 ? !read_info(iseq++, true, p, m0, n0, nkb, rows, kofs, sp, tn)
               : !tile_info(tile, p, m0, n0, nkb, rows, kofs, sp, tn))
          continue;
      for (int kb = 0; kb < nkb; ++kb, ++kg) {
        const int s = kg % SR, l = kg % SL;
        TC2_T0(t2);
        mbar_wait(bar(RAW_FULL + s), (kg / SR) & 1);
        if (!BF16 && kg >= SL) mbar_wait(bar(LO_EMPTY + l), ((kg / SL) - 1) & 1);  // lo slot's MMAs done
        TC2_T1(t2, 2);
        const uint32_t hi = raw_base + s * TC2_STAGE, lo = raw_base + (SR + l) * TC2_STAGE;
        const int n16 = BF16 ? 0 : (TC2_A_BYTES + (tn / 2) * TC2_BK * 4) / 16;  // A + B-half 16-byte chunks
#pragma unroll
        for (int h = 0; h < NPART; ++h) {
          if ((h * PART) * CT >= n16) break;
          uint4 v[PART];
#pragma unroll
          for (int u = 0; u < PART; ++u) v[u] = lds128(hi + 16 * (ct + (h * PART + u) * CT));
#pragma unroll
          for (int u = 0; u < PART; ++u) {
            // lo = rna_tf32(x - trunc_tf32(x)) (truncating lo instead moved Adam's first-step
            // weights by 3.3e-4 relative against the oracle: above the per-step tolerance)
            uint4 o;
            o.x = tf32_bits(__float_as_uint(__uint_as_float(v[u].x) - __uint_as_float(v[u].x & 0xFFFFE000u)));
            o.y = tf32_bits(__float_as_uint(__uint_as_float(v[u].y) - __uint_as_float(v[u].y & 0xFFFFE000u)));
            o.z = tf32_bits(__float_as_uint(__uint_as_float(v[u].z) - __uint_as_float(v[u].z & 0xFFFFE000u)));
            o.w = tf32_bits(__float_as_uint(__uint_as_float(v[u].w) - __uint_as_float(v[u].w & 0xFFFFE000u)));
            sts128(lo + 16 * (ct + (h * PART + u) * CT), o);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(lo_full_leader + 8 * l);
      }
    }
  }
  } else {
#if HNN_TC2_REGS_ACC
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(HNN_TC2_REGS_ACC));
#endif
    // ---------------- accumulators + epilogue (warps 4..11): lane quarter warp % 4, column half
    constexpr int HALF = TC2_BN / 2;  // up to 128 columns per warp (tile_n / 2)
    const int aw = warp - 4, q = warp & 3, half = aw >> 2;
    const uint32_t lane_quarter = tmem + (uint32_t(q * 32) << 16);
    const uint32_t stg = epi_base + aw * 4096;
    const uint32_t acc_empty_leader = map_cluster(bar(ACC_EMPTY), 0);
    uint32_t cg = 0, nstore = 0, iseq = 0;
    for (int ti = t_begin; ti < t_end; ti += t_step) {
        const int tile = tile_id(ti);
      const hnn_gemm_problem* p;
      int m0, n0, nkb, rows, kofs, sp, tn;
      TC2_T0(t9);
      if (BF16 ? !read_info(iseq++, true, p, m0, n0, nkb, rows, kofs, sp, tn)
               : !tile_info(tile, p, m0, n0, nkb, rows, kofs, sp, tn))
          continue;
      TC2_T1(t9, 9);
      const int ckb = tc2_chunk_kb<OP>(p, nkb);
      const int nchunks = BF16 ? 1 : (nkb + ckb - 1) / ckb;
      const int hn = tn / 2;  // this warp's columns: [half * hn, half * hn + hn)
      const uint32_t lane_base = lane_quarter + half * hn;
      // Fused plain SGD over a single chunk (K <= 128: C1 / C2 / C5 weight gradients): nothing to
      // promote, so the epilogue reads TMEM block by block and the registers the running sum
      // would hold carry the weights instead, loaded ahead (block 0's before the MMAs finish).
      const bool direct = OP == HNN_WGRAD && nchunks == 1 && p->opt_w != nullptr && p->opt_wm == nullptr;
      if (direct) {
        TC2_T0(t5);
        const uint32_t buf = cg & 1;
        nstore = tc2_sgd_direct(lane_base, buf, bar(ACC_FULL + buf), (cg >> 1) & 1, acc_empty_leader, stg,
                                m0 + int(rank) * TC2_BM + q * 32, n0 + half * hn, hn, p->m, p->n, p->ldc, p->opt_w,
                                p->c, p->tmap_c, cur[p->model].lr, sp, nstore);
        ++cg;
        TC2_T1(t5, 7);
        continue;
      }
      // bf16 (kind::f16, exact products, fp32 accumulation in the tensor core): the whole K is one
      // chunk and the epilogue reads the accumulators straight from TMEM, block by block, releasing
      // the buffer after the last block; fp32 (3xTF32): running sum in registers, promoted per chunk
      float sum[BF16 ? 1 : HALF];
#pragma unroll
      for (int j = 0; j < (BF16 ? 1 : HALF); ++j) sum[j] = 0.0f;  // defined on every path: not live across tiles
      const uint32_t dbuf = cg & 1, dpar = (cg >> 1) & 1;  // (bf16) the tile's accumulator buffer
      // bf16: the wait for the accumulators comes after the problem fields and biases are loaded
      // (their global-memory latency then overlaps the MMAs instead of following them)
      if (BF16) ++cg;
      for (int c = 0; c < (BF16 ? 0 : nchunks); ++c, ++cg) {
        const uint32_t buf = cg & 1;
        TC2_T0(t4);
        mbar_wait(bar(ACC_FULL + buf), (cg >> 1) & 1);
        TC2_T1(t4, 4);
        tc_fence_after();
#pragma unroll
        for (int cb = 0; cb < HALF; cb += TC2_PROMO_COLS) {
          if (cb >= hn) break;
          // TC2_PROMO_COLS columns per TMEM round trip (one tcgen05.wait::ld each)
          uint32_t r0[TC2_PROMO_COLS];
          if (TC2_PROMO_COLS >= 32) {
#pragma unroll
            for (int h = 0; h < TC2_PROMO_COLS / 32; ++h)
              tmem_ld32_nowait(lane_base + buf * TC2_BN + cb + 32 * h, *reinterpret_cast<uint32_t(*)[32]>(r0 + 32 * h));
            tmem_wait_ld();
          } else {
            tmem_ld16(lane_base + buf * TC2_BN + cb, *reinterpret_cast<uint32_t(*)[16]>(r0));
          }
#pragma unroll
          for (int j = 0; j < TC2_PROMO_COLS; ++j)
            sum[cb + j] = (c == 0) ? __uint_as_float(r0[j]) : __fadd_rn(sum[cb + j], __uint_as_float(r0[j]));
        }
        TC2_T1(t4, 6);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acc_empty_leader + 8 * buf);
      }
      TC2_T0(t5);
      // epilogue: this CTA's rows m0 + rank*128 + q*32 + lane, columns n0 + half*128 + cb + j.
      // Problem fields are copied to registers first: the smem stores below carry a "memory"
      // clobber, which would otherwise reload them from global memory per element.
      const int pm = p->m, pn = p->n, ldc = p->ldc;
      const float* bias = p->bias;
      const bool relu = (p->relu & 1) != 0;
      float* const cptr = p->c;
      const void* tmap_c = p->tmap_c;
      const void* xh_out = BF16 ? p->xh_out : nullptr;  // (bf16 NCHW forward: NHWC copy for the next layer)
      const void* tmap_xh = p->tmap_xh;
      float* const ow = p->opt_w;
      float* const owm = p->opt_wm;
      const bool fuse = OP == HNN_WGRAD && ow != nullptr;
      const bool nchw = OP == HNN_FWD && p->c_mode >= 1;  // conv output straight to NCHW (c_mode >= 2: a parity class)
      const float* nmask = nchw ? p->mask : nullptr;
      const int nchw_b = nchw ? (m0 + int(rank) * TC2_BM + q * 32 + lane) / p->row_mult : 0;  // row's sample
      const int nchw_hw = nchw ? (m0 + int(rank) * TC2_BM + q * 32 + lane) - nchw_b * p->row_mult : 0;
      const int hw_n = p->row_mult;
      const Update u = fuse ? make_update(cur[p->model], p->opt_kind, p->opt_momentum) : Update{};
      if (fuse && u.kind == HNN_OPT_ADAM) __trap();  // fused epilogues take SGD / momentum (hnn_b200.h)
      const int row0 = m0 + int(rank) * TC2_BM + q * 32, row = row0 + lane;
      const int nh = n0 + half * hn;
      const bool zero_row = (OP != HNN_WGRAD) && row >= rows;
      float bvp[BF16 ? HALF / 32 : 1];  // (bf16) each 32-column block's bias, lane j = column j
#pragma unroll
      for (int blk = 0; blk < (BF16 ? HALF / 32 : 1); ++blk)
        bvp[blk] = (BF16 && OP == HNN_FWD && bias && blk * 32 < hn && nh + blk * 32 + lane < pn)
                       ? __ldg(bias + nh + blk * 32 + lane)
                       : 0.0f;
      if (BF16) {
        TC2_T0(t4b);
        mbar_wait(bar(ACC_FULL + dbuf), dpar);
        TC2_T1(t4b, 4);
        tc_fence_after();
      }
      const float* mrow = (OP == HNN_DGRAD && p->mask && row < pm) ? p->mask + size_t(row) * ldc : nullptr;
#pragma unroll
      for (int cb = 0; cb < HALF; cb += 32) {
        if (cb >= hn) break;
        if (nh + cb >= pn || row0 >= pm) continue;  // 32 x 32 block outside the problem
        if (lane == 0 && nstore > 0) tma_store_wait_read();  // previous store done reading staging
        __syncwarp();
        // registers (lane = row) -> 128B-swizzled staging (16-byte chunk j of row r at chunk
        // j ^ (r & 7): conflict-free STS.128) -> one TMA store per 32 x 32 block
        const float bv = BF16 ? bvp[(cb / 32) % (BF16 ? HALF / 32 : 1)]  // lane j: column j
                              : ((OP == HNN_FWD && bias && nh + cb + lane < pn) ? __ldg(bias + nh + cb + lane) : 0.0f);
        float tv[32];
        TC2_T0(t10);
        if (BF16) {
          uint32_t r0[16], r1[16];
          tmem_ld16(lane_base + dbuf * TC2_BN + cb, r0);
          tmem_ld16(lane_base + dbuf * TC2_BN + cb + 16, r1);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            tv[j] = __uint_as_float(r0[j]);
            tv[16 + j] = __uint_as_float(r1[j]);
          }
        }
        TC2_T1(t10, 10);
#define TC2_ACC(j) (BF16 ? tv[(j)] : sum[(cb + (j)) % (BF16 ? 1 : HALF)])
        if (nchw) {
          // element (pixel row, filter n) -> y[b][n][hw]: for a fixed n the 32 lanes (rows =
          // consecutive pixels) write consecutive addresses.  NG columns at a time: their relu-mask
          // loads (a conv input gradient as a forward conv of dy) are all issued before any store
          // (interleaved, each load waited behind the previous store: the epilogue was 75% of the
          // dgrad launches' time)
          constexpr int NG = BF16 ? 8 : 2;  // (fp32: the running sum holds 128 registers)
          const bool rok = row < pm;
          // c_mode >= 2: pixel (i, j) of parity class (ph, pw) lands at (2i + ph, 2j + pw) of a
          // 4x larger plane
          const int cm = p->c_mode, par = cm >= 2;
          const int plane = par ? 4 * hw_n : hw_n;
          const int pix = par ? (2 * (nchw_hw / p->im_ow) + ((cm - 2) >> 1)) * 2 * p->im_ow + 2 * (nchw_hw % p->im_ow) +
                                    ((cm - 2) & 1)
                              : nchw_hw;
          const size_t ybase = rok ? size_t(nchw_b) * pn * plane + pix : 0;
          if (BF16 && cm == 1 && (hw_n & 31) == 0) {  // (bf16 convs; fp32 keeps the direct stores)
            // whole 32-pixel runs of one image: stage the block as [channel][pixel] (for a fixed
            // channel the lanes write consecutive words) and store it with one 3D TMA box
            // {32 pixels, 32 channels, 1 image}; rows / channels past the tensor are clipped
#pragma unroll
            for (int g = 0; g < 32 / NG; ++g) {
              float mk[NG];
#pragma unroll
              for (int jj = 0; jj < NG; ++jj) {
                const int n = nh + cb + g * NG + jj;
                mk[jj] = (nmask && rok && n < pn) ? __ldg(nmask + ybase + size_t(n) * plane) : 1.0f;
              }
#pragma unroll
              for (int jj = 0; jj < NG; ++jj) {
                float x = TC2_ACC(g * NG + jj);
                const float b = __shfl_sync(0xffffffffu, bv, g * NG + jj);  // column's bias
                if (zero_row) x = 0.0f;
                else {
                  x = __fadd_rn(x, b);
                  if (relu) x = np_relu(x);
                }
                sts32(stg + (g * NG + jj) * 128 + lane * 4, nmask ? (zero_row ? 0.0f : np_mask(x, mk[jj])) : x);
              }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) tma_store_3d(tmap_c, stg, row0 % hw_n, nh + cb, row0 / hw_n);
            ++nstore;
            if (xh_out) {
              // the next layer's NHWC bf16 input: the same 32 x 32 block as [pixel][channel] rows
              // (64 bytes per pixel) once the NCHW store has read the staging block
              if (lane == 0) tma_store_wait_read();
              __syncwarp();
#pragma unroll
              for (int j8 = 0; j8 < 4; ++j8) {
                uint32_t w[4];
#pragma unroll
                for (int h2 = 0; h2 < 4; ++h2) {
                  float y2[2];
#pragma unroll
                  for (int e = 0; e < 2; ++e) {
                    const int jj = j8 * 8 + h2 * 2 + e;
                    float x = TC2_ACC(jj);
                    const float b = __shfl_sync(0xffffffffu, bv, jj);
                    if (zero_row) x = 0.0f;
                    else {
                      x = __fadd_rn(x, b);
                      if (relu) x = np_relu(x);
                    }
                    y2[e] = x;
                  }
                  const __nv_bfloat162 pr = __floats2bfloat162_rn(y2[0], y2[1]);
                  w[h2] = *reinterpret_cast<const uint32_t*>(&pr);
                }
                sts128(stg + lane * 64 + j8 * 16, make_uint4(w[0], w[1], w[2], w[3]));
              }
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) tma_store_2d(tmap_xh, stg, nh + cb, row0);
              ++nstore;
            }
            continue;
          }
#pragma unroll
          for (int g = 0; g < 32 / NG; ++g) {
            float mk[NG];
#pragma unroll
            for (int jj = 0; jj < NG; ++jj) {
              const int n = nh + cb + g * NG + jj;
              mk[jj] = (nmask && rok && n < pn) ? __ldg(nmask + ybase + size_t(n) * plane) : 1.0f;
            }
#pragma unroll
            for (int jj = 0; jj < NG; ++jj) {
              const int n = nh + cb + g * NG + jj;
              float x = TC2_ACC(g * NG + jj);
              const float b = __shfl_sync(0xffffffffu, bv, g * NG + jj);  // column's bias
              if (zero_row) x = 0.0f;
              else {
                x = __fadd_rn(x, b);
                if (relu) x = np_relu(x);
              }
              if (rok && n < pn) cptr[ybase + size_t(n) * plane] = nmask ? (zero_row ? 0.0f : np_mask(x, mk[jj])) : x;
            }
          }
          continue;
        }
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          float v[4], mv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
          if (OP == HNN_DGRAD && mrow) {  // this row's relu mask, 4 columns
            const int n = nh + cb + j4 * 4;
            if (n + 3 < pn && (ldc & 3) == 0) {
              const float4 m4 = __ldg(reinterpret_cast<const float4*>(mrow + n));
              mv[0] = m4.x; mv[1] = m4.y; mv[2] = m4.z; mv[3] = m4.w;
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) mv[e] = n + e < pn ? __ldg(mrow + n + e) : 0.0f;
            }
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int jj = j4 * 4 + e;
            float x = TC2_ACC(jj);
            if (OP == HNN_FWD) {
              const float b = __shfl_sync(0xffffffffu, bv, jj);  // column jj's bias
              if (zero_row) x = 0.0f;
              else {
                x = __fadd_rn(x, b);  // columns >= n are clipped by the TMA store
                if (relu) x = np_relu(x);
              }
            } else if (OP == HNN_DGRAD) {
              if (zero_row) x = 0.0f;
              else if (mrow) x = np_mask(x, mv[e]);
            }
            v[e] = x;
          }
          sts128(stg + lane * 128 + ((j4 ^ (lane & 7)) << 4),
                 make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3])));
        }
        __syncwarp();
        if (fuse) {
          // fused optimizer: lane = column, so W / moment accesses of a row are one coalesced
          // 128-byte transaction; the gradient comes back out of the swizzled staging block
          // 8 rows at a time: their weight / moment loads are all in flight together (a row-by-row
          // loop serialised one HBM round trip per row: 130 us for C5's weight gradients)
          const int n = nh + cb + lane;
          if (n < pn) {
            const int rmax = min(32, pm - row0);
            if (!owm) {  // plain SGD: 16 rows' weights in flight at once
              for (int r16 = 0; r16 < rmax; r16 += 16) {
                float w[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                  w[i] = r16 + i < rmax ? ow[size_t(row0 + r16 + i) * ldc + n] : 0.0f;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const int rr = r16 + i;
                  if (rr >= rmax) break;
                  const float g = lds32(stg + rr * 128 + ((((lane >> 2) ^ (rr & 7))) << 4) + ((lane & 3) << 2));
                  ow[size_t(row0 + rr) * ldc + n] = __fsub_rn(w[i], __fmul_rn(u.lr, g));
                }
              }
            } else {  // momentum: 8 rows' weights + velocities in flight
              for (int r8 = 0; r8 < rmax; r8 += 8) {
                float w[8], mm[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const size_t off = size_t(row0 + r8 + i) * ldc + n;
                  const bool in = r8 + i < rmax;
                  w[i] = in ? ow[off] : 0.0f;
                  mm[i] = in ? owm[off] : 0.0f;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const int rr = r8 + i;
                  if (rr >= rmax) break;
                  const float g = lds32(stg + rr * 128 + ((((lane >> 2) ^ (rr & 7))) << 4) + ((lane & 3) << 2));
                  const size_t off = size_t(row0 + rr) * ldc + n;
                  update_sgd(u, w[i], g, mm[i]);
                  ow[off] = w[i];
                  owm[off] = mm[i];
                }
              }
            }
          }
          __syncwarp();
        }
        if (cptr != nullptr) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) tma_store_2d(tmap_c, stg, nh + cb, row0 + sp * ((pm + 31) & ~31));  // split sp's rows
          ++nstore;
        }
      }
#undef TC2_ACC
      if (BF16) {  // accumulators read: the buffer goes back to the MMA issuer
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acc_empty_leader + 8 * dbuf);
      }
      TC2_T1(t5, 7);
    }
    if (lane == 0) tma_store_wait_all();
  }
  TC2_T0(t6);
  tc_fence_before();
  __syncthreads();
  TC2_T1(t6, 8);
#ifdef HNN_TC2_TRACE
  if (threadIdx.x == 0) g_tc2_trace[blockIdx.x * 16 + 15] += clock64() - t_start;
  if ((threadIdx.x & 31) == 0)
    for (int i = 0; i < 11; ++i)
      if (tr[i]) atomicAdd(&g_tc2_trace[blockIdx.x * 16 + i], (unsigned long long)tr[i]);
#endif
  cluster_sync_all();  // the leader's MMAs into the peer's TMEM are complete
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int gemm_tc2_chunk_terms() { return TC2_CHUNK_KB * TC2_BK; }

int gemm_tc2_tile_shape(int op, int32_t* tm, int32_t* tn) {
  *tm = 2 * TC2_BM;
  *tn = TC2_BN;
  return HNN_OK;
}

int launch_colsum(const hnn_gemm_problem* probs, int nprob, const hnn_step_row* cur, const hnn_model_status* status,
                  cudaStream_t s);

template <int KIND>
int launch_tc2(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
               const hnn_model_status* status, cudaStream_t s) {
  static bool configured[3] = {false, false, false};
  if (!configured[op]) {
    cudaError_t e;
    if (op == HNN_FWD) e = cudaFuncSetAttribute(gemm_tc2_kernel<HNN_FWD, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC2_SMEM_BYTES);
    else if (op == HNN_DGRAD) e = cudaFuncSetAttribute(gemm_tc2_kernel<HNN_DGRAD, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC2_SMEM_BYTES);
    else e = cudaFuncSetAttribute(gemm_tc2_kernel<HNN_WGRAD, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC2_SMEM_BYTES);
    if (e != cudaSuccess) {
      set_error("hnn_grouped_gemm(tc2)", cudaGetErrorString(e));
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
  int pairs = total_tiles < sms / 2 ? total_tiles : sms / 2;
  if (const char* g = getenv("HNN_TC2_PAIRS")) pairs = std::max(1, std::min(pairs, atoi(g)));  // (probe: SM share)
  const int grid = 2 * pairs;
  if (op == HNN_FWD)
    hnn::launch_pdl(gemm_tc2_kernel<HNN_FWD, KIND>, dim3(grid), dim3(TC2_THREADS), TC2_SMEM_BYTES, s, probs, nprob, total_tiles, cur, status);
  else if (op == HNN_DGRAD)
    hnn::launch_pdl(gemm_tc2_kernel<HNN_DGRAD, KIND>, dim3(grid), dim3(TC2_THREADS), TC2_SMEM_BYTES, s, probs, nprob, total_tiles, cur, status);
  else {
    hnn::launch_pdl(gemm_tc2_kernel<HNN_WGRAD, KIND>, dim3(grid), dim3(TC2_THREADS), TC2_SMEM_BYTES, s, probs, nprob, total_tiles, cur, status);
    int rc = check_launch("hnn_grouped_gemm(tc2)");
    if (rc) return rc;
    return launch_colsum(probs, nprob, cur, status, s);
  }
  return check_launch("hnn_grouped_gemm(tc2)");
}

int grouped_gemm_tc2(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                     const hnn_model_status* status, cudaStream_t s) {
  return launch_tc2<0>(op, probs, nprob, total_tiles, cur, status, s);
}

int grouped_gemm_bf16(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                      const hnn_model_status* status, cudaStream_t s) {
  return launch_tc2<1>(op, probs, nprob, total_tiles, cur, status, s);
}

}  // namespace hnn

#ifdef HNN_TC2_TRACE
extern "C" int hnn_debug_tc2_trace(void* host_out, int reset) {
  cudaMemcpyFromSymbol(host_out, hnn::g_tc2_trace, sizeof(hnn::g_tc2_trace));
  if (reset) {
    static unsigned long long zeros[296 * 16] = {};
    cudaMemcpyToSymbol(hnn::g_tc2_trace, zeros, sizeof(zeros));
  }
  return 0;
}
#endif
