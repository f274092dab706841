// K1 (fp32), production variant: 3xTF32 strided batched GEMM on
// tcgen05.mma.cta_group::2 (UMMA 256 x 256), TMA-fed, persistent.
//
//   C = alpha * (A_hi B_hi + A_hi B_lo + A_lo B_hi) + beta * C
//
// The tensor core TRUNCATES fp32 operands to TF32 (measured: feeding the raw
// fp32 tile as "hi" together with lo = x - trunc(x) reproduces the explicit
// split to the last bit of accuracy, while lo = x - rna(x) does not).  So the
// raw tile that TMA lands in shared memory IS the hi operand, and only the
// residual lo = x - (x & ~0x1fff) has to be produced -- two ALU ops per
// element, written at the same (swizzled) offset, so the converter never needs
// to know the layout.
//
// Operand staging is in place at the operands' strides: a 4-D TMA tensor map
// (contiguous mode, other mode, batch, batch2) per operand; K-major operands
// use 128 B swizzle, MN-major ones 128 B swizzle with 32 B atoms (the only
// MN-major layout UMMA accepts for tf32).  TMA zero-fills every M/N/K tail.
//
// CTA pair: each CTA holds its 128 rows of A and 128 of B's 256 columns; the
// leader issues M=256 MMAs reading both CTAs' smem.  SPLIT_ACC keeps the two
// small cross terms in a second TMEM accumulator: the tensor core truncates on
// every accumulate, so folding 2^-11-sized terms into the main accumulator
// would cost a full ulp(acc) each; with the split the error of K=1024 sums
// drops ~3x.  (Two accumulators use all 512 TMEM columns, so SPLIT_ACC runs
// with a single accumulator buffer; the default double-buffers instead.)
//
// Warp roles per CTA (14 warps): 0-3 epilogue, 4-11 lo converters (two groups
// of 4 warps taking alternate K-blocks, so each has two K-blocks of time),
// 12 TMA producer + TMEM allocator, 13 MMA issuer (leader).
//
// Problem sets: the kernel walks the tiles of up to MAXP independent problems
// (each with its own operands, strides, K-major / MN-major layouts, fold and
// tensor maps, passed by value in the kernel parameters) in one persistent
// launch.  A single contraction is MAXP = 1; a group of independent
// contractions (e.g. the 36-case sweep) shares one pipeline fill, one drain
// and one tile-quantisation tail instead of paying them per contraction.
//
// Unbiased narrow tiles (FLUSH: BNT <= 64 with split accumulators, the
// HBM-bound rank-r products of Tucker/HOOI).  Two biases of the default path
// matter when such products are chained and their norms compared (the HOOI
// fit, reference tucker.py:164-167): (1) the raw tile used as hi is x
// truncated, so the residual that the tensor core truncates again is always of
// x's sign -- every operand is shrunk by ~2^-22 on average; (2) the main
// accumulator is truncated on every MMA, a shrink of ~K/16 ulp for coherent
// sums.  FLUSH removes both: the converters write lo = rna_tf32(x - trunc(x))
// (the rounding of the residual is now unbiased), and the hi*hi MMA of
// every group of G K=8 steps writes a FRESH TMEM step accumulator (8 rotating
// slots) that the epilogue warps add into registers in round-to-nearest fp32,
// in k order; the 2^-11-sized cross terms keep their own accumulator.  The
// tiles are HBM-paced (~700 cycles per K-block), so the extra TMEM loads and
// adds are hidden.
//
// Batch-blocked A (BB, the exceptional cases, reference kernels.py:179-204):
// the A operand is unit-stride along the BATCH mode (apt = 1) while C is
// unit-stride along m.  Each CTA's 128 MMA rows are (4 consecutive batch
// entries) x (32 consecutive m): row r = b_l + 4 m_l.  Per 32-row MN atom one
// dense 3-D TMA box (4 batch, 8 m, BK k) lands as [k][m8][b4]: 128 B of MN per
// k row, the MN-major SW128_BASE32B atom minus its swizzle (TMA cannot swizzle
// a 16-byte-wide box; UMMA takes no unswizzled MN-major tf32).  The converter
// warps, which read every raw element anyway to form lo, write A_hi and A_lo
// at the swizzled offset (16-byte chunks move whole: off ^ ((off>>7)&3)<<5),
// so the permutation costs one extra 16 KB smem write per K-block, and in
// the epilogue a
// warp's 32 lanes are 8 consecutive m x 4 batch entries: every store
// instruction writes four full 32-byte sectors of C instead of 32 scattered
// 4-byte words.  B must not depend on the batch (bps = 0).
#pragma once
#include <cuda.h>

#include <type_traits>

#include "sbt_common.cuh"
#include "sm100_ptx.cuh"

namespace sbt {
namespace tf32tma {

constexpr int BM = 256, BN = 256, HM = 128, HN = 128;
constexpr int kThreads = 14 * 32;
constexpr int kConvWarps = 8;                      // two groups of 4, alternating K-blocks
constexpr int kGroupWarps = 4;

// K-block depth BK (32: 128 B rows, SW128; 16: 64 B rows, SW64).  Raw (TMA) ring
// and lo ring share 192 KB: raw slots are held from TMA issue to MMA
// retirement, lo slots only from conversion to MMA retirement, so the raw ring
// is the deeper one; a smaller BK gives more, finer slots in flight.
// BB: the converted slot also holds A_hi (the converter re-lays the dense raw
// A box into the swizzled MN-major atom), so it is 3 operand halves wide.
// BNT: tile width (N of the MMA): 256, or 128 / 64 / 32 for narrow problems
// (each CTA holds BNT/2 columns of B; narrow accumulators leave TMEM room for
// double-buffered split accumulators).  BNT = 32 serves the rank-32 Tucker
// products (M' = 262144, N = 32), which are HBM-bound: the MMA's shared-memory
// reads per flop grow as N shrinks, but the tile still outruns HBM.
template <int BK, bool BB = false, int BNT = 256, int EPIB = 2>
struct Geo {
  static constexpr int A_BYTES = 128 * BK * 4;               // A half (128 rows)
  static constexpr int B_BYTES = (BNT / 2) * BK * 4;         // B half (BNT/2 columns)
  static constexpr int OP_BYTES = A_BYTES;
  static constexpr int SLOT_BYTES = A_BYTES + B_BYTES;       // raw A half + raw B half
  static constexpr int LO_SLOT_BYTES = SLOT_BYTES + (BB ? A_BYTES : 0);
  // The lo ring bounds how far conversion runs ahead of the MMAs: a lo slot
  // cycles through MMA retire -> commit -> converter -> full barrier (both
  // CTAs) -> MMA issue, ~2.4K cycles measured (SBT_TRACE).  Wide tiles spend
  // 1536 cycles of MMA per K-block, so 2 slots cover it; narrow tiles are
  // HBM-paced (~700 cycles per K-block at BNT = 32), where 3 lo slots keep the
  // converters ahead and leave 7 raw slots for TMA depth (measured on the
  // 512^3 rank-32 Tucker products: 2 / 3 / 4 / 5 lo slots = 5.2 / 5.7 / 5.3 /
  // 5.0 TB/s).
#ifndef SBT_LO_NARROW
#define SBT_LO_NARROW 3
#endif
#ifndef SBT_LO_128
#define SBT_LO_128 3
#endif
  static constexpr int LO_SLOTS =
      (BK == 32 ? 1 : 2) * (BNT >= 256 ? 2 : BNT >= 128 ? SBT_LO_128 : SBT_LO_NARROW);
  // epilogue staging for the TMA-store epilogue: EPIB x (128 rows x 32
  // columns).  Each buffer is one TMA store in flight: short-K tiles (K <= 128,
  // e.g. the 4th-order contraction) are bound by the C writes, which need ~64 KB
  // in flight per SM, so they take 4 buffers at the price of raw-ring depth
  static constexpr int EPI_BYTES = BB ? 0 : EPIB * 128 * 32 * 4;
  // as many raw slots as fit in 227 KB: TMA latency under load is ~4.3K cycles
  // (measured), ~3 K-blocks of MMA time, and a raw slot stays held until the
  // MMAs that read it retire
  static constexpr int RAW_SLOTS =
      (232448 - 1024 - 512 - LO_SLOTS * LO_SLOT_BYTES - EPI_BYTES) / SLOT_BYTES;
  static constexpr int SMEM_BYTES =
      RAW_SLOTS * SLOT_BYTES + LO_SLOTS * LO_SLOT_BYTES + EPI_BYTES + 1024 + 512;
  static constexpr uint32_t TX = SLOT_BYTES;                 // raw A + raw B per K-block
  static constexpr int NV = SLOT_BYTES / 16 / 128;           // float4 per converter thread
  static_assert(SLOT_BYTES % (16 * 128) == 0, "converter chunks");
  static_assert(RAW_SLOTS <= 16 && LO_SLOTS <= 16, "barrier area");
  static_assert(RAW_SLOTS >= 3, "TMA depth");
};

// Debug timeline (SBT_TRACE builds only): per-event clock64 stamps of pair 0.
#ifdef SBT_TRACE
__device__ long long g_trace[8][4096];
#define TRACE(row, idx) do { if (blockIdx.x < 2 && (idx) < 4096) g_trace[(row) + 4 * rank][(idx)] = clock64(); } while (0)
__device__ long long g_trace_epi[2][64][4];
__device__ long long g_trace_mma[64][2];       // per tile: accumulator acquired, last commit
__device__ long long g_trace_tepi[2][64][8];   // TMA-store epilogue: wait, acquired, released, end, phase sums
__device__ long long g_trace_flush[2][4096];   // FLUSH: epilogue warp 0 got step group eg
#else
#define TRACE(row, idx) do { } while (0)
#endif

struct Tile {
  int64_t m0, n0, pb, qb;
};
// Batch folding: a batch mode that only one operand (and C) depends on can be
// folded into that operand's MMA dimension when the dimension is a multiple of
// the CTA block (128): M' = m x batch_X rows, row r' = (r' % m, x = r' / m),
// each CTA's 128 rows inside one x.  This turns e.g. the 4th-order contraction
// C[mnpq] = A[mkp] B[nkq] (m = n = 128, two batch modes: the planner's
// LoopStep fused as batch2) into one 16384 x 16384 x 128 GEMM of full 256x256
// tiles instead of 16384 half-empty 128x128 ones.
struct Fold {
  int64_t m_in, n_in;  // inner extents (p.m, p.n)
  int64_t mtot, ntot;  // folded extents M', N'
  int fm, fn;          // 0 = none, 1 = folds `batch`, 2 = folds `batch2`
  // epilogue: 0 = direct st.global; TMA store through smem staging with the C
  // tensor map over (1) rows contiguous (crs = 1) or (2) columns contiguous
  int cmode;
};

// One problem of a set.  Tensor maps first (64-byte aligned).
struct Problem {
  CUtensorMap ta, tb, tc;
  GemmParams<float> p;
  Fold f;
  int64_t tiles_m, tiles_n, nbatch;  // tile grid (nbatch: batch units the tiles run over)
  int64_t tile_begin;                // first global tile index of this problem
  int a_k, b_k;                      // operand majorness: 1 = K-major
  int nkb;                           // K-blocks per tile
  int pad;
};
template <int MAXP>
struct ProblemSet {
  Problem pr[MAXP];
  int64_t total;  // tiles over all problems
  int n;
};

// problem owning global tile t; `cur` only moves forward (every role walks
// its tiles in increasing order)
__device__ __forceinline__ const Problem& locate(const Problem* pr, int n, int64_t t, int& cur) {
  while (cur + 1 < n && t >= pr[cur + 1].tile_begin) ++cur;
  return pr[cur];
}

// BB tiles cover 64 m (32 per CTA) x 4 batch entries; pb is then the batch group
template <bool BB = false, int BNT = BN>
__device__ __forceinline__ Tile tile_of(int64_t t, int64_t tiles_m, int64_t tiles_n,
                                        int64_t batch) {
  Tile c;
  c.m0 = (t % tiles_m) * (BB ? 64 : BM);
  t /= tiles_m;
  c.n0 = (t % tiles_n) * BNT;
  t /= tiles_n;
  c.pb = t % batch;
  c.qb = t / batch;
  return c;
}

// TMA loads of one operand half (ROWS = 128 or 64 rows/cols of the MMA
// dimension x BK k).  K-major: one box (BK k, ROWS mn).  MN-major: ROWS/32 boxes
// (32 mn, BK k), one per 32-wide MN atom column, each a contiguous slab of BK
// 128-byte rows.  PREFETCH: the same boxes as L2 prefetches (no smem).
template <int BK, bool PREFETCH = false, int ROWS = 128>
__device__ __forceinline__ void tma_operand(bool kmaj, const CUtensorMap* tm, uint8_t* dst,
                                            uint64_t* bar, int64_t mn0, int64_t k0, int64_t b,
                                            int64_t b2, bool bcast, bool bcast2) {
  const int cb = bcast ? 0 : int(b), cb2 = bcast2 ? 0 : int(b2);
  if (kmaj) {
    if (PREFETCH) ptx::tma_prefetch_4d(tm, int(k0), int(mn0), cb, cb2);
    else ptx::tma_load_4d(dst, tm, bar, int(k0), int(mn0), cb, cb2);
  } else {
#pragma unroll
    for (int c = 0; c < ROWS / 32; ++c) {
      if (PREFETCH) ptx::tma_prefetch_4d(tm, int(mn0 + 32 * c), int(k0), cb, cb2);
      else ptx::tma_load_4d(dst + c * (BK * 128), tm, bar, int(mn0 + 32 * c), int(k0), cb, cb2);
    }
  }
}

// FLUSH configuration (see the header): step-accumulator slots after the
// NBUF x ACC_W accumulator columns
template <bool SPLIT_ACC, bool BB, int BNT>
struct FlushCfg {
  static constexpr bool ON = SPLIT_ACC && !BB && BNT <= 64;
  static constexpr int ACC_W = (SPLIT_ACC ? 2 : 1) * BNT;
  static constexpr int NBUF = 512 / ACC_W >= 2 ? 2 : 1;
  static constexpr int BASE = NBUF * ACC_W;
  static constexpr int NSLOT = ON ? ((512 - BASE) / BNT < 12 ? (512 - BASE) / BNT : 12) : 1;
};

template <int MAXP, bool SPLIT_ACC, int BK, bool BB = false, int BNT = 256, int EPIB = 2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
tf32x3_pair_tma_kernel(const __grid_constant__ ProblemSet<MAXP> ps, int p_prefetch) {
  const Problem* __restrict__ prs = ps.pr;
  const int nprob = ps.n;
  const int64_t total = ps.total;
  // problem of global tile t; a single-problem launch indexes ps.pr[0] at
  // compile time so its fields stay in the constant bank / uniform registers
  auto prob = [&](int64_t t, int& cur) -> const Problem& {
    if constexpr (MAXP == 1) { (void)t; (void)cur; return ps.pr[0]; }
    else return locate(prs, nprob, t, cur);
  };
  using Gm = Geo<BK, BB, BNT, EPIB>;
  constexpr int HNT = BNT / 2;  // B columns per CTA (MN-major B needs HNT >= 32: host-checked)
  constexpr int RAW_SLOTS = Gm::RAW_SLOTS, LO_SLOTS = Gm::LO_SLOTS;
  constexpr int OP_BYTES = Gm::OP_BYTES, SLOT_BYTES = Gm::SLOT_BYTES;
  constexpr int LO_SLOT_BYTES = Gm::LO_SLOT_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* raw_ring = smem;
  uint8_t* lo_ring = smem + RAW_SLOTS * SLOT_BYTES;
  uint8_t* epi_stage = smem + RAW_SLOTS * SLOT_BYTES + LO_SLOTS * LO_SLOT_BYTES;  // 1 KB aligned
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(epi_stage + Gm::EPI_BYTES);
  uint64_t* raw_empty = raw_full + RAW_SLOTS;
  uint64_t* full = raw_empty + RAW_SLOTS;         // converted (leader's copy is the one used)
  uint64_t* lo_empty = full + RAW_SLOTS;
  uint64_t* acc_full = lo_empty + LO_SLOTS;
  uint64_t* acc_empty = acc_full + 2;
  using FC = FlushCfg<SPLIT_ACC, BB, BNT>;
  constexpr bool FLUSH = FC::ON;
  constexpr int NSLOT = FC::NSLOT;
  uint64_t* step_full = acc_empty + 2;           // FLUSH step accumulators
  uint64_t* step_empty = step_full + NSLOT;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(step_empty + NSLOT);
  static_assert((3 * RAW_SLOTS + LO_SLOTS + 4 + 2 * NSLOT) * 8 + 4 <= 512, "barrier area");
  // FLUSH: K=8 steps per step-accumulator group (1, 2, 4 or 8; log2 in bits 12-13)
  const int flush_lg = (p_prefetch >> 12) & 3;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t rank = ptx::cluster_rank();
  const int64_t pair = blockIdx.x >> 1;
  const int64_t npairs = gridDim.x >> 1;
  // TMEM: NBUF buffers of (main [+ small]) BNT-column accumulators in 512 columns
  constexpr int ACC_W = (SPLIT_ACC ? 2 : 1) * BNT;
  constexpr int NBUF = 512 / ACC_W >= 2 ? 2 : 1;

  if (warp == 12) {
    if (lane == 0) {
      for (int s = 0; s < RAW_SLOTS; ++s) {
        ptx::mbar_init(&raw_full[s], 1);
        ptx::mbar_init(&raw_empty[s], 1);
        ptx::mbar_init(&full[s], 2 * kGroupWarps);
      }
      for (int s = 0; s < LO_SLOTS; ++s) ptx::mbar_init(&lo_empty[s], 1);
      for (int b = 0; b < 2; ++b) {
        ptx::mbar_init(&acc_full[b], 1);
        ptx::mbar_init(&acc_empty[b], 2 * 4);  // one arrival per epilogue warp of each CTA
      }
      for (int s = 0; s < NSLOT; ++s) {
        ptx::mbar_init(&step_full[s], 1);
        ptx::mbar_init(&step_empty[s], 2 * 4);
      }
      ptx::fence_mbarrier_init();
      for (int i = 0; i < nprob; ++i) {
        ptx::prefetch_tmap(&prs[i].ta);
        ptx::prefetch_tmap(&prs[i].tb);
        if (!BB && prs[i].f.cmode) ptx::prefetch_tmap(&prs[i].tc);
      }
    }
    __syncwarp();
    ptx::tmem_alloc2(tmem_slot, 512);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 12) {
    {
      // -------------------------------------------------------- TMA producer
      // warp-uniform loop (coordinates in uniform registers); one elected lane
      // issues the TMA boxes
      // Per-tile TMA coordinates, decoded once per tile
      struct Coord {
        const Problem* pr;
        int am, ab, ab2, bn, bb, bb2;
        int qm[4], qb[4], qb2[4];  // MN-major A: the four 32-row boxes (fold per box)
      };
      auto decode = [&](int64_t tile_idx, int& cur) {
        const Problem& P = prob(tile_idx, cur);
        const GemmParams<float>& p = P.p;
        const Fold& f = P.f;
        const bool a_bc = p.aps == 0, a_bc2 = p.aps2 == 0, b_bc = p.bps == 0, b_bc2 = p.bps2 == 0;
        const Tile tc = tile_of<BB, BNT>(tile_idx - P.tile_begin, P.tiles_m, P.tiles_n, P.nbatch);
        Coord c;
        c.pr = &P;
        if (BB) {
          c.am = int(tc.m0 + rank * 32); c.ab = int(tc.pb * 4); c.ab2 = a_bc2 ? 0 : int(tc.qb);
          c.bn = int(tc.n0 + rank * HNT); c.bb = b_bc ? 0 : int(tc.pb); c.bb2 = b_bc2 ? 0 : int(tc.qb);
          return c;
        }
        // (un)fold: CTA row / column block -> (inner index, folded batch index)
        int64_t am = tc.m0 + rank * HM, ab = tc.pb, ab2 = tc.qb;
        if (f.fm) {
          const int64_t x = am / f.m_in;
          am -= x * f.m_in;
          if (f.fm == 1) ab = x; else ab2 = x;
        }
        int64_t bn = tc.n0 + rank * HNT, bb = tc.pb, bb2 = tc.qb;
        if (f.fn) {
          const int64_t y = bn / f.n_in;
          bn -= y * f.n_in;
          if (f.fn == 1) bb = y; else bb2 = y;
        }
        c.am = int(am); c.ab = a_bc ? 0 : int(ab); c.ab2 = a_bc2 ? 0 : int(ab2);
        c.bn = int(bn); c.bb = b_bc ? 0 : int(bb); c.bb2 = b_bc2 ? 0 : int(bb2);
        // MN-major A loads 32-row boxes: with a fold of m_in < 128 rows (a
        // multiple of 32) consecutive boxes belong to different batch entries
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int64_t qm = am + 32 * q, qx = 0;
          if (f.fm && qm >= f.m_in) {
            qx = qm / f.m_in;
            qm -= qx * f.m_in;
          }
          c.qm[q] = int(qm);
          c.qb[q] = (f.fm == 1 && !a_bc) ? int(ab + qx) : c.ab;
          c.qb2[q] = (f.fm == 2 && !a_bc2) ? int(ab2 + qx) : c.ab2;
        }
        return c;
      };
      // issue the TMA boxes of one K-block: into raw slot st (PF = false) or
      // as L2 prefetches (PF = true, st unused)
      auto boxes = [&](const Coord& c, int k0, uint8_t* st, uint64_t* bar, auto pf) {
        constexpr bool PF = decltype(pf)::value;
        const CUtensorMap* tmA = &c.pr->ta;
        if (BB) {  // four dense (4 batch, 8 m, BK k) boxes [k][m8][b4], one per MN atom
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (PF) ptx::tma_prefetch_4d(tmA, c.ab, c.am + 8 * q, k0, c.ab2);
            else ptx::tma_load_4d(st + q * (BK * 128), tmA, bar, c.ab, c.am + 8 * q, k0, c.ab2);
          }
        } else if (c.pr->a_k) {
          tma_operand<BK, PF>(true, tmA, st, bar, c.am, k0, c.ab, c.ab2, false, false);
        } else {  // MN-major A: four 32-row boxes [32 m][BK k]
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (PF) ptx::tma_prefetch_4d(tmA, c.qm[q], k0, c.qb[q], c.qb2[q]);
            else ptx::tma_load_4d(st + q * (BK * 128), tmA, bar, c.qm[q], k0, c.qb[q], c.qb2[q]);
          }
        }
        tma_operand<BK, PF, HNT>(c.pr->b_k, &c.pr->tb, st + Gm::A_BYTES, bar, c.bn, k0, c.bb,
                                 c.bb2, false, false);
      };
      // L2 prefetch distance (K-blocks ahead of the smem ring)
      const int pfd = p_prefetch & 0xff;
      const bool dbg_no_tma = (p_prefetch >> 8) & 1;  // diagnostics: MMA/convert loop only
      int64_t pf_tile = pair;       // prefetch cursor (tile, k-block)
      int pf_kb = 0, pf_cur = 0, cur = 0;
      Coord pf_c{};
      if (pf_tile < total) pf_c = decode(pf_tile, pf_cur);
      auto prefetch_next = [&]() {
        if (pf_tile >= total) return;
        boxes(pf_c, pf_kb * BK, nullptr, nullptr, std::true_type{});
        if (++pf_kb == pf_c.pr->nkb) {
          pf_kb = 0;
          pf_tile += npairs;
          if (pf_tile < total) pf_c = decode(pf_tile, pf_cur);
        }
      };
      if (ptx::elect_one_sync())
        for (int i = 0; i < pfd; ++i) prefetch_next();
      __syncwarp();
      int64_t g = 0;
      for (int64_t t = pair; t < total; t += npairs) {
        const Coord c = decode(t, cur);
        const int nkb = c.pr->nkb;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const uint32_t s = uint32_t(g % RAW_SLOTS);
          ptx::mbar_wait(&raw_empty[s], (uint32_t(g / RAW_SLOTS) & 1u) ^ 1u);
          TRACE(0, int(g));
          uint8_t* st = raw_ring + s * SLOT_BYTES;
          if (ptx::elect_one_sync()) {
            if (pfd > 0) prefetch_next();
            if (dbg_no_tma) {
              ptx::mbar_arrive(&raw_full[s]);
            } else {
              ptx::mbar_arrive_expect_tx(&raw_full[s], Gm::TX);
              boxes(c, kb * BK, st, &raw_full[s], std::false_type{});
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4 && warp < 4 + kConvWarps) {
    // -------------------------------------------------------- lo converters
    // group c converts K-blocks g = c, c+2, ... into lo slot g % LO_SLOTS
    const int grp = (warp - 4) / kGroupWarps;
    const int ct = tid - 128 - grp * kGroupWarps * 32;  // 0..127
    uint32_t full_leader[RAW_SLOTS];
#pragma unroll
    for (int s = 0; s < RAW_SLOTS; ++s) full_leader[s] = ptx::mapa(&full[s], 0);
    int64_t n_iter = 0;  // K-blocks of this pair's tiles
    {
      int cur = 0;
      for (int64_t t = pair; t < total; t += npairs) n_iter += prob(t, cur).nkb;
    }
    for (int64_t g = grp; g < n_iter; g += kConvWarps / kGroupWarps) {
      const uint32_t s = uint32_t(g % RAW_SLOTS);
      const uint32_t ls = uint32_t(g % LO_SLOTS);
      const uint32_t lo_base = ptx::smem_addr(lo_ring + ls * LO_SLOT_BYTES);
      ptx::mbar_wait(&lo_empty[ls], (uint32_t(g / LO_SLOTS) & 1u) ^ 1u);
      ptx::mbar_wait(&raw_full[s], uint32_t(g / RAW_SLOTS) & 1u);
      if (ct == 0) TRACE(1, int(g));
      const uint32_t raw = ptx::smem_addr(raw_ring + s * SLOT_BYTES);
      constexpr int NV = Gm::NV;  // float4 chunks per thread (A and B halves)
#pragma unroll
      for (int h = 0; h < ((p_prefetch >> 9) & 1 ? 0 : (NV + 3) / 4); ++h) {
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (h * 4 + i < NV) v[i] = ptx::lds_v4(raw + (ct + (h * 4 + i) * 128) * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (h * 4 + i >= NV) continue;
          uint32_t off = (ct + (h * 4 + i) * 128) * 16;
          if (BB && (h * 4 + i) * 128 < Gm::A_BYTES / 16) {  // chunk lies in the A half
            // dense [k][m8][b4] A chunk -> 32 B-atom swizzle (k row % 4 XOR granule)
            off ^= ((off >> 7) & 3u) << 5;
            ptx::sts_v4(lo_base + Gm::SLOT_BYTES + off, __float_as_uint(v[i].x),
                        __float_as_uint(v[i].y), __float_as_uint(v[i].z), __float_as_uint(v[i].w));
          }
          if constexpr (FLUSH) {
            // unbiased split at the cost of one cvt per element: the raw tile
            // stays the hi operand (the tensor core truncates it to trunc(x)),
            // and the exact residual x - trunc(x) -- always of x's sign -- is
            // rounded to TF32 to nearest here instead of truncated by the
            // tensor core.  (Writing hi = rna(x) back into the raw slot as well
            // cost ~150 cycles per K-block at the HBM pace.)
            ptx::sts_v4(lo_base + off, ptx::to_tf32(ptx::tf32_residual(v[i].x)),
                        ptx::to_tf32(ptx::tf32_residual(v[i].y)),
                        ptx::to_tf32(ptx::tf32_residual(v[i].z)),
                        ptx::to_tf32(ptx::tf32_residual(v[i].w)));
          } else {
            ptx::sts_v4(lo_base + off, __float_as_uint(ptx::tf32_residual(v[i].x)),
                        __float_as_uint(ptx::tf32_residual(v[i].y)),
                        __float_as_uint(ptx::tf32_residual(v[i].z)),
                        __float_as_uint(ptx::tf32_residual(v[i].w)));
          }
        }
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) ptx::mbar_arrive(&full[s]);
        else ptx::mbar_arrive_remote(full_leader[s]);
      }
      if (ct == 0) TRACE(2, int(g));
    }
  } else if (warp < 4) {
    // -------------------------------------------------------- epilogue
    const uint32_t lane_addr = uint32_t(warp * 32) << 16;
    const uint32_t empty_leader[2] = {ptx::mapa(&acc_empty[0], 0), ptx::mapa(&acc_empty[1], 0)};
    const int r = warp * 32 + lane;
    const bool leader = (r == 0);
    uint32_t nchunk = 0, tcount = 0;
    uint32_t eg = 0;  // FLUSH: step-accumulator groups consumed (all tiles)
    const uint32_t step_empty_leader = FLUSH ? ptx::mapa(&step_empty[0], 0) : 0u;
    int cur = 0;
    for (int64_t t = pair; t < total; t += npairs, ++tcount) {
      const Problem& P = prob(t, cur);
      const GemmParams<float>& p = P.p;
      const Fold& f = P.f;
      const Tile tc = tile_of<BB, BNT>(t - P.tile_begin, P.tiles_m, P.tiles_n, P.nbatch);
      // FLUSH: sum the tile's hi*hi step accumulators in round-to-nearest fp32
      // (k order), then park the sum in the tile's main accumulator columns,
      // which the MMAs do not write in this mode
      float facc[FLUSH ? BNT : 1];
      if constexpr (FLUSH) {
#pragma unroll
        for (int j = 0; j < BNT; ++j) facc[j] = 0.f;
        const int lg_t = (flush_lg == 3 && (P.nkb & 1)) ? 2 : flush_lg;
        const uint32_t ngroups = uint32_t(P.nkb * (BK / 8)) >> lg_t;
#pragma unroll 1
        for (uint32_t gi = 0; gi < ngroups; ++gi, ++eg) {
          const uint32_t slot = eg % NSLOT;
          ptx::mbar_wait(&step_full[slot], (eg / NSLOT) & 1u);
          ptx::tc_fence_after();
#ifdef SBT_TRACE
          if (blockIdx.x < 2 && tid == 0 && eg < 4096) g_trace_flush[rank][eg] = clock64();
#endif
          uint32_t v[BNT];
#if defined(SBT_FLUSH_DEBUG) && SBT_FLUSH_DEBUG == 2   // timing only: no slot reads
#pragma unroll
          for (int c = 0; c < BNT; ++c) v[c] = 0u;
#else
#pragma unroll
          for (int c = 0; c < BNT; c += 16)
            ptx::tmem_ld16(tmem + lane_addr + FC::BASE + slot * BNT + c,
                           *reinterpret_cast<uint32_t(*)[16]>(v + c));
          ptx::tmem_ld_wait();
#endif
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (rank == 0) ptx::mbar_arrive(&step_empty[slot]);
            else ptx::mbar_arrive_remote(step_empty_leader + slot * 8);
          }
#pragma unroll
          for (int j = 0; j < BNT; ++j) facc[j] += __uint_as_float(v[j]);
        }
      }
      auto park_flush = [&](uint32_t acc_col) {
        if constexpr (FLUSH) {
#pragma unroll
          for (int c = 0; c < BNT; c += 16)
            ptx::tmem_st16(tmem + lane_addr + acc_col + c,
                           *reinterpret_cast<const uint32_t(*)[16]>(
                               reinterpret_cast<const uint32_t*>(facc) + c));
          ptx::tmem_st_wait();
        }
      };
    if (!BB && f.cmode) {
      // TMA-store epilogue: per 32-column chunk, TMEM -> registers (alpha) ->
      // per-warp smem staging (EPIB buffers) -> one TMA store of a 32 x 32 box
      // per warp.
      // The TMA engine writes full lines and clips the M / N tails.
      {
        const uint32_t b = NBUF == 2 ? (tcount & 1u) : 0u;
        const uint32_t ph = NBUF == 2 ? ((tcount >> 1) & 1u) : (tcount & 1u);
#ifdef SBT_TRACE
        const long long tt0 = clock64();
#endif
        ptx::mbar_wait(&acc_full[b], ph);
        ptx::tc_fence_after();
        park_flush(b * ACC_W);
#ifdef SBT_TRACE
        const long long tt1 = clock64();
        long long tt2 = 0, ph_ld = 0, ph_bw = 0, ph_st = 0;
#endif
        // CTA row block -> (inner row, folded batch index)
        int64_t row0 = tc.m0 + rank * HM, rb = tc.pb, rb2 = tc.qb;
        if (f.fm) {
          const int64_t x = row0 / f.m_in;
          row0 -= x * f.m_in;
          if (f.fm == 1) rb = x; else rb2 = x;
        }
        int64_t ecol = tc.n0, ecy = 0;  // tile's first column, unfolded
        if (f.fn) {
          ecy = ecol / f.n_in;
          ecol -= ecy * f.n_in;
        }
        const uint32_t acc_col = b * ACC_W;
        // TMEM loads run one chunk ahead: chunk cc + 32 is in flight while
        // chunk cc is staged and stored
        uint32_t v[32];
        ptx::tmem_ld16(tmem + lane_addr + acc_col, *reinterpret_cast<uint32_t(*)[16]>(v));
        ptx::tmem_ld16(tmem + lane_addr + acc_col + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
#pragma unroll 1
        for (int cc = 0; cc < BNT; cc += 32, ++nchunk) {
          float o[32];
#ifdef SBT_TRACE
          const long long q0 = clock64();
#endif
          if (SPLIT_ACC) {
            uint32_t w[32];
            ptx::tmem_ld16(tmem + lane_addr + acc_col + BNT + cc,
                           *reinterpret_cast<uint32_t(*)[16]>(w));
            ptx::tmem_ld16(tmem + lane_addr + acc_col + BNT + cc + 16,
                           *reinterpret_cast<uint32_t(*)[16]>(w + 16));
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j)
              o[j] = p.alpha * (__uint_as_float(v[j]) + __uint_as_float(w[j]));
          } else {
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = p.alpha * __uint_as_float(v[j]);
          }
          if (cc + 32 < BNT) {
            ptx::tmem_ld16(tmem + lane_addr + acc_col + cc + 32,
                           *reinterpret_cast<uint32_t(*)[16]>(v));
            ptx::tmem_ld16(tmem + lane_addr + acc_col + cc + 48,
                           *reinterpret_cast<uint32_t(*)[16]>(v + 16));
          }
          if (cc + 32 == BNT) {  // accumulator buffer drained: hand it back to the MMA
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (rank == 0) ptx::mbar_arrive(&acc_empty[b]);
              else ptx::mbar_arrive_remote(empty_leader[b]);
            }
#ifdef SBT_TRACE
            tt2 = clock64();
#endif
          }
          // each warp stages and stores its own 32 rows (a 32 x 32 box): no
          // barrier between the four epilogue warps
          const uint32_t buf = nchunk % uint32_t(EPIB);
          uint8_t* stg_p = epi_stage + (warp * EPIB + buf) * (32 * 32 * 4);
          const uint32_t stg = ptx::smem_addr(stg_p);
#ifdef SBT_TRACE
          const long long q1 = clock64();
#endif
          if (lane == 0) ptx::bulk_wait_group_read<EPIB - 1>();  // the store that used `buf` read it
          __syncwarp();
#ifdef SBT_TRACE
          const long long q2 = clock64();
#endif
          if (f.cmode == 1) {  // [32 cols][32 rows]: 128 B per column
#pragma unroll
            for (int j = 0; j < 32; ++j) ptx::sts_f32(stg + j * 128 + lane * 4, o[j]);
          } else {  // [32 rows][32 cols], 128 B swizzle (16 B chunk q at q ^ (row & 7))
#pragma unroll
            for (int q = 0; q < 8; ++q)
              ptx::sts_v4(stg + lane * 128 + ((q ^ (lane & 7)) << 4), __float_as_uint(o[4 * q]),
                          __float_as_uint(o[4 * q + 1]), __float_as_uint(o[4 * q + 2]),
                          __float_as_uint(o[4 * q + 3]));
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
#ifdef SBT_TRACE
          const long long q3 = clock64();
          ph_ld += q1 - q0;
          ph_bw += q2 - q1;
          ph_st += q3 - q2;
#endif
          if (lane == 0) {
            // (un)fold the chunk's first column: one division per tile, then a
            // carry per chunk (32 | n_in for N folds)
            int64_t col0 = ecol + cc, cb = rb, cb2 = rb2;
            if (f.fn) {
              int64_t y = ecy;
              while (col0 >= f.n_in) col0 -= f.n_in, ++y;
              if (f.fn == 1) cb = y; else cb2 = y;
            }
            const int wrow = int(row0) + 32 * warp;
            if (f.cmode == 1)
              ptx::tma_store_4d(&P.tc, stg_p, wrow, int(col0), int(cb), int(cb2));
            else
              ptx::tma_store_4d(&P.tc, stg_p, int(col0), wrow, int(cb), int(cb2));
            ptx::bulk_commit_group();
          }
        }
#ifdef SBT_TRACE
        if (blockIdx.x < 2 && tid == 0 && tcount < 64) {
          g_trace_tepi[rank][tcount][0] = tt0;
          g_trace_tepi[rank][tcount][1] = tt1;
          g_trace_tepi[rank][tcount][2] = tt2;
          g_trace_tepi[rank][tcount][3] = clock64();
          g_trace_tepi[rank][tcount][4] = ph_ld;
          g_trace_tepi[rank][tcount][5] = ph_bw;
          g_trace_tepi[rank][tcount][6] = ph_st;
        }
#endif
      }
    } else {
    {
      const uint32_t b = NBUF == 2 ? (tcount & 1u) : 0u;
      const uint32_t ph = NBUF == 2 ? ((tcount >> 1) & 1u) : (tcount & 1u);
      ptx::mbar_wait(&acc_full[b], ph);
      ptx::tc_fence_after();
      park_flush(b * ACC_W);
#ifdef SBT_TRACE
      long long t_ld = 0, t_begin = clock64();
#endif
      // BB: MMA row r is (batch entry 4*pb + r%4, m = m0 + 32*rank + r/4);
      // fold: row r' = m0 + 128*rank + r of M' is (m = r' % m_in, x = r' / m_in)
      int64_t row = BB ? tc.m0 + rank * 32 + (r >> 2) : tc.m0 + rank * HM + r;
      int64_t bidx = BB ? tc.pb * 4 + (r & 3) : tc.pb, qidx = tc.qb;
      bool row_ok = BB ? (row < p.m && bidx < p.batch) : row < f.mtot;
      if (!BB && f.fm) {
        const int64_t x = row / f.m_in;
        row -= x * f.m_in;
        if (f.fm == 1) bidx = x; else qidx = x;
      }
      float* __restrict__ crow =
          p.c + (row_ok ? bidx * p.cps + row * p.crs + qidx * p.cps2 : 0);
      const int64_t ncols = BB ? p.n : f.ntot;
      const bool full_tile = (tc.n0 + BNT <= ncols) && p.beta == 0.f;
      const bool vec = (p.ccs == 1) && full_tile;
      const uint32_t acc_col = b * ACC_W;
#pragma unroll 1
      for (int cc = 0; cc < BNT; cc += 16) {
        uint32_t v[16];
        float o[16];
#ifdef SBT_TRACE
        long long t0 = clock64();
#endif
        ptx::tmem_ld16(tmem + lane_addr + acc_col + cc, v);
        if (SPLIT_ACC) {
          uint32_t w[16];
          ptx::tmem_ld16(tmem + lane_addr + acc_col + BNT + cc, w);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = __uint_as_float(v[j]) + __uint_as_float(w[j]);
        } else {
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = __uint_as_float(v[j]);
        }
#ifdef SBT_TRACE
        long long t1 = clock64();
        t_ld += t1 - t0;
#endif
        if (!row_ok) continue;
        // column chunk base: fold keeps a 16-column chunk inside one y (16 | n_in)
        int64_t col0 = tc.n0 + cc, ycol = 0;
        if (!BB && f.fn) {
          const int64_t y = col0 / f.n_in;
          col0 -= y * f.n_in;
          ycol = y * (f.fn == 1 ? p.cps : p.cps2);
        }
        float* dst = crow + ycol + col0 * p.ccs;
        if (vec && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(dst + j) =
                make_float4(p.alpha * o[j], p.alpha * o[j + 1], p.alpha * o[j + 2],
                            p.alpha * o[j + 3]);
        } else if (full_tile) {
          // interior tile, beta == 0: straight-line stores, one address add each
#pragma unroll
          for (int j = 0; j < 16; ++j) dst[j * p.ccs] = p.alpha * o[j];
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (tc.n0 + cc + j < ncols) store_out(dst + j * p.ccs, o[j], p.alpha, p.beta);
          }
        }
      }
#ifdef SBT_TRACE
      if (blockIdx.x < 2 && tid == 0 && tcount < 64) {
        long long t_end = clock64();
        g_trace_epi[rank][tcount][0] = t_begin;
        g_trace_epi[rank][tcount][1] = t_end;
        g_trace_epi[rank][tcount][2] = t_ld;
        g_trace_epi[rank][tcount][3] = t_end - t_begin - t_ld;
      }
#endif
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) ptx::mbar_arrive(&acc_empty[b]);
        else ptx::mbar_arrive_remote(empty_leader[b]);
      }
    }
    }  // direct-store epilogue
    }  // tiles
    if (lane == 0) ptx::bulk_wait_group<0>();  // each warp's own stores
  } else if (warp == 13 && rank == 0) {
    // -------------------------------------------------------- MMA issuer
    // The whole warp walks the loop (waits and descriptor math are
    // warp-uniform); one elected lane issues the MMAs and commits.
    // per-problem operand layouts (uniform registers)
    // K-major: rows of BK*4 bytes (SW128 for BK=32, SW64 for BK=16), 8-row
    // groups at SBO = 8*BK*4, K=8 step = 32 B inside the row.
    // MN-major: 32-wide MN slabs of BK k-rows: LBO = slab stride (BK*128 B),
    // SBO 512 (4-row K groups), K=8 step = 1024 B.
    constexpr uint32_t k_lay = BK == 32 ? ptx::kLayoutSW128 : ptx::kLayoutSW64;
    uint32_t it = 0, tcount = 0;
    uint32_t u = 0, u_in = 0;  // FLUSH: step groups started (all tiles), steps in the current one
    int cur = 0;
    for (int64_t t = pair; t < total; t += npairs, ++tcount) {
      const Problem& P = prob(t, cur);
      const bool A_K = !BB && P.a_k, B_K = P.b_k;
      const int nkb = P.nkb;
      const uint32_t idesc = ptx::idesc_tf32(BM, BNT, !A_K, !B_K);
      const uint32_t a_lbo = A_K ? 16u : uint32_t(BK * 128), a_sbo = A_K ? 8u * BK * 4 : 512u;
      const uint32_t b_lbo = B_K ? 16u : uint32_t(BK * 128), b_sbo = B_K ? 8u * BK * 4 : 512u;
      const uint32_t a_step = A_K ? 32u : 1024u, b_step = B_K ? 32u : 1024u;
      const uint32_t a_lay = A_K ? k_lay : ptx::kLayoutSW128Base32B;
      const uint32_t b_lay = B_K ? k_lay : ptx::kLayoutSW128Base32B;
      const uint32_t b = NBUF == 2 ? (tcount & 1u) : 0u;
      const uint32_t ph = NBUF == 2 ? ((tcount >> 1) & 1u) : (tcount & 1u);
      ptx::mbar_wait(&acc_empty[b], ph ^ 1u);
      ptx::tc_fence_after();
#ifdef SBT_TRACE
      if (blockIdx.x < 2 && tcount < 64) g_trace_mma[tcount][0] = clock64();
#endif
      const uint32_t d_main = tmem + b * ACC_W;
      const uint32_t d_small = SPLIT_ACC ? d_main + BNT : d_main;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const uint32_t s = it % RAW_SLOTS;
        const uint32_t ls = it % LO_SLOTS;
        ptx::mbar_wait(&full[s], (it / RAW_SLOTS) & 1u);
        TRACE(3, int(it));
        ptx::tc_fence_after();
        const uint32_t b_raw = ptx::smem_addr(raw_ring + s * SLOT_BYTES) + Gm::A_BYTES;
        const uint32_t a_lo = ptx::smem_addr(lo_ring + ls * LO_SLOT_BYTES);
        const uint32_t b_lo = a_lo + Gm::A_BYTES;
        // BB: A_hi is the converter's swizzled copy, not the dense raw box
        const uint32_t a_raw = BB ? a_lo + Gm::SLOT_BYTES : b_raw - Gm::A_BYTES;
        if constexpr (FLUSH) {
          // group size 2^lg_t K=8 steps; 8-step groups need an even K-block count.
          // One elected lane issues the whole K-block (and waits for the step
          // slots it opens), as in the default path: per-step warp-wide elect /
          // syncwarp rounds doubled the K-block issue time.
          const int lg_t = (flush_lg == 3 && (nkb & 1)) ? 2 : flush_lg;
          const uint32_t gmask = (1u << lg_t) - 1u;
          if (ptx::elect_one_sync()) {
            uint32_t gu = u, gin = u_in;
#pragma unroll
            for (int j = 0; j < BK / 8; ++j) {
              const uint32_t slot = gu % NSLOT;
              if (gin == 0) {  // the epilogue drained this slot's previous group
                ptx::mbar_wait(&step_empty[slot], ((gu / NSLOT) & 1u) ^ 1u);
                ptx::tc_fence_after();
              }
              const uint64_t dar = ptx::umma_desc(a_raw + j * a_step, a_lbo, a_sbo, a_lay);
              const uint64_t dal = ptx::umma_desc(a_lo + j * a_step, a_lbo, a_sbo, a_lay);
              const uint64_t dbr = ptx::umma_desc(b_raw + j * b_step, b_lbo, b_sbo, b_lay);
              const uint64_t dbl = ptx::umma_desc(b_lo + j * b_step, b_lbo, b_sbo, b_lay);
              ptx::mma2_tf32_ss(d_small, dal, dbr, idesc, (kb | j) ? 1u : 0u);
              ptx::mma2_tf32_ss(d_small, dar, dbl, idesc, 1u);
#if defined(SBT_FLUSH_DEBUG) && SBT_FLUSH_DEBUG == 1   // timing only: no slot rotation
              ptx::mma2_tf32_ss(tmem + FC::BASE, dar, dbr, idesc, 1u);
#else
              ptx::mma2_tf32_ss(tmem + FC::BASE + slot * BNT, dar, dbr, idesc, gin ? 1u : 0u);
#endif
              if (gin == gmask) {
                ptx::tc_commit2_mc(&step_full[slot], 0x3);
                ++gu;
                gin = 0;
              } else {
                ++gin;
              }
            }
            ptx::tc_commit2_mc(&raw_empty[s], 0x3);
            ptx::tc_commit2_mc(&lo_empty[ls], 0x3);
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < BK / 8; ++j) {   // the same step accounting on every lane
            if (u_in == gmask) ++u, u_in = 0;
            else ++u_in;
          }
        } else if (ptx::elect_one_sync()) {
#pragma unroll
          for (int j = 0; j < BK / 8; ++j) {
            const uint64_t dar = ptx::umma_desc(a_raw + j * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t dal = ptx::umma_desc(a_lo + j * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t dbr = ptx::umma_desc(b_raw + j * b_step, b_lbo, b_sbo, b_lay);
            const uint64_t dbl = ptx::umma_desc(b_lo + j * b_step, b_lbo, b_sbo, b_lay);
            const uint32_t first = (kb | j) ? 1u : 0u;
            ptx::mma2_tf32_ss(d_small, dal, dbr, idesc, first);
            ptx::mma2_tf32_ss(d_small, dar, dbl, idesc, 1u);
            ptx::mma2_tf32_ss(d_main, dar, dbr, idesc, SPLIT_ACC ? first : 1u);
          }
          ptx::tc_commit2_mc(&raw_empty[s], 0x3);
          ptx::tc_commit2_mc(&lo_empty[ls], 0x3);
        }
        __syncwarp();
#ifdef SBT_TRACE
        if (blockIdx.x < 2 && it < 4096) g_trace[7][it] = clock64();  // issue done (rank-1 row 3)
#endif
      }
      if (ptx::elect_one_sync()) ptx::tc_commit2_mc(&acc_full[b], 0x3);
      __syncwarp();
#ifdef SBT_TRACE
      if (blockIdx.x < 2 && tcount < 64) g_trace_mma[tcount][1] = clock64();
#endif
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, 512);
  }
}

}  // namespace tf32tma
}  // namespace sbt
