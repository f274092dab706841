// Kernel-family selection for one strided (batched) GEMM request.
//
// The reference picks its arithmetic core by entry point only
// (kernels.py:107,174,223).  Here the same request is routed by stride class:
//   tensor-core tiles (fp32: tcgen05 3xTF32; fp64: DMMA) when each operand has
//       a unit-stride mode and 16-byte aligned other strides -- after
//       orienting the problem (C^T = B^T A^T) so the larger extent is the
//       128-row MMA dimension;
//   small-matrix batched kernel for many tiny GEMMs;
//   generic SIMT kernel for everything else (odd extents / strides).
#pragma once
#include <cstdlib>
#include <cstring>
#include <utility>

#include "sbt_common.cuh"
#include "k_generic.cuh"
#include "k_skinny_dmma.cuh"
#include "k_tf32x3.cuh"
#include "k_tf32x3_pair_tma.cuh"
#include "k_dmma.cuh"
#include "k_small.cuh"
#include "k_small_dmma.cuh"
#include "k_small64.cuh"
#include "k_gemv.cuh"
#include "sbt_tma.cuh"

namespace sbt {

template <typename T, int BM, int BN, int BK, int TM, int TN>
static void launch_generic_cfg(const GemmParams<T>& p, cudaStream_t stream, const char* name) {
  const int64_t tiles_m = ceil_div(p.m, BM), tiles_n = ceil_div(p.n, BN);
  const int64_t total = tiles_m * tiles_n * p.batch * p.batch2;
  const int64_t grid = total < int64_t(kNumSMs) * 32 ? total : int64_t(kNumSMs) * 32;
  const int a_m_fast = p.ars <= p.acs ? 1 : 0;
  const int b_k_fast = p.brs <= p.bcs ? 1 : 0;
  generic_gemm_kernel<T, BM, BN, BK, TM, TN>
      <<<dim3(unsigned(grid)), dim3(GenericCfg<T, BM, BN, BK, TM, TN>::NT), 0, stream>>>(
          p, tiles_m, tiles_n, total, a_m_fast, b_k_fast);
  note_launch(name);
}

template <typename T>
static void launch_generic(const GemmParams<T>& p, cudaStream_t stream) {
  const bool small = p.m <= 48 || p.n <= 48;
  if constexpr (sizeof(T) == 4) {
    if (small) launch_generic_cfg<T, 32, 32, 16, 2, 2>(p, stream, "generic_f32_32x32");
    else       launch_generic_cfg<T, 128, 128, 8, 8, 8>(p, stream, "generic_f32_128x128");
  } else {
    if (small) launch_generic_cfg<T, 32, 32, 8, 2, 2>(p, stream, "generic_f64_32x32");
    else       launch_generic_cfg<T, 64, 64, 8, 4, 4>(p, stream, "generic_f64_64x64");
  }
}

// C = A B  <=>  C^T = B^T A^T : swap operand roles and output strides.
template <typename T>
static GemmParams<T> transposed(const GemmParams<T>& p) {
  GemmParams<T> q = p;
  q.m = p.n; q.n = p.m;
  q.a = p.b; q.ars = p.bcs; q.acs = p.brs; q.aps = p.bps; q.aps2 = p.bps2;
  q.b = p.a; q.brs = p.acs; q.bcs = p.ars; q.bps = p.aps; q.bps2 = p.aps2;
  q.crs = p.ccs; q.ccs = p.crs;
  return q;
}

static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// 16-byte vectors: 4 fp32 or 2 fp64 elements
template <typename T>
static inline bool vmult(int64_t v) { return v % int64_t(16 / sizeof(T)) == 0; }
static inline bool aligned16(const void* ptr) {
  return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0;
}

// Operand major-ness for the 16-byte-vector tensor-core producers.
// returns 1 = K-major, 2 = MN-major, 0 = not eligible
template <typename T>
static int a_major(const GemmParams<T>& p) {
  if (!aligned16(p.a) || !vmult<T>(p.aps) || !vmult<T>(p.aps2)) return 0;
  if (p.acs == 1 && vmult<T>(p.ars) && vmult<T>(p.k)) return 1;
  if (p.ars == 1 && vmult<T>(p.acs) && vmult<T>(p.m)) return 2;
  return 0;
}
template <typename T>
static int b_major(const GemmParams<T>& p) {
  if (!aligned16(p.b) || !vmult<T>(p.bps) || !vmult<T>(p.bps2)) return 0;
  if (p.brs == 1 && vmult<T>(p.bcs) && vmult<T>(p.k)) return 1;
  if (p.bcs == 1 && vmult<T>(p.brs) && vmult<T>(p.n)) return 2;
  return 0;
}

template <int BN, bool AK, bool BK_>
static int launch_tf32x3_cfg(const GemmParams<float>& p, cudaStream_t stream) {
  using C_ = tf32x3::Cfg<BN>;
  auto kern = tf32x3::tf32x3_gemm_kernel<BN, AK, BK_>;
  if (set_smem_attr(reinterpret_cast<const void*>(kern), C_::SMEM_BYTES) != 0) return -3;
  const int64_t tiles_m = ceil_div(p.m, tf32x3::BM), tiles_n = ceil_div(p.n, BN);
  const int64_t total = tiles_m * tiles_n * p.batch * p.batch2;
  if (total > int64_t(0x7fffffff)) return -2;
  kern<<<dim3(unsigned(total)), dim3(tf32x3::kThreads), C_::SMEM_BYTES, stream>>>(
      p, tiles_m, tiles_n);
  note_launch("tc_tf32x3");
  return 0;
}

// Fold a batch mode into M (only A and C depend on it) and / or into N (only B
// and C) when the extent is a multiple of the CTA block but not of the 256-wide
// pair tile (see k_tf32x3_pair_tma.cuh, struct Fold).
static tf32tma::Fold make_fold(const GemmParams<float>& p, bool a_mn) {
  tf32tma::Fold f{p.m, p.n, p.m, p.n, 0, 0, 0};
  auto cnt = [&](int w) { return w == 1 ? p.batch : p.batch2; };
  auto as = [&](int w) { return w == 1 ? p.aps : p.aps2; };
  auto bs = [&](int w) { return w == 1 ? p.bps : p.bps2; };
  // M folds need whole A boxes per batch entry: 128 rows for K-major A, 32
  // for MN-major A (its boxes are 32-row MN atoms, each with its own batch)
  const int64_t m_unit = a_mn ? 32 : tf32tma::HM;
  if (p.m % tf32tma::BM != 0 && p.m % m_unit == 0) {
    for (int w : {2, 1})
      if (cnt(w) > 1 && bs(w) == 0 && as(w) > 0 && vmult<float>(as(w))) {
        f.fm = w;
        f.mtot = p.m * cnt(w);
        break;
      }
  }
  if (p.n % tf32tma::BN != 0 && p.n % tf32tma::HN == 0) {
    for (int w : {1, 2})
      if (w != f.fm && cnt(w) > 1 && as(w) == 0 && bs(w) > 0 && vmult<float>(bs(w))) {
        f.fn = w;
        f.ntot = p.n * cnt(w);
        break;
      }
  }
  return f;
}

// ---- CTA-pair tcgen05 kernel: planning, problem sets, launches --------------

// How one GEMM request maps onto the pair kernel (orientation, layouts, fold,
// tile width, accumulator split).
struct PairPlan {
  GemmParams<float> p;  // oriented problem
  tf32tma::Fold f;
  int am = 0, bm = 0;   // 1 = K-major, 2 = MN-major
  bool bb = false, split = false;
  int bnt = 256;
};

static bool pick_split(const GemmParams<float>& p) {
  static const int split_env = env_int("SBT_TC_SPLITACC", -1);
  return split_env < 0 ? (p.k > 512) : (split_env != 0);
}

// Decide whether (and how) the pair kernel runs this request.
// variant (SBT_TC_VARIANT): 0 auto, 1 = 1-CTA tiles only, 4 = force pair,
// 5 = batch-blocked pair only, 6 = auto without batch folding
static bool plan_pair(const GemmParams<float>& p0, PairPlan* out) {
  static const int variant = env_int("SBT_TC_VARIANT", 0);
  if (variant == 1) return false;
  if (variant == 0 || variant == 5) {
    // exceptional cases: A unit-stride along the batch, B batch-independent
    for (int o = 0; o < 2; ++o) {
      const GemmParams<float> p = o ? transposed(p0) : p0;
      if (p.aps != 1 || p.bps != 0 || p.batch < 2 || !aligned16(p.a)) continue;
      if (p.ars < 4 || p.acs < 4 || !vmult<float>(p.ars) || !vmult<float>(p.acs) ||
          !vmult<float>(p.aps2))
        continue;
      if (p.m < 64 || p.n < 96) continue;
      const int bm = b_major(p);
      if (!bm) continue;
      out->p = p;
      out->f = tf32tma::Fold{p.m, p.n, p.m, p.n, 0, 0, 0};
      out->am = 2; out->bm = bm; out->bb = true; out->bnt = p.n < 192 ? 128 : 256;
      out->split = pick_split(p);
      return true;
    }
    if (variant == 5) return false;
  }
  // among the two orientations (C = AB, C^T = B^T A^T) take the one whose
  // (folded) M reaches a full 256-row tile, larger M first
  bool found = false;
  for (int o = 0; o < 2; ++o) {
    const GemmParams<float> q = o ? transposed(p0) : p0;
    const int qa = a_major(q), qb = b_major(q);
    if (!qa || !qb) continue;
    const tf32tma::Fold f =
        variant == 6 ? tf32tma::Fold{q.m, q.n, q.m, q.n, 0, 0, 0} : make_fold(q, qa == 2);
    // narrow N (< 96) only pays off for many M rows in total (HBM-bound skinny
    // products: rank-r Tucker mode products, any rank -- the unbiased FLUSH
    // mode runs there); narrow tiles need K-major B
    const int64_t rows = f.mtot * ((f.fm == 1 || f.fn == 1) ? 1 : q.batch) *
                         ((f.fm == 2 || f.fn == 2) ? 1 : q.batch2);
    const bool ok = variant == 4 ||
                    (f.mtot >= 256 && (f.ntot >= 96 || (rows >= 8192 && qb == 1)));
    // ties: prefer C unit-stride along N (vector staging stores in the
    // TMA-store epilogue: 8 x 16 B per thread and chunk instead of 32 x 4 B)
    static const int prefer_rowmajor_c = env_int("SBT_TC_PREFER_CN", 1);
    const bool better_c = prefer_rowmajor_c && q.ccs == 1 && out->p.ccs != 1;
    if (ok && (!found || f.mtot > out->f.mtot ||
               (f.mtot == out->f.mtot && (f.ntot > out->f.ntot ||
                                          (f.ntot == out->f.ntot && better_c))))) {
      out->p = q; out->f = f; out->am = qa; out->bm = qb; found = true;
    }
  }
  if (!found) return false;
  const int64_t nt = out->f.ntot;
  out->bnt = nt <= 32 ? 32 : nt <= 64 ? 64 : nt < 192 ? 128 : 256;
  if (out->bnt < 64 && out->bm != 1) return false;  // 16-column B halves must be K-major
  out->bb = false;
  out->split = pick_split(out->p);
  // narrow tiles run the unbiased FLUSH mode (k_tf32x3_pair_tma.cuh header),
  // which keeps the cross terms in the split accumulator
  static const int narrow_flush = env_int("SBT_TC_FLUSH", 1);
  if (narrow_flush && accumulation_mode() && out->bnt <= 64) out->split = true;
  // split accumulators (K > 512) fill TMEM at 256 columns: 128-wide tiles keep
  // them double-buffered, so the epilogue overlaps the next tile's MMAs
  static const int split_bnt = env_int("SBT_TC_SPLIT_BNT", 256);
  if (out->split && out->bnt == 256 && split_bnt == 128) out->bnt = 128;
  static const int force_bnt = env_int("SBT_TC_BNT", 0);   // A/B: cap the tile width
  if (force_bnt >= 128 && out->bnt > force_bnt) out->bnt = force_bnt;
  return true;
}

// Tensor maps, tile grid and epilogue mode of one planned problem.
template <bool BB, int BNT, int KB>
static bool fill_problem(const PairPlan& pl, tf32tma::Problem* pr) {
  const GemmParams<float>& p = pl.p;
  tf32tma::Fold f = pl.f;
  constexpr uint32_t HNT = BNT / 2;
  const bool AK = pl.am == 1, BK_ = pl.bm == 1;
  const CUtensorMapSwizzle kswz = KB == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  const bool ok_a =
      BB ? make_tmap_f32(&pr->ta, p.a, p.batch, p.m, p.ars, p.k, p.acs, p.batch2, p.aps2, 4, 8,
                         CU_TENSOR_MAP_SWIZZLE_NONE, KB)
      : AK ? make_tmap_f32(&pr->ta, p.a, p.k, p.m, p.ars, p.batch, p.aps, p.batch2, p.aps2, KB,
                           128, kswz)
           : make_tmap_f32(&pr->ta, p.a, p.m, p.k, p.acs, p.batch, p.aps, p.batch2, p.aps2, 32,
                           KB, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  const bool ok_b =
      BK_ ? make_tmap_f32(&pr->tb, p.b, p.k, p.n, p.bcs, p.batch, p.bps, p.batch2, p.bps2, KB,
                          HNT, kswz)
          : make_tmap_f32(&pr->tb, p.b, p.n, p.k, p.brs, p.batch, p.bps, p.batch2, p.bps2, 32,
                          KB, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!ok_a || !ok_b) return false;  // not expressible as TMA: caller falls back
  // TMA-store epilogue when C is expressible as a tensor map (beta == 0: C not read)
  std::memset(&pr->tc, 0, sizeof(pr->tc));
  f.cmode = 0;
  static const int tma_epi = env_int("SBT_TC_TMA_EPI", 1);
  // (128-row store boxes: not with an M fold of fewer rows per batch entry)
  if (!BB && tma_epi && p.beta == 0.f && aligned16(p.c) && vmult<float>(p.cps) &&
      vmult<float>(p.cps2) && !(f.fm && f.m_in % tf32tma::HM != 0)) {
    // 32 x 32 boxes: each epilogue warp stores its own 32 rows
    if (p.crs == 1 && vmult<float>(p.ccs) &&
        make_tmap_f32(&pr->tc, p.c, p.m, p.n, p.ccs, p.batch, p.cps, p.batch2, p.cps2, 32, 32,
                      CU_TENSOR_MAP_SWIZZLE_NONE))
      f.cmode = 1;
    else if (p.ccs == 1 && vmult<float>(p.crs) &&
             make_tmap_f32(&pr->tc, p.c, p.n, p.m, p.crs, p.batch, p.cps, p.batch2, p.cps2, 32,
                           32, CU_TENSOR_MAP_SWIZZLE_128B))
      f.cmode = 2;
  }
  pr->p = p;
  pr->f = f;
  pr->tiles_m = ceil_div(f.mtot, BB ? 64 : tf32tma::BM);
  pr->tiles_n = ceil_div(f.ntot, BNT);
  pr->nbatch = BB ? ceil_div(p.batch, 4) : ((f.fm == 1 || f.fn == 1) ? 1 : p.batch);
  pr->a_k = AK ? 1 : 0;
  pr->b_k = BK_ ? 1 : 0;
  pr->nkb = int(ceil_div(p.k, KB));
  pr->pad = 0;
  return true;
}

// Launch one problem set (tile_begin of each problem must be set, total summed).
template <int MAXP, bool SPLIT, bool BB, int BNT, int KB = 32, int EPIB = 2>
static int launch_pair_set(const tf32tma::ProblemSet<MAXP>& ps, cudaStream_t stream,
                           const char* name) {
  static_assert(sizeof(tf32tma::ProblemSet<MAXP>) <= 32000, "kernel parameter space");
  auto kern = tf32tma::tf32x3_pair_tma_kernel<MAXP, SPLIT, KB, BB, BNT, EPIB>;
  constexpr int smem = tf32tma::Geo<KB, BB, BNT, EPIB>::SMEM_BYTES;
  if (set_smem_attr(reinterpret_cast<const void*>(kern), smem) != 0) return -3;
  const int64_t pairs = ps.total < kNumSMs / 2 ? ps.total : kNumSMs / 2;
  // low byte: L2 prefetch distance (measured: no gain, 0); bits 8/9: diagnostics
  // (SBT_TC_DEBUG=1 skips the TMA loads, 2 the lo conversion -- wrong results)
  // bits 12-13: log2 of the K=8 steps per FLUSH step-accumulator group
  // (SBT_TC_FLUSH_G = 1 / 2 / 4 / 8; narrow tiles only)
  // 4 K=8 steps per group: fit of the 512^3 rank-32 HOOI within 5.1e-6 of the
  // fp64 oracle (8 steps: 7.3e-6; north_star bound 1e-5) for ~2% of its time
  static const int flush_g = env_int("SBT_TC_FLUSH_G", 4);
  static const int prefetch = env_int("SBT_TC_PREFETCH", 0) | (env_int("SBT_TC_DEBUG", 0) << 8) |
                              ((flush_g >= 8 ? 3 : flush_g >= 4 ? 2 : flush_g >= 2 ? 1 : 0) << 12);
  kern<<<dim3(unsigned(2 * pairs)), dim3(tf32tma::kThreads), smem, stream>>>(ps, prefetch);
  note_launch(name);
  return 1;
}

static const char* pair_name(bool bb, bool split, int bnt, bool fold, bool group) {
  if (group) return bb ? "tc_tf32x3_pair_group_bb" : "tc_tf32x3_pair_group";
  if (bb) return split ? "tc_tf32x3_pair_bb_splitacc" : "tc_tf32x3_pair_bb";
  if (fold) {
    if (bnt < 256) return split ? "tc_tf32x3_pair_fold_narrow_splitacc" : "tc_tf32x3_pair_fold_narrow";
    return split ? "tc_tf32x3_pair_fold_splitacc" : "tc_tf32x3_pair_fold";
  }
  if (bnt < 256) return split ? "tc_tf32x3_pair_narrow_splitacc" : "tc_tf32x3_pair_narrow";
  return split ? "tc_tf32x3_pair_tma_splitacc" : "tc_tf32x3_pair_tma";
}

template <bool SPLIT, bool BB, int BNT>
static int launch_pair_single_t(const PairPlan& pl, cudaStream_t stream) {
  tf32tma::ProblemSet<1> ps;
  if (!fill_problem<BB, BNT, 32>(pl, &ps.pr[0])) return 0;
  ps.pr[0].tile_begin = 0;
  ps.n = 1;
  ps.total = ps.pr[0].tiles_m * ps.pr[0].tiles_n * ps.pr[0].nbatch *
             ((ps.pr[0].f.fm == 2 || ps.pr[0].f.fn == 2) ? 1 : pl.p.batch2);
  const char* name = pair_name(BB, SPLIT, BNT, pl.f.fm || pl.f.fn, false);
  // short K with the TMA-store epilogue: the C writes bound the tile, so more
  // stores in flight (4 staging buffers) beat raw-ring depth
  if constexpr (!SPLIT && !BB && BNT == 256) {
    static const int epib4 = env_int("SBT_TC_EPIB4", 0);  // measured: no gain (kept for A/B)
    if (epib4 && ps.pr[0].nkb <= 4 && ps.pr[0].f.cmode != 0)
      return launch_pair_set<1, SPLIT, BB, BNT, 32, 4>(ps, stream, name);
  }
  if constexpr (BB) {   // A/B: 16-deep K-blocks for the batch-blocked tiles
    static const int bb_kb = env_int("SBT_TC_BB_KB", 32);
    if (bb_kb == 16) {
      tf32tma::ProblemSet<1> ps16;
      if (!fill_problem<BB, BNT, 16>(pl, &ps16.pr[0])) return 0;
      ps16.pr[0].tile_begin = 0;
      ps16.n = 1;
      ps16.total = ps.total;
      return launch_pair_set<1, SPLIT, BB, BNT, 16>(ps16, stream, name);
    }
  }
  return launch_pair_set<1, SPLIT, BB, BNT>(ps, stream, name);
}

// dispatch on the compile-time configuration of a plan
template <template <bool, bool, int> class F, typename... Args>
static int with_pair_cfg(const PairPlan& pl, Args&&... args) {
  if (pl.bb) {
    if (pl.bnt == 128)
      return pl.split ? F<true, true, 128>::run(args...) : F<false, true, 128>::run(args...);
    return pl.split ? F<true, true, 256>::run(args...) : F<false, true, 256>::run(args...);
  }
  switch (pl.bnt) {
    case 32: return pl.split ? F<true, false, 32>::run(args...) : F<false, false, 32>::run(args...);
    case 64: return pl.split ? F<true, false, 64>::run(args...) : F<false, false, 64>::run(args...);
    case 128:
      return pl.split ? F<true, false, 128>::run(args...) : F<false, false, 128>::run(args...);
    default:
      return pl.split ? F<true, false, 256>::run(args...) : F<false, false, 256>::run(args...);
  }
}

template <bool SPLIT, bool BB, int BNT>
struct SingleLaunch {
  static int run(const PairPlan& pl, cudaStream_t stream) {
    return launch_pair_single_t<SPLIT, BB, BNT>(pl, stream);
  }
};

static int try_pair_f32(const GemmParams<float>& p0, cudaStream_t stream) {
  PairPlan pl;
  if (!plan_pair(p0, &pl)) return 0;
  return with_pair_cfg<SingleLaunch>(pl, pl, stream);
}

// ---- grouped launch: many independent problems, one persistent pair kernel --
constexpr int kMaxGroup = 40;

template <bool SPLIT, bool BB, int BNT>
struct GroupLaunch {
  // plans[idx[0..count)] share this configuration
  static int run(const PairPlan* plans, const int* idx, int count, cudaStream_t stream,
                 bool* launched) {
    thread_local tf32tma::ProblemSet<kMaxGroup> ps;  // host staging (the launch copies it)
    int rc = 0;
    for (int base = 0; base < count && rc >= 0; base += kMaxGroup) {
      const int nb = (count - base) < kMaxGroup ? (count - base) : kMaxGroup;
      int n = 0;
      int64_t total = 0;
      int members[kMaxGroup];
      static const int bb_kb = BB ? env_int("SBT_TC_BB_KB", 32) : 32;
      for (int i = 0; i < nb; ++i) {
        const PairPlan& pl = plans[idx[base + i]];
        bool filled;
        if constexpr (BB)
          filled = bb_kb == 16 ? fill_problem<BB, BNT, 16>(pl, &ps.pr[n])
                               : fill_problem<BB, BNT, 32>(pl, &ps.pr[n]);
        else
          filled = fill_problem<BB, BNT, 32>(pl, &ps.pr[n]);
        if (!filled) continue;  // caller relaunches singly
        ps.pr[n].tile_begin = total;
        total += ps.pr[n].tiles_m * ps.pr[n].tiles_n * ps.pr[n].nbatch *
                 ((ps.pr[n].f.fm == 2 || ps.pr[n].f.fn == 2) ? 1 : pl.p.batch2);
        members[n++] = idx[base + i];
      }
      if (n == 0) continue;
      ps.n = n;
      ps.total = total;
      if constexpr (BB) {
        rc = bb_kb == 16
                 ? launch_pair_set<kMaxGroup, SPLIT, BB, BNT, 16>(
                       ps, stream, pair_name(BB, SPLIT, BNT, false, true))
                 : launch_pair_set<kMaxGroup, SPLIT, BB, BNT>(
                       ps, stream, pair_name(BB, SPLIT, BNT, false, true));
      } else {
        rc = launch_pair_set<kMaxGroup, SPLIT, BB, BNT>(ps, stream,
                                                        pair_name(BB, SPLIT, BNT, false, true));
      }
      if (rc >= 0)
        for (int i = 0; i < n; ++i) launched[members[i]] = true;
    }
    return rc;
  }
};

template <int BN>
static int launch_tf32x3_bn(const GemmParams<float>& p, int am, int bm, cudaStream_t s) {
  if (am == 1 && bm == 1) return launch_tf32x3_cfg<BN, true, true>(p, s);
  if (am == 1 && bm == 2) return launch_tf32x3_cfg<BN, true, false>(p, s);
  if (am == 2 && bm == 1) return launch_tf32x3_cfg<BN, false, true>(p, s);
  return launch_tf32x3_cfg<BN, false, false>(p, s);
}

// Batch <-> row role swap: the batch index becomes the MMA row index (and the
// old rows a batch mode).  Valid when B does not depend on the batch.  This is
// how the exceptional ("extended") cases reach the tensor cores: their first
// operand is unit-stride along the batch mode, which becomes an MN-major MMA
// operand (reference kernels.py:179-204 puts apt = 1 there).
template <typename T>
static bool batch_row_swapped(const GemmParams<T>& p, GemmParams<T>* q) {
  if (p.bps != 0 || p.batch < 2) return false;
  *q = p;
  q->m = p.batch; q->batch = p.m;
  q->ars = p.aps; q->aps = p.ars;
  q->crs = p.cps; q->cps = p.crs;
  return true;
}

// Candidate orientations: as given, transposed (C^T = B^T A^T), and the
// batch<->row swaps of both; pick the tensor-core-eligible one with the
// largest MMA M.  Returns false if none is eligible.
template <typename T>
static bool orient(const GemmParams<T>& p0, GemmParams<T>* out, int* am, int* bm) {
  GemmParams<T> cand[4];
  int nc = 0;
  cand[nc++] = p0;
  cand[nc++] = transposed(p0);
  GemmParams<T> q;
  if (batch_row_swapped(p0, &q)) cand[nc++] = q;
  if (batch_row_swapped(transposed(p0), &q)) cand[nc++] = q;
  int best = -1;
  for (int i = 0; i < nc; ++i) {
    const int a = a_major(cand[i]), b = b_major(cand[i]);
    if (!a || !b) continue;
    if (best < 0 || cand[i].m > cand[best].m ||
        (cand[i].m == cand[best].m && cand[i].n > cand[best].n)) {
      best = i; *am = a; *bm = b;
    }
  }
  if (best < 0) return false;
  *out = cand[best];
  return true;
}

template <bool AK, bool BK_, bool BB, int NW, int BNT = 128, bool BB16 = false>
static int launch_dmma_nw(const GemmParams<double>& p, cudaStream_t stream) {
  auto kern = dmma::dmma_gemm_kernel<AK, BK_, BB, NW, BNT, BB16>;
  // BNT = 64: the B tile is half as wide (two CTAs per SM need <= 113 KB each)
  const int smem = BNT == 128 ? dmma::SMEM_BYTES : dmma::SMEM_BYTES_N64;
  if (set_smem_attr(reinterpret_cast<const void*>(kern), smem) != 0) return -3;
  const int64_t tiles_m = ceil_div(p.m, BB ? 32 : dmma::BM), tiles_n = ceil_div(p.n, BNT);
  const int64_t total = tiles_m * tiles_n * (BB ? ceil_div(p.batch, 4) : p.batch) * p.batch2;
  if (total > int64_t(0x7fffffff)) return -2;
  kern<<<dim3(unsigned(total)), dim3(NW * 32), smem, stream>>>(p, tiles_m, tiles_n);
  note_launch(BB ? "tc_dmma_f64_bb" : "tc_dmma_f64");
  return 1;
}

// 16 warps per 128 x 128 tile (each 32 x 32) for short reductions, where a
// tile's cp.async prologue and epilogue are a large share and more warps hide
// them; 8 warps (64 x 32 each, more fragment reuse) for long ones.  Measured
// (36-case fp64 sweeps, TF/s, 8 -> 16 warps): n=128 20.0 -> 23.9, n=256 27.7 ->
// 27.7, n=512 29.7 -> 29.1, 4th order (K=128) 25.6 -> 26.1.
template <bool AK, bool BK_, bool BB = false>
static int launch_dmma_cfg(const GemmParams<double>& p, cudaStream_t stream) {
  static const int nw_env = env_int("SBT_DMMA_WARPS", 0);  // 0 = by K
  // plain tiles: 128 x 64 with two CTAs per SM (one CTA's cp.async prologue and
  // C epilogue overlap the other's DMMA loop).  Measured (36-case fp64 sweep,
  // plain-case launches, 128 -> 64): n=128 24.7 -> 26.8, n=256 28.6 -> 30.3
  // TF/s; the batch-blocked tiles lose (25.0 -> 23.4) and keep 128 x 128.
  static const int bn_env = env_int("SBT_DMMA_BN", 0);     // 0 = by tile kind
  // batch-blocked tiles: 8 warps (25.0 -> 25.6 TF/s on the 8 exceptional cases at n=256);
  // 16-byte A staging when the batch pairs are 16-byte aligned (SBT_DMMA_BB16=0: 8-byte),
  // then also 128 x 64 tiles, two CTAs per SM (36-case step 28.7 -> 29.0 TF/s)
  static const int bb16_env = env_int("SBT_DMMA_BB16", 1);
  if (BB && bb16_env && nw_env == 0 && p.ars % 2 == 0 && p.acs % 2 == 0 &&
      reinterpret_cast<uintptr_t>(p.a) % 16 == 0)
    return bn_env == 128 ? launch_dmma_nw<AK, BK_, BB, 8, 128, true>(p, stream)
                         : launch_dmma_nw<AK, BK_, BB, 8, 64, true>(p, stream);
  const int bn = bn_env ? bn_env : (BB ? 128 : 64);
  // N <= 32 (the rank-r Tucker products of fp64 tensors): 128 x 32 tiles, no idle columns
  static const int narrow32 = env_int("SBT_DMMA_N32", 1);
  if (!BB && narrow32 && bn_env == 0 && nw_env == 0 && p.n <= 32)
    return launch_dmma_nw<AK, BK_, BB, 8, 32>(p, stream);
  if (bn == 64 && nw_env == 0) return launch_dmma_nw<AK, BK_, BB, 8, 64>(p, stream);
  const int nw = nw_env ? nw_env : ((p.k <= 256 && !BB) ? 16 : 8);
  return nw == 16 ? launch_dmma_nw<AK, BK_, BB, 16>(p, stream)
                  : launch_dmma_nw<AK, BK_, BB, 8>(p, stream);
}

// fp64 exceptional cases: batch-blocked DMMA tiles (k_dmma.cuh), as given or
// transposed.  Returns 1 if launched, 0 if not eligible.
static int try_dmma_bb(const GemmParams<double>& p0, cudaStream_t stream) {
  for (int orient = 0; orient < 2; ++orient) {
    const GemmParams<double> p = orient ? transposed(p0) : p0;
    if (p.aps != 1 || p.bps != 0 || p.batch < 4 || p.m < 16 || p.n < 64) continue;
    const int bm = b_major(p);
    if (!bm) continue;
    return bm == 1 ? launch_dmma_cfg<false, true, true>(p, stream)
                   : launch_dmma_cfg<false, false, true>(p, stream);
  }
  return 0;
}

static int try_tensor_f64(const GemmParams<double>& p0, cudaStream_t stream, bool forced) {
  static const int use_bb = env_int("SBT_DMMA_BB", 1);
  if (use_bb) {
    const int rc = try_dmma_bb(p0, stream);
    if (rc != 0) return rc;
  }
  GemmParams<double> p;
  int am = 0, bm = 0;
  if (!orient(p0, &p, &am, &bm)) return 0;
  if (!forced && (p.m < 32 || p.n < 8 || double(p.m) * p.n * p.k * p.batch * p.batch2 < 1e6))
    return 0;
  if (am == 1 && bm == 1) return launch_dmma_cfg<true, true>(p, stream);
  if (am == 1) return launch_dmma_cfg<true, false>(p, stream);
  if (bm == 1) return launch_dmma_cfg<false, true>(p, stream);
  return launch_dmma_cfg<false, false>(p, stream);
}

// Returns 1 if launched, 0 if not eligible, <0 on error.
static int try_tensor_f32(const GemmParams<float>& p0, cudaStream_t stream, bool forced) {
  {
    const int rc = try_pair_f32(p0, stream);
    if (rc != 0) return rc;
  }
  GemmParams<float> p;
  int am = 0, bm = 0;
  if (!orient(p0, &p, &am, &bm)) return 0;
  // M >= 32: a 32-row problem pads the 128-row tile 4x, but the many-batch
  // shapes that reach here (Tucker products with a rank-32 mode first) are
  // HBM-bound, where the padding costs nothing and the SIMT fallback does
  if (!forced && (p.m < 32 || p.n < 8 || double(p.m) * p.n * p.k * p.batch * p.batch2 < 2e6))
    return 0;
  int bn = env_int("SBT_TC_BN", 0);
  if (bn != 32 && bn != 64 && bn != 128 && bn != 256)
    bn = p.n > 128 ? 256 : (p.n > 64 ? 128 : (p.n > 32 ? 64 : 32));
  int rc;
  switch (bn) {
    case 256: rc = launch_tf32x3_bn<256>(p, am, bm, stream); break;
    case 128: rc = launch_tf32x3_bn<128>(p, am, bm, stream); break;
    case 64:  rc = launch_tf32x3_bn<64>(p, am, bm, stream); break;
    default:  rc = launch_tf32x3_bn<32>(p, am, bm, stream); break;
  }
  return rc < 0 ? rc : 1;
}

// ---- K3 small-matrix batched ----------------------------------------------------
template <typename T, int S, bool AM, bool BK_>
static int launch_small_cfg(const GemmParams<T>& p, cudaStream_t stream) {
  auto kern = small::small_batched_kernel<T, S, AM, BK_>;
  constexpr int smem = small::smem_bytes<T, S>();
  if (set_smem_attr(reinterpret_cast<const void*>(kern), smem) != 0) return -3;
  const int64_t ngroups = ceil_div(p.batch, small::Shape<S>::G);
  const int per_sm = smem <= 110 * 1024 ? 2 : 1;
  const int64_t grid = ngroups < int64_t(kNumSMs) * per_sm ? ngroups : int64_t(kNumSMs) * per_sm;
  kern<<<dim3(unsigned(grid)), dim3(small::kThreads), smem, stream>>>(p, ngroups);
  note_launch(sizeof(T) == 4 ? "small_batched_f32" : "small_batched_f64");
  return 1;
}

template <typename T, int S>
static int launch_small_s(const GemmParams<T>& p, bool am, bool bk, cudaStream_t s) {
  if (am && bk) return launch_small_cfg<T, S, true, true>(p, s);
  if (am) return launch_small_cfg<T, S, true, false>(p, s);
  if (bk) return launch_small_cfg<T, S, false, true>(p, s);
  return launch_small_cfg<T, S, false, false>(p, s);
}

// fp64 16 < n <= 32 with column-major A, B and C: the DMMA variant of K3.
template <int NMAX>
static int launch_small_dmma(const GemmParams<double>& p, cudaStream_t stream) {
  using namespace small_dmma;
  using C_ = Cfg<NMAX>;
  auto kern = small_dmma_kernel<NMAX>;
  if (set_smem_attr(reinterpret_cast<const void*>(kern), C_::SMEM_BYTES) != 0) return -3;
  CUtensorMap ta, tb;
  if (!make_tmap_f64_3d(&ta, p.a, p.m, p.k, p.acs, p.batch, p.aps, ld_of(int(p.m)),
                        uint32_t(p.k), C_::G) ||
      !make_tmap_f64_3d(&tb, p.b, p.k, p.n, p.bcs, p.batch, p.bps, ld_of(int(p.k)),
                        uint32_t(p.n), C_::G))
    return 0;
  const int64_t ngroups = ceil_div(p.batch, C_::G);
  const int64_t cap = int64_t(kNumSMs) * C_::CTAS_PER_SM;
  const int64_t grid = ngroups < cap ? ngroups : cap;
  kern<<<dim3(unsigned(grid)), dim3(kThreads), C_::SMEM_BYTES, stream>>>(p, ta, tb, ngroups);
  note_launch(NMAX == 32 ? "small_batched_dmma_f64" : "small_batched_dmma64_f64");
  return 1;
}

// fp64 16 < n <= 64 with column-major A, B and C: the DMMA variants of K3.
static int try_small_dmma(const GemmParams<double>& p, cudaStream_t stream) {
  if (p.m % 8 || p.n % 8 || p.k % 4 || p.m > 64 || p.n > 64 || p.k > 64) return 0;
  if (!(p.ars == 1 && p.acs == p.m && p.brs == 1 && p.bcs == p.k && p.crs == 1 && p.ccs == p.m))
    return 0;
  if (p.aps % 2 || p.bps % 2 || p.aps < p.m * p.k || p.bps < p.k * p.n) return 0;
  if (!aligned16(p.a) || !aligned16(p.b) || p.batch > (int64_t(1) << 31)) return 0;
  static const int use64 = env_int("SBT_SMALL_DMMA64", 1);
  if (p.m > 32 || p.n > 32 || p.k > 32) return use64 ? launch_small_dmma<64>(p, stream) : 0;
  return launch_small_dmma<32>(p, stream);
}

// fp32 64 x 64 x 64 batches with column-major A, B and C: 8 x 8 register blocks.
// fp32 n = 32 / 64 packed batches on the tensor pipe (k_small64.cuh
// small_mma_kernel); 0 = not eligible.  SBT_SMALL_MMA=0 keeps the FFMA kernels.
template <int S>
static int try_small_mma(const GemmParams<float>& p, cudaStream_t stream) {
  using namespace small64mma;
  using C_ = Cfg<S>;
  static const int on = env_int("SBT_SMALL_MMA", env_int("SBT_SMALL64_MMA", 1));
  if (!on) return 0;
  if (p.m != S || p.n != S || p.k != S) return 0;
  if (!(p.ars == 1 && p.acs == S && p.brs == 1 && p.bcs == S && p.crs == 1 && p.ccs == S))
    return 0;
  if (p.aps % 4 || p.bps % 4 || p.aps < S * S || p.bps < S * S || !aligned16(p.a) ||
      !aligned16(p.b) || p.batch > (int64_t(1) << 31))
    return 0;
  auto kern = small_mma_kernel<S>;
  if (set_smem_attr(reinterpret_cast<const void*>(kern), C_::SMEM_BYTES) != 0) return -3;
  CUtensorMap ta, tb;
  if (!make_tmap_f32(&ta, p.a, S, S, S, p.batch, p.aps, 1, 0, C_::LDA, S,
                     CU_TENSOR_MAP_SWIZZLE_NONE, C_::G) ||
      !make_tmap_f32(&tb, p.b, S, S, S, p.batch, p.bps, 1, 0, C_::LDB, S,
                     CU_TENSOR_MAP_SWIZZLE_NONE, C_::G))
    return 0;
  const int64_t ngroups = ceil_div(p.batch, C_::G);
  const int64_t cap = int64_t(kNumSMs) * C_::CTAS_PER_SM;
  const int64_t grid = ngroups < cap ? ngroups : cap;
  kern<<<dim3(unsigned(grid)), dim3(C_::kThreads), C_::SMEM_BYTES, stream>>>(p, ta, tb, ngroups);
  note_launch(S == 64 ? "small64_mma_f32" : "small32_mma_f32");
  return 1;
}

static int try_small64(const GemmParams<float>& p, cudaStream_t stream) {
  using namespace small64;
  if (p.m != 64 || p.n != 64 || p.k != 64) return 0;
  if (!(p.ars == 1 && p.acs == 64 && p.brs == 1 && p.bcs == 64 && p.crs == 1 && p.ccs == 64))
    return 0;
  if (p.aps % 4 || p.bps % 4 || p.aps < 4096 || p.bps < 4096 || !aligned16(p.a) ||
      !aligned16(p.b) || p.batch > (int64_t(1) << 31))
    return 0;
  {
    const int rc = try_small_mma<64>(p, stream);
    if (rc != 0) return rc;
  }
  if (set_smem_attr(reinterpret_cast<const void*>(small64_kernel), SMEM_BYTES) != 0) return -3;
  CUtensorMap ta, tb;
  if (!make_tmap_f32(&ta, p.a, 64, 64, 64, p.batch, p.aps, 1, 0, 64, 64,
                     CU_TENSOR_MAP_SWIZZLE_NONE, G) ||
      !make_tmap_f32(&tb, p.b, 64, 64, 64, p.batch, p.bps, 1, 0, LDB, 64,
                     CU_TENSOR_MAP_SWIZZLE_NONE, G))
    return 0;
  const int64_t ngroups = ceil_div(p.batch, G);
  const int64_t cap = int64_t(kNumSMs) * CTAS_PER_SM;
  const int64_t grid = ngroups < cap ? ngroups : cap;
  small64_kernel<<<dim3(unsigned(grid)), dim3(kThreads), SMEM_BYTES, stream>>>(p, ta, tb,
                                                                              ngroups);
  note_launch("small64_f32");
  return 1;
}

// Many tiny dense matrices: every extent <= 64, each matrix stored densely.
template <typename T>
static int try_small(const GemmParams<T>& p, cudaStream_t stream, bool forced) {
  const int64_t mx = p.m > p.n ? (p.m > p.k ? p.m : p.k) : (p.n > p.k ? p.n : p.k);
  if (mx > 64 || p.batch2 != 1) return 0;
  if (!forced && p.batch < 512) return 0;
  const bool am = p.ars == 1 && p.acs == p.m, ak = p.acs == 1 && p.ars == p.k;
  const bool bk = p.brs == 1 && p.bcs == p.k, bn = p.bcs == 1 && p.brs == p.n;
  if (!(am || ak) || !(bk || bn) || !(p.crs == 1 && p.ccs == p.m)) return 0;
  if (!vmult<T>(p.m * p.k) || !vmult<T>(p.k * p.n) || !vmult<T>(p.aps) || !vmult<T>(p.bps) ||
      !aligned16(p.a) || !aligned16(p.b))
    return 0;
  if constexpr (sizeof(T) == 4) {
    static const int use64 = env_int("SBT_SMALL64", 1);
    if (use64 && mx == 64) {
      const int rc = try_small64(p, stream);
      if (rc != 0) return rc;
    }
    if (mx == 32) {
      const int rc = try_small_mma<32>(p, stream);
      if (rc != 0) return rc;
    }
  }
  if constexpr (sizeof(T) == 8) {
    static const int use_dmma = env_int("SBT_SMALL_DMMA", 1);
    if (use_dmma && mx > 16 && mx <= 64) {
      const int rc = try_small_dmma(p, stream);
      if (rc != 0) return rc;
    }
  }
  if (mx <= 8) return launch_small_s<T, 8>(p, am, bk, stream);
  if (mx <= 16) return launch_small_s<T, 16>(p, am, bk, stream);
  if (mx <= 32) return launch_small_s<T, 32>(p, am, bk, stream);
  return launch_small_s<T, 64>(p, am, bk, stream);
}

// ---- split-K for tall-skinny reductions --------------------------------------------
// A single output tile with a huge K (e.g. the Tucker HOSVD Gram matrices,
// 512 x 512 with K = 262144) leaves most SMs idle.  Split K into S contiguous
// chunks as a batched GEMM into a stream-ordered workspace, then reduce the S
// partials (fixed S and order: deterministic).
template <typename T>
__global__ void reduce_splits_kernel(const T* __restrict__ w, int64_t nsplit, int64_t m,
                                     int64_t n, T alpha, T beta, T* c, int64_t crs,
                                     int64_t ccs) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    T acc = T(0);
    for (int64_t s = 0; s < nsplit; ++s) acc += w[s * total + e];
    const int64_t i = e % m, j = e / m;
    store_out(c + i * crs + j * ccs, acc, alpha, beta);
  }
}

template <typename T>
static int launch_gemm_core(const GemmParams<T>& p, cudaStream_t stream);
template <typename T>
static int launch_chunked(const GemmParams<T>& p, cudaStream_t stream);

template <typename T>
static int try_split_k(const GemmParams<T>& p, cudaStream_t stream) {
  // fp64 (DMMA, 128x128 tiles, 4096 cycles per 16-deep K step): split as soon
  // as few tiles leave SMs idle -- the HOOI Grams (512 x 512, K = 1024) and the
  // Rayleigh-Ritz products (512 x 48 and 48 x 48, K = 512) would otherwise run
  // on 16 / 4 / 1 CTAs; fp32 tiles are larger and faster, so only very long
  // reductions split
  const int64_t min_k = sizeof(T) == 8 ? 256 : 16384, min_chunk = sizeof(T) == 8 ? 64 : 4096;
  if (p.batch != 1 || p.batch2 != 1 || p.k < min_k || p.m == 1 || p.n == 1) return 0;
  const int64_t tiles = ceil_div(p.m, 128) * ceil_div(p.n, 128);
  if (tiles >= kNumSMs / 2) return 0;
  int64_t S = (2 * kNumSMs) / tiles;
  const int64_t max_s = p.k / min_chunk;
  if (S > max_s) S = max_s;
  if (S < 2) return 0;
  // chunk length: multiple of 32 so every chunk keeps the operands' alignment
  const int64_t kc = ((ceil_div(p.k, S) + 31) / 32) * 32;
  if (kc >= p.k) return 0;
  S = ceil_div(p.k, kc);
  T* w = nullptr;
  static bool pool_kept = [] {  // keep freed workspaces in the stream-ordered pool
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~uint64_t(0);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return true;
  }();
  (void)pool_kept;
  {
    const cudaError_t e =
        cudaMallocAsync(reinterpret_cast<void**>(&w), size_t(S) * p.m * p.n * sizeof(T), stream);
    if (e != cudaSuccess) return cuda_fail(e, "split-K workspace (cudaMallocAsync)");
  }
  GemmParams<T> q = p;
  q.alpha = T(1); q.beta = T(0);
  q.c = w; q.crs = 1; q.ccs = p.m; q.cps = p.m * p.n;
  const bool even = p.k == S * kc;
  q.k = kc; q.batch = even ? S : S - 1;   // full chunks
  q.aps = kc * p.acs; q.bps = kc * p.brs;
  int rc = 0;
  if (q.batch > 0) rc = launch_chunked<T>(q, stream);
  if (rc == 0 && !even) {                 // ragged last chunk
    GemmParams<T> t = q;
    t.batch = 1; t.k = p.k - (S - 1) * kc;
    t.a = p.a + (S - 1) * kc * p.acs; t.b = p.b + (S - 1) * kc * p.brs;
    t.c = w + (S - 1) * p.m * p.n;
    rc = launch_chunked<T>(t, stream);
  }
  if (rc == 0) {
    const int64_t total = p.m * p.n;
    const int64_t blocks = ceil_div(total, 256) < 4096 ? ceil_div(total, 256) : 4096;
    reduce_splits_kernel<T><<<unsigned(blocks), 256, 0, stream>>>(w, S, p.m, p.n, p.alpha,
                                                                  p.beta, p.c, p.crs, p.ccs);
    note_launch("split_k_reduce");
  }
  cudaFreeAsync(w, stream);
  return rc < 0 ? rc : 1;
}

// fp32 accuracy guard for long reductions.  The tensor core truncates its fp32
// accumulator on every MMA, a bias that grows linearly with K (measured 3xTF32
// max_rel_err with the split small-term accumulator: 3.3e-6 at K=1024, 6.8e-6
// at K=2048, 1.1e-5 at K=4096).  Longer reductions run as K-chunks of at most
// kMaxChunkK, the first with the caller's beta, the rest accumulating into C
// (beta = 1): the cross-chunk sums are round-to-nearest fp32 adds, so the error
// stays at the K = kMaxChunkK level for any K.
constexpr int64_t kMaxChunkK = 2048;

template <typename T>
static int launch_chunked(const GemmParams<T>& p, cudaStream_t stream) {
  if constexpr (sizeof(T) == 4) {
    if (p.k > kMaxChunkK) {
      const int64_t nch = ceil_div(p.k, kMaxChunkK);
      const int64_t kc = ceil_div(ceil_div(p.k, nch), 32) * 32;  // keep 16 B alignment
      for (int64_t k0 = 0; k0 < p.k; k0 += kc) {
        GemmParams<T> q = p;
        q.k = (p.k - k0) < kc ? (p.k - k0) : kc;
        q.a = p.a + k0 * p.acs;
        q.b = p.b + k0 * p.brs;
        if (k0 > 0) q.beta = T(1);
        const int rc = launch_gemm_core<T>(q, stream);
        if (rc != 0) return rc;
      }
      return 0;
    }
  }
  return launch_gemm_core<T>(p, stream);
}

// fp64 skinny products (no batch, N <= 64 in one orientation, enough work to
// matter): 64 x 32 DMMA tiles, in-kernel deterministic split-K (k_skinny_dmma).
static void keep_pool_memory() {
  static bool done = [] {  // keep freed workspaces in the stream-ordered pool
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~uint64_t(0);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return true;
  }();
  (void)done;
}

template <bool AK, bool BK_>
static int launch_skinny_cfg(const GemmParams<double>& p, cudaStream_t stream) {
  using namespace skinny;
  auto kern = skinny_dmma_kernel<AK, BK_>;
  if (set_smem_attr(reinterpret_cast<const void*>(kern), SMEM_BYTES) != 0) return -3;
  const int64_t tiles_m = ceil_div(p.m, BM), tiles = tiles_m * ceil_div(p.n, BN);
  const int64_t nz = p.batch * p.batch2;
  if (tiles > 65535 * 16 || nz > 65535) return 0;
  // splits (unbatched only): fill ~2 waves of CTAs, at least 2 K-chunks per split
  int64_t S = nz > 1 ? 1 : (2 * kNumSMs + tiles - 1) / tiles;
  const int64_t max_s = p.k / (2 * KC);
  if (S > max_s) S = max_s;
  if (S > 64) S = 64;
  if (S < 1) S = 1;
  const int64_t kper = ceil_div(ceil_div(p.k, S), KC) * KC;
  S = ceil_div(p.k, kper);
  double* ws = nullptr;
  unsigned* cnt = nullptr;
  if (S > 1) {
    keep_pool_memory();
    const size_t wbytes = size_t(tiles) * S * TILE * sizeof(double);
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws),
                                          wbytes + tiles * sizeof(unsigned), stream);
    if (e != cudaSuccess) return cuda_fail(e, "skinny split-K workspace (cudaMallocAsync)");
    cnt = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ws) + wbytes);
    cudaMemsetAsync(cnt, 0, tiles * sizeof(unsigned), stream);
  }
  kern<<<dim3(unsigned(tiles), unsigned(S), unsigned(nz)), NT, SMEM_BYTES, stream>>>(
      p, int(tiles_m), kper, ws, cnt);
  note_launch("skinny_dmma_f64");
  if (ws) cudaFreeAsync(ws, stream);
  return 1;
}

static int try_skinny_f64(const GemmParams<double>& p0, cudaStream_t stream) {
  static const int enabled = env_int("SBT_SKINNY", 1);
  if (!enabled || p0.m == 1 || p0.n == 1) return 0;
  // batched: only when every entry fills a 64-row tile (the narrow side <= 64
  // would waste most of a 128 x 128 DMMA tile)
  if ((p0.batch > 1 || p0.batch2 > 1) && (p0.m < 64 && p0.n < 64)) return 0;
  // many tiny matrices belong to the K3 small-matrix kernels
  if (p0.batch >= 512 && p0.batch2 == 1 && p0.m <= 64 && p0.n <= 64 && p0.k <= 64) return 0;
  // orientation with the narrow side as N
  const GemmParams<double> p = (p0.n <= skinny::BN * 2 || p0.m > skinny::BN * 2) ? p0
                                                                                  : transposed(p0);
  if (p.n > 2 * skinny::BN || p.m < 16 || p.k < 32) return 0;
  if (double(p.m) * p.n * p.k < 2e5) return 0;  // tiny: the generic kernel
  const bool ak = p.acs == 1, amn = p.ars == 1;
  const bool bk = p.brs == 1, bn = p.bcs == 1;
  if (!(ak || amn) || !(bk || bn)) return 0;
  if (ak && bk) return launch_skinny_cfg<true, true>(p, stream);
  if (ak) return launch_skinny_cfg<true, false>(p, stream);
  if (bk) return launch_skinny_cfg<false, true>(p, stream);
  return launch_skinny_cfg<false, false>(p, stream);
}

template <typename T>
static int launch_gemm(const GemmParams<T>& p, cudaStream_t stream) {
  if constexpr (sizeof(T) == 8) {
    if (kernel_override() == 0) {
      const int rc = try_skinny_f64(p, stream);
      if (rc != 0) return rc < 0 ? rc : 0;
    }
  }
  if (kernel_override() == 0) {
    const int rc = try_split_k<T>(p, stream);
    if (rc < 0) return rc;
    if (rc == 1) return 0;
  }
  return launch_chunked<T>(p, stream);
}

// GEMV-shaped calls (one of M, N is 1): bandwidth-bound streaming kernels
template <typename T>
static int try_gemv(const GemmParams<T>& p0, cudaStream_t stream) {
  if (p0.n != 1 && p0.m != 1) return 0;
  const GemmParams<T> p = p0.n == 1 ? p0 : transposed(p0);
  if (p.n != 1) return 0;
  if (p.acs == 1 && p.ars != 1) {
    const int64_t warps = p.m * p.batch * p.batch2;
    const int64_t blocks = ceil_div(warps, gemv::kThreads / 32);
    const int64_t grid = blocks < int64_t(kNumSMs) * 16 ? blocks : int64_t(kNumSMs) * 16;
    gemv::gemv_dot_kernel<T><<<unsigned(grid), gemv::kThreads, 0, stream>>>(p);
    note_launch(sizeof(T) == 4 ? "gemv_dot_f32" : "gemv_dot_f64");
  } else {
    const int64_t nblk = ceil_div(p.m, gemv::kThreads);
    const int64_t work = nblk * p.batch * p.batch2;
    const int64_t grid = work < int64_t(kNumSMs) * 16 ? work : int64_t(kNumSMs) * 16;
    gemv::gemv_rows_kernel<T><<<unsigned(grid), gemv::kThreads, 0, stream>>>(p, nblk);
    note_launch(sizeof(T) == 4 ? "gemv_rows_f32" : "gemv_rows_f64");
  }
  return 1;
}

template <typename T>
static int launch_gemm_core(const GemmParams<T>& p, cudaStream_t stream) {
  const int ov = kernel_override();
  if (ov == 0) {
    const int rc = try_gemv<T>(p, stream);
    if (rc < 0) return rc;
    if (rc == 1) return 0;
  }
  if (ov == 0 || ov == 3) {
    const int rc = try_small<T>(p, stream, ov == 3);
    if (rc < 0) return rc;
    if (rc == 1) return 0;
  }
  if (ov == 0 || ov == 2) {
    int rc;
    if constexpr (sizeof(T) == 4) rc = try_tensor_f32(p, stream, ov == 2);
    else rc = try_tensor_f64(p, stream, ov == 2);
    if (rc < 0) return rc;
    if (rc == 1) return 0;
  }
  launch_generic<T>(p, stream);
  return 0;
}

}  // namespace sbt
