// tt_launch_tpl.cuh — the templated launchers of the three GEMM engines (tile configuration,
// split-K, tensor maps); instantiated once per operand layout in tt_launch_l{0..3}.cu so the
// four layouts compile in parallel.  Policy helpers live in tt_launch.cu.
#pragma once
#include "tt_internal.cuh"
#include "tt_gemm_v3.cuh"
#include <cudaTypedefs.h>

namespace ttint {

// ---- non-template policy helpers (tt_launch.cu) ----------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
bool make_map(CUtensorMap* m, const double* base, long long inner, long long outer, long long ld,
              int box_outer);
bool make_map3(CUtensorMap* m, const double* base, long long M, long long K, long long ld,
               int nslab);
int store_mode(bool a_kc, bool b_kc, const GemmParams& p);
int latency_choice(const GemmParams& p, bool a_kc, bool b_kc, int& ks_out);

struct TileCand {
  int id, bm, bn, warps, minb;
  double eff;
};
// threshold swept on the W5 sweep (TT_LAT_FLOPS, profiles/r01e/latflops*.log): 5 GFLOP brings
// the config-5 interface-update stages (2.7-4.8 GFLOP, 3.5-3.9 waves of default tiles) under
// the model: update 0.443 -> 0.430 ms, W5 -0.1 %; 10 GFLOP adds the first stage of cores 3 / 8
// (9.7 GFLOP, K = 64): W5 another -0.07 %; 3 GFLOP neutral, 25 GFLOP +0.1 %
constexpr double kLatencyFlops = 1.0e10;
constexpr TileCand kLatencyCands[] = {
    {10, 128, 64, 8, 2, 0.90}, {11, 64, 64, 8, 2, 0.83}, {12, 64, 64, 4, 4, 0.85},
    {13, 64, 32, 4, 4, 0.82},  {14, 32, 64, 4, 4, 0.82}, {15, 32, 32, 4, 4, 0.75},
    {16, 64, 112, 8, 2, 0.80}, {21, 64, 144, 8, 2, 0.85}, {17, 64, 48, 8, 2, 0.78},
    // one 16-warp CTA per SM: with a non-power-of-two split it fills 144 of 148 SMs where the
    // 128 x 64 tiles reach 128 (the K = 1 matvec's last stage at r = 256: 16 tiles x 9 splits)
    {18, 128, 128, 16, 1, 0.93},
    // (12-warp 128 x 144 / 128 x 96 and 6-warp 64 x 144 / 64 x 96 candidates were measured
    // and dropped: config-4 W34 0.73 -> 0.84 ms; the 6-warp tiles reach only 28 TF/s at scale)
};


// ----------------------------------------------------------------------------------------
// GEMM launch: tile configuration chosen from the stage's N extent
// ----------------------------------------------------------------------------------------
template <int BM, int BN, int BK, int WM, int WN, int ST, bool AK, bool BK_>
cudaError_t launch_cfg(const GemmParams& p0, cudaStream_t s) {
  using Cfg = tt::GemmCfg<BM, BN, BK, WM, WN, ST, AK, BK_>;
  auto kern = tt::dmma_gemm_kernel<BM, BN, BK, WM, WN, ST, AK, BK_>;
  if (cudaError_t attr_err = smem_attr((const void*)kern, (int)Cfg::kSmemBytes)) return attr_err;
  GemmParams p = p0;
  const long long tm = (p.M + BM - 1) / BM;
  p.tiles_n = (p.N + BN - 1) / BN;
  const long long tiles = tm * p.tiles_n;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const long long tr = trace_begin(BN, p.M, p.N, p.K, s);
  if (cudaError_t e = launch_pdl(2.0 * p.M * p.N * p.K <= pdl_flops(), kern, dim3((unsigned)tiles), dim3(Cfg::kThreads), Cfg::kSmemBytes, s, p))
    return e;
  trace_end(tr, s);
  ++g_launches;
  return cudaGetLastError();
}

template <bool AK, bool BK_>
cudaError_t launch_gemm_l(const GemmParams& p, cudaStream_t s) {
  // Narrow-N configurations keep the whole N extent of the operator-core stage in one tile
  // (N = n*R <= 160 in every config: 16, 36, 64, 100, 144); wide N uses 128x128 tiles.
  if (p.N <= 16) return launch_cfg<128, 16, 16, 8, 1, 4, AK, BK_>(p, s);
  if (p.N <= 40) return launch_cfg<128, 40, 16, 8, 1, 4, AK, BK_>(p, s);
  if (p.N <= 64) return launch_cfg<128, 64, 16, 4, 2, 4, AK, BK_>(p, s);
  if (p.N <= 104) return launch_cfg<128, 104, 16, 8, 1, 4, AK, BK_>(p, s);
  if (p.N <= 144) return launch_cfg<128, 144, 16, 4, 2, 4, AK, BK_>(p, s);
  return launch_cfg<128, 128, 16, 2, 4, 4, AK, BK_>(p, s);
}


constexpr int stages_for(size_t stage_bytes, size_t budget) {
  return (int)(budget / stage_bytes) > 4 ? 4 : (int)(budget / stage_bytes);
}

template <bool AK, bool BK_, int BM, int BN, int WM, int WN, int MINB>
cudaError_t launch_v2_cfg(const GemmParams& p0, cudaStream_t s) {
  using Probe = tt::GemmV2Cfg<AK, BK_, BM, BN, WM, WN, 1, MINB>;
  constexpr size_t budget = MINB == 1 ? 220 * 1024 : 110 * 1024;
  constexpr int ST = stages_for(Probe::kSmemBytes, budget);
  static_assert(ST >= 2, "shared memory budget");
  using Cfg = tt::GemmV2Cfg<AK, BK_, BM, BN, WM, WN, ST, MINB>;
  auto kern = tt::dmma_gemm_v2_kernel<AK, BK_, BM, BN, WM, WN, ST, MINB>;
  if (cudaError_t attr_err = smem_attr((const void*)kern, (int)Cfg::kSmemBytes)) return attr_err;
  tt::GemmParamsV2 p;
  p.A = p0.A;
  p.B = p0.B;
  p.C = p0.C;
  p.P = nullptr;
  p.dbg = g_dbg_flags;
  p.gate = p0.gate;
  p.M = (int)p0.M;
  p.N = (int)p0.N;
  p.K = (int)p0.K;
  p.lda = p0.lda;
  p.ldb = p0.ldb;
  p.rowmap = tt::to_map32(p0.rowmap);
  p.colmap = tt::to_map32(p0.colmap);
  const long long tm = (p0.M + BM - 1) / BM;
  const long long tn = (p0.N + BN - 1) / BN;
  const long long tiles = tm * tn;
  p.tiles_n = (int)tn;
  p.KT = (int)((p0.K + Cfg::BK - 1) / Cfg::BK);
  // split-K when the tile count quantises badly onto the persistent CTAs (e.g. the
  // matvec's last stage: 512 tiles on 148 SMs = 3.46 waves) and K is long enough
  const long long slots = (long long)num_sms() * MINB;
  int ks = 1;
  double best = 0.0;
  for (int cand = 1; cand <= 4; ++cand) {
    if (cand > 1 && (p.KT / cand < 24 || g_pscratch == nullptr ||
                     (long long)cand * p0.M * p0.N > g_pscratch_elems))
      break;
    const long long units = tiles * cand;
    const long long waves = (units + slots - 1) / slots;
    const double eff = (double)units / (double)(waves * slots) * (cand == 1 ? 1.0 : 0.97);
    if (eff > best + 1e-9) {
      best = eff;
      ks = cand;
    }
  }
  // no empty K-split: the unit stream assumes every unit has at least one k-tile
  ks = (p.KT + (p.KT + ks - 1) / ks - 1) / ((p.KT + ks - 1) / ks);
  p.ksplit = ks;
  p.kt_per_split = (p.KT + ks - 1) / ks;
  p.total_units = (int)(tiles * ks);
  if (ks > 1) p.P = g_pscratch;
  const int grid = (int)std::min<long long>((long long)p.total_units, slots);
  const long long tr = trace_begin(BN + 1000 * ks, p0.M, p0.N, p0.K, s);
  if (cudaError_t e = launch_pdl(2.0 * p0.M * p0.N * p0.K <= pdl_flops(), kern, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmemBytes, s, p))
    return e;
  if (ks > 1) {
    const long long mn = p0.M * p0.N;
    long long blocks = (mn / 2 + 255) / 256;   // two columns per thread
    if (blocks > 8L * num_sms()) blocks = 8L * num_sms();
    if (blocks < 1) blocks = 1;
    if (cudaError_t e = launch_pdl(2.0 * p0.M * p0.N * p0.K <= pdl_flops(), tt::splitk_reduce_kernel,
                                   dim3((unsigned)blocks), dim3(256), 0,
                                   s, (const double*)p.P, p.C, p.M, p.N, ks, p.rowmap, p.colmap,
                                   tt::make_fastdiv((uint32_t)p.N), p.gate))
      return e;
    ++g_launches;
  }
  trace_end(tr, s);
  ++g_launches;
  return cudaGetLastError();
}

template <bool AK, bool BK_>
cudaError_t launch_v2_l(const GemmParams& p, cudaStream_t s) {
  const int v = g_variant < 0 ? 1 : g_variant;
  if (v == 0) {   // one 512-thread CTA per SM, BM = 128
    if (p.N <= 16) return launch_v2_cfg<AK, BK_, 128, 16, 16, 1, 1>(p, s);
    if (p.N <= 40) return launch_v2_cfg<AK, BK_, 128, 40, 16, 1, 1>(p, s);
    if (p.N <= 64) return launch_v2_cfg<AK, BK_, 128, 64, 8, 2, 1>(p, s);
    if (p.N <= 104) return launch_v2_cfg<AK, BK_, 128, 104, 16, 1, 1>(p, s);
    if (p.N <= 144) return launch_v2_cfg<AK, BK_, 128, 144, 8, 2, 1>(p, s);
    return launch_v2_cfg<AK, BK_, 128, 128, 4, 4, 1>(p, s);
  }
  // two 256-thread CTAs per SM (independent barriers: one CTA's epilogue and pipeline
  // bubbles overlap the other's DMMA stream)
  if (p.N <= 16) return launch_v2_cfg<AK, BK_, 64, 16, 8, 1, 2>(p, s);
  if (p.N <= 40) return launch_v2_cfg<AK, BK_, 64, 40, 8, 1, 2>(p, s);
  if (p.N <= 64) return launch_v2_cfg<AK, BK_, 64, 64, 4, 2, 2>(p, s);
  if (p.N <= 104) return launch_v2_cfg<AK, BK_, 64, 104, 8, 1, 2>(p, s);
  if (p.N <= 144) return launch_v2_cfg<AK, BK_, 64, 144, 4, 2, 2>(p, s);
  return launch_v2_cfg<AK, BK_, 128, 64, 4, 2, 2>(p, s);
}


// RR (round-robin producer, tt_gemm_v3.cuh) by default on tiles of 8 and more warps: the
// 4-warp latency tiles of configs 2 / 3 lost 3 % with it (W34 87 -> 90 us, 152 -> 156 us; its
// extra block barrier after the prologue), the 8- to 16-warp tiles gain 1-2 %.
template <bool AK, bool BK_, int BM, int BN, int WM, int WN, int MINB, bool BRES = false,
          bool RR = (WM * WN >= 8)>
cudaError_t launch_v3_cfg(const GemmParams& p0, cudaStream_t s, bool& ok) {
  using Probe = tt::GemmV3Cfg<AK, BK_, BM, BN, WM, WN, 1, MINB, BRES>;
  constexpr size_t budget = (MINB == 1 ? 224 : MINB == 2 ? 110 : 54) * 1024 - 1024;
  constexpr int ST0 = (int)((budget - Probe::BRES_BYTES) / Probe::STAGE_BYTES);
  constexpr int ST = ST0 > 6 ? 6 : ST0;
  static_assert(ST >= 2, "shared memory budget");
  using Cfg = tt::GemmV3Cfg<AK, BK_, BM, BN, WM, WN, ST, MINB, BRES>;
  ok = false;
  CUtensorMap ta, tb;
  // A: K-contiguous -> inner K, outer M (box rows BM); M-contiguous -> inner M, outer K (box 16)
  const bool use3d = !(g_dbg_flags & 128);
  const bool a3d = !AK && use3d && make_map3(&ta, p0.A, p0.M, p0.K, p0.lda, BM / 16);
  const bool b3d = !BK_ && use3d && make_map3(&tb, p0.B, p0.N, p0.K, p0.ldb, BN / 16);
  if (!a3d &&
      !(AK ? make_map(&ta, p0.A, p0.K, p0.M, p0.lda, BM) : make_map(&ta, p0.A, p0.M, p0.K, p0.lda, 16)))
    return cudaSuccess;
  if (!b3d &&
      !(BK_ ? make_map(&tb, p0.B, p0.K, p0.N, p0.ldb, BN) : make_map(&tb, p0.B, p0.N, p0.K, p0.ldb, 16)))
    return cudaSuccess;
  if (BRES && (!b3d || p0.N > BN || (p0.K + 15) / 16 > tt::kBresMaxKT)) return cudaSuccess;
  ok = true;
  auto kern = tt::dmma_gemm_v3_kernel<AK, BK_, BM, BN, WM, WN, ST, MINB, BRES, RR>;
  if (cudaError_t attr_err = smem_attr((const void*)kern, (int)Cfg::kSmemBytes)) return attr_err;
  tt::GemmParamsV3 p;
  p.C = p0.C;
  p.P = nullptr;
  p.dbg = g_dbg_flags;
  p.gate = p0.gate;
  // warp skew (tt_gemm_v3.cuh): 1 k-tile for the 16-warp tiles (W5 sweep -0.18 % in a
  // one-process A/B, S1 +0.4 %); debug bit 16384 disables it, bit 32768 sets 2 k-tiles
  p.skew = (Cfg::kWarps >= 12 && ST >= 4 && !(g_dbg_flags & 16384))
               ? ((g_dbg_flags & 32768) ? 2 : 1) : 0;
  p.M = (int)p0.M;
  p.N = (int)p0.N;
  p.K = (int)p0.K;
  p.rowmap = tt::to_map32(p0.rowmap);
  p.colmap = tt::to_map32(p0.colmap);
  p.store_mode = store_mode(AK, BK_, p0);
  p.a3d = a3d ? 1 : 0;
  p.b3d = b3d ? 1 : 0;
  // L2 policies: an operand that fits comfortably in L2 and is re-read by many tiles is kept
  // (evict_last); an operand larger than L2 is streamed (evict_first) when that protects a
  // kept partner of some size (a streamed operand with a tiny partner gains nothing and was
  // measured to lose ~1% on config 5's S2).  Config 5: S3 +1.5% (T2 streamed, PhiR kept),
  // S2 +0.6% (A-hat kept).
  {
    const long long a_bytes = 8LL * (AK ? p0.M * p0.lda : p0.K * p0.lda);
    const long long b_bytes = 8LL * (BK_ ? p0.N * p0.ldb : p0.K * p0.ldb);
    const long long a_reads = (p0.N + BN - 1) / BN, b_reads = (p0.M + BM - 1) / BM;
    const long long l2_keep = 80LL << 20, l2_size = 126LL << 20;
    p.l2_a = (g_dbg_flags & 16) || a_reads < 2 || a_bytes > l2_keep ? 0 : 1;
    p.l2_b = (g_dbg_flags & 16) || b_reads < 2 || b_bytes > l2_keep ? 0 : 1;
    if (p.l2_a == 1 && p.l2_b == 1 && a_bytes + b_bytes > l2_keep) {
      if (a_bytes > b_bytes) p.l2_a = 0; else p.l2_b = 0;
    }
    const long long min_protect = 4LL << 20;
    if (!(g_dbg_flags & 16)) {
      if (a_bytes > l2_size && p.l2_b == 1 && b_bytes >= min_protect) p.l2_a = 2;
      if (b_bytes > l2_size && p.l2_a == 1 && a_bytes >= min_protect) p.l2_b = 2;
    }
    if (g_dbg_flags & 32) { if (p.l2_a == 2) p.l2_a = 0; if (p.l2_b == 2) p.l2_b = 0; }
    if (g_dbg_flags & 64) { if (p.l2_a == 1) p.l2_a = 0; if (p.l2_b == 1) p.l2_b = 0; }
#ifdef TT_DEBUG_HOOKS
    static const bool l2_debug = getenv("TT_L2_DEBUG") != nullptr;
#else
    constexpr bool l2_debug = false;
#endif
    if (l2_debug)
      fprintf(stderr, "v3 %dx%d M=%lld N=%lld K=%lld AK=%d BK=%d a=%lldMB(r%lld,p%d) b=%lldMB(r%lld,p%d)\n",
              BM, BN, (long long)p0.M, (long long)p0.N, (long long)p0.K, AK, BK_, a_bytes >> 20,
              a_reads, p.l2_a, b_bytes >> 20, b_reads, p.l2_b);
  }
  p.store_mode = store_mode(AK, BK_, p0);
  const long long tm = (p0.M + BM - 1) / BM;
  const long long tn = (p0.N + BN - 1) / BN;
  const long long tiles = tm * tn;
  p.tiles_n = (int)tn;
  p.tiles_n_div = tt::make_fastdiv((uint32_t)tn);
  p.tiles_m = (int)tm;
  p.group_m = (g_dbg_flags & 512) ? 8 : (g_dbg_flags & 1024) ? (int)tm : 1;
  p.KT = (int)((p0.K + Cfg::BK - 1) / Cfg::BK);
  const long long slots = (long long)num_sms() * MINB;
  // Split-K choice from a small cost model: GEMM time = waves x (k-tiles per unit) x
  // (k-tile time), plus the deterministic reduction (reads ks*M*N, writes M*N doubles).
  // Big stages rarely split (only to fix wave quantisation); skinny ones (few output tiles,
  // long K — e.g. config 4's last matvec stage, 4 tiles x 200 k-tiles) split up to 64 ways.
  int ks = 1;
  if (BRES) {   // resident B: one N tile, whole K per unit
  } else if (g_force_ks > 0) {   // probe hook (tt_debug_set_variant >= 100)
    ks = g_force_ks;
    while (ks > 1 && (p.KT < ks || g_pscratch == nullptr ||
                      (long long)ks * p0.M * p0.N > g_pscratch_elems))
      --ks;
  } else {
    const double ktile_s = 2.0 * BM * BN * Cfg::BK / (37.0e12 / (double)slots);
    double best_t = 1e30;
    for (int cand = 1; cand <= 64; ++cand) {
      if (cand > 1 && (p.KT < 4 * cand || g_pscratch == nullptr ||
                       (long long)cand * p0.M * p0.N > g_pscratch_elems))
        break;
      const long long units = tiles * cand;
      const long long waves = (units + slots - 1) / slots;
      const long long kper = (p.KT + cand - 1) / cand;
      double t = (double)waves * (double)kper * ktile_s + 2.0e-6 * waves;
      if (cand > 1) t += (double)(cand + 1) * p0.M * p0.N * 8.0 / 5.0e12 + 3.0e-6;
      if (t < best_t * 0.98) {
        best_t = t;
        ks = cand;
      }
    }
  }
  // no empty K-split: the unit stream assumes every unit has at least one k-tile
  ks = (p.KT + (p.KT + ks - 1) / ks - 1) / ((p.KT + ks - 1) / ks);
  p.ksplit = ks;
  p.kt_per_split = (p.KT + ks - 1) / ks;
  p.total_units = (int)(tiles * ks);
  if (ks > 1) p.P = g_pscratch;
  const int grid = (int)std::min<long long>((long long)p.total_units, slots);
  const long long tr = trace_begin(BN + 1000 * ks + 100000, p0.M, p0.N, p0.K, s);
  if (cudaError_t e = launch_pdl(2.0 * p0.M * p0.N * p0.K <= pdl_flops(), kern, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmemBytes, s, ta, tb, p))
    return e;
  if (ks > 1) {
    const long long mn = p0.M * p0.N;
    long long blocks = (mn / 2 + 255) / 256;   // two columns per thread
    if (blocks > 8L * num_sms()) blocks = 8L * num_sms();
    if (blocks < 1) blocks = 1;
    if (cudaError_t e = launch_pdl(2.0 * p0.M * p0.N * p0.K <= pdl_flops(), tt::splitk_reduce_kernel,
                                   dim3((unsigned)blocks), dim3(256), 0,
                                   s, (const double*)p.P, p.C, p.M, p.N, ks, p.rowmap, p.colmap,
                                   tt::make_fastdiv((uint32_t)p.N), p.gate))
      return e;
    ++g_launches;
  }
  trace_end(tr, s);
  ++g_launches;
  return cudaGetLastError();
}


template <bool AK, bool BK_>
cudaError_t launch_v3_l(const GemmParams& p, cudaStream_t s, bool& ok) {
  {
    int ks = 1;
    const int li = (g_variant < 10 && g_variant != 4) ? latency_choice(p, AK, BK_, ks) : -1;
    if (li >= 0) {
      struct KsScope {   // the planned split-K factor, for this launch only
        int saved;
        explicit KsScope(int k) : saved(g_force_ks) { g_force_ks = k; }
        ~KsScope() { g_force_ks = saved; }
      } ks_scope(ks);
      switch (kLatencyCands[li].id) {
        case 10: return launch_v3_cfg<AK, BK_, 128, 64, 4, 2, 2>(p, s, ok);
        case 11: return launch_v3_cfg<AK, BK_, 64, 64, 4, 2, 2>(p, s, ok);
        case 12: return launch_v3_cfg<AK, BK_, 64, 64, 2, 2, 4>(p, s, ok);
        case 13: return launch_v3_cfg<AK, BK_, 64, 32, 2, 2, 4>(p, s, ok);
        case 14: return launch_v3_cfg<AK, BK_, 32, 64, 2, 2, 4>(p, s, ok);
        case 15: return launch_v3_cfg<AK, BK_, 32, 32, 2, 2, 4>(p, s, ok);
        case 16: return launch_v3_cfg<AK, BK_, 64, 112, 8, 1, 2>(p, s, ok);
        case 17: return launch_v3_cfg<AK, BK_, 64, 48, 8, 1, 2>(p, s, ok);
        case 21: return launch_v3_cfg<AK, BK_, 64, 144, 4, 2, 2>(p, s, ok);
        case 18: return launch_v3_cfg<AK, BK_, 128, 128, 4, 4, 1>(p, s, ok);
        default: break;
      }
    }
  }
  if (g_variant >= 10) {   // probe hook: forced tile configuration (variant % 100)
    switch (g_variant % 100) {
      case 10: return launch_v3_cfg<AK, BK_, 128, 64, 4, 2, 2>(p, s, ok);
      case 11: return launch_v3_cfg<AK, BK_, 64, 64, 4, 2, 2>(p, s, ok);
      case 12: return launch_v3_cfg<AK, BK_, 64, 64, 2, 2, 4>(p, s, ok);
      case 13: return launch_v3_cfg<AK, BK_, 64, 32, 2, 2, 4>(p, s, ok);
      case 14: return launch_v3_cfg<AK, BK_, 32, 64, 2, 2, 4>(p, s, ok);
      case 15: return launch_v3_cfg<AK, BK_, 32, 32, 2, 2, 4>(p, s, ok);
      case 16: return launch_v3_cfg<AK, BK_, 64, 112, 8, 1, 2>(p, s, ok);
      case 17: return launch_v3_cfg<AK, BK_, 64, 48, 8, 1, 2>(p, s, ok);
      case 18: return launch_v3_cfg<AK, BK_, 128, 128, 4, 4, 1>(p, s, ok);
      case 19: return launch_v3_cfg<AK, BK_, 64, 128, 2, 4, 2>(p, s, ok);
      case 20: return launch_v3_cfg<AK, BK_, 128, 32, 4, 2, 2>(p, s, ok);
      case 21: return launch_v3_cfg<AK, BK_, 64, 144, 4, 2, 2>(p, s, ok);
      case 22: return launch_v3_cfg<AK, BK_, 32, 112, 2, 2, 4>(p, s, ok);
      case 23: return launch_v3_cfg<AK, BK_, 128, 144, 16, 1, 1>(p, s, ok);
      case 24: return launch_v3_cfg<AK, BK_, 128, 128, 8, 2, 1>(p, s, ok);
      case 25: return launch_v3_cfg<AK, BK_, 128, 128, 2, 8, 1>(p, s, ok);
      case 26: return launch_v3_cfg<AK, BK_, 128, 144, 4, 3, 1>(p, s, ok);
      case 27: return launch_v3_cfg<AK, BK_, 128, 144, 2, 6, 1>(p, s, ok);
      case 29: return launch_v3_cfg<AK, BK_, 128, 96, 4, 3, 1>(p, s, ok);
      case 31: return launch_v3_cfg<AK, BK_, 128, 128, 4, 2, 1>(p, s, ok);
      default: break;
    }
  }
  if (g_variant == 4) {   // all two-CTA tiles (previous default), kept for comparison
    if (p.N <= 16) return launch_v3_cfg<AK, BK_, 64, 16, 8, 1, 2>(p, s, ok);
    if (p.N <= 48) return launch_v3_cfg<AK, BK_, 64, 48, 8, 1, 2>(p, s, ok);
    if (p.N <= 64) return launch_v3_cfg<AK, BK_, 64, 64, 4, 2, 2>(p, s, ok);
    if (p.N <= 112) return launch_v3_cfg<AK, BK_, 64, 112, 8, 1, 2>(p, s, ok);
    if (p.N <= 144) return launch_v3_cfg<AK, BK_, 64, 144, 4, 2, 2>(p, s, ok);
    return launch_v3_cfg<AK, BK_, 128, 64, 4, 2, 2>(p, s, ok);
  }
  // Measured per stage shape (tools/stage_probe.py, config-5 interior core):
  //  * narrow N (the operator-core stage, N = n R <= 144): one 16-warp CTA per SM with a
  //    128 x N tile and a 6-deep TMA ring (the streamed operand comes from HBM);
  //  * wide N with a K-contiguous B (the last matvec stage): one 16-warp CTA per SM,
  //    128 x 128 tiles (+ split-K), 95% of the DMMA peak;
  //  * wide N with an N-contiguous B (the first stage): one 16-warp CTA per SM, 128 x 128
  //    (two 8-warp CTAs of 128 x 64 were the earlier choice; with the 3-D TMA slabs and L2
  //    hints the 128 x 128 tile is 1.2 % faster on the whole W5 sweep), warps 8 x 2 (16 x 64
  //    warp tiles: S1 +0.9 %, W5 -0.28 % against 4 x 4, tools/flags_ab.py 0 v6); since then
  //    one 12-warp CTA per SM with a 128 x 144 tile (warps 4 x 3 of 32 x 48), below.
  //  * 12 warps (3 per sub-partition, up to 168 registers) fit 32 x 48 warp tiles: 10
  //    fragment loads per 24 DMMAs instead of 10-11 per 16-18 (tools/stage_probe.py 26-31,
  //    tools/flags_ab.py 0 5242880: W5 sweep 105.65 -> 104.18 ms).
  if (p.N <= 16) return launch_v3_cfg<AK, BK_, 64, 16, 8, 1, 2>(p, s, ok);
  if (p.N <= 48) return launch_v3_cfg<AK, BK_, 64, 48, 8, 1, 2>(p, s, ok);
  // small problems: 64-row tiles on two CTAs per SM double the tile count
  const bool small = (p.M + 127) / 128 < (long long)num_sms() && p.N <= 144;
  if (small) {
    if (p.N <= 64) return launch_v3_cfg<AK, BK_, 64, 64, 4, 2, 2>(p, s, ok);
    if (p.N <= 112) return launch_v3_cfg<AK, BK_, 64, 112, 8, 1, 2>(p, s, ok);
    return launch_v3_cfg<AK, BK_, 64, 144, 4, 2, 2>(p, s, ok);
  }
  if (p.N <= 64) return launch_v3_cfg<AK, BK_, 128, 64, 8, 2, 1>(p, s, ok);
  if (p.N <= 112) return launch_v3_cfg<AK, BK_, 128, 112, 8, 2, 1>(p, s, ok);
  if (p.N <= 144) {
    // 12 warps of 32 x 48 (fewer fragment loads per DMMA than 8 x 2 warps of 16 x 72:
    // operator-core stage 33.5 -> 34.6 TFLOP/s, W5 sweep -0.6 %); bit 20 restores 8 x 2
    if (g_dbg_flags & 1048576) return launch_v3_cfg<AK, BK_, 128, 144, 8, 2, 1>(p, s, ok);
    if ((g_dbg_flags & 33554432) && !BK_ && (p.K + 15) / 16 <= tt::kBresMaxKT) {
      cudaError_t e = launch_v3_cfg<AK, BK_, 128, 144, 4, 3, 1, true>(p, s, ok);
      if (e != cudaSuccess || ok) return e;
    }
    if (g_dbg_flags & 2097152) return launch_v3_cfg<AK, BK_, 128, 144, 2, 6, 1>(p, s, ok);
    // round-robin producer (tt_gemm_v3.cuh RR): S1 / S2 / S3 of the config-5 interior matvec
    // 4.379 / 2.515 / 4.425 -> 4.328 / 2.466 / 4.360 ms; debug bit 30 restores thread 0
    if (g_dbg_flags & (1 << 30)) return launch_v3_cfg<AK, BK_, 128, 144, 4, 3, 1, false, false>(p, s, ok);
    return launch_v3_cfg<AK, BK_, 128, 144, 4, 3, 1>(p, s, ok);
  }
  if (BK_ && (g_dbg_flags & (1 << 30))) return launch_v3_cfg<AK, BK_, 128, 128, 4, 4, 1, false, false>(p, s, ok);
  if (BK_) return launch_v3_cfg<AK, BK_, 128, 128, 4, 4, 1>(p, s, ok);
  if (g_variant == 5) return launch_v3_cfg<AK, BK_, 128, 64, 4, 2, 2>(p, s, ok);   // probes
  if (g_variant == 6) return launch_v3_cfg<AK, BK_, 128, 128, 4, 4, 1>(p, s, ok);
  if (g_variant == 7) return launch_v3_cfg<AK, BK_, 64, 128, 2, 4, 2>(p, s, ok);
  // 128 x 144 tiles on 12 warps of 32 x 48 (first stage 34.0 -> 35.4 TFLOP/s, W5 sweep
  // -0.75 % on top of the operator-core change; bit 22 restores 128 x 128 on 8 x 2 warps)
  if (g_dbg_flags & 4194304) return launch_v3_cfg<AK, BK_, 128, 128, 8, 2, 1>(p, s, ok);
  if (g_dbg_flags & (1 << 30)) return launch_v3_cfg<AK, BK_, 128, 144, 4, 3, 1, false, false>(p, s, ok);
  return launch_v3_cfg<AK, BK_, 128, 144, 4, 3, 1>(p, s, ok);
}


// v3 (TMA) when eligible and a tensor map can be encoded, else v2 (16-byte cp.async), else v1
template <bool AK, bool BK_>
cudaError_t launch_layout(const GemmParams& p, cudaStream_t s) {
  const int v = g_variant < 0 ? 2 : g_variant;
  if (!g_force_v1 && v >= 2 && v2_eligible(AK, BK_, p)) {
    bool ok = false;
    cudaError_t e = launch_v3_l<AK, BK_>(p, s, ok);
    if (ok || e != cudaSuccess) return e;
  }
  if (!g_force_v1 && v2_eligible(AK, BK_, p)) return launch_v2_l<AK, BK_>(p, s);
  return launch_gemm_l<AK, BK_>(p, s);
}

extern template cudaError_t launch_layout<true, true>(const GemmParams&, cudaStream_t);
extern template cudaError_t launch_layout<true, false>(const GemmParams&, cudaStream_t);
extern template cudaError_t launch_layout<false, true>(const GemmParams&, cudaStream_t);
extern template cudaError_t launch_layout<false, false>(const GemmParams&, cudaStream_t);

}  // namespace ttint
