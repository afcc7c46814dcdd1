// tt_launch.cu — GEMM launch policy: tile configuration, split-K and the latency model for
// the DMMA engines of tt_gemm.cuh / tt_gemm_v2.cuh / tt_gemm_v3.cuh.
#include "tt_internal.cuh"
#include "tt_launch_tpl.cuh"

namespace ttint {

// ---- v2 (persistent, 16 warps, 16-byte loads) --------------------------------------------
int num_sms() {   // of the current device (cached per device and thread)
  constexpr int kMaxDev = 64;
  thread_local int sms[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 148;
  if (sms[dev] <= 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v > 0 ? v : 148;
  }
  return sms[dev];
}

thread_local int g_variant = -1;
thread_local int g_force_ks = 0;   // probe hook: split-K factor forced by tt_debug_set_variant
// device flag gating every GEMM launch of the calling thread (set by the iterative solvers
// around their matvecs so that iterations after convergence cost launches only)
thread_local const int* g_gate = nullptr;

// split-K scratch for the current stage (set by the stage planners; nullptr = no split)
thread_local double* g_pscratch = nullptr;
thread_local long long g_pscratch_elems = 0;

// ---- v3 (TMA + mbarrier pipeline) ---------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 2-D FP64 tensor map of a plain view: inner extent `inner` (unit stride), outer extent
// `outer` with stride `ld` doubles; box {16, box_outer}, 128-byte swizzle, zero OOB fill.
bool make_map(CUtensorMap* m, const double* base, long long inner, long long outer, long long ld,
              int box_outer) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {16u, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D view of an MN-contiguous operand: dims {16 (m_lo), K, M/16 (m_hi)}, strides
// {ld, 16} doubles, box {16, 16, nslab}: one TMA loads a whole BM x 16 tile as nslab
// swizzled 2 KB slabs.  Needs M % 16 == 0 (no element past M is ever addressed).
bool make_map3(CUtensorMap* m, const double* base, long long M, long long K, long long ld,
               int nslab) {
  if (M % 16 != 0 || (ld * 8) % 16 != 0) return false;
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {16u, (cuuint64_t)K, (cuuint64_t)(M / 16)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 8), 128u};
  cuuint32_t box[3] = {16u, 16u, (cuuint32_t)nslab};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool even_strides(const IndexMap& m) {
  return ((m.s0 | m.s1 | m.s2) & 1) == 0;
}
// 16-byte epilogue stores (tt_gemm_v3.cuh store_mode): the output must be contiguous in
// pairs along the paired fragment dimension, with every other offset even and C aligned.
int store_mode(bool a_kc, bool b_kc, const GemmParams& p) {
  if (reinterpret_cast<uintptr_t>(p.C) & 15) return 0;
  const IndexMap &r = p.rowmap, &c = p.colmap;
  // 32-byte stores: columns contiguous in aligned fours (measured: S1 +3 % with no stores at
  // all; the 16-byte pairs wrote every sector half by half in two instructions)
  auto quad = [](long long v) { return (v & 3) == 0; };
  auto quad_strides = [&](const IndexMap& m) {
    return quad(m.s0) && (m.d0 >= tt::kBig || quad(m.s1)) && (m.d0 >= tt::kBig || m.d1 >= tt::kBig || quad(m.s2));
  };
  if (!b_kc && !(g_dbg_flags & 131072) && !(reinterpret_cast<uintptr_t>(p.C) & 31) &&
      c.s0 == 1 && (c.d0 >= tt::kBig || (quad(c.d0) && quad(c.s1) && (c.d1 >= tt::kBig || quad(c.s2)))) &&
      quad_strides(r) && quad(p.N))
    return 3;
  if (!b_kc && c.s0 == 1 && (c.d0 & 1) == 0 && ((c.s1 | c.s2) & 1) == 0 && even_strides(r) &&
      (p.N & 1) == 0)
    return 1;
  if (!a_kc && r.s0 == 1 && (r.d0 & 1) == 0 && ((r.s1 | r.s2) & 1) == 0 && even_strides(c) &&
      (p.M & 1) == 0)
    return 2;
  return 0;
}

// ---- latency policy for small stage GEMMs (configs 3/4, boundary cores) -------------------
// A stage of a few tens of MFLOP is bound by how many SMs it occupies (one SM retires
// 37.2 TF / 148 = 251 GFLOP/s of DMMA), not by tile efficiency: config 3's interior left-update
// stages (~34 MFLOP) ran as 32-64 CTAs of 128 x 64.  For GEMMs below kLatencyFlops the tile
// configuration and split-K factor are chosen by a small model over a candidate list:
//   t = ceil(units / SMs) x k-tiles per unit x 2 BM BN 16 / (251 GF/s x eff x occ)
//       + ceil(units / SMs) x 3 us + split-K reduction (reads ks M N, writes M N doubles)
//       + a fixed 1 us if ks > 1  (occ = 1 by default; knobs below),
// eff = the configuration's measured fraction of peak at scale (tools/stage_probe.py, config-5
// interior shapes) and occ the warp-occupancy factor of a sparsely filled SM (a DMMA blocks
// its warp ~16 cycles; fewer than 2 warps per sub-partition leave the pipe idle).
// Debug flag 8192 disables it (A/B).
// model knobs (probe overrides: TT_LAT_FLOPS, TT_LAT_UNIT_US, TT_LAT_MASK = candidate bitmask
// to exclude), read once
struct LatKnobs {
  // unit_s: a per-unit cost (epilogue, pipeline refill, the smaller tiles' lower efficiency)
  // that favours fewer, larger units; swept on the W34 DAG (tools/w34_knobs.py): config 4
  // 0.808 ms (0 us) -> 0.761 (1 us) -> 0.750 (3 us), config 3 unchanged (0.173-0.176 ms)
  // split_s: fixed cost of a split-K reduction launch; occ_model: the warp-occupancy factor
  // (off: with the per-unit term it only cost config 3, 0.175 -> 0.165 ms without it)
  double flops = kLatencyFlops, unit_s = 3.0e-6, split_s = 1.0e-6;
  int occ_model = 0;
  unsigned mask = 0;
};
const LatKnobs& lat_knobs() {
  static LatKnobs k = [] {
    LatKnobs r;
#ifdef TT_DEBUG_HOOKS   // probe overrides exist only in a debug build
    if (const char* e = getenv("TT_LAT_FLOPS")) r.flops = atof(e);
    if (const char* e = getenv("TT_LAT_UNIT_US")) r.unit_s = atof(e) * 1e-6;
    if (const char* e = getenv("TT_LAT_MASK")) r.mask = (unsigned)strtoul(e, nullptr, 0);
    if (const char* e = getenv("TT_LAT_SPLIT_US")) r.split_s = atof(e) * 1e-6;
    if (const char* e = getenv("TT_LAT_OCC")) r.occ_model = atoi(e);
#endif
    return r;
  }();
  return k;
}

double latency_estimate(const TileCand& c, long long M, long long N, long long K, int ks) {
  const long long sms = num_sms();
  const long long tiles = ((M + c.bm - 1) / c.bm) * ((N + c.bn - 1) / c.bn);
  const long long KT = (K + 15) / 16;
  const long long kper = (KT + ks - 1) / ks;
  const long long units = tiles * ks;
  const long long grid = std::min<long long>(units, sms * c.minb);
  const long long per_sm = (units + sms - 1) / sms;
  const long long ctas_per_sm = std::min<long long>(c.minb, (grid + sms - 1) / sms);
  const long long w = ctas_per_sm * c.warps;
  const double occ = !lat_knobs().occ_model ? 1.0 : w >= 12 ? 1.0 : w >= 8 ? 0.9 : w >= 4 ? 0.6 : 0.35;
  double t = (double)per_sm * (double)kper * 2.0 * c.bm * c.bn * 16.0 / (251.0e9 * c.eff * occ);
  t += (double)per_sm * lat_knobs().unit_s;   // per-unit epilogue / pipeline refill
  if (ks > 1) t += (double)(ks + 1) * M * N * 8.0 / 5.0e12 + lat_knobs().split_s;
  return t;
}

// best (candidate index, ks) for a small GEMM, or -1 when the stage is not small
int latency_choice(const GemmParams& p, bool a_kc, bool b_kc, int& ks_out) {
  if (g_dbg_flags & 8192) return -1;
  if (2.0 * p.M * p.N * p.K > lat_knobs().flops) return -1;
  double best = 1e30;
  int bi = -1;
  const long long KT = (p.K + 15) / 16;
  for (int i = 0; i < (int)(sizeof(kLatencyCands) / sizeof(kLatencyCands[0])); ++i) {
    const TileCand& c = kLatencyCands[i];
    if (lat_knobs().mask & (1u << i)) continue;
    // the one-CTA-per-SM 128 x 128 tile only for the multi-GFLOP stages (config-5 interior,
    // K = 1): under config 4's concurrent chains it cost 10 % (W34 597 -> 654 us)
    if (c.id == 18 && 2.0 * p.M * p.N * p.K < 2.0e9) continue;
    (void)a_kc; (void)b_kc;   // every candidate's BM, BN are multiples of 16 (any operand layout)
    static const int kSplits[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 14, 16};
    for (int ks : kSplits) {
      if (ks > 1 && (KT < 2 * ks || g_pscratch == nullptr || (long long)ks * p.M * p.N > g_pscratch_elems))
        break;
      const double t = latency_estimate(c, p.M, p.N, p.K, ks);
      if (t < best * 0.97) {
        best = t;
        bi = i;
        ks_out = ks;
      }
    }
  }
  return bi;
}

bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

// the v2 preconditions (tt_gemm_v2.cuh header)
bool v2_eligible(bool a_kc, bool b_kc, const GemmParams& p) {
  const long long lim = (1LL << 31) - 256;
  if (p.M >= lim || p.N >= lim || p.K >= lim) return false;
  if (!aligned16(p.A) || !aligned16(p.B) || (p.lda & 1) || (p.ldb & 1)) return false;
  if (a_kc ? (p.K & 1) : (p.M & 1)) return false;
  if (b_kc ? (p.K & 1) : (p.N & 1)) return false;
  const long long tiles = ((p.M + 127) / 128) * ((p.N + 15) / 16);
  return tiles < lim;
}

thread_local int g_force_v1 = 0;   // test hook (tt_debug_force_v1)

cudaError_t launch_gemm(bool a_kc, bool b_kc, const GemmParams& p, cudaStream_t s) {
  if (p.M <= 0 || p.N <= 0 || p.K <= 0) return cudaSuccess;
  if (g_dag) return g_dag->add(a_kc, b_kc, p);   // recording a persistent DAG (tt_dag.cu)
  if (a_kc && b_kc) return launch_layout<true, true>(p, s);
  if (a_kc && !b_kc) return launch_layout<true, false>(p, s);
  if (!a_kc && b_kc) return launch_layout<false, true>(p, s);
  return launch_layout<false, false>(p, s);
}

GemmParams gp(const double* A, long long lda, const double* B, long long ldb, double* C,
              long long M, long long N, long long K, IndexMap rm, IndexMap cm) {
  GemmParams p;
  p.A = A;
  p.B = B;
  p.C = C;
  p.M = M;
  p.N = N;
  p.K = K;
  p.lda = lda;
  p.ldb = ldb;
  p.rowmap = rm;
  p.colmap = cm;
  p.tiles_n = 1;
  p.gate = g_gate;
  return p;
}

}  // namespace ttint
