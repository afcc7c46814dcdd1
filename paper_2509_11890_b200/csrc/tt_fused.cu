// tt_fused.cu — launcher of the fused S1 -> S2 matvec kernel (tt_fused12.cuh): eligibility,
// the three tensor maps, unit count.  Called from enqueue_matvec (tt_core.cu).
#include "tt_internal.cuh"
#include "tt_launch_tpl.cuh"
#include "tt_fused12.cuh"

namespace ttint {

// tt_debug_set_fused: 0 policy (default), -1 never, m > 0 whenever eligible with warp-group
// skew {1, 0, 2}[(m - 1) % 3] k-tiles and option bits (m - 1) / 3 (tt_fused12.cuh)
thread_local int g_fused_mode = 0;

// 5-D FP64 view of the Krylov block X (a, j, m, b) for the phase-1 B operand: dims
// {16 (b lo), a (k), b / 16 (b hi), 4 (j), K (m)}, box {16, 16, 1, 4, 1}: one TMA brings the
// four swizzled 16 x 16 slabs (one per mode index j) of a k-tile.
static bool make_map_x(CUtensorMap* m, const double* X, long long a, long long N, long long K,
                       long long b) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[5] = {16u, (cuuint64_t)a, (cuuint64_t)(b / 16), (cuuint64_t)N, (cuuint64_t)K};
  cuuint64_t strides[4] = {(cuuint64_t)(N * K * b * 8), 128u, (cuuint64_t)(K * b * 8),
                           (cuuint64_t)(b * 8)};
  cuuint32_t box[5] = {16u, 16u, 1u, (cuuint32_t)N, 1u};
  cuuint32_t estr[5] = {1u, 1u, 1u, 1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(X), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool fused12_shape_ok(const Dims& d, long long K) {
  if (d.n != 4 || d.al > 36 || d.be > 36 || (4 * d.be) % 16 != 0) return false;
  if (d.b % 16 != 0 || d.a % 2 != 0 || K <= 0) return false;
  const long long units = ((d.a + 3) / 4) * (d.b / 16) * K;
  return units > 0 && units < (1LL << 31) - 1024 && d.a * d.al < (1LL << 31) &&
         d.a * K * 4 * d.be * d.b < (1LL << 62);
}

// The workspace is sized without T1 only under an explicit fused mode (TT_MATVEC_FUSED or a
// forced tt_debug_set_fused variant): there a misaligned operand is an error.
bool fused12_wanted(const Dims& d, long long K) {
  return g_fused_mode > 0 && fused12_shape_ok(d, K);
}

// TT_MATVEC_AUTO: the fused kernel where it was measured faster than the two stage GEMMs
// (tools/fused_probe.py, tools/iface_probe.py, tools/w5_fused_probe.py):
// every eligible core whose operator bond fills the kernel's 36-row a' blocks (Rl >= 28; at
// R = 16 / 20 / 24 the padded rows cost more than the fusion saves) and whose bonds give the
// 148 CTAs enough units.  The workspace keeps T1, so a misaligned operand falls back to the
// stage GEMMs.
bool fused12_auto(const Dims& d, long long K) {
  if (g_fused_mode != 0 || !fused12_shape_ok(d, K)) return false;
  return d.al >= 28 && d.a >= 64 && d.b >= 64;
}

// interface updates (their workspace always holds T1, so a misaligned operand just falls back)
bool fused12_iface_wanted(const Dims& d) {
  if (g_fused_mode < 0 || !fused12_shape_ok(d, 1)) return false;
  return g_fused_mode > 0 || fused12_auto(d, 1);
}

template <int G, bool PW, bool RR = false>
static cudaError_t launch_fused12_g(const Dims& d, long long K, int stage_tag, tt::Fused12Params p,
                                    const CUtensorMap& tl, const CUtensorMap& tx,
                                    const CUtensorMap& ta, cudaStream_t s) {
  using Cfg = tt::F12Cfg<G>;
  if (cudaError_t e = smem_attr((const void*)tt::fused_s12_kernel<G, PW, RR>, (int)Cfg::kSmemBytes)) return e;
  p.nag = (int)((d.a + 2 * G - 1) / (2 * G));
  p.total_units = (int)((long long)p.nag * p.nbt * K);
  p.nag_div = tt::make_fastdiv((uint32_t)p.nag);
  const int grid = (int)std::min<long long>(p.total_units, (long long)num_sms() * (3 - G));
  g_stage = stage_tag;
  // traced as one record with 2 M N K = the flops of both stages
  const long long tr = trace_begin(-12 - (G == 1) - 2 * (G == 2 && !RR ? 1 : 0), d.a * K * d.b, 4 * d.al, d.a + 4 * d.be, s);
  if (cudaError_t e = launch_pdl(false, tt::fused_s12_kernel<G, PW, RR>, dim3(grid), dim3(Cfg::kThreads + (PW ? 32 : 0)),
                                 Cfg::kSmemBytes, s, tl, tx, ta, p))
    return e;
  trace_end(tr, s);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_fused12(const Dims& d, long long K, const double* phiL, const double* Ah,
                           const double* X, double* T2, cudaStream_t s, bool& ok, int stage_tag) {
  ok = false;
  if (!fused12_shape_ok(d, K)) return cudaSuccess;
  if (!aligned16(phiL) || !aligned16(Ah) || !aligned16(X) || !aligned16(T2)) return cudaSuccess;
  CUtensorMap tl, tx, ta;
  if (!make_map(&tl, phiL, d.a, d.a * d.al, d.a, 72)) return cudaSuccess;
  if (!make_map_x(&tx, X, d.a, d.n, K, d.b)) return cudaSuccess;
  if (!make_map3(&ta, Ah, d.n * d.be, d.al * d.n, d.n * d.be, 9)) return cudaSuccess;
  ok = true;
  tt::Fused12Params p;
  p.T2 = T2;
  p.a = (int)d.a;
  p.b = (int)d.b;
  p.al = (int)d.al;
  p.be = (int)d.be;
  p.K = (int)K;
  p.nbt = (int)(d.b / 16);
  p.KT1 = (int)((d.a + 15) / 16);
  p.KT2 = (int)((4 * d.al + 15) / 16);
  p.nbt_div = tt::make_fastdiv((uint32_t)p.nbt);
  {
    const int m = g_fused_mode > 0 ? g_fused_mode - 1 : 1;   // policy default: skew 0
    const int sk[3] = {1, 0, 2};
    p.skew = sk[m % 3];
    p.opt = m / 3;
  }
  p.dbg = g_dbg_flags;
  p.gate = g_gate;
  // option bit 1: two independent 6-warp CTAs per SM instead of one 12-warp CTA
  if (p.opt & 2) return launch_fused12_g<1, false>(d, K, stage_tag, p, tl, tx, ta, s);
  // Producer placement (config-5 interior core, K = 32): thread 0 of the first consumer warp
  // 7.00-7.15 ms (option bit 5), a 13th producer warp 6.84 ms (bit 6; 13 warps cap the kernel at
  // 128 registers), the refill rotating over the 12 consumer warps 6.80 ms (default).
  if (p.opt & 32) return launch_fused12_g<2, false>(d, K, stage_tag, p, tl, tx, ta, s);
  if (p.opt & 64) return launch_fused12_g<2, true>(d, K, stage_tag, p, tl, tx, ta, s);
  return launch_fused12_g<2, false, true>(d, K, stage_tag, p, tl, tx, ta, s);
}

}  // namespace ttint
