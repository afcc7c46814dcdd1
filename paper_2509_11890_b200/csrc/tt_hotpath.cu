// tt_hotpath.cu — C-ABI (include/tt_hotpath.h) and stage plans of the TT hot path, sm_100a.
//
// Each ABI operation is a short sequence of kernels on the caller's stream:
//   * a permutation of the operator core A_k into the (contraction x output) GEMM layout
//     (a few KB; DESIGN.md §4 "P"),
//   * three DMMA GEMM stages (tt_gemm.cuh) = the paper's "three matrix products"
//     (§3.3), with the stage order chosen so that every operand is a plain
//     2-D view and every intermediate is written directly in the next stage's layout,
//   * a streaming kernel for the unrounded operator apply (H8).
// Index letters: a = r_k (rl), b = r_{k+1} (rr), al = R_k (Rl), be = R_{k+1}
// (Rr), N = mode size n, K = number of Krylov columns (nvec).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/tt_hotpath.h"
#include "tt_gemm.cuh"
#include "tt_gemm_v2.cuh"
#include "tt_gemm_v3.cuh"
#include <cudaTypedefs.h>
#include <cooperative_groups.h>

using tt::GemmParams;
using tt::IndexMap;

namespace {

thread_local std::string g_msg;
thread_local int64_t g_launches = 0;
thread_local int64_t g_launches_last = 0;

// ---- tracing (tt_trace_*): per-launch CUDA events on the launch stream ----------------
struct TraceRec {
  int stage, tile;
  long long M, N, K;
  cudaEvent_t e0, e1;
};
thread_local bool g_trace_on = false;
thread_local std::vector<TraceRec> g_trace;
thread_local std::vector<cudaEvent_t> g_trace_pool;
thread_local int g_stage = TT_ST_PERM;   // stage tag of the next launch

// ---- side stream for the sweeps' concurrent interface chains (per thread, per device) ------
struct SideStream {
  int dev = -1;
  cudaStream_t s = nullptr;
  cudaStream_t s_lo = nullptr;   // same, lowest priority (A/B hook: debug flag 2048)
  cudaEvent_t ev[64] = {};
  unsigned next = 0;
};
thread_local SideStream g_side;
thread_local int g_side_lowprio = 0;

cudaError_t side_stream(cudaStream_t* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (g_side.dev != dev) {
    // the side stream carries the interface chains, the sweeps' critical path: give it the
    // highest priority so its small GEMMs are scheduled ahead of the concurrent matvecs
    int lo = 0, hi = 0;
    if ((e = cudaDeviceGetStreamPriorityRange(&lo, &hi)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithPriority(&g_side.s, cudaStreamNonBlocking, hi)) != cudaSuccess)
      return e;
    if ((e = cudaStreamCreateWithPriority(&g_side.s_lo, cudaStreamNonBlocking, lo)) != cudaSuccess)
      return e;
    for (auto& ev : g_side.ev)
      if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
    g_side.dev = dev;
  }
  *out = g_side_lowprio ? g_side.s_lo : g_side.s;
  return cudaSuccess;
}
// `to` waits for all work enqueued on `from` so far (graph-capture compatible)
cudaError_t stream_dep(cudaStream_t from, cudaStream_t to) {
  cudaEvent_t ev = g_side.ev[g_side.next++ % 64];
  cudaError_t e = cudaEventRecord(ev, from);
  if (e != cudaSuccess) return e;
  return cudaStreamWaitEvent(to, ev, 0);
}

// ---- stream pool + dependency events for DAG-scheduled sweeps (per thread, per device) ----
constexpr int kPoolStreams = 4;
struct StreamPool {
  int dev = -1;
  cudaStream_t s[kPoolStreams] = {};
  cudaStream_t chain = nullptr;   // high priority (the W34 left chain)
  std::vector<cudaEvent_t> ev;
};
thread_local StreamPool g_pool;
cudaError_t pool_init(size_t nevents) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (g_pool.dev != dev) {
    int lo = 0, hi = 0;
    if ((e = cudaDeviceGetStreamPriorityRange(&lo, &hi)) != cudaSuccess) return e;
    for (auto& st : g_pool.s)
      if ((e = cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, lo)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithPriority(&g_pool.chain, cudaStreamNonBlocking, hi)) != cudaSuccess)
      return e;
    g_pool.ev.clear();
    g_pool.dev = dev;
  }
  while (g_pool.ev.size() < nevents) {
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
    g_pool.ev.push_back(ev);
  }
  return cudaSuccess;
}

long long trace_begin(int tile, long long M, long long N, long long K, cudaStream_t s) {
  if (!g_trace_on || 2 * (g_trace.size() + 1) > g_trace_pool.size()) return -1;
  TraceRec r;
  r.stage = g_stage;
  r.tile = tile;
  r.M = M;
  r.N = N;
  r.K = K;
  r.e0 = g_trace_pool[2 * g_trace.size()];
  r.e1 = g_trace_pool[2 * g_trace.size() + 1];
  cudaEventRecord(r.e0, s);
  g_trace.push_back(r);
  return (long long)g_trace.size() - 1;
}
void trace_end(long long idx, cudaStream_t s) {
  if (idx >= 0) cudaEventRecord(g_trace[idx].e1, s);
}

tt_status fail(tt_status s, const std::string& m) {
  g_msg = m;
  return s;
}

constexpr long long kMaxElems = (1LL << 62) / 8;

// checked product of positive extents
bool mulc(long long& acc, long long v) {
  if (v <= 0) return false;
  if (acc > kMaxElems / v) return false;
  acc *= v;
  return true;
}

long long prod(std::initializer_list<long long> xs, bool& ok) {
  long long p = 1;
  for (long long v : xs)
    if (!mulc(p, v)) ok = false;
  return ok ? p : 0;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Carves 256-byte aligned sub-buffers out of the caller's workspace.
struct Carver {
  char* base;
  size_t cap, off = 0;
  bool ok = true;
  double* take(long long elems) {
    uintptr_t p = reinterpret_cast<uintptr_t>(base) + off;
    uintptr_t q = (p + 255) & ~uintptr_t(255);
    size_t need = (q - reinterpret_cast<uintptr_t>(base)) + size_t(elems) * sizeof(double);
    if (need > cap) {
      ok = false;
      return nullptr;
    }
    off = need;
    return reinterpret_cast<double*>(q);
  }
};

// bytes of workspace for a list of buffers (each padded to 256 B, plus 256 B base slack)
size_t ws_bytes(std::initializer_list<long long> elems) {
  size_t s = 256;
  for (long long e : elems) s += align_up(size_t(e) * sizeof(double), 256);
  return s;
}

thread_local int g_dbg_flags = 0;   // tt_debug_set_flags (bits listed in the header)
// GEMMs up to this size are launched with PDL (config 3's ~34 MFLOP stages gain 8 %; config
// 4's ~0.16-0.4 GFLOP stages lose: the early-placed dependents unbalance the persistent grid;
// swept with tools/w34_knobs.py: 0.05 GFLOP gives config 3 0.166 ms and config 4 0.731 ms,
// 0.2 GFLOP 0.165 / 0.746, no PDL 0.193 / 0.734); g_no_pdl (tt_sweep_als scope) disables it.
constexpr double kPdlFlopsDefault = 0.05e9;
double pdl_flops() {   // probe override TT_PDL_FLOPS, read once
  static const double v = [] {
    const char* e = getenv("TT_PDL_FLOPS");
    return e ? atof(e) : kPdlFlopsDefault;
  }();
  return v;
}
thread_local bool g_no_pdl = false;

// Launch with programmatic stream serialisation (PDL, tt_gemm.cuh pdl_wait/pdl_trigger) when
// `pdl`: the kernel may be scheduled while its stream predecessor drains and waits for it on
// the device.  Only kernels that call pdl_wait() before touching global memory are launched
// this way, and only latency-bound ones (small GEMMs, their split-K reduction, the sweep
// preparation): for the large matvec GEMMs of W5 the early-resident dependents hold SMs the
// concurrent interface chain could use (measured +1.1 % on the W5 sweep with PDL everywhere).
// Debug flag 4096 disables PDL (A/B).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && !g_no_pdl && !(g_dbg_flags & 4096)) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ----------------------------------------------------------------------------------------
// GEMM launch: tile configuration chosen from the stage's N extent
// ----------------------------------------------------------------------------------------
template <int BM, int BN, int BK, int WM, int WN, int ST, bool AK, bool BK_>
cudaError_t launch_cfg(const GemmParams& p0, cudaStream_t s) {
  using Cfg = tt::GemmCfg<BM, BN, BK, WM, WN, ST, AK, BK_>;
  auto kern = tt::dmma_gemm_kernel<BM, BN, BK, WM, WN, ST, AK, BK_>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)Cfg::kSmemBytes);
  });
  if (attr_err != cudaSuccess) return attr_err;
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

// ---- v2 (persistent, 16 warps, 16-byte loads) --------------------------------------------
int num_sms() {
  static int sms = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  });
  return sms;
}

thread_local int g_variant = -1;
thread_local int g_force_ks = 0;   // probe hook: split-K factor forced by tt_debug_set_variant
// device flag gating every GEMM launch of the calling thread (set by the iterative solvers
// around their matvecs so that iterations after convergence cost launches only)
thread_local const int* g_gate = nullptr;

// split-K scratch for the current stage (set by the stage planners; nullptr = no split)
thread_local double* g_pscratch = nullptr;
thread_local long long g_pscratch_elems = 0;

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
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)Cfg::kSmemBytes);
  });
  if (attr_err != cudaSuccess) return attr_err;
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
    long long blocks = (mn + 255) / 256;
    if (blocks > 8L * num_sms()) blocks = 8L * num_sms();
    if (cudaError_t e = launch_pdl(2.0 * p0.M * p0.N * p0.K <= pdl_flops(), tt::splitk_reduce_kernel,
                                   dim3((unsigned)blocks), dim3(256), 0,
                                   s, (const double*)p.P, p.C, p.M, p.N, ks, p.rowmap, p.colmap,
                                   p.gate))
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

template <bool AK, bool BK_, int BM, int BN, int WM, int WN, int MINB, bool BRES = false>
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
  auto kern = tt::dmma_gemm_v3_kernel<AK, BK_, BM, BN, WM, WN, ST, MINB, BRES>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)Cfg::kSmemBytes);
  });
  if (attr_err != cudaSuccess) return attr_err;
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
    static const bool l2_debug = getenv("TT_L2_DEBUG") != nullptr;
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
    long long blocks = (mn + 255) / 256;
    if (blocks > 8L * num_sms()) blocks = 8L * num_sms();
    if (cudaError_t e = launch_pdl(2.0 * p0.M * p0.N * p0.K <= pdl_flops(), tt::splitk_reduce_kernel,
                                   dim3((unsigned)blocks), dim3(256), 0,
                                   s, (const double*)p.P, p.C, p.M, p.N, ks, p.rowmap, p.colmap,
                                   p.gate))
      return e;
    ++g_launches;
  }
  trace_end(tr, s);
  ++g_launches;
  return cudaGetLastError();
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
    // (12-warp 128 x 144 / 128 x 96 and 6-warp 64 x 144 / 64 x 96 candidates were measured
    // and dropped: config-4 W34 0.73 -> 0.84 ms; the 6-warp tiles reach only 28 TF/s at scale)
};

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
    if (const char* e = getenv("TT_LAT_FLOPS")) r.flops = atof(e);
    if (const char* e = getenv("TT_LAT_UNIT_US")) r.unit_s = atof(e) * 1e-6;
    if (const char* e = getenv("TT_LAT_MASK")) r.mask = (unsigned)strtoul(e, nullptr, 0);
    if (const char* e = getenv("TT_LAT_SPLIT_US")) r.split_s = atof(e) * 1e-6;
    if (const char* e = getenv("TT_LAT_OCC")) r.occ_model = atoi(e);
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
    (void)a_kc; (void)b_kc;   // every candidate's BM, BN are multiples of 16 (any operand layout)
    for (int ks = 1; ks <= 16; ks *= 2) {
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
    return launch_v3_cfg<AK, BK_, 128, 144, 4, 3, 1>(p, s, ok);
  }
  if (BK_) return launch_v3_cfg<AK, BK_, 128, 128, 4, 4, 1>(p, s, ok);
  if (g_variant == 5) return launch_v3_cfg<AK, BK_, 128, 64, 4, 2, 2>(p, s, ok);   // probes
  if (g_variant == 6) return launch_v3_cfg<AK, BK_, 128, 128, 4, 4, 1>(p, s, ok);
  if (g_variant == 7) return launch_v3_cfg<AK, BK_, 64, 128, 2, 4, 2>(p, s, ok);
  // 128 x 144 tiles on 12 warps of 32 x 48 (first stage 34.0 -> 35.4 TFLOP/s, W5 sweep
  // -0.75 % on top of the operator-core change; bit 22 restores 128 x 128 on 8 x 2 warps)
  if (g_dbg_flags & 4194304) return launch_v3_cfg<AK, BK_, 128, 128, 8, 2, 1>(p, s, ok);
  return launch_v3_cfg<AK, BK_, 128, 144, 4, 3, 1>(p, s, ok);
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
  const int v = g_variant < 0 ? 2 : g_variant;
  if (!g_force_v1 && v >= 2 && v2_eligible(a_kc, b_kc, p)) {
    bool ok = false;
    cudaError_t e;
    if (a_kc && b_kc) e = launch_v3_l<true, true>(p, s, ok);
    else if (a_kc && !b_kc) e = launch_v3_l<true, false>(p, s, ok);
    else if (!a_kc && b_kc) e = launch_v3_l<false, true>(p, s, ok);
    else e = launch_v3_l<false, false>(p, s, ok);
    if (ok || e != cudaSuccess) return e;
  }
  if (!g_force_v1 && v2_eligible(a_kc, b_kc, p)) {
    if (a_kc && b_kc) return launch_v2_l<true, true>(p, s);
    if (a_kc && !b_kc) return launch_v2_l<true, false>(p, s);
    if (!a_kc && b_kc) return launch_v2_l<false, true>(p, s);
    return launch_v2_l<false, false>(p, s);
  }
  if (a_kc && b_kc) return launch_gemm_l<true, true>(p, s);
  if (a_kc && !b_kc) return launch_gemm_l<true, false>(p, s);
  if (!a_kc && b_kc) return launch_gemm_l<false, true>(p, s);
  return launch_gemm_l<false, false>(p, s);
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

// ----------------------------------------------------------------------------------------
// small kernels
// ----------------------------------------------------------------------------------------
// Ahat[(al, j), (i, be)] = A[al, i, j, be]   (left / matvec stage S2 operand)
__global__ void perm_left_kernel(const double* __restrict__ A, double* __restrict__ Ah,
                                 long long al_n, long long n, long long be_n) {
  const long long total = al_n * n * n * be_n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long r = e;
    const long long be = r % be_n; r /= be_n;
    const long long j = r % n; r /= n;
    const long long i = r % n; r /= n;
    const long long al = r;
    Ah[(al * n + j) * (n * be_n) + i * be_n + be] = A[e];
  }
}

// Atil[(j, be), (al, i)] = A[al, i, j, be]   (right interface stage S2'' operand)
__global__ void perm_right_kernel(const double* __restrict__ A, double* __restrict__ At,
                                  long long al_n, long long n, long long be_n) {
  const long long total = al_n * n * n * be_n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long r = e;
    const long long be = r % be_n; r /= be_n;
    const long long j = r % n; r /= n;
    const long long i = r % n; r /= n;
    const long long al = r;
    At[(j * be_n + be) * (al_n * n) + al * n + i] = A[e];
  }
}


// xt[b, j, a] = x[a, j, b]: 32x32 shared-memory tiles per mode index j (coalesced both ways)
__global__ void transpose_core_kernel(const double* __restrict__ x, double* __restrict__ xt,
                                      int a_n, int n, int b_n) {
  __shared__ double tile[32][33];
  const int j = blockIdx.z;
  const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int a = a0 + r, b = b0 + threadIdx.x;
    if (a < a_n && b < b_n) tile[r][threadIdx.x] = x[((long long)a * n + j) * b_n + b];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int b = b0 + r, a = a0 + threadIdx.x;
    if (a < a_n && b < b_n) xt[((long long)b * n + j) * a_n + a] = tile[threadIdx.x][r];
  }
}

// All cores of a sweep prepared by ONE launch (a dependent launch costs ~4 us on the
// critical path of the small-rank sweeps): block range [start[c], start[c+1]) works on core c;
// the first block also writes the trivial boundary interfaces when given.
constexpr int kPrepMax = 40;
struct PrepTable {
  const double* A[kPrepMax];
  const double* x[kPrepMax];
  double* Ahl[kPrepMax];
  double* Ahr[kPrepMax];
  double* xt[kPrepMax];
  int al[kPrepMax], n[kPrepMax], be[kPrepMax], a[kPrepMax], b[kPrepMax];
  int start[kPrepMax + 1];
  int cores;
  double* one0;
  double* one1;
};

__global__ void __launch_bounds__(256) prep_all_kernel(const __grid_constant__ PrepTable t) {
  tt::pdl_wait();
  int c = 0;
  while (c + 1 < t.cores && (int)blockIdx.x >= t.start[c + 1]) ++c;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (t.one0) *t.one0 = 1.0;
    if (t.one1) *t.one1 = 1.0;
  }
  const long long al_n = t.al[c], n = t.n[c], be_n = t.be[c], a_n = t.a[c], b_n = t.b[c];
  const double* __restrict__ A = t.A[c];
  const double* __restrict__ x = t.x[c];
  double* __restrict__ Ahl = t.Ahl[c];
  double* __restrict__ Ahr = t.Ahr[c];
  double* __restrict__ xt = t.xt[c];
  const long long tA = al_n * n * n * be_n, tx = a_n * n * b_n;
  const long long nb = t.start[c + 1] - t.start[c];
  for (long long e = (blockIdx.x - t.start[c]) * (long long)blockDim.x + threadIdx.x; e < tA + tx;
       e += nb * blockDim.x) {
    if (e < tA) {
      long long r = e;
      const long long be = r % be_n; r /= be_n;
      const long long j = r % n; r /= n;
      const long long i = r % n;
      const long long al = r / n;
      const double v = A[e];
      Ahl[(al * n + j) * (n * be_n) + i * be_n + be] = v;
      Ahr[(be * n + j) * (n * al_n) + i * al_n + al] = v;
    } else {
      const long long f = e - tA;
      const long long b = f % b_n, r = f / b_n;
      const long long j = r % n, a = r / n;
      xt[(b * n + j) * a_n + a] = x[f];
    }
  }
  tt::pdl_trigger();
}

// At[be, i, j, al] = A[al, i, j, be]  (operator core with its two bonds swapped)
__global__ void swap_bonds_kernel(const double* __restrict__ A, double* __restrict__ At,
                                  long long al_n, long long nn, long long be_n) {
  const long long total = al_n * nn * be_n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long be = e % be_n, r = e / be_n;
    const long long ij = r % nn, al = r / nn;
    At[(be * nn + ij) * al_n + al] = A[e];
  }
}

cudaError_t launch_perm(bool left, const double* A, double* out, long long al, long long n,
                        long long be, cudaStream_t s) {
  const long long total = al * n * n * be;
  const int threads = 256;
  long long blocks = (total + threads - 1) / threads;
  if (blocks > 4096) blocks = 4096;
  const int saved = g_stage;
  g_stage = TT_ST_PERM;
  const long long tr = trace_begin(0, total, 0, 0, s);
  g_stage = saved;
  if (left)
    perm_left_kernel<<<(unsigned)blocks, threads, 0, s>>>(A, out, al, n, be);
  else
    perm_right_kernel<<<(unsigned)blocks, threads, 0, s>>>(A, out, al, n, be);
  trace_end(tr, s);
  ++g_launches;
  return cudaGetLastError();
}


// H8: z[(a,al), i, (b,be)] = sum_j A[al,i,j,be] x[a,j,b].  One CTA per (a, al) pair; the
// x[a,:,:] and A[al,:,:,:] slices are staged in shared memory; the output rows (one per i,
// each rr*Rr contiguous doubles) are written with streaming (evict-first) stores.
__global__ void __launch_bounds__(256) apply_kernel(const double* __restrict__ x,
                                                    const double* __restrict__ A,
                                                    double* __restrict__ z, int rl, int ni,
                                                    int nj, int rr, int Rl, int Rr) {
  extern __shared__ double sm[];
  double* xs = sm;                       // [nj][rr]
  double* As = sm + (size_t)nj * rr;     // [ni][nj][Rr]
  const long long pair = blockIdx.x;     // a * Rl + al
  const int a = (int)(pair / Rl), al = (int)(pair % Rl);
  const int xn = nj * rr, an = ni * nj * Rr;
  for (int e = threadIdx.x; e < xn; e += blockDim.x) xs[e] = x[(long long)a * xn + e];
  for (int e = threadIdx.x; e < an; e += blockDim.x) As[e] = A[(long long)al * an + e];
  __syncthreads();
  const int L = rr * Rr;
  const int step_b = blockDim.x / Rr, step_be = blockDim.x % Rr;
  for (int i = 0; i < ni; ++i) {
    double* zrow = z + (pair * ni + i) * (long long)L;
    const double* Ai = As + (size_t)i * nj * Rr;
    int b = threadIdx.x / Rr, be = threadIdx.x % Rr;
    for (int e = threadIdx.x; e < L; e += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < nj; ++j) s = fma(Ai[j * Rr + be], xs[j * rr + b], s);
      __stcs(zrow + e, s);
      b += step_b;
      be += step_be;
      if (be >= Rr) {
        be -= Rr;
        ++b;
      }
    }
  }
}

// H8, register-blocked: thread <-> one output column e = (b, beta) of the z rows; the thread
// keeps x[a, :, b] for AB consecutive a in registers and walks (alpha, i), reading the nj
// operator values A[alpha, i, :, beta] (L1-resident, coalesced across the warp's betas) once
// per AB outputs.  Every warp store is 32 consecutive doubles of one z row (evict-first).
template <int NJ, int AB>
__global__ void __launch_bounds__(256) apply_reg_kernel(const double* __restrict__ x,
                                                        const double* __restrict__ A,
                                                        double* __restrict__ z, int rl, int ni,
                                                        int rr, int Rl, int Rr, int az) {
  const long long L = (long long)rr * Rr;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= L) return;
  const int b = (int)(e / Rr), be = (int)(e - (long long)b * Rr);
  const int a0 = blockIdx.y * AB;
  // operator bond indices [al0, al1): split over blockIdx.z when the core is small
  const int al0 = blockIdx.z * az, al1 = min(Rl, al0 + az);
  double xv[AB][NJ];
#pragma unroll
  for (int u = 0; u < AB; ++u)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
      xv[u][j] = (a0 + u < rl) ? __ldg(x + ((long long)(a0 + u) * NJ + j) * rr + b) : 0.0;
  for (int al = al0; al < al1; ++al)
  for (int i = 0; i < ni; ++i) {
    double av[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) av[j] = __ldg(A + ((long long)(al * ni + i) * NJ + j) * Rr + be);
#pragma unroll
    for (int u = 0; u < AB; ++u) {
      if (a0 + u < rl) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j) s = fma(av[j], xv[u][j], s);
        __stcs(z + (((long long)(a0 + u) * Rl + al) * ni + i) * L + e, s);
      }
    }
  }
}

template <int NJ>
cudaError_t launch_apply_reg(const double* x, const double* A, double* z, long long rl,
                             long long ni, long long rr, long long Rl, long long Rr,
                             cudaStream_t s) {
  constexpr int AB = 4;
  const long long L = rr * Rr;
  const long long gx = (L + 255) / 256, gy = (rl + AB - 1) / AB;
  // enough CTAs to fill the machine, but as many bond indices per thread as possible
  long long az = (gx * gy * Rl) / 4096;
  az = az < 1 ? 1 : (az > Rl ? Rl : az);
  dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)((Rl + az - 1) / az));
  apply_reg_kernel<NJ, AB><<<grid, 256, 0, s>>>(x, A, z, (int)rl, (int)ni, (int)rr, (int)Rl,
                                                (int)Rr, (int)az);
  return cudaGetLastError();
}

// FP64 DMMA throughput probe: 8 independent accumulator chains per warp.
__global__ void __launch_bounds__(256) dmma_probe_kernel(double* out, long long iters) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (long long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) tt::dmma_8x8x4(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == -1.0) out[threadIdx.x] = s;   // never true; keeps the loop live
}

// ----------------------------------------------------------------------------------------
// stage plans
// ----------------------------------------------------------------------------------------
struct Dims {
  long long a, n, b, al, be;
};

bool dims_valid(const Dims& d) { return d.a > 0 && d.n > 0 && d.b > 0 && d.al > 0 && d.be > 0; }

// element counts of the matvec workspace buffers (K columns)
bool matvec_ws_elems(const Dims& d, long long K, long long& t1, long long& t2, long long& ah,
                     long long& pe) {
  bool ok = true;
  t1 = prod({d.a, d.al, d.n, K, d.b}, ok);
  t2 = prod({d.a, d.n, K, d.be, d.b}, ok);
  ah = prod({d.al, d.n, d.n, d.be}, ok);
  // split-K partials of the last stage: 4 slices, or up to 64 for small outputs (<= 128 MB)
  {
    const long long out = prod({d.a, d.n, K, d.b}, ok);
    pe = std::max(4 * out, std::min(64 * out, 16LL << 20));
  }
  return ok;
}

struct SplitScratch {   // scopes the split-K scratch to one stage launch
  SplitScratch(double* p, long long n) {
    g_pscratch = p;
    g_pscratch_elems = n;
  }
  ~SplitScratch() {
    g_pscratch = nullptr;
    g_pscratch_elems = 0;
  }
};

// Local matvec (K columns, Block-TT layout) — stages S1, S2^T, S3.
// S3: Y(a', i, m, b') = T2[(a' m i), (be b)] . phiR[b', (be b)]^T
cudaError_t enqueue_matvec_last(const Dims& d, long long K, const double* T2, const double* phiR,
                                double* Y, double* P, long long pe, cudaStream_t s) {
  const long long a = d.a, b = d.b, be = d.be, N = d.n;
  g_stage = TT_ST_MV_S3;
  SplitScratch scratch(P, pe);
  return launch_gemm(true, true,
                     gp(T2, be * b, phiR, be * b, Y, a * K * N, b, be * b,
                        tt::map3(N, K, K * b, b, N * K * b), tt::map_plain(1)),
                     s);
}

cudaError_t enqueue_matvec(const Dims& d, long long K, const double* phiL, const double* A,
                           const double* phiR, const double* X, double* Y, double* T1,
                           double* T2, double* Ah, double* P, long long pe, cudaStream_t s,
                           const double* Ah_pre = nullptr) {
  const long long a = d.a, b = d.b, al = d.al, be = d.be, N = d.n;
  cudaError_t e;
  if (Ah_pre)
    Ah = const_cast<double*>(Ah_pre);
  else if ((e = launch_perm(true, A, Ah, al, N, be, s)) != cudaSuccess)
    return e;
  // S1: T1(al, j, a', m, b) = phiL[(a' al), a] . X[a, (j m b)]
  g_stage = TT_ST_MV_S1;
  e = launch_gemm(true, false,
                  gp(phiL, a, X, N * K * b, T1, a * al, N * K * b, a,
                     tt::map2(al, N * a * K * b, K * b), tt::map2(K * b, 1, a * K * b)),
                  s);
  if (e != cudaSuccess) return e;
  // S2^T: T2(a', m, i, be, b) = T1^T[(a' m b), (al j)] . Ahat[(al j), (i be)]
  g_stage = TT_ST_MV_S2;
  e = launch_gemm(false, false,
                  gp(T1, a * K * b, Ah, N * be, T2, a * K * b, N * be, al * N,
                     tt::map2(b, 1, N * be * b), tt::map_plain(b)),
                  s);
  if (e != cudaSuccess) return e;
  return enqueue_matvec_last(d, K, T2, phiR, Y, P, pe, s);
}

bool iface_ws_elems(const Dims& d, long long& t1, long long& t2, long long& ah, long long& pe) {
  bool ok = true;
  // ah also holds the mirrored right update's swapped operator core and transposed core
  {
    const long long out = std::max(prod({d.b, d.be, d.b}, ok), prod({d.a, d.al, d.a}, ok));
    pe = std::max(4 * out, std::min(64 * out, 16LL << 20));
  }
  t1 = prod({d.a, d.al, d.n, d.b}, ok);
  long long t1r = prod({d.a, d.n, d.b, d.be}, ok);
  if (t1r > t1) t1 = t1r;
  t2 = prod({d.a, d.n, d.be, d.b}, ok);
  long long t2r = prod({d.a, d.al, d.n, d.b}, ok);
  if (t2r > t2) t2 = t2r;
  ah = prod({3, d.al, d.n, d.n, d.be}, ok) + prod({d.a, d.n, d.b}, ok);
  return ok;
}

// Left interface: S1, S2^T (K = 1), S3': phiL_next[b', (be b)] = x^T[b', (a' i)] . T2[(a' i), (be b)]
cudaError_t enqueue_left(const Dims& d, const double* phiL, const double* A, const double* x,
                         double* out, double* T1, double* T2, double* Ah, double* P,
                         long long pe, cudaStream_t s, int tag_s1 = TT_ST_IL_S1,
                         const double* Ah_pre = nullptr, cudaEvent_t ev_t2 = nullptr) {
  const long long a = d.a, b = d.b, al = d.al, be = d.be, N = d.n;
  cudaError_t e;
  if (Ah_pre)
    Ah = const_cast<double*>(Ah_pre);
  else if ((e = launch_perm(true, A, Ah, al, N, be, s)) != cudaSuccess)
    return e;
  g_stage = tag_s1;
  e = launch_gemm(true, false,
                  gp(phiL, a, x, N * b, T1, a * al, N * b, a, tt::map2(al, N * a * b, b),
                     tt::map2(b, 1, a * b)),
                  s);
  if (e != cudaSuccess) return e;
  g_stage = tag_s1 + 1;
  e = launch_gemm(false, false,
                  gp(T1, a * b, Ah, N * be, T2, a * b, N * be, al * N, tt::map2(b, 1, N * be * b),
                     tt::map_plain(b)),
                  s);
  if (e != cudaSuccess) return e;
  if (ev_t2 && (e = cudaEventRecord(ev_t2, s)) != cudaSuccess) return e;   // T2 complete
  g_stage = tag_s1 + 2;
  SplitScratch scratch(P, pe);
  return launch_gemm(false, false,
                     gp(x, b, T2, be * b, out, b, be * b, a * N, tt::map_plain(be * b),
                        tt::map_plain(1)),
                     s);
}

// Right interface: S1'': T1(j, be, a, b') = x[(a j), b] . phiR[(b' be), b]^T
//                  S2'': T2(i, b', al, a) = T1^T[(a b'), (j be)] . Atil[(j be), (al i)]
//                  S3'': phiR_prev[a', (al a)] = x[a', (i b')] . T2[(i b'), (al a)]
// Right interface as the mirror image of the left one: with
// xt[b, j, a] = x[a, j, b] and At[be, i, j, al] = A[al, i, j, be],
//   phiR_prev[a', al, a] = sum x[a',i,b'] A[al,i,j,be] phiR[b',be,b] x[a,j,b]
//                        = (left update of phiR through At, xt)[a', al, a],
// so the right update runs on the left update's stage kernels (their layouts give 16-byte
// epilogue stores and M/N-contiguous TMA operands).  Ah holds [perm | At | xt].
cudaError_t enqueue_right_mirror(const Dims& d, const double* phiR, const double* A,
                                 const double* x, double* out, double* T1, double* T2,
                                 double* Ah, double* P, long long pe, cudaStream_t s,
                                 const double* Ahr_pre = nullptr, const double* xt_pre = nullptr) {
  const long long a = d.a, b = d.b, al = d.al, be = d.be, N = d.n;
  if (Ahr_pre && xt_pre) {
    const Dims dm{b, N, a, be, al};
    return enqueue_left(dm, phiR, nullptr, xt_pre, out, T1, T2, Ah, P, pe, s, TT_ST_IR_S1,
                        Ahr_pre);
  }
  double* At = Ah + al * N * N * be;
  double* xt = At + al * N * N * be;
  {
    const long long total = al * N * N * be;
    long long blocks = (total + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    g_stage = TT_ST_PERM;
    const long long tr = trace_begin(0, total, 0, 0, s);
    swap_bonds_kernel<<<(unsigned)blocks, 256, 0, s>>>(A, At, al, N * N, be);
    trace_end(tr, s);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  {
    dim3 grid((unsigned)((b + 31) / 32), (unsigned)((a + 31) / 32), (unsigned)N);
    g_stage = TT_ST_PERM;
    const long long tr = trace_begin(0, a * N * b, 0, 0, s);
    transpose_core_kernel<<<grid, dim3(32, 8), 0, s>>>(x, xt, (int)a, (int)N, (int)b);
    trace_end(tr, s);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const Dims dm{b, N, a, be, al};
  return enqueue_left(dm, phiR, At, xt, out, T1, T2, Ah, P, pe, s, TT_ST_IR_S1);
}

cudaError_t enqueue_right(const Dims& d, const double* phiR, const double* A, const double* x,
                          double* out, double* T1, double* T2, double* At, double* P,
                          long long pe, cudaStream_t s) {
  const long long a = d.a, b = d.b, al = d.al, be = d.be, N = d.n;
  cudaError_t e;
  if ((e = launch_perm(false, A, At, al, N, be, s)) != cudaSuccess) return e;
  g_stage = TT_ST_IR_S1;
  e = launch_gemm(true, true,
                  gp(x, b, phiR, b, T1, a * N, b * be, b, tt::map2(N, be * a * b, b),
                     tt::map2(be, a * b, 1)),
                  s);
  if (e != cudaSuccess) return e;
  g_stage = TT_ST_IR_S2;
  e = launch_gemm(false, false,
                  gp(T1, a * b, At, al * N, T2, a * b, al * N, N * be, tt::map2(b, al * a, 1),
                     tt::map2(N, b * al * a, a)),
                  s);
  if (e != cudaSuccess) return e;
  g_stage = TT_ST_IR_S3;
  SplitScratch scratch(P, pe);
  return launch_gemm(true, false,
                     gp(x, N * b, T2, al * a, out, a, al * a, N * b, tt::map_plain(al * a),
                        tt::map_plain(1)),
                     s);
}

// ---- Petrov-Galerkin (bra train != ket train) variants --------------------------------------
// The same three-GEMM stage plans with the bra ranks (ap = a', bp = b') decoupled from the ket
// ranks (a, b): the local operator Z_{!=k}^T A X_{!=k} of two different trains, the projected
// right-hand side X_{!=k}^T b (identity operator) and the AMEn residual frame
// (PAPER.md:303).  Interfaces are [bra, op, ket]: phiL (ap, al, a), phiR (bp, be, b).
struct DimsPG {
  long long ap, a, n, bp, b, al, be;
};
bool dims_pg_valid(const DimsPG& d) {
  return d.ap > 0 && d.a > 0 && d.n > 0 && d.bp > 0 && d.b > 0 && d.al > 0 && d.be > 0;
}
// element counts for the matvec (K columns) and both interface updates
bool pg_ws_elems(const DimsPG& d, long long K, long long& t1, long long& t2, long long& ah,
                 long long& pe) {
  bool ok = true;
  t1 = std::max({prod({d.ap, d.al, d.n, K, d.b}, ok), prod({d.a, d.n, d.bp, d.be}, ok)});
  t2 = std::max({prod({d.ap, d.n, K, d.be, d.b}, ok), prod({d.n, d.bp, d.al, d.a}, ok)});
  ah = prod({d.al, d.n, d.n, d.be}, ok);
  const long long out = std::max({prod({d.ap, d.n, K, d.bp}, ok), prod({d.bp, d.be, d.b}, ok),
                                  prod({d.ap, d.al, d.a}, ok)});
  pe = std::max(4 * out, std::min(64 * out, 16LL << 20));
  return ok;
}

// Y (ap, n, K, bp) = phiL (ap, al, a) x A x phiR (bp, be, b) applied to X (a, n, K, b)
cudaError_t enqueue_matvec_pg(const DimsPG& d, long long K, const double* phiL, const double* A,
                              const double* phiR, const double* X, double* Y, double* T1,
                              double* T2, double* Ah, double* P, long long pe, cudaStream_t s) {
  const long long ap = d.ap, a = d.a, bp = d.bp, b = d.b, al = d.al, be = d.be, N = d.n;
  cudaError_t e;
  if ((e = launch_perm(true, A, Ah, al, N, be, s)) != cudaSuccess) return e;
  // S1: T1(al, j, a', m, b) = phiL[(a' al), a] . X[a, (j m b)]
  g_stage = TT_ST_MV_S1;
  e = launch_gemm(true, false,
                  gp(phiL, a, X, N * K * b, T1, ap * al, N * K * b, a,
                     tt::map2(al, N * ap * K * b, K * b), tt::map2(K * b, 1, ap * K * b)),
                  s);
  if (e != cudaSuccess) return e;
  // S2: T2(a', m, i, be, b) = T1^T[(a' m b), (al j)] . Ahat[(al j), (i be)]
  g_stage = TT_ST_MV_S2;
  e = launch_gemm(false, false,
                  gp(T1, ap * K * b, Ah, N * be, T2, ap * K * b, N * be, al * N,
                     tt::map2(b, 1, N * be * b), tt::map_plain(b)),
                  s);
  if (e != cudaSuccess) return e;
  // S3: Y(a', i, m, b') = T2[(a' m i), (be b)] . phiR[b', (be b)]^T
  g_stage = TT_ST_MV_S3;
  SplitScratch scratch(P, pe);
  return launch_gemm(true, true,
                     gp(T2, be * b, phiR, be * b, Y, ap * K * N, bp, be * b,
                        tt::map3(N, K, K * bp, bp, N * K * bp), tt::map_plain(1)),
                     s);
}

// phiL_next (bp, be, b) = sum x_bra[a', i, b'] phiL[a', al, a] A[al, i, j, be] x_ket[a, j, b]
cudaError_t enqueue_left_pg(const DimsPG& d, const double* phiL, const double* A,
                            const double* xb, const double* xk, double* out, double* T1,
                            double* T2, double* Ah, double* P, long long pe, cudaStream_t s) {
  const long long ap = d.ap, a = d.a, bp = d.bp, b = d.b, al = d.al, be = d.be, N = d.n;
  cudaError_t e;
  if ((e = launch_perm(true, A, Ah, al, N, be, s)) != cudaSuccess) return e;
  g_stage = TT_ST_IL_S1;   // T1(al, j, a', b) = phiL[(a' al), a] . x_ket[a, (j b)]
  e = launch_gemm(true, false,
                  gp(phiL, a, xk, N * b, T1, ap * al, N * b, a, tt::map2(al, N * ap * b, b),
                     tt::map2(b, 1, ap * b)),
                  s);
  if (e != cudaSuccess) return e;
  g_stage = TT_ST_IL_S2;   // T2(a', i, be, b) = T1^T[(a' b), (al j)] . Ahat[(al j), (i be)]
  e = launch_gemm(false, false,
                  gp(T1, ap * b, Ah, N * be, T2, ap * b, N * be, al * N, tt::map2(b, 1, N * be * b),
                     tt::map_plain(b)),
                  s);
  if (e != cudaSuccess) return e;
  g_stage = TT_ST_IL_S3;   // out[b', (be b)] = x_bra^T[b', (a' i)] . T2[(a' i), (be b)]
  SplitScratch scratch(P, pe);
  return launch_gemm(false, false,
                     gp(xb, bp, T2, be * b, out, bp, be * b, ap * N, tt::map_plain(be * b),
                        tt::map_plain(1)),
                     s);
}

// phiR_prev (ap, al, a) = sum x_bra[a', i, b'] A[al, i, j, be] phiR[b', be, b] x_ket[a, j, b]
cudaError_t enqueue_right_pg(const DimsPG& d, const double* phiR, const double* A,
                             const double* xb, const double* xk, double* out, double* T1,
                             double* T2, double* At, double* P, long long pe, cudaStream_t s) {
  const long long ap = d.ap, a = d.a, bp = d.bp, b = d.b, al = d.al, be = d.be, N = d.n;
  cudaError_t e;
  if ((e = launch_perm(false, A, At, al, N, be, s)) != cudaSuccess) return e;
  g_stage = TT_ST_IR_S1;   // T1(j, be, a, b') = x_ket[(a j), b] . phiR[(b' be), b]^T
  e = launch_gemm(true, true,
                  gp(xk, b, phiR, b, T1, a * N, bp * be, b, tt::map2(N, be * a * bp, bp),
                     tt::map2(be, a * bp, 1)),
                  s);
  if (e != cudaSuccess) return e;
  g_stage = TT_ST_IR_S2;   // T2(i, b', al, a) = T1^T[(a b'), (j be)] . Atil[(j be), (al i)]
  e = launch_gemm(false, false,
                  gp(T1, a * bp, At, al * N, T2, a * bp, al * N, N * be, tt::map2(bp, al * a, 1),
                     tt::map2(N, bp * al * a, a)),
                  s);
  if (e != cudaSuccess) return e;
  g_stage = TT_ST_IR_S3;   // out[a', (al a)] = x_bra[a', (i b')] . T2[(i b'), (al a)]
  SplitScratch scratch(P, pe);
  return launch_gemm(true, false,
                     gp(xb, N * bp, T2, al * a, out, ap, al * a, N * bp, tt::map_plain(al * a),
                        tt::map_plain(1)),
                     s);
}

tt_status cuda_fail(cudaError_t e, const char* where) {
  return fail(TT_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

struct CallScope {
  CallScope() {
    g_msg.clear();
    g_launches = 0;
  }
  ~CallScope() { g_launches_last = g_launches; }
};

tt_status check_dims(const Dims& d) {
  if (!dims_valid(d)) return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  bool ok = true;
  prod({d.a, d.al, d.n, d.b}, ok);
  prod({d.a, d.n, d.be, d.b}, ok);
  prod({d.al, d.n, d.n, d.be}, ok);
  prod({d.b, d.be, d.b}, ok);
  prod({d.a, d.al, d.a}, ok);
  if (!ok) return fail(TT_ERR_OVERFLOW, "extent product overflows");
  return TT_OK;
}

bool same(const void* p, const void* q) { return p != nullptr && p == q; }

#include "tt_gmres.cuh"
#include "tt_round.cuh"
#include "tt_lobpcg.cuh"

// Symmetric eigendecomposition of the n x n Gram matrix G: lam (descending) and V (columns)
// in the caller's buffers.  n <= 64: element-wise cooperative Jacobi (4 padded np x np
// buffers, np = n rounded up to even); larger n: block Jacobi (G and V padded to a multiple
// of 32 plus the per-pair rotations).  Scratch: sym_eigen_scratch(n) doubles.
constexpr int kBlockJacobiMin = 65;
long long sym_eigen_scratch(long long n) {
  const long long np = (n + 1) & ~1LL;
  const long long nb = (n + kJB2 - 1) / kJB2 * kJB2;
  const long long elem = 4 * np * np, blk = 2 * nb * nb + (nb / kJB2) * kJB2 * kJB2;
  return std::max(elem, blk) + 2 * 4096 + 8;
}
thread_local int g_eigen_elementwise = 0;   // test hook: force the element-wise kernel
cudaError_t launch_sym_eigen(const double* G, double* V, double* lam, int n, double* scratch,
                             cudaStream_t s) {
  g_stage = TT_ST_PERM;
  const long long tr = trace_begin(0, (long long)n * n, 0, 0, s);
  int dev = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaError_t e;
  if (n >= kBlockJacobiMin && !g_eigen_elementwise) {
    const int np = (n + kJB2 - 1) / kJB2 * kJB2;
    const long long NN = (long long)np * np;
    double* G0 = scratch;
    double* V0 = G0 + NN;
    double* Rbuf = V0 + NN;
    const int m = np / kJB2;   // block pairs per step
    double* part = Rbuf + (long long)m * kJB2 * kJB2;
    int* which = reinterpret_cast<int*>(part + 2 * 4096);
    long long eb = std::min<long long>(4096, (NN + 255) / 256);
    embed_kernel<<<(unsigned)eb, 256, 0, s>>>(G, G0, n, np);
    ++g_launches;
    if ((e = cudaMemsetAsync(which, 0, sizeof(int), s)) != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_block_coop_kernel, 256, 0);
    int grid = num_sms() * std::max(per_sm, 1);
    const int tasks = m * m + (np / kJB2) * m;
    if (grid > tasks) grid = tasks;
    if (grid > 4096) grid = 4096;
    int sweeps = 40;
    int npi = np;
    void* args[] = {&G0, &V0, (void*)&npi, &sweeps, &Rbuf, &part};
    e = cudaLaunchCooperativeKernel((const void*)jacobi_block_coop_kernel, grid, 256, args, 0, s);
    ++g_launches;
    if (e != cudaSuccess) return e;
    sort_padded_kernel<<<(n + 255) / 256, 256, 0, s>>>(G0, G0, V0, V0, which, V, lam, n, np);
    ++g_launches;
    trace_end(tr, s);
    return cudaGetLastError();
  }
  const int np = (n + 1) & ~1;
  const long long NN = (long long)np * np;
  double* G0 = scratch;
  double* G1 = G0 + NN;
  double* V0 = G1 + NN;
  double* V1 = V0 + NN;
  double* part = V1 + NN;
  int* which = reinterpret_cast<int*>(part + 2 * 4096);
  long long eb = (NN + 255) / 256;
  if (eb > 4096) eb = 4096;
  embed_kernel<<<(unsigned)eb, 256, 0, s>>>(G, G0, n, np);
  ++g_launches;
  const size_t smem = (size_t)np / 2 * (2 * sizeof(double) + 2 * sizeof(int));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_coop_kernel, 256, smem);
  int grid = num_sms() * std::max(per_sm, 1);
  const long long want = std::max<long long>(1, ((long long)(np / 2) * (np / 2) + 255) / 256);
  if (grid > want) grid = (int)want;
  if (grid > 4096) grid = 4096;
  int sweeps = 25;
  void* args[] = {&G0, &G1, &V0, &V1, (void*)&np, &sweeps, &part, &which};
  e = cudaLaunchCooperativeKernel((const void*)jacobi_coop_kernel, grid, 256, args, smem, s);
  ++g_launches;
  if (e != cudaSuccess) return e;
  sort_padded_kernel<<<(n + 255) / 256, 256, 0, s>>>(G0, G1, V0, V1, which, V, lam, n, np);
  ++g_launches;
  trace_end(tr, s);
  return cudaGetLastError();
}

// Block-TT column gather / scaled scatter-add: column `col` of X (rows, nb, rr) <-> v (rows, rr)
__global__ void gather_col_kernel(const double* __restrict__ X, double* __restrict__ v,
                                  long long rows, int nb, int rr, int col) {
  const long long tot = rows * rr;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / rr, b = e - row * rr;
    v[e] = X[(row * nb + col) * rr + b];
  }
}
__global__ void scatter_add_col_kernel(const double* __restrict__ v, double* __restrict__ Y,
                                       long long rows, int nb, int rr, int row_blk, double c) {
  const long long tot = rows * rr;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / rr, b = e - row * rr;
    double* y = Y + (row * nb + row_blk) * rr + b;
    *y = fma(c, v[e], *y);
  }
}

// W[r, c] = V[r * ldv + c] * f[c], r < rows, c < s
__global__ void scale_cols_ld_kernel(const double* __restrict__ V, long long ldv,
                                     const double* __restrict__ f, double* __restrict__ W,
                                     long long rows, int s) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < rows * s;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / s;
    const int c = (int)(e - r * s);
    W[e] = V[r * ldv + c] * f[c];
  }
}

// out (cols x rows) = in (rows x cols)^T, both row-major
__global__ void transpose2d_kernel(const double* __restrict__ in, double* __restrict__ out,
                                   long long rows, long long cols) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols, j = e - i * cols;
    out[j * rows + i] = in[e];
  }
}
// out (a, l, i, b) = in (a, i, l, b)   (the block index moved next to the left bond)
__global__ void swap_mid_kernel(const double* __restrict__ in, double* __restrict__ out,
                                long long a, long long ni, long long nl, long long b) {
  const long long total = a * ni * nl * b;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long r = e;
    const long long bb = r % b; r /= b;
    const long long l = r % nl; r /= nl;
    const long long i = r % ni;
    const long long aa = r / ni;
    out[((aa * nl + l) * ni + i) * b + bb] = in[e];
  }
}

// Two-site supercore operator: A12[al, (i1 i2), (j1 j2), be] = sum_g A1[al,i1,j1,g] A2[g,i2,j2,be]
// (the local operator of a pair of cores; tiny, one thread per output)
__global__ void merge_cores_kernel(const double* __restrict__ A1, const double* __restrict__ A2,
                                   double* __restrict__ A12, long long Rl, long long n1,
                                   long long n2, long long Rm, long long Rr) {
  const long long total = Rl * n1 * n2 * n1 * n2 * Rr;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long r = e;
    const long long be = r % Rr; r /= Rr;
    const long long j2 = r % n2; r /= n2;
    const long long j1 = r % n1; r /= n1;
    const long long i2 = r % n2; r /= n2;
    const long long i1 = r % n1;
    const long long al = r / n1;
    double s = 0.0;
    for (long long g = 0; g < Rm; ++g)
      s = fma(A1[((al * n1 + i1) * n1 + j1) * Rm + g], A2[((g * n2 + i2) * n2 + j2) * Rr + be], s);
    A12[e] = s;
  }
}

}  // namespace

// ========================================================================================
// C ABI
// ========================================================================================
extern "C" {

const char* tt_status_string(tt_status s) {
  switch (s) {
    case TT_OK: return "TT_OK";
    case TT_ERR_INVALID_ARGUMENT: return "TT_ERR_INVALID_ARGUMENT";
    case TT_ERR_NULL_POINTER: return "TT_ERR_NULL_POINTER";
    case TT_ERR_ALIASING: return "TT_ERR_ALIASING";
    case TT_ERR_WORKSPACE: return "TT_ERR_WORKSPACE";
    case TT_ERR_OVERFLOW: return "TT_ERR_OVERFLOW";
    case TT_ERR_CUDA: return "TT_ERR_CUDA";
  }
  return "TT_UNKNOWN_STATUS";
}

const char* tt_last_error_message(void) { return g_msg.c_str(); }
const char* tt_version(void) { return "tt_hotpath 0.1 (sm_100a, FP64 DMMA)"; }
int64_t tt_last_launch_count(void) { return g_launches_last; }
void tt_debug_force_v1(int on) { g_force_v1 = on; }
void tt_debug_set_variant(int v) {
  g_variant = v;
  g_force_ks = v >= 10 ? v / 100 : 0;
}
void tt_debug_set_flags(int f) {
  g_dbg_flags = f;
  g_side_lowprio = (f & 2048) ? 1 : 0;
}

size_t tt_local_matvec_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                                      int64_t nvec) {
  Dims d{rl, n, rr, Rl, Rr};
  long long t1, t2, ah, pe;
  if (!dims_valid(d) || nvec <= 0 || !matvec_ws_elems(d, nvec, t1, t2, ah, pe)) return 0;
  return ws_bytes({t1, t2, ah, pe});
}

tt_status tt_local_matvec_batched(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                                  int64_t nvec, const double* phiL, const double* A,
                                  const double* phiR, const double* X, double* Y,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  Dims d{rl, n, rr, Rl, Rr};
  tt_status st = check_dims(d);
  if (st != TT_OK) return st;
  if (nvec <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "nvec must be positive");
  if (!phiL || !A || !phiR || !X || !Y) return fail(TT_ERR_NULL_POINTER, "NULL tensor pointer");
  if (same(Y, phiL) || same(Y, A) || same(Y, phiR) || same(Y, X))
    return fail(TT_ERR_ALIASING, "output Y aliases an input");
  long long t1, t2, ah, pe;
  if (!matvec_ws_elems(d, nvec, t1, t2, ah, pe)) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  const size_t need = ws_bytes({t1, t2, ah, pe});
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  if (same(workspace, Y) || same(workspace, X) || same(workspace, phiL) || same(workspace, phiR) ||
      same(workspace, A))
    return fail(TT_ERR_ALIASING, "workspace aliases a tensor");
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  double* T1 = c.take(t1);
  double* T2 = c.take(t2);
  double* Ah = c.take(ah);
  double* Pp = c.take(pe);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  cudaError_t e = enqueue_matvec(d, nvec, phiL, A, phiR, X, Y, T1, T2, Ah, Pp, pe,
                                 static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_local_matvec_batched");
  return TT_OK;
}

tt_status tt_local_matvec(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                          const double* phiL, const double* A, const double* phiR,
                          const double* x, double* y, void* workspace, size_t workspace_bytes,
                          void* stream) {
  return tt_local_matvec_batched(rl, n, rr, Rl, Rr, 1, phiL, A, phiR, x, y, workspace,
                                 workspace_bytes, stream);
}

size_t tt_interface_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr) {
  Dims d{rl, n, rr, Rl, Rr};
  long long t1, t2, ah, pe;
  if (!dims_valid(d) || !iface_ws_elems(d, t1, t2, ah, pe)) return 0;
  return ws_bytes({t1, t2, ah, pe});
}

static tt_status iface_common(bool left, int64_t rl, int64_t n, int64_t rr, int64_t Rl,
                              int64_t Rr, const double* phi_in, const double* A,
                              const double* x, double* phi_out, void* workspace,
                              size_t workspace_bytes, void* stream) {
  Dims d{rl, n, rr, Rl, Rr};
  tt_status st = check_dims(d);
  if (st != TT_OK) return st;
  if (!phi_in || !A || !x || !phi_out) return fail(TT_ERR_NULL_POINTER, "NULL tensor pointer");
  if (same(phi_out, phi_in) || same(phi_out, A) || same(phi_out, x))
    return fail(TT_ERR_ALIASING, "output interface aliases an input");
  long long t1, t2, ah, pe;
  if (!iface_ws_elems(d, t1, t2, ah, pe)) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  const size_t need = ws_bytes({t1, t2, ah, pe});
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  if (same(workspace, phi_out) || same(workspace, phi_in) || same(workspace, x) ||
      same(workspace, A))
    return fail(TT_ERR_ALIASING, "workspace aliases a tensor");
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  double* T1 = c.take(t1);
  double* T2 = c.take(t2);
  double* Ah = c.take(ah);
  double* Pp = c.take(pe);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = left ? enqueue_left(d, phi_in, A, x, phi_out, T1, T2, Ah, Pp, pe, s)
                       : (g_dbg_flags & 8) ? enqueue_right(d, phi_in, A, x, phi_out, T1, T2, Ah, Pp, pe, s)
                                            : enqueue_right_mirror(d, phi_in, A, x, phi_out, T1, T2, Ah, Pp, pe, s);
  if (e != cudaSuccess) return cuda_fail(e, left ? "tt_interface_left" : "tt_interface_right");
  return TT_OK;
}

tt_status tt_interface_left(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                            const double* phiL_prev, const double* A, const double* x,
                            double* phiL_next, void* workspace, size_t workspace_bytes,
                            void* stream) {
  CallScope scope;
  return iface_common(true, rl, n, rr, Rl, Rr, phiL_prev, A, x, phiL_next, workspace,
                      workspace_bytes, stream);
}

tt_status tt_interface_right(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                             const double* phiR_next, const double* A, const double* x,
                             double* phiR_prev, void* workspace, size_t workspace_bytes,
                             void* stream) {
  CallScope scope;
  return iface_common(false, rl, n, rr, Rl, Rr, phiR_next, A, x, phiR_prev, workspace,
                      workspace_bytes, stream);
}

// ---- sweeps ------------------------------------------------------------------------------
static tt_status check_train(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R) {
  if (d <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "d must be >= 1");
  if (!n || !r || !R) return fail(TT_ERR_NULL_POINTER, "NULL shape array");
  if (r[0] != 1 || r[d] != 1) return fail(TT_ERR_INVALID_ARGUMENT, "r_1 and r_{d+1} must be 1");
  if (R[0] != 1 || R[d] != 1) return fail(TT_ERR_INVALID_ARGUMENT, "R_1 and R_{d+1} must be 1");
  for (int64_t k = 0; k < d; ++k) {
    Dims dk{r[k], n[k], r[k + 1], R[k], R[k + 1]};
    tt_status st = check_dims(dk);
    if (st != TT_OK) return fail(st, "core " + std::to_string(k) + ": " + g_msg);
  }
  return TT_OK;
}

// Sweep workspace = [per-stage scratch (max over cores and stage kinds)] [prepared operands
// of every core: Ahl, Ahr (alpha n^2 beta each), xt (r_k n r_{k+1})].
static long long prep_elems(const Dims& d) {
  return 2 * d.al * d.n * d.n * d.be + d.a * d.n * d.b;
}
static size_t sweep_step_ws(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                            int64_t nvec);
// [main-stream scratch: max over cores of the interface / matvec stage scratch]
// [side-stream scratch: max over cores of the interface stage scratch] [prepared operands]
static size_t sweep_prep_offset(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                                int64_t nvec) {
  const size_t main_b = sweep_step_ws(d, n, r, R, nvec);
  const size_t side_b = sweep_step_ws(d, n, r, R, 0);
  if (main_b == 0 || side_b == 0) return 0;
  return align_up(main_b, 256) + align_up(side_b, 256);
}
static size_t sweep_ws(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                       int64_t nvec) {
  size_t base = sweep_prep_offset(d, n, r, R, nvec);
  if (base == 0) return 0;
  for (int64_t k = 0; k < d; ++k) {
    Dims dk{r[k], n[k], r[k + 1], R[k], R[k + 1]};
    base += align_up(size_t(prep_elems(dk)) * sizeof(double), 256) + 256;
  }
  return base;
}
struct Prep {
  const double *Ahl, *Ahr, *xt;
};
// pointers of core k's prepared operands inside the workspace
static Prep prep_ptrs(int64_t k, int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                      int64_t nvec, void* ws) {
  size_t off = sweep_prep_offset(d, n, r, R, nvec);
  char* base = static_cast<char*>(ws);
  for (int64_t q = 0; q <= k; ++q) {
    Dims dq{r[q], n[q], r[q + 1], R[q], R[q + 1]};
    uintptr_t p = (reinterpret_cast<uintptr_t>(base) + off + 255) & ~uintptr_t(255);
    if (q == k) {
      const double* Ahl = reinterpret_cast<const double*>(p);
      const double* Ahr = Ahl + dq.al * dq.n * dq.n * dq.be;
      const double* xt = Ahr + dq.al * dq.n * dq.n * dq.be;
      return Prep{Ahl, Ahr, xt};
    }
    off = (p - reinterpret_cast<uintptr_t>(base)) + size_t(prep_elems(dq)) * sizeof(double);
  }
  return Prep{nullptr, nullptr, nullptr};
}
// one launch per kPrepMax cores (all of them in practice); one0/one1 (nullable) are set to 1
static cudaError_t launch_prep(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                               int64_t nvec, const double* const* xc, const double* const* Ac,
                               void* ws, cudaStream_t s, double* one0 = nullptr,
                               double* one1 = nullptr) {
  for (int64_t k0 = 0; k0 < d; k0 += kPrepMax) {
    PrepTable t;
    t.cores = (int)std::min<int64_t>(kPrepMax, d - k0);
    t.one0 = k0 == 0 ? one0 : nullptr;
    t.one1 = k0 == 0 ? one1 : nullptr;
    long long blocks = 0, total = 0;
    for (int c = 0; c < t.cores; ++c) {
      const int64_t k = k0 + c;
      Dims dk{r[k], n[k], r[k + 1], R[k], R[k + 1]};
      Prep pp = prep_ptrs(k, d, n, r, R, nvec, ws);
      t.A[c] = Ac[k];
      t.x[c] = xc[k];
      t.Ahl[c] = const_cast<double*>(pp.Ahl);
      t.Ahr[c] = const_cast<double*>(pp.Ahr);
      t.xt[c] = const_cast<double*>(pp.xt);
      t.al[c] = (int)dk.al; t.n[c] = (int)dk.n; t.be[c] = (int)dk.be;
      t.a[c] = (int)dk.a; t.b[c] = (int)dk.b;
      const long long el = prep_elems(dk);
      total += el;
      t.start[c] = (int)blocks;
      blocks += std::min<long long>(2048, (el + 255) / 256);
    }
    t.start[t.cores] = (int)blocks;
    g_stage = TT_ST_PERM;
    const long long tr = trace_begin(0, total, 0, 0, s);
    if (cudaError_t e = launch_pdl(true, prep_all_kernel, dim3((unsigned)blocks), dim3(256), 0, s, t))
      return e;
    trace_end(tr, s);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
static size_t sweep_step_ws(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                            int64_t nvec) {
  size_t best = 0;
  for (int64_t k = 0; k < d; ++k) {
    Dims dk{r[k], n[k], r[k + 1], R[k], R[k + 1]};
    long long t1, t2, ah, pe;
    if (!iface_ws_elems(dk, t1, t2, ah, pe)) return 0;
    size_t s = ws_bytes({t1, t2, ah, pe});
    if (s > best) best = s;
    if (nvec > 0) {
      if (!matvec_ws_elems(dk, nvec, t1, t2, ah, pe)) return 0;
      s = ws_bytes({t1, t2, ah, pe});
      if (s > best) best = s;
    }
  }
  return best;
}

size_t tt_sweep_workspace_size(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R) {
  if (d <= 0 || !n || !r || !R) return 0;
  return sweep_ws(d, n, r, R, 0);
}

size_t tt_sweep_als_workspace_size(int64_t d, const int64_t* n, const int64_t* r,
                                   const int64_t* R, int64_t nvec) {
  if (d <= 0 || !n || !r || !R || nvec <= 0) return 0;
  return sweep_ws(d, n, r, R, nvec);
}

// carve the workspace for core k (interface or matvec) and enqueue
static cudaError_t sweep_left_step(int64_t k, int64_t d, int64_t nvec, void* scratch, const int64_t* n,
                                   const int64_t* r, const int64_t* R, const double* const* xc,
                                   const double* const* Ac, double* const* phiL, void* ws,
                                   size_t wsb, cudaStream_t s, double* T2_keep = nullptr,
                                   cudaEvent_t ev_t2 = nullptr) {
  Dims dk{r[k], n[k], r[k + 1], R[k], R[k + 1]};
  long long t1, t2, ah, pe;
  iface_ws_elems(dk, t1, t2, ah, pe);
  Carver c{static_cast<char*>(scratch), wsb};
  double* T1 = c.take(t1);
  double* T2 = c.take(t2);
  double* Ah = c.take(ah);
  double* Pp = c.take(pe);
  if (!c.ok) return cudaErrorInvalidValue;
  if (T2_keep) T2 = T2_keep;
  const Prep pp = prep_ptrs(k, d, n, r, R, nvec, ws);
  return enqueue_left(dk, phiL[k], Ac[k], xc[k], phiL[k + 1], T1, T2, Ah, Pp, pe, s,
                      TT_ST_IL_S1, pp.Ahl, ev_t2);
}

static cudaError_t sweep_right_step(int64_t k, int64_t d, int64_t nvec, void* scratch, const int64_t* n,
                                    const int64_t* r, const int64_t* R, const double* const* xc,
                                    const double* const* Ac, double* const* phiR, void* ws,
                                    size_t wsb, cudaStream_t s) {
  Dims dk{r[k], n[k], r[k + 1], R[k], R[k + 1]};
  long long t1, t2, ah, pe;
  iface_ws_elems(dk, t1, t2, ah, pe);
  Carver c{static_cast<char*>(scratch), wsb};
  double* T1 = c.take(t1);
  double* T2 = c.take(t2);
  double* Ah = c.take(ah);
  double* Pp = c.take(pe);
  if (!c.ok) return cudaErrorInvalidValue;
  if (g_dbg_flags & 8) return enqueue_right(dk, phiR[k + 1], Ac[k], xc[k], phiR[k], T1, T2, Ah, Pp, pe, s);
  const Prep pp = prep_ptrs(k, d, n, r, R, nvec, ws);
  return enqueue_right_mirror(dk, phiR[k + 1], Ac[k], xc[k], phiR[k], T1, T2, Ah, Pp, pe, s,
                              pp.Ahr, pp.xt);
}

static cudaError_t sweep_matvec_step(int64_t k, int64_t d, void* scratch, const int64_t* n, const int64_t* r,
                                     const int64_t* R, int64_t nvec, const double* const* Ac,
                                     const double* const* Xb, double* const* Yb,
                                     double* const* phiL, double* const* phiR, void* ws,
                                     size_t wsb, cudaStream_t s) {
  Dims dk{r[k], n[k], r[k + 1], R[k], R[k + 1]};
  long long t1, t2, ah, pe;
  matvec_ws_elems(dk, nvec, t1, t2, ah, pe);
  Carver c{static_cast<char*>(scratch), wsb};
  double* T1 = c.take(t1);
  double* T2 = c.take(t2);
  double* Ah = c.take(ah);
  double* Pp = c.take(pe);
  if (!c.ok) return cudaErrorInvalidValue;
  const Prep pp = prep_ptrs(k, d, n, r, R, nvec, ws);
  return enqueue_matvec(dk, nvec, phiL[k], Ac[k], phiR[k + 1], Xb[k], Yb[k], T1, T2, Ah, Pp, pe,
                        s, pp.Ahl);
}

static tt_status check_ptrs(int64_t d, const void* const* arr, int64_t count, const char* what) {
  if (!arr) return fail(TT_ERR_NULL_POINTER, std::string("NULL array ") + what);
  for (int64_t k = 0; k < count; ++k)
    if (!arr[k]) return fail(TT_ERR_NULL_POINTER, std::string("NULL entry in ") + what);
  (void)d;
  return TT_OK;
}

// outputs (phi arrays, Y blocks) must not alias inputs (cores, blocks) nor each other
static tt_status check_outputs(int64_t d, const double* const* xc, const double* const* Ac,
                               const double* const* Xb,
                               std::initializer_list<std::pair<double* const*, int64_t>> outs,
                               void* ws) {
  std::vector<const void*> ins;
  for (int64_t k = 0; k < d; ++k) {
    ins.push_back(xc[k]);
    ins.push_back(Ac[k]);
    if (Xb) ins.push_back(Xb[k]);
  }
  std::vector<const void*> os;
  for (auto& pr : outs)
    if (pr.first)
      for (int64_t k = 0; k < pr.second; ++k) os.push_back(pr.first[k]);
  for (size_t i = 0; i < os.size(); ++i) {
    for (const void* q : ins)
      if (os[i] == q) return fail(TT_ERR_ALIASING, "an output aliases an input core");
    for (size_t j = i + 1; j < os.size(); ++j)
      if (os[i] == os[j]) return fail(TT_ERR_ALIASING, "two outputs alias");
    if (ws && os[i] == ws) return fail(TT_ERR_ALIASING, "an output aliases the workspace");
  }
  return TT_OK;
}

tt_status tt_sweep_interfaces(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                              const double* const* x_cores, const double* const* A_cores,
                              double* const* phiL, double* const* phiR, int directions,
                              void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  tt_status st = check_train(d, n, r, R);
  if (st != TT_OK) return st;
  if (directions < 1 || directions > 3) return fail(TT_ERR_INVALID_ARGUMENT, "bad directions");
  if ((st = check_ptrs(d, (const void* const*)x_cores, d, "x_cores")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)A_cores, d, "A_cores")) != TT_OK) return st;
  const bool doL = (directions & TT_SWEEP_LEFT) && phiL;
  const bool doR = (directions & TT_SWEEP_RIGHT) && phiR;
  if (doL && (st = check_ptrs(d, (const void* const*)phiL, d + 1, "phiL")) != TT_OK) return st;
  if (doR && (st = check_ptrs(d, (const void* const*)phiR, d + 1, "phiR")) != TT_OK) return st;
  if ((st = check_outputs(d, x_cores, A_cores, nullptr,
                          {{doL ? phiL : nullptr, d + 1}, {doR ? phiR : nullptr, d + 1}},
                          workspace)) != TT_OK)
    return st;
  const size_t need = sweep_ws(d, n, r, R, 0);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  char* wsb = static_cast<char*>(workspace);
  const size_t main_b = sweep_step_ws(d, n, r, R, 0);
  void* ws_main = wsb;
  void* ws_side = wsb + align_up(main_b, 256);
  if ((doL || doR) && (e = launch_prep(d, n, r, R, 0, x_cores, A_cores, workspace, s,
                                      doL ? phiL[0] : nullptr, doR ? phiR[d] : nullptr)) != cudaSuccess)
    return cuda_fail(e, "sweep prep");
  // the two chains are independent: left on the caller's stream, right on the side stream
  cudaStream_t sr = s;
  if (doL && doR) {
    if ((e = side_stream(&sr)) != cudaSuccess) return cuda_fail(e, "side stream");
    if ((e = stream_dep(s, sr)) != cudaSuccess) return cuda_fail(e, "fork");
  }
  if (doL) {
    for (int64_t k = 0; k < d; ++k)
      if ((e = sweep_left_step(k, d, 0, ws_main, n, r, R, x_cores, A_cores, phiL, workspace,
                               main_b, s)) != cudaSuccess)
        return cuda_fail(e, "sweep left");
  }
  if (doR) {
    void* wr = (sr == s) ? ws_main : ws_side;
    for (int64_t k = d - 1; k >= 0; --k)
      if ((e = sweep_right_step(k, d, 0, wr, n, r, R, x_cores, A_cores, phiR, workspace, main_b,
                                sr)) != cudaSuccess)
        return cuda_fail(e, "sweep right");
  }
  if (sr != s && (e = stream_dep(sr, s)) != cudaSuccess) return cuda_fail(e, "join");
  return TT_OK;
}

// ---- W34 as one DAG-scheduled call: both interface chains and one matvec per core ---------
// Workspace: [sweep workspace (chain scratch x2, prepared operands)] [kPoolStreams matvec
// scratches].  The left chain runs on the caller's stream, the right chain on the side
// stream, and core k's matvec on a pool stream as soon as phiL[k] and phiR[k+1] exist
// (events), middle cores first -- so the matvecs overlap the chains.
static size_t w34_mv_scratch(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R) {
  size_t best = 0;
  for (int64_t k = 0; k < d; ++k) {
    Dims dk{r[k], n[k], r[k + 1], R[k], R[k + 1]};
    long long t1, t2, ah, pe;
    if (!matvec_ws_elems(dk, 1, t1, t2, ah, pe)) return 0;
    best = std::max(best, ws_bytes({t1, t2, ah, pe}));
  }
  return best;
}

// W34 keeps every left update's stage-2 intermediate T2_k (a', i, be, b): with K = 1 it is
// also the matvec's stage-2 output at core k (same phiL[k], A_k, x_k), so the matvec is only
// its last stage, y_k = T2_k . phiR[k+1]^T
static size_t w34_t2_keep(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R) {
  size_t tot = 256;
  for (int64_t k = 0; k < d; ++k) {
    bool ok = true;
    const long long e = prod({r[k], n[k], R[k + 1], r[k + 1]}, ok);
    if (!ok) return 0;
    tot += align_up((size_t)e * 8, 256);
  }
  return tot;
}

size_t tt_sweep_w34_workspace_size(int64_t d, const int64_t* n, const int64_t* r,
                                   const int64_t* R) {
  if (d <= 0 || !n || !r || !R) return 0;
  const size_t base = sweep_ws(d, n, r, R, 0), mv = w34_mv_scratch(d, n, r, R);
  const size_t keep = w34_t2_keep(d, n, r, R);
  if (base == 0 || mv == 0 || keep == 0) return 0;
  return align_up(base, 256) + kPoolStreams * align_up(mv, 256) + keep + 256;
}

tt_status tt_sweep_w34(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                       const double* const* x_cores, const double* const* A_cores,
                       double* const* phiL, double* const* phiR, double* const* y_cores,
                       void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  tt_status st = check_train(d, n, r, R);
  if (st != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)x_cores, d, "x_cores")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)A_cores, d, "A_cores")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)phiL, d + 1, "phiL")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)phiR, d + 1, "phiR")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)y_cores, d, "y_cores")) != TT_OK) return st;
  if ((st = check_outputs(d, x_cores, A_cores, nullptr, {{phiL, d + 1}, {phiR, d + 1}, {y_cores, d}},
                          workspace)) != TT_OK)
    return st;
  const size_t need = tt_sweep_w34_workspace_size(d, n, r, R);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  char* wsb = static_cast<char*>(workspace);
  const size_t main_b = sweep_step_ws(d, n, r, R, 0);
  void* ws_main = wsb;
  void* ws_side = wsb + align_up(main_b, 256);
  const size_t mv_b = w34_mv_scratch(d, n, r, R);
  char* mv_base = wsb + align_up(sweep_ws(d, n, r, R, 0), 256);
  if ((e = pool_init(size_t(3 * (d + 1) + kPoolStreams + 4))) != cudaSuccess) return cuda_fail(e, "pool");
  cudaEvent_t* evL = g_pool.ev.data();         // evL[k]: phiL[k] ready
  cudaEvent_t* evR = evL + (d + 1);            // evR[k]: phiR[k] ready
  cudaEvent_t* evT = evR + (d + 1);            // evT[k]: the left update's T2_k ready
  cudaEvent_t* evJ = evT + (d + 1);            // joins
  // T2 reuse (debug bit 23 restores the three-stage matvecs)
  const bool reuse = !(g_dbg_flags & 8388608);
  std::vector<double*> T2k(d, nullptr);
  if (reuse) {
    char* kb = mv_base + kPoolStreams * align_up(mv_b, 256);
    kb += (256 - (reinterpret_cast<uintptr_t>(kb) & 255)) & 255;
    for (int64_t k = 0; k < d; ++k) {
      T2k[k] = reinterpret_cast<double*>(kb);
      kb += align_up((size_t)(r[k] * n[k] * R[k + 1] * r[k + 1]) * 8, 256);
    }
  }
  if ((e = launch_prep(d, n, r, R, 0, x_cores, A_cores, workspace, s, phiL[0], phiR[d])) != cudaSuccess)
    return cuda_fail(e, "sweep prep");
  cudaStream_t sr;
  if ((e = side_stream(&sr)) != cudaSuccess) return cuda_fail(e, "side stream");
  if ((e = stream_dep(s, sr)) != cudaSuccess) return cuda_fail(e, "fork");
  for (int q = 0; q < kPoolStreams; ++q)
    if ((e = stream_dep(s, g_pool.s[q])) != cudaSuccess) return cuda_fail(e, "fork");
  // the two chains, on high-priority streams (the critical path)
  cudaStream_t sl = g_pool.chain;
  if ((e = stream_dep(s, sl)) != cudaSuccess) return cuda_fail(e, "fork");
  if ((e = cudaEventRecord(evL[0], sl)) != cudaSuccess) return cuda_fail(e, "event");
  for (int64_t k = 0; k < d; ++k) {
    if ((e = sweep_left_step(k, d, 0, ws_main, n, r, R, x_cores, A_cores, phiL, workspace, main_b,
                             sl, T2k[k], reuse ? evT[k] : nullptr)) != cudaSuccess)
      return cuda_fail(e, "sweep left");
    if ((e = cudaEventRecord(evL[k + 1], sl)) != cudaSuccess) return cuda_fail(e, "event");
  }
  if ((e = cudaEventRecord(evR[d], sr)) != cudaSuccess) return cuda_fail(e, "event");
  for (int64_t k = d - 1; k >= 0; --k) {
    if ((e = sweep_right_step(k, d, 0, ws_side, n, r, R, x_cores, A_cores, phiR, workspace,
                              main_b, sr)) != cudaSuccess)
      return cuda_fail(e, "sweep right");
    if ((e = cudaEventRecord(evR[k], sr)) != cudaSuccess) return cuda_fail(e, "event");
  }
  // matvecs in readiness order (core k needs k left steps and d-1-k right steps)
  std::vector<int64_t> order(d);
  for (int64_t k = 0; k < d; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int64_t p, int64_t q) {
    return std::max(p, d - 1 - p) < std::max(q, d - 1 - q);
  });
  for (int64_t i = 0; i < d; ++i) {
    const int64_t k = order[i];
    const int q = (int)(i % kPoolStreams);
    cudaStream_t ps = g_pool.s[q];
    if ((e = cudaStreamWaitEvent(ps, reuse ? evT[k] : evL[k], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if ((e = cudaStreamWaitEvent(ps, evR[k + 1], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    Dims dk{r[k], n[k], r[k + 1], R[k], R[k + 1]};
    long long t1, t2, ah, pe;
    matvec_ws_elems(dk, 1, t1, t2, ah, pe);
    Carver c{mv_base + q * align_up(mv_b, 256), mv_b};
    double* T1 = c.take(t1);
    double* T2 = c.take(t2);
    double* Ah = c.take(ah);
    double* Pp = c.take(pe);
    if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
    if (reuse) {
      if ((e = enqueue_matvec_last(dk, 1, T2k[k], phiR[k + 1], y_cores[k], Pp, pe, ps)) != cudaSuccess)
        return cuda_fail(e, "sweep matvec");
      continue;
    }
    const Prep pp = prep_ptrs(k, d, n, r, R, 0, workspace);
    if ((e = enqueue_matvec(dk, 1, phiL[k], A_cores[k], phiR[k + 1], x_cores[k], y_cores[k], T1,
                            T2, Ah, Pp, pe, ps, pp.Ahl)) != cudaSuccess)
      return cuda_fail(e, "sweep matvec");
  }
  // join everything back into the caller's stream
  if ((e = cudaEventRecord(evJ[0], sr)) != cudaSuccess || (e = cudaStreamWaitEvent(s, evJ[0], 0)) != cudaSuccess)
    return cuda_fail(e, "join");
  if ((e = cudaEventRecord(evJ[1 + kPoolStreams], sl)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(s, evJ[1 + kPoolStreams], 0)) != cudaSuccess)
    return cuda_fail(e, "join");
  for (int q = 0; q < kPoolStreams; ++q)
    if ((e = cudaEventRecord(evJ[1 + q], g_pool.s[q])) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s, evJ[1 + q], 0)) != cudaSuccess)
      return cuda_fail(e, "join");
  return TT_OK;
}

tt_status tt_sweep_als(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                       int64_t nvec, const double* const* x_cores,
                       const double* const* A_cores, const double* const* X_blocks,
                       double* const* Y_fwd, double* const* Y_bwd, double* const* phiL,
                       double* const* phiR, void* workspace, size_t workspace_bytes,
                       void* stream) {
  CallScope scope;
  tt_status st = check_train(d, n, r, R);
  if (st != TT_OK) return st;
  if (nvec <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "nvec must be positive");
  if ((st = check_ptrs(d, (const void* const*)x_cores, d, "x_cores")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)A_cores, d, "A_cores")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)X_blocks, d, "X_blocks")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)Y_fwd, d, "Y_fwd")) != TT_OK) return st;
  if (Y_bwd && (st = check_ptrs(d, (const void* const*)Y_bwd, d, "Y_bwd")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)phiL, d + 1, "phiL")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)phiR, d + 1, "phiR")) != TT_OK) return st;
  if ((st = check_outputs(d, x_cores, A_cores, X_blocks,
                          {{Y_fwd, d}, {Y_bwd, d}, {phiL, d + 1}, {phiR, d + 1}}, workspace)) !=
      TT_OK)
    return st;
  const size_t need = sweep_ws(d, n, r, R, nvec);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  double* const* Yb = Y_bwd ? Y_bwd : Y_fwd;
  char* wsb = static_cast<char*>(workspace);
  const size_t main_b = sweep_step_ws(d, n, r, R, nvec);
  const size_t side_b = sweep_step_ws(d, n, r, R, 0);
  void* ws_main = wsb;
  void* ws_side = wsb + align_up(main_b, 256);
  // W5 is throughput-bound: plain launches (PDL measured 0.2 % slower on the whole sweep)
  struct NoPdl {
    bool saved = g_no_pdl;
    NoPdl() { g_no_pdl = true; }
    ~NoPdl() { g_no_pdl = saved; }
  } no_pdl;
  cudaStream_t ss;
  if ((e = side_stream(&ss)) != cudaSuccess) return cuda_fail(e, "side stream");
  if ((e = launch_prep(d, n, r, R, nvec, x_cores, A_cores, workspace, s, phiL[0], phiR[d])) !=
      cudaSuccess)
    return cuda_fail(e, "als prep");
  for (int64_t k = d - 1; k >= 1; --k)
    if ((e = sweep_right_step(k, d, nvec, ws_main, n, r, R, x_cores, A_cores, phiR, workspace,
                              main_b, s)) != cudaSuccess)
      return cuda_fail(e, "als initial right");
  // L->R: the left-interface chain runs on the side stream, one step ahead of the matvecs,
  // which wait only for the interface they read (matvec(k) needs phiL[k] = IL(k-1)).
  if ((e = stream_dep(s, ss)) != cudaSuccess) return cuda_fail(e, "fork");
  for (int64_t k = 0; k < d; ++k) {
    if (k > 0 && (e = stream_dep(ss, s)) != cudaSuccess) return cuda_fail(e, "dep");
    if ((e = sweep_matvec_step(k, d, ws_main, n, r, R, nvec, A_cores, X_blocks, Y_fwd, phiL, phiR,
                               workspace, main_b, s)) != cudaSuccess)
      return cuda_fail(e, "als matvec L->R");
    if (k < d - 1 && (e = sweep_left_step(k, d, nvec, ws_side, n, r, R, x_cores, A_cores, phiL,
                                          workspace, side_b, ss)) != cudaSuccess)
      return cuda_fail(e, "als left");
  }
  // R->L: the right chain recomputes phiR[k] (k = d-1..1) on the side stream; matvec(k)
  // needs phiR[k+1] = IR(k+1).  Both streams first wait for the whole L->R pass.
  if ((e = stream_dep(s, ss)) != cudaSuccess) return cuda_fail(e, "fork");
  for (int64_t k = d - 1; k >= 0; --k) {
    if (k < d - 1 && (e = stream_dep(ss, s)) != cudaSuccess) return cuda_fail(e, "dep");
    if ((e = sweep_matvec_step(k, d, ws_main, n, r, R, nvec, A_cores, X_blocks, Yb, phiL, phiR,
                               workspace, main_b, s)) != cudaSuccess)
      return cuda_fail(e, "als matvec R->L");
    if (k > 0 && (e = sweep_right_step(k, d, nvec, ws_side, n, r, R, x_cores, A_cores, phiR,
                                       workspace, side_b, ss)) != cudaSuccess)
      return cuda_fail(e, "als right");
  }
  if ((e = stream_dep(ss, s)) != cudaSuccess) return cuda_fail(e, "join");
  return TT_OK;
}

// ---- H8 ----------------------------------------------------------------------------------
tt_status tt_operator_apply(int64_t d, const int64_t* n_row, const int64_t* n_col,
                            const int64_t* r, const int64_t* R, const double* const* x_cores,
                            const double* const* A_cores, double* const* z_cores, void* stream) {
  CallScope scope;
  if (d <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "d must be >= 1");
  if (!n_row || !n_col || !r || !R) return fail(TT_ERR_NULL_POINTER, "NULL shape array");
  if (r[0] != 1 || r[d] != 1) return fail(TT_ERR_INVALID_ARGUMENT, "r_1 and r_{d+1} must be 1");
  if (R[0] != 1 || R[d] != 1) return fail(TT_ERR_INVALID_ARGUMENT, "R_1 and R_{d+1} must be 1");
  tt_status st;
  if ((st = check_ptrs(d, (const void* const*)x_cores, d, "x_cores")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)A_cores, d, "A_cores")) != TT_OK) return st;
  if ((st = check_ptrs(d, (const void* const*)z_cores, d, "z_cores")) != TT_OK) return st;
  if ((st = check_outputs(d, x_cores, A_cores, nullptr, {{z_cores, d}}, nullptr)) != TT_OK)
    return st;
  int dev = 0;
  cudaGetDevice(&dev);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  for (int64_t k = 0; k < d; ++k) {
    if (n_row[k] <= 0 || n_col[k] <= 0 || r[k] <= 0 || R[k] <= 0)
      return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
    bool ok = true;
    prod({r[k], R[k], n_row[k], r[k + 1], R[k + 1]}, ok);
    prod({R[k], n_row[k], n_col[k], R[k + 1]}, ok);
    prod({r[k], n_col[k], r[k + 1]}, ok);
    if (!ok) return fail(TT_ERR_OVERFLOW, "extent product overflows");
    const long long smem = 8LL * (n_col[k] * r[k + 1] + n_row[k] * n_col[k] * R[k + 1]);
    if (smem > smem_optin || r[k + 1] * R[k + 1] > 0x7fffffffLL || r[k] * R[k] > 0x7fffffffLL)
      return fail(TT_ERR_INVALID_ARGUMENT, "core too large for the apply kernel's staging");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem_optin);
  });
  if (attr_err != cudaSuccess) return cuda_fail(attr_err, "tt_operator_apply attr");
  for (int64_t k = 0; k < d; ++k) {
    const long long smem = 8LL * (n_col[k] * r[k + 1] + n_row[k] * n_col[k] * R[k + 1]);
    const long long blocks = r[k] * R[k];
    g_stage = TT_ST_APPLY;
    const long long tr = trace_begin(0, r[k] * R[k] * n_row[k] * r[k + 1] * R[k + 1], n_col[k], 0, s);
    cudaError_t e = cudaSuccess;
    const long long L = r[k + 1] * R[k + 1];
    if (n_col[k] <= 4 && L >= 256 && (r[k] + 3) / 4 <= 65535 && R[k] <= 65535) {
      switch (n_col[k]) {
        case 1: e = launch_apply_reg<1>(x_cores[k], A_cores[k], z_cores[k], r[k], n_row[k], r[k + 1], R[k], R[k + 1], s); break;
        case 2: e = launch_apply_reg<2>(x_cores[k], A_cores[k], z_cores[k], r[k], n_row[k], r[k + 1], R[k], R[k + 1], s); break;
        case 3: e = launch_apply_reg<3>(x_cores[k], A_cores[k], z_cores[k], r[k], n_row[k], r[k + 1], R[k], R[k + 1], s); break;
        default: e = launch_apply_reg<4>(x_cores[k], A_cores[k], z_cores[k], r[k], n_row[k], r[k + 1], R[k], R[k + 1], s); break;
      }
    } else {
      apply_kernel<<<(unsigned)blocks, 256, (size_t)smem, s>>>(
          x_cores[k], A_cores[k], z_cores[k], (int)r[k], (int)n_row[k], (int)n_col[k],
          (int)r[k + 1], (int)R[k], (int)R[k + 1]);
      e = cudaGetLastError();
    }
    trace_end(tr, s);
    ++g_launches;
    if (e != cudaSuccess) return cuda_fail(e, "tt_operator_apply");
  }
  return TT_OK;
}

// test hook: symmetric eigendecomposition of an n x n matrix (G overwritten), lam descending
tt_status tt_debug_sym_eigen(int64_t n, double* G, double* V, double* lam, void* workspace,
                             size_t workspace_bytes, void* stream) {
  CallScope scope;
  if (n <= 0 || n > 2048) return fail(TT_ERR_INVALID_ARGUMENT, "0 < n <= 2048");
  if (!G || !V || !lam || !workspace) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  if (workspace_bytes < (size_t)sym_eigen_scratch(n) * 8) return fail(TT_ERR_WORKSPACE, "workspace");
  g_eigen_elementwise = (g_dbg_flags & 256) ? 1 : 0;
  cudaError_t e = launch_sym_eigen(G, V, lam, (int)n, static_cast<double*>(workspace),
                                   static_cast<cudaStream_t>(stream));
  g_eigen_elementwise = 0;
  if (e != cudaSuccess) return cuda_fail(e, "tt_debug_sym_eigen");
  return TT_OK;
}

// ---- TT rounding ------------------------------------------------------
size_t tt_round_workspace_size(int64_t d, const int64_t* n, const int64_t* r) {
  if (d <= 0 || !n || !r) return 0;
  long long core_max = 0, rmax = 0, tot = 0;
  bool ok = true;
  for (int64_t k = 0; k < d; ++k) {
    const long long sz = prod({r[k], n[k], r[k + 1]}, ok);
    core_max = std::max(core_max, sz);
    tot += align_up((size_t)sz * 8, 256) / 8 + 32;
  }
  for (int64_t k = 0; k <= d; ++k) rmax = std::max<long long>(rmax, r[k]);
  if (!ok) return 0;
  // working cores, one temp core, G, V, Bm (rmax^2 each), d, lam (rmax), eigen scratch
  return ws_bytes({tot, core_max, rmax * rmax, rmax * rmax, rmax * rmax, rmax, rmax,
                   sym_eigen_scratch(rmax)});
}

// phases: bit 0 = right-to-left orthonormalisation, bit 1 = left-to-right truncation
// (delta = 0, max_rank = 0: plain left-to-right orthonormalisation)
static tt_status round_impl(int64_t d, const int64_t* n, const int64_t* r_in,
                            const double* const* cores_in, double delta, int64_t max_rank,
                            int64_t* r_out, double* const* cores_out, void* workspace,
                            size_t workspace_bytes, void* stream, int phases, const char* who) {
  if (d <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "d must be >= 1");
  if (!n || !r_in || !cores_in || !r_out || !cores_out) return fail(TT_ERR_NULL_POINTER, "NULL array");
  if (r_in[0] != 1 || r_in[d] != 1) return fail(TT_ERR_INVALID_ARGUMENT, "r_1 and r_{d+1} must be 1");
  if (!(delta >= 0.0)) return fail(TT_ERR_INVALID_ARGUMENT, "delta must be >= 0");
  long long rmax = 0;
  for (int64_t k = 0; k < d; ++k) {
    if (n[k] <= 0 || r_in[k] <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
    if (!cores_in[k] || !cores_out[k]) return fail(TT_ERR_NULL_POINTER, "NULL core");
    for (int64_t q = 0; q < d; ++q)
      if ((const void*)cores_out[k] == (const void*)cores_in[q])
        return fail(TT_ERR_ALIASING, "an output core aliases an input core");
    rmax = std::max<long long>(rmax, r_in[k]);
  }
  if (rmax > 512) return fail(TT_ERR_INVALID_ARGUMENT, "ranks above 512 are not supported");
  const size_t need = tt_round_workspace_size(d, n, r_in);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  std::vector<double*> W(d);
  long long core_max = 0;
  for (int64_t k = 0; k < d; ++k) {
    const long long sz = r_in[k] * n[k] * r_in[k + 1];
    W[k] = c.take(sz);
    core_max = std::max(core_max, sz);
  }
  double* Tmp = c.take(core_max);
  double* G = c.take(rmax * rmax);
  double* V = c.take(rmax * rmax);
  double* Bm = c.take(rmax * rmax);
  double* dg = c.take(rmax);
  double* lam = c.take(rmax);
  double* esc = c.take(sym_eigen_scratch(rmax));
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  std::vector<long long> r(r_in, r_in + d + 1);
  cudaError_t e = cudaSuccess;
  for (int64_t k = 0; k < d && e == cudaSuccess; ++k)
    e = cudaMemcpyAsync(W[k], cores_in[k], sizeof(double) * r[k] * n[k] * r[k + 1],
                        cudaMemcpyDeviceToDevice, s);
  std::vector<double> hl(rmax);
  auto eig = [&](int m) -> cudaError_t {   // G (m x m) -> V, lam (host copy in hl)
    cudaError_t er = launch_sym_eigen(G, V, lam, m, esc, s);
    if (er != cudaSuccess) return er;
    er = cudaMemcpyAsync(hl.data(), lam, sizeof(double) * m, cudaMemcpyDeviceToHost, s);
    if (er != cudaSuccess) return er;
    return cudaStreamSynchronize(s);
  };
  // scaled copies of the leading eigenvector columns: Bm[:, :s] = V[:, :s] * f
  std::vector<double> hf(rmax);
  auto scaled = [&](int m, int cols, const std::vector<double>& f) -> cudaError_t {
    cudaError_t er = cudaMemcpyAsync(dg, f.data(), sizeof(double) * cols, cudaMemcpyHostToDevice, s);
    if (er != cudaSuccess) return er;
    scale_cols_kernel<<<(m * cols + 255) / 256, 256, 0, s>>>(V, dg, Bm, m, cols);
    ++g_launches;
    return cudaGetLastError();
  };
  const double zero_rel = 1e-14;   // relative eigenvalue floor (numerical zero of the Gram)
  // right-to-left orthonormalisation: W_k = (V S)(S^-1 V^T W_k), W_{k-1} <- W_{k-1} V S
  for (int64_t k = d - 1; (phases & 1) && k >= 1 && e == cudaSuccess; --k) {
    const long long rk = r[k], q = n[k] * r[k + 1];
    g_stage = TT_ST_IL_S1;
    e = launch_gemm(true, true, gp(W[k], q, W[k], q, G, rk, rk, q, tt::map_plain(rk),
                                   tt::map_plain(1)), s);
    if (e == cudaSuccess) e = eig((int)rk);
    if (e != cudaSuccess) break;
    int sk = 0;
    for (long long i = 0; i < rk; ++i)
      if (hl[i] > zero_rel * hl[0] && hl[i] > 0.0) ++sk;
    if (sk == 0) sk = 1;
    for (int i = 0; i < sk; ++i) hf[i] = 1.0 / std::sqrt(std::max(hl[i], 1e-300));
    if ((e = scaled((int)rk, sk, hf)) != cudaSuccess) break;
    // Tmp (sk x q) = (V S^-1)^T W_k
    e = launch_gemm(false, false, gp(Bm, sk, W[k], q, Tmp, sk, q, rk, tt::map_plain(q),
                                     tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k], Tmp, sizeof(double) * sk * q, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) break;
    for (int i = 0; i < sk; ++i) hf[i] = std::sqrt(std::max(hl[i], 0.0));
    if ((e = scaled((int)rk, sk, hf)) != cudaSuccess) break;
    // W_{k-1} (r_{k-1} n x sk) = W_{k-1} (r_{k-1} n x rk) . (V S)
    const long long m1 = r[k - 1] * n[k - 1];
    e = launch_gemm(true, false, gp(W[k - 1], rk, Bm, sk, Tmp, m1, sk, rk, tt::map_plain(sk),
                                    tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k - 1], Tmp, sizeof(double) * m1 * sk, cudaMemcpyDeviceToDevice, s);
    r[k] = sk;
  }
  // left-to-right truncation with threshold delta / sqrt(d-1) ||T||
  double thr = 0.0;
  for (int64_t k = 0; (phases & 2) && k < d - 1 && e == cudaSuccess; ++k) {
    const long long m = r[k] * n[k], rk1 = r[k + 1];
    g_stage = TT_ST_IL_S2;
    e = launch_gemm(false, false, gp(W[k], rk1, W[k], rk1, G, rk1, rk1, m, tt::map_plain(rk1),
                                     tt::map_plain(1)), s);
    if (e == cudaSuccess) e = eig((int)rk1);
    if (e != cudaSuccess) break;
    if (k == 0) {
      double nrm2 = 0.0;
      for (long long i = 0; i < rk1; ++i) nrm2 += std::max(hl[i], 0.0);
      thr = delta / std::sqrt((double)std::max<int64_t>(d - 1, 1)) * std::sqrt(nrm2);
    }
    // smallest rank whose discarded tail has Frobenius norm <= thr; drop numerical zeros
    int nz = 0;
    for (long long i = 0; i < rk1; ++i)
      if (hl[i] > zero_rel * hl[0] && hl[i] > 0.0) ++nz;
    if (nz == 0) nz = 1;
    int sk = nz;
    double tail = 0.0;
    for (int i = nz - 1; i >= 1; --i) {
      tail += std::max(hl[i], 0.0);
      if (std::sqrt(tail) <= thr) sk = i; else break;
    }
    if (max_rank > 0 && sk > max_rank) sk = (int)max_rank;
    for (int i = 0; i < sk; ++i) hf[i] = 1.0 / std::sqrt(std::max(hl[i], 1e-300));
    if ((e = scaled((int)rk1, sk, hf)) != cudaSuccess) break;
    // U (m x sk) = W_k . (V S^-1)
    e = launch_gemm(true, false, gp(W[k], rk1, Bm, sk, Tmp, m, sk, rk1, tt::map_plain(sk),
                                    tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k], Tmp, sizeof(double) * m * sk, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) break;
    for (int i = 0; i < sk; ++i) hf[i] = std::sqrt(std::max(hl[i], 0.0));
    if ((e = scaled((int)rk1, sk, hf)) != cudaSuccess) break;
    // W_{k+1} (sk x q) = (V S)^T . W_{k+1} (rk1 x q)
    const long long q = n[k + 1] * r[k + 2];
    e = launch_gemm(false, false, gp(Bm, sk, W[k + 1], q, Tmp, sk, q, rk1, tt::map_plain(q),
                                     tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k + 1], Tmp, sizeof(double) * sk * q, cudaMemcpyDeviceToDevice, s);
    r[k + 1] = sk;
  }
  for (int64_t k = 0; k < d && e == cudaSuccess; ++k)
    e = cudaMemcpyAsync(cores_out[k], W[k], sizeof(double) * r[k] * n[k] * r[k + 1],
                        cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, who);
  for (int64_t k = 0; k <= d; ++k) r_out[k] = r[k];
  return TT_OK;
}

tt_status tt_round(int64_t d, const int64_t* n, const int64_t* r_in,
                   const double* const* cores_in, double delta, int64_t max_rank, int64_t* r_out,
                   double* const* cores_out, void* workspace, size_t workspace_bytes,
                   void* stream) {
  CallScope scope;
  return round_impl(d, n, r_in, cores_in, delta, max_rank, r_out, cores_out, workspace,
                    workspace_bytes, stream, 3, "tt_round");
}

size_t tt_orthonormalise_workspace_size(int64_t d, const int64_t* n, const int64_t* r) {
  return tt_round_workspace_size(d, n, r);
}

tt_status tt_orthonormalise(int64_t d, const int64_t* n, const int64_t* r_in,
                            const double* const* cores_in, int direction, int64_t* r_out,
                            double* const* cores_out, void* workspace, size_t workspace_bytes,
                            void* stream) {
  CallScope scope;
  if (direction != TT_SWEEP_LEFT && direction != TT_SWEEP_RIGHT)
    return fail(TT_ERR_INVALID_ARGUMENT, "direction must be TT_SWEEP_LEFT or TT_SWEEP_RIGHT");
  return round_impl(d, n, r_in, cores_in, 0.0, 0, r_out, cores_out, workspace, workspace_bytes,
                    stream, direction == TT_SWEEP_LEFT ? 2 : 1, "tt_orthonormalise");
}

// ---- block-index move ---------------------------------
// Thin SVD of an m x q matrix M through the Gram matrix of its smaller side: the leading s
// left singular vectors Us (m x s) and right singular vectors Vs (q x s), truncated at
// ||sigma_{s:}|| <= delta ||sigma|| (numerical zeros lambda <= 1e-14 lambda_max dropped) and
// s <= max_rank.  One host synchronisation (the truncation is data dependent).
struct SvdBufs {
  double *G, *E, *lam, *esc, *f, *Us, *Vs;
};
static long long svd_ws_elems(long long m, long long q) {
  const long long k = std::min(m, q), big = std::max(m, q);
  // G, E (<= k^2 + big k), lam, eigen scratch, f, Us + Vs (<= 2 big k), alignment slack
  return 2 * k * k + 3 * big * k + 3 * k + 128 + sym_eigen_scratch(k) + 12 * 32;
}
static cudaError_t svd_gram(const double* M, long long m, long long q, double delta,
                            long long max_rank, SvdBufs& b, int& s_out, cudaStream_t s) {
  const bool left = m <= q;   // Gram of the smaller side
  const long long k = left ? m : q;
  cudaError_t e;
  g_stage = TT_ST_IL_S1;
  if (left)   // G = M M^T (m x m)
    e = launch_gemm(true, true, gp(M, q, M, q, b.G, m, m, q, tt::map_plain(m), tt::map_plain(1)), s);
  else        // G = M^T M (q x q)
    e = launch_gemm(false, false, gp(M, q, M, q, b.G, q, q, m, tt::map_plain(q), tt::map_plain(1)), s);
  if (e != cudaSuccess) return e;
  if ((e = launch_sym_eigen(b.G, b.E, b.lam, (int)k, b.esc, s)) != cudaSuccess) return e;
  std::vector<double> hl(k);
  if ((e = cudaMemcpyAsync(hl.data(), b.lam, sizeof(double) * k, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  double tot = 0.0;
  int nz = 0;
  for (long long i = 0; i < k; ++i) {
    tot += std::max(hl[i], 0.0);
    if (hl[i] > 1e-14 * hl[0] && hl[i] > 0.0) ++nz;
  }
  if (nz == 0) nz = 1;
  const double thr = delta * std::sqrt(tot);
  int sk = nz;
  double tail = 0.0;
  for (int i = nz - 1; i >= 1; --i) {
    tail += std::max(hl[i], 0.0);
    if (std::sqrt(tail) <= thr) sk = i; else break;
  }
  if (max_rank > 0 && sk > max_rank) sk = (int)max_rank;
  s_out = sk;
  // E[:, :sk] (k x sk) -> the singular vectors of the Gram side; the other side by a GEMM
  std::vector<double> hf(sk);
  for (int i = 0; i < sk; ++i) hf[i] = 1.0;
  if ((e = cudaMemcpyAsync(b.f, hf.data(), sizeof(double) * sk, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  double* side = left ? b.Us : b.Vs;
  scale_cols_kernel<<<(unsigned)((k * sk + 255) / 256), 256, 0, s>>>(b.E, b.f, side, (int)k, sk);
  ++g_launches;
  for (int i = 0; i < sk; ++i) hf[i] = 1.0 / std::sqrt(std::max(hl[i], 1e-300));
  double* fin = b.f + 32 * ((sk + 31) / 32);
  if ((e = cudaMemcpyAsync(fin, hf.data(), sizeof(double) * sk, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  // the other side: Vs = M^T Us Sigma^-1  or  Us = M Vs Sigma^-1 (scale columns afterwards)
  double* other = left ? b.Vs : b.Us;
  if (left)   // Vs (q x sk) = M^T (q x m) . Us (m x sk)
    e = launch_gemm(false, false, gp(M, q, b.Us, sk, b.E, q, sk, m, tt::map_plain(sk), tt::map_plain(1)), s);
  else        // Us (m x sk) = M (m x q) . Vs (q x sk)
    e = launch_gemm(true, false, gp(M, q, b.Vs, sk, b.E, m, sk, q, tt::map_plain(sk), tt::map_plain(1)), s);
  if (e != cudaSuccess) return e;
  const long long ob = left ? q : m;
  scale_cols_ld_kernel<<<(unsigned)std::min<long long>(4096, (ob * sk + 255) / 256), 256, 0, s>>>(
      b.E, sk, fin, other, ob, sk);
  ++g_launches;
  return cudaGetLastError();
}

static bool block_move_ws(long long m, long long q, long long extra, long long& total) {
  total = svd_ws_elems(m, q) + m * q + extra;
  return m > 0 && q > 0;
}

size_t tt_block_move_workspace_size(int64_t r0, int64_t n0, int64_t l, int64_t r1, int64_t n1,
                                    int64_t r2) {
  if (r0 <= 0 || n0 <= 0 || l <= 0 || r1 <= 0 || n1 <= 0 || r2 <= 0) return 0;
  bool ok = true;
  // right move: M = (r0 n0) x (l r1);  left move: M = (r0 l) x (n0 r1) with (r0,n0,l,r1) the
  // core carrying the block index -- size for the larger of the two views
  const long long m1 = prod({r0, n0}, ok), q1 = prod({l, r1}, ok);
  const long long m2 = prod({r1, l}, ok), q2 = prod({n1, r2}, ok);
  const long long out = prod({std::max(m1, q1), std::max(n1 * r2, r0 * n0), l}, ok);
  if (!ok) return 0;
  long long a, b;
  block_move_ws(m1, q1, out, a);
  block_move_ws(m2, q2, out, b);
  return ws_bytes({std::max(a, b)});
}

tt_status tt_block_move_right(int64_t r0, int64_t n0, int64_t l, int64_t r1, int64_t n1,
                              int64_t r2, double delta, int64_t max_rank, const double* Wk_hat,
                              const double* Wk1, double* Wk_out, double* Wk1_hat_out,
                              int64_t* s_out, void* workspace, size_t workspace_bytes,
                              void* stream) {
  CallScope scope;
  if (r0 <= 0 || n0 <= 0 || l <= 0 || r1 <= 0 || n1 <= 0 || r2 <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  if (!(delta >= 0.0) || max_rank < 0) return fail(TT_ERR_INVALID_ARGUMENT, "need delta >= 0, max_rank >= 0");
  if (!Wk_hat || !Wk1 || !Wk_out || !Wk1_hat_out || !s_out) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  for (const void* o : {(const void*)Wk_out, (const void*)Wk1_hat_out})
    if (same(o, Wk_hat) || same(o, Wk1)) return fail(TT_ERR_ALIASING, "an output aliases an input");
  if (same(Wk_out, Wk1_hat_out)) return fail(TT_ERR_ALIASING, "two outputs alias");
  const long long m = r0 * n0, q = l * r1;
  if (std::min(m, q) > 2048)
    return fail(TT_ERR_INVALID_ARGUMENT, "min(r0 n0, l r1) above 2048 is not supported");
  const size_t need = tt_block_move_workspace_size(r0, n0, l, r1, n1, r2);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long k = std::min(m, q), big = std::max(m, q);
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  SvdBufs b;
  b.G = c.take(k * k);
  b.E = c.take(std::max(k * k, big * k));
  b.lam = c.take(k);
  b.esc = c.take(sym_eigen_scratch(k));
  b.f = c.take(2 * (k + 64));
  b.Us = c.take(m * k);
  b.Vs = c.take(q * k);
  double* C = c.take(k * q);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  int sk = 0;
  cudaError_t e = svd_gram(Wk_hat, m, q, delta, max_rank, b, sk, s);
  // Wk_out = Us (m x sk);  C (sk x q) = Us^T M
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(Wk_out, b.Us, sizeof(double) * m * sk, cudaMemcpyDeviceToDevice, s);
  g_stage = TT_ST_IL_S2;
  if (e == cudaSuccess)
    e = launch_gemm(false, false, gp(b.Us, sk, Wk_hat, q, C, sk, q, m, tt::map_plain(q),
                                     tt::map_plain(1)), s);
  // Wk1_hat_out[s, j, l, c] = sum_b C[s, l, b] Wk1[b, j, c]: rows (s, l), cols (j, c)
  if (e == cudaSuccess)
    e = launch_gemm(true, false, gp(C, r1, Wk1, n1 * r2, Wk1_hat_out, sk * l, n1 * r2, r1,
                                    tt::map2(l, r2, n1 * l * r2), tt::map2(r2, 1, l * r2)), s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "tt_block_move_right");
  *s_out = sk;
  return TT_OK;
}

tt_status tt_block_move_left(int64_t r0, int64_t n0, int64_t r1, int64_t n1, int64_t l,
                             int64_t r2, double delta, int64_t max_rank, const double* Wkm1,
                             const double* Wk_hat, double* Wkm1_hat_out, double* Wk_out,
                             int64_t* s_out, void* workspace, size_t workspace_bytes,
                             void* stream) {
  CallScope scope;
  if (r0 <= 0 || n0 <= 0 || l <= 0 || r1 <= 0 || n1 <= 0 || r2 <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  if (!(delta >= 0.0) || max_rank < 0) return fail(TT_ERR_INVALID_ARGUMENT, "need delta >= 0, max_rank >= 0");
  if (!Wkm1 || !Wk_hat || !Wk_out || !Wkm1_hat_out || !s_out) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  for (const void* o : {(const void*)Wk_out, (const void*)Wkm1_hat_out})
    if (same(o, Wk_hat) || same(o, Wkm1)) return fail(TT_ERR_ALIASING, "an output aliases an input");
  if (same(Wk_out, Wkm1_hat_out)) return fail(TT_ERR_ALIASING, "two outputs alias");
  const long long m = r1 * l, q = n1 * r2;
  if (std::min(m, q) > 2048)
    return fail(TT_ERR_INVALID_ARGUMENT, "min(r1 l, n1 r2) above 2048 is not supported");
  const size_t need = tt_block_move_workspace_size(r0, n0, l, r1, n1, r2);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long k = std::min(m, q), big = std::max(m, q);
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  SvdBufs b;
  b.G = c.take(k * k);
  b.E = c.take(std::max(k * k, big * k));
  b.lam = c.take(k);
  b.esc = c.take(sym_eigen_scratch(k));
  b.f = c.take(2 * (k + 64));
  b.Us = c.take(m * k);
  b.Vs = c.take(q * k);
  double* Mp = c.take(m * q);
  double* C = c.take(m * k);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  long long blocks = std::min<long long>(4096, (m * q + 255) / 256);
  // M (r1 l) x (n1 r2) from Wk_hat (r1, n1, l, r2)
  swap_mid_kernel<<<(unsigned)blocks, 256, 0, s>>>(Wk_hat, Mp, r1, n1, l, r2);
  ++g_launches;
  int sk = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = svd_gram(Mp, m, q, delta, max_rank, b, sk, s);
  // Wk_out (sk x q) = Vs^T;  C (m x sk) = M Vs = Us Sigma
  if (e == cudaSuccess) {
    transpose2d_kernel<<<(unsigned)std::min<long long>(4096, (q * sk + 255) / 256), 256, 0, s>>>(
        b.Vs, Wk_out, q, sk);
    ++g_launches;
    e = cudaGetLastError();
  }
  g_stage = TT_ST_IL_S2;
  if (e == cudaSuccess)
    e = launch_gemm(true, false, gp(Mp, q, b.Vs, sk, C, m, sk, q, tt::map_plain(sk),
                                    tt::map_plain(1)), s);
  // Wkm1_hat_out (r0 n0) x (l sk) = Wkm1 (r0 n0 x r1) . C (r1 x (l sk))
  if (e == cudaSuccess)
    e = launch_gemm(true, false, gp(Wkm1, r1, C, l * sk, Wkm1_hat_out, r0 * n0, l * sk, r1,
                                    tt::map_plain(l * sk), tt::map_plain(1)), s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "tt_block_move_left");
  *s_out = sk;
  return TT_OK;
}

// ---- AMEn enrichment ("enrichment of the TT cores by TT cores of the
// approximate residual, as in the AMEn algorithm") -----------------------------------------
// x_k (rl, n, rx) and the residual core z_k (rl, n, rz) are concatenated along the right bond,
// x_{k+1} (rx, n1, r2) is padded with rz zero rows (the represented tensor is unchanged), and
// the enlarged core is re-orthonormalised by one truncated SVD step (tt_block_move_right with
// l = 1): x_k' (rl, n, s) left-orthonormal, x_{k+1}' (s, n1, r2).
__global__ void enrich_concat_kernel(const double* __restrict__ x, const double* __restrict__ z,
                                     const double* __restrict__ x1, double* __restrict__ cat,
                                     double* __restrict__ cat1, long long rows, long long rx,
                                     long long rz, long long q1) {
  const long long r = rx + rz;
  const long long n0 = rows * r, n1 = r * q1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n0 + n1;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < n0) {
      const long long i = e / r, c = e - i * r;
      cat[e] = c < rx ? x[i * rx + c] : z[i * rz + (c - rx)];
    } else {
      const long long f = e - n0, row = f / q1;
      cat1[f] = row < rx ? x1[f] : 0.0;
    }
  }
}

size_t tt_enrich_right_workspace_size(int64_t rl, int64_t n, int64_t rx, int64_t rz, int64_t n1,
                                      int64_t r2) {
  if (rl <= 0 || n <= 0 || rx <= 0 || rz <= 0 || n1 <= 0 || r2 <= 0) return 0;
  bool ok = true;
  const long long cat = prod({rl, n, rx + rz}, ok), cat1 = prod({rx + rz, n1, r2}, ok);
  if (!ok) return 0;
  const size_t mv = tt_block_move_workspace_size(rl, n, 1, rx + rz, n1, r2);
  if (mv == 0) return 0;
  return mv + ws_bytes({cat, cat1});
}

tt_status tt_enrich_right(int64_t rl, int64_t n, int64_t rx, int64_t rz, int64_t n1, int64_t r2,
                          double delta, int64_t max_rank, const double* x_k, const double* z_k,
                          const double* x_k1, double* x_k_out, double* x_k1_out, int64_t* s_out,
                          void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  if (rl <= 0 || n <= 0 || rx <= 0 || rz <= 0 || n1 <= 0 || r2 <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  if (!x_k || !z_k || !x_k1 || !x_k_out || !x_k1_out || !s_out)
    return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  for (const void* o : {(const void*)x_k_out, (const void*)x_k1_out})
    if (same(o, x_k) || same(o, z_k) || same(o, x_k1))
      return fail(TT_ERR_ALIASING, "an output aliases an input");
  const size_t need = tt_enrich_right_workspace_size(rl, n, rx, rz, n1, r2);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  const size_t mv = tt_block_move_workspace_size(rl, n, 1, rx + rz, n1, r2);
  char* base = static_cast<char*>(workspace);
  Carver c{base + mv, workspace_bytes - mv};
  const long long r = rx + rz;
  double* cat = c.take(rl * n * r);
  double* cat1 = c.take(r * n1 * r2);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long tot = rl * n * r + r * n1 * r2;
  enrich_concat_kernel<<<(unsigned)std::min<long long>(4096, (tot + 255) / 256), 256, 0, s>>>(
      x_k, z_k, x_k1, cat, cat1, rl * n, rx, rz, n1 * r2);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "tt_enrich_right");
  const int64_t launches = g_launches;
  tt_status st = tt_block_move_right(rl, n, 1, r, n1, r2, delta, max_rank, cat, cat1, x_k_out,
                                     x_k1_out, s_out, base, mv, stream);
  g_launches += launches;
  g_launches_last = g_launches;
  return st;
}

// ---- projected KKT block system action -----------------------------
static bool block_ws(int64_t rl, int64_t n, int64_t rr, int64_t nops, const int64_t* Rl,
                     const int64_t* Rr, long long& t1, long long& t2, long long& ah, long long& pe,
                     long long& vec) {
  t1 = t2 = ah = pe = 0;
  bool ok = true;
  for (int64_t o = 0; o < nops; ++o) {
    Dims d{rl, n, rr, Rl[o], Rr[o]};
    long long a, b, c, e;
    if (!dims_valid(d) || !matvec_ws_elems(d, 1, a, b, c, e)) return false;
    t1 = std::max(t1, a);
    t2 = std::max(t2, b);
    ah = std::max(ah, c);
    pe = std::max(pe, e);
  }
  vec = prod({rl, n, rr}, ok);
  return ok;
}

size_t tt_block_local_matvec_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t nops,
                                            const int64_t* Rl, const int64_t* Rr) {
  if (nops <= 0 || !Rl || !Rr) return 0;
  long long t1, t2, ah, pe, vec;
  if (!block_ws(rl, n, rr, nops, Rl, Rr, t1, t2, ah, pe, vec)) return 0;
  return ws_bytes({t1, t2, ah, pe, vec, vec, vec});
}

tt_status tt_block_local_matvec(int64_t rl, int64_t n, int64_t rr, int64_t nblocks, int64_t nops,
                                const int64_t* Rl, const int64_t* Rr, const double* const* phiL,
                                const double* const* A, const double* const* phiR,
                                int64_t nterms, const tt_block_term* terms, const double* X,
                                double* Y, void* workspace, size_t workspace_bytes,
                                void* stream) {
  CallScope scope;
  if (rl <= 0 || n <= 0 || rr <= 0 || nblocks <= 0 || nops <= 0 || nterms < 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  if (!Rl || !Rr || !phiL || !A || !phiR || !X || !Y || (nterms > 0 && !terms))
    return fail(TT_ERR_NULL_POINTER, "NULL argument");
  for (int64_t o = 0; o < nops; ++o) {
    if (!phiL[o] || !A[o] || !phiR[o]) return fail(TT_ERR_NULL_POINTER, "NULL operator entry");
    tt_status st = check_dims(Dims{rl, n, rr, Rl[o], Rr[o]});
    if (st != TT_OK) return st;
    if (same(Y, phiL[o]) || same(Y, A[o]) || same(Y, phiR[o]))
      return fail(TT_ERR_ALIASING, "output Y aliases an operator");
  }
  if (same(Y, X)) return fail(TT_ERR_ALIASING, "output Y aliases X");
  for (int64_t t = 0; t < nterms; ++t) {
    const tt_block_term& tm = terms[t];
    if (tm.row < 0 || tm.row >= nblocks || tm.col < 0 || tm.col >= nblocks || tm.op < 0 ||
        tm.op >= nops || tm.op2 < -1 || tm.op2 >= nops)
      return fail(TT_ERR_INVALID_ARGUMENT, "term " + std::to_string(t) + " out of range");
  }
  long long t1, t2, ah, pe, vec;
  if (!block_ws(rl, n, rr, nops, Rl, Rr, t1, t2, ah, pe, vec))
    return fail(TT_ERR_OVERFLOW, "workspace overflow");
  const size_t need = ws_bytes({t1, t2, ah, pe, vec, vec, vec});
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  double* T1 = c.take(t1);
  double* T2 = c.take(t2);
  double* Ah = c.take(ah);
  double* Pp = c.take(pe);
  double* G = c.take(vec);
  double* G2 = c.take(vec);
  double* Tv = c.take(vec);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long rows = rl * n;
  long long blocks = (vec + 255) / 256;
  if (blocks > 4L * num_sms()) blocks = 4L * num_sms();
  cudaError_t e = cudaMemsetAsync(Y, 0, sizeof(double) * rows * nblocks * rr, s);
  for (int64_t t = 0; t < nterms && e == cudaSuccess; ++t) {
    const tt_block_term& tm = terms[t];
    gather_col_kernel<<<(unsigned)blocks, 256, 0, s>>>(X, G, rows, (int)nblocks, (int)rr,
                                                       (int)tm.col);
    ++g_launches;
    const double* in = G;
    if (tm.op2 >= 0) {
      const Dims d2{rl, n, rr, Rl[tm.op2], Rr[tm.op2]};
      e = enqueue_matvec(d2, 1, phiL[tm.op2], A[tm.op2], phiR[tm.op2], G, G2, T1, T2, Ah, Pp, pe, s);
      in = G2;
    }
    if (e != cudaSuccess) break;
    const Dims d1{rl, n, rr, Rl[tm.op], Rr[tm.op]};
    e = enqueue_matvec(d1, 1, phiL[tm.op], A[tm.op], phiR[tm.op], in, Tv, T1, T2, Ah, Pp, pe, s);
    if (e != cudaSuccess) break;
    scatter_add_col_kernel<<<(unsigned)blocks, 256, 0, s>>>(Tv, Y, rows, (int)nblocks, (int)rr,
                                                            (int)tm.row, tm.coeff);
    ++g_launches;
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return cuda_fail(e, "tt_block_local_matvec");
  return TT_OK;
}

// ---- two-site local matvec ------------------------------------------
size_t tt_local_matvec_two_site_workspace_size(int64_t rl, int64_t n1, int64_t n2, int64_t rr,
                                               int64_t Rl, int64_t Rm, int64_t Rr, int64_t nvec) {
  if (n1 <= 0 || n2 <= 0 || Rm <= 0 || nvec <= 0) return 0;
  Dims d{rl, n1 * n2, rr, Rl, Rr};
  long long t1, t2, ah, pe;
  if (!dims_valid(d) || !matvec_ws_elems(d, nvec, t1, t2, ah, pe)) return 0;
  return ws_bytes({t1, t2, ah, pe, d.al * d.n * d.n * d.be});
}

tt_status tt_local_matvec_two_site(int64_t rl, int64_t n1, int64_t n2, int64_t rr, int64_t Rl,
                                   int64_t Rm, int64_t Rr, int64_t nvec, const double* phiL,
                                   const double* A1, const double* A2, const double* phiR,
                                   const double* W, double* Y, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  CallScope scope;
  if (n1 <= 0 || n2 <= 0 || Rm <= 0 || nvec <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  bool ok = true;
  const long long N = prod({n1, n2}, ok);
  if (!ok) return fail(TT_ERR_OVERFLOW, "extent product overflows");
  Dims d{rl, N, rr, Rl, Rr};
  tt_status st = check_dims(d);
  if (st != TT_OK) return st;
  if (!phiL || !A1 || !A2 || !phiR || !W || !Y) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  if (same(Y, phiL) || same(Y, A1) || same(Y, A2) || same(Y, phiR) || same(Y, W))
    return fail(TT_ERR_ALIASING, "output Y aliases an input");
  long long t1, t2, ah, pe;
  if (!matvec_ws_elems(d, nvec, t1, t2, ah, pe)) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  const long long a12 = d.al * d.n * d.n * d.be;
  const size_t need = ws_bytes({t1, t2, ah, pe, a12});
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  double* T1 = c.take(t1);
  double* T2 = c.take(t2);
  double* Ah = c.take(ah);
  double* Pp = c.take(pe);
  double* A12 = c.take(a12);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  long long blocks = (a12 + 255) / 256;
  if (blocks > 2048) blocks = 2048;
  g_stage = TT_ST_PERM;
  const long long tr = trace_begin(0, a12, 0, 0, s);
  merge_cores_kernel<<<(unsigned)blocks, 256, 0, s>>>(A1, A2, A12, Rl, n1, n2, Rm, Rr);
  trace_end(tr, s);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = enqueue_matvec(d, nvec, phiL, A12, phiR, W, Y, T1, T2, Ah, Pp, pe, s);
  if (e != cudaSuccess) return cuda_fail(e, "tt_local_matvec_two_site");
  return TT_OK;
}

// ---- local GMRES --------------------------------------------------
size_t tt_local_gmres_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                                     int64_t nvec, int64_t m, int64_t k_aug) {
  Dims d{rl, n, rr, Rl, Rr};
  long long t1, t2, ah, pe;
  GmresWs gw;
  if (!dims_valid(d) || nvec <= 0 || nvec > 64 || m <= 0 || k_aug < 0 ||
      !matvec_ws_elems(d, nvec, t1, t2, ah, pe) || !gmres_ws_elems(d, nvec, m + k_aug, gw, k_aug))
    return 0;
  return ws_bytes({t1, t2, ah, pe, gw.basis, gw.w, gw.part, gw.small});
}

tt_status tt_local_gmres(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr, int64_t nvec,
                         int64_t m, int64_t k_aug, int64_t cycles, double tol, const double* phiL,
                         const double* A, const double* phiR, const double* F, double* X,
                         double* rel_res, int64_t* iters, void* workspace,
                         size_t workspace_bytes, void* stream) {
  CallScope scope;
  Dims d{rl, n, rr, Rl, Rr};
  tt_status st = check_dims(d);
  if (st != TT_OK) return st;
  if (nvec <= 0 || nvec > 64) return fail(TT_ERR_INVALID_ARGUMENT, "nvec must be in [1, 64]");
  if (m <= 0 || m > 512 || k_aug < 0 || k_aug > 64 || cycles < 0 || !(tol >= 0.0))
    return fail(TT_ERR_INVALID_ARGUMENT,
                "need 0 < m <= 512, 0 <= k_aug <= 64, cycles >= 0, tol >= 0");
  if (!phiL || !A || !phiR || !F || !X || !rel_res || !iters)
    return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  for (const void* o : {(const void*)X, (const void*)rel_res, (const void*)iters})
    for (const void* i : {(const void*)phiL, (const void*)A, (const void*)phiR, (const void*)F})
      if (o == i) return fail(TT_ERR_ALIASING, "an output aliases an input");
  if ((const void*)X == (const void*)rel_res || (const void*)X == (const void*)iters ||
      (const void*)rel_res == (const void*)iters)
    return fail(TT_ERR_ALIASING, "two outputs alias");
  const size_t need = tt_local_gmres_workspace_size(rl, n, rr, Rl, Rr, nvec, m, k_aug);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaError_t e = enqueue_gmres(d, nvec, m, k_aug, cycles, tol, phiL, A, phiR, F, X, rel_res,
                                reinterpret_cast<long long*>(iters), workspace, workspace_bytes,
                                static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_local_gmres");
  return TT_OK;
}

// ---- Petrov-Galerkin local operations (bra != ket) and AMEn enrichment ---------------------
static tt_status check_pg(const DimsPG& d) {
  if (!dims_pg_valid(d)) return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  long long t1, t2, ah, pe;
  if (!pg_ws_elems(d, 1, t1, t2, ah, pe)) return fail(TT_ERR_OVERFLOW, "extent product overflows");
  return TT_OK;
}

size_t tt_pg_workspace_size(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                            int64_t Rl, int64_t Rr, int64_t nvec) {
  DimsPG d{rl_bra, rl, n, rr_bra, rr, Rl, Rr};
  long long t1, t2, ah, pe;
  if (!dims_pg_valid(d) || nvec <= 0 || !pg_ws_elems(d, nvec, t1, t2, ah, pe)) return 0;
  return ws_bytes({t1, t2, ah, pe});
}

#define TT_PG_CARVE()                                                                      \
  long long t1, t2, ah, pe;                                                                \
  if (!pg_ws_elems(d, K, t1, t2, ah, pe)) return fail(TT_ERR_OVERFLOW, "workspace overflow"); \
  const size_t need = ws_bytes({t1, t2, ah, pe});                                          \
  if (!workspace || workspace_bytes < need)                                                \
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes"); \
  Carver c{static_cast<char*>(workspace), workspace_bytes};                                \
  double* T1 = c.take(t1);                                                                 \
  double* T2 = c.take(t2);                                                                 \
  double* Ah = c.take(ah);                                                                 \
  double* Pp = c.take(pe);                                                                 \
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");

tt_status tt_local_matvec_pg(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                             int64_t Rl, int64_t Rr, int64_t nvec, const double* phiL,
                             const double* A, const double* phiR, const double* X, double* Y,
                             void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  DimsPG d{rl_bra, rl, n, rr_bra, rr, Rl, Rr};
  tt_status st = check_pg(d);
  if (st != TT_OK) return st;
  if (nvec <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "nvec must be positive");
  if (!phiL || !A || !phiR || !X || !Y) return fail(TT_ERR_NULL_POINTER, "NULL tensor pointer");
  if (same(Y, phiL) || same(Y, A) || same(Y, phiR) || same(Y, X))
    return fail(TT_ERR_ALIASING, "output Y aliases an input");
  const long long K = nvec;
  TT_PG_CARVE();
  cudaError_t e = enqueue_matvec_pg(d, K, phiL, A, phiR, X, Y, T1, T2, Ah, Pp, pe,
                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_local_matvec_pg");
  return TT_OK;
}

tt_status tt_interface_left_pg(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                               int64_t Rl, int64_t Rr, const double* phiL_prev, const double* A,
                               const double* x_bra, const double* x_ket, double* phiL_next,
                               void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  DimsPG d{rl_bra, rl, n, rr_bra, rr, Rl, Rr};
  tt_status st = check_pg(d);
  if (st != TT_OK) return st;
  if (!phiL_prev || !A || !x_bra || !x_ket || !phiL_next)
    return fail(TT_ERR_NULL_POINTER, "NULL tensor pointer");
  if (same(phiL_next, phiL_prev) || same(phiL_next, A) || same(phiL_next, x_bra) ||
      same(phiL_next, x_ket))
    return fail(TT_ERR_ALIASING, "output aliases an input");
  const long long K = 1;
  TT_PG_CARVE();
  cudaError_t e = enqueue_left_pg(d, phiL_prev, A, x_bra, x_ket, phiL_next, T1, T2, Ah, Pp, pe,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_interface_left_pg");
  return TT_OK;
}

tt_status tt_interface_right_pg(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                                int64_t Rl, int64_t Rr, const double* phiR_next, const double* A,
                                const double* x_bra, const double* x_ket, double* phiR_prev,
                                void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  DimsPG d{rl_bra, rl, n, rr_bra, rr, Rl, Rr};
  tt_status st = check_pg(d);
  if (st != TT_OK) return st;
  if (!phiR_next || !A || !x_bra || !x_ket || !phiR_prev)
    return fail(TT_ERR_NULL_POINTER, "NULL tensor pointer");
  if (same(phiR_prev, phiR_next) || same(phiR_prev, A) || same(phiR_prev, x_bra) ||
      same(phiR_prev, x_ket))
    return fail(TT_ERR_ALIASING, "output aliases an input");
  const long long K = 1;
  TT_PG_CARVE();
  cudaError_t e = enqueue_right_pg(d, phiR_next, A, x_bra, x_ket, phiR_prev, T1, T2, Ah, Pp, pe,
                                   static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_interface_right_pg");
  return TT_OK;
}
#undef TT_PG_CARVE

// ---- LOBPCG ---------------------------------------------------------
size_t tt_local_lobpcg_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t RlA, int64_t RrA,
                                      int64_t RlB, int64_t RrB, int64_t nb) {
  Dims dA{rl, n, rr, RlA, RrA};
  const bool has_B = RlB > 0 || RrB > 0;
  Dims dB{rl, n, rr, has_B ? RlB : 1, has_B ? RrB : 1};
  if (!dims_valid(dA) || !dims_valid(dB) || nb <= 0 || nb > kLobMaxNb) return 0;
  long long t1a, t2a, aha, pea, t1b = 0, t2b = 0, ahb = 0, peb = 0;
  if (!matvec_ws_elems(dA, nb, t1a, t2a, aha, pea)) return 0;
  if (has_B && !matvec_ws_elems(dB, nb, t1b, t2b, ahb, peb)) return 0;
  LobWs lw;
  if (!lob_ws_elems(dA, nb, lw)) return 0;
  return ws_bytes({std::max(t1a, t1b), std::max(t2a, t2b), std::max(pea, peb), aha, ahb, lw.blocks,
                   lw.part, lw.gpart, lw.G, lw.Y, lw.small});
}

tt_status tt_local_lobpcg(int64_t rl, int64_t n, int64_t rr, int64_t RlA, int64_t RrA,
                          int64_t RlB, int64_t RrB, int64_t nb, int64_t maxiter,
                          int64_t refresh, double tol, const double* phiLA, const double* AA, const double* phiRA,
                          const double* phiLB, const double* AB, const double* phiRB, double* X,
                          double* lam, double* res, int64_t* iters, double* step,
                          void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  const bool has_B = phiLB || AB || phiRB;
  if (has_B && (!phiLB || !AB || !phiRB))
    return fail(TT_ERR_NULL_POINTER, "operator B needs all of phiL_B, A_B, phiR_B (or none: B = I)");
  Dims dA{rl, n, rr, RlA, RrA};
  tt_status st = check_dims(dA);
  if (st != TT_OK) return st;
  Dims dB{rl, n, rr, has_B ? RlB : 1, has_B ? RrB : 1};
  if ((st = check_dims(dB)) != TT_OK) return st;
  if (nb <= 0 || nb > kLobMaxNb) return fail(TT_ERR_INVALID_ARGUMENT, "nb must be in [1, 32]");
  if (nb > rl * n * rr) return fail(TT_ERR_INVALID_ARGUMENT, "nb exceeds the local dimension");
  if (maxiter < 0 || refresh < 0 || !(tol >= 0.0))
    return fail(TT_ERR_INVALID_ARGUMENT, "need maxiter >= 0, refresh >= 0, tol >= 0");
  if (!phiLA || !AA || !phiRA || !X || !lam || !res || !iters)
    return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  const void* outs[] = {X, lam, res, iters, step};
  const void* ins[] = {phiLA, AA, phiRA, phiLB, AB, phiRB};
  for (const void* o : outs) {
    for (const void* i : ins)
      if (same(o, i)) return fail(TT_ERR_ALIASING, "an output aliases an input");
    for (const void* o2 : outs)
      if (o != o2 && same(o, o2)) return fail(TT_ERR_ALIASING, "two outputs alias");
  }
  const size_t need = tt_local_lobpcg_workspace_size(rl, n, rr, RlA, RrA, has_B ? RlB : 0,
                                                     has_B ? RrB : 0, nb);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaError_t e = enqueue_lobpcg(dA, dB, has_B, nb, maxiter, refresh, tol, phiLA, AA, phiRA, phiLB, AB,
                                 phiRB, X, lam, res, reinterpret_cast<long long*>(iters), step,
                                 workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_local_lobpcg");
  return TT_OK;
}

tt_status tt_merge_operator_cores(int64_t Rl, int64_t n1, int64_t n2, int64_t Rm, int64_t Rr,
                                  const double* A1, const double* A2, double* A12, void* stream) {
  CallScope scope;
  if (Rl <= 0 || n1 <= 0 || n2 <= 0 || Rm <= 0 || Rr <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  bool ok = true;
  const long long total = prod({Rl, n1, n2, n1, n2, Rr}, ok);
  prod({Rl, n1, n1, Rm}, ok);
  prod({Rm, n2, n2, Rr}, ok);
  if (!ok) return fail(TT_ERR_OVERFLOW, "extent product overflows");
  if (!A1 || !A2 || !A12) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  if (same(A12, A1) || same(A12, A2)) return fail(TT_ERR_ALIASING, "output A12 aliases an input");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  long long blocks = (total + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  merge_cores_kernel<<<(unsigned)blocks, 256, 0, s>>>(A1, A2, A12, Rl, n1, n2, Rm, Rr);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "tt_merge_operator_cores");
  return TT_OK;
}

// ---- tracing / probe ----------------------------------------------------------------------
tt_status tt_trace_enable(int64_t capacity) {
  g_msg.clear();
  if (capacity <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "capacity must be positive");
  tt_trace_disable();
  g_trace_pool.resize(size_t(2 * capacity));
  for (auto& ev : g_trace_pool) {
    cudaError_t e = cudaEventCreate(&ev);
    if (e != cudaSuccess) {
      g_trace_pool.clear();
      return cuda_fail(e, "tt_trace_enable");
    }
  }
  g_trace.clear();
  g_trace.reserve(size_t(capacity));
  g_trace_on = true;
  return TT_OK;
}

tt_status tt_trace_disable(void) {
  for (auto& ev : g_trace_pool) cudaEventDestroy(ev);
  g_trace_pool.clear();
  g_trace.clear();
  g_trace_on = false;
  return TT_OK;
}

int64_t tt_trace_count(void) { return (int64_t)g_trace.size(); }

tt_status tt_trace_read(int64_t i, int* stage, int* tile, int64_t* M, int64_t* N, int64_t* K,
                        float* ms) {
  if (i < 0 || i >= (int64_t)g_trace.size()) return fail(TT_ERR_INVALID_ARGUMENT, "bad index");
  const TraceRec& r = g_trace[size_t(i)];
  if (stage) *stage = r.stage;
  if (tile) *tile = r.tile;
  if (M) *M = r.M;
  if (N) *N = r.N;
  if (K) *K = r.K;
  if (ms) {
    cudaError_t e = cudaEventSynchronize(r.e1);
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms, r.e0, r.e1);
    if (e != cudaSuccess) return cuda_fail(e, "tt_trace_read");
  }
  return TT_OK;
}

tt_status tt_fp64_peak_probe(int64_t iters, double* flops, void* stream) {
  CallScope scope;
  if (iters <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "iters must be positive");
  if (!flops) return fail(TT_ERR_NULL_POINTER, "flops");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = 2 * sms, threads = 256;   // 16 warps per SM
  dmma_probe_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(nullptr, iters);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "tt_fp64_peak_probe");
  *flops = 2.0 * 8 * 8 * 4 * 8.0 * double(iters) * blocks * (threads / 32);
  return TT_OK;
}

}  // extern "C"
