// tt_dag.cuh — persistent, device-scheduled executor for a DAG of small FP64 GEMMs (sm_100a).
//
// The latency-bound sweeps (configs 1-4: W34, the interface chains, single-vector matvecs)
// are long chains of stage GEMMs of a few to a few hundred MFLOP each (PAPER.md:526 three
// products per core, chained over the cores by PAPER.md:244-253).  Launched one kernel per
// stage, every dependent GEMM pays a launch gap and a grid drain.  Here ONE persistent kernel
// runs the whole DAG: a work queue of tile units in topological order, grabbed by the resident
// CTAs with one atomic each; a unit first waits (thread 0 spins on an acquire load) until every
// task it depends on has published all its tiles, computes its C tile with the DMMA inner loop
// of tt_gemm_v2.cuh (16-byte cp.async ring, or 8-byte loads for unaligned views), writes it
// through the stage's 3-level output maps and publishes it (fence + atomic add).  Split-K units
// write partial tiles; the last of a tile's splits (ticket counter) sums them in split order
// (deterministic) and publishes the tile.
//
// Deadlock freedom: units are taken in queue order and every dependency of a unit lies earlier
// in the queue, so the oldest unfinished unit is always runnable by the CTA holding it (CTAs
// only hold a unit while resident).  No co-residency of the whole grid is assumed.
//
// Memory model: producers store, __syncthreads, then thread 0 issues a gpu-scope fence and the
// atomic; consumers acquire-load the counter, __syncthreads, and read operands only through L2
// (cp.async.cg / ld.global.cg), so no stale L1 line of a re-used intermediate is ever read.
// Counters live in the caller's workspace and are zeroed (cudaMemsetAsync) before each launch.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tt_gemm.cuh"
#include "tt_gemm_v2.cuh"

namespace tt {

constexpr int kDagMaxTasks = 112;
constexpr int kDagMaxDeps = 3;
constexpr int kDagMaxSplit = 8;

struct DagTask {
  const double* A;   // (m,k) at m*lda+k if A K-contiguous else k*lda+m
  const double* B;   // (k,n) at n*ldb+k if B K-contiguous else k*ldb+n
  double* C;         // output through rowmap / colmap
  double* P;         // split-K partials [ksplit][M][N] (ksplit > 1)
  IndexMap32 rowmap, colmap;
  int M, N, K, lda, ldb;
  int flags;         // bit 0: A K-contiguous, 1: B K-contiguous, 2: A 16-byte loads, 3: B 16-byte
  int tiles_n, ksplit, kt_per_split, KT;
  int unit0;         // first queue index of this task's units
  int tick0;         // first split-K ticket of this task
  int ndeps;
  int dep[kDagMaxDeps];    // tasks that must have published all their tiles
  int need[kDagMaxDeps];   // = their tile counts
};

struct DagParams {
  int ntasks, total_units;
  int* ctr;          // [0] unit queue head, [1 .. 1+ntasks) published tiles, then tickets
  unsigned long long* trace;   // optional (debug): per unit {grab, ready, computed, done, smid}
  DagTask t[kDagMaxTasks];
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES>
struct DagCfg {
  static constexpr int BK = 16, kThreads = WARPS_M * WARPS_N * 32;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static_assert(WTM % 16 == 0 && WTN % 16 == 0, "warp tile multiple of 16 (paired fragments)");
  static constexpr int MI = WTM / 8, NI = WTN / 8;
  // padded shared-memory rows (doubles): K-contiguous rows 16 + 8 (192 B = 64 mod 128), M/N-
  // contiguous k-rows BX + 2 (16 mod 64 B): conflict-free LDS.128 fragment loads (tt_gemm_v2.cuh)
  static constexpr int KC_LD = BK + 8;
  static constexpr int A_MN_LD = BM + 2, B_MN_LD = BN + 2;
  static constexpr int A_ST = (BM * KC_LD > BK * A_MN_LD) ? BM * KC_LD : BK * A_MN_LD;
  static constexpr int B_ST = (BN * KC_LD > BK * B_MN_LD) ? BN * KC_LD : BK * B_MN_LD;
  static constexpr size_t kSmemBytes = sizeof(double) * (size_t)STAGES * (A_ST + B_ST);
};

// One C tile (or one K-split of it) of task T: k-tiles [kb, ke) accumulated into acc.
template <bool AK, bool BK_, int BM, int BN, int WARPS_M, int WARPS_N, int STAGES>
__device__ __forceinline__ void dag_mainloop(const DagTask& T, int m0, int n0, int kb, int ke,
                                             double* As, double* Bs,
                                             double (&acc)[BM / WARPS_M / 8][BN / WARPS_N / 8][2]) {
  using Cfg = DagCfg<BM, BN, WARPS_M, WARPS_N, STAGES>;
  constexpr int BK = Cfg::BK, NT = Cfg::kThreads, WTM = Cfg::WTM, WTN = Cfg::WTN;
  constexpr int MI = Cfg::MI, NI = Cfg::NI;
  constexpr int A_LD = AK ? Cfg::KC_LD : Cfg::A_MN_LD;
  constexpr int B_LD = BK_ ? Cfg::KC_LD : Cfg::B_MN_LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const bool avec = (T.flags & 4) != 0, bvec = (T.flags & 8) != 0;
  const double* __restrict__ Ag = T.A;
  const double* __restrict__ Bg = T.B;
  const int M = T.M, N = T.N, K = T.K;
  const long long lda = T.lda, ldb = T.ldb;

  auto load = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * Cfg::A_ST;
    double* bs = Bs + stage * Cfg::B_ST;
    if (avec) {
#pragma unroll
      for (int c = tid; c < BM * BK / 2; c += NT) {
        if (AK) {
          const int r = c >> 3, kc = (c & 7) * 2;
          const bool ok = (m0 + r < M) && (k0 + kc < K);
          cp_async16(as + r * A_LD + kc, ok ? Ag + (m0 + r) * lda + (k0 + kc) : Ag, ok);
        } else {
          constexpr int CPR = BM / 2;
          const int kr = c / CPR, mc = (c % CPR) * 2;
          const bool ok = (k0 + kr < K) && (m0 + mc < M);
          cp_async16(as + kr * A_LD + mc, ok ? Ag + (k0 + kr) * lda + (m0 + mc) : Ag, ok);
        }
      }
    } else {
      for (int c = tid; c < BM * BK; c += NT) {
        if (AK) {
          const int r = c >> 4, kk = c & 15;
          const bool ok = (m0 + r < M) && (k0 + kk < K);
          as[r * A_LD + kk] = ok ? __ldcg(Ag + (m0 + r) * lda + (k0 + kk)) : 0.0;
        } else {
          const int kr = c / BM, mm = c % BM;
          const bool ok = (k0 + kr < K) && (m0 + mm < M);
          as[kr * A_LD + mm] = ok ? __ldcg(Ag + (k0 + kr) * lda + (m0 + mm)) : 0.0;
        }
      }
    }
    if (bvec) {
#pragma unroll
      for (int c = tid; c < BN * BK / 2; c += NT) {
        if (BK_) {
          const int r = c >> 3, kc = (c & 7) * 2;
          const bool ok = (n0 + r < N) && (k0 + kc < K);
          cp_async16(bs + r * B_LD + kc, ok ? Bg + (n0 + r) * ldb + (k0 + kc) : Bg, ok);
        } else {
          constexpr int CPR = BN / 2;
          const int kr = c / CPR, nc = (c % CPR) * 2;
          const bool ok = (k0 + kr < K) && (n0 + nc < N);
          cp_async16(bs + kr * B_LD + nc, ok ? Bg + (k0 + kr) * ldb + (n0 + nc) : Bg, ok);
        }
      }
    } else {
      for (int c = tid; c < BN * BK; c += NT) {
        if (BK_) {
          const int r = c >> 4, kk = c & 15;
          const bool ok = (n0 + r < N) && (k0 + kk < K);
          bs[r * B_LD + kk] = ok ? __ldcg(Bg + (n0 + r) * ldb + (k0 + kk)) : 0.0;
        } else {
          const int kr = c / BN, nn = c % BN;
          const bool ok = (k0 + kr < K) && (n0 + nn < N);
          bs[kr * B_LD + nn] = ok ? __ldcg(Bg + (k0 + kr) * ldb + (n0 + nn)) : 0.0;
        }
      }
    }
  };

  // prologue: STAGES-1 k-tiles in flight (empty commit groups past ke keep the count uniform)
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (kb + s < ke) load(s, kb + s);
    cp_async_commit();
  }
  int st = 0;
#pragma unroll 1
  for (int kt = kb; kt < ke; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();   // stage st is complete for every thread; stage st-1 is free
    {
      const int nk = kt + STAGES - 1;
      if (nk < ke) load((st + STAGES - 1) % STAGES, nk);
      cp_async_commit();
    }
    const double* as = As + st * Cfg::A_ST;
    const double* bs = Bs + st * Cfg::B_ST;
    st = (st + 1 == STAGES) ? 0 : st + 1;
#pragma unroll
    for (int kp = 0; kp < BK / 8; ++kp) {   // pairs of DMMA k-steps (lane t <-> k = 2t + s)
      const int kb8 = kp * 8;
      double af[2][MI], bf[2][NI];
      if (AK) {
#pragma unroll
        for (int i = 0; i < MI; ++i)
          lds128(af[0][i], af[1][i], as + (wm * WTM + i * 8 + g) * A_LD + kb8 + 2 * t);
      } else {
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          const double* rowp = as + (kb8 + 2 * t + s2) * A_LD + wm * WTM;
#pragma unroll
          for (int pr = 0; pr < MI / 2; ++pr) lds128(af[s2][2 * pr], af[s2][2 * pr + 1], rowp + pr * 16 + 2 * g);
        }
      }
      if (BK_) {
#pragma unroll
        for (int j = 0; j < NI; ++j)
          lds128(bf[0][j], bf[1][j], bs + (wn * WTN + j * 8 + g) * B_LD + kb8 + 2 * t);
      } else {
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          const double* rowp = bs + (kb8 + 2 * t + s2) * B_LD + wn * WTN;
#pragma unroll
          for (int q2 = 0; q2 < NI / 2; ++q2) lds128(bf[s2][2 * q2], bf[s2][2 * q2 + 1], rowp + q2 * 16 + 2 * g);
        }
      }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma_8x8x4_nv(acc[i][j], af[s2][i], bf[s2][j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();   // the next unit's prologue overwrites the stages
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, int MINB>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, MINB)
dag_gemm_kernel(const __grid_constant__ DagParams p) {
  using Cfg = DagCfg<BM, BN, WARPS_M, WARPS_N, STAGES>;
  constexpr int WTM = Cfg::WTM, WTN = Cfg::WTN, MI = Cfg::MI, NI = Cfg::NI;
  constexpr int NT = Cfg::kThreads;
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;
  double* Bs = dsm + STAGES * Cfg::A_ST;
  __shared__ DagTask sT;
  __shared__ int s_unit, s_last;

  pdl_wait();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  int* const ctr = p.ctr;
  int* const done = ctr + 1;
  int* const ticks = ctr + 1 + p.ntasks;

  // tile rows / columns of this lane's accumulators (tt_gemm_v2.cuh fragment geometry)
  auto frag_row = [&](int i, bool ak) -> int {
    return ak ? wm * WTM + i * 8 + g : wm * WTM + (i >> 1) * 16 + 2 * g + (i & 1);
  };
  auto acc_col = [&](int j, int c, bool bk) -> int {
    return bk ? wn * WTN + j * 8 + c : wn * WTN + (j >> 1) * 16 + 2 * c + (j & 1);
  };

#pragma unroll 1
  for (;;) {
    unsigned long long t_grab = 0;
    if (tid == 0) {
      if (p.trace) t_grab = globaltimer();
      s_unit = atomicAdd(ctr, 1);
    }
    __syncthreads();
    const int u = s_unit;
    if (u >= p.total_units) break;
    if (tid == 0) {
      // task of unit u: the last task whose first unit is <= u
      int lo = 0, hi = p.ntasks - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p.t[mid].unit0 <= u) lo = mid; else hi = mid - 1;
      }
      sT = p.t[lo];
      s_last = lo;
      for (int q = 0; q < sT.ndeps; ++q) {
        const int* c = done + sT.dep[q];
        const int want = sT.need[q];
        int ns = 32;
        while (ld_acquire_gpu(c) < want) {
          __nanosleep(ns);
          if (ns < 256) ns <<= 1;
        }
      }
      if (p.trace) {
        unsigned long long* tr = p.trace + 5ULL * u;
        tr[0] = t_grab;
        tr[1] = globaltimer();
        unsigned sm;
        asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
        tr[4] = sm;
      }
    }
    __syncthreads();
    const DagTask& T = sT;
    const int ti = s_last;
    const int uu = u - T.unit0;
    const int tile = uu / T.ksplit, split = uu - tile * T.ksplit;
    const int tm = tile / T.tiles_n, tn = tile - tm * T.tiles_n;
    const int m0 = tm * BM, n0 = tn * BN;
    const int kb = split * T.kt_per_split, ke = min(T.KT, kb + T.kt_per_split);
    const bool ak = (T.flags & 1) != 0, bk = (T.flags & 2) != 0;

    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (ak && bk) dag_mainloop<true, true, BM, BN, WARPS_M, WARPS_N, STAGES>(T, m0, n0, kb, ke, As, Bs, acc);
    else if (ak) dag_mainloop<true, false, BM, BN, WARPS_M, WARPS_N, STAGES>(T, m0, n0, kb, ke, As, Bs, acc);
    else if (bk) dag_mainloop<false, true, BM, BN, WARPS_M, WARPS_N, STAGES>(T, m0, n0, kb, ke, As, Bs, acc);
    else dag_mainloop<false, false, BM, BN, WARPS_M, WARPS_N, STAGES>(T, m0, n0, kb, ke, As, Bs, acc);

    if (p.trace && tid == 0) p.trace[5ULL * u + 2] = globaltimer();
    bool publish = true;
    if (T.ksplit == 1) {
      long long roff[MI];
      bool rok[MI];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int r = m0 + frag_row(i, ak);
        rok[i] = r < T.M;
        roff[i] = rok[i] ? apply_map32(T.rowmap, (uint32_t)r) : 0;
      }
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + acc_col(j, 2 * t + h, bk);
          if (c < T.N) {
            const long long co = apply_map32(T.colmap, (uint32_t)c);
#pragma unroll
            for (int i = 0; i < MI; ++i)
              if (rok[i]) T.C[roff[i] + co] = acc[i][j][h];
          }
        }
    } else {
      // partial tile -> P[split]; the last split to arrive reduces all of them in split order
      const long long MN = (long long)T.M * T.N;
      double* P = T.P + split * MN;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int r = m0 + frag_row(i, ak);
        if (r < T.M) {
#pragma unroll
          for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = n0 + acc_col(j, 2 * t + h, bk);
              if (c < T.N) __stcg(P + (long long)r * T.N + c, acc[i][j][h]);
            }
        }
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        s_unit = atomicAdd(ticks + T.tick0 + tile, 1);
      }
      __syncthreads();
      publish = (s_unit == T.ksplit - 1);
      if (publish) {
        __threadfence();
        const int rows = min(BM, T.M - m0), cols = min(BN, T.N - n0);
        const int ks = T.ksplit;
        for (int e = tid; e < rows * cols; e += NT) {
          const int r = m0 + e / cols, c = n0 + e % cols;
          const double* src = T.P + (long long)r * T.N + c;
          // all partials in flight at once (ksplit <= kDagMaxSplit), summed in split order
          double v[kDagMaxSplit];
#pragma unroll
          for (int q = 0; q < kDagMaxSplit; ++q) v[q] = q < ks ? __ldcg(src + q * MN) : 0.0;
          double s = v[0];
#pragma unroll
          for (int q = 1; q < kDagMaxSplit; ++q)
            if (q < ks) s += v[q];
          T.C[apply_map32(T.rowmap, (uint32_t)r) + apply_map32(T.colmap, (uint32_t)c)] = s;
        }
      }
    }
    __syncthreads();
    if (publish && tid == 0) {
      __threadfence();
      atomicAdd(done + ti, 1);
    }
    if (p.trace && tid == 0) p.trace[5ULL * u + 3] = globaltimer();
  }
  pdl_trigger();
}

}  // namespace tt
