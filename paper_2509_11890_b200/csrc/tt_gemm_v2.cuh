// tt_gemm_v2.cuh — persistent FP64 DMMA GEMM for the TT contraction stages (sm_100a).
//
// Same contract as tt_gemm.cuh (C[m,n] = sum_k A[m,k] B[k,n], plain 2-D operand views,
// 3-level output index maps), tuned for the large stages:
//  * 16 warps / SM (one 512-thread CTA): DMMA.8x8x4 blocks its issuing warp for ~16 cycles,
//    so four warps per SM sub-partition are needed to keep the FP64 tensor pipe busy while
//    each warp also issues its loads and address arithmetic (measured: 2 warps/SMSP left
//    the pipe 38% idle, ncu stall "wait").
//  * persistent CTAs (grid = #SMs) walk their tiles as one continuous stream of k-tiles, so
//    the cp.async ring prefetches the next tile's operands during the current epilogue.
//  * 16-byte cp.async.cg (L2 only) with per-tile base pointers; zero-fill for M/N/K tails.
//  * 128-bit shared-memory fragment loads, conflict-free by construction:
//      K-contiguous tiles  [row][16+8]: one LDS.128 = the lane's A (or B) values of two
//                                      consecutive DMMA k-steps (lane t <-> k = 2t + s);
//      MN-contiguous tiles [k][BX+2]:   one LDS.128 = two fragments of one k-step (fragment
//                                      2p <-> rows 16p+2g, 2p+1 <-> rows 16p+2g+1).
//  * epilogue index maps with host-precomputed 32-bit magic-number division.
// Preconditions (checked by the host, which falls back to tt_gemm.cuh otherwise): base
// pointers 16-byte aligned, even leading dimensions, the contiguous extent of each operand
// (K for K-contiguous, M or N otherwise) even, M, N < 2^31.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tt_gemm.cuh"

namespace tt {

// q = x / d for 0 <= x < 2^31, 1 <= d < 2^31: q = (umulhi(x, mul) + x) >> shift
struct FastDiv {
  uint32_t d, mul, shift;
};
static inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.shift = l;
  f.mul = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
  return (__umulhi(x, f.mul) + x) >> f.shift;
}

// x -> (x % d0) * s0 + ((x / d0) % d1) * s1 + (x / (d0 d1)) * s2 with 32-bit index math
struct IndexMap32 {
  FastDiv d0, d1;
  long long s0, s1, s2;
};
static inline IndexMap32 to_map32(const IndexMap& m) {
  IndexMap32 r;
  const long long big = (1LL << 31) - 1;
  r.d0 = make_fastdiv((uint32_t)(m.d0 > big ? big : m.d0));
  r.d1 = make_fastdiv((uint32_t)(m.d1 > big ? big : m.d1));
  r.s0 = m.s0;
  r.s1 = m.s1;
  r.s2 = m.s2;
  return r;
}
__device__ __forceinline__ long long apply_map32(const IndexMap32& m, uint32_t x) {
  const uint32_t x1 = fdiv(x, m.d0);
  const uint32_t q0 = x - x1 * m.d0.d;
  const uint32_t q2 = fdiv(x1, m.d1);
  const uint32_t q1 = x1 - q2 * m.d1.d;
  return (long long)q0 * m.s0 + (long long)q1 * m.s1 + (long long)q2 * m.s2;
}

struct GemmParamsV2 {
  const double* A;
  const double* B;
  double* C;        // final output (ksplit == 1) ...
  double* P;        // ... or partial sums P[split][m][n] (ksplit > 1), reduced afterwards
  int M, N, K;
  long long lda, ldb;
  IndexMap32 rowmap, colmap;
  int tiles_n, total_units, KT, ksplit, kt_per_split;
  int dbg;          // benchmark hook: bit 0 = skip output stores, bit 1 = skip operand loads
  const int* gate;  // optional device flag: nonzero -> no-op
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int sz = ok ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(sz));
}
__device__ __forceinline__ void lds128(double& x, double& y, const double* p) {
  const double2 v = *reinterpret_cast<const double2*>(p);   // LDS.128 (p is 16-B aligned)
  x = v.x;
  y = v.y;
}
__device__ __forceinline__ double lds64(const double* p) { return *p; }
// non-volatile: a pure register operation the compiler may schedule freely
__device__ __forceinline__ void dmma_8x8x4_nv(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void stg_cs(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;\n" ::"l"(p), "d"(v));
}

template <bool A_KC, bool B_KC, int BM_, int BN, int WARPS_M, int WARPS_N, int STAGES, int MINB>
struct GemmV2Cfg {
  static constexpr int BM = BM_, BK = 16, kThreads = WARPS_M * WARPS_N * 32;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tile multiple of 8");
  static constexpr int MI = WTM / 8, NI = WTN / 8;
  // shared-memory row strides (doubles): K-contiguous rows 16+8 (= 192 B == 64 mod 128);
  // MN-contiguous rows BX+2 (== 16 mod 64 bytes)
  static constexpr int A_LD = A_KC ? (BK + 8) : (BM + 2);
  static constexpr int B_LD = B_KC ? (BK + 8) : (BN + 2);
  static constexpr int A_ST = A_KC ? BM * A_LD : BK * A_LD;
  static constexpr int B_ST = B_KC ? BN * B_LD : BK * B_LD;
  static constexpr int A_CHUNKS = BM * BK / 2, B_CHUNKS = BN * BK / 2;   // 16-byte chunks
  static constexpr size_t kSmemBytes = sizeof(double) * (size_t)STAGES * (A_ST + B_ST);
};

template <bool A_KC, bool B_KC, int BM_, int BN, int WARPS_M, int WARPS_N, int STAGES, int MINB>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, MINB)
dmma_gemm_v2_kernel(const GemmParamsV2 p) {
  pdl_wait();
  pdl_trigger();
  if (p.gate && *p.gate) return;
  using Cfg = GemmV2Cfg<A_KC, B_KC, BM_, BN, WARPS_M, WARPS_N, STAGES, MINB>;
  constexpr int BM = Cfg::BM, BK = Cfg::BK, NT = Cfg::kThreads;
  constexpr int WTM = Cfg::WTM, WTN = Cfg::WTN, MI = Cfg::MI, NI = Cfg::NI;
  constexpr int A_LD = Cfg::A_LD, B_LD = Cfg::B_LD, A_ST = Cfg::A_ST, B_ST = Cfg::B_ST;

  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_ST;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;

  // ---- loader: stage <- k-tile kt of the tile at (m0, n0) ------------------------------
  auto load = [&](int stage, int m0, int n0, int kt) {
    if (p.dbg & 2) return;
    const int k0 = kt * BK;
    double* as = As + stage * A_ST;
    double* bs = Bs + stage * B_ST;
#pragma unroll
    for (int c = tid; c < Cfg::A_CHUNKS; c += NT) {
      if (A_KC) {
        const int r = c >> 3, kc = (c & 7) * 2;
        const bool ok = (m0 + r < p.M) && (k0 + kc < p.K);
        const double* src = ok ? p.A + (long long)(m0 + r) * p.lda + (k0 + kc) : p.A;
        cp_async16(as + r * A_LD + kc, src, ok);
      } else {
        constexpr int CPR = BM / 2;   // chunks per k-row
        const int kr = c / CPR, mc = (c % CPR) * 2;
        const bool ok = (k0 + kr < p.K) && (m0 + mc < p.M);
        const double* src = ok ? p.A + (long long)(k0 + kr) * p.lda + (m0 + mc) : p.A;
        cp_async16(as + kr * A_LD + mc, src, ok);
      }
    }
#pragma unroll
    for (int c = tid; c < Cfg::B_CHUNKS; c += NT) {
      if (B_KC) {
        const int r = c >> 3, kc = (c & 7) * 2;
        const bool ok = (n0 + r < p.N) && (k0 + kc < p.K);
        const double* src = ok ? p.B + (long long)(n0 + r) * p.ldb + (k0 + kc) : p.B;
        cp_async16(bs + r * B_LD + kc, src, ok);
      } else {
        constexpr int CPR = BN / 2;
        const int kr = c / CPR, nc = (c % CPR) * 2;
        const bool ok = (k0 + kr < p.K) && (n0 + nc < p.N);
        const double* src = ok ? p.B + (long long)(k0 + kr) * p.ldb + (n0 + nc) : p.B;
        cp_async16(bs + kr * B_LD + nc, src, ok);
      }
    }
  };

  // work unit u -> (tile, k-split): m0, n0, [kt_begin, kt_end)
  struct Unit {
    int m0, n0, kb, ke, split;
  };
  auto unit_of = [&](int u) -> Unit {
    Unit w;
    const int tile = u / p.ksplit;
    w.split = u - tile * p.ksplit;
    const int tm = tile / p.tiles_n;
    w.m0 = tm * BM;
    w.n0 = (tile - tm * p.tiles_n) * BN;
    w.kb = w.split * p.kt_per_split;
    w.ke = min(p.KT, w.kb + p.kt_per_split);
    return w;
  };
  // ---- fragment geometry ---------------------------------------------------------------
  // row (within the CTA tile) of fragment i, lane-group g
  auto frag_row = [&](int i) -> int {
    if (A_KC) return wm * WTM + i * 8 + g;
    const int pr = i >> 1;
    if ((MI & 1) && i == MI - 1) return wm * WTM + pr * 16 + g;   // lone last fragment
    return wm * WTM + pr * 16 + 2 * g + (i & 1);
  };
  // column (within the CTA tile) of accumulator column c (0..7) of fragment j
  auto acc_col = [&](int j, int c) -> int {
    if (B_KC) return wn * WTN + j * 8 + c;
    const int q = j >> 1;
    if ((NI & 1) && j == NI - 1) return wn * WTN + q * 16 + c;
    return wn * WTN + q * 16 + 2 * c + (j & 1);
  };

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // this CTA's k-tile stream over units blockIdx.x, blockIdx.x + gridDim.x, ...
  int l_u = blockIdx.x;
  Unit lw = unit_of(l_u < p.total_units ? l_u : 0);
  int l_kt = lw.kb;
  int l_stage = 0;
#pragma unroll 1
  for (int s = 0; s < STAGES - 1; ++s) {
    if (l_u < p.total_units) {
      load(l_stage, lw.m0, lw.n0, l_kt);
      if (++l_kt == lw.ke) {
        l_u += gridDim.x;
        if (l_u < p.total_units) {
          lw = unit_of(l_u);
          l_kt = lw.kb;
        }
      }
    }
    l_stage = (l_stage + 1 == STAGES) ? 0 : l_stage + 1;
    cp_async_commit();
  }

  int c_u = blockIdx.x;
  Unit cw = unit_of(c_u < p.total_units ? c_u : 0);
  int c_kt = cw.kb;
  int st = 0;
#pragma unroll 1
  while (c_u < p.total_units) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (l_u < p.total_units) {
      load(l_stage, lw.m0, lw.n0, l_kt);
      if (++l_kt == lw.ke) {
        l_u += gridDim.x;
        if (l_u < p.total_units) {
          lw = unit_of(l_u);
          l_kt = lw.kb;
        }
      }
    }
    l_stage = (l_stage + 1 == STAGES) ? 0 : l_stage + 1;
    cp_async_commit();

    const double* as = As + st * A_ST;
    const double* bs = Bs + st * B_ST;
    st = (st + 1 == STAGES) ? 0 : st + 1;
#pragma unroll
    for (int kp = 0; kp < BK / 8; ++kp) {      // pairs of DMMA k-steps
      const int kb = kp * 8;
      double af[2][MI], bf[2][NI];             // [step s][fragment]
      // A fragments
      if (A_KC) {
#pragma unroll
        for (int i = 0; i < MI; ++i) lds128(af[0][i], af[1][i], as + frag_row(i) * A_LD + kb + 2 * t);
      } else {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const double* rowp = as + (kb + 2 * t + s) * A_LD + wm * WTM;
#pragma unroll
          for (int pr = 0; pr < MI / 2; ++pr) lds128(af[s][2 * pr], af[s][2 * pr + 1], rowp + pr * 16 + 2 * g);
          if (MI & 1) af[s][MI - 1] = lds64(rowp + (MI / 2) * 16 + g);
        }
      }
      // B fragments
      if (B_KC) {
#pragma unroll
        for (int j = 0; j < NI; ++j)
          lds128(bf[0][j], bf[1][j], bs + (wn * WTN + j * 8 + g) * B_LD + kb + 2 * t);
      } else {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const double* rowp = bs + (kb + 2 * t + s) * B_LD + wn * WTN;
#pragma unroll
          for (int q2 = 0; q2 < NI / 2; ++q2) lds128(bf[s][2 * q2], bf[s][2 * q2 + 1], rowp + q2 * 16 + 2 * g);
          if (NI & 1) bf[s][NI - 1] = lds64(rowp + (NI / 2) * 16 + g);
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma_8x8x4_nv(acc[i][j], af[s][i], bf[s][j]);
    }

    if (++c_kt == cw.ke) {
      // ---- epilogue of unit c_u ---------------------------------------------------------
      const int m0 = cw.m0, n0 = cw.n0;
      if (p.dbg & 1) {
        // skip stores (benchmark hook); keep the accumulators live
        double sink = 0.0;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) sink += acc[i][j][0] + acc[i][j][1];
        if (sink == 1.2345e-300) p.C[0] = sink;
      } else if (p.ksplit == 1) {
        long long roff[MI];
        bool rok[MI];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int r = m0 + frag_row(i);
          rok[i] = r < p.M;
          roff[i] = rok[i] ? apply_map32(p.rowmap, (uint32_t)r) : 0;
        }
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = n0 + acc_col(j, 2 * t + h);
            if (c < p.N) {
              const long long co = apply_map32(p.colmap, (uint32_t)c);
#pragma unroll
              for (int i = 0; i < MI; ++i)
                if (rok[i]) stg_cs(p.C + roff[i] + co, acc[i][j][h]);
            }
          }
      } else {
        double* P = p.P + (long long)cw.split * p.M * p.N;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int r = m0 + frag_row(i);
          if (r < p.M) {
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int c = n0 + acc_col(j, 2 * t + h);
                if (c < p.N) P[(long long)r * p.N + c] = acc[i][j][h];
              }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      c_u += gridDim.x;
      if (c_u < p.total_units) {
        cw = unit_of(c_u);
        c_kt = cw.kb;
      }
    }
  }
  cp_async_wait<0>();
}

// C[rowmap(m) + colmap(n)] = sum_s P[s][m][n]  (split-K reduction, fixed summation order).
// Streaming: the partials are read once (evict-first), two adjacent columns per thread when N
// is even (16-byte loads; one 16-byte store where the column map keeps the pair adjacent and
// aligned), the row/column split by a host-built magic divisor instead of a 64-bit division.
static __global__ void __launch_bounds__(256) splitk_reduce_kernel(const double* __restrict__ P,
                                                            double* __restrict__ C, int M, int N,
                                                            int ksplit, IndexMap32 rowmap,
                                                            IndexMap32 colmap, FastDiv ndiv,
                                                            const int* gate) {
  pdl_wait();
  if (gate && *gate) return;
  const long long MN = (long long)M * N;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if ((N & 1) == 0 && MN < (1LL << 31) && !(reinterpret_cast<uintptr_t>(P) & 15)) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; 2 * t < MN; t += stride) {
      const uint32_t e = (uint32_t)(2 * t);
      double2 acc = __ldcs(reinterpret_cast<const double2*>(P + e));
      int q = 1;
      for (; q + 1 < ksplit; q += 2) {
        const double2 v0 = __ldcs(reinterpret_cast<const double2*>(P + (long long)q * MN + e));
        const double2 v1 = __ldcs(reinterpret_cast<const double2*>(P + (long long)(q + 1) * MN + e));
        acc.x += v0.x;
        acc.y += v0.y;
        acc.x += v1.x;
        acc.y += v1.y;
      }
      if (q < ksplit) {
        const double2 v0 = __ldcs(reinterpret_cast<const double2*>(P + (long long)q * MN + e));
        acc.x += v0.x;
        acc.y += v0.y;
      }
      const uint32_t m = fdiv(e, ndiv), n = e - m * (uint32_t)N;
      double* row = C + apply_map32(rowmap, m);
      const long long c0 = apply_map32(colmap, n), c1 = apply_map32(colmap, n + 1);
      double* d0 = row + c0;
      if (c1 == c0 + 1 && !(reinterpret_cast<uintptr_t>(d0) & 15)) {
        asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};\n" ::"l"(d0), "d"(acc.x), "d"(acc.y));
      } else {
        stg_cs(d0, acc.x);
        stg_cs(row + c1, acc.y);
      }
    }
  } else {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < MN; e += stride) {
      double sum = P[e];
      for (int q = 1; q < ksplit; ++q) sum += P[q * MN + e];
      const int m = (int)(e / N), n = (int)(e - (long long)m * N);
      stg_cs(C + apply_map32(rowmap, (uint32_t)m) + apply_map32(colmap, (uint32_t)n), sum);
    }
  }
  pdl_trigger();
}

}  // namespace tt
