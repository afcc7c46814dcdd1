// tt_gemm.cuh — FP64 tensor-core (DMMA) GEMM engine for the TT contraction stages, sm_100a.
//
// Every stage of the local matvec / interface updates is ONE dense GEMM
//   C[m, n] = sum_k A[m, k] B[k, n]
// whose operands are plain 2-D strided views (one dimension unit-stride) of a core,
// interface or intermediate, and whose output is scattered through a 3-level index map so
// that the next stage reads a plain 2-D view again.  Blackwell has no FP64 UMMA (tcgen05
// rejects .kind::f64), so the math is warp-level mma.sync.m8n8k4.f64 -> DMMA.8x8x4, with
// accumulators in registers.  Tiles are staged global -> shared by an STAGES-deep cp.async
// ring (8-byte zero-filling copies: handles any alignment, ragged M/N/K and strided views);
// shared-memory rows are padded by 4 doubles so that every fragment load is conflict-free.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tt {

// x -> (x % d0) * s0 + ((x / d0) % d1) * s1 + (x / (d0 * d1)) * s2
struct IndexMap {
  long long d0, d1, s0, s1, s2;
};

static constexpr long long kBig = (1LL << 62);
static inline IndexMap map_plain(long long stride) { return IndexMap{kBig, kBig, stride, 0, 0}; }
static inline IndexMap map2(long long d0, long long s0, long long s1) {
  return IndexMap{d0, kBig, s0, s1, 0};
}
static inline IndexMap map3(long long d0, long long d1, long long s0, long long s1, long long s2) {
  return IndexMap{d0, d1, s0, s1, s2};
}

__device__ __forceinline__ long long apply_map(const IndexMap& m, long long x) {
  const long long x1 = x / m.d0;
  const long long q0 = x - x1 * m.d0;
  const long long q2 = x1 / m.d1;
  const long long q1 = x1 - q2 * m.d1;
  return q0 * m.s0 + q1 * m.s1 + q2 * m.s2;
}

struct GemmParams {
  const double* A;
  const double* B;
  double* C;
  long long M, N, K;
  long long lda, ldb;   // A: (m,k) at m*lda+k if A_KC else k*lda+m;  B: (k,n) at n*ldb+k if B_KC else k*ldb+n
  IndexMap rowmap, colmap;
  long long tiles_n;
  const int* gate;   // optional device flag: nonzero -> the launch is a no-op (iterative solvers)
};

// Programmatic dependent launch (PDL).  Every kernel the library may launch with the
// programmatic-serialisation attribute waits for its stream predecessor here, before its
// first global-memory access (read or write) and before any early return, so completion stays
// transitive along the stream; it then lets its own successor be launched, whose CTAs run
// their prologue (barrier init, descriptor prefetch) on SMs this grid leaves idle.
// Both instructions are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int sz = ok ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool A_KC, bool B_KC>
struct GemmCfg {
  static constexpr int kThreads = WARPS_M * WARPS_N * 32;
  static constexpr int kBM = BM, kBN = BN, kBK = BK;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MI = WTM / 8, NI = WTN / 8;
  static constexpr int A_LD = A_KC ? (BK + 4) : (BM + 4);
  static constexpr int B_LD = B_KC ? (BK + 4) : (BN + 4);
  static constexpr int A_ST = A_KC ? BM * A_LD : BK * A_LD;
  static constexpr int B_ST = B_KC ? BN * B_LD : BK * B_LD;
  static constexpr size_t kSmemBytes = sizeof(double) * (size_t)STAGES * (A_ST + B_ST);
  static_assert(BM % (8 * WARPS_M) == 0 && BN % (8 * WARPS_N) == 0, "warp tile must be 8-aligned");
  static_assert(BK % 4 == 0, "BK multiple of the DMMA k=4");
};

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool A_KC, bool B_KC>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, 1)
dmma_gemm_kernel(const GemmParams p) {
  pdl_wait();
  pdl_trigger();
  if (p.gate && *p.gate) return;
  using Cfg = GemmCfg<BM, BN, BK, WARPS_M, WARPS_N, STAGES, A_KC, B_KC>;
  constexpr int NT = Cfg::kThreads;
  constexpr int WTM = Cfg::WTM, WTN = Cfg::WTN, MI = Cfg::MI, NI = Cfg::NI;
  constexpr int A_LD = Cfg::A_LD, B_LD = Cfg::B_LD, A_ST = Cfg::A_ST, B_ST = Cfg::B_ST;

  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_ST;

  const long long tile = blockIdx.x;
  const long long tm = tile / p.tiles_n;
  const long long tn = tile - tm * p.tiles_n;
  const long long m0 = tm * BM, n0 = tn * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const long long KT = (p.K + BK - 1) / BK;

  auto load_tile = [&](int stage, long long kt) {
    const long long k0 = kt * BK;
    double* as = As + stage * A_ST;
    double* bs = Bs + stage * B_ST;
#pragma unroll
    for (int e = tid; e < BM * BK; e += NT) {
      const int mm = A_KC ? e / BK : e % BM;
      const int kk = A_KC ? e % BK : e / BM;
      const long long gm = m0 + mm, gk = k0 + kk;
      const bool ok = (gm < p.M) && (gk < p.K);
      const double* src = ok ? (A_KC ? p.A + gm * p.lda + gk : p.A + gk * p.lda + gm) : p.A;
      cp_async8(A_KC ? as + mm * A_LD + kk : as + kk * A_LD + mm, src, ok);
    }
#pragma unroll
    for (int e = tid; e < BN * BK; e += NT) {
      const int nn = B_KC ? e / BK : e % BN;
      const int kk = B_KC ? e % BK : e / BN;
      const long long gn = n0 + nn, gk = k0 + kk;
      const bool ok = (gn < p.N) && (gk < p.K);
      const double* src = ok ? (B_KC ? p.B + gn * p.ldb + gk : p.B + gk * p.ldb + gn) : p.B;
      cp_async8(B_KC ? bs + nn * B_LD + kk : bs + kk * B_LD + nn, src, ok);
    }
  };

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_tile(s, s);
    cp_async_commit();
  }

  for (long long kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const long long nk = kt + STAGES - 1;
      if (nk < KT) load_tile(static_cast<int>(nk % STAGES), nk);
      cp_async_commit();
    }
    const int st = static_cast<int>(kt % STAGES);
    const double* as = As + st * A_ST;
    const double* bs = Bs + st * B_ST;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double af[MI], bf[NI];
      const int kk = ks * 4 + t;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int mm = wm * WTM + i * 8 + g;
        af[i] = A_KC ? as[mm * A_LD + kk] : as[kk * A_LD + mm];
      }
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int nn = wn * WTN + j * 8 + g;
        bf[j] = B_KC ? bs[nn * B_LD + kk] : bs[kk * B_LD + nn];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // Epilogue: D fragment lane (g,t) holds rows g, cols 2t, 2t+1 of each 8x8 tile.
  long long roff[MI];
  bool rok[MI];
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const long long r = m0 + wm * WTM + i * 8 + g;
    rok[i] = r < p.M;
    roff[i] = rok[i] ? apply_map(p.rowmap, r) : 0;
  }
  long long coff[NI][2];
  bool cok[NI][2];
#pragma unroll
  for (int j = 0; j < NI; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long c = n0 + wn * WTN + j * 8 + 2 * t + h;
      cok[j][h] = c < p.N;
      coff[j][h] = cok[j][h] ? apply_map(p.colmap, c) : 0;
    }
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (rok[i] && cok[j][h]) p.C[roff[i] + coff[j][h]] = acc[i][j][h];
}

}  // namespace tt
