// tt_gemm_v3.cuh — TMA + mbarrier FP64 DMMA GEMM for the TT contraction stages (sm_100a).
//
// Same contract as tt_gemm.cuh / tt_gemm_v2.cuh (C[m,n] = sum_k A[m,k] B[k,n] over plain 2-D
// operand views, 3-level output index maps, optional split-K), with the operand path moved
// to the Blackwell copy engine:
//  * operand tiles arrive by TMA (cp.async.bulk.tensor.2d, SWIZZLE_128B, OOB zero-fill),
//    issued by one thread; per-stage `full` mbarriers carry the transaction count, per-stage
//    `empty` mbarriers collect one arrival per consumer warp.  There is no CTA-wide barrier
//    in the main loop: each warp runs ahead as soon as its stage is full, so one warp's
//    epilogue or fragment-load latency overlaps the other warps' DMMA stream.
//  * two 256-thread CTAs per SM (4 warps per sub-partition), persistent over work units,
//    the k-tile stream continuing across tiles.
//  * fragment loads are 128-bit and bank-conflict-free under the 128-byte swizzle:
//      K-contiguous tiles (rows of 16 doubles = 128 B): fragment row g <-> tile row
//        8i + 4(g&1) + (g>>1), so the two rows a quarter-warp reads differ by 4 mod 8 and the
//        XOR swizzle sends them to disjoint 64-byte halves; one LDS.128 = two DMMA k-steps
//        (lane t <-> k = 2t + s).
//      M/N-contiguous tiles (16-wide boxes of 16 k-rows): fragment pair (2p, 2p+1) <-> rows
//        (16p+2g, 16p+2g+1); the quarter-warp's four k-rows 2t+s carry XOR keys 2t+s, so the
//        eight 16-byte chunks are distinct.
// Preconditions (host-checked; else tt_gemm_v2/v1): 16-byte aligned bases, even leading
// dimensions, even contiguous extents, M/N-contiguous tile extents multiples of 16.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "tt_gemm_v2.cuh"

namespace tt {

struct GemmParamsV3 {
  double* C;
  double* P;
  int M, N, K;
  IndexMap32 rowmap, colmap;
  int tiles_n, total_units, KT, ksplit, kt_per_split;
  FastDiv tiles_n_div;   // magic division by tiles_n (unit decode)
  int a3d, b3d;     // MN-contiguous operand described by a 3-D map (one TMA per stage)
  int tiles_m, group_m;   // tile order: groups of group_m M-tiles, M fastest inside a group
                          // (group_m = 1: N-fastest rows of tiles)
  int l2_a, l2_b;   // TMA L2 policy per operand: 0 default, 1 evict_last (reused, L2-sized),
                    // 2 evict_first (streamed once, larger than L2)
  int store_mode;   // 0 scalar; 1 column pairs (N-contiguous B, output contiguous along n);
                    // 2 row pairs (M-contiguous A, output contiguous along m) -> 16-byte stores;
                    // 3 column quads (as 1, contiguous in fours) -> 32-byte stores
  int dbg;
  int skew;         // k-tiles by which the second half of the warps trails the first (0 = off)
  const int* gate;  // optional device flag: nonzero -> no-op
};

// 32-byte store (sm_100: STG.E.EF.256)
__device__ __forceinline__ void stg_cs4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d));
}
__device__ __forceinline__ void stg_cs2(double* p, double a, double b) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// 3-D box {16 (m_lo), 16 (k), nslab (m_hi)}: the BM/16 swizzled 2 KB slabs of an
// M-contiguous operand tile in one instruction (same shared-memory layout as nslab 2-D boxes)
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar, uint64_t pol, bool hint) {
  if (hint)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)),
        "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint64_t l2_policy(int kind) {
  uint64_t pol = 0;
  if (kind == 1)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// B_RES: the whole B operand of a single-N-tile GEMM (the operator-core stage's A-hat,
// K x N <= kBresMaxKT x 16 x BN doubles) is loaded once per CTA into a resident shared-memory
// block; the ring then carries only A tiles.
constexpr int kBresMaxKT = 9;
template <bool A_KC, bool B_KC, int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, int MINB,
          bool B_RES = false>
struct GemmV3Cfg {
  static constexpr int BK = 16, kThreads = WARPS_M * WARPS_N * 32, kWarps = WARPS_M * WARPS_N;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tile multiple of 8");
  static_assert(A_KC || BM % 16 == 0, "M-contiguous A needs 16-wide boxes");
  static_assert(B_KC || BN % 16 == 0, "N-contiguous B needs 16-wide boxes");
  static constexpr int MI = WTM / 8, NI = WTN / 8;
  static constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128;   // 16 doubles per row/column
  static constexpr int STAGE_BYTES = B_RES ? A_BYTES : A_BYTES + B_BYTES;
  static constexpr int BRES_BYTES = B_RES ? kBresMaxKT * B_BYTES : 0;
  static_assert(A_BYTES % 1024 == 0 || BM % 8 == 0, "");
  // +1024 alignment slack for the 128-byte swizzle atoms
  static constexpr size_t kSmemBytes = (size_t)STAGES * STAGE_BYTES + BRES_BYTES + 1024;
};

// RR: the refill of the ring (an empty-barrier wait plus the TMA issue) rotates over the warps
// -- the warp q mod kWarps issues the load that follows k-tile q, in stream order through a
// shared turn counter -- instead of always falling on warp 0, whose critical path it lengthened
// (an extra producer warp costs a quarter of the register file: 13 warps put 4 on one
// sub-partition, 128 registers per thread).
template <bool A_KC, bool B_KC, int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, int MINB,
          bool B_RES = false, bool RR = false>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, MINB)
dmma_gemm_v3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmParamsV3 p) {
  using Cfg = GemmV3Cfg<A_KC, B_KC, BM, BN, WARPS_M, WARPS_N, STAGES, MINB, B_RES>;
  constexpr int WTM = Cfg::WTM, WTN = Cfg::WTN, MI = Cfg::MI, NI = Cfg::NI;
  constexpr int A_BYTES = Cfg::A_BYTES, STAGE_BYTES = Cfg::STAGE_BYTES;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], bres_bar;
  // align to the 1 KB swizzle atom by integer offset so the compiler keeps the shared
  // address space (generic pointer arithmetic would turn every LDS into a generic LD)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  constexpr int kProdTid = 0;   // the thread that issues the prologue's TMA loads
  __shared__ volatile int prod_turn;   // RR: the k-tile whose refill is due next

  // Column offsets of the output map: when the whole N extent is one tile (the operator-core
  // stage, N = n R <= 144) every unit has c_n0 = 0, so the BN offsets are evaluated once into
  // shared memory instead of two magic divisions per column per unit in the epilogue.
  __shared__ long long ctab[BN];
  const bool col_cached = p.tiles_n == 1 && !(p.dbg & 262144);
  if (col_cached)
    for (int c = threadIdx.x; c < BN; c += blockDim.x)
      ctab[c] = c < p.N ? apply_map32(p.colmap, (uint32_t)c) : 0;
  auto col_off = [&](int c) -> long long {
    return col_cached ? ctab[c] : apply_map32(p.colmap, (uint32_t)c);
  };
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], Cfg::kWarps);
    }
    if constexpr (B_RES) mbar_init(&bres_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  __syncthreads();
  // PDL: the barrier setup above overlaps the predecessor's tail (tt_gemm.cuh).  The
  // successor is released when every CTA has started its LAST unit (below), so its CTAs are
  // placed on SMs as this grid's CTAs retire rather than piling onto the few with spare room.
  pdl_wait();
  if (p.gate && *p.gate) return;

  // (the common cases ksplit == 1 and a single N tile skip the integer divisions: the
  // operator-core stage switches units every 9 k-tiles; debug bit 19 forces the generic path)
  const bool fast_units = !(p.dbg & 524288);
  auto unit_of = [&](int u, int& m0, int& n0, int& kb, int& ke, int& split) {
    const int tile = (fast_units && p.ksplit == 1) ? u : u / p.ksplit;
    split = u - tile * p.ksplit;
    int tm, tn;
    if (fast_units && p.group_m <= 1 && p.tiles_n == 1) {
      tm = tile;
      tn = 0;
    } else if (fast_units && p.group_m <= 1) {
      tm = (int)fdiv((uint32_t)tile, p.tiles_n_div);
      tn = tile - tm * p.tiles_n;
    } else if (p.group_m <= 1) {
      tm = tile / p.tiles_n;
      tn = tile - tm * p.tiles_n;
    } else {
      const int per_group = p.group_m * p.tiles_n;
      const int grp = tile / per_group, first = grp * p.group_m;
      const int gsz = min(p.tiles_m - first, p.group_m);
      const int r = tile - grp * per_group;
      tm = first + r % gsz;
      tn = r / gsz;
    }
    m0 = tm * BM;
    n0 = tn * BN;
    kb = split * p.kt_per_split;
    ke = min(p.KT, kb + p.kt_per_split);
  };

  const bool may_produce = RR ? lane == 0 : tid == kProdTid;
  const uint64_t pol_a = (may_produce && p.l2_a) ? l2_policy(p.l2_a) : 0;
  const uint64_t pol_b = (may_produce && p.l2_b) ? l2_policy(p.l2_b) : 0;
  // ---- producer state (thread 0 only; kept in shared memory to spare registers) ---------
  __shared__ int prod_state[7];   // u, m0, n0, kt, ke, split, q
  if (tid == kProdTid) {
    int* ps = prod_state;
    ps[0] = blockIdx.x;
    ps[6] = 0;
    if (ps[0] < p.total_units) unit_of(ps[0], ps[1], ps[2], ps[3], ps[4], ps[5]);
  }
  auto produce_one = [&]() {   // thread 0: issue the next k-tile of the stream, if any
    int* ps = prod_state;
    if (ps[0] >= p.total_units) return;
    const uint32_t lq = (uint32_t)ps[6];
    const int s = (int)(lq % STAGES);
    if (lq >= (uint32_t)STAGES) mbar_wait(&empty_bar[s], ((lq / STAGES) - 1) & 1);
    unsigned char* as = smem + s * STAGE_BYTES;
    unsigned char* bs = as + A_BYTES;
    const int k0 = ps[3] * Cfg::BK, m0 = ps[1], n0 = ps[2];
    mbar_expect_tx(&full_bar[s], STAGE_BYTES);
    (void)bs;
    if (!(p.dbg & 2)) {
      if (A_KC) {
        if (p.l2_a) tma_load_2d_hint(as, &tmA, k0, m0, &full_bar[s], pol_a);
        else tma_load_2d(as, &tmA, k0, m0, &full_bar[s]);
      } else if (p.a3d) {
        tma_load_3d(as, &tmA, 0, k0, m0 / 16, &full_bar[s], pol_a, p.l2_a != 0);
      } else {
#pragma unroll
        for (int b = 0; b < BM / 16; ++b) {
          if (p.l2_a) tma_load_2d_hint(as + b * 2048, &tmA, m0 + 16 * b, k0, &full_bar[s], pol_a);
          else tma_load_2d(as + b * 2048, &tmA, m0 + 16 * b, k0, &full_bar[s]);
        }
      }
      if constexpr (B_RES) {
      } else if (B_KC) {
        if (p.l2_b) tma_load_2d_hint(bs, &tmB, k0, n0, &full_bar[s], pol_b);
        else tma_load_2d(bs, &tmB, k0, n0, &full_bar[s]);
      } else if (p.b3d) {
        tma_load_3d(bs, &tmB, 0, k0, n0 / 16, &full_bar[s], pol_b, p.l2_b != 0);
      } else {
#pragma unroll
        for (int b = 0; b < BN / 16; ++b) {
          if (p.l2_b) tma_load_2d_hint(bs + b * 2048, &tmB, n0 + 16 * b, k0, &full_bar[s], pol_b);
          else tma_load_2d(bs + b * 2048, &tmB, n0 + 16 * b, k0, &full_bar[s]);
        }
      }
    } else {
      // benchmark hook: no loads; complete the transaction count locally
      asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&full_bar[s])),
                   "r"((uint32_t)STAGE_BYTES)
                   : "memory");
    }
    ps[6] = (int)(lq + 1);
    if (++ps[3] == ps[4]) {
      ps[0] += gridDim.x;
      if (ps[0] < p.total_units) unit_of(ps[0], ps[1], ps[2], ps[3], ps[4], ps[5]);
    }
  };
  // Warp skew: when every warp reaches a unit's epilogue at once, the DMMA pipe idles for the
  // epilogue's duration (S1 / S2 of the matvec switch units every 9-16 k-tiles).  With skew L
  // the second half of the warps starts L k-tiles after the first (named barrier 1), so the two
  // halves' epilogues fall on each other's DMMA stream; the producer then runs only
  // STAGES-1-L k-tiles ahead so that refilling a stage never waits for the trailing half.
  const int skew = p.skew;
  const bool trail = skew > 0 && warp >= Cfg::kWarps / 2;
  unsigned char* const bres = smem + STAGES * STAGE_BYTES;   // B_RES: resident B k-tiles
  if (tid == kProdTid) {
    if constexpr (B_RES) {   // the whole B once (one N tile, ksplit 1, KT <= kBresMaxKT)
      mbar_expect_tx(&bres_bar, (uint32_t)(p.KT * Cfg::B_BYTES));
      for (int kt = 0; kt < p.KT; ++kt)
        tma_load_3d(bres + kt * Cfg::B_BYTES, &tmB, 0, kt * Cfg::BK, 0, &bres_bar, pol_b, p.l2_b != 0);
    }
    for (int s = 0; s < STAGES - 1 - skew; ++s) produce_one();
    prod_turn = 0;
  }
  if constexpr (RR) __syncthreads();   // the prologue's producer state is visible to every warp
  if (trail) asm volatile("bar.sync 1, %0;\n" ::"r"(Cfg::kThreads) : "memory");
  if constexpr (B_RES) mbar_wait(&bres_bar, 0);

  // ---- fragment geometry ---------------------------------------------------------------
  auto frag_row = [&](int i) -> int {   // tile row of fragment i, lane group g
    if (A_KC) return wm * WTM + i * 8 + 4 * (g & 1) + (g >> 1);
    if ((MI & 1) && i == MI - 1) return wm * WTM + (i >> 1) * 16 + g;
    return wm * WTM + (i >> 1) * 16 + 2 * g + (i & 1);
  };
  auto acc_col = [&](int j, int c) -> int {   // tile column of accumulator column c of fragment j
    if (B_KC) return wn * WTN + j * 8 + 4 * (c & 1) + (c >> 1);
    if ((NI & 1) && j == NI - 1) return wn * WTN + (j >> 1) * 16 + c;
    return wn * WTN + (j >> 1) * 16 + 2 * c + (j & 1);
  };
  // ---- per-lane shared-memory byte offsets (loop invariant) ------------------------------
  // K-contiguous tile, rows R0 + 8i + Rg (Rg = 4(g&1) + (g>>1)), k = kb + 2t:
  //   off = (R0 + Rg)*128 + ((t ^ Rg) << 4) + i*1024, and the kb = 8 half is off ^ 64.
  const int Rg = 4 * (g & 1) + (g >> 1);
  const int a_kc = (wm * WTM + Rg) * 128 + ((t ^ Rg) << 4);
  const int b_kc = (wn * WTN + Rg) * 128 + ((t ^ Rg) << 4);
  // M/N-contiguous tile of 16-wide boxes, k-row kb + 2t + s2, column m:
  //   off = (m >> 4)*2048 + (kb + 2t + s2)*128 + ((((m & 15) >> 1) ^ (2t + s2)) << 4) + (m & 1)*8
  // pair p of a warp tile starting at column C0 uses m = C0 + 16p + 2g (-> + p*2048).
  auto mn_off = [&](int m, int s2) -> int {
    const int k = 2 * t + s2;
    return (m >> 4) * 2048 + k * 128 + ((((m & 15) >> 1) ^ k) << 4) + (m & 1) * 8;
  };
  const int a_mn0 = mn_off(wm * WTM + 2 * g, 0), a_mn1 = mn_off(wm * WTM + 2 * g, 1);
  const int b_mn0 = mn_off(wn * WTN + 2 * g, 0), b_mn1 = mn_off(wn * WTN + 2 * g, 1);
  const int a_lo0 = mn_off(wm * WTM + (MI / 2) * 16 + g, 0), a_lo1 = mn_off(wm * WTM + (MI / 2) * 16 + g, 1);
  const int b_lo0 = mn_off(wn * WTN + (NI / 2) * 16 + g, 0), b_lo1 = mn_off(wn * WTN + (NI / 2) * 16 + g, 1);

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  int c_u = blockIdx.x, c_m0 = 0, c_n0 = 0, c_kt = 0, c_ke = 0, c_split = 0;
  if (c_u < p.total_units) unit_of(c_u, c_m0, c_n0, c_kt, c_ke, c_split);
  if (c_u + (int)gridDim.x >= p.total_units) pdl_trigger();
  uint32_t q = 0;
#pragma unroll 1
  while (c_u < p.total_units) {
    const int s = (int)(q % STAGES);
    mbar_wait(&full_bar[s], (q / STAGES) & 1);
    const unsigned char* as = smem + s * STAGE_BYTES;
    const unsigned char* bs = B_RES ? bres + c_kt * Cfg::B_BYTES : as + A_BYTES;
#pragma unroll
    for (int kp = 0; kp < 2; ++kp) {   // two pairs of DMMA k-steps per 16-deep k-tile
      // K-contiguous operands: one LDS.128 yields both k-steps of the pair
      double akc[A_KC ? 2 : 1][A_KC ? MI : 1], bkc[B_KC ? 2 : 1][B_KC ? NI : 1];
      if (A_KC) {
        const unsigned char* base = as + (kp ? (a_kc ^ 64) : a_kc);
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const double2 v = *reinterpret_cast<const double2*>(base + i * 1024);
          akc[0][i] = v.x;
          akc[A_KC ? 1 : 0][i] = v.y;
        }
      }
      if (B_KC) {
        const unsigned char* base = bs + (kp ? (b_kc ^ 64) : b_kc);
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const double2 v = *reinterpret_cast<const double2*>(base + j * 1024);
          bkc[0][j] = v.x;
          bkc[B_KC ? 1 : 0][j] = v.y;
        }
      }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        // M/N-contiguous operands: loaded per k-step (fewer live registers)
        double af[MI], bf[NI];
        if (A_KC) {
#pragma unroll
          for (int i = 0; i < MI; ++i) af[i] = akc[A_KC ? s2 : 0][i];
        } else {
          const unsigned char* base = as + (s2 ? a_mn1 : a_mn0) + kp * 1024;
#pragma unroll
          for (int pr = 0; pr < MI / 2; ++pr) {
            const double2 v = *reinterpret_cast<const double2*>(base + pr * 2048);
            af[2 * pr] = v.x;
            af[2 * pr + 1] = v.y;
          }
          if (MI & 1) af[MI - 1] = *reinterpret_cast<const double*>(as + (s2 ? a_lo1 : a_lo0) + kp * 1024);
        }
        if (B_KC) {
#pragma unroll
          for (int j = 0; j < NI; ++j) bf[j] = bkc[B_KC ? s2 : 0][j];
        } else {
          const unsigned char* base = bs + (s2 ? b_mn1 : b_mn0) + kp * 1024;
#pragma unroll
          for (int q2 = 0; q2 < NI / 2; ++q2) {
            const double2 v = *reinterpret_cast<const double2*>(base + q2 * 2048);
            bf[2 * q2] = v.x;
            bf[2 * q2 + 1] = v.y;
          }
          if (NI & 1) bf[NI - 1] = *reinterpret_cast<const double*>(bs + (s2 ? b_lo1 : b_lo0) + kp * 1024);
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma_8x8x4_nv(acc[i][j], af[i], bf[j]);
      }
    }
    // release the stage (one arrival per warp), then thread 0 refills the stream
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
    if constexpr (RR) {
      if (lane == 0 && (int)(q % Cfg::kWarps) == warp) {
        while (prod_turn != (int)q) {
        }
        __threadfence_block();
        produce_one();
        __threadfence_block();
        prod_turn = (int)q + 1;
      }
    } else {
      if (tid == 0) produce_one();
    }
    __syncwarp();
    ++q;
    if (skew > 0 && !trail && q == (uint32_t)skew)
      asm volatile("bar.arrive 1, %0;\n" ::"r"(Cfg::kThreads) : "memory");

    if (++c_kt == c_ke) {
      // ---- epilogue of unit c_u (registers -> global) --------------------------------
      if (p.dbg & 1) {
        double sink = 0.0;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) sink += acc[i][j][0] + acc[i][j][1];
        if (sink == 1.2345e-300) p.C[0] = sink;
      } else if (p.ksplit == 1 && !B_KC && p.store_mode == 3 && NI % 2 == 0 && WTN % 16 == 0) {
        // lane t holds output columns 4t..4t+3 of every 16-column group (fragments 2q, 2q+1,
        // both accumulator halves): one 32-byte store per row and group (full sectors)
        long long roff[MI];
        bool rok[MI];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int r = c_m0 + frag_row(i);
          rok[i] = r < p.M;
          roff[i] = rok[i] ? apply_map32(p.rowmap, (uint32_t)r) : 0;
        }
#pragma unroll
        for (int j = 0; j < NI; j += 2) {
          const int c = c_n0 + acc_col(j, 2 * t);
          if (c < p.N) {
            const long long co = col_off(c);
#pragma unroll
            for (int i = 0; i < MI; ++i)
              if (rok[i])
                stg_cs4(p.C + roff[i] + co, acc[i][j][0], acc[i][j + 1][0], acc[i][j][1],
                        acc[i][j + 1][1]);
          }
        }
      } else if (p.ksplit == 1 && !B_KC && (p.store_mode == 1 || p.store_mode == 3)) {
        // fragments 2q and 2q+1 hold adjacent output columns: one 16-byte store per pair
        long long roff[MI];
        bool rok[MI];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int r = c_m0 + frag_row(i);
          rok[i] = r < p.M;
          roff[i] = rok[i] ? apply_map32(p.rowmap, (uint32_t)r) : 0;
        }
#pragma unroll
        for (int j = 0; j + 1 < NI; j += 2)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = c_n0 + acc_col(j, 2 * t + h);
            if (c < p.N) {
              const long long co = col_off(c);
#pragma unroll
              for (int i = 0; i < MI; ++i)
                if (rok[i]) stg_cs2(p.C + roff[i] + co, acc[i][j][h], acc[i][j + 1][h]);
            }
          }
        if (NI & 1) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = c_n0 + acc_col(NI - 1, 2 * t + h);
            if (c < p.N) {
              const long long co = col_off(c);
#pragma unroll
              for (int i = 0; i < MI; ++i)
                if (rok[i]) stg_cs(p.C + roff[i] + co, acc[i][NI - 1][h]);
            }
          }
        }
      } else if (p.ksplit == 1 && !A_KC && p.store_mode == 2) {
        // fragments 2p and 2p+1 hold adjacent output rows: one 16-byte store per pair
        constexpr int MP = MI / 2;
        long long rpo[MP > 0 ? MP : 1];
        bool rpk[MP > 0 ? MP : 1];
#pragma unroll
        for (int ip = 0; ip < MP; ++ip) {
          const int r = c_m0 + frag_row(2 * ip);
          rpk[ip] = r < p.M;
          rpo[ip] = rpk[ip] ? apply_map32(p.rowmap, (uint32_t)r) : 0;
        }
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = c_n0 + acc_col(j, 2 * t + h);
            if (c < p.N) {
              const long long co = col_off(c);
#pragma unroll
              for (int ip = 0; ip < MP; ++ip)
                if (rpk[ip]) stg_cs2(p.C + rpo[ip] + co, acc[2 * ip][j][h], acc[2 * ip + 1][j][h]);
            }
          }
        if (MI & 1) {
          const int r = c_m0 + frag_row(MI - 1);
          if (r < p.M) {
            const long long ro = apply_map32(p.rowmap, (uint32_t)r);
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int c = c_n0 + acc_col(j, 2 * t + h);
                if (c < p.N) stg_cs(p.C + ro + col_off(c), acc[MI - 1][j][h]);
              }
          }
        }
      } else if (p.ksplit == 1) {
        long long roff[MI];
        bool rok[MI];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int r = c_m0 + frag_row(i);
          rok[i] = r < p.M;
          roff[i] = rok[i] ? apply_map32(p.rowmap, (uint32_t)r) : 0;
        }
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = c_n0 + acc_col(j, 2 * t + h);
            if (c < p.N) {
              const long long co = col_off(c);
#pragma unroll
              for (int i = 0; i < MI; ++i)
                if (rok[i]) stg_cs(p.C + roff[i] + co, acc[i][j][h]);
            }
          }
      } else {
        double* P = p.P + (long long)c_split * p.M * p.N;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int r = c_m0 + frag_row(i);
          if (r < p.M) {
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int c = c_n0 + acc_col(j, 2 * t + h);
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
      if (c_u < p.total_units) unit_of(c_u, c_m0, c_n0, c_kt, c_ke, c_split);
      if (c_u < p.total_units && c_u + (int)gridDim.x >= p.total_units) pdl_trigger();
    }
  }
  if (skew > 0 && !trail && q < (uint32_t)skew)   // fewer k-tiles than the skew: release
    asm volatile("bar.arrive 1, %0;\n" ::"r"(Cfg::kThreads) : "memory");
  // drain: thread 0 may still owe nothing (every issued stage was consumed)
}

}  // namespace tt
