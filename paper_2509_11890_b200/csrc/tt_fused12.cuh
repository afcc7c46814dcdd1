// tt_fused12.cuh — the first two stages of the local matvec (the three-product
// evaluation of y = Phi_L x_1 A x_2 Phi_R applied to a core) in ONE kernel: the intermediate
//   T1(a', al, j, m, b) = sum_a Phi_L[a', al, a] X[a, j, m, b]                      (S1)
// of a tile never leaves shared memory; the kernel writes only
//   T2(a', m, i, be, b) = sum_{al, j} A[al, i, j, be] T1(a', al, j, m, b)           (S2)
// so the matvec's HBM traffic and workspace lose the T1 round trip.
//
// One unit = 4 left-bond indices a' x 16 right-bond indices b of one Krylov column m:
//   phase 1: T1 tile (4 al) x (4 j x 16 b), K = a, operands by TMA into a 5-deep mbarrier ring
//            (Phi_L rows K-contiguous, X tile as 4 swizzled 16 x 16 slabs, one per j);
//   hand-over: accumulators -> shared memory in the layout phase 2 reads as an M-contiguous
//            A operand (k-rows (al, j), 16 b contiguous, 128-byte swizzle);
//   phase 2: per a': T2 tile (16 b) x (4 be), K = 4 al, B = the prepared operator core
//            Ahat[(al j), (i be)] streamed through the same ring (k-tiles of 16 x 144).
// 12 warps in two groups of 6; a group owns two of the four a' in both phases, so the
// hand-over needs only a group-local named barrier.  The k-tile stream is continuous across
// phases and units (persistent CTAs, one per SM); the refill of the ring rotates over the 12
// consumer warps (template RR: warp q mod 12 issues the load that follows k-tile q, in stream
// order through a shared turn counter) -- with thread 0 of warp 0 as the only producer that
// warp's critical path set the pace of the whole CTA (7.15 ms against 6.80 ms at the config-5
// interior core, K = 32; a 13th producer warp, template PW: 6.84 ms at 128 registers).
// Probe variants kept for A/B: G = 1 (two 6-warp CTAs per SM), a start skew
// between the two groups, the barrier before the hand-over.
//
// Preconditions (host-checked in tt_fused.cu, else the three-stage path): n = 4, al <= 36,
// be <= 36 with 4 be a multiple of 16, b a multiple of 16, a even, 16-byte aligned bases.
#pragma once
#include "tt_gemm_v3.cuh"

namespace tt {

constexpr int kF12ABytes = 72 * 128;                       // Phi_L rows of one warp group
constexpr int kF12XBytes = 4 * 2048;                       // X tile: 4 slabs (j) of 16 k x 16 b
constexpr int kF12AhBytes = 9 * 2048;                      // phase-2 k-tile: 16 k x 144 columns
// T1 of one a': 9 k-tiles (144 k-rows) x 16 b, the 2 KB slabs 16 bytes apart so that the
// hand-over stores of fragment rows g and g + 1 (k-rows 16 apart) fall on different banks
constexpr int kF12T1Slab = 2048 + 16;
constexpr int kF12T1PerA = 9 * kF12T1Slab;
// G warp groups of 6 warps per CTA, each owning two a' of the unit: G = 2 is one 12-warp CTA
// per SM (4 a' per unit, X tile and Ahat k-tiles shared by the groups, 5 stages); G = 1 is two
// independent 6-warp CTAs per SM (2 a' per unit, own 4-stage rings: twice the X / Ahat reads
// from L2, but one CTA's hand-over and epilogue fall on the other's DMMA stream).
template <int G>
struct F12Cfg {
  static constexpr int kThreads = 192 * G, kWarps = 6 * G;
  static constexpr int kPhase1Bytes = G * kF12ABytes + kF12XBytes;
  static constexpr int kStageBytes = kPhase1Bytes > kF12AhBytes ? kPhase1Bytes : kF12AhBytes;
  static constexpr int kStages = G == 2 ? 5 : 4;
  static constexpr int kT1Bytes = 2 * G * kF12T1PerA;
  static constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + kT1Bytes + 1024;
};

struct Fused12Params {
  double* T2;        // (a, K, 4, be, b)
  int a, b, al, be, K;
  int nag, nbt;      // groups of 2 G a', tiles of 16 b
  int total_units;   // nag * nbt * K, a' group fastest
  int KT1, KT2;      // k-tiles of 16: ceil(a / 16), ceil(4 al / 16)
  FastDiv nag_div, nbt_div;
  int skew;          // k-tiles by which warp group 1 trails group 0 (0..2)
  int opt;           // bit 0: keep the barrier before the hand-over even when KT1 > stages
  int dbg;
  const int* gate;   // optional device flag: nonzero -> no-op
};

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void sts2(unsigned char* p, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(smem_u32(p)), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// PW: a 13th warp whose lane 0 is the TMA producer (G = 2 only), so that no consumer warp
// carries the refill on its critical path.
// RR: no producer warp; the refill rotates over the consumer warps (tt_gemm_v3.cuh RR).
template <int G, bool PW = false, bool RR = false>
__global__ void __launch_bounds__(192 * G + (PW ? 32 : 0), 3 - G)
fused_s12_kernel(const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ CUtensorMap tmA, const Fused12Params p) {
  using Cfg = F12Cfg<G>;
  constexpr int ST = Cfg::kStages, kF12StageBytes = Cfg::kStageBytes, kF12Threads = Cfg::kThreads;
  constexpr int kProdTid = PW ? kF12Threads : 0;   // the thread that issues the TMA loads
  __shared__ volatile int prod_turn;   // RR: the k-tile whose refill is due next
  constexpr int kF12Warps = Cfg::kWarps, kF12T1Bytes = Cfg::kT1Bytes;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[ST], empty_bar[ST];
  __shared__ int prod_state[6];   // u, ag, bt, m, kt, q
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* const t1s = smem + ST * kF12StageBytes;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int gm = G == 1 ? 0 : warp / 6, wl = warp - 6 * gm;   // warp group, warp within the group
  const int wr = wl >> 1, wc = wl & 1;           // phase 1: 3 x 2 warps of 24 rows x 32 columns
  const int wa = wl / 3, wn2 = wl - 3 * wa;      // phase 2: 2 (a') x 3 warps of 16 rows x 48 columns

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kF12Warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmL)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
  }
  // the k-rows of T1 past 4 al (the last phase-2 k-tile's padding) stay zero for the whole run
  static_assert(kF12T1Bytes % 16 == 0, "");
  for (int e = tid; e < kF12T1Bytes / 16; e += (int)blockDim.x)
    *reinterpret_cast<double2*>(t1s + 16 * e) = make_double2(0.0, 0.0);
  __syncthreads();
  pdl_wait();
  if (p.gate && *p.gate) return;

  auto decode = [&](int u, int& ag, int& bt, int& m) {
    const int rest = (int)fdiv((uint32_t)u, p.nag_div);
    ag = u - rest * p.nag;
    m = (int)fdiv((uint32_t)rest, p.nbt_div);
    bt = rest - m * p.nbt;
  };

  const uint64_t pol_keep = (RR ? lane == 0 : tid == kProdTid) ? l2_policy(1) : 0;   // Phi_L and Ahat: re-read by every unit
  const int KTU = p.KT1 + p.KT2;
  if (tid == kProdTid) {
    int* ps = prod_state;
    ps[0] = blockIdx.x;
    ps[4] = 0;
    ps[5] = 0;
    if (ps[0] < p.total_units) decode(ps[0], ps[1], ps[2], ps[3]);
  }
  auto produce_one = [&]() {   // thread 0: issue the next k-tile of the stream, if any
    int* ps = prod_state;
    if (ps[0] >= p.total_units) return;
    const uint32_t lq = (uint32_t)ps[5];
    const int s = (int)(lq % ST);
    if (lq >= (uint32_t)ST) mbar_wait(&empty_bar[s], ((lq / ST) - 1) & 1);
    unsigned char* st = smem + s * kF12StageBytes;
    const int kt = ps[4];
#ifdef TT_DEBUG_HOOKS
    if (p.opt & 4) {   // timing probe: no loads, the transaction count completed locally
      const uint32_t nbytes = kt < p.KT1 ? Cfg::kPhase1Bytes : kF12AhBytes;
      mbar_expect_tx(&full_bar[s], nbytes);
      asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&full_bar[s])),
                   "r"(nbytes)
                   : "memory");
    } else
#endif
    if (kt < p.KT1) {
      const int k0 = kt * 16, r0 = ps[1] * 2 * G * p.al;
      mbar_expect_tx(&full_bar[s], Cfg::kPhase1Bytes);
      tma_load_2d_hint(st, &tmL, k0, r0, &full_bar[s], pol_keep);
      if (G == 2) tma_load_2d_hint(st + kF12ABytes, &tmL, k0, r0 + 2 * p.al, &full_bar[s], pol_keep);
      tma_load_5d(st + G * kF12ABytes, &tmX, 0, k0, ps[2], 0, ps[3], &full_bar[s]);
    } else {
      mbar_expect_tx(&full_bar[s], kF12AhBytes);
      tma_load_3d(st, &tmA, 0, (kt - p.KT1) * 16, 0, &full_bar[s], pol_keep, true);
    }
    ps[5] = (int)(lq + 1);
    if (++ps[4] == KTU) {
      ps[4] = 0;
      ps[0] += gridDim.x;
      if (ps[0] < p.total_units) decode(ps[0], ps[1], ps[2], ps[3]);
    }
  };
  const int skew = G == 2 ? p.skew : 0;
  const bool trail = skew > 0 && gm == 1;
  if (PW) {
    if (warp == kF12Warps) {   // producer warp: runs as far ahead as the ring allows
      if (lane == 0)
        while (prod_state[0] < p.total_units) produce_one();
      return;
    }
  } else if (tid == 0) {
    for (int s = 0; s < ST - 1 - skew; ++s) produce_one();
    prod_turn = 0;
  }
  if (RR) __syncthreads();
  if (trail) bar_sync(3, kF12Threads);

  // ---- per-lane shared-memory byte offsets (tt_gemm_v3.cuh fragment geometry) ------------
  const int Rg = 4 * (g & 1) + (g >> 1);
  // phase 1 A (Phi_L rows, K-contiguous): group tile row wr*24 + 8 i + Rg
  const int a1_off = gm * kF12ABytes + (wr * 24 + Rg) * 128 + ((t ^ Rg) << 4);
  // M/N-contiguous slabs: k-row 2t + s2 of a 16 x 16 slab, columns 2g, 2g + 1
  const int mn0 = (2 * t) * 128 + ((g ^ (2 * t)) << 4);
  const int mn1 = (2 * t + 1) * 128 + ((g ^ (2 * t + 1)) << 4);
  // phase 1 B (X tile): slabs j = 2 wc + q;  phase 2 B (Ahat k-tile): slabs 3 wn2 + q
  const int x_off = G * kF12ABytes + wc * 2 * 2048;
  const int ah_off = wn2 * 3 * 2048;
  // phase 2 A: the T1 block of this warp's a' (= 2 gm + wa), one slab per k-tile
  const unsigned char* const t1a = t1s + (2 * gm + wa) * kF12T1PerA;

  const int NB = 4 * p.be;   // valid phase-2 columns (i, be)
  const bool pre_barrier = p.KT1 <= ST || (p.opt & 1);
  uint32_t q = 0;
  bool released = skew == 0 || gm == 1;
#pragma unroll 1
  for (int u = blockIdx.x; u < p.total_units; u += gridDim.x) {
    int ag, bt, m;
    decode(u, ag, bt, m);
    // ================= phase 1: T1 tile =================
    double acc[3][4][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 1
    for (int kt = 0; kt < p.KT1; ++kt) {
      const int s = (int)(q % ST);
      mbar_wait(&full_bar[s], (q / ST) & 1);
      const unsigned char* st = smem + s * kF12StageBytes;
#pragma unroll
      for (int kp = 0; kp < 2; ++kp) {
        double ak[2][3];
        {
          const unsigned char* base = st + (kp ? (a1_off ^ 64) : a1_off);
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const double2 v = *reinterpret_cast<const double2*>(base + i * 1024);
            ak[0][i] = v.x;
            ak[1][i] = v.y;
          }
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          double bf[4];
          const unsigned char* base = st + x_off + (s2 ? mn1 : mn0) + kp * 1024;
#pragma unroll
          for (int q2 = 0; q2 < 2; ++q2) {
            const double2 v = *reinterpret_cast<const double2*>(base + q2 * 2048);
            bf[2 * q2] = v.x;
            bf[2 * q2 + 1] = v.y;
          }
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_8x8x4_nv(acc[i][j], ak[s2][i], bf[j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
      if (RR) {
        if (lane == 0 && (int)(q % kF12Warps) == warp) {
          while (prod_turn != (int)q) {
          }
          __threadfence_block();
          produce_one();
          __threadfence_block();
          prod_turn = (int)q + 1;
        }
      } else if (!PW && tid == 0) {
        produce_one();
      }
      __syncwarp();
      ++q;
      if (!released && q == (uint32_t)skew) {
        bar_arrive(3, kF12Threads);
        released = true;
      }
    }
    // ================= hand-over: accumulators -> T1 in shared memory =================
    // Every warp of the group has finished reading the previous unit's T1: with KT1 > ST the
    // ring guarantees it (the load of this unit's last phase-1 k-tile was issued only after
    // all 12 warps released a stage of this unit's phase 1), otherwise a barrier does.
    if (pre_barrier) bar_sync(1 + gm, 192);
#ifdef TT_DEBUG_HOOKS
    if (!(p.opt & 16))   // timing probe: no hand-over stores
#endif
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int lr = wr * 24 + 8 * i + Rg;           // Phi_L row within the group: (a', al)
      const int ain = lr >= p.al ? 1 : 0;
      const int alv = lr - ain * p.al;
      if (alv < p.al) {                              // rows past 2 al belong to other groups
        unsigned char* rowp = t1s + (2 * gm + ain) * kF12T1PerA;
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
          const int k2 = alv * 4 + 2 * wc + q2;      // phase-2 k-row (al, j)
          unsigned char* kp = rowp + (k2 >> 4) * kF12T1Slab + (k2 & 15) * 128;
          const int key = k2 & 7;
          // this lane's columns 4t .. 4t + 3 of the 16 b: chunks 2t and 2t + 1
          sts2(kp + (((2 * t) ^ key) << 4), acc[i][2 * q2][0], acc[i][2 * q2 + 1][0]);
          sts2(kp + (((2 * t + 1) ^ key) << 4), acc[i][2 * q2][1], acc[i][2 * q2 + 1][1]);
        }
      }
    }
    bar_sync(1 + gm, 192);
    // ================= phase 2: T2 tile of this warp's a' =================
    double ac2[2][6][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 6; ++j) ac2[i][j][0] = ac2[i][j][1] = 0.0;
#pragma unroll 1
    for (int kt = 0; kt < p.KT2; ++kt) {
      const int s = (int)(q % ST);
      mbar_wait(&full_bar[s], (q / ST) & 1);
      const unsigned char* bs = smem + s * kF12StageBytes + ah_off;
      const unsigned char* as = t1a + kt * kF12T1Slab;
#pragma unroll
      for (int kp = 0; kp < 2; ++kp) {
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          const int mo = (s2 ? mn1 : mn0) + kp * 1024;
          const double2 av = *reinterpret_cast<const double2*>(as + mo);
          double bf[6];
#pragma unroll
          for (int q2 = 0; q2 < 3; ++q2) {
            const double2 v = *reinterpret_cast<const double2*>(bs + mo + q2 * 2048);
            bf[2 * q2] = v.x;
            bf[2 * q2 + 1] = v.y;
          }
#pragma unroll
          for (int j = 0; j < 6; ++j) {
            dmma_8x8x4_nv(ac2[0][j], av.x, bf[j]);
            dmma_8x8x4_nv(ac2[1][j], av.y, bf[j]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
      if (RR) {
        if (lane == 0 && (int)(q % kF12Warps) == warp) {
          while (prod_turn != (int)q) {
          }
          __threadfence_block();
          produce_one();
          __threadfence_block();
          prod_turn = (int)q + 1;
        }
      } else if (!PW && tid == 0) {
        produce_one();
      }
      __syncwarp();
      ++q;
      if (!released && q == (uint32_t)skew) {
        bar_arrive(3, kF12Threads);
        released = true;
      }
    }
    // ================= epilogue: T2(a', m, i, be, b0 + 2g .. 2g + 1) =================
    const int ap = ag * 2 * G + 2 * gm + wa;
#ifdef TT_DEBUG_HOOKS
    if (p.opt & 8) {   // timing probe: no T2 stores (accumulators kept live)
      double sink = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) sink += ac2[0][j][0] + ac2[0][j][1] + ac2[1][j][0] + ac2[1][j][1];
      if (sink == 1.2345e-300) p.T2[0] = sink;
    } else
#endif
    if (ap < p.a) {
      double* rowp = p.T2 + ((long long)ap * p.K + m) * ((long long)NB * p.b) + bt * 16 + 2 * g;
#pragma unroll
      for (int j = 0; j < 6; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = wn2 * 48 + (j >> 1) * 16 + 2 * (2 * t + h) + (j & 1);   // (i, be)
          if (c < NB) stg_cs2(rowp + (long long)c * p.b, ac2[0][j][h], ac2[1][j][h]);
        }
    }
  }
  if (!released) bar_arrive(3, kF12Threads);
  pdl_trigger();
}

}  // namespace tt
