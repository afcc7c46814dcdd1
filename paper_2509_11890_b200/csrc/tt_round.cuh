// tt_round.cuh — TT rounding on the GPU.
//
// Oseledets' TT-rounding (right-to-left orthonormalisation -- cluster Householder QR,
// tt_qr.cuh -- then left-to-right truncated SVD).  This header holds the Gram route of the
// truncating SVDs (and of orthonormalisations too large for one cluster):
//   G = M^T M (a DMMA GEMM of the engine) = V diag(sigma^2) V^T   (parallel Jacobi
//   eigensolver on all SMs, cooperative launch), U = M V diag(1/sigma) (a GEMM).
// Exactly rank-deficient unfoldings (e.g. the formal sum T + T) are handled: zero singular
// values are dropped.  The truncation decisions are data dependent: tt_round reads the
// singular values of every core on the host (one synchronisation per core), tt_round_async
// takes them on the device (trunc_decide_kernel, tt_solvers.cu).
// Kernels: jacobi_coop_kernel (element-wise, n < 24), jacobi_block2_kernel (block Jacobi,
// the default), jacobi_block_coop_kernel (the first block kernel, kept for A/B).
// Included by tt_solvers.cu inside namespace ttint.

// Multi-CTA parallel Jacobi (cooperative launch, one grid barrier per step).  The n x n
// matrix is embedded in an np x np one (np even; a dummy isolated index if n is odd) and
// ping-ponged between two buffers: in every step each CTA recomputes the np/2 rotation angles
// of the round-robin pairs from the current buffer (cheap) and writes its share of the
// updated matrix, J^T G J, as 2x2 blocks (row pair, column pair), and of V J, into the other
// buffer, so no CTA ever reads what another writes within a step.  Convergence (off-diagonal
// Frobenius mass <= 1e-26 of the diagonal mass) is decided identically by every CTA from
// per-CTA partial sums added in a fixed order (deterministic).
__global__ void __launch_bounds__(256) jacobi_coop_kernel(double* __restrict__ G0,
                                                          double* __restrict__ G1,
                                                          double* __restrict__ V0,
                                                          double* __restrict__ V1, int np,
                                                          int sweeps, double* __restrict__ part,
                                                          int* __restrict__ result_buf) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  extern __shared__ double sh[];
  double* cs = sh;                 // [np/2]
  double* sn = sh + np / 2;        // [np/2]
  int* pp = reinterpret_cast<int*>(sn + np / 2);
  int* qq = pp + np / 2;
  __shared__ double red[16];
  const int tid = threadIdx.x, nt = blockDim.x, bid = blockIdx.x, nb = gridDim.x;
  const long long gt = (long long)bid * nt + tid, gstride = (long long)nb * nt;
  const long long NN = (long long)np * np;
  for (long long e = gt; e < NN; e += gstride) V0[e] = (e / np == e % np) ? 1.0 : 0.0;
  grid.sync();
  double *Gc = G0, *Gn = G1, *Vc = V0, *Vn = V1;
  int cur = 0;
  for (int sw = 0; sw < sweeps; ++sw) {
    double off = 0.0, dia = 0.0;
    for (long long e = gt; e < NN; e += gstride) {
      const double v = Gc[e];
      if (e / np == e % np) dia += v * v; else off += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_down_sync(0xffffffffu, off, o);
      dia += __shfl_down_sync(0xffffffffu, dia, o);
    }
    if ((tid & 31) == 0) {
      red[(tid >> 5) * 2] = off;
      red[(tid >> 5) * 2 + 1] = dia;
    }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < nt / 32; ++w) {
        a += red[2 * w];
        b += red[2 * w + 1];
      }
      part[2 * bid] = a;
      part[2 * bid + 1] = b;
    }
    grid.sync();
    double offs = 0.0, dias = 0.0;
    for (int c = 0; c < nb; ++c) {   // same fixed order in every thread of every CTA
      offs += part[2 * c];
      dias += part[2 * c + 1];
    }
    grid.sync();   // everyone has read `part` before it is rewritten next sweep
    if (offs <= 1e-26 * dias) break;
    for (int step = 0; step < np - 1; ++step) {
      for (int k = tid; k < np / 2; k += nt) {
        int a = (k == 0) ? 0 : 1 + (k - 1 + step) % (np - 1);
        int b = 1 + (np - 2 - k + step) % (np - 1);
        if (a > b) { const int t = a; a = b; b = t; }
        pp[k] = a;
        qq[k] = b;
        double c = 1.0, s = 0.0;
        const double apq = Gc[(long long)a * np + b];
        if (apq != 0.0) {
          const double app = Gc[(long long)a * np + a], aqq = Gc[(long long)b * np + b];
          const double tau = (aqq - app) / (2.0 * apq);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
        }
        cs[k] = c;
        sn[k] = s;
      }
      __syncthreads();
      const long long nblk = (long long)(np / 2) * (np / 2);
      for (long long e = gt; e < nblk; e += gstride) {   // 2x2 blocks of J^T G J
        const int kr = (int)(e / (np / 2)), kc = (int)(e - (long long)kr * (np / 2));
        const int p = pp[kr], q = qq[kr], u = pp[kc], w = qq[kc];
        const double cr = cs[kr], sr = sn[kr], cc = cs[kc], sc = sn[kc];
        const double gpu_ = Gc[(long long)p * np + u], gpw = Gc[(long long)p * np + w];
        const double gqu = Gc[(long long)q * np + u], gqw = Gc[(long long)q * np + w];
        // rows: (p, q) <- (c p - s q, s p + c q); then columns likewise
        const double rpu = cr * gpu_ - sr * gqu, rpw = cr * gpw - sr * gqw;
        const double rqu = sr * gpu_ + cr * gqu, rqw = sr * gpw + cr * gqw;
        Gn[(long long)p * np + u] = cc * rpu - sc * rpw;
        Gn[(long long)p * np + w] = sc * rpu + cc * rpw;
        Gn[(long long)q * np + u] = cc * rqu - sc * rqw;
        Gn[(long long)q * np + w] = sc * rqu + cc * rqw;
      }
      const long long nv = (long long)np * (np / 2);
      for (long long e = gt; e < nv; e += gstride) {      // V J: rows i, column pairs
        const int i = (int)(e / (np / 2)), kc = (int)(e - (long long)i * (np / 2));
        const int u = pp[kc], w = qq[kc];
        const double cc = cs[kc], sc = sn[kc];
        const double vu = Vc[(long long)i * np + u], vw = Vc[(long long)i * np + w];
        Vn[(long long)i * np + u] = cc * vu - sc * vw;
        Vn[(long long)i * np + w] = sc * vu + cc * vw;
      }
      grid.sync();
      double* t = Gc; Gc = Gn; Gn = t;
      t = Vc; Vc = Vn; Vn = t;
      cur ^= 1;
      __syncthreads();
    }
  }
  if (gt == 0) result_buf[0] = cur;   // which buffer holds the result
}

// Block Jacobi (cooperative launch): the np x np matrix (np a multiple of 2 BS) is split into
// 2m blocks of BS indices, paired round-robin.  In each step every pair (P, Q) of blocks is
// handled by one CTA, which runs one cyclic Jacobi sweep on its 2BS x 2BS diagonal block in
// shared memory and records the accumulated rotation R_PQ; after a grid barrier every
// 2BS x 2BS block of G is replaced by R_rows^T G_blk R_cols and every 2BS-row slab of V by
// V R (each block is owned by one task, so the update is in place); a second barrier ends the
// step.  2m - 1 steps per sweep: two grid barriers per BS-wide pair instead of one per index
// pair, i.e. ~BS/2 times fewer barriers than the element-wise kernel above.
constexpr int kJBS = 16, kJB2 = 2 * kJBS;
__global__ void __launch_bounds__(256) jacobi_block_coop_kernel(double* __restrict__ G,
                                                                double* __restrict__ V, int np,
                                                                int sweeps,
                                                                double* __restrict__ Rbuf,
                                                                double* __restrict__ part) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ double S[kJB2][kJB2 + 1];
  __shared__ double R[kJB2][kJB2 + 1];
  __shared__ double T[kJB2][kJB2 + 1];
  __shared__ double cs[kJBS], sn[kJBS];
  __shared__ int pp[kJBS], qq[kJBS];
  __shared__ double red[16];
  __shared__ int pb[2];
  const int tid = threadIdx.x, nt = blockDim.x, bid = blockIdx.x, nb = gridDim.x;
  const int nblk = np / kJBS, m = nblk / 2;
  const long long gt = (long long)bid * nt + tid, gstride = (long long)nb * nt;
  const long long NN = (long long)np * np;
  for (long long e = gt; e < NN; e += gstride) V[e] = (e / np == e % np) ? 1.0 : 0.0;
  grid.sync();
  int extra = 0;
  auto pair_of = [&](int k, int step, int& a, int& b) {   // round-robin over nblk blocks
    a = (k == 0) ? 0 : 1 + (k - 1 + step) % (nblk - 1);
    b = 1 + (nblk - 2 - k + step) % (nblk - 1);
    if (a > b) { const int t = a; a = b; b = t; }
  };
  for (int sw = 0; sw < sweeps; ++sw) {
    double off = 0.0, dia = 0.0;
    for (long long e = gt; e < NN; e += gstride) {
      const double v = G[e];
      if (e / np == e % np) dia += v * v; else off += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_down_sync(0xffffffffu, off, o);
      dia += __shfl_down_sync(0xffffffffu, dia, o);
    }
    if ((tid & 31) == 0) {
      red[(tid >> 5) * 2] = off;
      red[(tid >> 5) * 2 + 1] = dia;
    }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < nt / 32; ++w) {
        a += red[2 * w];
        b += red[2 * w + 1];
      }
      part[2 * bid] = a;
      part[2 * bid + 1] = b;
    }
    grid.sync();
    double offs = 0.0, dias = 0.0;
    for (int c = 0; c < nb; ++c) {
      offs += part[2 * c];
      dias += part[2 * c + 1];
    }
    grid.sync();
    // below 1e-13 relative off-diagonal mass, two more sweeps: the one-sweep inner solves
    // converge more slowly than the element-wise kernel, and eigenvectors of eigenvalues
    // ~1e-6 of the largest need the off-diagonal mass near the rounding floor
    if (offs <= 1e-26 * dias && ++extra > 2) break;
    for (int step = 0; step < nblk - 1; ++step) {
      // ---- phase A: one inner Jacobi sweep per block pair -> R_PQ ----
      for (int k = bid; k < m; k += nb) {
        if (tid == 0) pair_of(k, step, pb[0], pb[1]);
        __syncthreads();
        const int P = pb[0], Q = pb[1];
        for (int e = tid; e < kJB2 * kJB2; e += nt) {
          const int i = e / kJB2, j = e % kJB2;
          const int gi = (i < kJBS ? P * kJBS + i : Q * kJBS + i - kJBS);
          const int gj = (j < kJBS ? P * kJBS + j : Q * kJBS + j - kJBS);
          S[i][j] = G[(long long)gi * np + gj];
          R[i][j] = (i == j) ? 1.0 : 0.0;
        }
        __syncthreads();
        for (int st = 0; st < kJB2 - 1; ++st) {
          if (tid < kJBS) {
            int a = (tid == 0) ? 0 : 1 + (tid - 1 + st) % (kJB2 - 1);
            int b = 1 + (kJB2 - 2 - tid + st) % (kJB2 - 1);
            if (a > b) { const int t = a; a = b; b = t; }
            pp[tid] = a;
            qq[tid] = b;
            double c = 1.0, sv = 0.0;
            const double apq = S[a][b], app = S[a][a], aqq = S[b][b];
            if (fabs(apq) > 1e-300) {
              const double tau = (aqq - app) / (2.0 * apq);
              const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
              c = 1.0 / sqrt(1.0 + t * t);
              sv = t * c;
            }
            cs[tid] = c;
            sn[tid] = sv;
          }
          __syncthreads();
          for (int e = tid; e < kJBS * kJBS; e += nt) {   // 2x2 blocks of J^T S J (in place)
            const int kr = e / kJBS, kc = e % kJBS;
            const int p = pp[kr], q = qq[kr], u = pp[kc], w = qq[kc];
            const double cr = cs[kr], sr = sn[kr], cc = cs[kc], sc = sn[kc];
            const double mpu = S[p][u], mpw = S[p][w], mqu = S[q][u], mqw = S[q][w];
            const double rpu = cr * mpu - sr * mqu, rpw = cr * mpw - sr * mqw;
            const double rqu = sr * mpu + cr * mqu, rqw = sr * mpw + cr * mqw;
            S[p][u] = cc * rpu - sc * rpw;
            S[p][w] = sc * rpu + cc * rpw;
            S[q][u] = cc * rqu - sc * rqw;
            S[q][w] = sc * rqu + cc * rqw;
          }
          for (int e = tid; e < kJB2 * kJBS; e += nt) {   // R <- R J
            const int i = e / kJBS, kc = e % kJBS;
            const int u = pp[kc], w = qq[kc];
            const double ru = R[i][u], rw = R[i][w];
            R[i][u] = cs[kc] * ru - sn[kc] * rw;
            R[i][w] = sn[kc] * ru + cs[kc] * rw;
          }
          __syncthreads();
        }
        double* Rg = Rbuf + (long long)k * kJB2 * kJB2;
        for (int e = tid; e < kJB2 * kJB2; e += nt) Rg[e] = R[e / kJB2][e % kJB2];
        __syncthreads();
      }
      grid.sync();
      // ---- phase B: G[PQ, RS] <- R_PQ^T G[PQ, RS] R_RS;  V[rows, PQ] <- V[rows, PQ] R_PQ ----
      const int gtasks = m * m, vtasks = (np / kJB2) * m;
      for (int task = bid; task < gtasks + vtasks; task += nb) {
        const bool isG = task < gtasks;
        const int t2 = isG ? task : task - gtasks;
        const int kr = isG ? t2 / m : -1, kc = t2 % m;
        const int rb = isG ? -1 : t2 / m;   // V row slab
        if (tid == 0) {
          int a, b;
          pair_of(kc, step, a, b);
          pb[0] = a * 32768 + b;   // column pair
          if (isG) {
            pair_of(kr, step, a, b);
            pb[1] = a * 32768 + b;
          }
        }
        __syncthreads();
        const int Pc = pb[0] / 32768, Qc = pb[0] % 32768;
        const int Pr = isG ? pb[1] / 32768 : 0, Qr = isG ? pb[1] % 32768 : 0;
        const double* Rc = Rbuf + (long long)kc * kJB2 * kJB2;
        for (int e = tid; e < kJB2 * kJB2; e += nt) {
          const int i = e / kJB2, j = e % kJB2;
          const int gj = (j < kJBS ? Pc * kJBS + j : Qc * kJBS + j - kJBS);
          int gi;
          if (isG) gi = (i < kJBS ? Pr * kJBS + i : Qr * kJBS + i - kJBS);
          else gi = rb * kJB2 + i;
          S[i][j] = isG ? G[(long long)gi * np + gj] : V[(long long)gi * np + gj];
          R[i][j] = Rc[e];
        }
        __syncthreads();
        // T = S R_cols
        for (int e = tid; e < kJB2 * kJB2; e += nt) {
          const int i = e / kJB2, j = e % kJB2;
          double v = 0.0;
#pragma unroll 8
          for (int q = 0; q < kJB2; ++q) v = fma(S[i][q], R[q][j], v);
          T[i][j] = v;
        }
        __syncthreads();
        if (isG) {   // S = R_rows^T T
          const double* Rr = Rbuf + (long long)kr * kJB2 * kJB2;
          for (int e = tid; e < kJB2 * kJB2; e += nt) R[e / kJB2][e % kJB2] = Rr[e];
          __syncthreads();
          for (int e = tid; e < kJB2 * kJB2; e += nt) {
            const int i = e / kJB2, j = e % kJB2;
            double v = 0.0;
#pragma unroll 8
            for (int q = 0; q < kJB2; ++q) v = fma(R[q][i], T[q][j], v);
            S[i][j] = v;
          }
          __syncthreads();
        }
        double (*Out)[kJB2 + 1] = isG ? S : T;
        for (int e = tid; e < kJB2 * kJB2; e += nt) {
          const int i = e / kJB2, j = e % kJB2;
          const int gj = (j < kJBS ? Pc * kJBS + j : Qc * kJBS + j - kJBS);
          if (isG) {
            const int gi = (i < kJBS ? Pr * kJBS + i : Qr * kJBS + i - kJBS);
            G[(long long)gi * np + gj] = Out[i][j];
          } else {
            V[(long long)(rb * kJB2 + i) * np + gj] = Out[i][j];
          }
        }
        __syncthreads();
      }
      grid.sync();
    }
  }
}

// Block Jacobi, second version (the default): the same block pairing and barriers as
// jacobi_block_coop_kernel, with
//  * cross-pair inner sweeps: only the first block step of a sweep rotates the pairs inside a
//    block (every block belongs to exactly one pair there, so each index pair of the matrix is
//    still rotated exactly once per sweep); the other 2m - 2 steps rotate only the BS x BS
//    cross pairs (p in P, q in Q) in BS inner steps of BS disjoint rotations instead of
//    2BS - 1.  A sweep is then 2BS - 1 + (2m - 2) BS ~ n inner steps for ANY block size, so
//    the block size only sets the number of block steps (two grid barriers and one update
//    round trip each): BS = 32 (64 x 64 diagonal problems, 512 threads) halves them;
//  * rotations from two reciprocal square roots (jb2_rotation);
//  * the 2BS x 2BS x 2BS products of the update phase on the FP64 tensor cores (DMMA.8x8x4;
//    the scalar version made n >= 512 shared-memory bound), all three operands of a task
//    loaded in one round trip, T = S R_cols written over S for the second product.
// Dynamic shared memory: 3 (2BS)(2BS + 4) doubles.
__device__ __forceinline__ void jb2_rotation(double app, double aqq, double apq, double& c,
                                             double& s) {
  // (c, s) annihilating apq, |theta| <= pi/4, without the textbook three divisions and two
  // square roots (a ~1500-cycle dependent chain that bounded the inner sweeps): with
  // d = aqq - app, h = 2 apq, r = hypot(d, h): cos 2theta = |d| / r,
  // c = sqrt((1 + cos 2theta) / 2), s = sign(d) h / (2 r c) -- no cancellation in either.
  // d and h are scaled by a power of two first (exact), so the squares neither overflow nor
  // underflow.
  c = 1.0;
  s = 0.0;
  double d = aqq - app, h = 2.0 * apq;
  const double mx = fmax(fabs(d), fabs(h));
  if (!(fabs(apq) > 1e-300) || !(mx < 1.7e308)) return;
  const int ex = min(max((__double2hiint(mx) >> 20) & 0x7ff, 2), 2044);   // biased exponent
  const double sc = __hiloint2double((2046 - ex) << 20, 0);               // 2^(1023 - ex)
  d *= sc;
  h *= sc;
  const double rinv = rsqrt(d * d + h * h);
  const double c2 = 0.5 + 0.5 * (fabs(d) * rinv);
  const double cinv = rsqrt(c2);
  c = c2 * cinv;
  s = (d >= 0.0 ? 0.5 : -0.5) * (h * rinv) * cinv;
}
__device__ __forceinline__ void jb2_dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
template <int BS>
struct Jb2 {
  static constexpr int B2 = 2 * BS, LD = B2 + 1;        // odd stride: the inner sweeps' accesses
  static constexpr int LDB = B2 + 4;                    // update phase: conflict-free DMMA fragments
  static constexpr int kThreads = BS * 16;              // update warps: 256 / 512 threads
  static constexpr int kLaunch = kThreads + 32;         // + the rotation warp of the inner sweeps
  static constexpr int kRowTiles = B2 / 8;              // 8-row DMMA tiles of a block
  static constexpr int kNT = B2 / 16;                   // 8-column tiles per warp (half a block)
  static constexpr size_t kSmem = 3 * (size_t)B2 * LDB * sizeof(double);
};
template <int BS>
__global__ void __launch_bounds__(Jb2<BS>::kLaunch) jacobi_block2_kernel(
    double* __restrict__ G, double* __restrict__ V, int np, int sweeps,
    double* __restrict__ Rbuf, double* __restrict__ part) {
  using C = Jb2<BS>;
  constexpr int B2 = C::B2, LD = C::LD, NTL = C::kNT;
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  extern __shared__ double jsm[];
  constexpr int LDB = C::LDB;
  double (*S)[LD] = reinterpret_cast<double (*)[LD]>(jsm);
  double (*R)[LD] = reinterpret_cast<double (*)[LD]>(jsm + B2 * LDB);
  double (*R2)[LD] = reinterpret_cast<double (*)[LD]>(jsm + 2 * B2 * LDB);
  double (*Sb)[LDB] = reinterpret_cast<double (*)[LDB]>(jsm);               // update-phase views
  double (*Rb)[LDB] = reinterpret_cast<double (*)[LDB]>(jsm + B2 * LDB);
  double (*R2b)[LDB] = reinterpret_cast<double (*)[LDB]>(jsm + 2 * B2 * LDB);
  __shared__ double cs[2][BS], sn[2][BS];
  __shared__ int pp[2][BS], qq[2][BS], pos[2][B2];
  __shared__ double red[2 * C::kLaunch / 32];
  __shared__ int pb[2];
  const int tid = threadIdx.x, nt = blockDim.x, bid = blockIdx.x, nb = gridDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nblk = np / BS, m = nblk / 2;
  const long long gt = (long long)bid * nt + tid, gstride = (long long)nb * nt;
  const long long NN = (long long)np * np;
  for (long long e = gt; e < NN; e += gstride) V[e] = (e / np == e % np) ? 1.0 : 0.0;
  // rot_ready[k] = number of the last block step whose rotation R_k is in Rbuf: the update
  // tasks wait for the two rotations they need instead of a grid barrier after phase A
  int* rot_ready = reinterpret_cast<int*>(part + 4096);
  if (bid == 0)
    for (int k = tid; k < m; k += nt) rot_ready[k] = 0;
  int gstep = 0;
  // (only while every CTA has at most one update task: with several per CTA -- n >= 1024 --
  // the per-task wait costs more than the barrier it replaces: 27.1 -> 29.7 ms measured)
  const bool use_flags = 2 * m * m <= nb;
  grid.sync();
  int extra = 0;
  auto pair_of = [&](int k, int step, int& a, int& b) {   // round-robin over nblk blocks
    if (nblk == 2) { a = 0; b = 1; return; }
    a = (k == 0) ? 0 : 1 + (k - 1 + step) % (nblk - 1);
    b = 1 + (nblk - 2 - k + step) % (nblk - 1);
    if (a > b) { const int t = a; a = b; b = t; }
  };
  // fragment coordinates of this warp's 8 x BS slice of a 2BS x 2BS product
  const int half = warp / C::kRowTiles;                 // 0: columns of P, 1: columns of Q
  const int fr = 8 * (warp % C::kRowTiles) + (lane >> 2), fk = lane & 3;
  const int fc = BS * half + (lane >> 2), oc = BS * half + 2 * (lane & 3);
  for (int sw = 0; sw < sweeps; ++sw) {
    double off = 0.0, dia = 0.0;
    for (long long e = gt; e < NN; e += gstride) {
      const double v = G[e];
      if (e / np == e % np) dia += v * v; else off += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_down_sync(0xffffffffu, off, o);
      dia += __shfl_down_sync(0xffffffffu, dia, o);
    }
    if (lane == 0) {
      red[warp * 2] = off;
      red[warp * 2 + 1] = dia;
    }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < nt / 32; ++w) {
        a += red[2 * w];
        b += red[2 * w + 1];
      }
      part[2 * bid] = a;
      part[2 * bid + 1] = b;
    }
    grid.sync();
    double offs = 0.0, dias = 0.0;
    for (int c = 0; c < nb; ++c) {
      offs += part[2 * c];
      dias += part[2 * c + 1];
    }
    grid.sync();
    if (offs <= 1e-26 * dias && ++extra > 1) break;   // one more sweep after the test passes (the first kernel: two; none: residual 3.5x larger)
    for (int step = 0; step < nblk - 1; ++step) {
      // ---- phase A: one inner Jacobi sweep per block pair -> R_PQ ----
      const bool full = (step == 0);
      const int isteps = full ? B2 - 1 : BS;
      for (int k = bid; k < m; k += nb) {
        if (tid == 0) pair_of(k, step, pb[0], pb[1]);
        __syncthreads();
        const int P = pb[0], Q = pb[1];
        for (int e = tid; e < B2 * B2; e += nt) {
          const int i = e / B2, j = e % B2;
          const int gi = (i < BS ? P * BS + i : Q * BS + i - BS);
          const int gj = (j < BS ? P * BS + j : Q * BS + j - BS);
          S[i][j] = G[(long long)gi * np + gj];
          R[i][j] = (i == j) ? 1.0 : 0.0;
        }
        __syncthreads();
        // Inner sweep, software-pipelined: while the update warps apply step st (S_nxt =
        // J^T S_cur J into the other buffer, R <- R J), the rotation warp already computes the
        // rotations of step st + 1 -- the three entries each needs are transformed from S_cur
        // with the very expressions of the update -- so a step costs one barrier and
        // max(update, rotation) instead of their sum plus two barriers.
        double (*Sc)[LD] = S;
        double (*Sn)[LD] = R2;
        const bool rotw = warp == C::kThreads / 32;
        auto pair_at = [&](int st, int i, int& a, int& b) {
          if (full) {
            a = (i == 0) ? 0 : 1 + (i - 1 + st) % (B2 - 1);
            b = 1 + (B2 - 2 - i + st) % (B2 - 1);
            if (a > b) { const int t = a; a = b; b = t; }
          } else {
            a = i;
            b = BS + ((i + st) & (BS - 1));
          }
        };
        if (rotw && lane < BS) {
          int a, b;
          pair_at(0, lane, a, b);
          pp[0][lane] = a;
          qq[0][lane] = b;
          pos[0][a] = 2 * lane;
          pos[0][b] = 2 * lane + 1;
          double c, sv;
          jb2_rotation(Sc[a][a], Sc[b][b], Sc[a][b], c, sv);
          cs[0][lane] = c;
          sn[0][lane] = sv;
        }
        __syncthreads();
        for (int st = 0; st < isteps; ++st) {
          const int cur = st & 1, nxt = cur ^ 1;
          if (!rotw) {
            constexpr int NB = BS * BS / C::kThreads, NR = B2 * BS / C::kThreads;
            int bp[NB], bq[NB], bu[NB], bw[NB];
            double cr[NB], sr[NB], cc[NB], sc[NB], m0[NB], m1[NB], m2[NB], m3[NB];
            int ri[NR], ru[NR], rw[NR];
            double rc[NR], rs[NR], r0[NR], r1[NR];
#pragma unroll
            for (int x = 0; x < NB; ++x) {
              const int e = tid + x * C::kThreads, kr = e / BS, kc = e % BS;
              bp[x] = pp[cur][kr]; bq[x] = qq[cur][kr]; bu[x] = pp[cur][kc]; bw[x] = qq[cur][kc];
              cr[x] = cs[cur][kr]; sr[x] = sn[cur][kr]; cc[x] = cs[cur][kc]; sc[x] = sn[cur][kc];
            }
#pragma unroll
            for (int x = 0; x < NR; ++x) {
              const int e = tid + x * C::kThreads, kc = e % BS;
              ri[x] = e / BS; ru[x] = pp[cur][kc]; rw[x] = qq[cur][kc];
              rc[x] = cs[cur][kc]; rs[x] = sn[cur][kc];
            }
#pragma unroll
            for (int x = 0; x < NB; ++x) {
              m0[x] = Sc[bp[x]][bu[x]]; m1[x] = Sc[bp[x]][bw[x]];
              m2[x] = Sc[bq[x]][bu[x]]; m3[x] = Sc[bq[x]][bw[x]];
            }
#pragma unroll
            for (int x = 0; x < NR; ++x) {
              r0[x] = R[ri[x]][ru[x]]; r1[x] = R[ri[x]][rw[x]];
            }
#pragma unroll
            for (int x = 0; x < NB; ++x) {   // 2x2 blocks of J^T S J
              const double rpu = cr[x] * m0[x] - sr[x] * m2[x], rpw = cr[x] * m1[x] - sr[x] * m3[x];
              const double rqu = sr[x] * m0[x] + cr[x] * m2[x], rqw = sr[x] * m1[x] + cr[x] * m3[x];
              Sn[bp[x]][bu[x]] = cc[x] * rpu - sc[x] * rpw;
              Sn[bp[x]][bw[x]] = sc[x] * rpu + cc[x] * rpw;
              Sn[bq[x]][bu[x]] = cc[x] * rqu - sc[x] * rqw;
              Sn[bq[x]][bw[x]] = sc[x] * rqu + cc[x] * rqw;
            }
#pragma unroll
            for (int x = 0; x < NR; ++x) {   // R <- R J
              R[ri[x]][ru[x]] = rc[x] * r0[x] - rs[x] * r1[x];
              R[ri[x]][rw[x]] = rs[x] * r0[x] + rc[x] * r1[x];
            }
          } else if (lane < BS && st + 1 < isteps) {
            int a, b;
            pair_at(st + 1, lane, a, b);
            pp[nxt][lane] = a;
            qq[nxt][lane] = b;
            pos[nxt][a] = 2 * lane;
            pos[nxt][b] = 2 * lane + 1;
            // entry (x, y) of J^T S_cur J: x in pair kx (side sx), y in pair ky (side sy)
            auto entry = [&](int kx, int sx, int ky, int sy) {
              const int p = pp[cur][kx], q = qq[cur][kx], u = pp[cur][ky], w = qq[cur][ky];
              const double cr = cs[cur][kx], sr = sn[cur][kx], cc = cs[cur][ky], sc = sn[cur][ky];
              const double m0 = Sc[p][u], m1 = Sc[p][w], m2 = Sc[q][u], m3 = Sc[q][w];
              const double rpu = cr * m0 - sr * m2, rpw = cr * m1 - sr * m3;
              const double rqu = sr * m0 + cr * m2, rqw = sr * m1 + cr * m3;
              const double ru_ = sx ? rqu : rpu, rw_ = sx ? rqw : rpw;
              return sy ? sc * ru_ + cc * rw_ : cc * ru_ - sc * rw_;
            };
            const int pa = pos[cur][a], pbb = pos[cur][b];
            const double naa = entry(pa >> 1, pa & 1, pa >> 1, pa & 1);
            const double nbb = entry(pbb >> 1, pbb & 1, pbb >> 1, pbb & 1);
            const double nab = entry(pa >> 1, pa & 1, pbb >> 1, pbb & 1);
            double c, sv;
            jb2_rotation(naa, nbb, nab, c, sv);
            cs[nxt][lane] = c;
            sn[nxt][lane] = sv;
          }
          __syncthreads();
          double (*t)[LD] = Sc; Sc = Sn; Sn = t;
        }
        double* Rg = Rbuf + (long long)k * B2 * B2;
        for (int e = tid; e < B2 * B2; e += nt) Rg[e] = R[e / B2][e % B2];
        __threadfence();
        __syncthreads();
        if (tid == 0)
          asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(rot_ready + k), "r"(gstep + 1)
                       : "memory");
      }
      ++gstep;
      if (!use_flags) grid.sync();
      // ---- phase B: G[PQ, RS] <- R_PQ^T G[PQ, RS] R_RS;  V[rows, PQ] <- V[rows, PQ] R_PQ ----
      const int gtasks = m * m, vtasks = (np / B2) * m;
      for (int task = bid; task < gtasks + vtasks; task += nb) {
        const bool isG = task < gtasks;
        const int t2 = isG ? task : task - gtasks;
        const int kr = isG ? t2 / m : -1, kc = t2 % m;
        const int rb = isG ? -1 : t2 / m;   // V row slab
        int Pc, Qc, Pr = 0, Qr = 0;
        pair_of(kc, step, Pc, Qc);
        if (isG) pair_of(kr, step, Pr, Qr);
        const double* Rc = Rbuf + (long long)kc * B2 * B2;
        const double* Rr = Rbuf + (long long)(isG ? kr : kc) * B2 * B2;
        if (use_flags && tid == 0) {   // the two rotations of this task (bounded spin: never a hang)
          const int need[2] = {kc, isG ? kr : kc};
          for (int w = 0; w < 2; ++w) {
            int v = 0;
            for (long long it = 0; it < (1LL << 28); ++it) {
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(rot_ready + need[w]) : "memory");
              if (v >= gstep) break;
            }
          }
        }
        __syncthreads();
        for (int e = tid; e < B2 * B2; e += nt) {
          const int i = e / B2, j = e % B2;
          const int gj = (j < BS ? Pc * BS + j : Qc * BS + j - BS);
          int gi;
          if (isG) gi = (i < BS ? Pr * BS + i : Qr * BS + i - BS);
          else gi = rb * B2 + i;
          Sb[i][j] = isG ? G[(long long)gi * np + gj] : V[(long long)gi * np + gj];
          Rb[i][j] = Rc[e];
          if (isG) R2b[i][j] = Rr[e];
        }
        __syncthreads();
        const bool mmaw = warp < C::kThreads / 32;   // the rotation warp only helps with loads
        double c[NTL][2];
#pragma unroll
        for (int t = 0; t < NTL; ++t) c[t][0] = c[t][1] = 0.0;
#pragma unroll 4
        for (int kk = 0; mmaw && kk < B2 / 4; ++kk) {   // T = S R_cols
          const double a = Sb[fr][4 * kk + fk];
#pragma unroll
          for (int t = 0; t < NTL; ++t) jb2_dmma(c[t], a, Rb[4 * kk + fk][fc + 8 * t]);
        }
        if (isG) {   // S <- T, then out = R_rows^T T
          __syncthreads();
#pragma unroll
          for (int t = 0; mmaw && t < NTL; ++t) {
            Sb[fr][oc + 8 * t] = c[t][0];
            Sb[fr][oc + 8 * t + 1] = c[t][1];
            c[t][0] = c[t][1] = 0.0;
          }
          __syncthreads();
#pragma unroll 4
          for (int kk = 0; mmaw && kk < B2 / 4; ++kk) {
            const double a = R2b[4 * kk + fk][fr];
#pragma unroll
            for (int t = 0; t < NTL; ++t) jb2_dmma(c[t], a, Sb[4 * kk + fk][fc + 8 * t]);
          }
        }
        if (mmaw) {   // the thread's outputs: row fr, columns oc + 8 t, + 1 (one BS-column half)
          const int i = fr;
          const long long gi = isG ? (i < BS ? Pr * BS + i : Qr * BS + i - BS)
                                   : (long long)rb * B2 + i;
          double* dst = (isG ? G : V) + gi * np + (half ? Qc * BS - BS : Pc * BS);
#pragma unroll
          for (int t = 0; t < NTL; ++t) {
            dst[oc + 8 * t] = c[t][0];
            dst[oc + 8 * t + 1] = c[t][1];
          }
        }
        __syncthreads();
      }
      grid.sync();
    }
  }
}

// copy an n x n matrix into the top-left of an np x np zero-padded buffer
__global__ void embed_kernel(const double* __restrict__ G, double* __restrict__ P, int n, int np) {
  const long long NN = (long long)np * np;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < NN;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / np), j = (int)(e - (long long)i * np);
    P[e] = (i < n && j < n) ? G[(long long)i * n + j] : 0.0;
  }
}

// eigenvalues (diag of the padded result, first n entries) and vectors sorted descending;
// `which` selects the buffer the cooperative kernel finished in
__global__ void sort_padded_kernel(const double* __restrict__ Ga, const double* __restrict__ Gb,
                                   const double* __restrict__ Va, const double* __restrict__ Vb,
                                   const int* __restrict__ which, double* __restrict__ V,
                                   double* __restrict__ lam, int n, int np) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* Gf = which[0] ? Gb : Ga;
  const double* Vf = which[0] ? Vb : Va;
  const double li = Gf[(long long)i * np + i];
  int rank = 0;
  for (int j = 0; j < n; ++j) {
    const double lj = Gf[(long long)j * np + j];
    rank += (lj > li) || (lj == li && j < i);
  }
  lam[rank] = li;
  for (int r = 0; r < n; ++r) V[(long long)r * n + rank] = Vf[(long long)r * np + i];
}

// W[r, c] = V[r, c] * f[c] for c < s (an n x s scaled column block of V)
__global__ void scale_cols_kernel(const double* __restrict__ V, const double* __restrict__ f,
                                  double* __restrict__ W, int n, int s) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * s) return;
  const int r = e / s, c = e - r * s;
  W[e] = V[r * n + c] * f[c];
}
