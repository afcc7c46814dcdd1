// tt_round.cuh — TT rounding on the GPU.
//
// Oseledets' TT-rounding (right-to-left orthonormalisation, left-to-right truncated SVD)
// with every SVD taken through the Gram matrix of the core unfolding:
//   G = M^T M (a DMMA GEMM of the engine) = V diag(sigma^2) V^T   (parallel cyclic Jacobi
//   eigensolver on all SMs, cooperative launch, n <= 512), U = M V diag(1/sigma) (a GEMM).
// Exactly rank-deficient unfoldings (e.g. the formal sum T + T) are handled: zero singular
// values are dropped.  The truncation decisions are data dependent, so the host reads the
// singular values of every core (one synchronisation per core).
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
