// tt_round.cuh — TT rounding on the GPU.
//
// Oseledets' TT-rounding (right-to-left orthonormalisation, left-to-right truncated SVD)
// with every SVD taken through the Gram matrix of the core unfolding:
//   G = M^T M (a DMMA GEMM of the engine) = V diag(sigma^2) V^T   (parallel cyclic Jacobi
//   eigensolver on all SMs, cooperative launch, n <= 512), U = M V diag(1/sigma) (a GEMM).
// Exactly rank-deficient unfoldings (e.g. the formal sum T + T) are handled: zero singular
// values are dropped.  The truncation decisions are data dependent, so the host reads the
// singular values of every core (one synchronisation per core).
// Included by tt_hotpath.cu inside its anonymous namespace.

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
