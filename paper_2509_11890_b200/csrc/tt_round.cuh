// tt_round.cuh — TT rounding on the GPU.
//
// Oseledets' TT-rounding (right-to-left orthonormalisation, left-to-right truncated SVD)
// with every SVD taken through the Gram matrix of the core unfolding:
//   G = M^T M (a DMMA GEMM of the engine) = V diag(sigma^2) V^T   (parallel cyclic Jacobi
//   eigensolver, one CTA, n <= 512), U = M V diag(1/sigma) (another GEMM).
// Exactly rank-deficient unfoldings (e.g. the formal sum T + T) are handled: zero singular
// values are dropped.  The truncation decisions are data dependent, so the host reads the
// singular values of every core (one synchronisation per core).
// Included by tt_hotpath.cu inside its anonymous namespace.

// Parallel cyclic Jacobi for a symmetric n x n matrix G (row-major, global, overwritten);
// On exit diag(G) holds the eigenvalues and V (n x n, column i = vector i) the eigenvectors
// (unsorted; sort_eigvecs_kernel orders them).
// Round-robin ordering: in every step the n/2 disjoint pairs rotate simultaneously (their
// rotations commute), rows first, then columns; `sweeps` full sweeps or until the
// off-diagonal mass is below eps of the diagonal.
__global__ void __launch_bounds__(1024) jacobi_eigen_kernel(double* __restrict__ G,
                                                            double* __restrict__ V, int n,
                                                            int sweeps) {
  extern __shared__ double sh[];
  const int np = (n + 1) & ~1;         // even number of players (one dummy if n is odd)
  double* cs = sh;                     // [np/2]
  double* sn = sh + np / 2;            // [np/2]
  int* pp = reinterpret_cast<int*>(sn + np / 2);   // [np/2] p of each pair
  int* qq = pp + np / 2;                            // [np/2] q of each pair
  __shared__ double red[32];
  __shared__ int stop;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < n * n; e += nt) V[e] = (e / n == e % n) ? 1.0 : 0.0;
  __syncthreads();
  for (int sw = 0; sw < sweeps; ++sw) {
    // convergence test: off-diagonal vs diagonal Frobenius mass
    double off = 0.0, dia = 0.0;
    for (int e = tid; e < n * n; e += nt) {
      const double v = G[e];
      if (e / n == e % n) dia += v * v; else off += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_down_sync(0xffffffffu, off, o);
      dia += __shfl_down_sync(0xffffffffu, dia, o);
    }
    if ((tid & 31) == 0) red[tid >> 5] = off;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < nt / 32; ++w) s += red[w];
      red[31] = s;
    }
    __syncthreads();
    const double offsum = red[31];
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = dia;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < nt / 32; ++w) s += red[w];
      stop = (offsum <= 1e-30 * s) ? 1 : 0;
    }
    __syncthreads();
    if (stop) break;
    for (int step = 0; step < np - 1; ++step) {
      // round-robin schedule: player 0 fixed, the others rotate
      for (int k = tid; k < np / 2; k += nt) {
        int a = (k == 0) ? 0 : 1 + (k - 1 + step) % (np - 1);
        int b = 1 + (np - 2 - k + step) % (np - 1);
        if (a > b) { const int t = a; a = b; b = t; }
        pp[k] = a;
        qq[k] = b;
        double c = 1.0, s = 0.0;
        if (b < n) {
          const double apq = G[a * n + b];
          if (apq != 0.0) {
            const double app = G[a * n + a], aqq = G[b * n + b];
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        cs[k] = c;
        sn[k] = s;
      }
      __syncthreads();
      // rows: (row p, row q) <- (c row p - s row q, s row p + c row q)
      for (int e = tid; e < (np / 2) * n; e += nt) {
        const int k = e / n, j = e - k * n;
        const int p = pp[k], q = qq[k];
        if (q >= n) continue;
        const double c = cs[k], s = sn[k];
        const double gp = G[p * n + j], gq = G[q * n + j];
        G[p * n + j] = c * gp - s * gq;
        G[q * n + j] = s * gp + c * gq;
      }
      __syncthreads();
      // columns of G and V
      for (int e = tid; e < (np / 2) * n; e += nt) {
        const int k = e / n, i = e - k * n;
        const int p = pp[k], q = qq[k];
        if (q >= n) continue;
        const double c = cs[k], s = sn[k];
        const double gp = G[i * n + p], gq = G[i * n + q];
        G[i * n + p] = c * gp - s * gq;
        G[i * n + q] = s * gp + c * gq;
        const double vp = V[i * n + p], vq = V[i * n + q];
        V[i * n + p] = c * vp - s * vq;
        V[i * n + q] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  // on exit: diag(G) = eigenvalues (unsorted), V = eigenvectors (columns)
}

// Reorder eigenvector columns by descending eigenvalue: V[:, rank(i)] = G[:, i] where G holds
// the unsorted vectors and d the unsorted eigenvalues.
__global__ void sort_eigvecs_kernel(const double* __restrict__ Gvec, const double* __restrict__ d,
                                    double* __restrict__ V, double* __restrict__ lam, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double li = d[i];
  int rank = 0;
  for (int j = 0; j < n; ++j) rank += (d[j] > li) || (d[j] == li && j < i);
  lam[rank] = li;
  for (int r = 0; r < n; ++r) V[r * n + rank] = Gvec[r * n + i];
}

__global__ void diag_kernel(const double* __restrict__ G, double* __restrict__ d, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = G[i * n + i];
}

// W[r, c] = V[r, c] * f[c] for c < s (an n x s scaled column block of V)
__global__ void scale_cols_kernel(const double* __restrict__ V, const double* __restrict__ f,
                                  double* __restrict__ W, int n, int s) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * s) return;
  const int r = e / s, c = e - r * s;
  W[e] = V[r * n + c] * f[c];
}
