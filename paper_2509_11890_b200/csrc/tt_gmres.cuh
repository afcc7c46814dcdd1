// tt_gmres.cuh — GPU-resident restarted GMRES(m) on the projected local operator
// ("we can solve them in a matrix-free fashion via
// GMRES ... perform the constituent multiplications sequentially").
//
// nvec independent right-hand sides (the columns of a Block-TT core, layout (rl,n,nvec,rr))
// are solved in lock step: every Arnoldi step is ONE batched local matvec (the hot path,
// enqueue_matvec) plus column-wise reductions.  Orthogonalisation is classical Gram-Schmidt
// with one re-orthogonalisation pass (CGS2; equal in exact arithmetic to the modified
// Gram-Schmidt of the textbook algorithm).  The Hessenberg least-squares problem of every column is updated by Givens
// rotations in a one-thread-per-column kernel; converged columns are frozen by a device-side
// flag, so the whole solve is a fixed sequence of launches (asynchronous, graph-capturable).
// Included by tt_solvers.cu inside namespace ttint.

constexpr int kMaxL = 32;   // basis vectors per reduction pass

// Column-segmented reduction: part[(l*K + j)*chunks + c] = sum over the rows of chunk c of
// sum_b A_l[row, j, b] * B[row, j, b], for l < L <= LMAX (A_l = A + l*S).  Grid (chunks, K).
// Column j of a row is the contiguous run [(row K + j) rr, + rr); with VEC = 2 a thread
// reads b pairs as 16-byte loads (rr even).  LMAX bounds the accumulators: fewer registers,
// more resident warps, more loads in flight (the kernel is HBM-bound).
template <int LMAX, int VEC>
__global__ void __launch_bounds__(256) colreduce_kernel(const double* __restrict__ A, long long S,
                                                        int L, const double* __restrict__ B,
                                                        long long rows, int K, int rr,
                                                        long long rows_per_chunk,
                                                        double* __restrict__ part,
                                                        const int* __restrict__ gate) {
  if (gate && *gate) return;
  const int c = blockIdx.x, j = blockIdx.y, chunks = gridDim.x;
  const long long r0 = c * rows_per_chunk;
  const long long r1 = min(rows, r0 + rows_per_chunk);
  double acc[LMAX];
#pragma unroll
  for (int l = 0; l < LMAX; ++l) acc[l] = 0.0;
  if (VEC == 2) {
    const int half = rr / 2;
    for (long long row = r0; row < r1; ++row) {
      const long long base = (row * K + j) * rr;
      for (int bb = threadIdx.x; bb < half; bb += blockDim.x) {
        const long long e = base + 2 * bb;
        const double2 bv = *reinterpret_cast<const double2*>(B + e);
        double2 av[LMAX];
#pragma unroll
        for (int l = 0; l < LMAX; ++l)
          if (l < L) av[l] = *reinterpret_cast<const double2*>(A + l * S + e);
#pragma unroll
        for (int l = 0; l < LMAX; ++l)
          if (l < L) acc[l] = fma(av[l].y, bv.y, fma(av[l].x, bv.x, acc[l]));
      }
    }
  } else {
    const unsigned nel = (unsigned)((r1 - r0) * rr);
    for (unsigned t = threadIdx.x; t < nel; t += blockDim.x) {
      const unsigned rowo = t / (unsigned)rr, bb = t - rowo * (unsigned)rr;
      const long long e = ((r0 + rowo) * K + j) * rr + bb;
      const double bv = B[e];
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) acc[l] = fma(A[l * S + e], bv, acc[l]);
    }
  }
  __shared__ double red[8][LMAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int l = 0; l < LMAX; ++l) {
    if (l < L) {
      double v = acc[l];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][l] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < L) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w][threadIdx.x];
    part[((long long)threadIdx.x * K + j) * chunks + c] = v;
  }
}

// out[l*K + j] = sum_c part[(l*K + j)*chunks + c]   (fixed order: deterministic)
__global__ void colreduce_finish_kernel(const double* __restrict__ part, int LK, int chunks,
                                        double* __restrict__ out, const int* __restrict__ gate) {
  if (gate && *gate) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= LK) return;
  double v = 0.0;
  for (int c = 0; c < chunks; ++c) v += part[(long long)i * chunks + c];
  out[i] = v;
}

// B[e] += sign * sum_{l<L} coef[l*K + j(e)] * A_l[e]
__global__ void __launch_bounds__(256) colaxpy_kernel(const double* __restrict__ A, long long S,
                                                      int L, const double* __restrict__ coef,
                                                      double sign, double* __restrict__ B,
                                                      int K, int rr, const int* __restrict__ gate) {
  if (gate && *gate) return;
  __shared__ double cf[kMaxL * 64];
  for (int i = threadIdx.x; i < L * K; i += blockDim.x) cf[i] = sign * coef[i];
  __syncthreads();
  // one (row, column) run of rr contiguous doubles per block iteration (no per-element
  // 64-bit division)
  const long long runs = S / rr;
  for (long long rc = blockIdx.x; rc < runs; rc += gridDim.x) {
    const int j = (int)(rc % K);
    const long long base = rc * rr;
    for (int bb = threadIdx.x; bb < rr; bb += blockDim.x) {
      const long long e = base + bb;
      double v = B[e];
      for (int l = 0; l < L; ++l) v = fma(cf[l * K + j], A[l * S + e], v);
      B[e] = v;
    }
  }
}

// dst[e] = src[e] * s[j(e)];  dst2 (optional) = src - dst2 (residual form: dst = F - W)
__global__ void colscale_kernel(const double* __restrict__ src, const double* __restrict__ s,
                                double* __restrict__ dst, long long S, int K, int rr,
                                const int* __restrict__ gate) {
  if (gate && *gate) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < S;
       e += (long long)gridDim.x * blockDim.x)
    dst[e] = src[e] * s[(e / rr) % K];
}
__global__ void add_kernel(const double* __restrict__ C, double* __restrict__ X, long long S) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < S;
       e += (long long)gridDim.x * blockDim.x)
    X[e] += C[e];
}
// per-column 1 / ||c|| (0 for a zero column)
__global__ void inv_norm_kernel(const double* __restrict__ nrm2, double* __restrict__ sc, int K) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < K) sc[j] = nrm2[j] > 0.0 ? 1.0 / sqrt(nrm2[j]) : 0.0;
}
__global__ void sub_kernel(const double* __restrict__ F, double* __restrict__ W, long long S) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < S;
       e += (long long)gridDim.x * blockDim.x)
    W[e] = F[e] - W[e];
}

// Per-column GMRES state.
struct GmresState {
  double* H;      // [K][m+1][m]  Hessenberg (rotated in place)
  double* cs;     // [K][m]
  double* sn;     // [K][m]
  double* g;      // [K][m+1]
  double* fnorm;  // [K]
  double* rel;    // [K]   current relative residual estimate (output)
  double* scale;  // [K]   per-column scale for the next basis vector
  double* coef;   // [m][K] back-substitution result y (for the solution update)
  int* active;    // [K]
  int* kcyc;      // [K]   Arnoldi steps in the current cycle
  long long* its; // [K]   total Arnoldi steps (output)
  int* done;      // [1]   all columns inactive in the current cycle
};

// cycle start: beta = ||r_j|| (true residual of the current iterate)
__global__ void gmres_cycle_init_kernel(GmresState st, const double* __restrict__ nrm2,
                                        int K, int m, double tol) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  const double beta = sqrt(nrm2[j]);
  const double fn = st.fnorm[j];
  const double rel = fn > 0.0 ? beta / fn : 0.0;
  st.rel[j] = rel;
  const int act = (fn > 0.0) && (rel > tol) && (beta > 0.0);
  st.active[j] = act;
  st.kcyc[j] = 0;
  for (int i = 0; i <= m; ++i) st.g[(long long)j * (m + 1) + i] = 0.0;
  st.g[(long long)j * (m + 1)] = beta;
  st.scale[j] = act ? 1.0 / beta : 0.0;
}

__global__ void gmres_set_fnorm_kernel(GmresState st, const double* __restrict__ nrm2, int K) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  st.fnorm[j] = sqrt(nrm2[j]);
  st.its[j] = 0;
  st.rel[j] = 0.0;
}

// Arnoldi step i: column of H from the two Gram-Schmidt passes (h1 + h2, rows 0..i) and
// ||w||^2; previous rotations, new rotation, residual estimate, convergence flag, and the
// scale 1/H[i+1,i] of the next basis vector (0 for frozen columns or breakdown).
__global__ void gmres_arnoldi_kernel(GmresState st, const double* __restrict__ h1,
                                     const double* __restrict__ h2,
                                     const double* __restrict__ wn2, int K, int m, int i,
                                     double tol) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  if (!st.active[j]) {
    st.scale[j] = 0.0;
    return;
  }
  double* H = st.H + (long long)j * (m + 1) * m;
  double* cs = st.cs + (long long)j * m;
  double* sn = st.sn + (long long)j * m;
  double* g = st.g + (long long)j * (m + 1);
  for (int l = 0; l <= i; ++l) H[l * m + i] = h1[l * K + j] + h2[l * K + j];
  const double hn = sqrt(wn2[j]);
  H[(i + 1) * m + i] = hn;
  for (int l = 0; l < i; ++l) {
    const double a = H[l * m + i], b = H[(l + 1) * m + i];
    H[l * m + i] = cs[l] * a + sn[l] * b;
    H[(l + 1) * m + i] = -sn[l] * a + cs[l] * b;
  }
  const double a = H[i * m + i], b = H[(i + 1) * m + i];
  const double den = hypot(a, b);
  cs[i] = a / den;
  sn[i] = b / den;
  H[i * m + i] = den;
  H[(i + 1) * m + i] = 0.0;
  g[i + 1] = -sn[i] * g[i];
  g[i] = cs[i] * g[i];
  st.kcyc[j] = i + 1;
  st.its[j] += 1;
  const double rel = fabs(g[i + 1]) / st.fnorm[j];
  st.rel[j] = rel;
  const bool done = (rel <= tol) || !(hn > 0.0);
  if (done) st.active[j] = 0;
  st.scale[j] = (!done && hn > 0.0) ? 1.0 / hn : 0.0;
}

// ---- fused Arnoldi step for one right-hand side (K = 1, the paper's GMRES: one matrix-free
// product per Arnoldi step) -------------------------------------------------------
// The ~12 dependent launches of an orthogonalisation step (CGS2 dots and updates, norm, Givens,
// scaling) are latency, not bandwidth, at the ranks of the paper (a vector of r n r <= 2^18
// doubles).  One thread-block cluster of kOrthCluster CTAs does the whole step: each CTA owns
// a contiguous segment of the vector, the three reductions (h1 = V^T w, h2 = V^T w after the
// first update, ||w||^2) combine the CTAs' partial sums through distributed shared memory
// (every CTA adds the kOrthCluster partials in rank order: identical, deterministic results in
// all CTAs), CTA 0 performs the Hessenberg / Givens update of gmres_arnoldi_kernel and
// broadcasts 1 / H[i+1,i], and every CTA writes its segment of v_{i+1}.
constexpr int kOrthMaxL = 32;
constexpr long long kOrthMaxS = 1LL << 17;

// Each CTA keeps its segment of w in shared memory for the whole step and reads the basis
// three times: h1 = V^T w; then (same loaded V values) w -= V h1 and h2 = V^T w; then
// w -= V h2 and ||w||^2.  Element loops are unrolled by U (2 for L <= 16) so that U (L + 1)
// independent loads are in flight per thread (the kernel is load-latency bound at these sizes).
template <int LMAX, int NT, int U>
__global__ void __launch_bounds__(NT) gmres_orth_cluster_kernel(
    GmresState st, const double* __restrict__ V, double* __restrict__ W, double* __restrict__ Vnext,
    long long S, int L, int m, int i, double tol, const int* __restrict__ gate) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank(), ncl = (int)cluster.num_blocks();
  extern __shared__ double wseg[];   // this CTA's segment of w
  __shared__ double inA[16][LMAX], inB[16][LMAX], inC[16][1];   // partials pushed by every CTA
  __shared__ double h1[LMAX], h2[LMAX], wn2;
  __shared__ double red[NT / 32][LMAX + 1];
  __shared__ double sh_scale;
  const bool gated = gate && *gate;   // uniform: written by an earlier, completed launch
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long per = (S + ncl - 1) / ncl;
  const long long s0 = rank * per, s1 = min(S, s0 + per);
  const int nseg = (int)max(0LL, s1 - s0);

  // block-reduce acc[0..n), then thread l pushes the CTA's partial l into slot [rank][l] of
  // EVERY CTA's inbox (remote DSMEM stores, nothing to wait for); after one cluster barrier
  // each CTA sums its inbox locally in rank order (identical, deterministic in every CTA)
  auto block_reduce = [&](double (&acc)[LMAX + 1], int n, double* inbox, int ldi) {
#pragma unroll
    for (int l = 0; l < LMAX; ++l) {
      if (l >= n) break;
      double v = acc[l];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][l] = v;
    }
    __syncthreads();
    if (tid < n) {
      double v = 0.0;
      for (int q = 0; q < NT / 32; ++q) v += red[q][tid];
      for (int r = 0; r < ncl; ++r) cluster.map_shared_rank(inbox, r)[rank * ldi + tid] = v;
    }
  };
  auto combine = [&](const double* inbox, int ldi, double* h, int n) {
    cluster.sync();
    if (tid < n) {
      double v = 0.0;
      for (int r = 0; r < ncl; ++r) v += inbox[r * ldi + tid];
      h[tid] = v;
    }
    __syncthreads();
  };
  if (!gated) {
    double acc[LMAX + 1];
    // pass 1: w -> shared memory, h1 = V^T w
#pragma unroll
    for (int l = 0; l < LMAX; ++l) acc[l] = 0.0;
    for (int t0 = tid; t0 < nseg; t0 += U * NT) {
      const int t1 = t0 + NT;
      const bool ok1 = U == 2 && t1 < nseg;
      const double w0 = W[s0 + t0], w1 = ok1 ? W[s0 + t1] : 0.0;
      wseg[t0] = w0;
      if (ok1) wseg[t1] = w1;
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) {
          const double v0 = V[l * S + s0 + t0], v1 = ok1 ? V[l * S + s0 + t1] : 0.0;
          acc[l] = fma(v1, w1, fma(v0, w0, acc[l]));
        }
    }
    block_reduce(acc, L, &inA[0][0], LMAX);
    combine(&inA[0][0], LMAX, h1, L);
    // pass 2: w -= V h1, h2 = V^T w (one read of V)
#pragma unroll
    for (int l = 0; l < LMAX; ++l) acc[l] = 0.0;
    for (int t0 = tid; t0 < nseg; t0 += U * NT) {
      const int t1 = t0 + NT;
      const bool ok1 = U == 2 && t1 < nseg;
      double vv0[LMAX], vv1[LMAX];
      double w0 = wseg[t0], w1 = ok1 ? wseg[t1] : 0.0;
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) {
          vv0[l] = V[l * S + s0 + t0];
          vv1[l] = ok1 ? V[l * S + s0 + t1] : 0.0;
        }
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) {
          w0 = fma(-h1[l], vv0[l], w0);
          w1 = fma(-h1[l], vv1[l], w1);
        }
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) acc[l] = fma(vv1[l], w1, fma(vv0[l], w0, acc[l]));
      wseg[t0] = w0;
      if (ok1) wseg[t1] = w1;
    }
    block_reduce(acc, L, &inB[0][0], LMAX);
    combine(&inB[0][0], LMAX, h2, L);
    // pass 3: w -= V h2, ||w||^2
    acc[0] = 0.0;
    for (int t0 = tid; t0 < nseg; t0 += U * NT) {
      const int t1 = t0 + NT;
      const bool ok1 = U == 2 && t1 < nseg;
      double vv0[LMAX], vv1[LMAX];
      double w0 = wseg[t0], w1 = ok1 ? wseg[t1] : 0.0;
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) {
          vv0[l] = V[l * S + s0 + t0];
          vv1[l] = ok1 ? V[l * S + s0 + t1] : 0.0;
        }
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) {
          w0 = fma(-h2[l], vv0[l], w0);
          w1 = fma(-h2[l], vv1[l], w1);
        }
      acc[0] = fma(w1, w1, fma(w0, w0, acc[0]));
      wseg[t0] = w0;
      if (ok1) wseg[t1] = w1;
    }
    block_reduce(acc, 1, &inC[0][0], 1);
    combine(&inC[0][0], 1, &wn2, 1);
    if (rank == 0 && tid == 0) {   // the Hessenberg column, Givens rotations, convergence
      double scale = 0.0;
      if (st.active[0]) {
        double* H = st.H;
        double* cs = st.cs;
        double* sn = st.sn;
        double* gg = st.g;
        for (int l = 0; l <= i; ++l) H[l * m + i] = h1[l] + h2[l];
        const double hn = sqrt(wn2);
        H[(i + 1) * m + i] = hn;
        for (int l = 0; l < i; ++l) {
          const double a = H[l * m + i], b = H[(l + 1) * m + i];
          H[l * m + i] = cs[l] * a + sn[l] * b;
          H[(l + 1) * m + i] = -sn[l] * a + cs[l] * b;
        }
        const double a = H[i * m + i], b = H[(i + 1) * m + i];
        const double den = hypot(a, b);
        cs[i] = a / den;
        sn[i] = b / den;
        H[i * m + i] = den;
        H[(i + 1) * m + i] = 0.0;
        gg[i + 1] = -sn[i] * gg[i];
        gg[i] = cs[i] * gg[i];
        st.kcyc[0] = i + 1;
        st.its[0] += 1;
        const double rel = fabs(gg[i + 1]) / st.fnorm[0];
        st.rel[0] = rel;
        const bool done = (rel <= tol) || !(hn > 0.0);
        if (done) st.active[0] = 0;
        scale = (!done && hn > 0.0) ? 1.0 / hn : 0.0;
      }
      st.scale[0] = scale;
      *st.done = !st.active[0];
      sh_scale = scale;
    }
    cluster.sync();
    const double scale = *cluster.map_shared_rank(&sh_scale, 0);
    for (int t = tid; t < nseg; t += NT) Vnext[s0 + t] = wseg[t] * scale;
  }
  cluster.sync();   // no CTA leaves while another may still read its shared memory
}

// cluster size: 16 CTAs where the device allows non-portable clusters, else 8 (per device)
template <int LMAX, int NT, int U>
cudaError_t orth_launch_t(const GmresState& st, const double* V, double* W, double* Vnext,
                          long long S, int L, int m, int i, double tol, cudaStream_t s) {
  auto kern = gmres_orth_cluster_kernel<LMAX, NT, U>;
  thread_local int cl_dev[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& cl = cl_dev[dev & 63];
  const size_t smem_max = sizeof(double) * (size_t)((kOrthMaxS + 7) / 8);   // w segment, 8 CTAs
  if (cl == 0) {
    cl = 8;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
        smem_attr((const void*)kern, (int)smem_max) == cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(16);
      q.blockDim = dim3(NT);
      q.dynamicSmemBytes = sizeof(double) * (size_t)((kOrthMaxS + 15) / 16);
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = 16;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      q.attrs = a;
      q.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &q) == cudaSuccess && nclusters > 0) cl = 16;
    }
    cudaGetLastError();
  }
  if (cudaError_t e = smem_attr((const void*)kern, (int)smem_max)) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = sizeof(double) * (size_t)((S + cl - 1) / cl);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, st, V, W, Vnext, S, L, m, i, tol, g_gate);
}

cudaError_t launch_orth_cluster(const GmresState& st, const double* V, double* W, double* Vnext,
                                long long S, int L, int m, int i, double tol, cudaStream_t s) {
  ++g_launches;
  g_stage = TT_ST_SET;
  const long long tr = trace_begin(-1, S, L, 0, s);
  cudaError_t e;
  if (L <= 8)
    e = orth_launch_t<8, 512, 2>(st, V, W, Vnext, S, L, m, i, tol, s);
  else if (L <= 16)
    e = orth_launch_t<16, 256, 2>(st, V, W, Vnext, S, L, m, i, tol, s);
  else
    e = orth_launch_t<32, 256, 1>(st, V, W, Vnext, S, L, m, i, tol, s);
  trace_end(tr, s);
  return e;
}

// *done = no column is active (gates the rest of the cycle's Arnoldi steps)
__global__ void gmres_alldone_kernel(const int* __restrict__ active, int K, int* __restrict__ done) {
  int any = 0;
  for (int j = 0; j < K; ++j) any |= active[j];
  *done = !any;
}

// back substitution H[:k,:k] y = g[:k] per column -> coef[l*K + j] (0 beyond k)
__global__ void gmres_backsolve_kernel(GmresState st, int K, int m) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  const int k = st.kcyc[j];
  const double* H = st.H + (long long)j * (m + 1) * m;
  const double* g = st.g + (long long)j * (m + 1);
  for (int l = m - 1; l >= 0; --l) {
    double y = 0.0;
    if (l < k) {
      y = g[l];
      for (int q = l + 1; q < k; ++q) y -= H[l * m + q] * st.coef[q * K + j];
      y /= H[l * m + l];
    }
    st.coef[l * K + j] = y;
  }
}

struct GmresDims {
  long long S;      // elements of one Block-TT vector (rl n K rr)
  long long rows;   // rl * n
  int K, rr;
  int chunks;
  long long rows_per_chunk;
};

GmresDims gmres_dims(const Dims& d, long long K) {
  GmresDims g;
  g.rows = d.a * d.n;
  g.K = (int)K;
  g.rr = (int)d.b;
  g.S = g.rows * K * d.b;
  // ~ 4 blocks per SM across (chunks x K)
  long long want = (4LL * num_sms() + K - 1) / K;
  if (want < 1) want = 1;
  if (want > g.rows) want = g.rows;
  g.rows_per_chunk = (g.rows + want - 1) / want;
  g.chunks = (int)((g.rows + g.rows_per_chunk - 1) / g.rows_per_chunk);
  return g;
}

// out[l*K+j] = <A_l[:,j], B[:,j]> for l < L (L any size; passes of kMaxL)
cudaError_t launch_coldots(const GmresDims& gd, const double* A, int L, const double* B,
                           double* part, double* out, cudaStream_t s) {
  constexpr int kPass = 16;   // accumulators per pass (colreduce_kernel LMAX)
  for (int l0 = 0; l0 < L; l0 += kPass) {
    const int Lp = std::min(kPass, L - l0);
    dim3 grid(gd.chunks, gd.K);
    const double* Al = A + l0 * gd.S;
    const bool v2 = (gd.rr % 2 == 0) && (gd.S % 2 == 0) &&
                    ((reinterpret_cast<uintptr_t>(Al) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
#define TT_COLRED(LM)                                                                         \
  do {                                                                                        \
    if (v2) colreduce_kernel<LM, 2><<<grid, 256, 0, s>>>(Al, gd.S, Lp, B, gd.rows, gd.K, gd.rr, \
                                                         gd.rows_per_chunk, part, g_gate);      \
    else colreduce_kernel<LM, 1><<<grid, 256, 0, s>>>(Al, gd.S, Lp, B, gd.rows, gd.K, gd.rr,    \
                                                      gd.rows_per_chunk, part, g_gate);         \
  } while (0)
    if (Lp <= 4) TT_COLRED(4);
    else if (Lp <= 8) TT_COLRED(8);
    else TT_COLRED(16);
#undef TT_COLRED
    ++g_launches;
    const int LK = Lp * gd.K;
    colreduce_finish_kernel<<<(LK + 255) / 256, 256, 0, s>>>(part, LK, gd.chunks,
                                                            out + (long long)l0 * gd.K, g_gate);
    ++g_launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_colaxpy(const GmresDims& gd, const double* A, int L, const double* coef,
                           double sign, double* B, cudaStream_t s) {
  long long blocks = (gd.S + 255) / 256;
  if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
  for (int l0 = 0; l0 < L; l0 += kMaxL) {
    const int Lp = std::min(kMaxL, L - l0);
    colaxpy_kernel<<<(unsigned)blocks, 256, 0, s>>>(A + l0 * gd.S, gd.S, Lp,
                                                     coef + (long long)l0 * gd.K, sign, B, gd.K,
                                                     gd.rr, g_gate);
    ++g_launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_elementwise(int kind, const double* a, const double* sc, double* b,
                               const GmresDims& gd, cudaStream_t s) {
  long long blocks = (gd.S + 255) / 256;
  if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
  if (kind == 0)
    colscale_kernel<<<(unsigned)blocks, 256, 0, s>>>(a, sc, b, gd.S, gd.K, gd.rr, g_gate);
  else if (kind == 1)
    sub_kernel<<<(unsigned)blocks, 256, 0, s>>>(a, b, gd.S);
  else
    add_kernel<<<(unsigned)blocks, 256, 0, s>>>(a, b, gd.S);
  ++g_launches;
  return cudaGetLastError();
}

// element counts of the GMRES workspace beyond the matvec's own
struct GmresWs {
  long long basis, w, part, small;
};
// m = Krylov steps per cycle plus augmentation vectors (the Hessenberg dimension); the
// basis holds m+1 orthonormal vectors, the k_aug error approximations and one correction.
bool gmres_ws_elems(const Dims& d, long long K, long long m, GmresWs& g, long long kaug = 0) {
  bool ok = true;
  const long long S = prod({d.a, d.n, K, d.b}, ok);
  g.basis = prod({m + 1 + kaug + 1, S}, ok);
  g.w = S;
  GmresDims gd = gmres_dims(d, K);
  g.part = (long long)kMaxL * K * gd.chunks;
  // H, cs, sn, g, fnorm, rel, scale, coef, h1, h2, wn2 (doubles) + active, kcyc, its
  g.small = K * ((m + 1) * m + 2 * m + (m + 1) + 4 + m) + 2 * (m + 1) * K + K + 3 * K + 8;
  return ok;
}

// The solve (host-side launch sequence; no synchronisation).  kaug > 0: LGMRES(m, kaug)
// (Baker, Jessup & Manteuffel 2005): each cycle's search space is [v_0..v_{m-1}] plus the
// kaug most recent normalised corrections z (newest first), orthonormalised into the
// growing Arnoldi basis; the new correction becomes the newest z.
cudaError_t enqueue_gmres(const Dims& d, long long K, long long m, long long kaug,
                          long long cycles, double tol, const double* phiL, const double* A,
                          const double* phiR, const double* F, double* X, double* rel_out,
                          long long* its_out, void* workspace, size_t workspace_bytes,
                          cudaStream_t s) {
  const long long ms = m + kaug;   // Hessenberg dimension
  long long t1, t2, ah, pe;
  matvec_ws_elems(d, K, t1, t2, ah, pe);
  GmresWs gw;
  gmres_ws_elems(d, K, ms, gw, kaug);
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  double* T1 = c.take(t1);
  double* T2 = c.take(t2);
  double* Ah = c.take(ah);
  double* Pp = c.take(pe);
  double* V = c.take(gw.basis);   // (ms + 2) vectors: ms + 1 basis, then Z slots / correction
  double* W = c.take(gw.w);
  double* part = c.take(gw.part);
  double* sm = c.take(gw.small);
  if (!c.ok) return cudaErrorInvalidValue;
  GmresState st;
  st.H = sm;
  st.cs = st.H + K * (ms + 1) * ms;
  st.sn = st.cs + K * ms;
  st.g = st.sn + K * ms;
  st.fnorm = st.g + K * (ms + 1);
  st.rel = rel_out;
  st.scale = st.fnorm + K;
  st.coef = st.scale + K;
  double* h1 = st.coef + ms * K;
  double* h2 = h1 + (ms + 1) * K;
  double* wn2 = h2 + (ms + 1) * K;
  st.active = reinterpret_cast<int*>(wn2 + K);
  st.kcyc = st.active + K;
  st.done = st.kcyc + K;
  st.its = its_out;
  const GmresDims gd = gmres_dims(d, K);
  // vector slots: V_0..V_{m+nz} (Arnoldi basis, at most ms + 1), then the kaug Z slots
  double* Zs = V + (ms + 1) * gd.S;
  double* C = W;   // the correction reuses W after the cycle's last Arnoldi step
  std::vector<int> zorder;   // Z slot indices, newest first
  const int kb = (int)((K + 127) / 128), kt = 128;
  // K = 1 at the paper's ranks: the fused cluster kernel for the orthogonalisation step
  // (debug flag 1 << 26 keeps the separate kernels)
  const bool fused_orth = K == 1 && ms + 1 <= kOrthMaxL && gd.S <= kOrthMaxS &&
                          !(g_dbg_flags & (1 << 26));
  cudaError_t e;
  g_stage = TT_ST_PERM;
  if ((e = launch_perm(true, A, Ah, d.al, d.n, d.be, s)) != cudaSuccess) return e;
  // ||f||
  if ((e = launch_coldots(gd, F, 1, F, part, wn2, s)) != cudaSuccess) return e;
  gmres_set_fnorm_kernel<<<kb, kt, 0, s>>>(st, wn2, (int)K);
  ++g_launches;
  for (long long cyc = 0; cyc < cycles; ++cyc) {
    const long long nz = (long long)zorder.size();
    // r = f - L(x), beta = ||r||, v0 = r / beta
    if ((e = enqueue_matvec(d, K, phiL, A, phiR, X, W, T1, T2, Ah, Pp, pe, s, Ah)) != cudaSuccess)
      return e;
    if ((e = launch_elementwise(1, F, nullptr, W, gd, s)) != cudaSuccess) return e;
    if ((e = launch_coldots(gd, W, 1, W, part, wn2, s)) != cudaSuccess) return e;
    gmres_cycle_init_kernel<<<kb, kt, 0, s>>>(st, wn2, (int)K, (int)ms, tol);
    ++g_launches;
    gmres_alldone_kernel<<<1, 1, 0, s>>>(st.active, (int)K, st.done);
    ++g_launches;
    if ((e = launch_elementwise(0, W, st.scale, V, gd, s)) != cudaSuccess) return e;
    // once every column has converged the rest of the cycle's Arnoldi steps are no-ops
    // (device flag read by every launch of the step, the matvec's GEMMs included)
    struct GateScope {
      GateScope(const int* g) { g_gate = g; }
      ~GateScope() { g_gate = nullptr; }
    } gscope(st.done);
    for (long long i = 0; i < m + nz; ++i) {
      const double* in = (i < m) ? V + i * gd.S : Zs + (long long)zorder[i - m] * gd.S;
      if ((e = enqueue_matvec(d, K, phiL, A, phiR, in, W, T1, T2, Ah, Pp, pe, s, Ah)) !=
          cudaSuccess)
        return e;
      const int L = (int)(i + 1);
      if (fused_orth) {   // one cluster launch for the whole orthogonalisation step
        if ((e = launch_orth_cluster(st, V, W, V + (i + 1) * gd.S, gd.S, L, (int)ms, (int)i, tol, s)) !=
            cudaSuccess)
          return e;
        continue;
      }
      // CGS2: two classical Gram-Schmidt passes against v_0..v_i
      if ((e = launch_coldots(gd, V, L, W, part, h1, s)) != cudaSuccess) return e;
      if ((e = launch_colaxpy(gd, V, L, h1, -1.0, W, s)) != cudaSuccess) return e;
      if ((e = launch_coldots(gd, V, L, W, part, h2, s)) != cudaSuccess) return e;
      if ((e = launch_colaxpy(gd, V, L, h2, -1.0, W, s)) != cudaSuccess) return e;
      if ((e = launch_coldots(gd, W, 1, W, part, wn2, s)) != cudaSuccess) return e;
      gmres_arnoldi_kernel<<<kb, kt, 0, s>>>(st, h1, h2, wn2, (int)K, (int)ms, (int)i, tol);
      ++g_launches;
      gmres_alldone_kernel<<<1, 1, 0, s>>>(st.active, (int)K, st.done);
      ++g_launches;
      if ((e = launch_elementwise(0, W, st.scale, V + (i + 1) * gd.S, gd, s)) != cudaSuccess)
        return e;
    }
    g_gate = nullptr;
    gmres_backsolve_kernel<<<kb, kt, 0, s>>>(st, (int)K, (int)ms);
    ++g_launches;
    // correction C = sum_{i<m} y_i v_i + sum_{j<nz} y_{m+j} z_j;  x += C
    if ((e = cudaMemsetAsync(C, 0, sizeof(double) * gd.S, s)) != cudaSuccess) return e;
    if ((e = launch_colaxpy(gd, V, (int)m, st.coef, 1.0, C, s)) != cudaSuccess) return e;
    for (long long j = 0; j < nz; ++j)
      if ((e = launch_colaxpy(gd, Zs + (long long)zorder[j] * gd.S, 1, st.coef + (m + j) * K, 1.0,
                              C, s)) != cudaSuccess)
        return e;
    if ((e = launch_elementwise(2, C, nullptr, X, gd, s)) != cudaSuccess) return e;
    if (kaug > 0) {   // newest error approximation z = C / ||C||
      if ((e = launch_coldots(gd, C, 1, C, part, wn2, s)) != cudaSuccess) return e;
      inv_norm_kernel<<<kb, kt, 0, s>>>(wn2, st.scale, (int)K);
      ++g_launches;
      const int slot = (nz < kaug) ? (int)nz : zorder.back();
      if ((e = launch_elementwise(0, C, st.scale, Zs + (long long)slot * gd.S, gd, s)) !=
          cudaSuccess)
        return e;
      if (nz == kaug) zorder.pop_back();
      zorder.insert(zorder.begin(), slot);
    }
  }
  return cudaGetLastError();
}
