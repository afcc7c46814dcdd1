// tt_lobpcg.cuh — GPU-resident block LOBPCG for the step-length local eigenproblem
// (PAPER.md:556-567).
//
// The paper poses the optimal step length as d local generalised eigenproblems
//   max_E  vec(E)^T E_{!=k}^T dM E_{!=k} vec(E)   s.t.  vec(E)^T E_{!=k}^T M E_{!=k} vec(E) = 1
// and notes they "can also be implemented in a matrix-free fashion by using iterative
// eigenvalue solvers (such as LOBPCG [Knyazev 2001])".  Here both projected
// operators act through the hot-path local matvec (enqueue_matvec, H1-H4) on the nb columns of
// a Block-TT block, and everything else stays on the device:
//
//   X <- Rayleigh-Ritz(X); loop:  W = A X - B X diag(lam)         (residual, no preconditioner)
//                                 AW = A W, BW = B W               (2 batched local matvecs)
//                                 S = [X W P], G_A = S^T A S, G_B = S^T B S
//                                 G_B = U mu U^T (Jacobi), drop mu <= 1e-12 mu_max,
//                                 T = U mu^{-1/2}, T^T G_A T = V theta V^T (Jacobi)
//                                 C = T V[:, largest nb]:  X <- S C,  P <- [W P] C_{W,P}
//
// (Knyazev 2001, Alg. 4.1 "LOBPCG" with the Rayleigh-Ritz step done by an SVQB-style
// eigen-reduction of the Gram matrix (Stathopoulos & Wu 2002) instead of a Cholesky
// factorisation, so nearly dependent directions are dropped instead of failing.)  The
// images A S, B S are carried by the same linear combinations, so each iteration costs two
// batched matvecs.  Convergence (max over columns of ||A x - lam B x|| / (||A x|| +
// |lam| ||B x||) <= tol) sets a device flag that turns every later launch, the GEMMs of the
// matvecs included (GemmParams::gate), into a no-op: the solve is a fixed, asynchronous,
// graph-capturable launch sequence whose iterations after convergence cost launches only.
// Included by tt_solvers.cu inside namespace ttint.

constexpr int kLobMaxNb = 32;
// Cholesky pivot floor of the equilibrated Gram matrix (squared norm of the new direction a
// column adds): below it the Rayleigh-Ritz step restarts without P / falls back to SVQB
#ifndef TT_LOB_PIVOT
#define TT_LOB_PIVOT 1e-4
#endif
constexpr double kLobPivot = TT_LOB_PIVOT;
constexpr int kLobMaxS = 3 * kLobMaxNb;   // Rayleigh-Ritz basis [X W P]

struct LobDims {
  long long rows;   // rl * n
  long long S;      // elements of one block (rl n nb rr)
  int nb, rr;
  int chunks;       // column-norm partial sums
  long long rows_per_chunk;
  int gchunks;      // Gram partial sums
  long long k_per_gchunk;
};

LobDims lob_dims(const Dims& d, long long nb) {
  LobDims L;
  L.rows = d.a * d.n;
  L.nb = (int)nb;
  L.rr = (int)d.b;
  L.S = L.rows * nb * d.b;
  long long want = (4LL * num_sms() + nb - 1) / nb;
  want = std::max(1LL, std::min(want, L.rows));
  L.rows_per_chunk = (L.rows + want - 1) / want;
  L.chunks = (int)((L.rows + L.rows_per_chunk - 1) / L.rows_per_chunk);
  const long long kt = L.rows * d.b;   // contraction length of the Gram matrices
  long long g = std::max(1LL, std::min<long long>(2LL * num_sms(), (kt + 255) / 256));
  L.k_per_gchunk = (kt + g - 1) / g;
  L.gchunks = (int)((kt + L.k_per_gchunk - 1) / L.k_per_gchunk);
  return L;
}

// Residual and column norms in one pass: W = AX - BX diag(lam) is written, and
// part[(t*nb + j)*chunks + c] = sum over chunk c of the squared entries of column j of block t
// (t < 3: W, AX, BX).  Grid (chunks, nb).
__global__ void __launch_bounds__(256) lob_colnorm_kernel(double* __restrict__ W,
                                                          const double* __restrict__ AX,
                                                          const double* __restrict__ BX,
                                                          const double* __restrict__ lam,
                                                          long long rows, int nb, int rr,
                                                          long long rows_per_chunk,
                                                          double* __restrict__ part,
                                                          const int* __restrict__ gate) {
  if (gate && *gate) return;
  const int c = blockIdx.x, j = blockIdx.y, chunks = gridDim.x;
  const long long r0 = c * rows_per_chunk, r1 = min(rows, r0 + rows_per_chunk);
  const double lj = lam[j];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (long long t = threadIdx.x; t < (r1 - r0) * rr; t += blockDim.x) {
    const long long e = ((r0 + t / rr) * nb + j) * rr + (t % rr);
    const double x1 = AX[e], x2 = BX[e];
    const double x0 = fma(-lj, x2, x1);
    W[e] = x0;
    a0 = fma(x0, x0, a0);
    a1 = fma(x1, x1, a1);
    a2 = fma(x2, x2, a2);
  }
  __shared__ double red[3][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_down_sync(0xffffffffu, a0, o);
    a1 += __shfl_down_sync(0xffffffffu, a1, o);
    a2 += __shfl_down_sync(0xffffffffu, a2, o);
  }
  if (lane == 0) {
    red[0][warp] = a0;
    red[1][warp] = a1;
    red[2][warp] = a2;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
    part[((long long)threadIdx.x * nb + j) * chunks + c] = v;
  }
}

struct LobState {
  double* lam;      // [nb] Ritz values, descending (output)
  double* res;      // [nb] relative residuals (output)
  double* scale;    // [nb] 1 / ||w_j||
  int* done;        // convergence flag (the gate)
  long long* its;   // iterations performed (output)
  double* step;     // optional: min(1, 1 / lam_0) if lam_0 > 0 else 1
};

// Residual norms -> relative residuals, the normalisation of W, convergence; one block of
// 1024 threads: warp w sums the chunk partials of (array, column) pairs w, w + 32, ... (lanes
// over chunks, a fixed shuffle tree: deterministic), then the first nb threads finish.
__global__ void __launch_bounds__(1024) lob_check_kernel(const double* __restrict__ part, int chunks,
                                                         int nb, LobState st, double tol,
                                                         int final_pass) {
  if (!final_pass && *st.done) return;
  __shared__ double sums[3 * kLobMaxNb];
  __shared__ double rmax[kLobMaxNb];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int q = warp; q < 3 * nb; q += nw) {
    double v = 0.0;
    for (int c = lane; c < chunks; c += 32) v += part[(long long)q * chunks + c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sums[q] = v;
  }
  __syncthreads();
  const int j = threadIdx.x;
  double rel = 0.0;
  if (j < nb) {
    const double w = sums[j], a = sums[nb + j], b = sums[2 * nb + j];
    const double wn = sqrt(w), den = sqrt(a) + fabs(st.lam[j]) * sqrt(b);
    rel = den > 0.0 ? wn / den : 0.0;
    st.res[j] = rel;
    st.scale[j] = wn > 0.0 ? 1.0 / wn : 0.0;
    rmax[j] = rel;
  }
  __syncthreads();
  if (j == 0) {
    double m = 0.0;
    for (int q = 0; q < nb; ++q) m = fmax(m, rmax[q]);
    if (!final_pass && m <= tol) *st.done = 1;
    if (final_pass && st.step) {
      const double l0 = st.lam[0];
      st.step[0] = l0 > 0.0 ? fmin(1.0, 1.0 / l0) : 1.0;
    }
  }
}

// Gram partial sums: part[c][p][m] = sum over the contraction indices k = (row, b) of chunk c
// of U_{p / nb}[row, p % nb, b] * V_{m / nb}[row, m % nb, b],  p < nu nb, m < nv nb.
struct GramArgs {
  const double* U[3];
  const double* V[6];
  int nu, nv, nb, rr;
  long long kt, k_per_chunk;
  const int* gate;
  tt::FastDiv rrdiv;   // k -> (row, b) with 32-bit magic division when kt < 2^31 (k32)
  int k32;
};

// Thread layout: G = 256 / (TU TV) groups split the 32 contraction indices of a staged chunk;
// inside a group a TU x TV grid of threads owns IU x JV outputs each (rows tu + TU i, columns
// tv + TV j); the G partial tiles are summed in shared memory in a fixed order.
template <int TU, int TV, int IU, int JV>
struct GramCfg {
  static constexpr int G = 256 / (TU * TV), KB = 32, LD = KB + 1;
  // two staging buffers (cp.async double buffering), reused for the group reduction
  static size_t smem(int su, int sv) {
    const size_t stage = 2 * (size_t)(su + sv) * LD, red = G > 1 ? (size_t)G * su * sv : 0;
    return sizeof(double) * std::max(stage, red) + sizeof(long long) * (KB + su + sv);
  }
};

template <int TU, int TV, int IU, int JV>
__global__ void __launch_bounds__(256) lob_gram_kernel(const GramArgs g, double* __restrict__ part) {
  if (g.gate && *g.gate) return;
  using Cfg = GramCfg<TU, TV, IU, JV>;
  constexpr int G = Cfg::G, KB = Cfg::KB, LD = Cfg::LD;
  extern __shared__ double gsm[];
  const int su = g.nu * g.nb, sv = g.nv * g.nb;
  const size_t stage = (size_t)(su + sv) * LD, redsz = G > 1 ? (size_t)G * su * sv : 0;
  const size_t dbl = 2 * stage > redsz ? 2 * stage : redsz;
  long long* koff = reinterpret_cast<long long*>(gsm + dbl);   // (unused slot kept for layout)
  const double** rptr = reinterpret_cast<const double**>(koff + KB);   // [su + sv] columns
  const int tid = threadIdx.x, grp = tid / (TU * TV), t2 = tid - grp * (TU * TV);
  const int tu = t2 % TU, tv = t2 / TU;
  if (tid == 0) {   // column r of the staged operands: its block's base + column offset
    for (int r = 0; r < su + sv; ++r) {
      const int q = (r < su ? r : r - su) / g.nb, p = (r < su ? r : r - su) - q * g.nb;
      const double* base = r < su ? (q == 0 ? g.U[0] : q == 1 ? g.U[1] : g.U[2])
                                  : (q == 0 ? g.V[0] : q == 1 ? g.V[1] : q == 2 ? g.V[2]
                                     : q == 3 ? g.V[3] : q == 4 ? g.V[4] : g.V[5]);
      rptr[r] = base + (long long)p * g.rr;
    }
  }
  __syncthreads();
  double acc[IU][JV];
#pragma unroll
  for (int i = 0; i < IU; ++i)
#pragma unroll
    for (int j = 0; j < JV; ++j) acc[i][j] = 0.0;
  const long long k0 = blockIdx.x * g.k_per_chunk;
  const long long k1 = min(g.kt, k0 + g.k_per_chunk);
  // Chunk kb -> staging buffer: every thread always stages contraction index bb = tid % 32 of
  // columns r = tid / 32 + 8 i (coalesced 256-byte runs along the b index), by 8-byte
  // cp.async with zero fill past k1; the next chunk's copies fly while this one is reduced.
  const int bb_t = tid & 31, r_t = tid >> 5;
  auto stage_chunk = [&](long long kb, double* buf) {
    const long long k = kb + bb_t;
    const bool in = k < k1;
    long long off = 0;
    if (in) {
      if (g.k32) {   // the division of every staged index is the kernel's largest cost otherwise
        const uint32_t row = tt::fdiv((uint32_t)k, g.rrdiv);
        off = (long long)row * g.nb * g.rr + ((uint32_t)k - row * (uint32_t)g.rr);
      } else {
        off = (k / g.rr) * (long long)g.nb * g.rr + (k % g.rr);
      }
    }
    for (int r = r_t; r < su + sv; r += 8) {
      double* dst = (r < su ? buf + r * LD : buf + su * LD + (r - su) * LD) + bb_t;
      tt::cp_async8(dst, rptr[r] + off, in);
    }
    tt::cp_async_commit();
  };
  if (k0 < k1) stage_chunk(k0, gsm);
  int cur = 0;
  for (long long kb = k0; kb < k1; kb += KB, cur ^= 1) {
    if (kb + KB < k1) {
      stage_chunk(kb + KB, gsm + (cur ^ 1) * stage);
      tt::cp_async_wait<1>();
    } else {
      tt::cp_async_wait<0>();
    }
    __syncthreads();
    const double* Us = gsm + cur * stage;
    const double* Vs = Us + su * LD;
#pragma unroll 2
    for (int bb = grp; bb < KB; bb += G) {
      double u[IU], v[JV];
#pragma unroll
      for (int i = 0; i < IU; ++i) u[i] = (tu + TU * i < su) ? Us[(tu + TU * i) * LD + bb] : 0.0;
#pragma unroll
      for (int j = 0; j < JV; ++j) v[j] = (tv + TV * j < sv) ? Vs[(tv + TV * j) * LD + bb] : 0.0;
#pragma unroll
      for (int i = 0; i < IU; ++i)
#pragma unroll
        for (int j = 0; j < JV; ++j) acc[i][j] = fma(u[i], v[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* out = part + (long long)blockIdx.x * su * sv;
  if (G == 1) {
#pragma unroll
    for (int i = 0; i < IU; ++i)
#pragma unroll
      for (int j = 0; j < JV; ++j)
        if (tu + TU * i < su && tv + TV * j < sv) out[(tu + TU * i) * sv + tv + TV * j] = acc[i][j];
    return;
  }
  double* red = gsm;   // [G][su][sv] (the staging area is free after the last barrier)
#pragma unroll
  for (int i = 0; i < IU; ++i)
#pragma unroll
    for (int j = 0; j < JV; ++j)
      if (tu + TU * i < su && tv + TV * j < sv)
        red[((size_t)grp * su + tu + TU * i) * sv + tv + TV * j] = acc[i][j];
  __syncthreads();
  for (int e = tid; e < su * sv; e += 256) {
    double v = 0.0;
    for (int q = 0; q < G; ++q) v += red[(size_t)q * su * sv + e];
    out[e] = v;
  }
}

// G[e] = sum_c part[c][e]  (fixed order: deterministic)
// One warp per entry: lane l sums chunks l, l + 32, ... and the 32 partials are combined by a
// fixed shuffle tree (the summation order is fixed, so the result is deterministic).
__global__ void lob_gram_finish_kernel(const double* __restrict__ part, int chunks, int n,
                                       double* __restrict__ G, const int* __restrict__ gate) {
  if (gate && *gate) return;
  const int e = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (e >= n) return;
  double v = 0.0;
  for (int c = lane; c < chunks; c += 32) v += part[(long long)c * n + e];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) G[e] = v;
}

// Cyclic parallel Jacobi on a symmetric np x np matrix (np even) in shared memory, one CTA:
// round-robin pairs, rotation angles from the current matrix, then J^T M J applied in 2x2
// blocks (each block owns its four entries, so the update is in place) and V <- V J.
// The step is latency-bound (one dependent chain per step: pair -> angle -> update ->
// barrier), so the chain is kept short: the round-robin pair of a step needs no division
// (one conditional subtraction), the angle is t = sgn(d) e / (|d| + hypot(d, e)) with
// d = a_qq - a_pp, e = 2 a_pq (one sqrt, one division, one rsqrt instead of three divisions
// and two square roots), the rotation flag is a plain store, and every thread walks its
// update items with incremental indices (no integer division inside the step loop).
__device__ void lob_jacobi_cta(double* M, double* V, int np, double* cs, double* sn, int* pp,
                               int* qq, double* red) {
  const int tid = threadIdx.x, nt = blockDim.x, h = np / 2, n1 = np - 1;
  __shared__ int nrot;
  for (int e = tid; e < np * np; e += nt) V[e] = (e / np == e % np) ? 1.0 : 0.0;
  if (tid == 0) nrot = 1;
  // first update items of this thread and the stride between its items, as (row, col) pairs
  const int m_r0 = tid / h, m_c0 = tid - m_r0 * h, st_r = nt / h, st_c = nt - st_r * h;
  __syncthreads();
  for (int sw = 0; sw < 60; ++sw) {
    // a sweep that applied no rotation (every off-diagonal entry negligible against its
    // diagonal pair) ends the iteration; so does a negligible off-diagonal mass
    if (nrot == 0) break;
    double off = 0.0, dia = 0.0;
    for (int e = tid; e < np * np; e += nt) {
      const double v = M[e];
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
    double offs = 0.0, dias = 0.0;
    for (int w = 0; w < nt / 32; ++w) {
      offs += red[2 * w];
      dias += red[2 * w + 1];
    }
    __syncthreads();
    if (!(offs > 1e-30 * dias)) break;   // also stops on an all-zero matrix
    // an entry is negligible below 1e-15 sqrt(|a_pp a_qq|) (the classical threshold: relative
    // accuracy) or below 1e-17 ||M||_F (rounding noise of the matrix itself)
    const double floor_abs = 1e-17 * sqrt(offs + dias);
    if (tid == 0) nrot = 0;
    __syncthreads();
    for (int step = 0; step < n1; ++step) {
      for (int k = tid; k < h; k += nt) {
        int a = 0, b;
        if (k > 0) {
          a = k - 1 + step;
          if (a >= n1) a -= n1;
          a += 1;
        }
        b = n1 - 1 - k + step;
        if (b >= n1) b -= n1;
        b += 1;
        if (a > b) { const int t = a; a = b; b = t; }
        pp[k] = a;
        qq[k] = b;
        double c = 1.0, s = 0.0;
        const double apq = M[a * np + b], app = M[a * np + a], aqq = M[b * np + b];
        if (apq * apq > 1e-30 * fabs(app * aqq) && fabs(apq) > floor_abs) {
          const double d = aqq - app, e2 = 2.0 * apq;
          const double r = sqrt(fma(d, d, e2 * e2));
          const double t = (d >= 0.0 ? e2 : -e2) / (fabs(d) + r);
          if (t != 0.0) {
            c = rsqrt(fma(t, t, 1.0));
            s = t * c;
            nrot = 1;
          }
        }
        cs[k] = c;
        sn[k] = s;
      }
      __syncthreads();
      for (int kr = m_r0, kc = m_c0; kr < h;) {
        const int p = pp[kr], q = qq[kr], u = pp[kc], w = qq[kc];
        const double cr = cs[kr], sr = sn[kr], cc = cs[kc], sc = sn[kc];
        if (sr != 0.0 || sc != 0.0) {
          const double mpu = M[p * np + u], mpw = M[p * np + w];
          const double mqu = M[q * np + u], mqw = M[q * np + w];
          const double rpu = cr * mpu - sr * mqu, rpw = cr * mpw - sr * mqw;
          const double rqu = sr * mpu + cr * mqu, rqw = sr * mpw + cr * mqw;
          M[p * np + u] = cc * rpu - sc * rpw;
          M[p * np + w] = sc * rpu + cc * rpw;
          M[q * np + u] = cc * rqu - sc * rqw;
          M[q * np + w] = sc * rqu + cc * rqw;
        }
        kr += st_r;
        kc += st_c;
        if (kc >= h) { kc -= h; ++kr; }
      }
      // V <- V J: items (row i, pair kc) over np x h, the same incremental walk
      for (int i = m_r0, kc = m_c0; i < np;) {
        const int u = pp[kc], w = qq[kc];
        const double vu = V[i * np + u], vw = V[i * np + w];
        V[i * np + u] = cs[kc] * vu - sn[kc] * vw;
        V[i * np + w] = sn[kc] * vu + cs[kc] * vw;
        i += st_r;
        kc += st_c;
        if (kc >= h) { kc -= h; ++i; }
      }
      __syncthreads();
    }
  }
}

// Shared-memory layout of the Rayleigh-Ritz kernel (doubles first, then ints):
//   Dg[np] cs[np/2] sn[np/2] red[16] Dn[nbp] | M0[np^2] M1[np^2] M2[np^2] extra | ints
// The P-coefficient step reuses M1.. as scratch: Cp, Tmp (s x nb each), N, U, H (nbp^2 each).
struct RrLayout {
  int np, nbp;
  size_t small, mats, extra, ints;
  __host__ __device__ size_t bytes() const { return sizeof(double) * (small + mats + extra) + sizeof(int) * ints; }
};
__host__ __device__ RrLayout rr_layout(int s, int nb) {
  RrLayout L;
  L.np = (s + 1) & ~1;
  L.nbp = (nb + 1) & ~1;
  L.small = (size_t)L.np + L.np + 16 + L.nbp;
  L.mats = 3 * (size_t)L.np * L.np;
  const long long need = 2LL * s * nb + 3LL * L.nbp * L.nbp;
  const long long have = 2LL * L.np * L.np;
  L.extra = (size_t)(need > have ? need - have : 0);
  L.ints = 3 * (size_t)L.np;
  return L;
}
size_t lob_rr_smem(int s, int nb) { return rr_layout(s, nb).bytes(); }

// Rayleigh-Ritz on S = [X W P] (s = nblk nb columns) from G = [G_A | G_B] (s x 2s), one CTA:
//   Y (s x nb) = D T V[:, top nb] (L_B-orthonormal Ritz coefficients) and the Ritz values;
//   with_p: Yp (s x nb), the coefficients of the next P: Y with its X rows zeroed,
//   G_B-orthogonalised against Y twice and G_B-orthonormalised (SVQB, near-dependent
//   directions dropped) -- so P is L_B-orthonormal and L_B-orthogonal to the new X, which
//   keeps the next Gram matrix well conditioned (cf. Duersch et al. 2018).
__global__ void __launch_bounds__(256) lob_rr_kernel(const double* __restrict__ G, int s, int nb,
                                                     double* __restrict__ Y,
                                                     double* __restrict__ Yp,
                                                     double* __restrict__ lam,
                                                     long long* __restrict__ its, int count,
                                                     const int* __restrict__ gate) {
  if (gate && *gate) return;
  extern __shared__ double rsm[];
  const RrLayout Ly = rr_layout(s, nb);
  const int np = Ly.np, nbp = Ly.nbp;
  double* Dg = rsm;
  double* cs = Dg + np;
  double* sn = cs + np / 2;
  double* red = sn + np / 2;
  double* Dn = red + 16;
  double* M0 = rsm + Ly.small;
  double* M1 = M0 + np * np;
  double* M2 = M1 + np * np;
  int* pp = reinterpret_cast<int*>(rsm + Ly.small + Ly.mats + Ly.extra);
  int* qq = pp + np / 2;
  int* keep = qq + np / 2;   // [np] (two arrays' worth: pp/qq are np/2 each)
  __shared__ int k_sh;
  const int tid = threadIdx.x, nt = blockDim.x, s2 = 2 * s;
  auto GA = [&](int i, int j) { return 0.5 * (G[i * s2 + j] + G[j * s2 + i]); };
  auto GB = [&](int i, int j) { return 0.5 * (G[i * s2 + s + j] + G[j * s2 + s + i]); };
  for (int i = tid; i < np; i += nt) {
    const double gb = i < s ? G[i * s2 + s + i] : 0.0;
    Dg[i] = gb > 0.0 ? 1.0 / sqrt(gb) : 0.0;
  }
  __syncthreads();
  // T with T^T G_B' T = I over the kept directions (G_B' = D G_B D, unit diagonal).  First
  // try a Cholesky factorisation G_B' = L L^T (T = L^{-T}; the basis is kept well conditioned
  // by construction: X L_B-orthonormal, W and P L_B-orthogonal to X, P L_B-orthonormal); on a
  // pivot below 1e-8 fall back to the eigen-decomposition G_B' = U mu U^T, T = U mu^{-1/2},
  // dropping mu <= 1e-12 mu_max (SVQB).  Zero columns (D = 0) are excluded either way.
  __shared__ int chol_ok;
  // attempt 0 on [X W P]; if G_B is too ill-conditioned for the Cholesky pivot test and P is
  // present, attempt 1 restarts without P (its columns get Dg = 0: excluded everywhere below,
  // so its Ritz coefficients are zero) -- the classical LOBPCG restart, which keeps runs past
  // convergence from drifting (nb = 32 on a 192-dimensional problem otherwise diverges)
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (tid == 0) {
      int k = 0;
      for (int i = 0; i < s; ++i)
        if (Dg[i] > 0.0) keep[k++] = i;
      k_sh = k;
      chol_ok = 1;
    }
    __syncthreads();
    const int kc = k_sh;
    // compacted equilibrated G_B over the nonzero columns -> M0 (kc x kc, ld np)
    for (int e = tid; e < kc * kc; e += nt) {
      const int i = e / kc, j = e - i * kc;
      M0[i * np + j] = GB(keep[i], keep[j]) * Dg[keep[i]] * Dg[keep[j]];
    }
    __syncthreads();
    for (int c = 0; c < kc; ++c) {   // right-looking Cholesky, lower triangle in place
      if (tid == 0) {
        const double d = M0[c * np + c];
        if (!(d > kLobPivot)) chol_ok = 0;
        M0[c * np + c] = d > 0.0 ? sqrt(d) : 1.0;
      }
      __syncthreads();
      if (!chol_ok) break;
      const double piv = M0[c * np + c];
      for (int i = c + 1 + tid; i < kc; i += nt) M0[i * np + c] /= piv;
      __syncthreads();
      for (int e = tid; e < (kc - c - 1) * (kc - c - 1); e += nt) {
        const int i = c + 1 + e / (kc - c - 1), j = c + 1 + e % (kc - c - 1);
        if (j <= i) M0[i * np + j] = fma(-M0[i * np + c], M0[j * np + c], M0[i * np + j]);
      }
      __syncthreads();
    }
    if (chol_ok) {
      // Z = L^{-1} (forward substitution, one column per thread) -> M1;  T = Z^T -> M2
      for (int j = tid; j < kc; j += nt) {
        for (int i = 0; i < kc; ++i) {
          double v = (i == j) ? 1.0 : 0.0;
          if (i >= j) {
            for (int l = j; l < i; ++l) v = fma(-M0[i * np + l], M1[l * np + j], v);
            v /= M0[i * np + i];
          } else {
            v = 0.0;
          }
          M1[i * np + j] = v;
        }
      }
      break;
    }
    if (s <= 2 * nb) break;
    for (int i = 2 * nb + tid; i < s; i += nt) Dg[i] = 0.0;   // restart without P
    __syncthreads();
  }
  __syncthreads();
  int k, kp;
  if (chol_ok) {
    k = k_sh;
    kp = (k + 1) & ~1;
    // T[q][c] = Z[c][pos(q)] for kept q (Z^T: row index of T is the original column q)
    for (int e = tid; e < np * kp; e += nt) M2[e] = 0.0;
    __syncthreads();
    for (int e = tid; e < k * k; e += nt) {
      const int r = e / k, c = e - r * k;   // r: position of the original column keep[r]
      M2[keep[r] * kp + c] = M1[c * np + r];
    }
  } else {
    // SVQB fallback: equilibrated G_B (unit diagonal on nonzero columns), zero-padded to np
    for (int e = tid; e < np * np; e += nt) {
      const int i = e / np, j = e - i * np;
      M0[e] = (i < s && j < s) ? GB(i, j) * Dg[i] * Dg[j] : 0.0;
    }
    __syncthreads();
    lob_jacobi_cta(M0, M1, np, cs, sn, pp, qq, red);
    __syncthreads();
    if (tid == 0) {
      double mx = 0.0;
      for (int i = 0; i < np; ++i) mx = fmax(mx, M0[i * np + i]);
      int kk = 0;
      for (int i = 0; i < np; ++i)
        if (mx > 0.0 && M0[i * np + i] > 1e-12 * mx) keep[kk++] = i;
      k_sh = kk;
    }
    __syncthreads();
    k = k_sh;
    kp = (k + 1) & ~1;
    // T = U[:, keep] mu^{-1/2}  -> M2 (np x kp, zero-padded)
    for (int e = tid; e < np * kp; e += nt) {
      const int i = e / kp, c = e - i * kp;
      M2[e] = c < k ? M1[i * np + keep[c]] / sqrt(M0[keep[c] * np + keep[c]]) : 0.0;
    }
  }
  __syncthreads();
  // equilibrated G_A -> M0
  for (int e = tid; e < np * np; e += nt) {
    const int i = e / np, j = e - i * np;
    M0[e] = (i < s && j < s) ? GA(i, j) * Dg[i] * Dg[j] : 0.0;
  }
  __syncthreads();
  // M1 = G_A T  (np x kp)
  for (int e = tid; e < np * kp; e += nt) {
    const int i = e / kp, c = e - i * kp;
    double v = 0.0;
    for (int q = 0; q < np; ++q) v = fma(M0[i * np + q], M2[q * kp + c], v);
    M1[e] = v;
  }
  __syncthreads();
  // M0 = T^T M1  (kp x kp; G_A is no longer needed), then symmetrised in place
  for (int e = tid; e < kp * kp; e += nt) {
    const int i = e / kp, j = e - i * kp;
    double v = 0.0;
    for (int q = 0; q < np; ++q) v = fma(M2[q * kp + i], M1[q * kp + j], v);
    M0[e] = v;
  }
  __syncthreads();
  for (int e = tid; e < kp * kp; e += nt) {
    const int i = e / kp, j = e - i * kp;
    if (i < j) {
      const double v = 0.5 * (M0[i * kp + j] + M0[j * kp + i]);
      M0[i * kp + j] = v;
      M0[j * kp + i] = v;
    }
  }
  __syncthreads();
  lob_jacobi_cta(M0, M1, kp, cs, sn, pp, qq, red);
  __syncthreads();
  // order the k genuine Ritz values (the padding index, if any, is excluded), descending
  if (tid == 0) {
    for (int i = 0; i < k; ++i) keep[i] = i;
    for (int i = 1; i < k; ++i) {   // insertion sort, stable
      const int v = keep[i];
      const double tv = M0[v * kp + v];
      int j = i - 1;
      while (j >= 0 && M0[keep[j] * kp + keep[j]] < tv) {
        keep[j + 1] = keep[j];
        --j;
      }
      keep[j + 1] = v;
    }
  }
  __syncthreads();
  for (int m = tid; m < nb; m += nt) lam[m] = m < k ? M0[keep[m] * kp + keep[m]] : 0.0;
  __syncthreads();
  // Y[q][m] = Dg[q] sum_c T[q][c] V[c][keep[m]]   (into M0, which is free now, and global)
  double* Ys = M0;
  for (int e = tid; e < s * nb; e += nt) {
    const int q = e / nb, m = e - q * nb;
    double v = 0.0;
    if (m < k)
      for (int c = 0; c < k; ++c) v = fma(M2[q * kp + c], M1[c * kp + keep[m]], v);
    v *= Dg[q];
    Ys[e] = v;
    Y[e] = v;
  }
  if (tid == 0 && count) ++its[0];
  if (!Yp) return;
  __syncthreads();
  // ---- P coefficients (scratch from M1 on: M1, M2 and the extra area are contiguous) ----
  double* Cp = M1;
  double* Tmp = Cp + s * nb;
  double* Nm = Tmp + s * nb;
  double* Um = Nm + nbp * nbp;
  double* H = Um + nbp * nbp;
  for (int e = tid; e < s * nb; e += nt) Cp[e] = (e / nb) < nb ? 0.0 : Ys[e];
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (int e = tid; e < s * nb; e += nt) {   // Tmp = G_B Cp
      const int i = e / nb, m = e - i * nb;
      double v = 0.0;
      for (int j = 0; j < s; ++j) v = fma(GB(i, j), Cp[j * nb + m], v);
      Tmp[e] = v;
    }
    __syncthreads();
    for (int e = tid; e < nb * nb; e += nt) {  // H = Y^T G_B Cp
      const int a = e / nb, m = e - a * nb;
      double v = 0.0;
      for (int q = 0; q < s; ++q) v = fma(Ys[q * nb + a], Tmp[q * nb + m], v);
      H[e] = v;
    }
    __syncthreads();
    for (int e = tid; e < s * nb; e += nt) {   // Cp -= Y H
      const int q = e / nb, m = e - q * nb;
      double v = Cp[e];
      for (int a = 0; a < nb; ++a) v = fma(-Ys[q * nb + a], H[a * nb + m], v);
      Cp[e] = v;
    }
    __syncthreads();
  }
  for (int e = tid; e < s * nb; e += nt) {     // Tmp = G_B Cp
    const int i = e / nb, m = e - i * nb;
    double v = 0.0;
    for (int j = 0; j < s; ++j) v = fma(GB(i, j), Cp[j * nb + m], v);
    Tmp[e] = v;
  }
  __syncthreads();
  for (int e = tid; e < nb * nb; e += nt) {    // H = Cp^T G_B Cp
    const int a = e / nb, m = e - a * nb;
    double v = 0.0;
    for (int q = 0; q < s; ++q) v = fma(Cp[q * nb + a], Tmp[q * nb + m], v);
    H[e] = v;
  }
  __syncthreads();
  for (int i = tid; i < nbp; i += nt) Dn[i] = (i < nb && H[i * nb + i] > 0.0) ? 1.0 / sqrt(H[i * nb + i]) : 0.0;
  __syncthreads();
  for (int e = tid; e < nbp * nbp; e += nt) {
    const int i = e / nbp, j = e - i * nbp;
    Nm[e] = (i < nb && j < nb) ? 0.5 * (H[i * nb + j] + H[j * nb + i]) * Dn[i] * Dn[j] : 0.0;
  }
  __syncthreads();
  lob_jacobi_cta(Nm, Um, nbp, cs, sn, pp, qq, red);
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int i = 0; i < nbp; ++i) mx = fmax(mx, Nm[i * nbp + i]);
    int kk = 0;
    for (int i = 0; i < nbp; ++i)
      if (mx > 0.0 && Nm[i * nbp + i] > 1e-12 * mx) keep[kk++] = i;
    k_sh = kk;
  }
  __syncthreads();
  const int kk = k_sh;
  // Yp[:, c] = Cp Dn U[:, keep[c]] / sqrt(mu) for the kept directions, zero beyond
  for (int e = tid; e < s * nb; e += nt) {
    const int q = e / nb, c = e - q * nb;
    double v = 0.0;
    if (c < kk) {
      const int u = keep[c];
      for (int a = 0; a < nb; ++a) v = fma(Cp[q * nb + a] * Dn[a], Um[a * nbp + u], v);
      v /= sqrt(Nm[u * nbp + u]);
    }
    Yp[e] = v;
  }
}

// Linear combinations: for every family f (X, AX, BX images) and position (row, b):
//   Xn_f[row, m, b] = sum_q sum_p S_f,q[row, p, b] Y[q nb + p, m]     (q over X, W, P)
//   Pn_f[row, m, b] = sum_q sum_p S_f,q[row, p, b] Yp[q nb + p, m]    (if Yp)
// In place (Xn_f = S_f,0, Pn_f = S_f,2): a thread reads every S_f,q[row, :, b] of its (row, b)
// positions before it writes Xn_f / Pn_f there, and no other thread touches them.
struct CombineArgs {
  const double* S[3][3];
  double* Xn[3];
  double* Pn[3];
  int nfam, nblk, nb, rr;
  long long rows;
  const double* Y;
  const double* Yp;
  const int* gate;
};

// NBT: compile-time bound on nb (accumulators); TB: consecutive b positions per thread
// (TB = 2 uses 16-byte loads/stores; needs rr even)
template <int NBT, int TB>
__global__ void __launch_bounds__(128) lob_combine_kernel(const CombineArgs a) {
  if (a.gate && *a.gate) return;
  extern __shared__ double csm[];
  const int s = a.nblk * a.nb, nb = a.nb;
  double* Ys = csm;
  double* Yps = csm + s * nb;
  for (int i = threadIdx.x; i < s * nb; i += blockDim.x) {
    Ys[i] = a.Y[i];
    if (a.Yp) Yps[i] = a.Yp[i];
  }
  __syncthreads();
  const long long rrt = a.rr / TB, total = a.rows * rrt;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / rrt, b = (e - row * rrt) * TB;
    for (int f = 0; f < a.nfam; ++f) {
      double ax[NBT][TB], ap[NBT][TB];
#pragma unroll
      for (int m = 0; m < NBT; ++m)
#pragma unroll
        for (int t = 0; t < TB; ++t) ax[m][t] = ap[m][t] = 0.0;
      for (int q = 0; q < a.nblk; ++q) {
        const double* src = a.S[f][q] + row * nb * a.rr + b;
#pragma unroll
        for (int p = 0; p < NBT; ++p) {
          if (p >= nb) break;
          double v[TB];
          if (TB == 2) {
            const double2 w = *reinterpret_cast<const double2*>(src + (long long)p * a.rr);
            v[0] = w.x;
            v[TB - 1] = w.y;
          } else {
            v[0] = src[(long long)p * a.rr];
          }
          const double* y = Ys + (q * nb + p) * nb;
          const double* yp = Yps + (q * nb + p) * nb;
#pragma unroll
          for (int m = 0; m < NBT; ++m)
            if (m < nb) {
              const double ym = y[m];
#pragma unroll
              for (int t = 0; t < TB; ++t) ax[m][t] = fma(v[t], ym, ax[m][t]);
              if (a.Yp) {
                const double ypm = yp[m];
#pragma unroll
                for (int t = 0; t < TB; ++t) ap[m][t] = fma(v[t], ypm, ap[m][t]);
              }
            }
        }
      }
      double* xo = a.Xn[f] + row * nb * a.rr + b;
      double* po = a.Yp ? a.Pn[f] + row * nb * a.rr + b : nullptr;
#pragma unroll
      for (int m = 0; m < NBT; ++m)
        if (m < nb) {
          if (TB == 2) {
            *reinterpret_cast<double2*>(xo + (long long)m * a.rr) = make_double2(ax[m][0], ax[m][TB - 1]);
            if (po) *reinterpret_cast<double2*>(po + (long long)m * a.rr) = make_double2(ap[m][0], ap[m][TB - 1]);
          } else {
            xo[(long long)m * a.rr] = ax[m][0];
            if (po) po[(long long)m * a.rr] = ap[m][0];
          }
        }
    }
  }
}

// W[row, m, b] -= sum_p X[row, p, b] C[p, m]   (in place; one thread per (row, b)).  NBT: a
// compile-time bound on nb, so the loads of a thread's nb values are unrolled and independent.
// With sc != nullptr the result columns are then scaled: W[:, m, :] *= sc[m] (the residual
// normalisation folded into the first pass: (W - X C) D = W D - X (C D)).
template <int NBT>
__global__ void __launch_bounds__(128) lob_orth_kernel(const double* __restrict__ X,
                                                       const double* __restrict__ C,
                                                       double* __restrict__ W, long long rows,
                                                       int nb, int rr, const double* __restrict__ sc,
                                                       const int* __restrict__ gate) {
  if (gate && *gate) return;
  __shared__ double Cs[NBT * NBT];
  __shared__ double Ds[NBT];
  for (int i = threadIdx.x; i < NBT * NBT; i += blockDim.x) {
    const int p = i / NBT, m = i - p * NBT;
    Cs[i] = (p < nb && m < nb) ? C[p * nb + m] : 0.0;
  }
  for (int i = threadIdx.x; i < NBT; i += blockDim.x) Ds[i] = (sc && i < nb) ? sc[i] : 1.0;
  __syncthreads();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < rows * rr;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / rr, b = e - row * rr;
    const double* x = X + row * nb * rr + b;
    double* w = W + row * nb * rr + b;
    double xv[NBT], acc[NBT];
#pragma unroll
    for (int p = 0; p < NBT; ++p) xv[p] = p < nb ? x[(long long)p * rr] : 0.0;
#pragma unroll
    for (int m = 0; m < NBT; ++m) acc[m] = m < nb ? w[(long long)m * rr] : 0.0;
#pragma unroll
    for (int p = 0; p < NBT; ++p)
#pragma unroll
      for (int m = 0; m < NBT; ++m) acc[m] = fma(-xv[p], Cs[p * NBT + m], acc[m]);
#pragma unroll
    for (int m = 0; m < NBT; ++m)
      if (m < nb) w[(long long)m * rr] = acc[m] * Ds[m];
  }
}

// workspace element counts beyond the matvec's (T1, T2, Pp shared; one Ahat per operator)
struct LobWs {
  long long blocks;   // 8 blocks of S: AX BX W AW BW P AP BP (the combination is in place)
  long long part, gpart, G, Y, small;
};

bool lob_ws_elems(const Dims& d, long long nb, LobWs& w) {
  bool ok = true;
  const long long S = prod({d.a, d.n, nb, d.b}, ok);
  w.blocks = prod({8, S}, ok);
  const LobDims L = lob_dims(d, nb);
  const long long s = 3 * nb;
  w.part = 3 * nb * (long long)L.chunks;
  w.gpart = prod({(long long)L.gchunks, s, 2 * s}, ok);
  w.G = s * 2 * s;
  w.Y = 2 * s * nb + nb * nb;   // Y, Yp, and the W-orthogonalisation coefficients
  w.small = 2 * nb + 8;
  return ok;
}

// opt-in shared memory of the kernels that can exceed 48 KB (per device)
cudaError_t lob_set_smem_attrs() {
  cudaError_t err = smem_attr((const void*)lob_gram_kernel<16, 16, 6, 12>,
                              (int)GramCfg<16, 16, 6, 12>::smem(kLobMaxS, 2 * kLobMaxS));
  if (err == cudaSuccess)
    err = smem_attr((const void*)lob_gram_kernel<16, 8, 3, 12>, (int)GramCfg<16, 8, 3, 12>::smem(48, 96));
  if (err == cudaSuccess)
    err = smem_attr((const void*)lob_rr_kernel, (int)lob_rr_smem(kLobMaxS, kLobMaxNb));
  for (auto fn : {lob_combine_kernel<16, 1>, lob_combine_kernel<16, 2>, lob_combine_kernel<32, 1>})
    if (err == cudaSuccess)
      err = smem_attr((const void*)fn, (int)(sizeof(double) * 2 * kLobMaxS * kLobMaxNb));
  return err;
}

// the launch sequence (no synchronisation).  refresh > 0: every `refresh` iterations the
// carried images A X, B X, A P, B P are recomputed by matvecs (the linear-combination updates
// accumulate rounding that otherwise corrupts the Gram matrices once the residual is small).
cudaError_t enqueue_lobpcg(const Dims& dA, const Dims& dB, bool has_B, long long nb,
                           long long maxiter, long long refresh, double tol, const double* phiLA,
                           const double* AA, const double* phiRA, const double* phiLB,
                           const double* AB, const double* phiRB, double* X, double* lam,
                           double* res, long long* its, double* step, void* workspace,
                           size_t wsb, cudaStream_t s) {
  long long t1a, t2a, aha, pea, t1b = 0, t2b = 0, ahb = 0, peb = 0;
  matvec_ws_elems(dA, nb, t1a, t2a, aha, pea);
  if (has_B) matvec_ws_elems(dB, nb, t1b, t2b, ahb, peb);
  LobWs lw;
  lob_ws_elems(dA, nb, lw);
  Carver c{static_cast<char*>(workspace), wsb};
  double* T1 = c.take(std::max(t1a, t1b));
  double* T2 = c.take(std::max(t2a, t2b));
  const long long pe = std::max(pea, peb);
  double* Pp = c.take(pe);
  double* AhA = c.take(aha);
  double* AhB = has_B ? c.take(ahb) : nullptr;
  double* blk = c.take(lw.blocks);
  double* part = c.take(lw.part);
  double* gpart = c.take(lw.gpart);
  double* G = c.take(lw.G);
  double* Y = c.take(lw.Y);
  double* sm = c.take(lw.small);
  if (!c.ok) return cudaErrorInvalidValue;
  double* Yp = Y + 3 * nb * nb;
  double* Cw = Yp + 3 * nb * nb;
  const LobDims L = lob_dims(dA, nb);
  const long long S = L.S;
  double* AX = blk;
  double* BX = blk + S;
  double* W = blk + 2 * S;
  double* AW = blk + 3 * S;
  double* BW = blk + 4 * S;
  double* P = blk + 5 * S;
  double* AP = blk + 6 * S;
  double* BP = blk + 7 * S;
  if (!has_B) {   // B = I: the B images are the blocks themselves
    BX = X;
    BW = W;
    BP = P;
  }
  LobState st;
  st.lam = lam;
  st.res = res;
  st.scale = sm;
  st.done = reinterpret_cast<int*>(sm + nb);
  st.its = its;
  st.step = step;
  cudaError_t e;
  if ((e = lob_set_smem_attrs()) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(sm, 0, sizeof(double) * lw.small, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(its, 0, sizeof(long long), s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(lam, 0, sizeof(double) * nb, s)) != cudaSuccess) return e;
  g_stage = TT_ST_PERM;
  if ((e = launch_perm(true, AA, AhA, dA.al, dA.n, dA.be, s)) != cudaSuccess) return e;
  if (has_B && (e = launch_perm(true, AB, AhB, dB.al, dB.n, dB.be, s)) != cudaSuccess) return e;
  const int* gate = st.done;
  struct GateScope {
    GateScope(const int* g) { g_gate = g; }
    ~GateScope() { g_gate = nullptr; }
  } gscope(gate);
  auto matvecs = [&](const double* in, double* outA, double* outB) -> cudaError_t {
    cudaError_t r = enqueue_matvec(dA, nb, phiLA, AA, phiRA, in, outA, T1, T2, AhA, Pp, pe, s, AhA);
    if (r != cudaSuccess || !has_B) return r;
    return enqueue_matvec(dB, nb, phiLB, AB, phiRB, in, outB, T1, T2, AhB, Pp, pe, s, AhB);
  };
  long long eb = (S + 255) / 256;
  eb = std::min<long long>(std::max(1LL, eb), 8LL * num_sms());
  long long cb = (L.rows * L.rr + 127) / 128;
  cb = std::min<long long>(std::max(1LL, cb), 16LL * num_sms());
  // Gram matrices of nu U blocks against nv V blocks -> out (nu nb x nv nb)
  auto gram = [&](int nu, const double* const* U, int nv, const double* const* V,
                  double* out) -> cudaError_t {
    GramArgs ga;
    for (int q = 0; q < 3; ++q) ga.U[q] = q < nu ? U[q] : nullptr;
    for (int q = 0; q < 6; ++q) ga.V[q] = q < nv ? V[q] : nullptr;
    ga.nu = nu;
    ga.nv = nv;
    ga.nb = (int)nb;
    ga.rr = L.rr;
    ga.kt = L.rows * L.rr;
    ga.k_per_chunk = L.k_per_gchunk;
    ga.gate = gate;
    ga.k32 = ga.kt < (1LL << 31) ? 1 : 0;
    ga.rrdiv = tt::make_fastdiv((uint32_t)L.rr);
    const int su = nu * (int)nb, sv = nv * (int)nb;
    if (su <= 8 && sv <= 8) {   // the orthogonalisation Gram X^T B W: 8 x 8 exactly, 32 groups
      using C = GramCfg<4, 2, 2, 4>;
      lob_gram_kernel<4, 2, 2, 4><<<L.gchunks, 256, C::smem(su, sv), s>>>(ga, gpart);
    } else if (su <= 12 && sv <= 24) {
      using C = GramCfg<4, 4, 3, 6>;
      lob_gram_kernel<4, 4, 3, 6><<<L.gchunks, 256, C::smem(su, sv), s>>>(ga, gpart);
    } else if (su <= 24 && sv <= 48) {
      using C = GramCfg<8, 8, 3, 6>;
      lob_gram_kernel<8, 8, 3, 6><<<L.gchunks, 256, C::smem(su, sv), s>>>(ga, gpart);
    } else if (su <= 48 && sv <= 96) {
      using C = GramCfg<16, 8, 3, 12>;
      lob_gram_kernel<16, 8, 3, 12><<<L.gchunks, 256, C::smem(su, sv), s>>>(ga, gpart);
    } else {
      using C = GramCfg<16, 16, 6, 12>;
      lob_gram_kernel<16, 16, 6, 12><<<L.gchunks, 256, C::smem(su, sv), s>>>(ga, gpart);
    }
    ++g_launches;
    const int n = su * sv;
    lob_gram_finish_kernel<<<(n + 7) / 8, 256, 0, s>>>(gpart, L.gchunks, n, out, gate);
    ++g_launches;
    return cudaGetLastError();
  };
  auto gram_rr = [&](int nblk, int count) -> cudaError_t {
    const double* U[3] = {X, W, P};
    const double* V[6] = {AX, AW, AP, BX, BW, BP};
    const double* Vc[6];
    for (int q = 0; q < nblk; ++q) {
      Vc[q] = V[q];
      Vc[nblk + q] = V[3 + q];
    }
    cudaError_t r = gram(nblk, U, 2 * nblk, Vc, G);
    if (r != cudaSuccess) return r;
    const int sdim = nblk * (int)nb;
    lob_rr_kernel<<<1, 256, lob_rr_smem(sdim, (int)nb), s>>>(G, sdim, (int)nb, Y,
                                                             nblk > 1 ? Yp : nullptr, lam, its,
                                                             count, gate);
    ++g_launches;
    return cudaGetLastError();
  };
  auto combine = [&](int nblk) -> cudaError_t {
    CombineArgs ca;
    const double* fam[3][3] = {{X, W, P}, {AX, AW, AP}, {BX, BW, BP}};
    double* xn[3] = {X, AX, BX};   // in place (lob_combine_kernel)
    double* pn[3] = {P, AP, BP};
    ca.nfam = has_B ? 3 : 2;
    for (int f = 0; f < 3; ++f) {
      for (int q = 0; q < 3; ++q) ca.S[f][q] = fam[f][q];
      ca.Xn[f] = xn[f];
      ca.Pn[f] = pn[f];
    }
    ca.nblk = nblk;
    ca.nb = (int)nb;
    ca.rr = L.rr;
    ca.rows = L.rows;
    ca.Y = Y;
    ca.Yp = nblk > 1 ? Yp : nullptr;
    ca.gate = gate;
    const size_t smem = sizeof(double) * 2 * (size_t)nblk * nb * nb;
    const bool tb2 = (L.rr % 2) == 0 && nb <= 16;   // 32 x 2 accumulators would spill
    long long cb2 = (L.rows * (tb2 ? L.rr / 2 : L.rr) + 127) / 128;
    cb2 = std::min<long long>(std::max(1LL, cb2), 16LL * num_sms());
#define LOB_COMBINE(NBT)                                                              \
  do {                                                                                \
    if (tb2) lob_combine_kernel<NBT, 2><<<(unsigned)cb2, 128, smem, s>>>(ca);          \
    else lob_combine_kernel<NBT, 1><<<(unsigned)cb2, 128, smem, s>>>(ca);              \
  } while (0)
    if (nb <= 4) LOB_COMBINE(4);
    else if (nb <= 8) LOB_COMBINE(8);
    else if (nb <= 16) LOB_COMBINE(16);
    else lob_combine_kernel<32, 1><<<(unsigned)cb2, 128, smem, s>>>(ca);
#undef LOB_COMBINE
    ++g_launches;
    return cudaGetLastError();
  };
  auto check = [&](int final_pass) -> cudaError_t {
    const int* g2 = final_pass ? nullptr : gate;
    dim3 grid(L.chunks, (unsigned)nb);
    lob_colnorm_kernel<<<grid, 256, 0, s>>>(W, AX, BX, lam, L.rows, (int)nb, L.rr,
                                            L.rows_per_chunk, part, g2);
    ++g_launches;
    lob_check_kernel<<<1, 1024, 0, s>>>(part, L.chunks, (int)nb, st, tol, final_pass);
    ++g_launches;
    return cudaGetLastError();
  };
  // initial Rayleigh-Ritz on X alone
  if ((e = matvecs(X, AX, BX)) != cudaSuccess) return e;
  if ((e = gram_rr(1, 0)) != cudaSuccess) return e;
  if ((e = combine(1)) != cudaSuccess) return e;
  for (long long it = 0; it < maxiter; ++it) {
    const int nblk = it == 0 ? 2 : 3;
    if (refresh > 0 && it > 0 && it % refresh == 0) {
      if ((e = matvecs(X, AX, BX)) != cudaSuccess) return e;
      if ((e = matvecs(P, AP, BP)) != cudaSuccess) return e;
    }
    if ((e = check(0)) != cudaSuccess) return e;
    for (int pass = 0; pass < 2; ++pass) {   // W <- W - X (B X)^T W, twice (pass 0 also scales)
      const double* U[1] = {BX};
      const double* V[1] = {W};
      const double* scp = pass == 0 ? st.scale : nullptr;
      if ((e = gram(1, U, 1, V, Cw)) != cudaSuccess) return e;
      if (nb <= 4) lob_orth_kernel<4><<<(unsigned)cb, 128, 0, s>>>(X, Cw, W, L.rows, (int)nb, L.rr, scp, gate);
      else if (nb <= 8) lob_orth_kernel<8><<<(unsigned)cb, 128, 0, s>>>(X, Cw, W, L.rows, (int)nb, L.rr, scp, gate);
      else if (nb <= 16) lob_orth_kernel<16><<<(unsigned)cb, 128, 0, s>>>(X, Cw, W, L.rows, (int)nb, L.rr, scp, gate);
      else lob_orth_kernel<32><<<(unsigned)cb, 128, 0, s>>>(X, Cw, W, L.rows, (int)nb, L.rr, scp, gate);
      ++g_launches;
    }
    if ((e = matvecs(W, AW, BW)) != cudaSuccess) return e;
    if ((e = gram_rr(nblk, 1)) != cudaSuccess) return e;
    if ((e = combine(nblk)) != cudaSuccess) return e;
  }
  return check(1);
}
