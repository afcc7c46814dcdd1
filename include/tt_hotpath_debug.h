/* tt_hotpath_debug.h -- test and benchmark hooks of libtt_hotpath.so.
 *
 * NOT part of the production ABI (include/tt_hotpath.h): these calls select alternative kernels,
 * tile configurations and scheduling paths of the calling thread for A/B measurements and
 * forced-path parity tests, or expose internal solvers to the tests.  Every path they select
 * computes the same results as the default (up to rounding order) and is parity-tested, except
 * the two result-corrupting timing bits of tt_debug_set_flags, which only a debug build
 * (-DTT_DEBUG_HOOKS) honours.  The probe environment variables (TT_LAT_*, TT_PDL_FLOPS,
 * TT_L2_DEBUG) are likewise read only by a debug build.
 */
#ifndef TT_HOTPATH_DEBUG_H
#define TT_HOTPATH_DEBUG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Test hook: eigendecomposition of a symmetric n x n matrix G (overwritten; n <= 2048) by the
 * rounding's parallel Jacobi solver (element-wise for n < 24, block Jacobi above; debug flag
 * 256 forces the element-wise kernel): V columns = eigenvectors, lam descending.  Workspace
 * >= max(4 ne^2, 2 nb^2 + 64 nb) + 8200 doubles, ne = n rounded up to even, nb = n rounded
 * up to a multiple of 64. */
tt_status tt_debug_sym_eigen(int64_t n, double* G, double* V, double* lam, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Test hook: on != 0 routes every GEMM stage of the calling thread through the generic
 * (unaligned-capable) kernel instead of the persistent 16-byte-load kernel. */
void tt_debug_force_v1(int on);
/* Benchmark hook: GEMM engine of the calling thread (-1 = default = 2; 0 = cp.async, one
 * 512-thread CTA per SM; 1 = cp.async, two 256-thread CTAs per SM; 2 = TMA + mbarrier). */
void tt_debug_set_variant(int v);
/* Benchmark hooks: bit 0 skips the GEMM output stores and bit 1 the operand loads (results
 * become WRONG; times the main loop / epilogue / load path in isolation) -- these two bits are
 * honoured only by a debug build (-DTT_DEBUG_HOOKS, `TT_DEBUG_HOOKS=1` at build time) and
 * masked off otherwise; bit 3 computes the
 * right interface update directly instead of as the mirrored left update (same result); bit 16
 * runs the Jacobi eigensolver's first block kernel (full inner sweeps, textbook rotations,
 * scalar updates) and bit 2 the current one with blocks of 32 instead of 16; bit 4
 * disables the TMA L2 cache-policy hints, bit 5 only the evict_first ones, bit 6 only the
 * evict_last ones, bit 7 issues M/N-contiguous tiles as 2-D boxes, bits 9/10 order the tiles
 * M-grouped by 8 / M-fastest, bit 8 forces the element-wise Jacobi (same results), bit 11
 * runs the W34 interface chains at the lowest stream priority, bit 12 disables programmatic
 * dependent launch, bit 13 the small-GEMM latency tile policy, bit 14 the one-k-tile warp skew
 * of the 16-warp GEMM tiles (bit 15: two k-tiles), bit 17 the 32-byte epilogue stores, bit 18
 * the shared-memory column-offset table of single-N-tile GEMMs, bit 19 the division-free unit
 * decode (ksplit == 1 / one N tile), bits 20 / 22 restore the 16-warp (8 x 2) tiles of the
 * operator-core / first matvec stages (bit 21: 2 x 6 warps), bit 23 runs tt_sweep_w34's
 * matvecs as three stages instead of reusing the left updates' T2_k, bit 25 runs the
 * operator-core stage with the whole A-hat resident in shared memory (3-deep T1 ring;
 * measured slower, kept as a probe), bit 24 forces tt_round's accurate truncation route
 * (Householder QR + cluster one-sided Jacobi SVD, otherwise used for delta / sqrt(d-1) < 1e-7), bit 26 runs tt_local_gmres's K = 1 orthogonalisation
 * step as separate kernels instead of the fused cluster kernel, bit 28 runs the small boundary
 * interface updates of the sweeps as three stage GEMMs each instead of fused one-CTA runs, bit 29
 * the orthonormalisation steps of tt_round / tt_orthonormalise through the Gram matrix instead
 * of the cluster Householder QR, bit 27 the operator apply with the register-blocked kernel instead
 * of the operator-stationary row-block kernel, bit 30 the 12- and 16-warp stage GEMM tiles with
 * thread 0 as the TMA producer instead of the round-robin producer (same results).
 * tt_debug_set_variant(v): v >= 10 forces
 * the GEMM tile configuration v % 100 (probe list in csrc/tt_launch_tpl.cuh) and split-K factor v / 100. */
void tt_debug_set_flags(int flags);
/* Benchmark hook: the experimental persistent DAG executor for tt_sweep_w34 on the calling
 * thread (one launch for the whole sweep, csrc/tt_dag.cuh): 0 = off (default: the stream/event
 * version, measured faster), 1 = on with 4-warp 64 x 64 tiles, 2 = 8-warp. */
void tt_debug_set_dag(int mode);
/* Benchmark / test hook: the fused S1 -> S2 matvec kernel (csrc/tt_fused12.cuh: T1 stays in
 * shared memory) on the calling thread: 0 = policy (default: TT_MATVEC_AUTO), -1 = never,
 * m > 0 = whenever the shape is eligible (workspaces sized without T1), with warp-group skew
 * {1, 0, 2}[(m - 1) % 3] k-tiles and option bits (m - 1) / 3: bit 0 keeps the barrier before
 * the hand-over, bit 1 two 6-warp CTAs per SM, bit 5 thread 0 as the TMA producer, bit 6 a
 * 13th producer warp (default: round-robin over the consumer warps); bits 2-4 are timing
 * probes of a debug build (no loads / no T2 stores / no hand-over: WRONG results).
 * m = 2 is what tt_set_matvec_mode(TT_MATVEC_FUSED) selects. */
void tt_debug_set_fused(int mode);
/* Measurement hook: while buf != NULL (device, 5 x uint64 per unit, cap_units units) the next
 * DAG launches of the calling thread record per unit {grab, ready, computed, published,
 * smid} (%globaltimer ns).  Copies the last DAG's per-task first-unit table into unit0 (host,
 * cap_tasks entries, + total) and returns (tasks << 32) | units of the last DAG launch. */
int64_t tt_debug_dag_trace(void* buf, int64_t cap_units, int32_t* unit0, int64_t cap_tasks);

/* Test hook: one-sided Jacobi SVD of a rows x c row-major matrix B (rows, c <= 256) in one
 * thread-block cluster (csrc/tt_qr.cuh): BJ = B J (rows x c, columns u_j sigma_j, unsorted),
 * J (c x c orthogonal), sigma (c), *sweeps (int32, device) the Jacobi sweeps run.  Device
 * pointers, asynchronous. */
tt_status tt_debug_svd(int64_t rows, int64_t c, const double* B, double* BJ, double* J,
                       double* sigma, int32_t* sweeps, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TT_HOTPATH_DEBUG_H */
