#!/bin/bash
# compute-sanitizer evidence: memcheck / racecheck / synccheck over
# smoke(), the config-1/2 parity tests, forced tile configurations (warp skew, split-K),
# ragged shapes, a small tt_round (cooperative Jacobi), LOBPCG and GMRES.
# usage: tools/sanitize.sh <memcheck|racecheck|synccheck|initcheck> [outdir]
set -u
TOOL=$1
OUT=${2:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS="compute-sanitizer --tool $TOOL --target-processes all --print-limit 200"
if [ "$TOOL" = memcheck ]; then CS="$CS --leak-check full"; fi
SEL_FULL='test_smoke or (test_config_w34_parity and (1-default or 2-default)) or (test_config_apply_parity and ([1] or [2])) or test_ragged or test_forced_tile_configs or test_sweep_als_small or (test_tt_round_vs_oracle and random) or (test_sweep_w34_call and ([1-0] or [2-0] or [2-8388608])) or test_identity_operator or test_single_core or test_rectangular or (test_local_gmres_vs_oracle and 2-3-4-12-2-0) or test_two_site_matvec or (test_block_local_matvec and 5-4-7-3) or (test_jacobi_eigen and ([7] or [65] or [129]))'
SEL_LIGHT='test_smoke or (test_config_w34_parity and 1-default) or (test_ragged_batched_matvec and (shape1 or shape2)) or (test_forced_tile_configs and ([1-1 or [3-2)) or (test_tt_round_vs_oracle and 0.01-random) or (test_local_gmres_vs_oracle and 2-3-4-12-2-0) or (test_jacobi_eigen and ([7] or [65]))'
SEL=$SEL_FULL
[ "$TOOL" != memcheck ] && SEL=$SEL_LIGHT
echo "== $TOOL smoke" > "$OUT/$TOOL.log"
timeout 900 $CS python __graft_entry__.py smoke >> "$OUT/$TOOL.log" 2>&1
echo "== rc=$?" >> "$OUT/$TOOL.log"
echo "== $TOOL pytest" >> "$OUT/$TOOL.log"
timeout 1800 $CS python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "$SEL" >> "$OUT/$TOOL.log" 2>&1
echo "== rc=$?" >> "$OUT/$TOOL.log"
echo "== $TOOL lobpcg" >> "$OUT/$TOOL.log"
timeout 900 $CS python -m pytest tests/test_gpu_lobpcg.py -q -m gpu -p no:cacheprovider -k "test_lobpcg_standard_vs_oracle or test_lobpcg_maxiter0 or test_lobpcg_early_stop" >> "$OUT/$TOOL.log" 2>&1
echo "== rc=$?" >> "$OUT/$TOOL.log"
grep -E "ERROR SUMMARY|== " "$OUT/$TOOL.log"
