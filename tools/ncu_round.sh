# ncu evidence for the current build (one GPU): full-set capture of the config-5 interior
# batched-matvec GEMM stages + the launch list of one bench step + the W34 launch lists.
# usage: bash tools/ncu_round.sh TAG
TAG=${1:-r01}
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python tools/profile_core.py --reps 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma_gemm -s 6 -c 3 -o gpurun_out/prof_$TAG python tools/profile_core.py --reps 3 > gpurun_out/ncu_prof_$TAG.log 2>&1
tail -2 gpurun_out/ncu_prof_$TAG.log
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweeps > gpurun_out/bench_l.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweeps > gpurun_out/ncu_l.log 2>&1
tail -1 gpurun_out/ncu_l.log | cut -c1-200
for c in 3 4; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w34_c${c}_$TAG.csv python tools/next_rows_probe.py w34 $c > /dev/null 2>&1
done
ls gpurun_out
