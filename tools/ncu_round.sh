# ncu evidence for the current build (one GPU): full-set capture of the config-5 interior
# batched-matvec GEMM stages + the launch list of one bench step.
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python tools/profile_core.py --reps 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dmma_gemm -s 6 -c 3 -o gpurun_out/prof_r01 python tools/profile_core.py --reps 3 > gpurun_out/ncu_prof_r01.log 2>&1
tail -2 gpurun_out/ncu_prof_r01.log
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweeps > gpurun_out/bench_l.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweeps > gpurun_out/ncu_l.log 2>&1
tail -1 gpurun_out/ncu_l.log | cut -c1-200
