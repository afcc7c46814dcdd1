python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k config5 2>&1 | tail -3
python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err
python tools/profile_core.py --reps 3 > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:dmma_gemm -s 6 -c 3 -o gpurun_out/prof_mv python tools/profile_core.py --reps 3 > gpurun_out/ncu_prof.log 2>&1; tail -3 gpurun_out/ncu_prof.log
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_l.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; tail -2 gpurun_out/ncu_l.log
