# one gpurun call: the closing evidence of the round (latest build)
# (GPU suite, smoke, bench line, then the ncu launch list of the same bench command)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_h.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest_h.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_h.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_h.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/launches_step_h.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-sweeps --no-cpu-baseline > gpurun_out/ncu_launches_h.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_launches_h.log
