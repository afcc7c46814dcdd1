python -c "import __graft_entry__ as g; g.build()" > /dev/null
(time timeout 1800 python -m pytest tests -m gpu -x -q) > gpurun_out/pytest_gpu_r01d.log 2>&1; tail -4 gpurun_out/pytest_gpu_r01d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01d.log 2>&1; echo smoke $?
timeout 900 python bench.py > gpurun_out/bench_r01d.json 2> gpurun_out/bench_r01d.err; tail -c 600 gpurun_out/bench_r01d.json
bash tools/ncu_round.sh r01d
