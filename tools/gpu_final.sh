python -c "import __graft_entry__ as g; g.build()" > /dev/null
(time timeout 1800 python -m pytest tests -m gpu -x -q) > gpurun_out/pytest_gpu_final.log 2>&1; tail -4 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke $?
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 200 gpurun_out/bench_final.json
bash tools/ncu_round.sh r01g
