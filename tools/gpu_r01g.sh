python -c "import __graft_entry__ as g; g.build()" > /dev/null
(time timeout 1800 python -m pytest tests -m gpu -x -q) > gpurun_out/pytest_gpu_r01g.log 2>&1; tail -4 gpurun_out/pytest_gpu_r01g.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01g.log 2>&1; echo smoke $?
timeout 900 python bench.py > gpurun_out/bench_r01g.json 2> gpurun_out/bench_r01g.err; tail -c 300 gpurun_out/bench_r01g.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r01g.json 2>&1; tail -c 300 gpurun_out/bench_ref_r01g.json
