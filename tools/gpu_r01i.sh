python -c "import __graft_entry__ as g; g.build()" > /dev/null
(time timeout 1800 python -m pytest tests -m gpu -x -q) > gpurun_out/pytest_gpu_r01i.log 2>&1; tail -4 gpurun_out/pytest_gpu_r01i.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01i.log 2>&1; echo smoke $?
timeout 900 python bench.py > gpurun_out/bench_r01i.json 2> gpurun_out/bench_r01i.err; tail -c 200 gpurun_out/bench_r01i.json
timeout 600 python tools/config5_certificate.py gpurun_out/cert_r01i.json > gpurun_out/cert_r01i.log 2>&1; tail -1 gpurun_out/cert_r01i.log
bash tools/ncu_round.sh r01i
