python -c "import __graft_entry__ as g; g.build()" > /dev/null
(time timeout 1800 python -m pytest tests -m gpu -x -q) > gpurun_out/pytest_gpu_r01h.log 2>&1; tail -4 gpurun_out/pytest_gpu_r01h.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01h.log 2>&1; echo smoke $?
timeout 900 python bench.py > gpurun_out/bench_r01h.json 2> gpurun_out/bench_r01h.err; tail -c 200 gpurun_out/bench_r01h.json
timeout 600 python tools/config5_certificate.py gpurun_out/cert_r01h.json > gpurun_out/cert_r01h.log 2>&1; tail -1 gpurun_out/cert_r01h.log
