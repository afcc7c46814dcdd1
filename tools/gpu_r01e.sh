python -c "import __graft_entry__ as g; g.build()" > /dev/null
(time timeout 1800 python -m pytest tests -m gpu -x -q) > gpurun_out/pytest_gpu_r01e.log 2>&1; tail -4 gpurun_out/pytest_gpu_r01e.log
timeout 900 python bench.py > gpurun_out/bench_r01e.json 2> gpurun_out/bench_r01e.err; tail -c 300 gpurun_out/bench_r01e.json
timeout 600 python tools/flags_ab.py 0 5242880 5 > gpurun_out/ab_r01e.log 2>&1; cat gpurun_out/ab_r01e.log
timeout 600 python tools/config5_certificate.py gpurun_out/cert_r01e.json > gpurun_out/cert_r01e.log 2>&1; tail -3 gpurun_out/cert_r01e.log
