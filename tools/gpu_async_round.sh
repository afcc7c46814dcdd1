set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_row3.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "round or eigen or orthonormalise" > gpurun_out/async_test.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/async_test.log
timeout 300 python tools/round_time_probe.py > gpurun_out/round_time.log 2>&1; tail -20 gpurun_out/round_time.log
timeout 300 python tools/eigen_probe.py 64 128 256 512 1024 > gpurun_out/eigen_time.log 2>&1; cat gpurun_out/eigen_time.log
