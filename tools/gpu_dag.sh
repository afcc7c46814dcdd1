set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "w34" > gpurun_out/dag_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/dag_tests.log
timeout 300 python tools/w34_dag_probe.py > gpurun_out/dag_probe.log 2>&1; echo "probe rc=$?"
cat gpurun_out/dag_probe.log
