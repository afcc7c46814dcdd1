set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest.log
timeout 300 python tools/w34_dag_probe.py > gpurun_out/dag_probe3.log 2>&1; echo "probe rc=$?"
cat gpurun_out/dag_probe3.log
