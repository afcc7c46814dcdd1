python -c "import __graft_entry__ as g; g.build()" > /dev/null
PROBE_SKEW=1 timeout 300 python tools/stage_probe.py -1 > gpurun_out/skew12.log 2>&1
timeout 600 python tools/flags_ab.py 0 32768 5 >> gpurun_out/skew12.log 2>&1
cat gpurun_out/skew12.log
