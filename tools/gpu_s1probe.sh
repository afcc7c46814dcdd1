python -c "import __graft_entry__ as g; g.build()" > /dev/null
PROBE_QUICK=1 timeout 300 python tools/stage_probe.py 26 28 29 30 31 > gpurun_out/s1probe.log 2>&1
timeout 600 python tools/flags_ab.py 1048576 5242880 7 >> gpurun_out/s1probe.log 2>&1
timeout 600 python tools/flags_ab.py 0 5242880 7 >> gpurun_out/s1probe.log 2>&1
cat gpurun_out/s1probe.log | tail -30
