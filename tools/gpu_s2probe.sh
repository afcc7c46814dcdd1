python -c "import __graft_entry__ as g; g.build()" > /dev/null
PROBE_QUICK=1 timeout 300 python tools/stage_probe.py 1 26 27 1 26 27 > gpurun_out/s2probe.log 2>&1
timeout 600 python tools/flags_ab.py 0 1048576 7 >> gpurun_out/s2probe.log 2>&1
timeout 600 python tools/flags_ab.py 0 2097152 7 >> gpurun_out/s2probe.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "forced or config5" >> gpurun_out/s2probe.log 2>&1
cat gpurun_out/s2probe.log | tail -30
