python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/dyn.log 2>&1; tail -2 gpurun_out/dyn.log
PROBE_QUICK=1 timeout 300 python tools/stage_probe.py -1 >> gpurun_out/dyn.log 2>&1
timeout 600 python tools/flags_ab.py 0 16777216 7 >> gpurun_out/dyn.log 2>&1
TT_FLAGS=0 timeout 300 python tools/w34_knobs.py >> gpurun_out/dyn.log 2>&1
TT_FLAGS=16777216 timeout 300 python tools/w34_knobs.py >> gpurun_out/dyn.log 2>&1
tail -8 gpurun_out/dyn.log
