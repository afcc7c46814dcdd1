python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "resident_b or ragged or config5" > gpurun_out/bres.log 2>&1; tail -2 gpurun_out/bres.log
PROBE_BRES=1 timeout 300 python tools/stage_probe.py -1 >> gpurun_out/bres.log 2>&1
timeout 600 python tools/flags_ab.py 0 33554432 5 >> gpurun_out/bres.log 2>&1
tail -7 gpurun_out/bres.log
