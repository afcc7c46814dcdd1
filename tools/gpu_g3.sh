python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "forced or ragged or config5 or resident or w34" > gpurun_out/g3.log 2>&1; tail -2 gpurun_out/g3.log
PROBE_G3=1 timeout 300 python tools/stage_probe.py -1 >> gpurun_out/g3.log 2>&1
timeout 600 python tools/flags_ab.py 0 67108864 7 >> gpurun_out/g3.log 2>&1
tail -6 gpurun_out/g3.log
