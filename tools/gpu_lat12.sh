python -c "import __graft_entry__ as g; g.build()" > /dev/null
PROBE_QUICK=1 timeout 300 python tools/stage_probe.py 35 36 > gpurun_out/lat12.log 2>&1
for rep in 1 2; do
for m in 7680 0 6144 1536; do TT_LAT_MASK=$m timeout 300 python tools/w34_knobs.py >> gpurun_out/lat12.log 2>&1; done
done
timeout 600 python -m pytest tests -m gpu -x -q -k "forced or latency or w34 or config3 or config4" >> gpurun_out/lat12.log 2>&1
cat gpurun_out/lat12.log | grep -v "^$" | tail -20
