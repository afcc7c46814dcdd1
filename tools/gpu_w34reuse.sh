python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "w34 or config3 or config4 or latency" > gpurun_out/w34reuse.log 2>&1; tail -2 gpurun_out/w34reuse.log
for rep in 1 2; do
TT_FLAGS=0 timeout 300 python tools/w34_knobs.py >> gpurun_out/w34reuse.log 2>&1
TT_FLAGS=8388608 timeout 300 python tools/w34_knobs.py >> gpurun_out/w34reuse.log 2>&1
done
tail -4 gpurun_out/w34reuse.log
