python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "apply" > gpurun_out/apply4.log 2>&1; tail -2 gpurun_out/apply4.log
for f in 0 134217728 0 134217728; do TT_FLAGS=$f timeout 120 python tools/apply_probe.py 2>&1 | head -1 >> gpurun_out/apply4.log; done
tail -5 gpurun_out/apply4.log
