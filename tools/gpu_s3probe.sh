python -c "import __graft_entry__ as g; g.build()" > /dev/null
PROBE_QUICK=1 timeout 300 python tools/stage_probe.py 18 32 33 34 18 32 33 > gpurun_out/s3probe.log 2>&1
cat gpurun_out/s3probe.log | grep normal
