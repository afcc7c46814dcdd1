python -c "import __graft_entry__ as g; g.build()" > /dev/null
for f in 1.5e9 3e9 5e9 1.5e9 3e9 5e9; do
  echo "TT_LAT_FLOPS=$f" >> gpurun_out/latflops.log
  TT_LAT_FLOPS=$f timeout 120 python tools/iface_probe.py 2>&1 | cut -c1-40 >> gpurun_out/latflops.log
  TT_LAT_FLOPS=$f timeout 300 python tools/flags_ab.py 0 0 3 2>&1 | head -1 >> gpurun_out/latflops.log
done
cat gpurun_out/latflops.log
