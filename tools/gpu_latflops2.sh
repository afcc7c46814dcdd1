python -c "import __graft_entry__ as g; g.build()" > /dev/null
for f in 5e9 1e10 2.5e10 5e9 1e10 2.5e10; do
  echo "TT_LAT_FLOPS=$f $(TT_LAT_FLOPS=$f timeout 300 python tools/flags_ab.py 0 0 3 2>&1 | head -1)" >> gpurun_out/latflops2.log
done
cat gpurun_out/latflops2.log
