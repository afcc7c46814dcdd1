python -c "import __graft_entry__ as g; g.build()" > /dev/null
for u in 3 1.5 6 3 1.5 6; do
  echo "TT_LAT_UNIT_US=$u $(TT_LAT_UNIT_US=$u timeout 300 python tools/flags_ab.py 0 0 3 2>&1 | head -1 | cut -c1-40) $(TT_LAT_UNIT_US=$u timeout 300 python tools/w34_knobs.py 2>&1 | tail -1)" >> gpurun_out/unitus.log
done
cat gpurun_out/unitus.log
