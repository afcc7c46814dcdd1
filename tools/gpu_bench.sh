set -x
free -g | head -2
nproc
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
echo rc=$?
tail -3 gpurun_out/bench_r02a.err
