python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python tools/stage_probe.py 2>&1 | tail -12
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 2; do python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --variant $v > gpurun_out/bench_v$v.json 2> gpurun_out/bench_v$v.err; tail -2 gpurun_out/bench_v$v.err; done
