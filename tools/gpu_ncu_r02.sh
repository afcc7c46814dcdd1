set -x
mkdir -p gpurun_out
bash tools/ncu_round.sh r02
python tools/profile_latency.py && timeout 300 ncu --set full --clock-control none --import-source on -k regex:"orth_cluster|small_chain" -c 4 -o gpurun_out/prof_lat_r02 python tools/profile_latency.py > gpurun_out/ncu_lat_r02.log 2>&1
tail -2 gpurun_out/ncu_lat_r02.log
ls -la gpurun_out
