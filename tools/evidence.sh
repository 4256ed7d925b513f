# Round evidence on a GPU box (gpurun): traffic stamps, the bench line, the C5 launch list and full capture.
# Afterwards here: cp gpurun_out/ncu_traffic.json profiles/; tools/make_profiles.py --round N --config c5 ...
set -x
python tools/capture_traffic.py run > gpurun_out/capture_traffic.log 2>&1
cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu --no-e2e > gpurun_out/c5_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:walk_kernel -c 1 -o gpurun_out/c5_walk_kernel python tools/profile_walk.py --config c5 --tune --launches 1 > gpurun_out/c5_full.log 2>&1
