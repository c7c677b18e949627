#!/bin/bash
# Launch list + one `ncu --set full` capture of the fused step kernel.
# Usage (on the GPU box, via gpurun):  bash scripts/profile.sh <tag>
# Each ncu run is preceded by the identical plain run (must exit 0).
set -e
TAG=${1:-r01}
CMD="python bench.py --steps 6 --warmup 2 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 2 -c 1 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
# the per-pass trajectory kernel (the e2e path)
python scripts/traj_probe.py 4 > gpurun_out/plain_traj_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_traj_pass -s 1 -c 1 \
    -o gpurun_out/prof_traj_$TAG python scripts/traj_probe.py 4 > gpurun_out/ncu_traj_$TAG.log 2>&1
