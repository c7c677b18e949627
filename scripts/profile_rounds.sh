#!/bin/bash
# Per-kernel DRAM traffic and duration of every launch of the per-round
# stages (scripts/round_probe.py), one lightweight ncu metric pass each.
# Usage (GPU box, via gpurun):  bash scripts/profile_rounds.sh <tag>
set -e
TAG=${1:-r08}
mkdir -p gpurun_out
for C in c4 c3; do
  python scripts/round_probe.py $C 3 > gpurun_out/round_${C}_$TAG.jsonl 2> gpurun_out/round_${C}_$TAG.err
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/round_launches_${C}_$TAG.csv \
      python scripts/round_probe.py $C 1 > gpurun_out/ncu_round_${C}_$TAG.log 2>&1
done
