#!/bin/bash
# Round-2 profiles (on the GPU box via gpurun):  bash scripts/profile_r2.sh <tag>
#  1. launch list of the driver's bench command (per-kernel times)
#  2. ncu --set full of the fused step (bench kernel, 128 chains)
#  3. ncu --set full of the per-pass trajectory kernel at 16 chains on C4
#     (heavy-row CTAs staged through SMEM)
#  4. ncu --set full of one k_two_scan_multi sweep (BA(1e6) one_two_flip x 8)
#  5. sector metrics of K1 on C5 at 8 / 16 / 64 chains (DRAM access granularity)
# Every ncu run is preceded by the identical plain run, which must exit 0.
set -e
TAG=${1:-r16}
mkdir -p gpurun_out
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ttq --e2e-steps 1"
$BENCH > gpurun_out/plain_bench_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $BENCH > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 3 -c 1 \
    -o gpurun_out/prof_kpass_$TAG $BENCH > gpurun_out/ncu_kpass_$TAG.log 2>&1
SB="python scripts/smallb_probe.py --graph c4 --chains 16 --steps 4 --traj 6"
$SB > gpurun_out/plain_sb_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_traj_pass -s 2 -c 1 \
    -o gpurun_out/prof_trajb16_$TAG $SB > gpurun_out/ncu_trajb16_$TAG.log 2>&1
LS="python scripts/ls_bench.py"
$LS > gpurun_out/plain_ls_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_two_scan_multi -s 9 -c 1 \
    -o gpurun_out/prof_scan_$TAG $LS > gpurun_out/ncu_scan_$TAG.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,dram__sectors_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,gpu__time_duration.sum
for B in 8 16 64; do
  C5="python scripts/smallb_probe.py --graph c5 --chains $B --steps 3 --traj 0"
  $C5 > gpurun_out/plain_c5_${B}_$TAG.log 2>&1
  ncu --metrics $M --clock-control none --csv -k regex:k_pass -s 2 -c 1 \
      --log-file gpurun_out/c5_sectors_B${B}_$TAG.csv $C5 > gpurun_out/ncu_c5_${B}_$TAG.log 2>&1
done
for r in prof_kpass prof_trajb16 prof_scan; do
  ncu -i gpurun_out/${r}_$TAG.ncu-rep --page raw --csv > gpurun_out/${r}_${TAG}_raw.csv
done
echo done
