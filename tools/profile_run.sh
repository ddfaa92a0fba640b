#!/bin/bash
# Bench + ncu evidence in one gpurun call.  Usage: tools/profile_run.sh <tag>
set -x
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu_$TAG.txt
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
cat $OUT/bench_$TAG.json
# launch list of the same command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
# one --set full capture of the top kernel and of the two split kernels (short command, exited 0 plain first)
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/plain_short_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_split|split_" -s 2 -c 2 \
    -o $OUT/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
