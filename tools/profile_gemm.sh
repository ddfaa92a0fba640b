#!/bin/bash
# ncu --set full of the GEMM kernel at the bench size (via bench.py) and at 16384^3.
TAG=${1:-r03}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/plain_short_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_split|split_" -s 6 -c 3 \
    -o $OUT/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu 4096 rc=$?"
timeout 300 python tools/gemm_once.py 16384 6 2 > $OUT/plain_16k_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_split" -s 1 -c 1 \
    -o $OUT/prof16k_$TAG python tools/gemm_once.py 16384 6 2 > $OUT/ncu_16k_$TAG.log 2>&1
echo "ncu 16k rc=$?"
