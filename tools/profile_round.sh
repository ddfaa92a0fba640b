#!/bin/bash
# Final-state evidence for a round in one gpurun call:  tools/profile_round.sh <tag>
#   GPU test suite + smoke, bench (plain), its ncu launch list, ncu --set full of the GEMM at
#   4096^3 and of the split pre-pass, LU factorisation time.  Everything lands in gpurun_out/.
TAG=${1:-r09}
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -2 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
tail -1 $OUT/bench_$TAG.json | cut -c1-300
timeout 300 python tools/lu_time.py 8192 3 4 > $OUT/lu_time_$TAG.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > $OUT/plain_bench_$TAG.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?"
timeout 300 python tools/gemm_once.py 4096 6 3 > $OUT/plain_once_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_split|split_" -s 2 -c 2 \
    -o $OUT/prof4096_$TAG python tools/gemm_once.py 4096 6 3 > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
timeout 300 python tools/gemm_once.py 16384 6 2 > $OUT/plain_16k_$TAG.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemm_split|split_" -s 2 -c 2 \
    -o $OUT/prof16k_$TAG python tools/gemm_once.py 16384 6 2 > $OUT/ncu_16k_$TAG.log 2>&1
echo "ncu 16k rc=$?"
