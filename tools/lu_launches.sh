#!/bin/bash
# launch list of one n=8192 bf16x3 gesv_ir (config 5, kappa 10): where the factorisation time goes
export CONFIG5_NO_SVD=1
timeout 300 python tools/config5.py 8192 3 1e1 > gpurun_out/c5_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"panel|laswp|trsm|trsv|residual|gemm_split|split_|build|gather|absmax|axpy|copy_matrix" -c 5000 --csv \
  --log-file gpurun_out/c5_launches.csv python tools/config5.py 8192 3 1e1 > gpurun_out/c5_ncu.log 2>&1
echo rc=$?
