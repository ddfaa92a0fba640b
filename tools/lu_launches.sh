#!/bin/bash
# launch list of one n=8192 solve (config 5): where the factorisation / refinement time goes
#   tools/lu_launches.sh [variant] [kappa] [solvers]
V=${1:-3}; K=${2:-1e1}; S=${3:-ir}
export CONFIG5_NO_SVD=1
timeout 300 python tools/config5.py 8192 $V $K $S > gpurun_out/c5_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"panel|laswp|trsm|trsv|residual|gemm_split|split_|build|gather|absmax|axpy|copy_matrix|arnoldi|krylov|diag_inverse" -c 20000 --csv \
  --log-file gpurun_out/c5_launches_${S}.csv python tools/config5.py 8192 $V $K $S > gpurun_out/c5_ncu.log 2>&1
echo rc=$?
