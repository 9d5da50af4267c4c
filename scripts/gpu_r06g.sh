#!/bin/bash
# r06g: k_pair_ws, relaxed drain arrives; 6 vs 10 converter warps (gemm shapes only)
O=gpurun_out/r06g; mkdir -p $O
for nc in 6 10; do
  TG_WS_CONV=$nc GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_ws$nc.log 2>&1; echo "exit $?" >> $O/gemm_ws$nc.log
done
TG_UMMA_WS=0 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_old.log 2>&1
