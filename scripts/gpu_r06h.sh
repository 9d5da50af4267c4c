#!/bin/bash
# r06h: k_pair_ws raw-ring (hi = landed fp32) vs in-place, 6 / 10 converter warps
O=gpurun_out/r06h; mkdir -p $O
for cfg in "10 1" "6 1" "10 0"; do
  set -- $cfg
  TG_WS_CONV=$1 TG_WS_RAW=$2 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_ws$1_raw$2.log 2>&1; echo "exit $?" >> $O/gemm_ws$1_raw$2.log
done
