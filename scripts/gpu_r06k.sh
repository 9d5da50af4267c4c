#!/bin/bash
# r06k: ablations of k_pair_ws (raw mode, relaxed relay): 2 no conversion, 4 no drain loads, 8 one MMA per k-step
O=gpurun_out/r06k; mkdir -p $O
for m in 1 3 5 9 15; do
  TG_WS_RELAX=$m GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_m$m.log 2>&1
done
TG_UMMA_WS=0 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_old.log 2>&1
