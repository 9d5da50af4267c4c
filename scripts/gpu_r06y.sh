#!/bin/bash
O=gpurun_out/r06y; mkdir -p $O
for v in 7 2055; do TG_LO_ONLY=$v timeout 300 python scripts/gpt_diag2.py $O/g$v.npy > $O/d$v.log 2>&1; done
for v in 7 2055 2048; do TG_LO_ONLY=$v GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_$v.log 2>&1; done
