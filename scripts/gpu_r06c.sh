#!/bin/bash
# r06c: pair GEMM diagnosis: throughput on cfg5 shapes + source-level ncu capture of fwd_l2
O=gpurun_out/r06c; mkdir -p $O
GB_S=262144 GB_ENGINES=1 timeout 600 python scripts/gemm_bench.py > $O/gemm_bench.log 2>&1
GB_S=131072 GB_ENGINES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_umma_pair \
   --launch-skip 4 --launch-count 1 -o /tmp/pair python scripts/gemm_bench.py > $O/ncu_pair.log 2>&1
ncu -i /tmp/pair.ncu-rep --page source --csv --print-source sass > $O/pair_source.csv 2>&1
ncu -i /tmp/pair.ncu-rep --page raw --csv > $O/pair_raw.csv 2>&1
python scripts/ncu_summary.py /tmp/pair.ncu-rep > $O/pair_summary.txt 2>&1
ls -la $O
