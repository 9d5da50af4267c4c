#!/bin/bash
O=gpurun_out/r06j; mkdir -p $O
TG_WS_FULLGRID=1 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_fullgrid.log 2>&1
TG_WS_FULLGRID=1 TG_WS_RELAX=1 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_fullgrid_relax.log 2>&1
TG_WS_RELAX=1 GB_S=131072 GB_ENGINES=1 timeout 300 ncu -f --set full --import-source on --clock-control none -k regex:k_pair_ws \
   --launch-skip 9 --launch-count 1 -o /tmp/ws2 python scripts/gemm_bench.py > $O/ncu_ws.log 2>&1
ncu -i /tmp/ws2.ncu-rep --page source --csv --print-source sass > $O/ws_source.csv 2>&1
ncu -i /tmp/ws2.ncu-rep --page raw --csv > $O/ws_raw.csv 2>&1
