#!/bin/bash
# r06i: is the relay's cluster release the limiter? + where the MMA issuer waits (raw mode)
O=gpurun_out/r06i; mkdir -p $O
TG_WS_RELAX=1 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_relax.log 2>&1
GB_S=131072 GB_ENGINES=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_pair_ws \
   --launch-skip 9 --launch-count 1 -o /tmp/ws python scripts/gemm_bench.py > $O/ncu_ws.log 2>&1
ncu -i /tmp/ws.ncu-rep --page source --csv --print-source sass > $O/ws_source.csv 2>&1
ncu -i /tmp/ws.ncu-rep --page raw --csv > $O/ws_raw.csv 2>&1
