#!/bin/bash
# r06e: where k_pair_ws waits (source-level), and the cfg5 launch list with it
O=gpurun_out/r06e; mkdir -p $O
GB_S=131072 GB_ENGINES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair_ws \
   --launch-skip 9 --launch-count 1 -o /tmp/ws python scripts/gemm_bench.py > $O/ncu_ws.log 2>&1
ncu -i /tmp/ws.ncu-rep --page source --csv --print-source sass > $O/ws_source.csv 2>&1
ncu -i /tmp/ws.ncu-rep --page raw --csv > $O/ws_raw.csv 2>&1
python scripts/ncu_summary.py /tmp/ws.ncu-rep > $O/ws_summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv \
   python scripts/one_cfg.py cfg5 1 > $O/ncu_launches.log 2>&1
TG_UMMA_WS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5_old.csv \
   python scripts/one_cfg.py cfg5 1 > $O/ncu_launches_old.log 2>&1
