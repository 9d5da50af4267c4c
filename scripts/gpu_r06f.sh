#!/bin/bash
# r06f: k_pair_ws with the peer relay; 6 vs 10 converter warps
O=gpurun_out/r06f; mkdir -p $O
for nc in 6 10; do
  TG_WS_CONV=$nc GB_S=262144 GB_ENGINES=1 timeout 300 python scripts/gemm_bench.py > $O/gemm_ws$nc.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x -k "gemm or umma or wide or char or gpt or bench_sizes" > $O/pytest_sel.log 2>&1; echo "exit $?" >> $O/pytest_sel.log
for nc in 6 10; do
  TG_WS_CONV=$nc timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $O/bench_cfg5_ws$nc.json 2> $O/bench_cfg5_ws$nc.err
done
TG_WS_CONV=10 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv \
   python scripts/one_cfg.py cfg5 1 > $O/ncu_launches.log 2>&1
