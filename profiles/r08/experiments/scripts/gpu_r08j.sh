#!/bin/bash
# r08j: row-wise L2 prefetch windows ahead of the CTA-pair ring (TG_PAIR_PF = k-tiles per window)
O=gpurun_out/r08j; mkdir -p $O
for pf in 0 2 4 8; do
  TG_PAIR_PF=$pf timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg5_pf$pf.json 2> $O/bench_cfg5_pf$pf.err
done
TG_PAIR_PF=4 GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/gemm_pf4.log 2>&1
for pf in 4 8; do
TG_PAIR_PF=$pf timeout 300 python scripts/one_cfg.py cfg5 1 > $O/plain_cfg5.log 2>&1 && \
TG_PAIR_PF=$pf timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg5_pf$pf.csv python scripts/one_cfg.py cfg5 1 > $O/ncu_launches_cfg5.log 2>&1
done
TG_PAIR_PF=4 timeout 600 python -m pytest tests -m gpu -q -x -k "gemm or bench_sizes or wide or full_size" > $O/pytest_pf4.log 2>&1; echo "exit $?" >> $O/pytest_pf4.log
