#!/bin/bash
# r07c: skinny weight gradients on the FP32 pipe
O=gpurun_out/r07c; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x -k "wide or bench_sizes or gemm or skinny" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv \
   python scripts/one_cfg.py cfg5 1 > $O/ncu_launches.log 2>&1
