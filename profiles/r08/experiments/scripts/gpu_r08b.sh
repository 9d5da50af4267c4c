#!/bin/bash
# r08b: k_dx_skinny (K <= 16 input adjoints as an HBM stream)
O=gpurun_out/r08b; mkdir -p $O
GB_SET=shortk GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/gemm_shortk.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "gemm or skinny or bench_sizes or wide" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 300 python scripts/one_cfg.py cfg5 1 > $O/plain_cfg5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg5.csv python scripts/one_cfg.py cfg5 1 > $O/ncu_launches_cfg5.log 2>&1
