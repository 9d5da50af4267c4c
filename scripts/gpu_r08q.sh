#!/bin/bash
# r08q: rolled store-only epilogue with hoisted addressing in k_umma_pair
O=gpurun_out/r08q; mkdir -p $O

GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/gemm.log 2>&1; echo "exit $?" >> $O/gemm.log
timeout 300 python scripts/gemm_shapes_err.py > $O/shapes.log 2>&1; echo "exit $?" >> $O/shapes.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --config cfg3 --steps 20 --no-cpu-baseline --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config cfg4 --steps 5 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 300 python scripts/one_cfg.py cfg5 1 > $O/plain_cfg5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg5.csv python scripts/one_cfg.py cfg5 1 > $O/ncu_launches_cfg5.log 2>&1
