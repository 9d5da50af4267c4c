#!/bin/bash
# r08c: persistent CTA pairs over a split ring (k_umma_pair_p) vs k_umma_pair
O=gpurun_out/r08c; mkdir -p $O
GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/gemm_pp.log 2>&1; echo "exit $?" >> $O/gemm_pp.log
TG_PAIR_PERSIST=0 GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/gemm_old.log 2>&1
timeout 300 python scripts/gemm_shapes_err.py > $O/shapes.log 2>&1; echo "exit $?" >> $O/shapes.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
