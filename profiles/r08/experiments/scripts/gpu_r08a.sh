#!/bin/bash
# r08a: state check after the container was re-created (tests, headline bench, GEMM engine bench)
O=gpurun_out/r08a; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
GB_S=262144 GB_ENGINES=1 timeout 300 python scripts/gemm_bench.py > $O/gemm.log 2>&1
