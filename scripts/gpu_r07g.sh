#!/bin/bash
# r07g: CTA-pair accumulator drained every 4 k-tiles (K = 128) instead of 2
O=gpurun_out/r07g; mkdir -p $O
GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/gemm.log 2>&1
timeout 300 python scripts/gemm_shapes_err.py > $O/shapes.log 2>&1
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python -m pytest tests -m gpu -q -x -k "wide or bench_sizes or gemm or char or gpt" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
