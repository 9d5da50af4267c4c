#!/bin/bash
# r08h: dact epilogue with all h segments in flight
O=gpurun_out/r08h; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "gemm or skinny or bench_sizes or wide or full_size or staged or fusions or gpt" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 python bench.py --config cfg3 --steps 20 --no-cpu-baseline --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config cfg4 --steps 5 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
