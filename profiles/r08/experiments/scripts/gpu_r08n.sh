#!/bin/bash
# r08n: non-persistent CTA pairs over the ring split by lifetime (4 raw/hi stages + 3 lo stages of 32 KB)
O=gpurun_out/r08n; mkdir -p $O
GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/gemm.log 2>&1; echo "exit $?" >> $O/gemm.log
timeout 200 python scripts/pair_trace.py fwd > $O/trace_fwd.log 2>&1
timeout 300 python scripts/gemm_shapes_err.py > $O/shapes.log 2>&1; echo "exit $?" >> $O/shapes.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --config cfg3 --steps 20 --no-cpu-baseline --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config cfg4 --steps 5 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
