#!/bin/bash
# r08d: persistent CTA pairs (old ring, 4-pass staged epilogue) vs k_umma_pair
O=gpurun_out/r08d; mkdir -p $O
GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/gemm_pp.log 2>&1; echo "exit $?" >> $O/gemm_pp.log
timeout 300 python scripts/gemm_shapes_err.py > $O/shapes.log 2>&1; echo "exit $?" >> $O/shapes.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
TG_PAIR_PERSIST=0 timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5_old.json 2> $O/bench_cfg5_old.err
timeout 600 python bench.py --config cfg4 --steps 5 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
TG_PAIR_PERSIST=0 timeout 600 python bench.py --config cfg4 --steps 5 --no-cpu-baseline --no-e2e > $O/bench_cfg4_old.json 2> $O/bench_cfg4_old.err
timeout 600 python bench.py --config cfg3 --steps 20 --no-cpu-baseline --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TG_PAIR_PERSIST=0 timeout 600 python bench.py --config cfg3 --steps 20 --no-cpu-baseline --no-e2e > $O/bench_cfg3_old.json 2> $O/bench_cfg3_old.err
