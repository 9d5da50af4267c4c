#!/bin/bash
O=gpurun_out/r05b; mkdir -p $O
GB_SET=shortk GB_ENGINES=0,1,2 timeout 600 python scripts/gemm_bench.py > $O/gemm_shortk.log 2>&1
timeout 300 python bench.py --config cfg1 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
