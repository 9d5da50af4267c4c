#!/bin/bash
# r07e: fused embedding-MLP / CE kernel (cfg3) + L2 prefetch in the CTA-pair producer
O=gpurun_out/r07e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "fused_embedding or char_mlp" > $O/pytest_fused.log 2>&1; echo "exit $?" >> $O/pytest_fused.log
timeout 600 python bench.py --config cfg3 --steps 20 --no-cpu-baseline --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
TG_FUSED_MLP=0 timeout 600 python bench.py --config cfg3 --steps 20 --no-cpu-baseline --no-e2e > $O/bench_cfg3_chain.json 2> $O/bench_cfg3_chain.err
GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/gemm.log 2>&1
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
