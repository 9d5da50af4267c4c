#!/bin/bash
# r06d: k_pair_ws (persistent warp-specialised CTA pairs) vs k_umma_pair
O=gpurun_out/r06d; mkdir -p $O
GB_S=262144 GB_ENGINES=1 TG_UMMA_WS=0 timeout 300 python scripts/gemm_bench.py > $O/gemm_old.log 2>&1
GB_S=262144 GB_ENGINES=1 timeout 300 python scripts/gemm_bench.py > $O/gemm_ws.log 2>&1; echo "exit $?" >> $O/gemm_ws.log
timeout 900 python -m pytest tests -m gpu -q -x -k "gemm or umma or wide or char or gpt or bench_sizes" > $O/pytest_sel.log 2>&1; echo "exit $?" >> $O/pytest_sel.log
timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
TG_UMMA_WS=0 timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $O/bench_cfg5_old.json 2> $O/bench_cfg5_old.err
