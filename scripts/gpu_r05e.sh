#!/bin/bash
O=gpurun_out/r05e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "simt or gemm or full_size or staged_fusions" > $O/pytest_sel.log 2>&1; echo "exit $?" >> $O/pytest_sel.log
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
TG_SKINNY=0 timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg5_noskinny.json 2> $O/bench_cfg5_noskinny.err
timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg5.csv python scripts/one_cfg.py cfg5 1 > /dev/null 2>&1
