#!/bin/bash
O=gpurun_out/r05c; mkdir -p $O
timeout 300 python bench.py --config cfg1 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python scripts/one_cfg.py cfg4 1 > $O/plain_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_tma_p --launch-skip 4 --launch-count 1 \
    -o /tmp/persist python scripts/one_cfg.py cfg4 1 > $O/ncu_persist.log 2>&1
ncu -i /tmp/persist.ncu-rep --page source --csv --print-source sass > $O/persist_source.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_level_range4 --launch-skip 24 --launch-count 1 \
    -o /tmp/level python scripts/one_cfg.py cfg4 1 > $O/ncu_level.log 2>&1
ncu -i /tmp/level.ncu-rep --page source --csv --print-source sass > $O/level_source.csv 2>&1
python scripts/ncu_summary.py /tmp/level.ncu-rep > $O/level.txt 2>&1
ls -la $O
