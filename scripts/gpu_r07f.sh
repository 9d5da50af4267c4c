#!/bin/bash
O=gpurun_out/r07f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "fused_embedding" > $O/pytest_fused.log 2>&1; echo "exit $?" >> $O/pytest_fused.log
timeout 600 python bench.py --config cfg3 --steps 20 --no-cpu-baseline --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 ncu --set full --import-source on --clock-control none -f -k regex:k_fused_mlp -c 1 -o /tmp/fm python scripts/one_cfg.py cfg3 1 > $O/ncu.log 2>&1
python scripts/ncu_summary.py /tmp/fm.ncu-rep > $O/fm_summary.txt 2>&1
ncu -i /tmp/fm.ncu-rep --page source --csv --print-source sass > $O/fm_source.csv 2>&1
