#!/bin/bash
O=gpurun_out/r05d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "gemm or staged or full_size or gpt or sequential or larger" > $O/pytest_sel.log 2>&1; echo "exit $?" >> $O/pytest_sel.log
for c in cfg3 cfg4 cfg5; do
  st=5; [ $c = cfg3 ] && st=20; [ $c = cfg5 ] && st=3
  timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
TG_SHORTK=0 timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg3_noshortk.json 2>&1
timeout 300 python scripts/one_cfg.py cfg3 1 > $O/plain_cfg3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg3.csv python scripts/one_cfg.py cfg3 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg4.csv python scripts/one_cfg.py cfg4 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg5.csv python scripts/one_cfg.py cfg5 1 > /dev/null 2>&1
