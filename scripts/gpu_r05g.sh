#!/bin/bash
O=gpurun_out/r05g; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
for c in cfg3 cfg4 cfg5; do
  st=5; [ $c = cfg3 ] && st=20; [ $c = cfg5 ] && st=3
  timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
for c in cfg3 cfg4 cfg5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_$c.csv python scripts/one_cfg.py $c 1 > /dev/null 2>&1
done
