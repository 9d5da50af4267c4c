O=gpurun_out/s15
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for c in cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2>&1
done
timeout 300 python scripts/one_cfg.py cfg4 1 > $O/plain_cfg4.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_cfg4.csv \
     python scripts/one_cfg.py cfg4 1 > $O/ncu_cfg4.log 2>&1
