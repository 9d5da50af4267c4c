O=gpurun_out/s9
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "gpt or workloads or larger or deterministic or shard or ragged" > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2>&1
timeout 300 python scripts/one_cfg.py cfg4 1 > $O/plain_cfg4.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_cfg4.csv \
     python scripts/one_cfg.py cfg4 1 > $O/ncu_cfg4.log 2>&1
