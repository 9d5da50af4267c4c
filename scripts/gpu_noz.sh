O=gpurun_out/s23
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "gpt or full_size or fusions or workloads or larger or gemm" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for c in cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2>&1
done
timeout 300 python scripts/one_cfg.py cfg4 1 > $O/plain4.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_cfg4.csv python scripts/one_cfg.py cfg4 1 > $O/ncu3.log 2>&1
