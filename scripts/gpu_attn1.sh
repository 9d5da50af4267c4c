O=gpurun_out/s8
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "gpt or workloads or larger or fusions or deterministic or shard or ragged" > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2>&1
