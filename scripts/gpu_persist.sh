O=gpurun_out/s18
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "gemm or gpt or full_size or fusions or workloads" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for p in 1 0; do
  echo "== persist $p" >> $O/gb.log
  TG_UMMA_PERSIST=$p GB_SET=cfg4 GB_S=524288 GB_ENGINES=1,2 timeout 300 python scripts/gemm_bench.py >> $O/gb.log 2>&1
done
for c in cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2>&1
done
