O=gpurun_out/s16
mkdir -p $O
for k1 in 32 64 128; do
  echo "== K1 $k1" >> $O/k1.log
  TG_UMMA_K1=$k1 GB_SET=cfg4 GB_S=524288 GB_ENGINES=1,2 timeout 300 python scripts/gemm_bench.py >> $O/k1.log 2>&1
done
for k1 in 32 64; do TG_UMMA_K1=$k1 timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_k1_$k1.json 2>&1; done
