O=gpurun_out/s17
mkdir -p $O
for e in 0 1 3 5; do
  echo "== exp $e" >> $O/abl.log
  TG_UMMA_EXP=$e GB_SET=cfg4 GB_S=524288 GB_ENGINES=2 timeout 300 python scripts/gemm_bench.py >> $O/abl.log 2>&1
done
