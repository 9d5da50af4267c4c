O=gpurun_out/s5
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "gemm" > $O/pytest_gemm.log 2>&1; echo "exit $?" >> $O/pytest_gemm.log
for e in 0 3; do
  echo "== exp $e" >> $O/ablation.log
  TG_UMMA_EXP=$e GB_S=262144 GB_ENGINES=1,2 timeout 300 python scripts/gemm_bench.py 2>&1 | head -3 >> $O/ablation.log
done
