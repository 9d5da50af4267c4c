O=gpurun_out/s4
mkdir -p $O
for e in 0 1 2 3; do
  echo "== exp $e" >> $O/ablation.log
  TG_UMMA_EXP=$e GB_S=262144 GB_ENGINES=1,2 timeout 300 python scripts/gemm_bench.py 2>&1 | head -3 >> $O/ablation.log
done
timeout 300 python scripts/gemm_one.py 1024 262144 1024 1 1 1 > $O/one.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma_pair -s 1 -c 1 -o $O/pair_fwd python scripts/gemm_one.py 1024 262144 1024 1 1 1 > $O/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma_tma -s 1 -c 1 -o $O/single_fwd python scripts/gemm_one.py 1024 262144 1024 1 1 2 >> $O/ncu.log 2>&1
