O=gpurun_out/s3
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "gemm" > $O/pytest_gemm.log 2>&1; echo "exit $?" >> $O/pytest_gemm.log
GB_S=262144 GB_ENGINES=1,2 timeout 600 python scripts/gemm_bench.py > $O/gemm_bench.log 2>&1
