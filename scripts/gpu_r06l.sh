#!/bin/bash
# r06l: one 3D TMA load per MN-major k-tile instead of four
O=gpurun_out/r06l; mkdir -p $O
GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_mn3.log 2>&1
TG_WS_RELAX=1 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_mn3_relax.log 2>&1
TG_WS_MN3=0 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_mn2.log 2>&1
