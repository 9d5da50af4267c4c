#!/bin/bash
O=gpurun_out/r06n; mkdir -p $O
TG_WS_CONV=14 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_c14.log 2>&1
TG_WS_CONV=14 TG_WS_RELAX=1 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_c14_relax.log 2>&1
TG_WS_CONV=14 TG_WS_RELAX=1 TG_WS_TRACE=1 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/trace_c14_relax.log 2>&1
TG_UMMA_WS=0 GB_S=262144 GB_ENGINES=1 timeout 90 python scripts/gemm_bench.py > $O/gemm_old.log 2>&1
