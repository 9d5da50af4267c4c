#!/bin/bash
O=gpurun_out/r06w; mkdir -p $O
TG_LO_ONLY=7 timeout 200 python scripts/gemm_n16.py > $O/n16_lo.log 2>&1
TG_LO_ONLY=0 timeout 200 python scripts/gemm_n16.py > $O/n16_rna.log 2>&1
