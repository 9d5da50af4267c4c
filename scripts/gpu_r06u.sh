#!/bin/bash
O=gpurun_out/r06u; mkdir -p $O
TG_GEMM_LOG=1 TG_LO_ONLY=4 timeout 300 python scripts/gpt_diag2.py $O/g4.npy > $O/d4.log 2>&1
TG_LO_ONLY=4 timeout 300 python scripts/gpt_diag2.py $O/g4b.npy 256 > $O/d4b.log 2>&1
