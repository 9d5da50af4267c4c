#!/bin/bash
O=gpurun_out/r06t; mkdir -p $O
TG_LO_ONLY=4 timeout 300 python scripts/gpt_diag2.py $O/g4.npy > $O/d4.log 2>&1
TG_LO_ONLY=0 timeout 300 python scripts/gpt_diag2.py $O/g0.npy > $O/d0.log 2>&1
