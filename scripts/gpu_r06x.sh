#!/bin/bash
O=gpurun_out/r06x; mkdir -p $O
for v in 132 260 516 1028; do TG_LO_ONLY=$v timeout 300 python scripts/gpt_diag2.py $O/g$v.npy > $O/d$v.log 2>&1; done
