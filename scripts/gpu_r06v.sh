#!/bin/bash
O=gpurun_out/r06v; mkdir -p $O
for v in 12 20 36 68; do TG_LO_ONLY=$v timeout 300 python scripts/gpt_diag2.py $O/g$v.npy > $O/d$v.log 2>&1; done
