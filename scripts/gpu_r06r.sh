#!/bin/bash
O=gpurun_out/r06r; mkdir -p $O
timeout 300 python scripts/gpt_diag.py $PWD $O/new.npy ref > $O/new.log 2>&1
timeout 300 python scripts/gpt_diag.py $PWD/build/old $O/old.npy > $O/old.log 2>&1
