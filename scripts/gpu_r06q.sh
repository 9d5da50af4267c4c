#!/bin/bash
O=gpurun_out/r06q; mkdir -p $O
timeout 300 python scripts/gemm_shapes_err.py > $O/shapes.log 2>&1
