#!/bin/bash
O=gpurun_out/r06z; mkdir -p $O
NCCL_DEBUG=WARN timeout 600 python -m pytest tests/test_gpu_dp.py -q -x > $O/dp.log 2>&1; echo "exit $?" >> $O/dp.log
