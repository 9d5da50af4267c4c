#!/bin/bash
O=gpurun_out/r06s; mkdir -p $O
T="tests/test_gpu.py::test_reference_recorded_token_models_on_gpu"
for v in 0 1 2 4 7; do TG_LO_ONLY=$v timeout 300 python -m pytest $T -q > $O/t_$v.log 2>&1; done
