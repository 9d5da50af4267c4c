#!/bin/bash
O=gpurun_out/r06p; mkdir -p $O
T="tests/test_gpu.py::test_reference_recorded_token_models_on_gpu"
timeout 300 python -m pytest $T -q > $O/t_default.log 2>&1
TG_UMMA_PAIR=0 timeout 300 python -m pytest $T -q > $O/t_nopair.log 2>&1
TG_UMMA_PERSIST=0 timeout 300 python -m pytest $T -q > $O/t_nopersist.log 2>&1
TG_UMMA_PAIR=0 TG_UMMA_PERSIST=0 timeout 300 python -m pytest $T -q > $O/t_neither.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "exit $?" >> $O/pytest_all.log
