#!/bin/bash
# r06m: event timeline of k_pair_ws k-tiles 100..163 (CTA 0 leader, CTA 1 peer), microseconds
# events: 0 TMA issue, 1 full seen by converter, 2 conv arrived, 3 relay saw local conv, 4 relay arrived remote,
#         5 MMA saw conv, 6 MMA issued+committed, 7 producer saw rempty (MMAs of that k-tile done)
O=gpurun_out/r06m; mkdir -p $O
TG_WS_TRACE=1 GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/trace.log 2>&1
TG_WS_TRACE=1 TG_WS_RELAX=1 GB_S=262144 GB_ENGINES=1 timeout 120 python scripts/gemm_bench.py > $O/trace_relax.log 2>&1
