#!/bin/bash
# New-row checks: chunked staged runs, device synth bit-exactness, bench keys.
O=gpurun_out/r05a; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "sequential or synth or device_generated" > $O/pytest_new.log 2>&1; echo "exit $?" >> $O/pytest_new.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
