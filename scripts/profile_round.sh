#!/bin/bash
# Round evidence: bench lines, reference arm, ncu launch lists + full captures of the step's kernels.
# Usage (on the GPU box): bash scripts/profile_round.sh r02
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O /tmp/tgsrc
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_cfg2_reference.json 2>&1
python bench.py --config cfg1 --no-cpu-baseline > $O/bench_cfg1.json 2>&1
python bench.py --config cfg3 --steps 20 --warmup 3 > $O/bench_cfg3.json 2>&1
python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2>&1
PYTHONPATH=. python scripts/e2e_probe.py > $O/e2e_probe.txt 2>&1
python scripts/link_bw.py > $O/link_bw.json 2>&1
# launch list of the bench command (ncu default: cold cache, serialised: shares, not absolutes)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
# same, warm caches (--cache-control none)
ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,smsp__inst_executed.sum --cache-control none \
    --clock-control none -c 400 --csv --log-file $O/launches_cfg2_warm.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_launches_warm.log 2>&1
# full captures of the step's two kernels (cfg2)
python scripts/one_cfg.py cfg2 3 > $O/plain1.log 2>&1 && \
TG_JIT_DUMP=/tmp/tgsrc ncu --set full --clock-control none --import-source on -k regex:tg_jit -s 2 -c 2 \
    -o $O/prof_cfg2 python scripts/one_cfg.py cfg2 3 > $O/ncu_full.log 2>&1
cp /tmp/tgsrc/*.cu $O/ 2>/dev/null
ls -la $O
