#!/bin/bash
# Round evidence: GPU tests, smoke, bench lines of every config (device value,
# e2e, roofline, cpu_baseline), the reference arm, ncu launch lists and full
# captures of the dominant kernels (summaries + raw pages as text).
# Usage (on the GPU box): bash scripts/profile_round.sh r09
R=${1:-r09}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_cfg5_reference.json 2>&1
timeout 600 python bench.py --config cfg1 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 600 python bench.py --config cfg2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --config cfg3 --steps 20 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 python bench.py --config cfg4 --steps 5 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 300 python scripts/one_cfg.py $c 1 > $O/plain_$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_$c.csv \
      python scripts/one_cfg.py $c 1 > $O/ncu_launches_$c.log 2>&1
done
cap() {   # name config kernel-regex launch-skip
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$3 --launch-skip $4 --launch-count 1 \
      -o /tmp/$1 python scripts/one_cfg.py $2 2 > $O/ncu_full_$1.log 2>&1
  python scripts/ncu_summary.py /tmp/$1.ncu-rep > $O/ncu_full_$1.txt 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > $O/ncu_full_$1_raw.csv 2>/dev/null
}
cap cfg5_pair cfg5 k_umma_pair 1
cap cfg5_pair_dx2 cfg5 k_umma_pair 2
cap cfg5_dw_skinny cfg5 k_dw_skinny 0
cap cfg5_dx_skinny cfg5 k_dx_skinny 0
cap cfg2_tape cfg2 tg_jit_tape 1
cap cfg1_tape cfg1 tg_jit_tape 1
cap cfg3_pair cfg3 k_umma_pair 0
cap cfg4_attn_bwd cfg4 k_attn_bwd 0
# DRAM traffic of one step (cold caches) for the staged configs whose kernels changed this round
for c in cfg3 cfg5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
      --print-units base --log-file $O/traffic_$c.csv python scripts/one_cfg.py $c 1 > $O/ncu_traffic_$c.log 2>&1
done
ls -la $O
