#!/bin/bash
# r08f: cfg1 timed as one graph launch of the K steps; ncu full captures of cfg5's weight-gradient and forward CTA-pair launches
O=gpurun_out/r08f; mkdir -p $O
timeout 600 python bench.py --config cfg1 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 600 python bench.py --config cfg1 --steps 100 --no-cpu-baseline --no-e2e > $O/bench_cfg1_k100.json 2> $O/bench_cfg1_k100.err
cap() {   # name config kernel-regex launch-skip
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$3 --launch-skip $4 --launch-count 1 \
      -o /tmp/$1 python scripts/one_cfg.py $2 1 > $O/ncu_full_$1.log 2>&1
  python scripts/ncu_summary.py /tmp/$1.ncu-rep > $O/ncu_full_$1.txt 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > $O/ncu_full_$1_raw.csv 2>/dev/null
}
cap cfg5_pair_dw2 cfg5 k_umma_pair 2
cap cfg5_pair_fwd2 cfg5 k_umma_pair 1
cap cfg5_dx_skinny cfg5 k_dx_skinny 0
