#!/bin/bash
# r06b: full GPU suite, tcgen05 / FMA peaks, per-config DRAM traffic, compute-sanitizer.
O=gpurun_out/r06b; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
./build/mma_peak $O/mma_peaks.json > $O/mma_peak.log 2>&1; echo "exit $?" >> $O/mma_peak.log
./build/fp_peak > $O/fp_peak.log 2>&1
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --print-units base \
     --clock-control none -c 5000 --csv --log-file $O/traffic_$c.csv python scripts/one_cfg.py $c 1 > $O/traffic_$c.log 2>&1
done
for t in memcheck racecheck synccheck; do
  for c in "cfg2 1024" "cfg3 512" "cfg5 256" "cfg4 8"; do
    set -- $c
    timeout 900 compute-sanitizer --tool $t --print-limit 50 python scripts/sanitize_run.py $1 $2 > $O/sanitizer_${t}_$1.log 2>&1
    echo "exit $?" >> $O/sanitizer_${t}_$1.log
  done
done
