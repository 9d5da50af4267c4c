# launch lists (ncu, one forward_backward per config) for the staged configs
O=gpurun_out/s2
mkdir -p $O
for c in cfg3 cfg4 cfg5; do
  timeout 300 python scripts/one_cfg.py $c 1 > $O/plain_$c.log 2>&1 && \
  TG_STAGED_VERBOSE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_$c.csv \
     python scripts/one_cfg.py $c 1 > $O/ncu_$c.log 2>&1
done
