O=gpurun_out/s14
mkdir -p $O
timeout 300 python scripts/one_cfg.py cfg4 1 > $O/plain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_level_range4 --launch-skip 97 --launch-count 1 -o $O/lv4096 python scripts/one_cfg.py cfg4 1 > $O/ncu1.log 2>&1
TG_LEVEL_GROUP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_level_range4 --launch-skip 97 --launch-count 1 -o $O/lv4096g python scripts/one_cfg.py cfg4 1 > $O/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_level_range4 --launch-skip 2 --launch-count 1 -o $O/lv128 python scripts/one_cfg.py cfg4 1 > $O/ncu3.log 2>&1
for g in 0 1; do TG_LEVEL_GROUP=$g timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_g$g.json 2>&1; done
for f in lv4096 lv4096g lv128; do python scripts/ncu_summary.py $O/$f.ncu-rep > $O/$f.txt 2>&1; done
rm -f $O/lv4096g.ncu-rep $O/lv128.ncu-rep
