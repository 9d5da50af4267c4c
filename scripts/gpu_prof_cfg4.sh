O=gpurun_out/s10
mkdir -p $O
timeout 300 python scripts/one_cfg.py cfg4 1 > $O/plain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_level_range --launch-skip 97 --launch-count 1 -o $O/lv4096 python scripts/one_cfg.py cfg4 1 > $O/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_level_range --launch-skip 2 --launch-count 1 -o $O/lv128 python scripts/one_cfg.py cfg4 1 > $O/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attn --launch-count 2 -o $O/attn python scripts/one_cfg.py cfg4 1 > $O/ncu3.log 2>&1
