set -x
O=gpurun_out/s1
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 300 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python bench.py --config cfg1 --no-cpu-baseline > $O/bench_cfg1.json 2>&1
timeout 300 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2>&1
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2>&1
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2>&1
