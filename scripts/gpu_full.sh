#!/bin/bash
# Full check: smoke, GPU suite, default bench line, grid/sort/deposit/PIC benches.
# Usage: bash scripts/gpu_full.sh <outdir>
OUT=${1:-gpurun_out/full}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke=$?" >> $OUT/rc.txt
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench=$?" >> $OUT/rc.txt
timeout 600 python scripts/bench_grid.py > $OUT/grid.jsonl 2> $OUT/grid.err; echo "grid=$?" >> $OUT/rc.txt
timeout 600 python scripts/bench_deposit.py > $OUT/dep.jsonl 2> $OUT/dep.err; echo "dep=$?" >> $OUT/rc.txt
timeout 600 python scripts/pic_cycle.py > $OUT/pic.jsonl 2> $OUT/pic.err; echo "pic=$?" >> $OUT/rc.txt
timeout 600 python scripts/pic_cycle.py --fused >> $OUT/pic.jsonl 2>> $OUT/pic.err
timeout 300 python scripts/bench_launch.py > $OUT/launch.jsonl 2>> $OUT/err.log
cat $OUT/rc.txt; tail -2 $OUT/pytest_gpu.log; grep -E "^FAILED" $OUT/pytest_gpu.log | head
