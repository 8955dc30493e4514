#!/bin/bash
# Session 2: full GPU suite, grid/sort/deposit benches, ncu DRAM bytes of the sort kernels.
OUT=gpurun_out/s2; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $OUT/rc.txt
timeout 600 python scripts/bench_grid.py > $OUT/grid.jsonl 2> $OUT/grid.err; echo "grid_rc=$?" >> $OUT/rc.txt
timeout 600 python scripts/bench_deposit.py > $OUT/dep.jsonl 2> $OUT/dep.err; echo "dep_rc=$?" >> $OUT/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_pack|k_unpack|k_rs|k_gather" --csv --log-file $OUT/sort_ncu.csv \
  python scripts/bench_grid.py --n 10000000 --steps 2 > $OUT/sort_ncu.log 2>&1; echo "ncu_rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -3 $OUT/pytest_gpu.log; cat $OUT/grid.jsonl $OUT/dep.jsonl
