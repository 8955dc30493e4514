#!/bin/bash
OUT=gpurun_out/s19; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "sort or grid or deposit" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_rs|k_scan|k_pack|k_unpack" --csv --log-file $OUT/sort.csv python scripts/prof_sort.py > $OUT/ncu.log 2>&1; echo "ncu=$?" >> $OUT/rc.txt
for rep in 1 2; do
  timeout 300 python scripts/pic_cycle.py --fused >> $OUT/pic.jsonl 2>> $OUT/err.log
  timeout 300 python scripts/bench_grid.py --steps 1 | grep sort >> $OUT/sort.jsonl 2>> $OUT/err.log
done
cat $OUT/rc.txt; tail -1 $OUT/pytest.log
