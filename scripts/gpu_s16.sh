#!/bin/bash
OUT=gpurun_out/s16; mkdir -p $OUT
for t in default gg_m2; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "grid or sort" -p no:cacheprovider > $OUT/pytest_$t.log 2>&1; echo "pytest_$t=$?" >> $OUT/rc.txt
done
for rep in 1 2; do
for t in default gg_m2 gg_off; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L timeout 300 python scripts/bench_grid.py --steps 1 | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/grid.jsonl 2>> $OUT/err.log
done; done
cat $OUT/rc.txt
