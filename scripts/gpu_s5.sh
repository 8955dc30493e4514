#!/bin/bash
# Session 5: grid-push state prefetch variants; lane-run deposition with register prefetch.
OUT=gpurun_out/s5; mkdir -p $OUT
for t in default gr_p1m2 gr_p1m3 dep_pf; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  for rep in 1 2; do
    LIBBORIS_PATH=$L timeout 300 python scripts/bench_grid.py --steps 1 | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/grid.jsonl 2>> $OUT/err.log
    LIBBORIS_PATH=$L timeout 300 python scripts/bench_deposit.py | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/dep.jsonl 2>> $OUT/err.log
  done
done
LIBBORIS_PATH=paper_2104_04579_b200/tuning_libs/libboris_gr_p1m2.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "grid or sort or deposit" -p no:cacheprovider > $OUT/pytest_p1m2.log 2>&1; echo "pytest_p1m2=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -1 $OUT/pytest_p1m2.log
