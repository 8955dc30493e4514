#!/bin/bash
OUT=gpurun_out/s18; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "mdipole or field_evaluate" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
LIBBORIS_PATH=paper_2104_04579_b200/tuning_libs/libboris_mdu2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "mdipole or grid" -p no:cacheprovider > $OUT/pytest_u2.log 2>&1; echo "pytest_u2=$?" >> $OUT/rc.txt
for rep in 1 2; do for t in default mdu2; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L timeout 600 python scripts/paper_table2.py --only analytic --iters 5 2>>$OUT/err.log | grep '^{' | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/t2.jsonl
  LIBBORIS_PATH=$L timeout 300 python scripts/bench_grid.py | grep '"steps": 100' | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/grid.jsonl 2>> $OUT/err.log
done; done
cat $OUT/rc.txt
