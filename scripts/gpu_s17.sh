#!/bin/bash
OUT=gpurun_out/s17; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "deposit" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
for rep in 1 2; do
for t in default dh1m2 dh1m3 dh1m4; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L timeout 300 python scripts/bench_deposit.py | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/dep.jsonl 2>> $OUT/err.log
done; done
cat $OUT/rc.txt
