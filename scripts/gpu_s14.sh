#!/bin/bash
OUT=gpurun_out/s14; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "type" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
for t in default t32 default t32; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L timeout 300 python scripts/bench_launch.py | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/launch.jsonl 2>> $OUT/err.log
done
cat $OUT/rc.txt; tail -2 $OUT/pytest.log; cat $OUT/launch.jsonl
