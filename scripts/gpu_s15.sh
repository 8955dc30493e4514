#!/bin/bash
OUT=gpurun_out/s15; mkdir -p $OUT
for t in default t32 default t32 default t32; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L timeout 300 python scripts/bench_launch.py | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/launch.jsonl 2>> $OUT/err.log
done
