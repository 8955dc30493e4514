#!/bin/bash
OUT=gpurun_out/s13; mkdir -p $OUT
for t in default pdm3; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  for rep in 1 2 3; do
    LIBBORIS_PATH=$L timeout 300 python scripts/pic_cycle.py --fused | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/pic.jsonl 2>> $OUT/err.log
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_push_deposit" -s 3 -c 1 \
  -o $OUT/pd -f python scripts/pic_cycle.py --fused --steps 5 > $OUT/ncu_pd.log 2>&1; echo "ncu=$?" >> $OUT/rc.txt
