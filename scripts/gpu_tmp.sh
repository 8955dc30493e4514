#!/bin/bash
OUT=gpurun_out/s35; mkdir -p $OUT
LIBBORIS_PATH=paper_2104_04579_b200/tuning_libs/libboris_axf.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "grid or sort or deposit or pic" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
for rep in 1 2; do for t in default axf; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L timeout 300 python scripts/bench_grid.py | grep grid_push | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/grid.jsonl 2>> $OUT/err.log
  LIBBORIS_PATH=$L timeout 300 python scripts/pic_cycle.py --fused | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/pic.jsonl 2>> $OUT/err.log
done; done
cat $OUT/rc.txt
