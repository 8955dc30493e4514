#!/bin/bash
# Session 4: ncu (full, source) of the sorted deposition: warp-run vs lane-run kernels.
OUT=gpurun_out/s4; mkdir -p $OUT
for t in default lane_runs; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_deposit" -s 1 -c 1 \
    -o $OUT/dep_$t -f python scripts/prof_deposit.py > $OUT/ncu_$t.log 2>&1; echo "ncu_$t=$?" >> $OUT/rc.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "mdipole or field_evaluate" -p no:cacheprovider > $OUT/pytest_md.log 2>&1; echo "pytest_md=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -3 $OUT/pytest_md.log
