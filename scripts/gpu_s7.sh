#!/bin/bash
# Session 7: folded m-dipole step: parity tests, Table-2 replica, ncu instruction mix.
OUT=gpurun_out/s7; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "mdipole or field_evaluate or alt_pusher" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
timeout 900 python scripts/paper_table2.py > $OUT/table2.txt 2> $OUT/table2.err; echo "table2=$?" >> $OUT/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 1 -c 1 \
  -o $OUT/md32 -f python scripts/prof_fused.py --field mdipole --n 2000000 --steps 200 --reps 2 > $OUT/ncu_md.log 2>&1; echo "md=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -2 $OUT/pytest.log
