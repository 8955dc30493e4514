#!/bin/bash
# Session 6: ncu full + source of the sorted single-step grid push and the fp32 m-dipole fused kernel.
OUT=gpurun_out/s6; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stream_soa_grid" -s 1 -c 1 \
  -o $OUT/grid -f python scripts/prof_kernels.py --case grid > $OUT/ncu_grid.log 2>&1; echo "grid=$?" >> $OUT/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 1 -c 1 \
  -o $OUT/md32 -f python scripts/prof_fused.py --field mdipole --n 2000000 --steps 200 --reps 2 > $OUT/ncu_md.log 2>&1; echo "md=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
