#!/bin/bash
# Round-end evidence: smoke, GPU suite, default bench line, Table-2 replica, grid/sort/
# deposition/PIC benches, ncu launch list of the bench.  Usage: bash scripts/gpu_final.sh <outdir>
OUT=${1:-gpurun_out/final}; mkdir -p $OUT
bash scripts/gpu_full.sh $OUT
timeout 900 python scripts/paper_table2.py --iters 5 > $OUT/table2.txt 2>&1; echo "table2=$?" >> $OUT/rc.txt
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stream|k_diag|k_fused" -c 40 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
  > $OUT/launches_bench.log 2>&1; echo "ncu_launches=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
