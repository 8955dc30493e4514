#!/bin/bash
# ncu evidence for the bench line (run under gpurun): the launch list of the bench's own
# command (per-launch time, cold and serialised -> the kernel's SHARE of the step) and one
# `--set full` capture of the timed kernel at the bench size (DRAM traffic per launch).
# Usage: bash scripts/gpu_evidence.sh <outdir>
OUT=${1:-gpurun_out/ev}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stream|k_diag|k_fused" -c 40 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
  --no-configs > $OUT/launches.log 2>&1; echo "launches=$?" >> $OUT/rc.txt
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:k_stream_soa_vec -s 3 -c 1 \
  -o $OUT/soa_8e8 -f python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-configs \
  > $OUT/full.log 2>&1; echo "full=$?" >> $OUT/rc.txt
$NCU -i $OUT/soa_8e8.ncu-rep --page raw --csv > $OUT/soa_8e8_raw.csv 2>/dev/null
$NCU -i $OUT/soa_8e8.ncu-rep --page details --csv > $OUT/soa_8e8_details.csv 2>/dev/null
cat $OUT/rc.txt
