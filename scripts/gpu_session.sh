#!/bin/bash
# One gpurun session: GPU tests, the perturbed-a10 tuning build, the bench line and the
# ncu instruction counts of the fused kernels.  Usage: scripts/gpu_session.sh <outdir>
OUT=${1:-gpurun_out/s}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $OUT/rc.txt
LIBBORIS_PATH=paper_2104_04579_b200/tuning_libs/libboris_perturb_cr.so timeout 300 \
  python -m pytest tests/test_gpu_parity.py -q -k "test_C2_arrays_parity" > $OUT/perturb_cr.log 2>&1; echo "perturb_rc=$?" >> $OUT/rc.txt
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench_rc=$?" >> $OUT/rc.txt
timeout 600 ncu --metrics smsp__inst_executed.sum,smsp__inst_executed_pipe_xu.sum,smsp__inst_executed_pipe_fp64.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --print-units base --csv --log-file $OUT/alu.csv python scripts/alu_counts.py run > $OUT/alu.log 2>&1; echo "ncu_rc=$?" >> $OUT/rc.txt
python scripts/alu_counts.py parse $OUT/alu.csv > $OUT/alu_counts.json 2>> $OUT/alu.log
cat $OUT/rc.txt; tail -3 $OUT/pytest_gpu.log; tail -3 $OUT/perturb_cr.log; head -c 600 $OUT/bench.json
