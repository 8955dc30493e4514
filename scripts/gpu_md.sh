#!/bin/bash
# m-dipole iteration: parity tests, Table-2 analytic cells, ncu instruction counts.
OUT=${1:-gpurun_out/md}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider -k "mdipole or field_evaluate or smoke" > $OUT/pytest_md.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
timeout 600 python scripts/paper_table2.py --only analytic --iters 5 > $OUT/table2.txt 2>&1; echo "table2=$?" >> $OUT/rc.txt
timeout 900 /usr/local/cuda/bin/ncu --metrics smsp__inst_executed.sum,smsp__inst_executed_pipe_xu.sum,smsp__inst_executed_pipe_fp64.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --csv --log-file $OUT/alu.csv python scripts/alu_counts.py run > $OUT/alu_run.log 2>&1; echo "alu=$?" >> $OUT/rc.txt
python scripts/alu_counts.py parse $OUT/alu.csv > $OUT/alu_counts.json 2>> $OUT/alu_run.log
cat $OUT/rc.txt; tail -2 $OUT/pytest_md.log
