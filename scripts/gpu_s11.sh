#!/bin/bash
# Session 11: deposition into the padded interleaved J4 scratch (vector atomics).
OUT=gpurun_out/s11; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "deposit or grid or sort" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
for rep in 1 2; do
  timeout 300 python scripts/bench_deposit.py >> $OUT/dep.jsonl 2>> $OUT/err.log
  timeout 300 python scripts/pic_cycle.py --fused >> $OUT/pic.jsonl 2>> $OUT/err.log
  timeout 300 python scripts/pic_cycle.py >> $OUT/pic.jsonl 2>> $OUT/err.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_deposit" -s 1 -c 1 \
  -o $OUT/dep -f python scripts/prof_deposit.py > $OUT/ncu_dep.log 2>&1; echo "ncu=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -2 $OUT/pytest.log
