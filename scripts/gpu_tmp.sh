#!/bin/bash
OUT=gpurun_out/s40; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "deposit or pic" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
for rep in 1 2 3; do timeout 300 python scripts/pic_cycle.py --fused >> $OUT/pic.jsonl 2>> $OUT/err.log; done
cat $OUT/rc.txt
