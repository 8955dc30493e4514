#!/bin/bash
OUT=gpurun_out/s20; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "deposit" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
for rep in 1 2; do
for t in default noTMA tA tB tC tD tE; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L timeout 300 python scripts/bench_deposit.py | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/dep.jsonl 2>> $OUT/err.log
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_deposit" -s 1 -c 1 \
  -o $OUT/dep -f python scripts/prof_deposit.py > $OUT/ncu_dep.log 2>&1; echo "ncu=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -2 $OUT/pytest.log
