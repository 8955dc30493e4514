#!/bin/bash
# Session 3: warp-run deposition variants (tests + bench), sort timings, ncu of the new kernels.
OUT=gpurun_out/s3; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "deposit or sort" -p no:cacheprovider > $OUT/pytest_default.log 2>&1; echo "pytest_default=$?" >> $OUT/rc.txt
for t in default dw_pd2_mb3 dw_pd3_mb2 dw_pd8_mb1; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  for rep in 1 2; do LIBBORIS_PATH=$L timeout 300 python scripts/bench_deposit.py | sed "s/^{/{\"v\": \"$t\", /" >> $OUT/dep.jsonl 2>> $OUT/dep.err; done
done
timeout 600 python scripts/bench_grid.py > $OUT/grid.jsonl 2> $OUT/grid.err; echo "grid_rc=$?" >> $OUT/rc.txt
timeout 600 python scripts/pic_cycle.py > $OUT/pic.jsonl 2> $OUT/pic.err; echo "pic_rc=$?" >> $OUT/rc.txt
timeout 600 python scripts/pic_cycle.py --fused > $OUT/pic_fused.jsonl 2>> $OUT/pic.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_deposit_warp" -s 2 -c 1 -o $OUT/dep_warp -f python scripts/bench_deposit.py > $OUT/ncu_dep.log 2>&1; echo "ncu_dep=$?" >> $OUT/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_pack|k_unpack|k_rs|k_deposit|k_zero" --csv --log-file $OUT/sort_ncu.csv \
  python scripts/bench_grid.py --n 10000000 --steps 2 > $OUT/sort_ncu.log 2>&1; echo "ncu_sort=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -2 $OUT/pytest_default.log
