#!/bin/bash
# streaming-kernel tuning variants (cache hints, block size), back to back at 1e8 and 8e8
mkdir -p gpurun_out
: > gpurun_out/exp2.jsonl
for t in default l2pf stwb t512 t128 l2pf_stwb default; do
  if [ $t = default ]; then L=paper_2104_04579_b200/libboris.so; else L=paper_2104_04579_b200/tuning_libs/libboris_$t.so; fi
  LIBBORIS_PATH=$L python scripts/exp_stream.py --tag $t --sizes 1e8,8e8 >> gpurun_out/exp2.jsonl 2>>gpurun_out/exp2.err
done
cat gpurun_out/exp2.jsonl; tail -3 gpurun_out/exp2.err
