#!/bin/bash
mkdir -p gpurun_out
python scripts/exp_stream.py --copy --tag default > gpurun_out/exp_stream.jsonl 2>gpurun_out/exp_stream.err
for t in precise minb3 precise_minb3; do
  LIBBORIS_PATH=paper_2104_04579_b200/build/libboris_$t.so python scripts/exp_stream.py --tag $t >> gpurun_out/exp_stream.jsonl 2>>gpurun_out/exp_stream.err
done
cat gpurun_out/exp_stream.jsonl
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python scripts/bench_variants.py > gpurun_out/variants.jsonl 2> gpurun_out/variants.err; echo variants rc=$?
cat gpurun_out/variants.jsonl; tail -3 gpurun_out/variants.err
