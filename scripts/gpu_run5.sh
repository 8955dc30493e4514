#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "C4 or mdipole or C3 or C1 or field_eval or host_resident_analytic or full_size" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
grep -E "^(fp32|fp64) " gpurun_out/pytest_gpu.log | head
python scripts/bench_variants.py --quick > gpurun_out/variants.jsonl 2> gpurun_out/variants.err; echo variants rc=$?
grep -E "C3|C4|mdipole" gpurun_out/variants.jsonl
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 \
  -o gpurun_out/prof_fused_pw_fp32 -f python scripts/prof_fused.py > gpurun_out/prof_fused.log 2>&1; echo ncu rc=$?
