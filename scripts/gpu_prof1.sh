#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 \
  -o gpurun_out/prof_fused_pw_fp32 -f python scripts/prof_fused.py > gpurun_out/prof_fused.log 2>&1; echo ncu rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 \
  -o gpurun_out/prof_fused_md_fp32 -f python scripts/prof_fused.py --field mdipole > gpurun_out/prof_fused_md.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/prof_fused.log
