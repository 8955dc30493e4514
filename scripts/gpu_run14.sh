#!/bin/bash
mkdir -p gpurun_out
BORIS_SOA_KERNEL=tma timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "soa or C2 or C5 or sharded or mixed or fused_arrays or kinetic or small" > gpurun_out/pytest_tma.log 2>&1; echo pytest-tma rc=$?
grep -E "passed|failed" gpurun_out/pytest_tma.log | tail -2; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_tma.log | head -20
python scripts/exp_stream.py --tag ldg --sizes 1e8,4e8,8e8 > gpurun_out/exp_tma.jsonl 2>gpurun_out/exp_tma.err
BORIS_SOA_KERNEL=tma python scripts/exp_stream.py --tag tma --sizes 1e8,4e8,8e8 >> gpurun_out/exp_tma.jsonl 2>>gpurun_out/exp_tma.err
python scripts/exp_stream.py --tag ldg2 --sizes 1e8,8e8 >> gpurun_out/exp_tma.jsonl 2>>gpurun_out/exp_tma.err
BORIS_SOA_KERNEL=tma python scripts/exp_stream.py --tag tma2 --sizes 1e8,8e8 >> gpurun_out/exp_tma.jsonl 2>>gpurun_out/exp_tma.err
cat gpurun_out/exp_tma.jsonl; tail -3 gpurun_out/exp_tma.err
