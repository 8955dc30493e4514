#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "grid or sort" -s > gpurun_out/pytest_grid.log 2>&1; echo pytest rc=$?
grep -E "passed|failed" gpurun_out/pytest_grid.log | tail -2; grep -E "^(FAILED|ERROR)|^fp|Error" gpurun_out/pytest_grid.log | head -20
timeout 600 python scripts/bench_grid.py > gpurun_out/bench_grid.jsonl 2> gpurun_out/bench_grid.err; echo grid rc=$?
cat gpurun_out/bench_grid.jsonl; tail -3 gpurun_out/bench_grid.err
