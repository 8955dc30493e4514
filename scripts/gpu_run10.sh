#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "deposit" > gpurun_out/pytest_dep.log 2>&1; echo pytest-dep rc=$?
grep -E "passed|failed" gpurun_out/pytest_dep.log | tail -2; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/pytest_dep.log | head -20
python scripts/bench_deposit.py > gpurun_out/bench_deposit.jsonl 2> gpurun_out/bench_deposit.err; echo dep rc=$?
cat gpurun_out/bench_deposit.jsonl; tail -3 gpurun_out/bench_deposit.err
