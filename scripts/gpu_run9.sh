#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "alt_pusher" -s > gpurun_out/pytest_alt.log 2>&1; echo pytest-alt rc=$?
grep -E "passed|failed" gpurun_out/pytest_alt.log | tail -2; grep -E "^(FAILED|ERROR)|Error" gpurun_out/pytest_alt.log | head -20
grep -E "^C[234] " gpurun_out/pytest_alt.log | head -20
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest-all rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head -20
