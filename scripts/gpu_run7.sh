#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head -20
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
python scripts/bench_variants.py > gpurun_out/variants.jsonl 2> gpurun_out/variants.err; echo variants rc=$?
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stream|k_diag|k_fused" -c 40 \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1; echo ncu-launches rc=$?
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:k_stream_soa_vec -s 3 -c 1 \
  -o gpurun_out/prof_soa_8e8 -f python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/prof_soa_8e8.log 2>&1; echo ncu-full-8e8 rc=$?
tail -3 gpurun_out/prof_soa_8e8.log
