set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --particles 100000000 --steps 20 --warmup 3 --e2e-steps 2 > gpurun_out/bench_1e8.json 2> gpurun_out/bench_1e8.err; echo bench rc=$?
cat gpurun_out/bench_1e8.json
tail -20 gpurun_out/bench_1e8.err
