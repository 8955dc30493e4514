# round-end style check 2: smoke, full GPU suite (incl. the > 2^31 tests), default bench
mkdir -p gpurun_out/r18
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r18/smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r18/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/r18/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/r18/bench.json 2> gpurun_out/r18/bench.err; echo bench rc=$?; cat gpurun_out/r18/bench.json
