# fused grid kernel: cell records cached in registers across steps vs per-step gathers
mkdir -p gpurun_out/gc
L=paper_2104_04579_b200/tuning_libs
timeout 900 python scripts/bench_grid.py > gpurun_out/gc/grid_cache.jsonl 2>gpurun_out/gc/err.txt; echo cache rc=$?
LIBBORIS_PATH=$L/libboris_gc0.so timeout 900 python scripts/bench_grid.py > gpurun_out/gc/grid_gc0.jsonl 2>>gpurun_out/gc/err.txt; echo gc0 rc=$?
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "grid or sort or deposit" > gpurun_out/gc/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/gc/pytest.log
