# single-step grid push: per-thread cell-record cache across its 4 consecutive particles
mkdir -p gpurun_out/gsc
L=paper_2104_04579_b200/tuning_libs
timeout 900 python scripts/bench_grid.py > gpurun_out/gsc/grid_default.jsonl 2>gpurun_out/gsc/err.txt; echo default rc=$?
for v in gsc2 gsc3; do
LIBBORIS_PATH=$L/libboris_$v.so timeout 900 python scripts/bench_grid.py > gpurun_out/gsc/grid_$v.jsonl 2>>gpurun_out/gsc/err.txt; echo $v rc=$?
done
LIBBORIS_PATH=$L/libboris_gsc2.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "grid or sort or deposit" > gpurun_out/gsc/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/gsc/pytest.log
