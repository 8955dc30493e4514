# single-step grid push: lane-consecutive particles (BORIS_GRID_KERNEL=lanes) vs default
mkdir -p gpurun_out/gl
for rep in 1 2; do
timeout 600 python scripts/bench_grid.py > gpurun_out/gl/grid_ldg_$rep.jsonl 2>gpurun_out/gl/err.txt; echo ldg rc=$?
BORIS_GRID_KERNEL=lanes timeout 600 python scripts/bench_grid.py > gpurun_out/gl/grid_lanes_$rep.jsonl 2>>gpurun_out/gl/err.txt; echo lanes rc=$?
done
BORIS_GRID_KERNEL=lanes timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "grid or sort or deposit" > gpurun_out/gl/pytest_lanes.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/gl/pytest_lanes.log
BORIS_GRID_KERNEL=lanes timeout 600 python scripts/pic_cycle.py > gpurun_out/gl/pic_lanes.jsonl 2>>gpurun_out/gl/err.txt; echo pic rc=$?
