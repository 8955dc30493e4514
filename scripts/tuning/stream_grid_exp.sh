# streaming kernel grid size under the board power cap (C5 8e8 bench, device-timed)
mkdir -p gpurun_out/sg
for rep in 1 2; do
for g in 0 148 296 592 1184; do
  BORIS_STREAM_GRID=$g timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sg/bench_g${g}_$rep.json 2>gpurun_out/sg/err.txt; echo g=$g rc=$?
done; done
