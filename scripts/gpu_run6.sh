#!/bin/bash
# multi-rank code path on one GPU (gloo), paper Table 2 replica, sanitizers
mkdir -p gpurun_out
BORIS_SHARE_GPU=1 BORIS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --particles 100000000 --steps 10 --warmup 3 --e2e-steps 1 \
  > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err; echo 2rank rc=$?
cat gpurun_out/bench_2rank_gloo.json; tail -3 gpurun_out/bench_2rank_gloo.err
timeout 900 python scripts/paper_table2.py > gpurun_out/paper_table2.txt 2> gpurun_out/paper_table2.err; echo table2 rc=$?
tail -15 gpurun_out/paper_table2.txt; tail -3 gpurun_out/paper_table2.err
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1; echo $tool rc=$?
  tail -3 gpurun_out/sanitize_$tool.log
done
