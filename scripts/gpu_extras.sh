#!/bin/bash
# Secondary measurements (run under gpurun from the repo root):
#   per-kernel variants, paper Table-2 replica, grid gather + sort, deposition,
#   ncu captures of every kernel family, compute-sanitizer on every variant.
# Usage: bash scripts/gpu_extras.sh [variants|table2|grid|deposit|ncu|sanitize|all]
what=${1:-all}
mkdir -p gpurun_out/extras gpurun_out/prof2
NCU=/usr/local/cuda/bin/ncu
if [ $what = variants ] || [ $what = all ]; then
  python scripts/bench_variants.py > gpurun_out/extras/variants.jsonl 2> gpurun_out/extras/variants.err; echo variants rc=$?
fi
if [ $what = table2 ] || [ $what = all ]; then
  timeout 900 python scripts/paper_table2.py > gpurun_out/extras/paper_table2.txt 2> gpurun_out/extras/paper_table2.err; echo table2 rc=$?
fi
if [ $what = grid ] || [ $what = all ]; then
  timeout 600 python scripts/bench_grid.py > gpurun_out/extras/bench_grid.jsonl 2> gpurun_out/extras/bench_grid.err; echo grid rc=$?
fi
if [ $what = deposit ] || [ $what = all ]; then
  timeout 600 python scripts/bench_deposit.py > gpurun_out/extras/bench_deposit.jsonl 2> gpurun_out/extras/bench_deposit.err; echo deposit rc=$?
fi
if [ $what = pic ] || [ $what = all ]; then
  for se in 1 10 1000000; do
    timeout 600 python scripts/pic_cycle.py --sort-every $se >> gpurun_out/extras/pic_cycle.jsonl 2>> gpurun_out/extras/pic_cycle.err
  done
  echo pic rc=$?
fi
if [ $what = ncu ] || [ $what = all ]; then
  run() {  # name case kernel-regex skip
    timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c 1 \
      -o gpurun_out/prof2/$1 -f python scripts/prof_kernels.py --case $2 > gpurun_out/prof2/$1.log 2>&1
    echo "ncu $1 rc=$?"
  }
  run aos32 aos32 k_stream_aos 1
  run aos64 aos64 k_stream_aos 1
  run soa64 soa64 k_stream_soa_vec 1
  run fusedarr fusedarr k_fused_arrays 1
  run grid grid '^k_fused$' 1
  run deposit deposit k_deposit 1
  run rs_scatter sort k_rs_scatter 0
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:'^k_fused$' -s 1 -c 1 \
    -o gpurun_out/prof2/fused_planewave_fp32 -f python scripts/prof_fused.py > gpurun_out/prof2/fused_pw.log 2>&1
  echo "ncu fused_planewave rc=$?"
fi
if [ $what = sanitize ] || [ $what = all ]; then
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
      python scripts/sanitize_cases.py > gpurun_out/extras/sanitize_$tool.log 2>&1; echo sanitize $tool rc=$?
  done
fi
