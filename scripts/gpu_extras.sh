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
    timeout 600 python scripts/pic_cycle.py --sort-every $se --fused >> gpurun_out/extras/pic_cycle.jsonl 2>> gpurun_out/extras/pic_cycle.err
  done
  echo pic rc=$?
fi
if [ $what = ncu ] || [ $what = all ]; then
  cap() {  # name kernel-regex skip command...
    local name=$1 rx=$2 skip=$3; shift 3
    timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c 1 \
      -o gpurun_out/prof2/$name -f "$@" > gpurun_out/prof2/$name.log 2>&1
    echo "ncu $name rc=$?"
    # keep the CSV pages, not the report (gpurun copies back at most 64 MiB)
    $NCU -i gpurun_out/prof2/$name.ncu-rep --page raw --csv > gpurun_out/prof2/${name}_raw.csv 2>/dev/null
    $NCU -i gpurun_out/prof2/$name.ncu-rep --page details --csv > gpurun_out/prof2/${name}_details.csv 2>/dev/null
    rm -f gpurun_out/prof2/$name.ncu-rep
  }
  PK="python scripts/prof_kernels.py --case"
  PF="python scripts/prof_fused.py"
  cap aos32 k_stream_aos 1 $PK aos32
  cap aos64 k_stream_aos 1 $PK aos64
  cap soa64 k_stream_soa_vec 1 $PK soa64
  cap fusedarr k_fused_arrays 1 $PK fusedarr
  cap grid '^k_stream_soa_grid' 1 $PK grid
  cap deposit '^k_deposit_runs' 1 $PK deposit
  cap rs_scatter k_rs_scatter 0 $PK sort
  cap permute_soa k_permute_soa 0 $PK sort
  cap fused_planewave_fp32 '^k_fused$' 1 $PF
  cap fused_planewave_fp64 '^k_fused$' 1 $PF --precision fp64
  cap fused_mdipole_fp32 '^k_fused$' 1 $PF --field mdipole
  cap fused_mdipole_fp64 '^k_fused$' 1 $PF --field mdipole --precision fp64
  cap fused_uniform_C3_fp64 '^k_fused$' 1 $PF --field uniform --precision fp64
  cap grid_fused20 '^k_fused$' 1 $PK grid --steps 20
  cap push_deposit 'k_push_deposit' 3 python scripts/pic_cycle.py --fused --steps 3
fi
if [ $what = sanitize ] || [ $what = all ]; then
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
      python scripts/sanitize_cases.py > gpurun_out/extras/sanitize_$tool.log 2>&1; echo sanitize $tool rc=$?
  done
fi
