# after the FMA rotation / deposit zero-kernel changes: variants, deposit, fused ncu,
# sanitizers on the new/opt-in kernels
mkdir -p gpurun_out/r10
NCU=/usr/local/cuda/bin/ncu
timeout 900 python scripts/bench_variants.py > gpurun_out/r10/variants.jsonl 2> gpurun_out/r10/variants.err; echo variants rc=$?
timeout 300 python scripts/bench_deposit.py > gpurun_out/r10/deposit.jsonl 2> gpurun_out/r10/deposit.err; echo deposit rc=$?
cat gpurun_out/r10/deposit.jsonl
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:'^k_fused$' -s 1 -c 1 \
  -o gpurun_out/r10/fused_planewave_fp32_yz -f python scripts/prof_fused.py > gpurun_out/r10/ncu_fused.log 2>&1; echo ncu fused rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:'^k_fused$' -s 1 -c 1 \
  -o gpurun_out/r10/fused_uniform_C3_fp64 -f python scripts/prof_fused.py --field uniform --precision fp64 > gpurun_out/r10/ncu_fused64.log 2>&1; echo ncu fused64 rc=$?
for tool in memcheck racecheck; do
  BORIS_GRID_KERNEL=tma timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
    python scripts/sanitize_cases.py > gpurun_out/r10/sanitize_gridtma_$tool.log 2>&1; echo sanitize gridtma $tool rc=$?
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
    python scripts/sanitize_cases.py > gpurun_out/r10/sanitize_$tool.log 2>&1; echo sanitize $tool rc=$?
done
