# ncu --set full of the grid gather kernels (single step LDG, fused 20 steps) and the
# launch list of one sort (per-kernel durations)
mkdir -p gpurun_out/gridncu
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:'^k_stream_soa_grid$' -s 1 -c 1 \
  -o gpurun_out/gridncu/grid_step -f python scripts/prof_kernels.py --case grid > gpurun_out/gridncu/step.log 2>&1; echo step rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:'^k_fused$' -s 1 -c 1 \
  -o gpurun_out/gridncu/grid_fused20 -f python scripts/prof_kernels.py --case grid --steps 20 > gpurun_out/gridncu/fused.log 2>&1; echo fused rc=$?
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gridncu/sort_launches.csv \
  python scripts/prof_kernels.py --case sort > gpurun_out/gridncu/sort.log 2>&1; echo sort rc=$?
