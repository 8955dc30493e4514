# launch/occupancy sections of the C4 fused kernel: resident grid vs 4-wave grid
mkdir -p gpurun_out/fg
NCU=/usr/local/cuda/bin/ncu
L=paper_2104_04579_b200/tuning_libs
for v in product waves; do
  lib=""; [ $v = waves ] && lib=$L/libboris_waves.so
  LIBBORIS_PATH=$lib timeout 300 $NCU --section LaunchStats --section Occupancy --section SpeedOfLight --metrics smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.max,smsp__warps_active.avg.per_cycle_active --clock-control none -k regex:'^k_fused$' -s 1 -c 1 --csv --page raw python scripts/prof_fused.py --reps 2 > gpurun_out/fg/ncu_$v.csv 2>gpurun_out/fg/ncu_$v.err; echo $v rc=$?
done
