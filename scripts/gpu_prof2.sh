#!/bin/bash
mkdir -p gpurun_out/prof2
NCU=/usr/local/cuda/bin/ncu
run() {  # name case kernel-regex skip
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c 1 \
    -o gpurun_out/prof2/$1 -f python scripts/prof_kernels.py --case $2 > gpurun_out/prof2/$1.log 2>&1
  echo "$1 rc=$?"
}
run aos32 aos32 k_stream_aos 1
run aos64 aos64 k_stream_aos 1
run soa64 soa64 k_stream_soa_vec 1
run fusedarr fusedarr k_fused_arrays 1
run grid grid "k_fused<" 1
run deposit deposit k_deposit 1
run rs_scatter sort k_rs_scatter 0
run rs_hist sort k_rs_hist 0
