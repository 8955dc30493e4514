# ncu --set full of the register-cached fused grid kernel (100 steps) and the
# m-dipole fp32 fused kernel (grouped, 16-step windows)
mkdir -p gpurun_out/prof3
NCU=/usr/local/cuda/bin/ncu
cap() {
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c 1 \
    -o gpurun_out/prof3/$name -f "$@" > gpurun_out/prof3/$name.log 2>&1
  echo "ncu $name rc=$?"
  $NCU -i gpurun_out/prof3/$name.ncu-rep --page raw --csv > gpurun_out/prof3/${name}_raw.csv 2>/dev/null
  $NCU -i gpurun_out/prof3/$name.ncu-rep --page details --csv > gpurun_out/prof3/${name}_details.csv 2>/dev/null
  rm -f gpurun_out/prof3/$name.ncu-rep
}
cap grid_fused100_cached '^k_fused$' 1 python scripts/prof_kernels.py --case grid --steps 100
cap fused_mdipole_fp32_grouped '^k_fused$' 1 python scripts/prof_fused.py --field mdipole
