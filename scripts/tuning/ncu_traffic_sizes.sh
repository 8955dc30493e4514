# dram traffic per launch of the bench kernel at the per-GPU sizes of N = 2 and 4 (4e8, 2e8)
mkdir -p gpurun_out/traffic
NCU=/usr/local/cuda/bin/ncu
for n in 400000000 200000000; do
  timeout 900 $NCU --set full --clock-control none -k regex:k_stream_soa_vec -s 3 -c 1 \
    -o gpurun_out/traffic/soa_$n -f python bench.py --particles $n --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/traffic/soa_$n.log 2>&1; echo ncu $n rc=$?
  $NCU -i gpurun_out/traffic/soa_$n.ncu-rep --page raw --csv > gpurun_out/traffic/soa_${n}_raw.csv 2>/dev/null
  rm -f gpurun_out/traffic/soa_$n.ncu-rep
done
