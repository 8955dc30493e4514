# fused grid kernel (register-cached records): fp32 occupancy 4 (default) / 5 / 6 blocks per SM
mkdir -p gpurun_out/gfm
L=paper_2104_04579_b200/tuning_libs
for rep in 1 2; do
timeout 600 python scripts/bench_grid.py > gpurun_out/gfm/grid_default_$rep.jsonl 2>gpurun_out/gfm/err.txt; echo default rc=$?
for v in gf5 gf6; do
LIBBORIS_PATH=$L/libboris_$v.so timeout 600 python scripts/bench_grid.py > gpurun_out/gfm/grid_${v}_$rep.jsonl 2>>gpurun_out/gfm/err.txt; echo $v rc=$?
done; done
