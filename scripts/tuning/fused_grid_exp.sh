# resident (one-wave) grid for the fused kernels and m-dipole branch grouping vs the
# earlier 4-wave grid: fused variant rows for each library build
mkdir -p gpurun_out/fg
L=paper_2104_04579_b200/tuning_libs
timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/fg/fused_product.jsonl 2>gpurun_out/fg/err_product.txt; echo product rc=$?
LIBBORIS_PATH=$L/libboris_waves.so timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/fg/fused_waves.jsonl 2>gpurun_out/fg/err_waves.txt; echo waves rc=$?
LIBBORIS_PATH=$L/libboris_mdg1.so timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/fg/md_mdg1.jsonl 2>gpurun_out/fg/err_mdg1.txt; echo mdg1 rc=$?
timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/fg/md_product.jsonl 2>>gpurun_out/fg/err_product.txt; echo md product rc=$?
LIBBORIS_PATH=$L/libboris_waves.so timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/fg/md_waves.jsonl 2>>gpurun_out/fg/err_waves.txt; echo md waves rc=$?
