# after the fused-kernel changes (grid, m-dipole grouping/radius, 16-step fp32 windows,
# fp64 merged rsqrt, fp64 1/xi via rcp_rn): fused rows, Table 2, ncu of every kernel family
mkdir -p gpurun_out/r16 gpurun_out/prof2
timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/r16/variants_fused.jsonl 2>gpurun_out/r16/err.txt; echo variants rc=$?
timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/r16/variants_md.jsonl 2>>gpurun_out/r16/err.txt; echo md rc=$?
timeout 1200 python scripts/paper_table2.py > gpurun_out/r16/table2.txt 2>>gpurun_out/r16/err.txt; echo table2 rc=$?
bash scripts/gpu_extras.sh ncu
