# fused-kernel grid policy (BORIS_FUSED_GRID 1: 4-wave grid-stride cap, 2: one block per
# 128 (x MD_GROUP) particles) and m-dipole branch grouping (BORIS_MD_GROUP)
mkdir -p gpurun_out/fg2
L=paper_2104_04579_b200/tuning_libs
for v in g1w g1a; do
  LIBBORIS_PATH=$L/libboris_$v.so timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/fg2/fused_$v.jsonl 2>gpurun_out/fg2/err_$v.txt; echo $v rc=$?
done
for v in g1w g1a g2a g4a g1w g1a g2a g4a; do
  LIBBORIS_PATH=$L/libboris_$v.so timeout 600 python scripts/bench_variants.py --mdipole-only >> gpurun_out/fg2/md_$v.jsonl 2>>gpurun_out/fg2/err_$v.txt; echo md $v rc=$?
done
