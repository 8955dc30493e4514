# one reciprocal square root for t and s in the fused uniform / plane-wave Boris step
mkdir -p gpurun_out/mr
L=paper_2104_04579_b200/tuning_libs
for rep in 1 2; do
for v in product mr; do
  lib=""; [ $v != product ] && lib=$L/libboris_$v.so
  LIBBORIS_PATH=$lib timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/mr/fused_${v}_$rep.jsonl 2>gpurun_out/mr/err_$v.txt; echo $v rc=$?
done; done
LIBBORIS_PATH=$L/libboris_mr.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "C4_plane or C3_crossed or C1_ or other_orientations or axis_aligned or host_resident_analytic or graph" > gpurun_out/mr/pytest_mr.log 2>&1; echo pytest mr rc=$?; tail -1 gpurun_out/mr/pytest_mr.log
