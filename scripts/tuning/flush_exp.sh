# fused-kernel fp64 flush window (BORIS_FUSED_FLUSH 8 / 12 / 16): speed and fp32 parity margin
mkdir -p gpurun_out/fl
L=paper_2104_04579_b200/tuning_libs
for v in product fl12 fl16; do
  lib=""; [ $v != product ] && lib=$L/libboris_$v.so
  LIBBORIS_PATH=$lib timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/fl/fused_$v.jsonl 2>gpurun_out/fl/err_$v.txt; echo $v rc=$?
  LIBBORIS_PATH=$lib timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "C4_plane or C3_crossed or mdipole_parity or C1_ or other_orientations or alt_pusher_parity" > gpurun_out/fl/pytest_$v.log 2>&1; echo pytest $v rc=$?; tail -1 gpurun_out/fl/pytest_$v.log
done
