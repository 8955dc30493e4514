# merged reciprocal square root on the fp64 uniform-field kernels: GPU suite + fused rows
mkdir -p gpurun_out/mrc
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/mrc/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/mrc/pytest_gpu.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "C3_crossed or C1_" > gpurun_out/mrc/pytest_print.log 2>&1; echo pytest-print rc=$?
timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/mrc/variants_fused.jsonl 2>gpurun_out/mrc/err.txt; echo variants rc=$?
