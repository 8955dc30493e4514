# fp32 flush window 16 as the default: GPU suite, fused rows, grid rows, Table-2 analytic
mkdir -p gpurun_out/flc
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/flc/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/flc/pytest_gpu.log
timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/flc/variants_fused.jsonl 2>gpurun_out/flc/err.txt; echo variants rc=$?
timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/flc/variants_md.jsonl 2>>gpurun_out/flc/err.txt; echo md rc=$?
timeout 900 python scripts/bench_grid.py > gpurun_out/flc/grid.jsonl 2>>gpurun_out/flc/err.txt; echo grid rc=$?
timeout 600 python scripts/paper_table2.py --only analytic > gpurun_out/flc/table2_analytic.txt 2>>gpurun_out/flc/err.txt; echo table2 rc=$?
