# after making BORIS_FUSED_GRID=2 / BORIS_MD_GROUP=2 the defaults: GPU suite, sanitizers,
# fused variant rows, Table-2 replica
mkdir -p gpurun_out/fgc
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fgc/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/fgc/pytest_gpu.log
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/fgc/sanitize_$tool.log 2>&1; echo sanitize $tool rc=$?
done
timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/fgc/variants_fused.jsonl 2>gpurun_out/fgc/variants.err; echo variants rc=$?
timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/fgc/variants_md.jsonl 2>>gpurun_out/fgc/variants.err; echo md rc=$?
timeout 900 python scripts/paper_table2.py > gpurun_out/fgc/table2.txt 2>gpurun_out/fgc/table2.err; echo table2 rc=$?
