# final round-end style check: smoke, full GPU suite, default bench, reference arm,
# sanitizers, fused rows, Table 2, ncu of the m-dipole fp32 kernel
mkdir -p gpurun_out/r21 gpurun_out/prof4
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r21/smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r21/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/r21/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/r21/bench.json 2> gpurun_out/r21/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r21/bench_ref.json 2>gpurun_out/r21/bench_ref.err; echo ref rc=$?
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/r21/sanitize_$tool.log 2>&1; echo sanitize $tool rc=$?
done
timeout 900 python scripts/bench_variants.py --fused-only > gpurun_out/r21/variants_fused.jsonl 2>gpurun_out/r21/err.txt; echo variants rc=$?
timeout 1200 python scripts/paper_table2.py > gpurun_out/r21/table2.txt 2>>gpurun_out/r21/err.txt; echo table2 rc=$?
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:'^k_fused$' -s 1 -c 1 -o gpurun_out/prof4/fused_mdipole_fp32 -f python scripts/prof_fused.py --field mdipole > gpurun_out/prof4/md.log 2>&1; echo ncu rc=$?
$NCU -i gpurun_out/prof4/fused_mdipole_fp32.ncu-rep --page raw --csv > gpurun_out/prof4/fused_mdipole_fp32_raw.csv 2>/dev/null
rm -f gpurun_out/prof4/fused_mdipole_fp32.ncu-rep
