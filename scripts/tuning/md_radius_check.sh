# m-dipole: MUFU-rsqrt radius + skipped zero E_z kicks: GPU suite, m-dipole rows, Table-2 analytic
mkdir -p gpurun_out/mdr
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/mdr/pytest_gpu.log 2>&1; echo pytest rc=$?; grep -E "passed|failed" gpurun_out/mdr/pytest_gpu.log | tail -1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "mdipole_parity or C4_plane" > gpurun_out/mdr/pytest_md_print.log 2>&1; echo pytest-print rc=$?
timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/mdr/variants_md.jsonl 2>gpurun_out/mdr/variants.err; echo md rc=$?
timeout 600 python scripts/paper_table2.py --only analytic > gpurun_out/mdr/table2_analytic.txt 2>gpurun_out/mdr/table2.err; echo table2 rc=$?
