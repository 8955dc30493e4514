# fp64 m-dipole closed form with the reduced-range sincos: parity, rows, Table 2 analytic
mkdir -p gpurun_out/msc
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "mdipole or field_evaluate or grid_fused_push_with" > gpurun_out/msc/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/msc/pytest.log
timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/msc/variants_md.jsonl 2>gpurun_out/msc/err.txt; echo md rc=$?
timeout 600 python scripts/paper_table2.py --only analytic > gpurun_out/msc/table2_analytic.txt 2>>gpurun_out/msc/err.txt; echo table2 rc=$?
