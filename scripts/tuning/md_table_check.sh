mkdir -p gpurun_out/mt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "mdipole or field_evaluate" > gpurun_out/mt/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/mt/pytest.log
timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/mt/variants_md.jsonl 2>gpurun_out/mt/err.txt; echo md rc=$?
timeout 600 python scripts/paper_table2.py --only analytic > gpurun_out/mt/table2.txt 2>>gpurun_out/mt/err.txt; echo t2 rc=$?
