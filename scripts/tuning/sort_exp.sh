# sort / grid changes: GPU tests of grid/sort/deposit, grid+sort timing, PIC cycle, launch list of one sort
mkdir -p gpurun_out/sortexp
timeout 600 python -m pytest tests -m gpu -q -k "grid or sort or deposit or pic" -p no:cacheprovider > gpurun_out/sortexp/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/sortexp/pytest.log
timeout 600 python scripts/bench_grid.py > gpurun_out/sortexp/bench_grid.jsonl 2> gpurun_out/sortexp/bench_grid.err; echo grid rc=$?
python - <<'PY'
import json
for l in open('gpurun_out/sortexp/bench_grid.jsonl'):
    d=json.loads(l); print(d['exp'], d['precision'], d.get('order', d.get('input')), d.get('steps',''), round(d.get('ps_per_particle_step', d.get('ns_per_particle',0)*1000),2))
PY
: > gpurun_out/sortexp/pic_cycle.jsonl
for se in 1 10 1000000; do timeout 600 python scripts/pic_cycle.py --sort-every $se >> gpurun_out/sortexp/pic_cycle.jsonl 2>> gpurun_out/sortexp/pic.err; done; cat gpurun_out/sortexp/pic_cycle.jsonl
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sortexp/sort_launches.csv \
  python scripts/prof_kernels.py --case sort > gpurun_out/sortexp/sort.log 2>&1; echo sortncu rc=$?
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:'^k_fused$' -s 1 -c 1 \
  -o gpurun_out/sortexp/grid_fused20 -f python scripts/prof_kernels.py --case grid --steps 20 > gpurun_out/sortexp/fused.log 2>&1; echo fused rc=$?
