# grid single-step kernel: LDG (default) vs TMA-staged state, back to back, twice;
# then the grid/sort/deposit GPU tests with the TMA kernel selected
mkdir -p gpurun_out/gridexp
: > gpurun_out/gridexp/bench.jsonl
for rep in 1 2; do
for k in ldg tma; do
  BORIS_GRID_KERNEL=$k timeout 300 python scripts/bench_grid.py --steps 1 2>>gpurun_out/gridexp/err.log | grep grid_push | sed "s/^{/{\"kernel\": \"$k\", /" >> gpurun_out/gridexp/bench.jsonl
done
done
python - <<'PY'
import json
for l in open('gpurun_out/gridexp/bench.jsonl'):
    d=json.loads(l); print(d['kernel'],d['precision'],d['order'],d['steps'],round(d['ps_per_particle_step'],2))
PY
BORIS_GRID_KERNEL=tma timeout 600 python -m pytest tests -m gpu -q -k "grid or sort or deposit or pic" -p no:cacheprovider > gpurun_out/gridexp/pytest_tma.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/gridexp/pytest_tma.log
