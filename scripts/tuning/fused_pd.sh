# fused push + deposit: GPU tests, PIC cycle fused vs separate
mkdir -p gpurun_out/fpd
timeout 900 python -m pytest tests -m gpu -q -k "push_deposit or deposit or grid or sort" -p no:cacheprovider > gpurun_out/fpd/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/fpd/pytest.log; grep -E "^(FAILED|ERROR)|Error" gpurun_out/fpd/pytest.log | head
: > gpurun_out/fpd/pic.jsonl
for rep in 1 2; do
for se in 10 1; do
  timeout 300 python scripts/pic_cycle.py --sort-every $se >> gpurun_out/fpd/pic.jsonl 2>> gpurun_out/fpd/pic.err
  timeout 300 python scripts/pic_cycle.py --sort-every $se --fused >> gpurun_out/fpd/pic.jsonl 2>> gpurun_out/fpd/pic.err
done
done
python - <<'PY'
import json
for l in open('gpurun_out/fpd/pic.jsonl'):
    d=json.loads(l); print(d['fused'], d['sort_every'], round(d['ps_per_particle_step'],2), {k: round(v*1e3,1) for k,v in d['ms_per_step'].items()})
PY
timeout 300 bash scripts/tuning/grid_tma_exp.sh
