# deposit tuning variants (tuning_libs/libboris_<tag>.so), back to back, twice
mkdir -p gpurun_out/dep
: > gpurun_out/dep/bench.jsonl
for rep in 1 2; do
for t in "$@"; do
  LIBBORIS_PATH=paper_2104_04579_b200/tuning_libs/libboris_$t.so timeout 300 python scripts/bench_deposit.py 2>>gpurun_out/dep/err.log | sed "s/^{/{\"lib\": \"$t\", /" >> gpurun_out/dep/bench.jsonl
done
done
python - <<'PY'
import json
for l in open('gpurun_out/dep/bench.jsonl'):
    d=json.loads(l); print(d['lib'],d['precision'],d['order'],round(d['ps_per_particle'],2))
PY
