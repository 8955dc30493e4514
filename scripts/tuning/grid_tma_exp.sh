# grid single step: LDG default vs TMA-staged state with 4 particles per thread (tile 1024)
mkdir -p gpurun_out/gridtma
: > gpurun_out/gridtma/bench.jsonl
for rep in 1 2; do
  BORIS_GRID_KERNEL=ldg timeout 300 python scripts/bench_grid.py --steps 1 2>>gpurun_out/gridtma/err.log | grep grid_push | sed "s/^{/{\"v\": \"ldg\", /" >> gpurun_out/gridtma/bench.jsonl
  for t in tp1024s3 tp1024s2 tp512s4; do
    BORIS_GRID_KERNEL=tma LIBBORIS_PATH=paper_2104_04579_b200/tuning_libs/libboris_$t.so timeout 300 python scripts/bench_grid.py --steps 1 2>>gpurun_out/gridtma/err.log | grep grid_push | sed "s/^{/{\"v\": \"$t\", /" >> gpurun_out/gridtma/bench.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/gridtma/bench.jsonl'):
    d=json.loads(l)
    if d['steps']==1: print(d['v'],d['precision'],d['order'],round(d['ps_per_particle_step'],2))
PY
