# fused push+deposit occupancy variants (PIC cycle, sort every 10) + grid TMA 4-per-thread variants + ncu of the fused kernel
mkdir -p gpurun_out/pdexp
: > gpurun_out/pdexp/pic.jsonl
for rep in 1 2; do
  timeout 300 python scripts/pic_cycle.py --fused | sed 's/^{/{"v": "minb2", /' >> gpurun_out/pdexp/pic.jsonl 2>> gpurun_out/pdexp/err.log
  for t in pdminb1 pdminb3; do
    LIBBORIS_PATH=paper_2104_04579_b200/tuning_libs/libboris_$t.so timeout 300 python scripts/pic_cycle.py --fused | sed "s/^{/{\"v\": \"$t\", /" >> gpurun_out/pdexp/pic.jsonl 2>> gpurun_out/pdexp/err.log
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/pdexp/pic.jsonl'):
    d=json.loads(l); print(d['v'], round(d['ps_per_particle_step'],2), {k: round(v*1e3,1) for k,v in d['ms_per_step'].items()})
PY
timeout 600 bash scripts/tuning/grid_tma_exp.sh
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:'k_push_deposit' -s 3 -c 1 \
  -o gpurun_out/pdexp/pd -f python scripts/pic_cycle.py --fused --steps 3 > gpurun_out/pdexp/ncu.log 2>&1; echo ncu rc=$?
$NCU -i gpurun_out/pdexp/pd.ncu-rep --page raw --csv > gpurun_out/pdexp/pd_raw.csv 2>/dev/null
$NCU -i gpurun_out/pdexp/pd.ncu-rep --page source --csv --print-source sass > gpurun_out/pdexp/pd_src.csv 2>/dev/null
rm -f gpurun_out/pdexp/pd.ncu-rep
