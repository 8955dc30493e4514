# deposition: per-lane chunks of 8M particles (merge once per chunk), M = 2, 4, 8
mkdir -p gpurun_out/dc
L=paper_2104_04579_b200/tuning_libs
for rep in 1 2; do
timeout 600 python scripts/bench_deposit.py > gpurun_out/dc/dep_default_$rep.jsonl 2>gpurun_out/dc/err.txt; echo default rc=$?
for v in dc2 dc4 dc8; do
  LIBBORIS_PATH=$L/libboris_$v.so timeout 600 python scripts/bench_deposit.py > gpurun_out/dc/dep_${v}_$rep.jsonl 2>>gpurun_out/dc/err.txt; echo $v rc=$?
done; done
for v in dc4 dc8; do
LIBBORIS_PATH=$L/libboris_$v.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "deposit" > gpurun_out/dc/pytest_$v.log 2>&1; echo pytest $v rc=$?; tail -1 gpurun_out/dc/pytest_$v.log
done
