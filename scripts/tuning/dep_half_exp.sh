# deposition: lane's 8 particles staged as two halves of 4 (BORIS_DEP_HALF), 2 or 3 blocks/SM
mkdir -p gpurun_out/dh
L=paper_2104_04579_b200/tuning_libs
for rep in 1 2; do
timeout 600 python scripts/bench_deposit.py > gpurun_out/dh/dep_default_$rep.jsonl 2>gpurun_out/dh/err.txt; echo default rc=$?
for v in dh2 dh3; do
  LIBBORIS_PATH=$L/libboris_$v.so timeout 600 python scripts/bench_deposit.py > gpurun_out/dh/dep_${v}_$rep.jsonl 2>>gpurun_out/dh/err.txt; echo $v rc=$?
done; done
LIBBORIS_PATH=$L/libboris_dh2.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "deposit" > gpurun_out/dh/pytest_dh2.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/dh/pytest_dh2.log
