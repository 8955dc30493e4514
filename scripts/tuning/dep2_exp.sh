# deposit with unwrapped-floor cell test: GPU tests + deposit bench + PIC cycle
mkdir -p gpurun_out/dep2
timeout 900 python -m pytest tests -m gpu -q -k "deposit" -p no:cacheprovider > gpurun_out/dep2/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/dep2/pytest.log
for rep in 1 2; do timeout 300 python scripts/bench_deposit.py 2>>gpurun_out/dep2/err.log; done
for f in "" "--fused"; do timeout 300 python scripts/pic_cycle.py $f; done
