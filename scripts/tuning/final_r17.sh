# round-end style check on the current tree: smoke, full GPU suite, default bench,
# reference arm, launch list, ncu full of the bench kernel, all sanitizers, PIC cycle, deposit
mkdir -p gpurun_out/r17
bash scripts/gpu_check.sh > gpurun_out/r17/gpu_check.log 2>&1; echo gpu_check rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r17/bench_ref.json 2>gpurun_out/r17/bench_ref.err; echo ref rc=$?
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/r17/sanitize_$tool.log 2>&1; echo sanitize $tool rc=$?
done
timeout 600 python scripts/pic_cycle.py --fused > gpurun_out/r17/pic_fused.jsonl 2>gpurun_out/r17/pic.err; echo pic rc=$?
timeout 600 python scripts/bench_deposit.py > gpurun_out/r17/deposit.jsonl 2>>gpurun_out/r17/pic.err; echo deposit rc=$?
