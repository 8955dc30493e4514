mkdir -p gpurun_out/md
for lib in "" paper_2104_04579_b200/tuning_libs/libboris_mdg1.so; do
  tag=${lib:+mdg1}; tag=${tag:-group4}
  LIBBORIS_PATH=$lib timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/md/variants_$tag.jsonl 2>gpurun_out/md/variants_$tag.err; echo variants $tag rc=$?
  LIBBORIS_PATH=$lib timeout 600 python scripts/bench_variants.py --mdipole-only > gpurun_out/md/variants2_$tag.jsonl 2>>gpurun_out/md/variants_$tag.err; echo variants2 $tag rc=$?
done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/md/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/md/pytest.log
timeout 900 python scripts/paper_table2.py > gpurun_out/md/table2.txt 2>gpurun_out/md/table2.err; echo table2 rc=$?
