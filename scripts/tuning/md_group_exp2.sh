# m-dipole branch grouping on the paper-replica workload (Table 2 analytic cells)
mkdir -p gpurun_out/mdg
L=paper_2104_04579_b200/tuning_libs
for rep in 1 2; do
for v in g1w g1a g2a g4a; do
  LIBBORIS_PATH=$L/libboris_$v.so timeout 600 python scripts/paper_table2.py --only analytic > gpurun_out/mdg/t2_${v}_$rep.txt 2>gpurun_out/mdg/err_$v.txt; echo $v rc=$?
done; done
