out=gpurun_out; mkdir -p $out
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_op_shared_atom.sum
for lib in ${LIBS:-default tree}; do
  if [ $lib = tree ]; then export LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:"csr_stream|vec_kernel" -s 900 -c 6 --csv --log-file $out/r2k_cg_$lib.csv python scripts/prof_late.py cg 305 > /dev/null 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:"csr_stream|vec_kernel" -s 1500 -c 10 --csv --log-file $out/r2k_bi_$lib.csv python scripts/prof_late.py bicgstab 305 > /dev/null 2>&1
done
