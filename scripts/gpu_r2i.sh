out=gpurun_out; mkdir -p $out
M=gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread,smsp__inst_executed_op_shared_atom.sum,smsp__sass_inst_executed_op_local_ld.sum
timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/r2i_exact.csv python scripts/prof_bicg.py > /dev/null 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/r2i_tree.csv python scripts/prof_bicg.py > /dev/null 2>&1
