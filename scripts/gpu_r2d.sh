out=gpurun_out; mkdir -p $out
M=gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread,smsp__inst_executed_op_shared_atom.sum,smsp__inst_executed_op_global_red.sum,dram__bytes_read.sum,smsp__sass_inst_executed_op_local_ld.sum
timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/r2d_exact.csv python scripts/prof_k1.py > /dev/null 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/r2d_tree.csv python scripts/prof_k1.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_stream -s 3 -c 2 -o $out/r2d_cg python scripts/prof_k1.py > /dev/null 2>&1
ncu -i $out/r2d_cg.ncu-rep --page details > $out/r2d_cg_details.txt 2>&1
ncu -i $out/r2d_cg.ncu-rep --page source --csv > $out/r2d_cg_source.csv 2>&1
rm -f $out/*.ncu-rep
ls -la $out/r2d*
