out=gpurun_out; mkdir -p $out
timeout 300 python scripts/ab_cg.py > $out/r2j.txt 2>&1
timeout 300 python scripts/phase_time.py >> $out/r2j.txt 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_XRED_STATS.so timeout 300 python scripts/xred_stats.py >> $out/r2j.txt 2>&1
M=gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread,smsp__inst_executed_op_shared_atom.sum,smsp__sass_inst_executed_op_local_ld.sum
timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/r2j_bicg.csv python scripts/prof_bicg.py > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/r2j_cg.csv python scripts/prof_k1.py > /dev/null 2>&1
cat $out/r2j.txt
