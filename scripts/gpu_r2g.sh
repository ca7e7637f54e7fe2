out=gpurun_out; mkdir -p $out
timeout 300 python scripts/ab_cg.py > $out/r2g_ab.txt 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 300 python scripts/ab_cg.py >> $out/r2g_ab.txt 2>&1
M=gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread
timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/r2g_exact.csv python scripts/prof_k1.py > /dev/null 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/r2g_tree.csv python scripts/prof_k1.py > /dev/null 2>&1
cat $out/r2g_ab.txt
