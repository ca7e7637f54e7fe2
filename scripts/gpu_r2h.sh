out=gpurun_out; mkdir -p $out
timeout 300 python scripts/phase_time.py > $out/r2h.txt 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 300 python scripts/phase_time.py >> $out/r2h.txt 2>&1
cat $out/r2h.txt
