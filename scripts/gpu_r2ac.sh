out=gpurun_out; mkdir -p $out; rm -f $out/r2ac.txt
timeout 300 python scripts/ab_cg.py >> $out/r2ac.txt 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 300 python scripts/ab_cg.py >> $out/r2ac.txt 2>&1
echo "== exact" >> $out/r2ac.txt; timeout 600 python scripts/scale_probe.py >> $out/r2ac.txt 2>&1
echo "== tree" >> $out/r2ac.txt; LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 600 python scripts/scale_probe.py >> $out/r2ac.txt 2>&1
cat $out/r2ac.txt
