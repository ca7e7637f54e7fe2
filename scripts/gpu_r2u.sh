out=gpurun_out; mkdir -p $out; rm -f $out/r2u.txt
echo "== exact" >> $out/r2u.txt; timeout 600 python scripts/scale_probe.py >> $out/r2u.txt 2>&1
echo "== tree" >> $out/r2u.txt; LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 600 python scripts/scale_probe.py >> $out/r2u.txt 2>&1
cat $out/r2u.txt
