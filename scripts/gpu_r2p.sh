out=gpurun_out; mkdir -p $out
for v in LBK_PIPE_TEST_1 LBK_SEQROW_64; do
  export LBK_LIB=$PWD/_variants/liblbk_$v.so
  echo "== $v" >> $out/r2p.txt
  timeout 300 python scripts/prof_pl.py >> $out/r2p.txt 2>&1
done
cat $out/r2p.txt
