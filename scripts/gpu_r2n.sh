out=gpurun_out; mkdir -p $out
for v in default LBK_SEQROW_64 LBK_SEQROW_32; do
  if [ $v != default ]; then export LBK_LIB=$PWD/_variants/liblbk_$v.so; fi
  echo "== $v" >> $out/r2n.txt
  timeout 300 python scripts/prof_pl.py >> $out/r2n.txt 2>&1
done
unset LBK_LIB
timeout 300 python -m pytest tests/test_gpu_spmv.py -q -k "stream or powerlaw" >> $out/r2n.txt 2>&1
cat $out/r2n.txt
