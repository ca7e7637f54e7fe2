out=gpurun_out; mkdir -p $out; rm -f $out/r2ag.txt
for v in default LBK_GATHER_NOALLOC LBK_GATHER_CG; do
  if [ $v != default ]; then export LBK_LIB=$PWD/_variants/liblbk_$v.so; fi
  echo "== $v" >> $out/r2ag.txt
  timeout 300 python scripts/prof_pl.py csr >> $out/r2ag.txt 2>&1
  timeout 300 python scripts/ab_spmv.py >> $out/r2ag.txt 2>&1
done
cat $out/r2ag.txt
