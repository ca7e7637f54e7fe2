out=gpurun_out; mkdir -p $out; rm -f $out/r2s.txt
for v in LBK_CSR_CAP_512_LBK_CSR_MINB_4_LBK_NO_FASTPATH LBK_CSR_CAP_512_LBK_CSR_MINB_4 LBK_NO_FASTPATH; do
  export LBK_LIB=$PWD/_variants/liblbk_$v.so
  echo "== $v" >> $out/r2s.txt
  timeout 300 python scripts/prof_pl.py csr >> $out/r2s.txt 2>&1
done
cat $out/r2s.txt
