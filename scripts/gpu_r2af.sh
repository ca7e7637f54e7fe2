out=gpurun_out; mkdir -p $out; rm -f $out/r2af.txt
timeout 300 python scripts/ab_cg.py >> $out/r2af.txt 2>&1
for v in LBK_CSR_WARPS_3_LBK_CSR_SLOTS_3 LBK_CSR_CAP_896_LBK_CSR_SLOTS_3_LBK_CSR_WARPS_3; do
  LBK_LIB=$PWD/_variants/liblbk_$v.so timeout 300 python scripts/ab_cg.py >> $out/r2af.txt 2>&1
done
cat $out/r2af.txt
