out=gpurun_out; mkdir -p $out; rm -f $out/r2an.txt
for lib in "" _variants/*.so; do
  if [ -n "$lib" ]; then export LBK_LIB=$PWD/$lib; else unset LBK_LIB; fi
  echo "lib=${lib:-default}" >> $out/r2an.txt
  timeout 300 python scripts/ab_spmv.py >> $out/r2an.txt 2>&1
  timeout 300 python scripts/prof_pl.py coo >> $out/r2an.txt 2>&1
done
cat $out/r2an.txt
