# cfg3 power-law: one full ncu capture per format, summarised into profiles/
out=gpurun_out; mkdir -p $out/r2ak_profiles
cp profiles/ncu_summary.json $out/r2ak_profiles/ 2>/dev/null
for w in csr coo f32; do
  k=csr_stream; [ $w = coo ] && k=coo_stream
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $out/r2ak_pl_$w python scripts/prof_pl.py $w > $out/r2ak_pl_$w.log 2>&1
done
python scripts/summarize_profiles.py r2ak 2 $out/r2ak_profiles --cfg3-only > $out/r2ak_summarize.log 2>&1
for w in csr coo f32; do ncu -i $out/r2ak_pl_$w.ncu-rep --page details > $out/r2ak_pl_${w}_details.txt 2>&1; done
rm -f $out/*.ncu-rep
cat $out/r2ak_summarize.log; cat $out/r2ak_profiles/r2_cfg3_ncu.txt
