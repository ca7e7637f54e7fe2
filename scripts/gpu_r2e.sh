out=gpurun_out; mkdir -p $out
timeout 300 python scripts/ab_cg.py > $out/r2e_ab.txt 2>&1
M=gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread,smsp__inst_executed_op_shared_atom.sum,dram__bytes_read.sum,smsp__sass_inst_executed_op_local_ld.sum,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/r2e_exact.csv python scripts/prof_k1.py > /dev/null 2>&1
cat $out/r2e_ab.txt
