out=gpurun_out; mkdir -p $out
M=gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size,launch__registers_per_thread
timeout 600 ncu --metrics $M --clock-control none -k regex:"csr_stream|vec_kernel|finish|peer|dist" -s 400 -c 40 --csv --log-file $out/r2w_exact.csv python scripts/scale_probe.py 8 60 > /dev/null 2>&1

