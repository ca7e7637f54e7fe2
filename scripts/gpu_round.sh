#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture.
# Usage (under gpurun): bash scripts/gpu_round.sh [tag]
tag=${1:-r}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/${tag}_smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> $out/${tag}_smoke.log
timeout 600 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc=$?" >> $out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $out/${tag}_bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/${tag}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-formats > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_stream -s 5 -c 1 -o $out/${tag}_csr python bench.py --steps 8 --warmup 3 --no-cg --no-cpu --no-formats > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'csr_stream|vec_kernel' -o $out/${tag}_cg python scripts/prof_k1.py > /dev/null 2>&1
# summarise on the box (the .ncu-rep captures exceed gpurun's 64 MiB return limit)
python scripts/summarize_profiles.py $tag ${ROUND:-1} $out/${tag}_profiles > $out/${tag}_summarize.log 2>&1
rm -f $out/*.ncu-rep
tail -3 $out/${tag}_pytest_gpu.log; tail -2 $out/${tag}_smoke.log; cat $out/${tag}_bench.json; tail -2 $out/${tag}_bench.err; cat $out/${tag}_bench_ref.json | tail -1
