#!/bin/bash
for V in base fam4; do
  L=""; [ $V != base ] && L="CHEB_LIB=build_variants/libchebld_$V.so"
  env $L timeout 1200 python scripts/bench_extras.py f2 > gpurun_out/extras_f2_$V.jsonl 2> gpurun_out/extras_f2_$V.err; echo "f2 $V rc=$?"; cat gpurun_out/extras_f2_$V.jsonl
done
for K in 16 64; do
  timeout 300 python scripts/prof_step.py --workload gmrf5000 --k $K --probes 128 --reps 3 > gpurun_out/k${K}_now.txt 2>&1; echo "k$K rc=$?"; tail -1 gpurun_out/k${K}_now.txt
done
timeout 1500 python -m pytest tests -m gpu -q -x -k "not full_m and not slow" > gpurun_out/t_q.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_q.log
