#!/bin/bash
CHEB_DEBUG=1 timeout 600 python scripts/exp_rank1.py > gpurun_out/exp_rank1.jsonl 2> gpurun_out/exp_rank1.err; echo "exp rc=$?"; cat gpurun_out/exp_rank1.jsonl; grep "persistent grid" gpurun_out/exp_rank1.err | sort | uniq -c
for V in base narrow; do
  L=""; [ $V != base ] && L="CHEB_LIB=build_variants/libchebld_$V.so"
  for K in 16 64; do
    env $L timeout 300 python scripts/prof_step.py --workload gmrf5000 --k $K --probes 128 --reps 3 > gpurun_out/k${K}_$V.txt 2>&1; echo "$V k$K rc=$?"; tail -1 gpurun_out/k${K}_$V.txt
  done
done
rm -f gpurun_out/parity.jsonl
PARITY_REPORT=gpurun_out/parity.jsonl timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_gpu.log
