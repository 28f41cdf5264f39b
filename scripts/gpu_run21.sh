#!/bin/bash
for V in base wide16; do
  L=""; [ $V != base ] && L="CHEB_LIB=build_variants/libchebld_$V.so"
  for K in 32 16; do
    env $L timeout 300 python scripts/prof_step.py --workload gmrf5000 --k $K --probes 128 --reps 3 > gpurun_out/k${K}_$V.txt 2>&1; echo "$V k$K rc=$?"; tail -1 gpurun_out/k${K}_$V.txt
  done
  env $L timeout 300 python scripts/prof_step.py --workload gmrf1000 --k 32 --probes 64 --reps 3 > gpurun_out/g1k_k32_$V.txt 2>&1; echo "$V gmrf1000 k32 rc=$?"; tail -1 gpurun_out/g1k_k32_$V.txt
done
timeout 2700 python -m pytest tests -m gpu -q -k "not slow" > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_gpu.log
