#!/bin/bash
timeout 1200 python scripts/bench_extras.py f2 > gpurun_out/extras_f2.jsonl 2> gpurun_out/extras_f2.err; echo "extras rc=$?"; cat gpurun_out/extras_f2.jsonl; tail -2 gpurun_out/extras_f2.err
timeout 600 python -m pytest tests -m gpu -q -x -k "family or likelihood" > gpurun_out/t_f2.log 2>&1; echo "pytest f2 rc=$?"; tail -2 gpurun_out/t_f2.log
for V in base dec dec3; do
  L=""; [ $V != base ] && L="CHEB_LIB=build_variants/libchebld_$V.so"
  for K in 16 64; do
    env $L timeout 300 python scripts/prof_step.py --workload gmrf5000 --k $K --probes 128 --reps 3 > gpurun_out/k${K}_$V.txt 2>&1; echo "$V k$K rc=$?"; tail -1 gpurun_out/k${K}_$V.txt
  done
done
CHEB_LIB=build_variants/libchebld_dec.so timeout 900 python -m pytest tests -m gpu -q -x -k "moments_and_gamma_small or full_m_parity and (gmrf1000 or gmrf32)" > gpurun_out/t_dec.log 2>&1; echo "pytest dec rc=$?"; tail -2 gpurun_out/t_dec.log
