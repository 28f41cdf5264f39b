#!/bin/bash
# New tests (f4 spectrum bounds, a7 triangular B, f1 accuracy, status, instantiations), f1 table,
# k = 16 tile experiments on configs[3].
timeout 1500 python -m pytest tests -m gpu -q -x -k "spectrum or triangular or accuracy or timeout or nonfinite or standard_geometry or dist_entry or launch_count or degrees_odd" > gpurun_out/t_new.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_new.log
timeout 900 python scripts/accuracy_51.py > gpurun_out/acc.jsonl 2> gpurun_out/acc.err; echo "acc rc=$?"
for V in base st0 s3; do
  E=""; L=""
  [ $V = st0 ] && E="CHEB_SMALL_TILES=0"
  [ $V = s3 ] && L="CHEB_LIB=build_variants/libchebld_s3.so"
  env $E $L timeout 300 python scripts/prof_step.py --workload gmrf5000 --k 16 --probes 128 --reps 4 > gpurun_out/k16_$V.txt 2>&1; echo "$V rc=$?"; tail -2 gpurun_out/k16_$V.txt
done
