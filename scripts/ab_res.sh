#!/bin/bash
# A/B of resident-kernel tuning builds (scripts/build_variants.py) against the in-tree library:
# configs[1] (torus256 + rank-1, k = 16) timings interleaved, Algorithm 1 and moment doubling;
# configs[0]; the resident parity tests on every variant; per-phase cycle counts (resprof builds).
#     VARIANTS="rest640" PROF_VARIANTS="resprof" bash scripts/ab_res.sh
mkdir -p gpurun_out
VARIANTS=${VARIANTS:-""}
VARIANTS="$VARIANTS" WORKLOAD=torus256 K=16 bash scripts/ab_variants.sh 2>&1 | tee gpurun_out/ab_res.txt
for v in default $VARIANTS; do
  if [ "$v" = default ]; then unset CHEB_LIB; else export CHEB_LIB=build_variants/libchebld_$v.so; fi
  echo "== $v"
  timeout 600 python scripts/exp_resident.py --cases torus256,gmrf32 --ks 16,64 --scheds resident --doubling 2>&1 | grep '^{' | cut -c1-220
done 2>&1 | tee gpurun_out/ab_res_cases.txt
for v in $VARIANTS; do
  CHEB_LIB=build_variants/libchebld_$v.so timeout 900 python -m pytest tests/test_resident_gpu.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/ab_res_test_$v.txt
done
unset CHEB_LIB
for v in ${PROF_VARIANTS:-}; do
  CHEB_LIB=build_variants/libchebld_$v.so timeout 300 python scripts/res_phases.py torus256 16 2>&1 | tee gpurun_out/ab_res_phases_$v.json
done
