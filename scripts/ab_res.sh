#!/bin/bash
# A/B of resident-kernel tuning builds at configs[1] (torus256 + rank-1, k = 16): timings interleaved
# with the in-tree library, the resident parity tests on every variant, per-phase cycle counts.
mkdir -p gpurun_out
VARIANTS=${VARIANTS:-""}
VARIANTS="$VARIANTS" WORKLOAD=torus256 K=16 bash scripts/ab_variants.sh > gpurun_out/ab_res.txt 2>&1
for v in $VARIANTS; do
  CHEB_LIB=build_variants/libchebld_$v.so timeout 900 python -m pytest tests/test_resident_gpu.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/ab_res_test_$v.txt
done
for v in ${PROF_VARIANTS:-resprof}; do
  CHEB_LIB=build_variants/libchebld_$v.so timeout 300 python scripts/res_phases.py torus256 16 > gpurun_out/ab_res_phases_$v.json 2>&1
done
cat gpurun_out/ab_res.txt; tail -n 2 gpurun_out/ab_res_test_*.txt; cat gpurun_out/ab_res_phases_*.json
