#!/bin/bash
# A/B of tuning builds (scripts/build_variants.py -> build_variants/libchebld_<name>.so) against the
# in-tree library on one B200, interleaved so clock / power-cap drift hits every variant alike:
#     VARIANTS="s3 sus1k" WORKLOAD=gmrf5000 K=16 bash scripts/ab_variants.sh
# prints the per-estimate times (ms, CUDA events) of the last 3 of 4 estimates per run.
for rep in 1 2; do for v in default ${VARIANTS}; do
  if [ "$v" = default ]; then unset CHEB_LIB; else export CHEB_LIB=build_variants/libchebld_$v.so; fi
  r=$(timeout 300 python scripts/prof_step.py --workload ${WORKLOAD:-gmrf5000} --k ${K:-16} --reps 4 2>&1 \
      | grep '^rep' | tail -3 | awk '{print $3}' | tr '\n' ' ')
  echo "$v: $r"
done; done
