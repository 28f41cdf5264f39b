#!/bin/bash
# A/B of a library environment switch on one B200, interleaved:
#     VAR=CHEB_SERPENTINE CASES="gmrf1000:16 gmrf1000:64 gmrf5000:16" bash scripts/ab_env.sh
# prints the per-estimate times (ms, CUDA events) of the last 3 of 4 estimates per run.
mkdir -p gpurun_out
for c in ${CASES:-gmrf1000:16}; do
  w=${c%%:*}; k=${c##*:}
  for rep in 1 2; do for s in 0 1; do
    r=$(env $VAR=$s timeout 300 python scripts/prof_step.py --workload $w --k $k --reps 4 2>&1 | grep '^rep' | tail -3 | awk '{print $3}' | tr '\n' ' ')
    echo "$w k=$k $VAR=$s: $r"
  done; done
done 2>&1 | tee gpurun_out/ab_env_$VAR.txt
