#!/bin/bash
# Profiling pass on one B200: rank-1 sync experiment, k=16 step kernel (configs[3]) under ncu --set full.
timeout 600 python scripts/exp_rank1.py > gpurun_out/exp_rank1.jsonl 2> gpurun_out/exp_rank1.err; echo "exp rc=$?"
CMD="python scripts/prof_step.py --workload gmrf5000 --k 16 --probes 16 --degree 12 --reps 1"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cheb_step_kernel -s 6 -c 1 \
  -o gpurun_out/k16_step $CMD > gpurun_out/ncu_k16.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/
