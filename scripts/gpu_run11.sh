#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -k "family or quadform or likelihood or launch_count or abi or degenerate" > gpurun_out/t_f2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_f2.log
timeout 1200 python scripts/bench_extras.py f2 f3 f4 > gpurun_out/extras.jsonl 2> gpurun_out/extras.err; echo "extras rc=$?"; cat gpurun_out/extras.jsonl; tail -3 gpurun_out/extras.err
T="python scripts/prof_step.py --workload torus256 --k 32 --reps 1"
timeout 300 $T > gpurun_out/plain_torus.log 2>&1 && \
timeout 900 ncu --replay-mode application --set full --import-source on --clock-control none -k regex:cheb_persist_kernel -c 1 -o gpurun_out/persist_torus $T > gpurun_out/ncu_torus.log 2>&1; echo "torus ncu rc=$?"; tail -3 gpurun_out/ncu_torus.log
