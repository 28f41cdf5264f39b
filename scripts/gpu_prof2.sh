#!/bin/bash
# ncu evidence: headline bench launch list; persistent rank-1 kernel at configs[1]; k = 16 step kernel traffic.
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-alt --no-weak"
timeout 600 $B > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
T="python scripts/prof_step.py --workload torus256 --k 32 --reps 1"
timeout 300 $T > gpurun_out/plain_torus.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cheb_persist_kernel -c 1 -o gpurun_out/persist_torus $T > gpurun_out/ncu_torus.log 2>&1; echo "torus ncu rc=$?"
S="python scripts/prof_step.py --workload gmrf5000 --k 16 --probes 16 --degree 12 --reps 1"
timeout 300 $S > gpurun_out/plain_k16.log 2>&1 && \
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:cheb_step_kernel -s 4 -c 4 --csv $S > gpurun_out/traffic_k16.csv 2>/dev/null; echo "traffic rc=$?"
ls -la gpurun_out | tail -8
