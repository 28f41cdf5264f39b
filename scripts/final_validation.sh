#!/bin/bash
# Round-end validation on one B200: GPU tests, smoke, headline bench, all configs, ncu evidence.
# Large .ncu-rep files are summarised on the box and removed (gpurun copies back <= 64 MiB).
SKIP_TESTS=${SKIP_TESTS:-0}
if [ "$SKIP_TESTS" = 0 ]; then
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/t_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
bash scripts/bench_all.sh; echo "bench_all done"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 420 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
for V in step dbl; do
  E=""; [ $V = dbl ] && E="CHEB_DOUBLING=1"
  env $E timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cheb_step_kernel" -s 10 -c 1 -o /tmp/full_$V python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 1 > /dev/null 2>&1; echo "full $V rc=$?"
  python scripts/ncu_brief.py /tmp/full_$V.ncu-rep > gpurun_out/full_${V}_brief.txt 2>&1
  python scripts/ncu_summary.py /tmp/full_$V.ncu-rep >> gpurun_out/full_${V}_brief.txt 2>&1
done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"cheb_step_kernel" -s 10 -c 3 --csv python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 1 > gpurun_out/traffic.csv 2>/dev/null; echo "traffic rc=$?"
du -sh gpurun_out
