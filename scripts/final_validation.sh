#!/bin/bash
# Round-end validation on one B200: GPU tests (full-m parity margins), smoke, headline bench, all
# configs, f rows, ncu launch list of the headline bench.  Writes gpurun_out/*.
rm -f gpurun_out/parity.jsonl
SKIP_TESTS=${SKIP_TESTS:-0}
if [ "$SKIP_TESTS" = 0 ]; then
PARITY_REPORT=gpurun_out/parity.jsonl timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/t_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/t_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
for W in gmrf32 torus256 gmrf1000 btb4m; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline > gpurun_out/all_$W.json 2> gpurun_out/all_$W.err; echo "bench $W rc=$?"
done
timeout 600 python bench.py --doubling --no-cpu-baseline --no-e2e > gpurun_out/all_gmrf5000_dbl.json 2> gpurun_out/all_gmrf5000_dbl.err; echo "bench dbl rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-alt --no-weak"
timeout 600 $B > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
S="python scripts/prof_step.py --workload gmrf5000 --k 16 --probes 16 --degree 12 --reps 1"
timeout 300 $S > gpurun_out/plain_k16.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cheb_step_kernel -s 6 -c 1 -o /tmp/k16_full $S > gpurun_out/ncu_k16.log 2>&1; echo "k16 full rc=$?"
python scripts/ncu_summary.py /tmp/k16_full.ncu-rep > gpurun_out/k16_summary.txt 2>&1
# the resident kernel at configs[1] (k = 16): ncu cannot replay a cooperative launch, so this capture
# launches the same grid without the cooperative attribute (CHEB_RES_NOCOOP=1, co-resident anyway)
R="python scripts/prof_res.py torus256 16"
CHEB_RES_NOCOOP=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:cheb_resident_kernel -c 1 -o /tmp/res16 $R > gpurun_out/ncu_res16.log 2>&1; echo "resident ncu rc=$?"
python scripts/ncu_summary.py /tmp/res16.ncu-rep > gpurun_out/res16_summary.txt 2>&1
ncu -i /tmp/res16.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/res16_sass.csv.gz
ncu -i /tmp/k16_full.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/k16_sass.csv.gz
du -sh gpurun_out
