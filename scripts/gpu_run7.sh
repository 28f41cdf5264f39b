#!/bin/bash
rm -f gpurun_out/parity.jsonl
CHEB_DEBUG=1 timeout 600 python scripts/exp_rank1.py > gpurun_out/exp_rank1.jsonl 2> gpurun_out/exp_rank1.err; echo "exp rc=$?"; cat gpurun_out/exp_rank1.jsonl
for V in base c3; do
  L=""; [ $V = c3 ] && L="CHEB_LIB=build_variants/libchebld_c3.so"
  env $L timeout 300 python scripts/prof_step.py --workload gmrf5000 --k 16 --probes 128 --reps 4 > gpurun_out/k16_$V.txt 2>&1; echo "$V rc=$?"; tail -1 gpurun_out/k16_$V.txt
done
PARITY_REPORT=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench.json
timeout 900 python bench.py --workload torus256 --no-cpu-baseline > gpurun_out/bench_torus.json 2> gpurun_out/bench_torus.err; echo "bench torus rc=$?"
