#!/bin/bash
rm -f gpurun_out/parity.jsonl
PARITY_REPORT=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python scripts/exp_rank1.py > gpurun_out/exp_rank1.jsonl 2> gpurun_out/exp_rank1.err; echo "exp rc=$?"; cat gpurun_out/exp_rank1.jsonl
timeout 1200 python scripts/bench_extras.py f2 > gpurun_out/extras_f2.jsonl 2> gpurun_out/extras_f2.err; echo "extras rc=$?"; cat gpurun_out/extras_f2.jsonl
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for W in gmrf32 torus256 gmrf1000 btb4m; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline > gpurun_out/all_$W.json 2> gpurun_out/all_$W.err; echo "bench $W rc=$?"
done
