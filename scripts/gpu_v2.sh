timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/v2_tgpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/v2_tgpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2_smoke.log 2>&1; echo "smoke rc=$?"
for W in gmrf32 torus256; do timeout 600 python bench.py --workload $W --no-cpu-baseline > gpurun_out/v2_$W.json 2> gpurun_out/v2_$W.err; echo "bench $W rc=$?"; done
