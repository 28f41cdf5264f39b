# resident kernel: parity tests, then per-estimate times of the schedules (Algorithm 1 and doubling)
timeout 900 python -m pytest tests/test_resident_gpu.py tests/test_doubling_gpu.py -q -x > gpurun_out/res_t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/res_t.log
python scripts/exp_resident.py --cases torus256,gmrf32 --ks 16,32 --scheds resident,persistent 2>&1 | cut -c1-150
CHEB_DOUBLING=1 python scripts/exp_resident.py --cases torus256,gmrf32 --ks 16,32 --scheds resident,persistent 2>&1 | cut -c1-150
