# compressed matrix copy: tests, then configs[3] bench A/B (CHEB_CV=0 vs default) and configs[2]
timeout 900 python -m pytest tests/test_compressed_gpu.py tests/test_parity_gpu.py -q -x -k "compressed or launch_count or timeout or moments_and_gamma" > gpurun_out/cv_t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/cv_t.log
for cv in 1 0 1 0; do CHEB_CV=$cv timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt --no-weak > gpurun_out/cv_b$cv.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/cv_b$cv.json').read().strip().splitlines()[-1]); r=d['roofline']
print('cv=$cv', round(d['value']), round(d['ms_per_step'],1), 'launch_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['power_w_median'])"; done
for cv in 1 0; do CHEB_CV=$cv timeout 600 python bench.py --workload gmrf1000 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt --no-weak > gpurun_out/cv_g$cv.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/cv_g$cv.json').read().strip().splitlines()[-1]); r=d['roofline']
print('gmrf1000 cv=$cv', round(d['value']), round(d['ms_per_step'],2), 'launch_ms', round(r['avg_launch_ms'],4), d['clocks']['sm_mhz'])"; done
