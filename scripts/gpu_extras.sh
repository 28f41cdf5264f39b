timeout 900 python -m pytest tests/test_compressed_gpu.py tests/test_parity_gpu.py tests/test_resident_gpu.py -q -x > gpurun_out/t4.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t4.log
timeout 1500 python scripts/bench_extras.py f1 f2 f3 f4 > gpurun_out/extras.jsonl 2> gpurun_out/extras.err; echo "extras rc=$?"
cut -c1-250 gpurun_out/extras.jsonl | grep -v '"f1"'
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/ab_final.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/ab_final.json').read().strip().splitlines()[-1]); w=d['weak_scaling']
print('k16', round(d['ms_per_step'],1), 'k64', round(w['ms_per_step'],1), d['roofline']['matrix_format'][:10], d['clocks']['sm_mhz'])"
