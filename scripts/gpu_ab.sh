# A/B: step kernels with / without the compressed-copy path (build_variants/libchebld_nocv.so)
for rep in 1 2; do for v in default nocv; do
  if [ $v = nocv ]; then export CHEB_LIB=build_variants/libchebld_nocv.so; else unset CHEB_LIB; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); w=d['weak_scaling']
print('$v', 'k16', round(d['ms_per_step'],1), 'k64', round(w['ms_per_step'],1), d['roofline']['matrix_format'][:10], d['clocks']['sm_mhz'])"
done; done
unset CHEB_LIB
timeout 900 python scripts/bench_extras.py f2 2>/dev/null | cut -c1-300
