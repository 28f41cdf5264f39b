#!/bin/bash
# bench.py on every BASELINE config, Algorithm 1 and moment doubling (one B200).
for W in ${WORKLOADS:-gmrf32 torus256 gmrf1000 gmrf5000 btb4m}; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline > gpurun_out/all_${W}.json 2> gpurun_out/all_${W}.err
  timeout 600 python bench.py --workload $W --doubling --no-cpu-baseline --no-alt --no-e2e > gpurun_out/all_${W}_dbl.json 2> gpurun_out/all_${W}_dbl.err
done
