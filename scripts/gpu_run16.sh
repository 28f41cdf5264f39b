#!/bin/bash
run() { # name, env...
  local N=$1; shift
  env "$@" timeout 300 python scripts/prof_step.py --workload gmrf5000 --k 16 --probes 128 --reps 3 > gpurun_out/k16_$N.txt 2>&1; echo "$N rc=$?"; tail -1 gpurun_out/k16_$N.txt
}
run base
run cap6dec_st0 CHEB_LIB=build_variants/libchebld_cap6dec.so CHEB_SMALL_TILES=0
run cap6_st0 CHEB_LIB=build_variants/libchebld_cap6.so CHEB_SMALL_TILES=0
run base2
run cap6dec_st1 CHEB_LIB=build_variants/libchebld_cap6dec.so
