#!/bin/bash
for V in base r1c4; do
  L=""; [ $V = r1c4 ] && L="CHEB_LIB=build_variants/libchebld_r1c4.so"
  env $L CHEB_DEBUG=1 timeout 600 python scripts/exp_rank1.py --cases torus256 > gpurun_out/exp_$V.jsonl 2> gpurun_out/exp_$V.err; echo "$V rc=$?"; cat gpurun_out/exp_$V.jsonl; grep "persistent grid" gpurun_out/exp_$V.err | sort | uniq -c
done
