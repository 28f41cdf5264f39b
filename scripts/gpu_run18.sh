#!/bin/bash
for V in base diag_r1nosync diag_r1nosync_c4; do
  L=""; [ $V != base ] && L="CHEB_LIB=build_variants/libchebld_$V.so"
  env $L CHEB_DEBUG=1 timeout 600 python scripts/exp_rank1.py --cases torus256 > gpurun_out/exp_$V.jsonl 2> gpurun_out/exp_$V.err; echo "$V rc=$?"; head -1 gpurun_out/exp_$V.jsonl; grep "persistent grid" gpurun_out/exp_$V.err | sort | uniq -c | head -2
done
