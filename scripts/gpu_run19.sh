#!/bin/bash
for RG in 0 8 4 2; do
  CHEB_RG=$RG CHEB_DEBUG=1 timeout 600 python scripts/exp_rank1.py --cases torus256 > gpurun_out/exp_rg$RG.jsonl 2> gpurun_out/exp_rg$RG.err; echo "rg$RG rc=$?"; head -1 gpurun_out/exp_rg$RG.jsonl; sed -n 3p gpurun_out/exp_rg$RG.jsonl; grep "persistent grid" gpurun_out/exp_rg$RG.err | sort | uniq -c | head -2
done
