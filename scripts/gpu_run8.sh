#!/bin/bash
CHEB_DEBUG=1 timeout 600 python scripts/exp_rank1.py --cases torus256 > gpurun_out/exp_rank1.jsonl 2> gpurun_out/exp_rank1.err; echo "exp rc=$?"; cat gpurun_out/exp_rank1.jsonl; grep "persistent grid" gpurun_out/exp_rank1.err | sort | uniq -c
timeout 1500 python -m pytest tests -m gpu -q -k "persistent or torus or rank1 or graph or shard or standard_geometry" > gpurun_out/t_sel.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_sel.log
