#!/bin/bash
rm -f gpurun_out/parity.jsonl
timeout 600 python scripts/exp_rank1.py > gpurun_out/exp_rank1.jsonl 2> gpurun_out/exp_rank1.err; echo "exp rc=$?"; cat gpurun_out/exp_rank1.jsonl
PARITY_REPORT=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/t_gpu.log
timeout 900 python scripts/accuracy_51.py > gpurun_out/acc.jsonl 2> gpurun_out/acc.err; echo "acc rc=$?"; tail -3 gpurun_out/acc.err
