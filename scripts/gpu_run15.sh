#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x -k "family or likelihood or quadform" > gpurun_out/t_f2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_f2.log
timeout 2400 python scripts/bench_extras.py f1 f2 f3 f4 > gpurun_out/extras.jsonl 2> gpurun_out/extras.err; echo "extras rc=$?"; cat gpurun_out/extras.jsonl; tail -3 gpurun_out/extras.err
