#!/bin/bash
# One B200 pass: GPU tests (full-m parity margins to gpurun_out/parity.jsonl), smoke, headline bench.
rm -f gpurun_out/parity.jsonl
PARITY_REPORT=gpurun_out/parity.jsonl timeout ${TEST_TIMEOUT:-2700} python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json
