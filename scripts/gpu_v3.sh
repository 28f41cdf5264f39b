# full GPU tests, headline bench, ncu traffic + full capture of the k=16 step kernel (compressed copy)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/v3_tgpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/v3_tgpu.log; grep FAILED gpurun_out/v3_tgpu.log | head
timeout 900 python bench.py > gpurun_out/v3_bench.json 2> gpurun_out/v3_bench.err; echo "bench rc=$?"
S="python scripts/prof_step.py --workload gmrf5000 --k 16 --probes 16 --degree 12 --reps 1"
timeout 300 $S > gpurun_out/v3_plain_k16.log 2>&1 && \
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:cheb_step_kernel -s 4 -c 4 --csv $S > gpurun_out/v3_traffic_k16.csv 2>/dev/null; echo "traffic rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cheb_step_kernel -s 6 -c 1 -o /tmp/k16cv $S > gpurun_out/v3_ncu_k16.log 2>&1; echo "k16 full rc=$?"
python scripts/ncu_summary.py /tmp/k16cv.ncu-rep > gpurun_out/v3_k16cv_summary.txt 2>&1
ncu -i /tmp/k16cv.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/v3_k16cv_sass.csv.gz
