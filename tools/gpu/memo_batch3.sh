mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/gputest.log
timeout 300 python tools/c5_probe.py > gpurun_out/c5_probe.json 2>&1; echo "probe rc=$?"; cat gpurun_out/c5_probe.json
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/c5_probe.py > gpurun_out/c5_ncu.log 2>&1; echo "ncu rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_v.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_v.log | cut -c1-300
RK_NO_MEMO=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-reduce-check > gpurun_out/bench_direct.log 2>&1; echo "direct rc=$?"
grep '^{' gpurun_out/bench_direct.log | cut -c1-300
