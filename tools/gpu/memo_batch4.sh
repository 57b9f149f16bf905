mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batch or c5 or strict or policy" > gpurun_out/gputest_mb.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest_mb.log
timeout 300 python tools/c5_probe.py > gpurun_out/c5_probe.json 2>&1; echo "probe rc=$?"; cat gpurun_out/c5_probe.json
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/c5_probe.py > gpurun_out/c5_ncu.log 2>&1; echo "ncu rc=$?"
