mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/gputest.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_v.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_v.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['fresh_sets'])"
RK_NO_MEMO=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-reduce-check > gpurun_out/bench_direct.log 2>&1; echo "direct rc=$?"
grep '^{' gpurun_out/bench_direct.log | cut -c1-260
timeout 300 python tools/c5_probe.py > gpurun_out/c5_probe2.json 2>&1; echo "c5 probe rc=$?"; cat gpurun_out/c5_probe2.json
