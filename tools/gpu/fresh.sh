mkdir -p gpurun_out
COMPACT=1 timeout 300 python tools/fresh_probe.py > gpurun_out/fresh_compact.json 2>&1; echo "compact rc=$?"
for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_f$i.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_f$i.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['fresh_sets'])"; done
