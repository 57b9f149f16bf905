# after moving strict RR out of line: gpu tests, C4 bench, C5 batch, direct-kernel C4 step
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/gputest.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_v.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_v.log | cut -c1-300
python tools/bench_c5.py > gpurun_out/c5_v.json 2>&1; echo "c5 rc=$?"; cut -c1-200 gpurun_out/c5_v.json
RK_NO_MEMO=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-reduce-check > gpurun_out/bench_direct.log 2>&1; echo "direct rc=$?"
grep '^{' gpurun_out/bench_direct.log | cut -c1-300
