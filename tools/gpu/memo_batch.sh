# memoised C5 batch: new parity tests, the C5 suite, C5 timing memo vs direct
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batch or c5" > gpurun_out/gputest_mb.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputest_mb.log
timeout 300 python tools/bench_c5.py > gpurun_out/c5_memo.json 2>&1; echo "c5 rc=$?"; cut -c1-220 gpurun_out/c5_memo.json
RK_NO_MEMO=1 timeout 300 python tools/bench_c5.py > gpurun_out/c5_direct.json 2>&1; echo "c5 direct rc=$?"; cut -c1-220 gpurun_out/c5_direct.json
