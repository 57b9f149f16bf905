for o in 0 1; do echo "overlap=$o $(RK_OVERLAP=$o python tools/memo_parts32.py 2>&1 | tail -2 | tr '\n' ' ')"; done
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:rk_dp_keys32_kernel -s 2 -c 1 -o /tmp/full_keys32 -f python tools/memo_parts32.py > /dev/null 2>&1; echo "ncu rc=$?"
$NCU -i /tmp/full_keys32.ncu-rep --page raw --csv > gpurun_out/full_keys32_raw.csv 2>/dev/null
$NCU -i /tmp/full_keys32.ncu-rep --page source --csv > gpurun_out/full_keys32_source.csv 2>/dev/null
python -m pytest tests/test_gpu_parity.py -x -q -k "compact" 2>&1 | tail -2
