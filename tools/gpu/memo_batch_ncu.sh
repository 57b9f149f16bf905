mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:rk_batch_memo_kernel -s 1 -c 1 -o /tmp/mb -f python tools/bench_c5.py > gpurun_out/mb_ncu.log 2>&1; echo "ncu rc=$?"
$NCU -i /tmp/mb.ncu-rep --page raw --csv > gpurun_out/mb_raw.csv 2>/dev/null
$NCU -i /tmp/mb.ncu-rep --page source --csv --print-source sass > gpurun_out/mb_source.csv 2>/dev/null
ls -la gpurun_out/mb_*
