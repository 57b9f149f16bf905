# r02 final evidence: gpu tests, smoke, bench (+ reference arm), shard projection, ncu launch list + full captures
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 300 python tools/bench_c5.py > gpurun_out/r02_c5_batch.json 2> gpurun_out/c5.err; echo "c5 rc=$?"
timeout 300 python tools/c5_probe.py > gpurun_out/c5_probe.json 2>&1; echo "c5 probe rc=$?"
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/c5_probe.py > gpurun_out/c5_ncu.log 2>&1; echo "c5 launches rc=$?"
python tools/shard_projection.py > gpurun_out/r02_shard_projection.json 2> gpurun_out/shard.err; echo "shard rc=$?"
$NCU --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-reduce-check > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
cap() { # name regex skip count
  $NCU --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 -o /tmp/full_$1 -f \
    python tools/memo_parts32.py > gpurun_out/ncu_full_$1.log 2>&1; echo "$1 rc=$?"
  $NCU -i /tmp/full_$1.ncu-rep --page raw --csv > gpurun_out/full_$1_raw.csv 2>/dev/null
}
cap keys32 rk_dp_keys32_kernel 2 1
cap suffix rk_dp_suffix_kernel 2 1
cap row24 rk_dp_row24_kernel 2 1
cap runs 'rk_dp_runs_kernel|rk_dp_parents_kernel|rk_dp_children_kernel' 6 3
cap ext rk_dp_ext_kernel 2 1
cap rows rk_dp_rows_kernel 2 1
cap levels rk_dp_level_kernel 24 8
$NCU --set full --clock-control none --import-source on -k regex:rk_batch_memo_kernel -s 1 -c 1 -o /tmp/full_mb -f python tools/bench_c5.py > gpurun_out/ncu_full_mb.log 2>&1; echo "memo batch rc=$?"
$NCU -i /tmp/full_mb.ncu-rep --page raw --csv > gpurun_out/full_memo_batch_raw.csv 2>/dev/null
du -sh gpurun_out
