# r02 ncu evidence after the pass-1 restructure: launch list of the bench step + full captures
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-reduce-check > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
cap() { # name regex skip count
  $NCU --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 -o /tmp/full_$1 -f \
    python tools/memo_step.py > gpurun_out/ncu_full_$1.log 2>&1; echo "$1 rc=$?"
  $NCU -i /tmp/full_$1.ncu-rep --page raw --csv > gpurun_out/full_$1_raw.csv 2>/dev/null
  $NCU -i /tmp/full_$1.ncu-rep --page source --csv > gpurun_out/full_$1_source.csv 2>/dev/null
}
cap keys rk_dp_keys_kernel 3 1
cap suffix rk_dp_suffix_kernel 3 1
cap row24 rk_dp_row24_kernel 3 1
cap runs rk_dp_runs_kernel 3 1
cap meta rk_dp_meta_kernel 3 1
cap rows rk_dp_rows_kernel 3 1
cap levels rk_dp_level_kernel 32 8
du -sh gpurun_out
