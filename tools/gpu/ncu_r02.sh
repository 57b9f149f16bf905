# round-2 ncu evidence: launch list of the bench step + full captures of the step's kernels
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
for k in rk_dp_keys_kernel rk_dp_suffix_kernel rk_dp_meta_kernel rk_dp_rows_kernel rk_dp_insert_kernel; do
  $NCU --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/full_$k -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$k.log 2>&1; echo "$k rc=$?"
done
$NCU --set full --clock-control none --import-source on -k regex:rk_dp_level_kernel -s 21 -c 7 -o gpurun_out/full_levels -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_levels.log 2>&1; echo "levels rc=$?"
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tools/sanitize_smoke.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"
RK_FORCE_MEMO=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tools/sanitize_smoke.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"
RK_FORCE_MEMO=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python tools/sanitize_smoke.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"
tail -3 gpurun_out/san_*.log
