mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
$CS --version > gpurun_out/san_version.log 2>&1; echo "version rc=$?"; head -5 gpurun_out/san_version.log
for tool in memcheck racecheck synccheck; do
  RK_FORCE_MEMO=1 timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_smoke.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; head -c 1500 gpurun_out/san_$tool.log; echo; tail -c 800 gpurun_out/san_$tool.log
done
