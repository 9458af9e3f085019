# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_small.py
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report analysis"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 python tools/sanitize_small.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|hazard" gpurun_out/sanitize_$tool.log | head -5
done
