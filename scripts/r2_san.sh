# usage: bash scripts/r2_san.sh <tool>   (one compute-sanitizer tool per gpurun call)
tool=$1
timeout 300 python scripts/sanitize_cases.py > gpurun_out/san_plain_$tool.log 2>&1; rc=$?; echo plain rc=$rc
tail -3 gpurun_out/san_plain_$tool.log
if [ $rc -eq 0 ]; then
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo sanitizer rc=$?
  tail -8 gpurun_out/san_$tool.log
fi
