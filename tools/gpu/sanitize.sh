# one compute-sanitizer tool per gpurun call (B200_PROFILING.md); TOOL=racecheck|synccheck|memcheck
set -x
mkdir -p gpurun_out/r2
T=${TOOL:-racecheck}
for spec in "fwd 16 16 32" "dgrad 16 16 32" "wgrad 16 16 40" "fwd 64 64 12" "wgrad 64 64 12" "fwd 32 32 34" "wgrad 32 32 34"; do
  timeout 600 compute-sanitizer --tool $T --print-limit 20 python tools/conv_one.py $spec 1 >> gpurun_out/r2/sanitize_$T.log 2>&1
  echo "$spec rc=$?" >> gpurun_out/r2/sanitize_$T.log
done
grep -E "rc=|ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/r2/sanitize_$T.log | tail -30
