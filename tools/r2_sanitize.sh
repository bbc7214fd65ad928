# compute-sanitizer over tools/sanitize_driver.py (GPU box) -> gpurun_out/r2_san_*.log
for t in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 40 python tools/sanitize_driver.py > gpurun_out/r2_san_$t.log 2>&1
  tail -3 gpurun_out/r2_san_$t.log
done
