# compute-sanitizer over tools/sanitize_driver.py (GPU box) -> gpurun_out/${1:-r2}_san_*.log
tag=${1:-r2}
for t in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 40 python tools/sanitize_driver.py > gpurun_out/${tag}_san_$t.log 2>&1
  tail -3 gpurun_out/${tag}_san_$t.log
done
