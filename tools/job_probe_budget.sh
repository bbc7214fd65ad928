cd $GRAFT_REPO_ROOT
for b in 24 26 28 24 26 28 22; do
  echo "$b $(RT_PROBE_BUDGET=$b timeout 300 python tools/eye_probe.py --reps 15)"
done > gpurun_out/s48_budget.log 2>&1
