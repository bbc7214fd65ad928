#!/bin/bash
# Round-2 session-2 final job (one GPU box): ncu captures (tools/r2_profile.sh), then the bench
# lines of every config + the reference arm (tools/job_r2_bench.sh), then the GPU test suite
# and smoke().
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 bash tools/r2_profile.sh > gpurun_out/r2d_profile.log 2>&1
bash tools/job_r2_bench.sh r2d
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2d_pytest.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1
echo done
