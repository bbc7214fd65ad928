#!/bin/bash
# Round-2 session-3 final job (one GPU box): the bench lines of every config + the reference
# arm (tools/job_r2_bench.sh) after the native render_frame readback and the asynchronous
# mesh validation, then the GPU test suite and smoke().  (The bench's dominant kernels are
# unchanged since the r2d ncu captures.)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/job_r2_bench.sh ${1:-r2e}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${1:-r2e}_pytest.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${1:-r2e}_smoke.log 2>&1
echo done
