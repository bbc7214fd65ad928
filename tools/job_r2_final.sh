#!/bin/bash
# Round-2 final measurement job (one GPU box): bench lines for every config + the reference
# arm, the ncu captures of tools/r2_profile.sh, then the GPU test suite.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2f_smi.txt
for c in 2 4 5; do
  timeout 900 python bench.py --config $c > gpurun_out/r2f_bench_c$c.json 2> gpurun_out/r2f_bench_c$c.err
done
timeout 900 python bench.py --config 3 --kernel mega > gpurun_out/r2f_bench_c3m.json 2> gpurun_out/r2f_bench_c3m.err
timeout 900 python bench.py --config 3 --kernel wavefront > gpurun_out/r2f_bench_c3w.json 2> gpurun_out/r2f_bench_c3w.err
timeout 900 python bench.py > gpurun_out/r2f_bench_default.json 2> gpurun_out/r2f_bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err
timeout 2400 bash tools/r2_profile.sh > gpurun_out/r2f_profile.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_pytest.log 2>&1
echo done
