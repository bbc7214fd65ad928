#!/bin/bash
# Round-2 bench lines for every config (one GPU box) -> gpurun_out/${1}_bench_*.json
cd "$(dirname "$0")/.."
tag=${1:-r2b}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt
for c in 2 4 5; do
  timeout 900 python bench.py --config $c > gpurun_out/${tag}_bench_c$c.json 2> gpurun_out/${tag}_bench_c$c.err
done
timeout 900 python bench.py --config 3 --kernel mega > gpurun_out/${tag}_bench_c3m.json 2> gpurun_out/${tag}_bench_c3m.err
timeout 900 python bench.py --config 3 --kernel wavefront > gpurun_out/${tag}_bench_c3w.json 2> gpurun_out/${tag}_bench_c3w.err
timeout 900 python bench.py > gpurun_out/${tag}_bench_default.json 2> gpurun_out/${tag}_bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
echo done
