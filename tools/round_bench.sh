#!/bin/bash
# Full measurement pass (GPU box): every bench config + the reference arm -> gpurun_out/bench_*.json
set -x
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config 3 --kernel mega --no-cpu > gpurun_out/bench_c3m.json 2> gpurun_out/bench_c3m.err
python bench.py --config 3 --kernel wavefront --no-cpu > gpurun_out/bench_c3w.json 2> gpurun_out/bench_c3w.err
python bench.py --config 4 --steps 10 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
