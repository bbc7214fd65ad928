#!/bin/bash
# Round-2 ncu captures for profiles/ (GPU box, one GPU, --clock-control none, cold caches):
# config-2 build, config-4 build, config-2 eye megakernel, config-3 PT megakernel and one
# wavefront wave (wf_raygen / wf_extend / wf_shade / wf_accumulate), config-4 eye megakernel,
# plus the launch list of two bench.py config-2 steps.  Outputs under gpurun_out/.
set -x
K='regex:lbvh_|onesweep'
# one 30-bit build = 7 kernels (bounds, Morton + histograms, 3 x onesweep10, emit, global emit)
ncu --set full --clock-control none --import-source on -k "$K" --launch-skip 7 --launch-count 7 \
    -o gpurun_out/r2_build -f python tools/drive_build.py 2 30 > gpurun_out/r2_ncu_build.log 2>&1
ncu --set full --clock-control none --import-source on -k "$K" --launch-skip 7 --launch-count 7 \
    -o gpurun_out/r2_soup_build -f python tools/drive_build.py 2 30 soup > gpurun_out/r2_ncu_soup_build.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pt_megakernel --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r2_mega_eye -f python tools/drive_render.py eye 2 > gpurun_out/r2_ncu_eye.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pt_megakernel --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r2_mega_pt -f python tools/drive_render.py pt 2 > gpurun_out/r2_ncu_pt.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wf_ --launch-skip 12 --launch-count 12 \
    -o gpurun_out/r2_wf_pt -f python tools/drive_render.py ptwf 2 > gpurun_out/r2_ncu_wf.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pt_megakernel --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r2_soup_trace -f python tools/drive_render.py soup 2 > gpurun_out/r2_ncu_soup.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-pt --no-e2e > gpurun_out/r2_ncu_launch_bench.log 2>&1
