# build-stage measurement job (GPU box): stage timings, compile probe, one emit capture, GPU tests
set -x
python tools/prof_build.py --reps 20 > gpurun_out/r2_prof_build_${TAG:-x}.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:lbvh_emit_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r2_soup_emit_${TAG:-x} -f python tools/drive_build.py 2 30 soup > gpurun_out/r2_ncu_emit.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2_gputest_${TAG:-x}.log
