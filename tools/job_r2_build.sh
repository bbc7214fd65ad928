set -x
python tools/prof_build.py --reps 20 > gpurun_out/r2_prof_build_wide.json 2>&1
RT_B200_LIB=variants/narrow/librt_b200.so python tools/prof_build.py --reps 20 > gpurun_out/r2_prof_build_narrow.json 2>&1
python tools/compile_probe.py > gpurun_out/r2_compile_probe2.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:lbvh_emit_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r2_soup_emit_wide -f python tools/drive_build.py 2 30 soup > gpurun_out/r2_ncu_emit.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2_gputest7.log
