#!/bin/bash
# Sort-variant check + A/B (one GPU box): bash tools/job_sort_ab.sh TAG VARIANT [more variants]
# LBVH parity tests and the rebuild stress run on VARIANT, then tools/ab_build.sh default + all.
cd "$(dirname "$0")/.."
tag=$1; shift
mkdir -p gpurun_out
RT_B200_LIB=variants/$1/librt_b200.so timeout 600 python -m pytest tests/test_gpu_lbvh.py -x -q > gpurun_out/${tag}_pytest.log 2>&1
RT_B200_LIB=variants/$1/librt_b200.so timeout 300 python tools/stress_build.py > gpurun_out/${tag}_stress.log 2>&1
bash tools/ab_build.sh default "$@" > gpurun_out/${tag}_ab.log 2>&1
