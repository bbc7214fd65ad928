cd "$(dirname "$0")/.."
mkdir -p gpurun_out
RT_B200_LIB=variants/t512i14/librt_b200.so timeout 600 python -m pytest tests/test_gpu_lbvh.py -x -q > gpurun_out/s71_pytest.log 2>&1
RT_B200_LIB=variants/t512i14/librt_b200.so timeout 300 python tools/stress_build.py > gpurun_out/s71_stress.log 2>&1
bash tools/ab_build.sh t512i13 t512i14 t512i15 > gpurun_out/s71_ab.log 2>&1
