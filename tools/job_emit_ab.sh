cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1; shift
timeout 300 env RT_B200_LIB=variants/$1/librt_b200.so python -m pytest tests/test_gpu_lbvh.py -x -q > gpurun_out/${tag}_pytest.log 2>&1
bash tools/ab_build.sh default "$@" > gpurun_out/${tag}_ab.log 2>&1
for v in default "$@"; do
  if [ $v = default ]; then unset RT_B200_LIB; else export RT_B200_LIB=variants/$v/librt_b200.so; fi
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,gpu__time_duration.sum --clock-control none -k regex:lbvh_emit_kernel --launch-skip 1 --launch-count 1 --csv python tools/drive_build.py 2 30 soup > gpurun_out/${tag}_ncu_$v.csv 2>/dev/null
done
unset RT_B200_LIB
