cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_render.py tests/test_gpu_spec.py tests/test_gpu_multi.py -x -q > gpurun_out/s65_pytest.log 2>&1
for v in nochunk default nochunk default; do
  if [ $v = default ]; then unset RT_B200_LIB; else export RT_B200_LIB=variants/$v/librt_b200.so; fi
  echo "$v $(timeout 600 python bench.py --config 3 --kernel mega --no-cpu --no-e2e --steps 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["value"],1))')"
done > gpurun_out/s65_chunk.log 2>&1
