#!/bin/bash
# radix/emit stage timings of the default build and every variants/* library (run on the GPU box)
for lib in "" variants/*/librt_b200.so; do
  name=${lib:-default}
  RT_B200_LIB=$lib python tools/prof_build.py --reps 10 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
print('$name', {k: (v['stages']['radix_passes'], v['stages']['emit_refit'], v['build_ms_median']) for k,v in d.items() if isinstance(v, dict)})"
done
