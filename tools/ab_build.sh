# A/B of build variants in one box: bash tools/ab_build.sh v1 v2 ... (each twice, interleaved)
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = default ]; then unset RT_B200_LIB; else export RT_B200_LIB=variants/$v/librt_b200.so; fi
  echo "== $v"; timeout 300 python tools/prof_build.py --reps 30 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(' '.join(f\"{k}:{v['build_ms_median']:.4f}/emit{v['stages']['emit_refit']:.4f}/sort{v['stages']['radix_passes']:.4f}\" for k,v in d.items()))"
done; done
