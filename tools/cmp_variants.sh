# usage: bash /tmp/.. variants...  (run on box)
for v in "$@"; do if [ $v = default ]; then unset RT_B200_LIB; else export RT_B200_LIB=variants/$v/librt_b200.so; fi; echo "== $v"; timeout 100 python tools/rebuild_check.py 2>&1 | grep -c same; timeout 200 python tools/prof_build.py --soup 10000000 --reps 10 2>&1 | grep -E "build_ms|emit|/30\"|/63\"" | paste -sd' ' ; done
