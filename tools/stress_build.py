"""Stress the LBVH build's inter-block hand-offs (global climb, programmatic dependent launch):
many sizes x both Morton widths x repeated in-place rebuilds, every rebuild compared with the
first build of its width (the build is deterministic), small sizes also with the CPU
restatement.   python tools/stress_build.py [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    from paper_2603_00292_b200 import compile_scene, scenes
    from oracle import oracle               # test infrastructure: the CPU restatement as the checker
    oracle.build()
    bad = 0
    for n in (2, 3, 255, 256, 257, 4096, 65537, 300000, 1000001, 4000000):
        desc = scenes.soup_description(n, seed=n)
        sc = compile_scene(desc, "lbvh30")
        for bits in (30, 63):
            sc.tlas.build(bits)
            first = sc.tlas.download()
            if n <= 300000:
                ref = oracle.lbvh_build(sc.tlas.tris, bits)
                for k in ("sorted_keys", "order", "child", "boxes"):
                    if not np.array_equal(first[k], ref[k]):
                        print("ORACLE MISMATCH", n, bits, k, flush=True)
                        bad += 1
            for r in range(reps):
                sc.tlas.build(63 if bits == 30 else 30)     # leave the other width's slot records behind
                sc.tlas.build(bits)
                got = sc.tlas.download()
                diff = [k for k in first if not np.array_equal(got[k], first[k])]
                if diff:
                    print("REBUILD MISMATCH", n, bits, r, diff, flush=True)
                    bad += 1
        print("n", n, "ok" if not bad else f"bad={bad}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
