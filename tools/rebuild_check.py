"""Rebuild a scene with alternating Morton widths and check every build against a fresh one
(stale device slot data across rebuilds must not leak into a build).
    python tools/rebuild_check.py [--soup N]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--soup", type=int, default=0)
    a = ap.parse_args()
    from paper_2603_00292_b200 import compile_scene, scenes
    desc = scenes.soup_description(a.soup) if a.soup else scenes.sphere_description()
    fresh = {}
    for bits in (30, 63):
        sc = compile_scene(desc, f"lbvh{bits}", device=0)
        fresh[bits] = sc.tlas.download()
        print("fresh", bits, "ok", flush=True)
    sc = compile_scene(desc, "lbvh30", device=0)
    bad = 0
    for k, bits in enumerate((63, 30, 63, 63, 30, 30)):
        sc.tlas.build(bits)
        got = sc.tlas.download()
        diff = [f for f in fresh[bits] if not np.array_equal(got[f], fresh[bits][f])]
        print("rebuild", k, bits, "same" if not diff else "DIFFERENT " + ",".join(diff), flush=True)
        bad += bool(diff)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
