"""Per-warp timeline of the megakernel (diagnostic build: tools/variants.sh timeline
"-DRT_TIMELINE=1"; RT_B200_LIB=variants/timeline/librt_b200.so): start / end spread per SM,
fetches per warp, for the config-2 eye frame and the config-3 PT frame."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_00292_b200 import IntegratorConfig, _native, compile_scene, render_into, scenes
    L = _native.lib()
    L.rt_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
    W, H = 1920, 1080
    acc = torch.zeros((H * W, 4), dtype=torch.float32, device="cuda")
    for name, desc, integ, spp in (("eye_sphere", scenes.sphere_description(), "eye", 1),
                                   ("pt_cornell", scenes.cornell_description(), "pt",
                                    int(os.environ.get("RT_TIMELINE_PT_SPP", "1"))),
                                   ("eye_soup4k", scenes.soup_description(), "eye", 1)):
        sc = compile_scene(desc)
        if name == "eye_soup4k":
            W, H = 3840, 2160
            acc = torch.zeros((H * W, 4), dtype=torch.float32, device="cuda")
        for _ in range(3):
            render_into(sc, acc, W, H, spp, integ, cfg=IntegratorConfig(max_depth=5), count_rays=False)
        torch.cuda.synchronize()
        nw = 1036 * 4
        buf = np.zeros(4 * nw, np.uint64)
        _native.check(L.rt_debug_timeline(buf.ctypes.data_as(ctypes.c_void_p), nw))
        t = buf.reshape(nw, 4).astype(np.float64)
        t0 = t[:, 0].min()
        st, en, sm, nf = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, t[:, 2].astype(int), t[:, 3]
        span = en.max()
        print(f"{name}: kernel span {span:.1f} us; warp start spread {st.min():.1f}-{st.max():.1f} us "
              f"(p50 {np.median(st):.1f}); end spread {en.min():.1f}-{en.max():.1f} us (p10 {np.percentile(en, 10):.1f}, "
              f"p50 {np.median(en):.1f}, p90 {np.percentile(en, 90):.1f}); fetches/warp min {nf.min():.0f} "
              f"p50 {np.median(nf):.0f} max {nf.max():.0f}; SMs used {len(set(sm))}")
        per_sm = {}
        for s_, a, b in zip(sm, st, en):
            lo, hi = per_sm.get(s_, (1e30, 0))
            per_sm[s_] = (min(lo, a), max(hi, b))
        act = np.array([b - a for a, b in per_sm.values()])
        print(f"  per-SM active span: min {act.min():.1f} p50 {np.median(act):.1f} max {act.max():.1f} us; "
              f"warps per SM min {min(np.bincount(sm)[list(per_sm)])} max {max(np.bincount(sm))}")
        busy = np.sum(en - st) / (len(st) * span)
        print(f"  mean warp busy fraction of the span: {busy:.3f}")


if __name__ == "__main__":
    main()
