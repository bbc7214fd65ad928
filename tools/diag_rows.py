"""Per-row cost of the config-2 eye frame: BVH4 node fetches + triangle tests per ray by
image row band (the persistent kernel fetches tiles top to bottom, so an expensive last
band makes a tail)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_00292_b200 import accel, compile_scene, scenes
    from paper_2603_00292_b200.integrators import raygen
    W, H = 1920, 1080
    for name, desc in (("sphere1M", scenes.sphere_description()),):
        sc = compile_scene(desc)
        rays = raygen(sc, W, H)
        hits = torch.empty((W * H, 4), dtype=torch.float32, device="cuda")
        st = torch.empty((W * H, 2), dtype=torch.int32, device="cuda")
        accel.trace_closest(sc.tlas, rays, hits, stats=st)
        torch.cuda.synchronize()
        s = st.cpu().numpy().reshape(H, W, 2).astype(np.float64)
        cost = s[:, :, 1] + 0.5 * s[:, :, 0]
        bands = cost.reshape(27, 40, W).mean(axis=(1, 2))
        print(name, "mean", cost.mean(), "per 40-row band:", " ".join(f"{b:.1f}" for b in bands))
        print(name, "max ray cost", cost.max(), "99.9% ray", np.percentile(cost, 99.9))


if __name__ == "__main__":
    main()
