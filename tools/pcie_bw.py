"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone, and both
directions at once on two streams (the bound of the e2e host-buffer path)."""
import json

import torch


def main():
    n = 128 << 20
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    out["h2d_gbs"] = n / t / 1e6
    t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
    out["d2h_gbs"] = n / t / 1e6
    t = timed(both)
    out["bidir_each_gbs"] = n / t / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
