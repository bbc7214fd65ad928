"""Benchmark: LBVH build + primary rays on the 1M-triangle UV sphere at 1920x1080
(BASELINE.json configs[1]); path tracing of the Cornell box (configs[2]) as a
secondary measurement.  Prints ONE JSON line (rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Step (our arm): rebuild the 30-bit LBVH over the device-resident triangles
(K1-K5) + render one 1920x1080 eye sample (raygen + closest-hit + shade fused in
the persistent megakernel, K7) [+ one NCCL reduce of the (H*W,4) f32
accumulation buffer to rank 0 when N > 1].  Weak scaling: rank g renders
sample index g of the same frame (global sample index in the stream hash), so
N GPUs trace N * 2,073,600 rays per step; value = all rays / max-over-ranks time.
Between timed steps a 256 MiB buffer is written to flush the 126 MB L2.

--impl reference: the reference's algorithm ported to C (oracle/, float64, the
reference itself is a numba library that cannot travel to the GPU box) on the
host cores: SAH compile + render_frame('eye') of the same frame, rank 0 only.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W, H = 1920, 1080
METRIC = "Mrays/s (primary + diffuse bounce) & LBVH build ms at 1/2/4/8 B200 vs CPU ref"
WORKLOAD = "config2: LBVH-30 build + 1920x1080 primary rays (eye, 1 spp/GPU, jitter, seed 0) on the synthetic " \
           "1M-triangle UV sphere (stacks 500 x slices 1000), camera (0,0,2.5)"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled in the background."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.proc = None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.device), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.perf_counter(), parts))

    def mark(self):
        self.marks.append(time.perf_counter())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        lo, hi = (self.marks[0], self.marks[-1]) if len(self.marks) >= 2 else (0, 1e30)
        inside = [s for t, s in self.samples if lo <= t <= hi] or [s for _, s in self.samples]
        sm = [float(s[1]) for s in inside if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in inside if s[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[k] for s in inside for k in range(4) if s[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside),
                "window": "warm-up + timed region" if len(self.marks) < 2 else "timed region"}


def dist_setup():
    import torch
    import torch.distributed as dist
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and not dist.is_initialized():
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle port (float64 C restatement)
# ---------------------------------------------------------------------------

def cpu_reference_step(orc_desc_fn, workers):
    """One reference step: SAH compile (reference algorithm, 1 thread as in the reference)
    + render_frame('eye') of the 1920x1080 frame on `workers` threads.  Returns (rays, secs, build_s)."""
    from oracle import oracle
    t0 = time.perf_counter()
    sc = oracle.scene_from_description(orc_desc_fn())
    t1 = time.perf_counter()
    _, rays = sc.render_frame(W, H, 1, "eye", seed=0, workers=workers)
    t2 = time.perf_counter()
    return rays, t2 - t0, t1 - t0


def run_reference(args, ws, rank):
    if rank != 0:
        return
    from oracle import oracle
    from paper_2603_00292_b200 import scenes
    oracle.build()
    cores = os.cpu_count() or 1
    desc = scenes.sphere_description()
    fn = lambda: desc
    for _ in range(args.warmup):
        cpu_reference_step(fn, cores)
    rays_tot, secs, builds = 0, 0.0, 0.0
    for _ in range(args.steps):
        r, s, b = cpu_reference_step(fn, cores)
        rays_tot += r
        secs += s
        builds += b
    value = rays_tot / secs / 1e6
    sample = (f"full config-2 step on the host: C float64 restatement of compile_scene (binned-SAH build, "
              f"accel.py:68-187, 1 thread) + render_frame('eye') 1920x1080 1 spp ({cores} threads); "
              f"mean SAH build {1e3 * builds / args.steps:.0f} ms")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "parallelism": f"cpu{cores}"},
            "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_build_ms": 1e3 * builds / args.steps}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, ws, rank, local):
    import torch
    import torch.distributed as dist
    from paper_2603_00292_b200 import IntegratorConfig, closest_hit_batch, compile_scene, render_into, scenes
    from paper_2603_00292_b200 import accel
    from paper_2603_00292_b200.integrators import raygen

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peak_gbs, peak_src = load_peaks()
    desc = scenes.sphere_description()
    sc = compile_scene(desc, "lbvh30", device=local)
    tl = sc.tlas
    n_tri = tl.n
    npix = W * H
    sample = rank                      # weak scaling: sample split, global sample index
    accum = torch.zeros((npix, 4), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # -- per-ray cost of this exact BVH (stats build of the trace kernel) -------
    rays_dev = raygen(sc, W, H, sample=sample)
    hits = torch.empty((npix, 4), dtype=torch.float32, device=dev)
    st = torch.empty((npix, 2), dtype=torch.int32, device=dev)
    accel.trace_closest(tl, rays_dev, hits, stats=st)
    torch.cuda.synchronize()
    n_tests = float(st[:, 0].double().mean())
    n_nodes = float(st[:, 1].double().mean())
    hit_frac = float((hits[:, 1].view(torch.int32) >= 0).double().mean())
    bytes_per_ray = 64.0 * n_nodes + 48.0 * n_tests + 32.0
    build_bytes = 328.0 * n_tri          # SURVEY 8(d) algorithmic bytes, 30-bit keys
    stages = tl.build_profiled(30)

    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step(timed=None):
        if timed:
            timed[0].record()
        tl.build(30)
        if timed:
            timed[1].record()
        render_into(sc, accum, W, H, 1, "eye", 0, None, True, "mega", samples=(sample, sample + 1),
                    count_rays=False)
        if timed:
            timed[2].record()
        if ws > 1:
            dist.reduce(accum, 0)
        if timed:
            timed[3].record()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    evs = [[ev() for _ in range(4)] for _ in range(args.steps)]
    for k in range(args.steps):
        flush.fill_(k & 0xFF)
        step(evs[k])
    torch.cuda.synchronize()
    clocks.mark()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    time.sleep(0.12)
    clocks.stop()
    t_build = sum(e[0].elapsed_time(e[1]) for e in evs)
    t_trace = sum(e[1].elapsed_time(e[2]) for e in evs)
    t_reduce = sum(e[2].elapsed_time(e[3]) for e in evs)
    t_total = sum(e[0].elapsed_time(e[3]) for e in evs)
    local_t = torch.tensor([t_total, t_build, t_trace, t_reduce], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(local_t, op=dist.ReduceOp.MAX)
    t_total, t_build, t_trace, t_reduce = (float(x) for x in local_t.cpu())
    K = args.steps
    rays_all = ws * npix * K
    value = rays_all / (t_total * 1e-3) / 1e6
    trace_mrays = ws * npix * K / (t_trace * 1e-3) / 1e6
    build_ms = t_build / K

    # -- end to end through the public API with host buffers ---------------------
    e2e = None
    if not args.no_e2e:
        r = rays_dev.cpu().numpy().astype(np.float64)
        O, D = np.ascontiguousarray(r[:, 0:3]), np.ascontiguousarray(r[:, 4:7])
        host_tris = tl.tris.copy()
        closest_hit_batch(sc, O, D)       # warm (staging buffers)
        ke = max(1, min(K, 5))
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(ke):
            tl.refit(host_tris, 30)
            res = closest_hit_batch(sc, O, D)
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        tt = torch.tensor([te], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
        e2e = {"value": ws * npix * ke / te / 1e6, "unit": "Mrays/s",
               "h2d_bytes_per_step": int(host_tris.nbytes + npix * (24 + 24 + 8 + 8)),
               "d2h_bytes_per_step": int(npix * (8 + 8 + 8 + 8 + 8 + 24)),
               "path": "GpuTlas.refit(host fp32 vertices) + closest_hit_batch(host float64 rays) -> host "
                       "float64/int64 (t, inst, prim, u, v, normal)", "steps": ke}

    # -- secondary: config 3 path tracing (Cornell 1080p, max_depth 5), rank 0 ------
    pt = None
    if rank == 0 and not args.no_pt:
        cfg = IntegratorConfig(max_depth=5)
        cs = compile_scene(scenes.cornell_description(), device=local)
        acc = torch.zeros((npix, 4), dtype=torch.float32, device=dev)
        pt = {"workload": f"config3: cornell 1920x1080, {args.pt_spp} spp, pt, max_depth 5, seed 0"}
        for kern in ("mega", "wavefront"):
            render_into(cs, acc, W, H, 2, "pt", 0, cfg, kernel=kern)        # warm
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record()
            rays = render_into(cs, acc, W, H, args.pt_spp, "pt", 0, cfg, kernel=kern, count_rays=False)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            rays = render_into(cs, acc, W, H, 1, "pt", 0, cfg, kernel=kern) * args.pt_spp  # count (1 spp probe)
            pt[kern] = {"ms": ms, "mrays_s_est": rays / (ms * 1e-3) / 1e6}
        acc.zero_()
        exact = render_into(cs, acc, W, H, args.pt_spp, "pt", 0, cfg, kernel="mega")
        for kern in ("mega", "wavefront"):
            pt[kern]["mrays_s"] = exact / (pt[kern]["ms"] * 1e-3) / 1e6
            pt[kern].pop("mrays_s_est")
        pt["rays_per_frame"] = exact
        pt["rays_per_path"] = exact / (npix * args.pt_spp)

    # -- CPU baseline (rank 0, N = 1): the oracle port on the host cores --------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        r, s, b = cpu_reference_step(lambda: desc, cores)
        cpu = {"value": r / s / 1e6, "unit": "Mrays/s", "cores": cores, "kind": "port",
               "sample": f"one full config-2 step: C float64 restatement of the reference (SAH compile "
                         f"{1e3 * b:.0f} ms on 1 thread + render_frame('eye') 1920x1080 on {cores} threads)"}

    if rank != 0:
        return
    trace_ms = t_trace / K
    trace_bytes = bytes_per_ray * npix
    trace_gbs = trace_bytes / (trace_ms * 1e-3) / 1e9
    build_gbs = build_bytes / (build_ms * 1e-3) / 1e9
    roof_trace = {"kernel": "pt_megakernel (eye: raygen + while-while trace + shade)", "bound": "hbm",
                  "achieved": trace_gbs, "peak": peak_gbs, "unit": "GB/s", "frac": trace_gbs / peak_gbs,
                  "traffic": None, "bytes_per_ray": bytes_per_ray,
                  "bytes_formula": f"64 B x {n_nodes:.2f} internal-node fetches + 48 B x {n_tests:.2f} tri tests "
                                   "+ 32 B accum RMW per ray (stats build of the same kernel)",
                  "peak_source": peak_src}
    roof_build = {"kernel": "LBVH build (K1-K5, 9 launches)", "bound": "hbm", "achieved": build_gbs,
                  "peak": peak_gbs, "unit": "GB/s", "frac": build_gbs / peak_gbs, "traffic": None,
                  "bytes_formula": "328 B/tri x 1,000,000 tris (SURVEY 8(d))", "stage_ms": stages,
                  "peak_source": peak_src}
    dominant = roof_trace if t_trace >= t_build else roof_build
    line = {
        "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": ws, "steps": K, "warmup": args.warmup,
        "ms_per_step": t_total / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (config-2 UV sphere generated in-process; no dataset)",
        "config": {"workload": WORKLOAD, "triangles": n_tri, "rays_per_gpu_per_step": npix,
                   "parallelism": f"sample-split x{ws} + NCCL reduce" if ws > 1 else "1 GPU",
                   "l2": "256 MiB buffer written between timed steps (flush)", "hit_fraction": hit_frac},
        "lbvh_build_ms": build_ms, "trace_mrays_s": trace_mrays, "reduce_ms": t_reduce / K,
        "roofline": dominant, "roofline_other": roof_build if dominant is roof_trace else roof_trace,
        "per_ray": {"internal_node_fetches": n_nodes, "triangle_tests": n_tests},
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
        "gpu_launches": K * (9 + 1), "gpu_launches_detail": "per step: 9 LBVH kernels (bounds, bounds_finish, "
                                                            "morton, histogram, 4 onesweep passes, fused emit+refit) + "
                                                            "1 megakernel",
        "pt": pt,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--pt-spp", type=int, default=64)
    ap.add_argument("--no-pt", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, ws, rank)
        return
    ws, rank, local = dist_setup()
    run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
