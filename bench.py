#!/usr/bin/env python
"""Benchmark of the B200 pcSIR / SIR filter step (BASELINE.json metric:
particle-updates/sec per filter step).

One "step" = one frame of the filter (propagate+gather -> bin -> dummies ->
likelihood -> normalise/estimate/ESS -> exact systematic resampling) over
all N particles. Default workload = BASELINE config 2: 256x256 frames,
N = 1e6, pcSIR with 1 px bins (the other bin sizes and SIR are reported
under "variants").

  python bench.py [--gpus N --steps K --warmup W]            # our arm
  python bench.py --impl reference [...]                     # CPU reference arm

Multi-GPU (torchrun): config 2 is a single filter, so ranks run independent
replicas ("replicas only"); time = max over ranks.
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

WORKLOADS = {
    # name: (width, n_particles, start_xy, cells_per_pixel or None for SIR)
    "c2": dict(width=256, n=1_000_000, start=(103.0, 128.0)),
    "c1": dict(width=64, n=10_000, start=(20.0, 32.0)),
}
VARIANTS = {"pcSIR-1px": 1.0, "pcSIR-0.5px": 0.5, "pcSIR-0.25px": 0.25, "pcSIR-2px": 2.0,
            "SIR": None}
ALGO_BYTES = {  # algorithmic bytes per particle per launch
    # pcSIR: R anc 4 + R state 20 + W state 20 + W cell 4; scan: R cell 4 + W ancestor 4
    "k_pc_step1": 48, "k_scan_emit:pc": 8,
    # SIR: + W loglik 8; sum: R 8; stats: R 8 + R 20; scan: R 8 + W 4
    "k_sir_propagate_lik": 52, "k_sir_sum": 8, "k_sir_stats": 28, "k_scan_emit:sir": 12,
}
STEP_BYTES = 60  # canonical fused minimum per particle-update


def frames_for(width, count, start, seed=0):
    """Synthetic config frames: one Gaussian spot (sigma 1.5, I0 20, bg 10)
    moving +0.5 px/frame along x, Poisson noise, seed 0 (BASELINE configs)."""
    rng = np.random.default_rng(seed)
    x, y = start
    xs = np.arange(width)
    out = np.empty((count, width, width), dtype=np.float32)
    truth = np.empty((count, 2))
    for k in range(count):
        x += 0.5
        gx = np.exp(-((xs - x) ** 2) / (2 * 1.5 ** 2))
        gy = np.exp(-((xs - y) ** 2) / (2 * 1.5 ** 2))
        out[k] = rng.poisson(20.0 * np.outer(gy, gx) + 10.0)
        truth[k] = (x, y)
    return out, truth


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout
                    self.rows.append([c.strip() for c in out.strip().split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def make_cfg(pc, wl, cpp, seed):
    width, n = wl["width"], wl["n"]
    init = pc.InitSpec(pc.StateVector(wl["start"][0], wl["start"][1], 0.5, 0.0, 20.0), "gauss",
                       sigma=2.0)
    dyn = pc.DynamicsParams(0.5, 0.1, 1.0)
    lik = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5))
    res = pc.ResampleConfig(1.0, "systematic")
    if cpp is None:
        return pc.FilterConfig(n, init, dyn, res, lik), None
    grid = pc.BinGrid(-0.5, -0.5, cpp, cpp, int(round(width / cpp)), int(round(width / cpp)))
    return pc.PcFilterConfig(n, init, dyn, res, lik, grid=grid), grid


def c_cfg(pc, _lib, cfg, grid, seed, use_graph=True):
    c = _lib.PcsTrackCfg()
    c.method = 0 if grid is None else 1
    c.placement = 0
    c.n_particles = cfg.n_particles
    c.init = cfg.init.to_c()
    c.dyn = cfg.dynamics.to_c()
    c.spot = cfg.likelihood.spot_c()
    if grid is not None:
        c.grid = grid.to_c()
    c.seed = seed
    c.frame0 = 0
    c.use_graph = 1 if use_graph else 0
    return c


def run_device_steps(torch, pc, _lib, cfg, grid, dev_frames, warmup, steps, seed, flush,
                     sampler=None):
    """Warm-up W frames, then time K frames one graph replay at a time with an
    L2 flush (write > L2) between timed steps. Returns (per-step ms list, outs)."""
    import ctypes
    k_total = warmup + steps
    c = c_cfg(pc, _lib, cfg, grid, seed)
    st = _lib.stream()
    _lib.check(_lib.lib().pcs_track_begin(_lib.ctx(), ctypes.byref(c), dev_frames.shape[1],
                                          dev_frames.shape[2], st), "pcs_track_begin")
    est = torch.empty((k_total, 5), dtype=torch.float64, device="cuda")
    ess = torch.empty(k_total, dtype=torch.float64, device="cuda")
    res = torch.empty(k_total, dtype=torch.uint8, device="cuda")
    occ = torch.empty(k_total, dtype=torch.int64, device="cuda")

    def step(k0, k1):
        fr = dev_frames[k0:k1]
        _lib.check(_lib.lib().pcs_track_steps(_lib.ctx(), _lib.ptr(fr), k0, k1,
                                              _lib.ptr(est[k0:]), _lib.ptr(ess[k0:]),
                                              _lib.ptr(res[k0:]), _lib.ptr(occ[k0:]), st),
                   "pcs_track_steps")

    step(0, warmup)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    if sampler:
        sampler.start()
    for i in range(steps):
        flush.zero_()                      # > L2: every timed step starts cold
        ev[i][0].record()
        step(warmup + i, warmup + i + 1)
        ev[i][1].record()
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    out = _lib.PcsTrackResult()
    rc = _lib.lib().pcs_track_end(_lib.ctx(), ctypes.byref(out), st)
    _lib.check(rc, "pcs_track_end")
    ms = [a.elapsed_time(b) for a, b in ev]
    return ms, dict(est=est.cpu().numpy(), ess=ess.cpu().numpy(), occ=occ.cpu().numpy(),
                    flags=int(out.flags), clocks=clocks,
                    launches=int(_lib.lib().pcs_track_launches_per_step(_lib.ctx())))


def kernel_profile(torch, pc, _lib, cfg, grid, dev_frames, warmup, frames_n, seed, flush):
    """Per-kernel device time (CUDA events on the launching stream, no graph),
    L2 flushed before every frame."""
    import ctypes
    c = c_cfg(pc, _lib, cfg, grid, seed, use_graph=False)
    st = _lib.stream()
    _lib.check(_lib.lib().pcs_track_begin(_lib.ctx(), ctypes.byref(c), dev_frames.shape[1],
                                          dev_frames.shape[2], st), "pcs_track_begin")
    k_total = warmup + frames_n
    est = torch.empty((k_total, 5), dtype=torch.float64, device="cuda")
    ess = torch.empty(k_total, dtype=torch.float64, device="cuda")
    res = torch.empty(k_total, dtype=torch.uint8, device="cuda")
    occ = torch.empty(k_total, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().pcs_track_steps(_lib.ctx(), _lib.ptr(dev_frames), 0, warmup,
                                          _lib.ptr(est), _lib.ptr(ess), _lib.ptr(res),
                                          _lib.ptr(occ), st))
    acc = np.zeros(8)
    buf = (ctypes.c_double * 8)()
    for k in range(warmup, k_total):
        flush.zero_()
        fr = dev_frames[k:k + 1]
        _lib.check(_lib.lib().pcs_track_steps_timed(
            _lib.ctx(), _lib.ptr(fr), k, k + 1, _lib.ptr(est[k:]), _lib.ptr(ess[k:]),
            _lib.ptr(res[k:]), _lib.ptr(occ[k:]), buf, 8, st), "pcs_track_steps_timed")
        acc += np.array(buf[:])
    out = _lib.PcsTrackResult()
    _lib.lib().pcs_track_end(_lib.ctx(), ctypes.byref(out), st)
    n_k = int(_lib.lib().pcs_track_launches_per_step(_lib.ctx()))
    names = [_lib.lib().pcs_track_kernel_name(_lib.ctx(), i).decode() for i in range(n_k)]
    return {nm: acc[i] / frames_n for i, nm in enumerate(names)}


def cpu_port_track(width, n, frames, start, cpp):
    """The oracle port of the reference driver (filtering.py:148-182 /
    binning.py:175-226), numpy Generator draws like the reference, and the
    reference's own compiled likelihood kernel when oracle/_ref has it."""
    from oracle import pcsir_oracle as orc
    ssd = orc.reference_ssd_kernel()
    lik = orc.SpotModel(1.5, 10.0, 10.0, 5, ssd=ssd)
    grid = None if cpp is None else (-0.5, -0.5, cpp, cpp, int(round(width / cpp)),
                                     int(round(width / cpp)))
    rng = np.random.default_rng(0)
    t0 = time.perf_counter()
    orc.track([f.astype(np.float64) for f in frames], n, [start[0], start[1], 0.5, 0.0, 20.0],
              2.0, [0.5, 0.5, 0.1, 0.1, 1.0], 1.0, lik, rng, grid=grid)
    dt = time.perf_counter() - t0
    return n * len(frames) / dt, dt, ("reference _speedups.pyx kernel (oracle/_ref)"
                                      if ssd is not None else "oracle C kernel")


def reference_arm(args, wl, cpp):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    frames, _ = frames_for(wl["width"], args.warmup + args.steps, wl["start"])
    n = wl["n"]
    # warm-up frames then K timed frames; each step = one frame over all N particles
    t0 = time.perf_counter()
    v, dt, kern = cpu_port_track(wl["width"], n, frames, wl["start"], cpp)
    total = time.perf_counter() - t0
    per_step = dt / (args.warmup + args.steps)
    value = n / per_step
    line = {
        "impl": "reference", "metric": "particle-updates/sec per filter step",
        "value": value, "unit": "particle-updates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}:{args.variant}", "n_particles": n,
                   "frame": f"{wl['width']}x{wl['width']}"},
        "cpu_baseline": {"value": value, "unit": "particle-updates/s", "cores": 1,
                         "kind": "port",
                         "sample": f"{args.warmup + args.steps} frames x N={n} "
                                   f"(reference driver restated in oracle/, {kern}), "
                                   f"{total:.1f} s"},
        "e2e": {"value": value, "unit": "particle-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="pcSIR-1px", choices=sorted(VARIANTS))
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    cpp_main = VARIANTS[args.variant]
    if args.impl == "reference":
        return reference_arm(args, wl, None if cpp_main is None else cpp_main)

    import torch
    import paper_1310_5541_b200 as pc
    from paper_1310_5541_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = wl["n"]
    k_total = args.warmup + args.steps
    frames_host, truth = frames_for(wl["width"], k_total, wl["start"])
    dev_frames = torch.from_numpy(frames_host).cuda()
    info = _lib.device_info(local)
    flush = torch.empty(int(max(2 * info["l2_bytes"], 256 << 20)) // 4, dtype=torch.float32,
                        device="cuda")

    def timed_variant(cpp, sampler=None, steps=None, warmup=None):
        steps = steps or args.steps
        warmup = warmup or args.warmup
        cfg, grid = make_cfg(pc, wl, cpp, args.seed)
        return run_device_steps(torch, pc, _lib, cfg, grid, dev_frames, warmup, steps,
                                args.seed, flush, sampler)

    # ---- headline: K timed steps of the main variant ----
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    ms, out = timed_variant(cpp_main, sampler)
    total_ms = float(np.sum(ms))
    if dist:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    torch.cuda.synchronize()
    value = n * args.steps * world / (total_ms * 1e-3)
    rmse = float(np.sqrt(np.mean(np.sum((out["est"][args.warmup:, :2]
                                         - truth[args.warmup:]) ** 2, axis=1))))

    # ---- per-kernel profile (dominant kernel roofline) ----
    cfg, grid = make_cfg(pc, wl, cpp_main, args.seed)
    kprof = kernel_profile(torch, pc, _lib, cfg, grid, dev_frames, args.warmup,
                           min(args.steps, 20), args.seed, flush)
    dom = max(kprof, key=kprof.get)
    peak, peak_kind = peaks()
    key = dom if dom != "k_scan_emit" else ("k_scan_emit:pc" if cpp_main else "k_scan_emit:sir")
    dom_bytes = ALGO_BYTES.get(key, 0) * n
    achieved = dom_bytes / (kprof[dom] * 1e-3) / 1e9 if kprof[dom] > 0 else 0.0
    step_ms = total_ms / args.steps
    l2 = info["l2_bytes"]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "algo_bytes_per_launch": dom_bytes,
                "kernel_ms": {k: round(v, 5) for k, v in kprof.items()},
                "kernel_share": {k: round(v / sum(kprof.values()), 4) for k, v in kprof.items()},
                "step_bytes_per_particle": STEP_BYTES,
                "step_achieved_gbs": STEP_BYTES * n / (step_ms * 1e-3) / 1e9,
                "step_frac": STEP_BYTES * n / (step_ms * 1e-3) / 1e9 / peak,
                "working_set_mb": round(60 * n / 1e6, 1), "l2_mb": round(l2 / 2 ** 20, 1)}

    # ---- e2e: the public call with host frames (H2D + D2H inside the timed region) ----
    cfg_e, _ = make_cfg(pc, wl, cpp_main, args.seed)
    host_frames = [pc.ImageFrame(f) for f in frames_host[:args.warmup]]
    track = pc.pcsir_track if cpp_main is not None else pc.sir_track
    track(host_frames, cfg_e, pc.PhiloxRng(args.seed))          # warm (allocs, graph)
    e_frames = [pc.ImageFrame(f) for f in frames_host[args.warmup:k_total]]
    cfg_e, _ = make_cfg(pc, wl, cpp_main, args.seed)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = track(e_frames, cfg_e, pc.PhiloxRng(args.seed))
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": n * args.steps * world / e2e_s, "unit": "particle-updates/s",
           "h2d_bytes_per_step": int(wl["width"] * wl["width"] * 4),
           "d2h_bytes_per_step": 5 * 8 + 8 + 1 + 8, "path": r.path,
           "note": "pcsir_track(list of host ImageFrame) wall time incl. frame upload, "
                   "graph capture and result download"}

    # ---- other variants (SIR and the other bin sizes), shorter runs ----
    variants = {}
    if not args.no_variants:
        for name, cpp in VARIANTS.items():
            if name == args.variant:
                continue
            vms, vout = timed_variant(cpp, None, steps=min(args.steps, 30))
            vt = float(np.sum(vms))
            variants[name] = {"value": n * len(vms) / (vt * 1e-3),
                              "ms_per_step": vt / len(vms),
                              "mean_occupied_bins": float(np.mean(vout["occ"][args.warmup:]))}

    # ---- CPU baseline: oracle port on this host (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nf = 10
        v, dt, kern = cpu_port_track(wl["width"], n, frames_host[:nf], wl["start"], cpp_main)
        cpu = {"value": v, "unit": "particle-updates/s", "cores": 1, "kind": "port",
               "sample": f"{nf} frames x N={n} {args.variant} (reference driver restated in "
                         f"oracle/, {kern}) = {dt:.1f} s on 1 host core"}

    if rank == 0:
        line = {
            "metric": "particle-updates/sec per filter step", "value": value,
            "unit": "particle-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.workload}:{args.variant}", "n_particles": n,
                       "frame": f"{wl['width']}x{wl['width']}", "bin_px": cpp_main,
                       "likelihood": "gauss-ssd 11x11, sigma_xi 10",
                       "resampling": "systematic every frame (threshold 1.0)",
                       "l2": "flushed (write > L2) before every timed step",
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "rmse_px": rmse, "mean_occupied_bins":
                           float(np.mean(out["occ"][args.warmup:]))},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": out["launches"] * args.steps,
            "clocks": out["clocks"], "variants": variants, "flags": out["flags"],
        }
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
