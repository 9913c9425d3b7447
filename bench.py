#!/usr/bin/env python
"""Benchmark of the B200 pcSIR / SIR filter step (BASELINE.json metric:
particle-updates/sec per filter step; one line of JSON on rank 0).

A "step" is one frame of the filter over all N particles of the workload
(gather -> propagate -> bin -> dummies -> likelihood -> normalise / estimate /
ESS -> exact systematic resampling). Workloads (BASELINE.json configs):

  c1  64x64,   N=1e4, pcSIR 1 px (the reference's CPU-scale case)
  c2  256x256, N=1e6, pcSIR 1 px
      (SIR and the 0.25/0.5/2 px grids are reported under "variants")
  c3  512x512, N=1e7, erf-PSF Poisson likelihood 15x15, pcSIR 0.5 px (+ SIR)
  c4  2048x2048, 4096 targets x 1e5 particles, pcSIR 1 px; targets sharded
      across GPUs with no communication
  c5  4096x4096, N=2^30, pcSIR 0.25 px; one filter sharded by particle
      across GPUs (NCCL all-reduce / all-gather / all-to-all); 1 GPU = fused
                                                    <- default headline: the
      largest BASELINE.json config that fits one B200 (20 GiB of states)

The default line also carries "likelihood_roofline": the per-particle SIR
likelihood kernel measured at c3 (erf-PSF Poisson 15x15, N=1e7) and c2
(Gaussian SSD 11x11, N=1e6) against the FP32 / SFU pipe bound of SURVEY
§8(d)'s minimal operation counts.

  python bench.py [--gpus N --steps K --warmup W --workload c2]
  python bench.py --impl reference [...]     # the reference CPU path, rank 0
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
    "c1": dict(width=64, n=10_000, start=(20.0, 32.0), variant="pcSIR-1px", model="gauss", hw=5),
    "c2": dict(width=256, n=1_000_000, start=(103.0, 128.0), variant="pcSIR-1px", model="gauss",
               hw=5),
    "c3": dict(width=512, n=10_000_000, start=(203.0, 256.0), variant="pcSIR-0.5px", model="erf",
               hw=7),
    "c4": dict(width=2048, n=100_000, targets=4096, variant="pcSIR-1px", model="gauss", hw=5),
    "c5": dict(width=4096, n=1 << 30, start=(2043.0, 2048.0), variant="pcSIR-0.25px",
               model="gauss", hw=5),
}
VARIANTS = {"pcSIR-1px": 1.0, "pcSIR-0.5px": 0.5, "pcSIR-0.25px": 0.25, "pcSIR-2px": 2.0,
            "SIR": None}
OTHER_VARIANTS = {"c2": ["SIR", "pcSIR-0.5px", "pcSIR-0.25px", "pcSIR-2px"], "c3": ["SIR"],
                  "c1": ["SIR"]}
ALGO_BYTES = {  # algorithmic bytes per particle per launch
    # pcSIR step1: R anc 4 + R state 20 + W state 20 + W cell 4; scan: R cell 4 + W anc 4
    "k_pc_step1": 48, "k_sys_resample:pc": 8,
    # SIR: + W loglik 8; sum: R 8; stats: R 8 + R 20; scan: R 8 + W 4
    "k_sir_propagate_lik": 52, "k_sir_sum": 8, "k_sir_stats": 28, "k_sys_resample:sir": 12,
    # multi-target frame kernel: step1 48 + scan R cell 4 + W anc 4
    "k_mt_frame": 56,
}
STEP_BYTES = 60  # canonical fused minimum per particle-update
L2_BYTES = 132_644_864   # B200 L2 (126.5 MiB): decides the L2 flush, same rule in both arms
# Minimal likelihood operation counts per evaluation (separable
# forms): FP32 FLOPs and SFU (MUFU) operations; redundant non-separable
# arithmetic does not count.
#   Gaussian SSD S x S: 2S exp (MUFU) + ~4 FLOP each, S amp*gx hoists, 5 S^2
#   erf-PSF Poisson S x S: 2(S+1) erf edges (~20 FLOP each, no MUFU) + per pixel
#   one lg2 (MUFU) and ~6 FLOP
def lik_min_ops(model, hw):
    S = 2 * hw + 1
    if model == "gauss":
        return {"flop": 2 * S * 4 + S + 5 * S * S, "mufu": 2 * S}
    return {"flop": 2 * (S + 1) * 20 + 6 * S * S, "mufu": S * S}
# what bounds the dominant kernel, from the committed ncu captures (profiles/)
LIMITERS = {
    "k_pc_step1": ("instruction issue: ~9.2 warp instructions per particle at 60 % issue active "
                   "(16 warps/SM at 120 registers), Philox + Box-Muller ~2.8 of them; DRAM "
                   "traffic ~= the algorithmic bytes (profiles/r5_c5s_ncu_summary.txt)"),
    "k_sys_resample": ("latency of pass 2 (u128 prefix -> slot -> run head chains, emission "
                       "stage): ~2.75 warp instructions per particle, 42 % issue active "
                       "(profiles/r5_c5s_ncu_summary.txt)"),
    "k_sir_propagate_lik": "FP32/SFU/XU pipes and latency of the per-pixel likelihood",
    "k_mt_frame": ("instruction issue and shared-atomic serialisation (step-1 machinery per "
                   "target, two CTAs per SM; replicated accumulators for compact clouds)"),
}


# ---------------------------------------------------------------------------
# synthetic inputs (BASELINE configs; the paper and reference use synthetic scenes)
# ---------------------------------------------------------------------------
def frames_for(width, count, start, seed=0):
    """One Gaussian spot (sigma 1.5 px, I0 20, bg 10) moving +0.5 px/frame
    along x (direction unstated in the configs), Poisson noise, seed 0."""
    rng = np.random.default_rng(seed)
    x, y = start
    out = np.empty((count, width, width), dtype=np.float32)
    truth = np.empty((count, 2))
    r = 12
    for k in range(count):
        x += 0.5
        ideal = np.full((width, width), 10.0)
        cx, cy = int(round(x)), int(round(y))
        xa, xb, ya, yb = max(cx - r, 0), min(cx + r + 1, width), max(cy - r, 0), min(cy + r + 1, width)
        gx = np.exp(-((np.arange(xa, xb) - x) ** 2) / (2 * 1.5 ** 2))
        gy = np.exp(-((np.arange(ya, yb) - y) ** 2) / (2 * 1.5 ** 2))
        ideal[ya:yb, xa:xb] += 20.0 * np.outer(gy, gx)
        out[k] = rng.poisson(ideal)
        truth[k] = (x, y)
    return out, truth


def scene(wl_name, wl, count, torch):
    """Frames of a single-spot workload: host numpy (c1, c2) or rendered on
    the GPU (c3, c5: 512^2 / 4096^2 frames, paper_1310_5541_b200.synthesis).
    Returns (device frames, host frames, truth positions (count, 2), source)."""
    if wl_name in ("c3", "c5"):
        from paper_1310_5541_b200 import synthesis as syn
        dev, truth = syn.spot_scene(count, wl["width"], wl["start"], seed=0)
        return dev, dev.cpu().numpy(), truth, "GPU Poisson synthesis (pcs_render_frames), seed 0"
    host, truth = frames_for(wl["width"], count, wl["start"])
    return torch.from_numpy(host).cuda(), host, truth, "host numpy Poisson, seed 0"


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
                self._stop.wait(0.1)
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


def bench_config(wl_name, wl, variant, world):
    """The workload-defining config dict, identical in both arms (results
    such as RMSE go under "quality", not here)."""
    cpp = VARIANTS[variant]
    n = wl["n"]
    if wl_name == "c4":
        return {"workload": f"c4:{variant}", "targets": wl["targets"],
                "n_particles_per_target": n, "frame": f"{wl['width']}x{wl['width']}",
                "frames": "4096 Gaussian spots (uniform positions, v~N(0,1), I0~U[10,40]), "
                          "bg 10, Poisson, seed 0",
                "bin_px": cpp, "likelihood": "gauss-ssd 11x11",
                "resampling": "systematic every frame (threshold 1.0)",
                "parallelism": f"targets sharded x{world}, no communication",
                "l2": "working set larger than L2"}
    working_set = STEP_BYTES * n
    lik = (f"{'gauss-ssd' if wl['model'] == 'gauss' else 'erf-poisson'}"
           f" {2 * wl['hw'] + 1}x{2 * wl['hw'] + 1}")
    if wl_name == "c5":
        par = (f"particles sharded x{world} (NCCL all-reduce / all-gather / all-to-all)"
               if world > 1 else "single GPU (one filter, fused device loop)")
    else:
        par = f"replicas x{world}" if world > 1 else "single GPU"
    return {"workload": f"{wl_name}:{variant}", "n_particles": n,
            "frame": f"{wl['width']}x{wl['width']}",
            "frames": "one Gaussian spot (sigma 1.5 px, I0 20, bg 10), +0.5 px/frame, Poisson, "
                      "seed 0",
            "bin_px": cpp, "likelihood": lik,
            "resampling": "systematic every frame (threshold 1.0)",
            "l2": ("flushed (write > L2) before every timed step" if working_set < 2 * L2_BYTES
                   else "working set larger than L2"),
            "parallelism": par}


def make_cfg(pc, wl, cpp, n=None, center=None):
    width = wl["width"]
    n = n or wl["n"]
    c = center if center is not None else (wl["start"][0], wl["start"][1], 0.5, 0.0, 20.0)
    init = pc.InitSpec(pc.StateVector(*c), "gauss", sigma=2.0)
    dyn = pc.DynamicsParams(0.5, 0.1, 1.0)
    if wl["model"] == "gauss":
        lik = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, wl["hw"]))
    else:
        lik = pc.PoissonSpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, wl["hw"]),
                                       "erf")
    res = pc.ResampleConfig(1.0, "systematic")
    if cpp is None:
        return pc.FilterConfig(n, init, dyn, res, lik), None
    cells = int(round(width / cpp))
    grid = pc.BinGrid(-0.5, -0.5, cpp, cpp, cells, cells)
    return pc.PcFilterConfig(n, init, dyn, res, lik, grid=grid), grid


def c_cfg(pc, _lib, cfg, grid, seed, use_graph=True):
    c = _lib.PcsTrackCfg()
    c.method = 0 if grid is None else 1
    c.placement = 0
    c.n_particles = cfg.n_particles
    c.init = cfg.init.to_c()
    c.dyn = cfg.dynamics.to_c()
    c.spot = cfg.likelihood.spot_c(cells=grid is not None)
    if grid is not None:
        c.grid = grid.to_c()
    c.seed = seed
    c.frame0 = 0
    c.use_graph = 1 if use_graph else 0
    return c


# ---------------------------------------------------------------------------
# single-filter workloads (c1, c2, c3, c5 on one GPU): fused device loop
# ---------------------------------------------------------------------------
def run_fused(torch, pc, _lib, cfg, grid, dev_frames, warmup, steps, seed, flush, sampler=None):
    """W warm-up frames, then K frames timed one graph replay at a time
    (optionally flushing L2 before each). Returns per-step ms and outputs."""
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
        if flush is not None:
            flush.zero_()                  # > L2: every timed step starts cold
        ev[i][0].record()
        step(warmup + i, warmup + i + 1)
        ev[i][1].record()
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    out = _lib.PcsTrackResult()
    _lib.check(_lib.lib().pcs_track_end(_lib.ctx(), ctypes.byref(out), st), "pcs_track_end")
    ms = [a.elapsed_time(b) for a, b in ev]
    return ms, dict(est=est.cpu().numpy(), ess=ess.cpu().numpy(), occ=occ.cpu().numpy(),
                    flags=int(out.flags), clocks=clocks,
                    launches=int(_lib.lib().pcs_track_launches_per_step(_lib.ctx())))


def measured_traffic(wl_name, variant, kernel, n):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture (profiles/traffic.json), scaled to
    this run's N when the capture used a smaller N; None if not captured."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as f:
            tab = json.load(f)
    except (OSError, ValueError):
        return None
    rec = tab.get(f"{wl_name}:{variant}", {}).get(kernel)
    if not rec:
        return None
    return rec["bytes_per_launch"] * n / rec["n"]


def kernel_profile(torch, pc, _lib, cfg, grid, dev_frames, warmup, frames_n, seed, flush):
    """Per-kernel device time (CUDA events on the launching stream, no graph)."""
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
        if flush is not None:
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


# measured pipe utilisation of k_sir_propagate_lik (ncu --set full, one launch;
# profiles/r2_sir_likelihood_ncu.txt): % of each pipe's peak while active
LIK_PIPES = {
    "c3": {"fma_pct": 59.2, "xu_pct": 47.5, "alu_pct": 30.8, "fp64_pct": 0.31,
           "issue_active_pct": 83.9, "measured_limiter": "FP32 FMA pipe / issue (two 256-thread "
           "CTAs per SM at 128 registers)"},
    "c2": {"fma_pct": 24.4, "xu_pct": 53.0, "alu_pct": 25.7, "fp64_pct": 11.2,
           "issue_active_pct": 57.9, "measured_limiter": "XU (expf + float->double "
           "conversions of the exact r^2 sums)"},
}


def likelihood_roofline(torch, pc, _lib, info, args, clock_mhz):
    """FP32 / SFU roofline of the per-particle likelihood kernel
    (k_sir_propagate_lik, one evaluation per particle): c3's erf-PSF Poisson
    15x15 at N=1e7 and c2's Gaussian SSD 11x11 at N=1e6, CUDA events around
    each launch (kernel_profile). Achieved = minimal operation count (SURVEY
    §8(d), lik_min_ops) x N / kernel time; peaks from the SM count and the SM
    clock sampled during the timed region: FP32 = SMs x 128 lanes x 2 FLOP x f,
    SFU = SMs x 16 MUFU x f. The kernel also gathers, draws and propagates (52 B
    per particle of HBM traffic), which the count leaves out."""
    f = (clock_mhz or 1965.0) * 1e6
    sms = info["sm_count"]
    peak_fp32 = sms * 128 * 2 * f
    peak_sfu = sms * 16 * f
    out = {}
    for wl_name in ("c3", "c2"):
        wl = dict(WORKLOADS[wl_name])
        frames_n = 4
        dev_frames, _, _, _ = scene(wl_name, wl, args.warmup + frames_n, torch)
        cfg, grid = make_cfg(pc, wl, None)
        prof = kernel_profile(torch, pc, _lib, cfg, grid, dev_frames, args.warmup, frames_n,
                              args.seed, None)
        ms = prof.get("k_sir_propagate_lik")
        ops = lik_min_ops(wl["model"], wl["hw"])
        n = wl["n"]
        t = ms * 1e-3
        flop_s, mufu_s = ops["flop"] * n / t, ops["mufu"] * n / t
        t_bound = max(ops["flop"] * n / peak_fp32, ops["mufu"] * n / peak_sfu)
        out[f"{wl_name}:SIR"] = {
            "bound": "fp32/sfu", "kernel": "k_sir_propagate_lik", "kernel_ms": round(ms, 5),
            "likelihood": ("erf-poisson 15x15" if wl["model"] != "gauss" else "gauss-ssd 11x11"),
            "n_evals": n, "min_flop_per_eval": ops["flop"], "min_mufu_per_eval": ops["mufu"],
            "achieved_tflops": flop_s / 1e12, "peak_fp32_tflops": peak_fp32 / 1e12,
            "fp32_frac": flop_s / peak_fp32,
            "achieved_mufu_per_s": mufu_s, "peak_mufu_per_s": peak_sfu, "sfu_frac": mufu_s / peak_sfu,
            "frac": t_bound / t, "limiter": "sfu" if ops["mufu"] / peak_sfu >= ops["flop"] / peak_fp32
            else "fp32",
            "clock_mhz": f / 1e6, "peak_kind": "SMs x lanes x clock (sampled)",
            "ncu_pipes": dict(LIK_PIPES[wl_name],
                              source="profiles/r2_sir_likelihood_ncu.txt")}
        del dev_frames
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# CPU reference path (oracle port of the reference driver + the reference's
# compiled likelihood kernel when oracle/_ref holds it)
# ---------------------------------------------------------------------------
def cpu_port_track(wl, n, frames, start, cpp):
    from oracle import pcsir_oracle as orc
    ssd = orc.reference_ssd_kernel()
    model = wl["model"]
    lik = orc.SpotModel(1.5, 10.0, 10.0, wl["hw"], model=model,
                        ssd=ssd if model == "gauss" else None)
    width = wl["width"]
    grid = None if cpp is None else (-0.5, -0.5, cpp, cpp, int(round(width / cpp)),
                                     int(round(width / cpp)))
    rng = np.random.default_rng(0)
    t0 = time.perf_counter()
    orc.track([f.astype(np.float64) for f in frames], n, [start[0], start[1], 0.5, 0.0, 20.0],
              2.0, [0.5, 0.5, 0.1, 0.1, 1.0], 1.0, lik, rng, grid=grid)
    dt = time.perf_counter() - t0
    kern = ("reference _speedups.pyx kernel (oracle/_ref)" if (ssd is not None and model == "gauss")
            else "oracle C likelihood")
    return n * len(frames) / dt, dt, kern


def _c4_cpu_worker(args):
    wl, n, frames, center, cpp = args
    v, dt, kern = cpu_port_track(wl, n, frames, center, cpp)
    return n * len(frames), dt, kern


def cpu_sample(wl_name, wl, frames_host, cpp, pool_cores=1):
    """A bounded sample (~10-30 s of CPU work) of the workload on this host."""
    if wl_name in ("c1", "c2"):
        nf = {"c1": 50, "c2": 40}[wl_name]   # c2: ~10 s on one core
        v, dt, kern = cpu_port_track(wl, wl["n"], frames_host[:nf], wl["start"], cpp)
        return v, 1, f"{nf} frames x N={wl['n']} ({kern}), {dt:.1f} s on 1 core"
    if wl_name in ("c3", "c5"):
        n = 1_000_000 if wl_name == "c3" else 1 << 23   # c5: ~8 s on one core
        v, dt, kern = cpu_port_track(wl, n, frames_host[:3], wl["start"], cpp)
        return v, 1, (f"3 frames x N={n} (1/{wl['n'] // n} of the config's N; particle-updates/s "
                      f"is per-particle so it scales with N) ({kern}), {dt:.1f} s on 1 core")
    # c4: independent targets -> process pool over the host cores
    frames, truth = frames_host
    nt = max(2, pool_cores)
    jobs = [(wl, wl["n"], frames[:3], (truth[t, 0, 0], truth[t, 0, 1]), cpp) for t in range(nt)]
    import multiprocessing as mp
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(pool_cores) as pool:
        out = pool.map(_c4_cpu_worker, jobs)
    dt = time.perf_counter() - t0
    tot = sum(o[0] for o in out)
    return tot / dt, pool_cores, (f"{nt} of {wl['targets']} targets x N={wl['n']} x 3 frames, "
                                  f"process pool of {pool_cores} ({out[0][2]}), {dt:.1f} s")


def scaling_of(wl_name):
    """c4 / c5 fix the total work (targets / particles) as GPUs are added;
    c1-c3 run one filter per GPU (replicas)."""
    return "strong" if wl_name in ("c4", "c5") else "weak"


def reference_arm(args, wl_name, wl, cpp):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    cores = len(os.sched_getaffinity(0))
    if wl_name == "c4":
        from paper_1310_5541_b200.multitarget import multi_target_scene
        fh = multi_target_scene(min(wl["targets"], 64), 4, wl["width"], seed=0)
        v, used, sample = cpu_sample(wl_name, wl, fh, cpp, pool_cores=cores)
    else:
        k_total = args.warmup + args.steps
        if wl_name in ("c1", "c2"):
            frames, _ = frames_for(wl["width"], k_total, wl["start"])
            t0 = time.perf_counter()
            v, dt, kern = cpu_port_track(wl, wl["n"], frames, wl["start"], cpp)
            used = 1
            sample = (f"{k_total} frames x N={wl['n']} (reference driver restated in oracle/, "
                      f"{kern}), {time.perf_counter() - t0:.1f} s")
        else:
            frames, _ = frames_for(wl["width"], 3, wl["start"])
            v, used, sample = cpu_sample(wl_name, wl, frames, cpp)
    line = {
        "impl": "reference", "metric": "particle-updates/sec per filter step",
        "value": v, "unit": "particle-updates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wl.get("targets", 1) * wl["n"] / v * 1e3,
        "higher_is_better": True, "scaling": scaling_of(wl_name), "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(wl_name, wl, args.variant or wl["variant"], args.gpus),
        "cpu_baseline": {"value": v, "unit": "particle-updates/s", "cores": used, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "particle-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default=None, choices=sorted(VARIANTS))
    ap.add_argument("--targets", type=int, default=None, help="c4: number of targets")
    ap.add_argument("--n", type=int, default=None, help="override particles (per target for c4)")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl_name = args.workload
    wl = dict(WORKLOADS[wl_name])
    if args.n:
        wl["n"] = args.n
    if args.targets:
        wl["targets"] = args.targets
    if args.steps is None:
        args.steps = {"c1": 50, "c2": 100, "c3": 20, "c4": 10, "c5": 10}[wl_name]
    variant = args.variant or wl["variant"]
    cpp_main = VARIANTS[variant]
    if args.impl == "reference":
        return reference_arm(args, wl_name, wl, cpp_main)

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

    from paper_1310_5541_b200.distributed import max_over_ranks

    info = _lib.device_info(local)
    peak, peak_kind = peaks()
    k_total = args.warmup + args.steps
    sampler = ClockSampler(local)
    extra = {}

    if wl_name == "c4":
        line = bench_c4(args, wl, cpp_main, world, rank, dist, torch, pc, _lib, sampler,
                        max_over_ranks, peak, peak_kind)
    elif wl_name == "c5" and world > 1:
        line = bench_c5_sharded(args, wl, cpp_main, world, rank, dist, torch, pc, _lib, sampler,
                                max_over_ranks, peak, peak_kind)
    else:
        n = wl["n"]
        dev_frames, frames_host, truth, frames_src = scene(wl_name, wl, k_total, torch)
        working_set = STEP_BYTES * n
        flush = None
        if working_set < 2 * info["l2_bytes"]:
            flush = torch.empty(int(max(2 * info["l2_bytes"], 256 << 20)) // 4,
                                dtype=torch.float32, device="cuda")
        cfg, grid = make_cfg(pc, wl, cpp_main)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ms, out = run_fused(torch, pc, _lib, cfg, grid, dev_frames, args.warmup, args.steps,
                            args.seed, flush, sampler)
        total_ms = max_over_ranks(float(np.sum(ms)))
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        value = n * args.steps * world / (total_ms * 1e-3)
        step_ms = total_ms / args.steps
        rmse = float(np.sqrt(np.mean(np.sum((out["est"][args.warmup:, :2]
                                             - truth[args.warmup:]) ** 2, axis=1))))
        cfg, grid = make_cfg(pc, wl, cpp_main)
        kprof = kernel_profile(torch, pc, _lib, cfg, grid, dev_frames, args.warmup,
                               min(args.steps, 10), args.seed, flush)
        dom = max(kprof, key=kprof.get)
        key = dom if dom != "k_sys_resample" else ("k_sys_resample:pc" if cpp_main else "k_sys_resample:sir")
        dom_bytes = ALGO_BYTES.get(key, 0) * n
        achieved = dom_bytes / (kprof[dom] * 1e-3) / 1e9 if kprof[dom] > 0 else 0.0
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                    "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": measured_traffic(wl_name, variant, dom, n),
                    "algo_bytes_per_launch": dom_bytes,
                    "kernel_ms": {k: round(v, 5) for k, v in kprof.items()},
                    "kernel_share": {k: round(v / sum(kprof.values()), 4)
                                     for k, v in kprof.items()},
                    "step_bytes_per_particle": STEP_BYTES,
                    "step_achieved_gbs": STEP_BYTES * n / (step_ms * 1e-3) / 1e9,
                    "step_frac": STEP_BYTES * n / (step_ms * 1e-3) / 1e9 / peak,
                    "working_set_mb": round(working_set / 1e6, 1),
                    "l2_mb": round(info["l2_bytes"] / 2 ** 20, 1),
                    "limiter": LIMITERS.get(dom, ""),
                    "note": ("kernel times from a non-graph pass with CUDA events around every "
                             "launch (include ~5 us launch gaps); the headline is graph replay")}
        # e2e: the public call on host frames (H2D + D2H inside the timed region).
        # The frames sit in pinned host memory (a (K,H,W) float32 tensor, as a
        # camera/loader pipeline would hand them over); the call uploads them,
        # runs the filter and downloads estimates / ESS / resampled flags.
        track = pc.pcsir_track if cpp_main is not None else pc.sir_track
        warm = torch.from_numpy(np.ascontiguousarray(frames_host[:args.warmup],
                                                     dtype=np.float32)).pin_memory()
        cfg_e, _ = make_cfg(pc, wl, cpp_main)
        track(warm, cfg_e, pc.PhiloxRng(args.seed))
        e_frames = torch.from_numpy(np.ascontiguousarray(frames_host[args.warmup:k_total],
                                                         dtype=np.float32)).pin_memory()
        e_runs = []
        for _ in range(3):   # median of three whole calls
            cfg_e, _ = make_cfg(pc, wl, cpp_main)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = track(e_frames, cfg_e, pc.PhiloxRng(args.seed))
            torch.cuda.synchronize()
            e_runs.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(float(np.median(e_runs)))
        e2e = {"value": n * args.steps * world / e2e_s, "unit": "particle-updates/s",
               "h2d_bytes_per_step": int(wl["width"] * wl["width"] * 4),
               "d2h_bytes_per_step": 5 * 8 + 8 + 1 + 8, "path": r.path,
               "note": "pcsir_track/sir_track on a pinned (K,H,W) float32 host tensor: wall "
                       "time incl. frame upload (chunks on a side stream overlapping the "
                       "filter), particle init, graph capture and result download; median "
                       "of 3 calls"}
        variants = {}
        if not args.no_variants:
            for name in OTHER_VARIANTS.get(wl_name, []):
                cfg_v, grid_v = make_cfg(pc, wl, VARIANTS[name])
                vsteps = min(args.steps, 20)
                vms, vout = run_fused(torch, pc, _lib, cfg_v, grid_v, dev_frames, args.warmup,
                                      vsteps, args.seed, flush)
                vt = max_over_ranks(float(np.sum(vms)))
                variants[name] = {"value": n * vsteps * world / (vt * 1e-3),
                                  "ms_per_step": vt / vsteps,
                                  "mean_occupied_bins": float(np.mean(vout["occ"][args.warmup:]))}
        lik_roof = None
        if wl_name == "c5" and not args.no_variants:
            del dev_frames
            torch.cuda.empty_cache()
            lik_roof = likelihood_roofline(torch, pc, _lib, info, args,
                                           (out["clocks"] or {}).get("sm_mhz"))
        cpu = None
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            v, used, sample = cpu_sample(wl_name, wl, frames_host, cpp_main)
            cpu = {"value": v, "unit": "particle-updates/s", "cores": used, "kind": "port",
                   "sample": sample + "; reference driver restated in oracle/"}
        line = {
            "metric": "particle-updates/sec per filter step", "value": value,
            "unit": "particle-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": scaling_of(wl_name), "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": bench_config(wl_name, wl, variant, world),
            "quality": {"rmse_px": rmse, "frames_source": frames_src,
                        "mean_occupied_bins": float(np.mean(out["occ"][args.warmup:]))},
            "roofline": roofline, "likelihood_roofline": lik_roof, "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": out["launches"] * args.steps,
            "clocks": out["clocks"], "variants": variants, "flags": out["flags"],
        }
    if rank == 0 and line is not None:
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def bench_c4(args, wl, cpp, world, rank, dist, torch, pc, _lib, sampler, max_over_ranks, peak,
             peak_kind):
    """Config 4: T targets, targets partitioned over ranks (no communication)."""
    from paper_1310_5541_b200 import multitarget as mt
    T = wl["targets"]
    k_total = args.warmup + args.steps
    from paper_1310_5541_b200 import synthesis as syn
    dev_frames, truth = syn.multi_target_scene_device(T, k_total, wl["width"], seed=0)
    frames_host = dev_frames.cpu().numpy()
    lo, hi = mt.target_range(T, rank, world)
    n = wl["n"]
    cfg, _ = make_cfg(pc, wl, cpp, n=n, center=(0, 0, 0, 0, 20.0))
    tr = mt.MultiTargetTracker(cfg, truth[lo:hi, 0], args.seed, k_total, wl["width"],
                               wl["width"], target_offset=lo)
    for k in range(args.warmup):
        tr.step(dev_frames[k])
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sampler.start()
    for i in range(args.steps):
        ev[i][0].record()
        tr.step(dev_frames[args.warmup + i])
        ev[i][1].record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = float(np.sum([a.elapsed_time(b) for a, b in ev]))
    total_ms = max_over_ranks(ms)
    res = tr.results()
    value = T * n * args.steps / (total_ms * 1e-3)
    step_ms = total_ms / args.steps
    local_particles = (hi - lo) * n
    achieved = ALGO_BYTES["k_mt_frame"] * local_particles / (ms / args.steps * 1e-3) / 1e9
    d = np.sqrt(np.sum((res.estimates[:, args.warmup:, :2]
                        - truth[lo:hi, 1 + args.warmup:, :2]) ** 2, axis=2))
    err = float(np.sqrt(np.mean(d ** 2)))
    err_median = float(np.median(d))
    lost = float(np.mean(d[:, -1] > 2.0))   # dim (I0 ~ 10 on bg 10) or fast (|v| > 2) spots
    # e2e: the public call on pinned host frames (upload inside the timed region)
    e_frames = torch.from_numpy(np.ascontiguousarray(frames_host[:args.steps],
                                                     dtype=np.float32)).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = mt.multi_pcsir_track(e_frames, cfg, truth[lo:hi, 0], args.seed, target_offset=lo)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        v, used, sample = cpu_sample("c4", wl, (frames_host, truth), cpp, pool_cores=cores)
        cpu = {"value": v, "unit": "particle-updates/s", "cores": used, "kind": "port",
               "sample": sample}
    return {
        "metric": "particle-updates/sec per filter step", "value": value,
        "unit": "particle-updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config("c4", wl, args.variant or wl["variant"], world),
        "quality": {"rmse_px": err, "median_err_px": err_median, "lost_target_frac": lost},
        "roofline": {"bound": "hbm", "kernel": "k_mt_frame", "limiter": LIMITERS["k_mt_frame"],
                     "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None,
                     "algo_bytes_per_launch": ALGO_BYTES["k_mt_frame"] * local_particles},
        "cpu_baseline": cpu,
        "e2e": {"value": T * n * args.steps / e2e_s, "unit": "particle-updates/s",
                "h2d_bytes_per_step": int(wl["width"] ** 2 * 4),
                "d2h_bytes_per_step": int((hi - lo) * (5 * 8 + 8 + 1 + 8)), "path": "multi"},
        "gpu_launches": args.steps, "clocks": clocks,
        "flags_nonzero_targets": int(np.count_nonzero(res.flags)),
    }


def bench_c5_sharded(args, wl, cpp, world, rank, dist, torch, pc, _lib, sampler, max_over_ranks,
                     peak, peak_kind):
    """Config 5 over >1 GPU: one filter sharded by particle (distributed.py,
    pcs_shard.cuh). The protocol has no host synchronisation inside the frame
    loop, so the K timed frames are bracketed by CUDA events on the stream
    (max over ranks); e2e uploads pinned host frames inside its timed region."""
    from paper_1310_5541_b200 import distributed as D
    k_total = args.warmup + args.steps
    dev_frames, frames_host, truth, _ = scene("c5", wl, k_total, torch)
    cfg, _ = make_cfg(pc, wl, cpp)
    ops = D.DeviceShardOps(k_total)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    orig_step1, orig_flags = ops.step1, ops.flags

    def step1(frame, k):
        if k == args.warmup:
            ev0.record()
        return orig_step1(frame, k)

    def flags():
        ev1.record()
        return orig_flags()

    ops.step1, ops.flags = step1, flags
    dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    est, ess, res, evals = D.sharded_pcsir_track(dev_frames, cfg, args.seed, ops)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    elapsed = max_over_ranks(ev0.elapsed_time(ev1) * 1e-3)
    n = wl["n"]
    value = n * args.steps / elapsed
    # e2e: pinned host frames -> device inside the timed region, host outputs
    host = torch.from_numpy(np.ascontiguousarray(frames_host[:args.steps])).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D.sharded_pcsir_track(host.cuda(non_blocking=True), make_cfg(pc, wl, cpp)[0], args.seed,
                          D.DeviceShardOps(args.steps))
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    rmse = float(np.sqrt(np.mean(np.sum((est[args.warmup:, :2] - truth[args.warmup:]) ** 2,
                                        axis=1))))
    return {
        "metric": "particle-updates/sec per filter step", "value": value,
        "unit": "particle-updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": bench_config("c5", wl, args.variant or wl["variant"], world),
        "quality": {"rmse_px": rmse},
        "timing": "CUDA events on the stream around the K timed frames, max over ranks (no "
                  "host synchronisation inside the sharded frame loop)",
        "roofline": None, "cpu_baseline": None,
        "e2e": {"value": n * args.steps / e2e_s, "unit": "particle-updates/s",
                "h2d_bytes_per_step": int(wl["width"] ** 2 * 4),
                "d2h_bytes_per_step": 5 * 8 + 8 + 1 + 8,
                "note": "sharded_pcsir_track on pinned host frames (upload, init, K frames, "
                        "result download), wall clock, max over ranks"},
        "gpu_launches": None, "clocks": clocks,
    }


if __name__ == "__main__":
    sys.exit(main())
