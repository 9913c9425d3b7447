"""Device side of the sharded giant filter (config 5) on one B200: a world of
one rank through the full sharded protocol (limb export/all-reduce/import,
rank-prefix scan, slot emission, all-to-all, state install) reproduces the
fused single-GPU filter bit for bit. (Multi-rank equality is covered on CPU
by tests/test_distributed_cpu.py; only one GPU is available per run.)"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import distributed as D

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def group(cuda):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("cpp,n,res", [(1, 20000, (1.0, "systematic")), (4, 50000, (1.0, "systematic")),
                                       (1, 20000, (0.5, "systematic")),
                                       (2, 20000, (0.25, "multinomial"))])
def test_sharded_world1_equals_fused(group, cpp, n, res):
    rng = np.random.default_rng(5)
    width, k = 96, 8
    xs = np.arange(width)
    frames = []
    x, y = 40.0, 45.0
    for _ in range(k):
        x += 0.5
        ideal = 20.0 * np.outer(np.exp(-((xs - y) ** 2) / 4.5), np.exp(-((xs - x) ** 2) / 4.5)) + 10
        frames.append(rng.poisson(ideal).astype(np.float32))
    frames = np.stack(frames)
    init = pc.InitSpec(pc.StateVector(40.0, 45.0, 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    dyn = pc.DynamicsParams(0.5, 0.1, 1.0)
    grid = pc.BinGrid.pixel_aligned(width, width, cpp)

    def cfg():
        return pc.PcFilterConfig(n, init, dyn, pc.ResampleConfig(*res),
                                 pc.SpotLikelihood(pc.PsfParams(1.5, 10.0),
                                                   pc.LikelihoodParams(10.0, 5)), grid=grid)

    fused = pc.pcsir_track([pc.ImageFrame(f) for f in frames], cfg(), pc.PhiloxRng(77))
    assert fused.path == "fused"
    if res[0] < 1.0:
        assert 0 < int(fused.resampled.sum()) < k   # both kinds of frames occur
    ops = D.DeviceShardOps(k)
    est, ess, res, evals = D.sharded_pcsir_track(torch.from_numpy(frames).cuda(), cfg(), 77, ops,
                                                 group=group)
    assert np.array_equal(est, fused.estimates)
    assert np.array_equal(ess, fused.ess)
    assert np.array_equal(res, fused.resampled)
    assert evals == fused.likelihood_evals


def _emulated_ranks(frames, cfg, seed, world, wcap=1 << 14, bcap=None):
    """The sharded protocol for `world` ranks run one after another on this
    GPU, one pcs_ctx per rank, the collectives done as tensor ops between the
    ranks' launches (nothing waits on another rank's kernel: every exchange
    is complete before the next call) — exercises the multi-rank device
    kernels (window export / import, rank totals, slot ranges, boundary
    pack / unpack) with a single B200."""
    from dataclasses import replace
    from paper_1310_5541_b200 import _lib
    n_global = cfg.n_particles
    n = n_global // world
    multi = cfg.resampling.scheme == "multinomial"
    cond = cfg.resampling.threshold_fraction < 1.0
    bcap = bcap or D.default_bcap(n, world, multi)
    k_frames, h, w = frames.shape
    ops = [D.DeviceShardOps(k_frames, _lib.new_ctx()) for _ in range(world)]
    for r, o in enumerate(ops):
        o.begin(replace(cfg, n_particles=n), h, w, r, world, n_global, wcap, bcap, seed)
    for k in range(k_frames):
        boxes = [o.step1(frames[k], k).clone() for o in ops]
        box = torch.stack(boxes).max(dim=0).values
        limbs = torch.stack([o.export(box).clone() for o in ops]).sum(dim=0)
        for o in ops:
            o.import_bins(box, limbs)
        if cond:
            mx = torch.stack([o.prior(0)[0].clone() for o in ops]).max(dim=0).values
            s3 = torch.stack([o.prior(1, mx)[0].clone() for o in ops]).sum(dim=0)
            outs = [tuple(t.clone() for t in o.prior(2, s3)) for o in ops]
            st = torch.stack([a for a, _ in outs]).sum(dim=0)
            mm = torch.stack([b for _, b in outs]).max(dim=0).values
            for o in ops:
                o.prior(3, st, mm)
        totals = torch.cat([o.total().clone() for o in ops])
        if multi:   # all-to-all: chunk q of rank r's buffer goes to rank q
            reqs = [o.route(totals).clone().view(world, -1) for o in ops]
            resps = [o.serve(torch.stack([reqs[q][r] for q in range(world)]).reshape(-1)).clone()
                     .view(world, -1) for r, o in enumerate(ops)]
            for r, o in enumerate(ops):
                o.install(torch.stack([resps[q][r] for q in range(world)]).reshape(-1))
            continue
        sends = [tuple(t.clone() for t in o.emit(totals)) for o in ops]
        for r, o in enumerate(ops):
            rp = sends[r - 1][1] if r > 0 else torch.zeros_like(sends[r][0])
            rn = sends[r + 1][0] if r < world - 1 else torch.zeros_like(sends[r][1])
            o.unpack(rp, rn)
    flags = [o.flags()[0] for o in ops]
    outs = [o.outputs() for o in ops]
    return flags, outs


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cpp,res", [(1, (1.0, "systematic")), (4, (1.0, "systematic")),
                                     (1, (0.5, "systematic")), (4, (0.3, "systematic")),
                                     (2, (1.0, "multinomial")), (4, (0.25, "multinomial"))])
def test_sharded_device_kernels_multi_rank_equal_fused(cuda, world, cpp, res):
    rng = np.random.default_rng(7)
    width, k, n = 96, 8, 40000
    xs = np.arange(width)
    frames = []
    x, y = 40.0, 45.0
    for _ in range(k):
        x += 0.5
        ideal = 20.0 * np.outer(np.exp(-((xs - y) ** 2) / 4.5), np.exp(-((xs - x) ** 2) / 4.5)) + 10
        frames.append(rng.poisson(ideal).astype(np.float32))
    frames = np.stack(frames)
    init = pc.InitSpec(pc.StateVector(40.0, 45.0, 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    dyn = pc.DynamicsParams(0.5, 0.1, 1.0)
    grid = pc.BinGrid.pixel_aligned(width, width, cpp)

    def cfg():
        return pc.PcFilterConfig(n, init, dyn, pc.ResampleConfig(*res),
                                 pc.SpotLikelihood(pc.PsfParams(1.5, 10.0),
                                                   pc.LikelihoodParams(10.0, 5)), grid=grid)

    fused = pc.pcsir_track([pc.ImageFrame(f) for f in frames], cfg(), pc.PhiloxRng(77))
    assert fused.path == "fused"
    if res[0] < 1.0:
        assert 0 < int(fused.resampled.sum()) < k   # both kinds of frames occur
    flags, outs = _emulated_ranks(torch.from_numpy(frames).cuda(), cfg(), 77, world)
    assert flags == [0] * world
    for est, ess, res, occ in outs:   # every rank holds the same results
        assert np.array_equal(est, fused.estimates)
        assert np.array_equal(ess, fused.ess)
        assert np.array_equal(res, fused.resampled)
        assert int(np.sum(occ)) == fused.likelihood_evals


def test_sharded_device_capacity_flag_on_every_rank(cuda):
    rng = np.random.default_rng(8)
    frames = torch.from_numpy(rng.poisson(12.0, size=(3, 48, 48)).astype(np.float32)).cuda()
    init = pc.InitSpec(pc.StateVector(20.0, 24.0, 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    cfg = pc.PcFilterConfig(4000, init, pc.DynamicsParams(0.5, 0.1, 1.0),
                            pc.ResampleConfig(1.0, "systematic"),
                            pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5)),
                            grid=pc.BinGrid.pixel_aligned(48, 48, 1))
    flags, _ = _emulated_ranks(frames, cfg, 5, 4, bcap=1)   # one-slot boundary buffers
    assert all(f & 4 for f in flags)                          # PCS_FLAG_CAPACITY on every rank
