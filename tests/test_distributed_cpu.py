"""The sharded giant-filter orchestration (config 5) on CPU with gloo: the
results for 2 ranks equal those for 1 rank bit for bit (exact limb
all-reduce, exact rank prefixes, global-index Philox), plus unit checks of
the slot-range / exchange planning."""

import os
import pathlib
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = pathlib.Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _scene(k=5, width=48, seed=0):
    rng = np.random.default_rng(seed)
    xs = np.arange(width)
    frames = []
    x, y = 20.0, 24.0
    for _ in range(k):
        x += 0.5
        gx = np.exp(-((xs - x) ** 2) / (2 * 1.5 ** 2))
        gy = np.exp(-((xs - y) ** 2) / (2 * 1.5 ** 2))
        frames.append(rng.poisson(20.0 * np.outer(gy, gx) + 10.0).astype(np.float32))
    return np.stack(frames)


def _run(rank, world, port, n, cpp, out_dir, bcap=None, res=(1.0, "systematic")):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1310_5541_b200 as pc
    from paper_1310_5541_b200 import distributed as D
    from shard_cpu_ops import CpuShardOps

    frames = _scene()
    cfg = pc.PcFilterConfig(n, pc.InitSpec(pc.StateVector(20.0, 24.0, 0.5, 0.0, 20.0), "gauss",
                                           sigma=2.0),
                            pc.DynamicsParams(0.5, 0.1, 1.0), pc.ResampleConfig(*res),
                            likelihood=object(), grid=pc.BinGrid.pixel_aligned(48, 48, cpp))
    ops = CpuShardOps(len(frames), frames)
    try:
        est, ess, res, evals = D.sharded_pcsir_track(torch.from_numpy(frames), cfg, 1234, ops,
                                                     wcap=4096, bcap=bcap)
    except Exception as err:   # every rank must raise the same error
        np.savez(os.path.join(out_dir, f"err_w{world}_r{rank}.npz"), kind=type(err).__name__)
        dist.barrier()
        dist.destroy_process_group()
        return
    if rank == 0:
        np.savez(os.path.join(out_dir, f"w{world}.npz"), est=est, ess=ess, res=res, evals=evals)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cpp", [1, 2])
def test_ranks_equal_one_rank(tmp_path, cpp):
    """P = 2 and P = 4 reproduce P = 1 bit for bit: the exact limb all-reduce,
    the exact rank prefixes and the boundary exchange with the neighbours."""
    n = 1200
    for world in (1, 2, 4):
        mp.spawn(_run, args=(world, _free_port(), n, cpp, str(tmp_path)), nprocs=world, join=True)
    a = np.load(tmp_path / "w1.npz")
    for world in (2, 4):
        b = np.load(tmp_path / f"w{world}.npz")
        assert np.array_equal(a["est"], b["est"])
        assert np.array_equal(a["ess"], b["ess"])
        assert np.array_equal(a["res"], b["res"])
        assert int(a["evals"]) == int(b["evals"])
    assert a["res"].all()
    truth_x = 20.0 + 0.5 * np.arange(1, 6)
    assert np.max(np.abs(a["est"][:, 0] - truth_x)) < 1.0


@pytest.mark.parametrize("frac,scheme,cpp", [(0.5, "systematic", 1), (1.0, "multinomial", 2),
                                              (0.5, "multinomial", 1)])
def test_ranks_equal_one_rank_threshold_multinomial(tmp_path, frac, scheme, cpp):
    """ESS-threshold frames (prior weights finished per particle through the
    MAX / SUM all-reduces) and multinomial resampling (requests and states
    through the two all-to-alls): P = 2 and P = 4 reproduce P = 1 bit for bit."""
    n = 1200
    for world in (1, 2, 4):
        mp.spawn(_run, args=(world, _free_port(), n, cpp, str(tmp_path), None, (frac, scheme)),
                 nprocs=world, join=True)
    a = np.load(tmp_path / "w1.npz")
    if frac < 1.0:
        assert 0 < int(a["res"].sum()) < len(a["res"])   # both kinds of frames occur
    for world in (2, 4):
        b = np.load(tmp_path / f"w{world}.npz")
        assert np.array_equal(a["est"], b["est"])
        assert np.array_equal(a["ess"], b["ess"])
        assert np.array_equal(a["res"], b["res"])
        assert int(a["evals"]) == int(b["evals"])
    truth_x = 20.0 + 0.5 * np.arange(1, 6)
    assert np.max(np.abs(a["est"][:, 0] - truth_x)) < 1.0


def test_capacity_error_raised_on_every_rank(tmp_path):
    """A boundary buffer too small for the slots a rank must hand to its
    neighbour: the check is evaluated identically on every rank (same
    gathered totals) and the flags are all-reduced, so all ranks raise."""
    world = 4
    mp.spawn(_run, args=(world, _free_port(), 1200, 1, str(tmp_path), 1), nprocs=world, join=True)
    kinds = [str(np.load(tmp_path / f"err_w{world}_r{r}.npz")["kind"]) for r in range(world)]
    assert kinds == ["CapacityError"] * world


def test_slot_ranges_and_plan():
    from paper_1310_5541_b200 import distributed as D
    # 3 ranks x 4 particles, weights concentrated on rank 1
    n_global, p = 12, 3
    one = 1 << 120
    totals = [one // 8, one // 2, one - one // 8 - one // 2]
    ranges, prefixes = D.slot_ranges(totals, 0.3, n_global, True)
    assert ranges[0][0] == 0 and ranges[-1][1] == n_global
    assert all(ranges[r][1] == ranges[r + 1][0] for r in range(p - 1))
    assert prefixes == [0, one // 8, one // 8 + one // 2]
    plan = D.exchange_plan(ranges, n_global, p)
    # every destination receives exactly n_local slots
    for q in range(p):
        assert sum(plan[r][q][1] for r in range(p)) == n_global // p
    # no resampling: identity ranges
    ranges, _ = D.slot_ranges(totals, 0.3, n_global, False)
    assert ranges == [(0, 4), (4, 8), (8, 12)]


def test_first_slot_matches_points():
    from paper_1310_5541_b200 import distributed as D
    rng = np.random.default_rng(0)
    n = 1000
    u = float(rng.random())
    pts = (u + np.arange(n)) / n
    for c in list(rng.random(200)) + [0.0, 1.0, pts[5], pts[999]]:
        j = D.first_slot(float(c), u, n)
        assert j == int(np.searchsorted(pts, c, side="left"))

