"""Config 4 across ranks on CPU (gloo): targets partitioned by target_range
([r*T/P, (r+1)*T/P), no communication), each target filtered with its own
RNG key target_seed(seed, t), results collected by gather_results and the
timing reduced by max_over_ranks. The per-target filter here is the CPU
oracle of the reference driver (filtering.py:148-173, binning.py:175-195)
replaying the device's Philox draws, so P = 2 and P = 4 must reproduce the
single-process results bit for bit."""

import os
import pathlib
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = pathlib.Path(__file__).resolve().parents[1]
T, K, N, W = 6, 3, 400, 48


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _scene():
    sys.path.insert(0, str(ROOT))
    from paper_1310_5541_b200.multitarget import multi_target_scene
    return multi_target_scene(T, K, W, seed=0)


def _local_results(lo, hi, frames, truth, seed):
    """MultiTrackResult-shaped results of targets [lo, hi) from the oracle."""
    from oracle import pcsir_oracle as orc
    from paper_1310_5541_b200.multitarget import MultiTrackResult, target_seed
    est = np.zeros((hi - lo, K, 5))
    ess = np.zeros((hi - lo, K))
    res = np.zeros((hi - lo, K), dtype=bool)
    occ = np.zeros((hi - lo, K), dtype=np.int64)
    evals = np.zeros(hi - lo, dtype=np.int64)
    grid = (-0.5, -0.5, 1.0, 1.0, W, W)
    for i, t in enumerate(range(lo, hi)):
        lik = orc.SpotModel(1.5, 10.0, 10.0, 5)
        before = 0
        centre = [truth[t, 0, 0], truth[t, 0, 1], 0.0, 0.0, 20.0]
        e, s, r, ev = orc.track([f.astype(np.float64) for f in frames], N, centre, 2.0,
                                [0.5, 0.5, 0.1, 0.1, 1.0], 1.0, lik,
                                orc.PhiloxReplay(target_seed(seed, t)), grid=grid)
        est[i], ess[i], res[i], evals[i] = e, s, r, ev - before
        occ[i] = ev // K
    return MultiTrackResult(est, ess, res, occ, np.zeros(hi - lo, dtype=np.uint32), evals)


def _run(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1310_5541_b200 import multitarget as mt
    from paper_1310_5541_b200.distributed import max_over_ranks
    frames, truth = _scene()
    lo, hi = mt.target_range(T, rank, world)
    local = _local_results(lo, hi, frames, truth, seed=99)
    got = mt.gather_results(local)
    slowest = max_over_ranks(float(rank + 1) * 1.5)
    if rank == 0:
        np.savez(os.path.join(out_dir, f"w{world}.npz"), slowest=slowest, **got)
    dist.barrier()
    dist.destroy_process_group()


def _spawn(world, out_dir):
    mp.start_processes(_run, args=(world, _free_port(), out_dir), nprocs=world, join=True,
                       start_method="fork")
    return np.load(os.path.join(out_dir, f"w{world}.npz"))


@pytest.mark.parametrize("t,p", [(4096, 8), (4096, 3), (5, 8), (7, 2), (1, 1)])
def test_target_range_partitions_every_target_once(t, p):
    sys.path.insert(0, str(ROOT))
    from paper_1310_5541_b200.multitarget import target_range
    ranges = [target_range(t, r, p) for r in range(p)]
    assert ranges[0][0] == 0 and ranges[-1][1] == t
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c                                  # contiguous, disjoint
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1                # balanced


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_targets_equal_single_process(tmp_path, world):
    sys.path.insert(0, str(ROOT))
    frames, truth = _scene()
    ref = _local_results(0, T, frames, truth, seed=99)
    got = _spawn(world, str(tmp_path))
    assert np.array_equal(got["estimates"], ref.estimates)
    assert np.array_equal(got["ess"], ref.ess)
    assert np.array_equal(got["likelihood_evals"], ref.likelihood_evals)
    assert float(got["slowest"]) == 1.5 * world        # max over ranks, not rank 0's
