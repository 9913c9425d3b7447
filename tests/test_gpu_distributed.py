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


@pytest.mark.parametrize("cpp,n", [(1, 20000), (4, 50000)])
def test_sharded_world1_equals_fused(group, cpp, n):
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
        return pc.PcFilterConfig(n, init, dyn, pc.ResampleConfig(1.0, "systematic"),
                                 pc.SpotLikelihood(pc.PsfParams(1.5, 10.0),
                                                   pc.LikelihoodParams(10.0, 5)), grid=grid)

    fused = pc.pcsir_track([pc.ImageFrame(f) for f in frames], cfg(), pc.PhiloxRng(77))
    assert fused.path == "fused"
    ops = D.DeviceShardOps(k)
    est, ess, res, evals = D.sharded_pcsir_track(torch.from_numpy(frames).cuda(), cfg(), 77, ops,
                                                 group=group)
    assert np.array_equal(est, fused.estimates)
    assert np.array_equal(ess, fused.ess)
    assert np.array_equal(res, fused.resampled)
    assert evals == fused.likelihood_evals
