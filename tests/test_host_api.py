"""Host-side logic of the drop-in API (validation, window convention, RNG
handles, reference inline known answers) — CPU only. The product path must
fail loudly without a GPU."""

import numpy as np
import pytest
import torch

import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import binning, imaging, kernels, rng as prng


def test_config_validation():
    with pytest.raises(ValueError):
        pc.BinGrid(0, 0, 0.0, 1.0, 4, 4)
    with pytest.raises(ValueError):
        pc.BinGrid(0, 0, 1.0, 1.0, 0, 4)
    with pytest.raises(ValueError):
        pc.DynamicsParams(-1.0)
    with pytest.raises(ValueError):
        pc.DynamicsParams(dt=0.0)
    with pytest.raises(ValueError):
        pc.InitSpec(pc.StateVector(0, 0, 0, 0, 1), "bogus")
    with pytest.raises(ValueError):
        pc.InitSpec(pc.StateVector(0, 0, 0, 0, 1), "uniform")
    with pytest.raises(ValueError):
        pc.InitSpec(pc.StateVector(0, 0, 0, 0, 1), "gauss")
    with pytest.raises(ValueError):
        pc.ResampleConfig(threshold_fraction=0.0)
    with pytest.raises(ValueError):
        pc.ResampleConfig(scheme="stratified")
    with pytest.raises(ValueError):
        pc.LikelihoodParams(0.0, 4)
    with pytest.raises(ValueError):
        pc.LikelihoodParams(1.0, -1)
    with pytest.raises(ValueError):
        pc.PsfParams(0.0)
    with pytest.raises(ValueError):
        pc.StateVector(0, 0, 0, 0, -1.0)
    with pytest.raises(ValueError):
        pc.Particle(pc.StateVector(0, 0, 0, 0, 1), float("nan"))
    with pytest.raises(ValueError):
        pc.PoissonSpotLikelihood(pc.PsfParams(1.5, 0.0), pc.LikelihoodParams(10.0, 7))


def test_filter_config_validation():
    init = pc.InitSpec(pc.StateVector(0, 0, 0, 0, 1))
    with pytest.raises(ValueError):
        pc.FilterConfig(0, init, likelihood=object())
    with pytest.raises(ValueError):
        pc.FilterConfig(10, init)
    with pytest.raises(ValueError):
        pc.PcFilterConfig(10, init, likelihood=object())


def test_pixel_grid_known_answers():
    grid = pc.BinGrid.pixel_aligned(512, 512, 1)
    assert grid.cell_indices(10.0, 20.0) == (10, 20)
    assert grid.cell_indices(10.49, 20.49) == (10, 20)
    assert grid.cell_indices(10.5, 20.5) == (11, 21)
    assert grid.cell_center(10, 20) == (10.0, 20.0)
    g2 = pc.BinGrid.pixel_aligned(512, 512, 2)
    assert g2.cell_width == 0.5 and g2.n_cols == 1024
    assert g2.cell_indices(-0.3, -0.3) == (0, 0)
    assert g2.cell_indices(0.3, -0.3) == (1, 0)


def test_window_convention_known_answers():
    small = pc.ImageFrame(np.zeros((512, 512)))
    assert imaging.window_pixel_count(small, 100.2, 340.9, 4) == 81
    assert imaging.window_pixel_count(small, 100.2, 340.9, 32) == 65 * 65
    frame = pc.ImageFrame(np.zeros((32, 32)))
    assert imaging.window_pixel_count(frame, 0.0, 0.0, 4) == 25
    assert imaging.window_pixel_count(frame, -50.0, 16.0, 4) == 9
    assert imaging.window_pixel_count(frame, 1000.0, 1000.0, 4) == 1
    assert pc.default_halfwidth(1.16) == 4
    assert pc.default_halfwidth(13.0) == 39


def test_make_dummy_rejects_empty_before_any_device_work():
    with pytest.raises(ValueError):
        pc.make_dummy([], (0, 1, 0, 1), pc.DummyPlacement.CENTER_OF_MASS)


def test_render_object_known_answers():
    import math
    assert pc.render_object((5.0, 7.0), 20.0, pc.PsfParams(1.16, 3.0), (5.0, 7.0)) == 23.0
    v = pc.render_object((0.0, 0.0), 10.0, pc.PsfParams(2.0, 1.0), (2.0, 0.0))
    assert v == pytest.approx(10.0 * math.exp(-0.5) + 1.0, rel=1e-15)


def test_single_backend_only():
    assert kernels.available_backends() == ["cuda"]
    assert kernels.set_backend("auto") == "cuda"
    with pytest.raises(ValueError):
        kernels.set_backend("python")


def test_rng_handles():
    r = prng.as_philox(np.random.default_rng(42))
    r2 = prng.as_philox(np.random.default_rng(42))
    assert r.seed == r2.seed
    assert prng.as_philox(r) is r
    assert prng.as_philox(7).seed == 7
    f0 = r.next_frame()
    assert r.next_frame() == f0 + 1
    with pytest.raises(TypeError):
        prng.as_philox("seed")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_product_path_fails_loudly_without_gpu():
    with pytest.raises(RuntimeError, match="CUDA"):
        pc.init_particle_set(10, pc.InitSpec(pc.StateVector(0, 0, 0, 0, 1)), 0)
    with pytest.raises(RuntimeError, match="CUDA"):
        kernels.spot_window_ssd(np.zeros((4, 4)), np.zeros(1), np.zeros(1), np.zeros(1), 1.0, 0, 1)


def test_bounds_partition_host_semantics():
    # test_bounds.py:131-144 (partition validation / geometry, host only)
    from paper_1310_5541_b200 import bounds as bd
    with pytest.raises(ValueError):
        bd.DomainPartition(np.array([0.0, 0.0, 1.0]), np.array([0.0, 1.0]))
    with pytest.raises(ValueError):
        bd.DomainPartition(np.array([0.0]), np.array([0.0, 1.0]))
    part = bd.DomainPartition(np.array([0.0, 1.0, 3.0]), np.array([0.0, 2.0]))
    assert part.n_cells == 2
    assert np.array_equal(part.cell_widths, [1.0, 2.0])
    assert np.array_equal(part.cell_heights, [2.0])
    assert part.domain == (0.0, 3.0, 0.0, 2.0)
