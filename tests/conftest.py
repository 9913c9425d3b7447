import pathlib
import subprocess
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_oracle():
    lib = ROOT / "oracle" / "liboracle.so"
    if not lib.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)


_ensure_oracle()


def assert_propagation_close(got, want, s32, z32, dyn):
    """|got - want| <= 2^-22 x max(|state in|, |state out|, |noise term|,
    |v dt| for positions): two float32 ulps of the operands' scale."""
    sig = np.array([dyn[0], dyn[0], dyn[1], dyn[1], dyn[2]])[:, None]
    scale = np.maximum.reduce([np.abs(s32.astype(np.float64)), np.abs(want),
                               np.abs(z32.astype(np.float64)) * sig])
    scale[:2] = np.maximum(scale[:2], np.abs(s32[2:4].astype(np.float64)) * dyn[3])
    err = np.abs(got.astype(np.float64) - want)
    assert np.all(err <= 2.0 ** -22 * scale), float(np.max(err / scale))


def golden(name):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


@pytest.fixture
def rng():
    return np.random.default_rng(20240)  # reference conftest.py:9-11


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)


def spot_pixels(x, y, i0, sigma, bg, width=64, height=64):
    """Noise-free frame (synthesis.py:124-129 form)."""
    gx = np.exp(-((np.arange(width) - x) ** 2) / (2.0 * sigma ** 2))
    gy = np.exp(-((np.arange(height) - y) ** 2) / (2.0 * sigma ** 2))
    return i0 * np.outer(gy, gx) + bg
