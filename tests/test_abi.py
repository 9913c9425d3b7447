"""The C-ABI library loads and exports every symbol include/pcsir_b200.h
declares; the ctypes table matches the header. CPU only (no compute calls)."""

import ctypes
import pathlib
import re
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pcsir_b200.h"
LIB = ROOT / "paper_1310_5541_b200" / "libpcsir_b200.so"


def _declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pcs_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib_path():
    srcs = list((ROOT / "paper_1310_5541_b200" / "csrc").glob("*")) + [HEADER]
    if not LIB.exists() or max(p.stat().st_mtime for p in srcs) > LIB.stat().st_mtime:
        subprocess.run(["bash", str(ROOT / "build.sh")], check=True, cwd=ROOT)
    return LIB


def test_header_declares_entry_points():
    names = _declared()
    for must in ("pcs_propagate", "pcs_partition", "pcs_dummies", "pcs_loglik",
                 "pcs_spot_window_ssd_f64", "pcs_normalize", "pcs_resample_systematic",
                 "pcs_track"):
        assert must in names


def test_library_exports_every_declared_symbol(lib_path):
    dll = ctypes.CDLL(str(lib_path))
    missing = [n for n in _declared() if not hasattr(dll, n)]
    assert not missing, missing


def test_ctypes_table_matches_header(lib_path):
    from paper_1310_5541_b200 import _lib
    assert sorted(_lib.EXPORTED_SYMBOLS) == _declared()
    _lib.load_library()  # binds every signature (raises on a missing export)


def test_sm100a_cubin_embedded(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib_path)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_host_only_calls_work_without_gpu(lib_path):
    from paper_1310_5541_b200 import _lib
    L = _lib.load_library()
    assert L.pcs_version() >= 10000
    # the systematic offset is a pure host computation (same Philox as the device)
    from oracle import pcsir_oracle as orc
    for f in (0, 1, 17, 2 ** 31 + 5):
        assert L.pcs_philox_resample_u(123456789, f) == orc.resample_u(123456789, f)


def test_invalid_arguments_are_rejected(lib_path):
    from paper_1310_5541_b200 import _lib
    L = _lib.load_library()
    spot = _lib.PcsSpot(-1.0, 10.0, 10.0, 4, 0)  # sigma_psf <= 0
    rc = L.pcs_loglik(None, 1, 1, None, None, None, 1, ctypes.byref(spot), None, None)
    assert rc == _lib.PCS_E_INVALID
    assert "sigma_psf" in _lib.last_error()


def test_ctypes_struct_layouts_match_the_library(lib_path):
    from paper_1310_5541_b200 import _lib
    L = _lib.load_library()
    out = (ctypes.c_int64 * 6)()
    assert L.pcs_abi_struct_sizes(out, 6) == 6
    mine = [ctypes.sizeof(t) for t in (_lib.PcsGrid, _lib.PcsDynamics, _lib.PcsSpot,
                                       _lib.PcsInit, _lib.PcsTrackCfg, _lib.PcsTrackResult)]
    assert list(out) == mine
