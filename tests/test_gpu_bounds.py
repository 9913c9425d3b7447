"""The appendix bound study on the device against the
unmodified reference (tests/golden/bounds.npz from bounds.py:121-180 and
experiments.py:370-388): derivative maxima bit for bit (an exact max over
the same np.linspace samples, within an ulp where CUDA's exp / sin round
differently), bounds to 1e-12 and the quadrature error to 1e-11 relative
(the reference's einsum order differs from the device's fixed order), plus
the reference tests' known answers (test_bounds.py)."""

import numpy as np
import pytest

from conftest import golden
from paper_1310_5541_b200 import bounds as bd
from paper_1310_5541_b200.experiments import run_bounds_study

pytestmark = pytest.mark.gpu

FIELDS = {"quadratic": bd.quadratic_field(), "linear": bd.linear_field(),
          "sinsin": bd.sinsin_field(), "gaussian": bd.gaussian_spot_field(),
          "gauss2": bd.gaussian_spot_field(1.5, 20.0, 10.0, (0.3, -0.2))}
DOMAINS = {"quadratic": (0.0, 4.0, 0.0, 4.0), "linear": (0.0, 1.0, 0.0, 1.0),
           "sinsin": (0.0, np.pi, 0.0, np.pi), "gaussian": (-4.0, 4.0, -4.0, 4.0),
           "gauss2": (-3.0, 5.0, -4.0, 2.0)}


def _close(got, want, rtol, atol=1e-15):
    np.testing.assert_allclose(got, want, rtol=rtol, atol=atol)


@pytest.mark.parametrize("name", list(FIELDS))
@pytest.mark.parametrize("cells", [(4, 4), (7, 3), (16, 16), (33, 20), "irr"])
def test_bounds_match_reference(cuda, name, cells):
    g = golden("bounds")
    fld = FIELDS[name]
    if cells == "irr":
        part = bd.DomainPartition(g[f"{name}_irr_x"], g[f"{name}_irr_y"])
        key = f"{name}_irr"
    else:
        part = bd.DomainPartition.uniform(DOMAINS[name], *cells)
        key = f"{name}_{cells[0]}x{cells[1]}"
    _close(bd.derivative_maxima(fld, part), g[f"{key}_dmax"], rtol=4e-16)
    _close(bd.rect_bound(fld, part), g[f"{key}_rect"], rtol=1e-12)
    _close(bd.midpoint_error(fld, part), g[f"{key}_mid64"], rtol=1e-11, atol=1e-14)
    if cells != "irr":
        _close(bd.midpoint_error(fld, part, quad_points=16), g[f"{key}_mid16"], rtol=1e-11,
               atol=1e-14)


def test_bounds_study_matches_reference(cuda):
    g = golden("bounds")
    for name, rows in run_bounds_study().items():
        _close(np.array(rows), g[f"study_{name}"], rtol=1e-11, atol=1e-14)


def test_reference_known_answers(cuda):
    # test_bounds.py:14-79
    unit = (0.0, 1.0, 0.0, 1.0)
    part = bd.DomainPartition.uniform(unit, 1, 1)
    assert bd.rect_bound(bd.quadratic_field(), part) == pytest.approx(1.0 / 6.0, rel=1e-12)
    part4 = bd.DomainPartition.uniform(unit, 4, 4)
    assert bd.rect_bound(bd.linear_field(), part4) == 0.0
    assert bd.midpoint_error(bd.linear_field(), part4) == pytest.approx(0.0, abs=1e-15)
    constant = bd.polynomial_field("constant", e=4.2)
    assert bd.midpoint_error(constant, bd.DomainPartition.uniform(unit, 3, 3)) == 0.0
    xsq = bd.polynomial_field("xsq", a=1.0)
    assert bd.midpoint_error(xsq, part) == pytest.approx(1.0 / 12.0, abs=1e-10)
    field = bd.gaussian_spot_field(sigma=1.16)
    ratio = (bd.square_bound(field, 1.0, (-4.0, 4.0, -4.0, 4.0))
             / bd.square_bound(field, 0.5, (-4.0, 4.0, -4.0, 4.0)))
    assert ratio == pytest.approx(4.0, rel=1e-9)
    with pytest.raises(ValueError):
        bd.square_bound(bd.quadratic_field(), 0.3, unit)
    for name, dom in (("quadratic", (0.0, 4.0, 0.0, 4.0)), ("gaussian", (-4.0, 4.0, -4.0, 4.0)),
                      ("sinsin", (0.0, 4.0, 0.0, 4.0))):
        fld = bd.builtin_fields()[name]
        for cells in ((4, 4), (7, 3), (16, 16)):
            p = bd.DomainPartition.uniform(dom, *cells)
            assert bd.midpoint_error(fld, p) <= bd.rect_bound(fld, p) + 1e-12


def test_large_partition_runs_on_device(cuda):
    # 512 x 512 cells x 64^2 nodes = 1.07e9 field evaluations
    fld = bd.gaussian_spot_field(1.5, 20.0, 10.0)
    part = bd.DomainPartition.uniform((-8.0, 8.0, -8.0, 8.0), 512, 512)
    err = bd.midpoint_error(fld, part)
    assert 0.0 < err <= bd.rect_bound(fld, part)
