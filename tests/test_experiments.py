"""GPU sweep harness and micro-benchmark (experiments.py, cli.py of the
reference): variant parsing, summary aggregation and CSV columns on the host,
a small paired sweep and the CLI on the GPU."""

import math

import numpy as np
import pytest

from paper_1310_5541_b200 import experiments as ex
from paper_1310_5541_b200.binning import DummyPlacement


def test_parse_variant_labels():
    assert ex.parse_variant("SIR").label == "SIR" and not ex.parse_variant("sir").is_pc
    v = ex.parse_variant("pcSIR-2x2-coc")
    assert v.label == "pcSIR-2x2-CoC" and v.cells_per_pixel == 2
    assert v.placement is DummyPlacement.CELL_CENTER
    assert ex.parse_variant("pcsir-1x1").label == "pcSIR-1x1-CoM"
    for bad in ("pcSIR", "pcSIR-2x3", "foo-1x1", "pcSIR-1x1-xyz"):
        with pytest.raises(ex.ConfigError):
            ex.parse_variant(bad)


def test_summarize_matches_reference_rules(tmp_path):
    R = ex.RunRecord
    recs = [R("e", "SIR", 100, 0, 1.0, 2.0, 500), R("e", "SIR", 100, 1, 3.0, 4.0, 700),
            R("e", "pcSIR-1x1-CoM", 100, 0, 2.0, 1.0, 50),
            R("e", "pcSIR-1x1-CoM", 100, 1, float("nan"), 9.0, 0, failed=True)]
    rows = ex.summarize(recs)
    sir, pc = rows
    assert sir.rmse_mean == 2.0 and math.isclose(sir.rmse_std, math.sqrt(2.0))
    assert sir.time_mean_s == 3.0 and sir.lik_evals_mean == 600 and sir.speedup_vs_sir == 1.0
    assert pc.time_mean_s == 1.0 and pc.rmse_std == 0.0 and pc.speedup_vs_sir == 3.0
    p = ex.write_summary_csv(rows, tmp_path / "s.csv")
    lines = p.read_text().splitlines()
    assert lines[0].split(",") == list(ex.SUMMARY_COLUMNS) and len(lines) == 3


def test_sweep_validation():
    with pytest.raises(ex.ConfigError):
        ex.run_tracking_experiment(["SIR"], [100, 100], 1)
    with pytest.raises(ex.ConfigError):
        ex.run_tracking_experiment(["SIR"], [100], 0)


@pytest.mark.gpu
def test_gpu_sweep_paired(cuda):
    from paper_1310_5541_b200 import synthesis as syn
    from paper_1310_5541_b200.imaging import PsfParams
    scene = syn.SceneConfig(PsfParams(1.5, 10.0), frames=6, width=64, height=64)
    recs = ex.run_tracking_experiment(["SIR", "pcSIR-1x1-CoM"], [2000, 8000], 2, scene=scene,
                                      seed=3)
    assert len(recs) == 8 and not any(r.failed for r in recs)
    by = {(r.variant, r.n_particles, r.repetition): r for r in recs}
    for n in (2000, 8000):
        for rep in range(2):
            assert by[("SIR", n, rep)].lik_evals == n * 6
            assert by[("pcSIR-1x1-CoM", n, rep)].lik_evals < n * 6 / 10
            assert by[("pcSIR-1x1-CoM", n, rep)].rmse < 1.0
    rows = ex.summarize(recs)
    assert {r.variant for r in rows} == {"SIR", "pcSIR-1x1-CoM"}
    assert all(np.isfinite(r.speedup_vs_sir) for r in rows)
    # repeatable: same seed -> same trajectories
    again = ex.run_tracking_experiment(["pcSIR-1x1-CoM"], [2000], 1, scene=scene, seed=3)
    assert np.array_equal(again[0].trajectory, by[("pcSIR-1x1-CoM", 2000, 0)].trajectory)


@pytest.mark.gpu
def test_cli_backends_and_track(cuda, tmp_path, capsys):
    from paper_1310_5541_b200.__main__ import main
    assert main(["backends", "--repeats", "2"]) == 0
    out = capsys.readouterr().out
    assert "small spot (9x9)" in out and "evals/s" in out
    csv = tmp_path / "t.csv"
    assert main(["track", "--variants", "SIR,pcSIR-2x2-CoM", "--n", "1000", "--reps", "1",
                 "--frames", "4", "--size", "64", "--out", str(csv)]) == 0
    assert csv.read_text().startswith(",".join(ex.SUMMARY_COLUMNS))
    assert main(["track", "--variants", "bogus"]) == 2


def test_parse_prior_and_pseudo_summary():
    c = ex.StateVector(1.0, 2.0, 0.0, 0.0, 20.0)
    assert ex.parse_prior("uniform3x3", c).width == 3.0
    assert ex.parse_prior("gauss0.8", c).sigma == 0.8
    assert ex.parse_prior("point", c).mode == "point"
    with pytest.raises(ex.ConfigError):
        ex.parse_prior("cauchy1", c)
    R = ex.RunRecord
    rows = ex.summarize([R("pseudo_tracking", "SIR", 10, 0, 3.0, 1.0, 10),
                         R("pseudo_tracking", "SIR", 10, 1, 4.0, 1.0, 10)])
    assert rows[0].rmse_mean == math.sqrt(12.5)   # RMS of single-shot errors


@pytest.mark.gpu
def test_gpu_pseudo_tracking(cuda):
    recs = ex.run_pseudo_tracking(["SIR", "pcSIR-1x1-CoM", "pcSIR-2x2-CoC"], [300, 30000], 12,
                                  prior="uniform3x3", seed=1)
    assert len(recs) == 2 * 12 * 3 and not any(r.failed for r in recs)
    rows = {(r.variant, r.n_particles): r for r in ex.summarize(recs)}
    for v in ("SIR", "pcSIR-1x1-CoM", "pcSIR-2x2-CoC"):
        assert rows[(v, 30000)].rmse_mean < rows[(v, 300)].rmse_mean
    # the 1x1 grid cannot resolve sub-pixel offsets better than SIR at large N
    assert rows[("SIR", 30000)].rmse_mean < 0.1
    assert rows[("pcSIR-1x1-CoM", 30000)].lik_evals_mean <= 16
    again = ex.run_pseudo_tracking(["pcSIR-1x1-CoM"], [300], 2, prior="uniform3x3", seed=1)
    assert [r.rmse for r in again] == [r.rmse for r in recs
                                       if r.variant == "pcSIR-1x1-CoM" and r.n_particles == 300][:2]


# --- the reference's own harness on the same scenes -----------
def _golden_scenes(g):
    reps = len([k for k in g.files if k.startswith("frames_")])
    return [{"frames": g[f"frames_{r}"].astype(np.float32), "positions": g[f"positions_{r}"],
             "init_state": g[f"init_{r}"]} for r in range(reps)]


def test_summary_columns_match_reference():
    from conftest import golden
    from paper_1310_5541_b200 import experiments as ex
    g = golden("experiments")
    assert tuple(ex.SUMMARY_COLUMNS) == tuple(str(c) for c in g["summary_columns"])


@pytest.mark.gpu
def test_sweep_matches_reference_harness_on_its_scenes(cuda):
    """The reference's run_tracking_experiment (reduced small_object preset,
    8 repetitions, N = 2000 / 8000, its default ResampleConfig: ESS threshold
    0.5, multinomial) against the device harness on the SAME rendered frames
    (tests/golden/experiments.npz). The RNG streams differ (numpy vs Philox),
    so the comparison is statistical: SIR evaluation counts equal exactly,
    pcSIR occupied-cell counts and RMSE agree within sampling error, and the
    1x1-cell bias of pcSIR over SIR that the reference shows is reproduced."""
    from conftest import golden
    import paper_1310_5541_b200 as pc
    from paper_1310_5541_b200 import experiments as ex
    g = golden("experiments")
    d = g["filter_dyn"]
    recs = ex.run_tracking_on_scenes(
        _golden_scenes(g), [str(v) for v in g["variants"]], [int(n) for n in g["n_particles"]],
        pc.PsfParams(float(g["sigma_psf"]), float(g["i_bg"])), float(g["sigma_xi"]), int(g["hw"]),
        filter_dynamics=pc.DynamicsParams(float(d[0]), float(d[1]), float(d[2]), float(d[3])),
        prior=str(g["prior"]), seed=3)
    rows = {(r.variant, r.n_particles): r for r in ex.summarize(recs)}
    ref = {(str(v), int(n)): (float(e), float(m)) for v, n, e, m in
           zip(g["sum_variant"], g["sum_n"], g["sum_rmse_mean"], g["sum_evals_mean"])}
    assert set(rows) == set(ref)
    assert not any(r.failed for r in recs)
    k = g["frames_0"].shape[0]
    for r in recs:
        if r.variant == "SIR":
            assert r.lik_evals == r.n_particles * k
    for key, (rmse_ref, evals_ref) in ref.items():
        row = rows[key]
        assert abs(row.rmse_mean - rmse_ref) <= 0.06, (key, row.rmse_mean, rmse_ref)
        assert abs(row.lik_evals_mean - evals_ref) <= 0.12 * evals_ref, (key, row.lik_evals_mean,
                                                                         evals_ref)
    for n in (2000, 8000):   # the 1x1-cell approximation costs accuracy in both
        assert rows[("pcSIR-1x1-CoM", n)].rmse_mean > rows[("SIR", n)].rmse_mean
        assert ref[("pcSIR-1x1-CoM", n)][0] > ref[("SIR", n)][0]
