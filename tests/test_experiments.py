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
