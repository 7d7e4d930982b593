"""The paper's §4 grid protocol (paper_2110_03423_b200/grid.py), mirroring the reference's
bench suite (tests/test_bench.cpp): statistics, ratio band, CSV format, presets; and one
small GPU grid whose fast-decay rows meet the 1e-8 accuracy gate (bench.hpp:75)."""
import io

import pytest

from paper_2110_03423_b200 import grid as G


def test_summarize_and_ratio_band():
    ours = G.summarize("rsvd", [1.0, 2.0, 3.0])
    assert ours.n_runs == 3 and ours.mean_seconds == 2.0 and abs(ours.std_seconds - 1.0) < 1e-15
    comp = G.summarize("full", [10.0])
    assert comp.std_seconds == 0.0
    row = G.speedup_ratio(comp, ours)
    assert row.ratio == 5.0
    assert row.band_lo == 10.0 / 3.0 and row.band_hi == 10.0 / 1.0
    # mean_ours <= std_ours: no upper band
    row = G.speedup_ratio(comp, G.summarize("rsvd", [0.1, 3.0]))
    assert row.band_hi is None
    with pytest.raises(ValueError):
        G.speedup_ratio(comp, G.BenchStats("rsvd", 1, 0.0, 0.0))


def test_csv_format():
    r = G.SpeedupRow("fast", 500, 100, 0.03, 3, "full_svd_gpu", 1.0, 0.1, 0.5, 0.05, 2.0,
                     1.5, None, 1e-12)
    buf = io.StringIO()
    G.write_csv([r], buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == G.CSV_HEADER
    assert lines[1] == "fast,500,100,0.029999999999999999,3,full_svd_gpu,1,0.10000000000000001," \
                       "0.5,0.050000000000000003,2,1.5,,9.9999999999999998e-13"


def test_presets():
    for name in ("fast-small", "sharp-small", "slow-small", "fast-2000", "sharp-2000",
                 "slow-2000", "perf-2000"):
        g = G.preset(name)
        assert g.m in (500, 2000) and g.n_grid
    assert G.preset("fast-2000").power_q == 12 and G.preset("sharp-small").power_q == 4
    assert G.preset("perf-2000").k_fractions == [0.01]
    with pytest.raises(ValueError):
        G.preset("nope")


@pytest.mark.gpu
def test_gpu_grid_fast_small(solver):
    cfg = G.preset("fast-small")
    cfg.repetitions = 2
    rows, errors = G.run_grid(cfg, solver)
    assert not errors and len(rows) == 12
    assert all(r.max_rel_err <= cfg.tolerance for r in rows), [r.max_rel_err for r in rows]
    assert all(r.ratio > 0 for r in rows)
