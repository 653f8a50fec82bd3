"""Footprint KPI pins — the paper's own Squidtab identity and
the SPEC.md worked examples."""
import csv
import json
import os

import pytest

from oracle import footprint

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_spec_examples():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        g = json.load(f)
    for ex in g["ram_pct"]:
        assert footprint.ram_pct(ex["data"], ex["buffer"]) == pytest.approx(ex["out"]), ex["cite"]
    for ex in g["footprint"]:
        assert footprint.t_footprint(ex["ram_pct"], ex["cost"]) == pytest.approx(ex["out"]), ex["cite"]


def test_squidtab_footprint_is_ram_times_cost():
    """Table Squidtab: r(pcdF) = r(%M) * r(pcdE) per row,
    within the table's 2-decimal rounding.  A footprint defined any other way
    (sum, ratio, avg of the wrong thing) fails this."""
    with open(os.path.join(GOLDEN, "squidtab.csv")) as f:
        rows = [r for r in csv.DictReader(line for line in f if not line.startswith("#"))]
    assert len(rows) == 9
    for r in rows:
        rm, re, rf = float(r["r_M"]), float(r["r_pcdE"]), float(r["r_pcdF"])
        # footprint ratio of (Squid, Knuth) = (M_s*E_s)/(M_k*E_k)
        f = footprint.ratio(footprint.t_footprint(rm, re), footprint.t_footprint(1.0, 1.0))
        # each input carries +-0.005 rounding: |d f| <= 0.005*(rm+re) + 0.005
        assert abs(f - rf) <= 0.005 * (rm + re) + 0.005 + 1e-12, r["pattern"]


def test_gns_modes_nominal():
    n = 1 << 27
    s = 12
    assert footprint.ram_pct(n * s, n * s) == 2.0
    assert footprint.ram_pct(n * s, (n // 2) * s) == 1.5
    with pytest.raises(ValueError):
        footprint.ram_pct(0, 1)
