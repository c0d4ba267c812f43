"""B200 cost-model calibration against the reference's own fit.

tests/golden/costmodel.json holds seeded (x, latency) profiles with dllmsim's fit of
each (costmodel.py:118-176) and its profile CSV (costmodel.py:179-186), written by
tests/golden/make_golden.py from the reference itself.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2605_24832_b200 import costmodel as cm
from paper_2605_24832_b200.errors import ConfigError

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "costmodel.json").read_text())


@pytest.mark.parametrize("k", range(len(GOLD["fits"])))
def test_fit_matches_reference(k):
    case = GOLD["fits"][k]
    samples = [tuple(s) for s in case["samples"]]
    got = cm.fit(samples)
    ref = case["fit"]
    for a, b in zip(got["segments"], ref["segments"]):
        assert a["x_start"] == b["x_start"]
        for key in ("slope_us_per_token", "intercept_ms"):
            assert a[key] == pytest.approx(b[key], rel=1e-9, abs=1e-12)
    # and the model evaluates like the reference's latency() on a grid
    for x in np.linspace(0, 5000, 37):
        seg = ref["segments"][0]
        for s in ref["segments"][1:]:
            if x >= s["x_start"]:
                seg = s
        want = seg["intercept_ms"] * 1e-3 + seg["slope_us_per_token"] * 1e-6 * (x - seg["x_start"])
        assert cm.latency(got, x) == pytest.approx(want, rel=1e-9)


@pytest.mark.parametrize("k", range(len(GOLD["fits"])))
def test_profile_csv_is_the_reference_format(k):
    case = GOLD["fits"][k]
    assert cm.profile_csv([tuple(s) for s in case["samples"]]) == case["csv"]


def test_fit_rejects_short_profiles():
    with pytest.raises(ConfigError):
        cm.fit([(float(i), 1e-3) for i in range(5)])
    with pytest.raises(ConfigError):
        cm.fit([(float(i % 4), 1e-3) for i in range(20)])


def test_committed_b200_calibration_is_a_valid_model():
    """profiles/b200_cost_model.json (tools/calibrate_b200.py on a B200) is continuous,
    nondecreasing and convex, as the reference's CostModel requires (costmodel.py:39-55)."""
    p = Path(__file__).resolve().parents[1] / "profiles" / "b200_cost_model.json"
    if not p.exists():
        pytest.skip("no B200 calibration committed yet")
    m = json.loads(p.read_text())
    segs = m["segments"]
    assert len(segs) == 3 and segs[0]["x_start"] == 0
    for a, b in zip(segs, segs[1:]):
        assert b["x_start"] > a["x_start"]
        assert b["slope_us_per_token"] >= a["slope_us_per_token"] >= 0
        joint = a["intercept_ms"] + a["slope_us_per_token"] * 1e-3 * (b["x_start"] - a["x_start"])
        assert joint == pytest.approx(b["intercept_ms"], rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("name", ["b200_cost_model.json", "b200_b64_cost_model.json"])
def test_reference_loads_and_refits_the_b200_calibration(name):
    """The committed B200 model loads with dllmsim's CostModel.from_json and equals
    dllmsim's own fit of the committed profile CSV (run only where the reference
    checkout exists; the GPU box has none)."""
    import sys
    ref = Path("/root/reference/pkg/src")
    prof = Path(__file__).resolve().parents[1] / "profiles"
    if not ref.exists() or not (prof / name).exists():
        pytest.skip("reference checkout or committed calibration absent")
    sys.path.insert(0, str(ref))
    from dllmsim.costmodel import CostModel, fit, profile_from_csv

    ours = CostModel.from_json((prof / name).read_text())
    csv_name = name.replace("_cost_model.json", "_step_profile.csv")
    theirs = fit(profile_from_csv((prof / csv_name).read_text()))
    for x in (0, 10, 100, 500, 1000, 1500, 3000):
        assert ours.latency(x) == pytest.approx(theirs.latency(x), rel=1e-9)
