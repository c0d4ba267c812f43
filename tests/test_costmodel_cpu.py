"""B200 cost-model calibration.  The fit is the reference's own
(``dllmsim.costmodel.fit``, costmodel.py:118-176) applied to the B200 step profile
that tools/calibrate_b200.py measures; these tests check the committed calibration
is a valid model and that the reference reproduces it from the committed CSV."""

import json
from pathlib import Path

import numpy as np
import pytest



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
    dllmsim's own fit of the committed profile CSV."""
    costmodel = pytest.importorskip("dllmsim.costmodel")
    prof = Path(__file__).resolve().parents[1] / "profiles"
    if not (prof / name).exists():
        pytest.skip("committed calibration absent")
    CostModel, fit, profile_from_csv = costmodel.CostModel, costmodel.fit, costmodel.profile_from_csv

    ours = CostModel.from_json((prof / name).read_text())
    csv_name = name.replace("_cost_model.json", "_step_profile.csv")
    theirs = fit(profile_from_csv((prof / csv_name).read_text()))
    for x in (0, 10, 100, 500, 1000, 1500, 3000):
        assert ours.latency(x) == pytest.approx(theirs.latency(x), rel=1e-9)
