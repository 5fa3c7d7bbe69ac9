"""oracle/synthetic.py (the SyntheticGradSpec restatement used for cfg3's inputs) against the
reference's own synthetic_round outputs (tests/golden/synthetic.npz, make_golden.py)."""
import json
import os

import numpy as np
import pytest

from oracle.synthetic import SyntheticGradSpec, SyntheticStream, synthetic_round

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "synthetic.npz")


def test_synthetic_round_matches_reference():
    z = np.load(GOLD)
    for i, m in enumerate(json.loads(str(z["meta"]))):
        got = synthetic_round(SyntheticGradSpec(dim=m["d"], **m["kw"]), m["seed"], m["round"], m["n"])
        assert np.array_equal(np.stack(got), z[f"g_{i}"]), m


def test_stream_reuses_shared_part_across_rounds():
    spec = SyntheticGradSpec(dim=5000)
    s = SyntheticStream(spec, 3)
    for r in range(3):
        assert np.array_equal(np.stack(s.round(r, 2)), np.stack(synthetic_round(spec, 3, r, 2)))


def test_validation():
    with pytest.raises(ValueError):
        SyntheticGradSpec(dim=1)
    with pytest.raises(ValueError):
        SyntheticGradSpec(dim=10, rho=1.0)
