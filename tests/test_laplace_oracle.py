"""Laplace evidence oracles: the CPU restatement against
the reference's own values (tests/golden/laplace.npz from
tests/golden/make_golden_laplace.py), and the product wrapper's validation
(no GPU needed: it validates before touching the device)."""

import numpy as np
import pytest

import oracle
from paper_2511_06407_b200 import rrgp
from paper_2511_06407_b200.evidence import GridSpec, laplace_grid_oracle

G = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "laplace.npz"))


def conj():
    x, y = G["conj_x"], G["conj_y"]
    data = rrgp.Dataset(x, y)
    fixed = rrgp.build_model("nl-mean", x, feature_count=8, intercept_variance=1e-4,
                             fixed_hypers={"c_g": 1.3, "sigma_g": 2.1, "c_l": 1.0})
    free = rrgp.build_model("nl-mean", x, feature_count=8, intercept_variance=1e-4)
    return data, fixed, free


def logi():
    data = rrgp.Dataset(G["logi_x"], G["logi_y"])
    return data, rrgp.build_model("logistic", data.x, feature_count=8)


def test_laplace_full_matches_reference():
    data, fixed, _ = conj()
    assert oracle.laplace_full(oracle.OTarget(fixed, data)) == float(G["laplace_full_fixed"])
    ld, lm = logi()
    assert oracle.laplace_full(oracle.OTarget(lm, ld)) == float(G["laplace_full_logi"])


@pytest.mark.parametrize("key,args", [
    ("grid_single", (2.6, 2.6, 4.2, 4.2)),
    ("grid_conj_4x4", (2.0, 0.5, 2.0, 0.5)),
])
def test_grid_serpentine_matches_reference(key, args):
    data, _, free = conj()
    v, st, _ = oracle.laplace_grid_nodes(oracle.OTarget(free, data), *args, (("c_l", 1.0),))
    assert oracle.laplace_grid_combine(v, st) == float(G[key])


def test_grid_logistic_and_zero_start():
    ld, lm = logi()
    t = oracle.OTarget(lm, ld)
    v, st, _ = oracle.laplace_grid_nodes(t, 3.0, 1.0, 3.0, 1.0, (("c_l", 1.0),))
    assert oracle.laplace_grid_combine(v, st) == float(G["grid_logi_3x3"])
    # independent nodes from a = 0 (what the device does): same optimum to the optimiser tolerance
    v0, st0, _ = oracle.laplace_grid_nodes(t, 3.0, 1.0, 3.0, 1.0, (("c_l", 1.0),), warm="zero")
    assert abs(oracle.laplace_grid_combine(v0, st0) - float(G["grid_logi_3x3"])) < 1e-6


def test_wrapper_validation_errors():
    data, fixed, free = conj()
    with pytest.raises(ValueError, match="Gaussian-kernel hyperparameters"):
        laplace_grid_oracle(fixed, data)
    with pytest.raises(ValueError, match="must be pinned"):
        laplace_grid_oracle(free, data, GridSpec())
    with pytest.raises(ValueError, match="must be positive"):
        laplace_grid_oracle(free, data, GridSpec(pinned=(("c_l", -1.0),)))


def test_grid_centers_match_reference_definition():
    c, s = GridSpec(c_max=2.0, c_mesh=0.5, sigma_max=1.0, sigma_mesh=0.25).centers()
    np.testing.assert_array_equal(c, [0.25, 0.75, 1.25, 1.75])
    np.testing.assert_array_equal(s, [0.125, 0.375, 0.625, 0.875])
