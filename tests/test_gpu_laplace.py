"""Device Laplace-grid oracle (csrc/sgp_grid.cuh) against the CPU oracle's
zero-start restatement node by node and against the reference's own grid
evidence (tests/golden/laplace.npz).  B200 only."""

import math

import numpy as np
import pytest

import oracle
from paper_2511_06407_b200 import rrgp
from paper_2511_06407_b200.evidence import GridSpec, laplace_grid_nodes, laplace_grid_oracle

pytestmark = pytest.mark.gpu

G = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "laplace.npz"))


def conj():
    x, y = G["conj_x"], G["conj_y"]
    data = rrgp.Dataset(x, y)
    free = rrgp.build_model("nl-mean", x, feature_count=8, intercept_variance=1e-4)
    return data, free


def logi():
    data = rrgp.Dataset(G["logi_x"], G["logi_y"])
    return data, rrgp.build_model("logistic", data.x, feature_count=8)


@pytest.mark.parametrize("case", ["conj", "logi"])
def test_nodes_match_oracle_zero_start(case):
    if case == "conj":
        data, model = conj()
        args = (2.0, 0.5, 2.0, 0.5)
    else:
        data, model = logi()
        args = (3.0, 1.0, 3.0, 1.0)
    spec = GridSpec(*args, pinned=(("c_l", 1.0),))
    v, st, it = laplace_grid_nodes(model, data, spec, mode="robust")  # pass 1 = a = 0 starts
    ov, ost, _ = oracle.laplace_grid_nodes(oracle.OTarget(model, data), *args, (("c_l", 1.0),), warm="zero")
    np.testing.assert_array_equal(st, ost)
    ok = st == 0
    # same algorithm and start; reductions differ in order -> optimiser-tolerance agreement
    assert np.max(np.abs(v[ok] - ov[ok])) < 1e-7
    assert np.all(it[ok] > 0)


@pytest.mark.parametrize("case", ["conj", "logi"])
def test_reference_mode_nodes_match_serpentine_oracle(case):
    """mode="reference": every node from the reference's serpentine a_warm; the oracle runs the
    reference's sequential chain (bit-exact with it, tests/test_laplace_oracle.py)."""
    if case == "conj":
        data, model = conj()
        args = (2.0, 0.5, 2.0, 0.5)
    else:
        data, model = logi()
        args = (3.0, 1.0, 3.0, 1.0)
    v, st, it = laplace_grid_nodes(model, data, GridSpec(*args, pinned=(("c_l", 1.0),)))
    ov, ost, _ = oracle.laplace_grid_nodes(oracle.OTarget(model, data), *args, (("c_l", 1.0),))
    np.testing.assert_array_equal(st, ost)
    ok = st == 0
    assert np.max(np.abs(v[ok] - ov[ok])) < 1e-6


def test_default_grid_fails_like_the_reference():
    """The paper's grid use (simulated logistic, N = 500, default 400 x 200 GridSpec): the
    reference's serpentine chain fails 3 678 of 80 000 nodes there and raises "untrustworthy"
    (CPU restatement, bit-exact with the reference's code path: profiles/r1_laplace_grid.md).
    mode="reference" reproduces the failure rate and the error; mode="robust" returns a value."""
    data, _ = rrgp.simulate_logistic(1, n=500, seed=0)
    model = rrgp.build_model("logistic", data.x)
    spec = GridSpec(pinned=(("c_l", 1.0),))
    v, st, _ = laplace_grid_nodes(model, data, spec)
    failed = int(np.count_nonzero(st))
    assert 0.8 * 3678 <= failed <= 1.2 * 3678, failed
    with pytest.raises(RuntimeError, match="untrustworthy"):
        laplace_grid_oracle(model, data, spec)
    assert math.isfinite(laplace_grid_oracle(model, data, spec, mode="robust"))


def test_grid_evidence_matches_reference():
    data, free = conj()
    value = laplace_grid_oracle(free, data, GridSpec(2.0, 0.5, 2.0, 0.5, pinned=(("c_l", 1.0),)))
    assert abs(value - float(G["grid_conj_4x4"])) < 1e-6
    value = laplace_grid_oracle(free, data, GridSpec(2.6, 2.6, 4.2, 4.2, pinned=(("c_l", 1.0),)))
    assert abs(value - float(G["grid_single"])) < 1e-6
    ld, lm = logi()
    value = laplace_grid_oracle(lm, ld, GridSpec(3.0, 1.0, 3.0, 1.0, pinned=(("c_l", 1.0),)))
    assert abs(value - float(G["grid_logi_3x3"])) < 1e-6


def test_single_node_is_fixed_hyper_laplace_plus_prior_and_area():
    """Reference tests/test_evidence.py:378-395 on the device."""
    data, free = conj()
    value = laplace_grid_oracle(free, data, GridSpec(2.6, 2.6, 4.2, 4.2, pinned=(("c_l", 1.0),)))

    def ig(theta, a, b):
        return a * math.log(b) - math.lgamma(a) - (a + 1.0) * math.log(theta) - b / theta

    expected = (float(G["laplace_full_fixed"]) + ig(1.3, *free.priors["c_g"]) + ig(2.1, *free.priors["sigma_g"])
                + math.log(2.6) + math.log(4.2))
    assert value == pytest.approx(expected, abs=1e-5)


def test_unsolvable_nodes_poison_the_result():
    """Reference tests/test_evidence.py:440-446."""
    data, free = conj()
    grid = GridSpec(c_max=0.5, c_mesh=0.25, sigma_max=0.5, sigma_mesh=0.25, pinned=(("c_l", 1.0),))
    with pytest.raises(RuntimeError, match="grid oracle skipped"):
        laplace_grid_oracle(free, data, grid, gtol=1e-15, max_iters=1)


def test_laplace_full_matches_reference():
    """evidence.py:277-304 on the device: mode search + cold Jacobi log-determinant."""
    from paper_2511_06407_b200.evidence import laplace_full

    x, y = G["conj_x"], G["conj_y"]
    data = rrgp.Dataset(x, y)
    fixed = rrgp.build_model("nl-mean", x, feature_count=8, intercept_variance=1e-4,
                             fixed_hypers={"c_g": 1.3, "sigma_g": 2.1, "c_l": 1.0})
    assert abs(laplace_full(fixed, data) - float(G["laplace_full_fixed"])) < 1e-8
    ld, lm = logi()
    assert abs(laplace_full(lm, ld) - float(G["laplace_full_logi"])) < 1e-8
