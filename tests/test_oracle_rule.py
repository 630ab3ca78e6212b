"""Pins for the oracle's HHT quadrature rule (App. B; Lemma 3).

The oracle evaluates eq. quad_points_and_locations literally with complex arguments (mpmath).
Pins, none of which re-call that routine:
* an independent REAL-arithmetic route through scipy.special.ellipj/ellipk and the Jacobi
  imaginary transforms sn(ix|k)=i sc(x|k'), cn(ix|k)=nc(x|k'), dn(ix|k)=dc(x|k');
* the 1x1 case of eq. contour_integral_quad, lambda * sum_q w_q/(t_q+lambda) ~ sqrt(lambda), within
  the Hale bound O(exp(-2 Q pi^2 / (log kappa + 3))) (Lemma hale);
* the paper's claim that Q=8 gives < 1e-4 for kappa ~ 1e4;
* positivity t_q, w_q > 0, strict ordering, exact homogeneity in lambda;
* Lemma 3: sum_q w_q/t_q < 4 Q log(5 sqrt(kappa)) / (pi sqrt(lambda_min))."""
import math

import numpy as np
import pytest
import scipy.special as sp

from oracle import hht_rule


def real_form_rule(lmin, lmax, q):
    k2 = lmin / lmax
    mp_ = 1.0 - k2                                    # parameter of k'
    kp = sp.ellipk(mp_)
    u = (np.arange(1, q + 1) - 0.5) / q
    sn, cn, dn, _ = sp.ellipj(u * kp, mp_)
    t = lmin * (sn / cn) ** 2
    w = 2.0 * math.sqrt(lmin) * kp / (math.pi * q) * dn / cn ** 2
    return t, w


def scalar_rel_err(t, w, lam):
    lam = np.asarray(lam, dtype=np.float64)
    approx = lam * np.sum(w[None, :] / (t[None, :] + lam[:, None]), axis=1)
    return np.abs(approx - np.sqrt(lam)) / np.sqrt(lam)


def hale(q, kappa):
    return math.exp(-2.0 * q * math.pi ** 2 / (math.log(kappa) + 3.0))


@pytest.mark.parametrize("lmin,lmax,q", [(1e-4, 1.0, 8), (0.05, 104.0, 8), (1e-3, 3.0, 15), (1.0, 1e8, 20), (2.0, 3.0, 4)])
def test_rule_matches_independent_real_form(lmin, lmax, q):
    t, w = hht_rule(lmin, lmax, q)
    tr, wr = real_form_rule(lmin, lmax, q)
    # scipy's ellipj loses digits as the parameter m' = 1 - 1/kappa -> 1 (measured 5e-9 at 1e8)
    rtol = 1e-11 if lmax / lmin <= 1e6 else 1e-8
    np.testing.assert_allclose(t, tr, rtol=rtol)
    np.testing.assert_allclose(w, wr, rtol=rtol)


@pytest.mark.parametrize("kappa", [10.0, 1e2, 1e4, 1e6, 1e8])
@pytest.mark.parametrize("q", [2, 4, 8, 12, 16, 20])
def test_scalar_identity_within_hale_bound(kappa, q):
    lmin = 0.37
    lmax = lmin * kappa
    t, w = hht_rule(lmin, lmax, q)
    assert np.all(t > 0) and np.all(w > 0)
    assert np.all(np.diff(t) > 0)
    lam = np.geomspace(lmin, lmax, 400)
    err = scalar_rel_err(t, w, lam).max()
    assert err <= max(10.0 * hale(q, kappa), 1e-13), (err, hale(q, kappa))
    # Lemma 3
    assert np.sum(w / t) < 4 * q * math.log(5 * math.sqrt(kappa)) / (math.pi * math.sqrt(lmin))


def test_paper_claim_q8_kappa_1e4():
    t, w = hht_rule(1.0, 1e4, 8)
    lam = np.geomspace(1.0, 1e4, 200)
    assert scalar_rel_err(t, w, lam).max() < 1e-4
    # SPEC S:240 "lambda = 4, rule for [1, 16], Q=8 -> ~2 to 1e-6"
    t, w = hht_rule(1.0, 16.0, 8)
    assert abs(4.0 * np.sum(w / (t + 4.0)) - 2.0) < 1e-6


def test_error_decays_with_q():
    lam = np.geomspace(1.0, 1e5, 300)
    errs = [scalar_rel_err(*hht_rule(1.0, 1e5, q), lam).max() for q in (2, 4, 6, 8, 10, 12)]
    assert all(b < a for a, b in zip(errs, errs[1:])), errs


def test_homogeneity():
    t, w = hht_rule(0.01, 50.0, 8)
    t2, w2 = hht_rule(0.04, 200.0, 8)
    np.testing.assert_allclose(t2, 4.0 * t, rtol=1e-13)
    np.testing.assert_allclose(w2, 2.0 * w, rtol=1e-13)


def test_clamped_kappa_one():
    # lambda_min = lambda_max = 1, Q = 4 -> rule exists, scalar check passes
    t, w = hht_rule(1.0, 1.0, 4)
    assert np.all(np.isfinite(t)) and np.all(np.isfinite(w))
    assert abs(1.0 * np.sum(w / (t + 1.0)) - 1.0) < 1e-6


def test_invalid_arguments():
    with pytest.raises(ValueError):
        hht_rule(1.0, 2.0, 0)
    with pytest.raises(ValueError):
        hht_rule(0.0, 2.0, 4)
