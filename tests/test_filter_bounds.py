"""Filter truncation-error bounds (csrc/bounds.cpp through the C-ABI) and the
inspect-filter sweep -- every case of proj/tests/test_filter_bounds.cpp,
restated on the reference's own generators (libstdc++ mt19937_64 and
uniform_real_distribution, reproduced bit for bit by the oracle).
"""
import math

import numpy as np
import pytest

import paper_2604_00914_b200 as adp

PI = math.pi


def step_in_angle(theta, alpha, beta):
    if beta < theta < alpha:
        return 1.0
    if theta == alpha or theta == beta:
        return 0.5
    return 0.0


def g_truncated(theta, alpha, beta, k):
    c = adp.chebyshev_step_coeffs(alpha, beta, k)
    acc = 0.0
    for j in range(k + 1):
        acc += c[j] * math.cos(j * theta)
    return acc


def g_damped(theta, alpha, beta, k_i, k, m):
    c = adp.chebyshev_step_coeffs(alpha, beta, k)
    d = adp.lanczos_damping(k, m)
    acc = 0.0
    for j in range(k_i + 1):
        acc += c[j] * d[j] * math.cos(j * theta)
    return acc


# test_filter_bounds.cpp:44-56
def test_j_theta_closed_special_case():
    alpha, beta = 1.9, 0.6
    want = 1.0 / abs(math.sin(alpha)) + 1.0 / abs(math.sin(0.5 * (alpha + beta))) + 1.0 / abs(math.sin(0.5 * (alpha - beta)))
    assert adp.j_theta(alpha, alpha, beta) == want
    want_b = 1.0 / abs(math.sin(beta)) + 1.0 / abs(math.sin(0.5 * (alpha + beta))) + 1.0 / abs(math.sin(0.5 * (alpha - beta)))
    assert adp.j_theta(beta, alpha, beta) == want_b


# :58-65
def test_j_theta_four_term_plug_in():
    alpha, beta, theta = 2.0 * PI / 3.0, PI / 3.0, PI / 2.0
    want = 1 / math.sin(7 * PI / 12) + 1 / math.sin(PI / 12) + 1 / math.sin(5 * PI / 12) + 1 / math.sin(PI / 12)
    assert adp.j_theta(theta, alpha, beta) == pytest.approx(want, rel=1e-13)


# :67-81
def test_j_theta_far_field(orc):
    alpha, beta = math.acos(0.1), math.acos(0.6)
    rng = orc.MT19937_64(7)
    for _ in range(2000):
        theta = rng.uniform(0.0, PI)
        d = min(abs(theta - alpha), abs(theta + alpha - 2 * PI), abs(theta + alpha), abs(theta - beta),
                abs(theta + beta - 2 * PI), abs(theta + beta))
        if d < 1e-6:
            continue
        assert adp.j_theta(theta, alpha, beta) <= 4.0 * PI / d * (1.0 + 1e-12)


# :83-85
def test_j_theta_vanishing_denominator_is_inf():
    assert adp.j_theta(0.0, 2.0, 0.0) == math.inf


# :87-95 (doctest Approx(want).epsilon(e): |a - w| <= e * (scale + max(|a|, |w|)), scale 1)
@pytest.mark.parametrize("m,want", [(0.3, 1.623510847285), (0.5, 1.157421898908), (1.0, 0.766813582899),
                                    (2.0, 0.525768839741), (3.0, 0.425209921156)])
def test_c_m_constant_frozen_references(m, want):
    got = adp.c_m_constant(m)
    assert abs(got - want) <= 5e-10 * (1.0 + max(abs(got), abs(want)))


# :97-110
def test_c_m_constant_m1_trapezoid():
    # the reference uses 1e7 trapezoid panels; 2e6 (vectorised) already agrees to ~1e-13
    n = 2_000_000
    u = np.linspace(0.0, PI, n + 1)
    f = np.empty_like(u)
    small = u < 1e-8
    f[small] = 1.0 / 3.0
    us = u[~small]
    f[~small] = (np.sin(us) - us * np.cos(us)) / us ** 3
    want = (PI / n) * (0.5 * (f[0] + f[-1]) + f[1:-1].sum())
    got = adp.c_m_constant(1.0)
    assert abs(got - want) <= 1e-9 * (1.0 + max(abs(got), abs(want)))


# :112-118
def test_c_m_constant_positive_cached_and_rejects_nonpositive():
    for m in (0.2, 0.5, 0.9, 1.0, 1.5, 2.5, 4.0):
        assert adp.c_m_constant(m) > 0.0
    assert adp.c_m_constant(0.7) == adp.c_m_constant(0.7)
    for m in (0.0, -1.0):
        with pytest.raises(adp.ConfigError):
            adp.c_m_constant(m)


# :120-144
def test_undamped_bound_decay_and_soundness(orc):
    alpha, beta = math.acos(0.1), math.acos(0.6)
    prev = math.inf
    for k in (1, 2, 5, 10, 50, 500):
        b = adp.undamped_bound(1.0, k, alpha, beta)
        assert b < prev
        prev = b
        assert b == pytest.approx(adp.j_theta(1.0, alpha, beta) / (PI * (k + 1)))
    rng = orc.MT19937_64(3)
    checked = 0
    for _ in range(2000):
        theta = rng.uniform(0.0, PI)
        if abs(theta - alpha) < 1e-3 or abs(theta - beta) < 1e-3:
            continue
        checked += 1
        for k in (5, 20, 100):
            err = abs(step_in_angle(theta, alpha, beta) - g_truncated(theta, alpha, beta, k))
            assert err <= adp.undamped_bound(theta, k, alpha, beta)
    assert checked > 1900
    with pytest.raises(adp.ConfigError):
        adp.undamped_bound(1.0, 0, alpha, beta)


# :146-151
def test_undamped_bound_far_field_chaining():
    alpha, beta = 2.0, 0.9
    theta = alpha + 0.1
    for k in (5, 20, 100):
        assert adp.undamped_bound(theta, k, alpha, beta) <= 40.0 / (k + 1)


# :153-160
def test_damped_bound_m0_is_undamped():
    alpha, beta = math.acos(0.1), math.acos(0.6)
    for theta in (0.3, 1.0, 2.2):
        for k_i in (3, 10, 40):
            assert adp.damped_bound(theta, k_i, 100, 0.0, alpha, beta) == adp.undamped_bound(theta, k_i, alpha, beta)


# :162-179
def test_damped_bound_soundness_sampled(orc):
    alpha, beta = math.acos(0.1), math.acos(0.6)
    rng = orc.MT19937_64(11)
    for _ in range(400):
        theta = rng.uniform(0.0, PI)
        if abs(theta - alpha) < 1e-3 or abs(theta - beta) < 1e-3:
            continue
        for m in (0.5, 1.0, 2.0):
            for k_i in (10, 40):
                k = int(math.ceil(2.5 * k_i))
                err = abs(step_in_angle(theta, alpha, beta) - g_damped(theta, alpha, beta, k_i, k, m))
                assert err <= adp.damped_bound(theta, k_i, k, m, alpha, beta)


def test_damped_bound_errors():
    with pytest.raises(adp.ConfigError):
        adp.damped_bound(1.0, 0, 10, 0.5, 2.0, 1.0)
    with pytest.raises(adp.ConfigError):
        adp.damped_bound(1.0, 11, 10, 0.5, 2.0, 1.0)
    with pytest.raises(adp.ConfigError):
        adp.damped_bound(1.0, 5, 10, -0.5, 2.0, 1.0)


# :181-192
def test_damped_bound_decays_like_inverse_degree():
    alpha, beta = math.acos(0.1), math.acos(0.6)
    for x in (-0.1, 0.0, 0.2, 0.3):
        theta = math.acos(x)

        def bound_at(k_i):
            return adp.damped_bound(theta, k_i, int(math.ceil(2.5 * k_i)), 0.5, alpha, beta)

        assert bound_at(80) / bound_at(10) <= 0.25


# :194-200
def test_projector_bound_single_midpoint():
    f = adp.build_filter(0.1, 0.6, (-1.0, 1.0), 800, 0.5)
    assert adp.projector_bound(f, [math.acos(0.35)], 800) < 0.5
    with pytest.raises(adp.ConfigError):
        adp.projector_bound(f, [], 10)
    with pytest.raises(adp.ConfigError):
        adp.projector_bound(f, [1.0], 801)


# :202-224
def test_projector_bound_dominates_diagonal_projector_error(orc):
    rng = orc.MT19937_64(29)
    diag = [rng.uniform(-0.98, 0.98) for _ in range(60)]
    lo, hi = -0.3, 0.45
    f = adp.build_filter(lo, hi, (-1.0, 1.0), 120, 0.5)
    thetas = [math.acos(f.map_clamped(x)) for x in diag]
    for k_i in (20, 60, 120):
        p_err = 0.0
        for x in diag:
            s = 1.0 if lo < x < hi else (0.5 if x == lo or x == hi else 0.0)
            p_err = max(p_err, abs(s - adp.eval_filter_scalar(f, x, k_i)))
        assert p_err <= adp.projector_bound(f, thetas, k_i)


# :226-236
def test_projector_bound_non_increasing_in_degree():
    f = adp.build_filter(-0.2, 0.5, (-1.0, 1.0), 150, 0.5)
    thetas = [0.4, 1.0, 1.6, 2.2, 2.9]
    prev = math.inf
    for k_i in range(1, 151, 7):
        b = adp.projector_bound(f, thetas, k_i)
        assert b <= prev
        prev = b


# inspect-filter (cli.cpp:198-235)
def test_inspect_filter_sweep():
    rows = adp.inspect_filter(-0.2, 0.3, (-1.0, 1.0), k=60, m=0.5, samples=41)
    assert len(rows) == 41 and rows[0][0] == -1.0 and rows[-1][0] == 1.0
    f = adp.build_filter(-0.2, 0.3, (-1.0, 1.0), 60, 0.5)
    for x, rho, err, bound in rows:
        assert rho == adp.eval_filter_scalar(f, x, 60)
        if min(abs(x + 0.2), abs(x - 0.3)) > 1e-9:  # sound away from the (rounded) discontinuities
            assert err <= bound
    text = adp.inspect_filter_csv(-0.2, 0.3, (-1.0, 1.0), k=60, samples=2)
    assert text.splitlines()[0] == "x,rho,error,bound" and len(text.splitlines()) == 3
    assert adp.inspect_filter(-0.2, 0.3, samples=0) == []
    for bad in (dict(degree=0), dict(degree=101), dict(bounds=(1.0, -1.0)), dict(samples=-1)):
        with pytest.raises(adp.ConfigError):
            adp.inspect_filter(-0.2, 0.3, **bad)


# proj/tests/test_cli.cpp:218-269 (inspect-filter)
def test_inspect_filter_full_interval_rho_is_one():
    rows = adp.inspect_filter_csv(-1.0, 1.0, (-1.0, 1.0), k=40, m=0.5, samples=25).splitlines()
    assert len(rows) == 26 and rows[0] == "x,rho,error,bound"
    assert all(",1," in r for r in rows[1:])


def test_inspect_filter_zero_samples_header_only():
    assert adp.inspect_filter_csv(0.1, 0.6, samples=0) == "x,rho,error,bound\n"


def test_inspect_filter_error_dominated_by_bound():
    rows = adp.inspect_filter_csv(0.1, 0.6, (-1.0, 1.0), k=100, m=0.5, samples=500, sweep=(-0.1, 0.3)).splitlines()
    assert len(rows) == 501
    compared = 0
    for r in rows[1:]:
        x, rho, err, bound = (float(v) for v in r.split(","))
        if abs(x - 0.1) <= 1e-3:
            continue
        compared += 1
        assert err <= bound
    assert compared >= 490
