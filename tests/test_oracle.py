"""Pins for the CPU oracle (oracle/rhg_oracle.c) against things other than itself:
NVIDIA's Philox implementation, closed forms, printed examples (SPEC.md / SURVEY.md,
cited in tests/golden), 50-digit mpmath evaluation of the paper's literal Eq. 3,
brute force on tiny inputs, exact-integral expectations and invariants.
All CPU-only (no GPU marker)."""
import json
import math
import os
import shutil
import subprocess
import tempfile

import mpmath as mp
import numpy as np
import pytest
from scipy import stats

GOLD = os.path.join(os.path.dirname(__file__), "golden")
mp.mp.dps = 60


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------- RNG
CURAND_HOST = r"""
#define QUALIFIERS static inline
#define __device__
#define __forceinline__ inline
#include <vector_types.h>
#include <vector_functions.h>
#include <curand_philox4x32_x.h>
#include <stdio.h>
#include <stdlib.h>
int main(int argc, char** argv){
  unsigned long long seed = strtoull(argv[1], 0, 0);
  unsigned long long i0 = strtoull(argv[2], 0, 0), cnt = strtoull(argv[3], 0, 0);
  uint2 k = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
  for (unsigned long long i = i0; i < i0 + cnt; ++i) {
    uint4 c = make_uint4((unsigned)i, (unsigned)(i >> 32), 0, 0);
    uint4 o = curand_Philox4x32_10(c, k);
    printf("%u %u %u %u\n", o.x, o.y, o.z, o.w);
  }
}
"""


def _cuda_include():
    for p in ("/usr/local/cuda/include", "/usr/local/cuda-12.9/include"):
        if os.path.exists(os.path.join(p, "curand_philox4x32_x.h")):
            return p
    return None


@pytest.mark.skipif(_cuda_include() is None or shutil.which("g++") is None,
                    reason="curand headers or g++ missing")
@pytest.mark.parametrize("seed,i0", [(1, 0), (3, 0), (0x123456789ABCDEF0, 2**32 - 5),
                                     (5, 99_999_000)])
def test_philox_matches_curand_header(orc, seed, i0):
    """Pin: oracle Philox4x32-10 == NVIDIA curand_philox4x32_x.h (host-compiled),
    counter (i_lo, i_hi, 0, 0), key (seed_lo, seed_hi) -- Reading Z12."""
    d = tempfile.mkdtemp()
    src = os.path.join(d, "c.cpp")
    exe = os.path.join(d, "c")
    open(src, "w").write(CURAND_HOST)
    subprocess.run(["g++", "-O1", "-I", _cuda_include(), src, "-o", exe], check=True)
    cnt = 2000
    out = subprocess.run([exe, str(seed), str(i0), str(cnt)], check=True, capture_output=True,
                         text=True).stdout.split()
    ref = np.array(out, dtype=np.uint64).astype(np.uint32).reshape(cnt, 4)
    mine = orc.philox_words(seed, i0, cnt)
    assert np.array_equal(ref, mine)


def test_uniform_bit_mapping(orc):
    """u = (w_hi:w_lo >> 11) * 2^-53: closed-form corner cases (Reading Z12)."""
    a, b = orc.uniforms([0, 0, 0xFFFFFFFF, 0xFFFFFFFF])
    assert a == 0.0 and b == 1.0 - 2.0**-53
    a, b = orc.uniforms([1 << 11, 0, 0, 1 << 31])
    assert a == 2.0**-53 and b == 0.5


# --------------------------------------------------------------------------- params
def test_alpha_examples(orc):
    for g, a in gold("spec_examples.json")["alpha_from_gamma"]["cases"]:
        assert orc.alpha(g) == pytest.approx(a, abs=1e-15)


def test_target_radius_matches_survey(orc):
    """Pin: R for the five configs against the survey's independent mpmath
    bisection of Eq. 22."""
    for c in gold("survey_radii.json")["configs"]:
        R = orc.target_radius(c["n"], c["kbar"], orc.alpha(c["gamma"]))
        assert R == pytest.approx(c["R"], abs=2e-10)


def _kbar_mp(n, a, R):
    # Eq. 22 typed from PAPER.md:180-181 in 60-digit arithmetic (zeta = 1)
    n, a, R = mp.mpf(n), mp.mpf(a), mp.mpf(R)
    xi = a / (a - mp.mpf(1) / 2)
    pre = 2 / mp.pi * xi**2 * n
    return pre * mp.e**(-R / 2) + pre * (mp.e**(-a * R) *
                                         (a * R / 2 * (mp.pi / 4 / a**2 - (mp.pi - 1) / a + (mp.pi - 2)) - 1))


def test_kbar_formula_vs_mpmath(orc):
    for n, a, R in [(1e4, 1.0, 18.42), (1e6, 0.6, 26.5), (1e8, 0.85, 33.9), (50, 0.75, 3.0)]:
        assert orc.kbar_formula(n, a, R) == pytest.approx(float(_kbar_mp(n, a, R)), rel=1e-13)


def test_kbar_decreasing_on_search_branch(orc):
    """the formula decreases in R on the bracket searched."""
    for n, a in [(1e4, 1.0), (1e6, 0.6), (1e8, 0.85)]:
        Rs = np.linspace(3.0, 10 * math.log(n) + 50, 2000)
        k = np.array([orc.kbar_formula(n, a, R) for R in Rs])
        assert np.all(np.diff(k) < 0)


def _exact_mean_degree(n, a, R, m=1600):
    """(n-1) E[P(edge)] with P = dphi/pi from the LITERAL acos form of Eqs. 6-9
    (PAPER.md:205-208), by tensor Gauss-Legendre quadrature in x = R - r.
    Independent of Eq. 22 (an approximation) and of the oracle's stable window."""
    # density of x = R - r:  a sinh(a (R-x)) / (cosh aR - 1); mass concentrated near x=0
    xs, ws = [], []
    edges = np.concatenate([np.linspace(0, min(R, 12.0 / a), 40), [R]])
    edges = np.unique(edges)
    g, gw = np.polynomial.legendre.leggauss(m // len(edges) + 8)
    for lo, hi in zip(edges[:-1], edges[1:]):
        xs.append(0.5 * (hi - lo) * g + 0.5 * (hi + lo))
        ws.append(0.5 * (hi - lo) * gw)
    x = np.concatenate(xs)
    w = np.concatenate(ws)
    r = R - x
    f = a * np.sinh(a * r) / (np.cosh(a * R) - 1.0)
    r1, r2 = np.meshgrid(r, r, indexing="ij")
    with np.errstate(divide="ignore", invalid="ignore"):
        g_ = (np.cosh(r1) * np.cosh(r2) - np.cosh(R)) / (np.sinh(r1) * np.sinh(r2))
    P = np.where(g_ <= -1, 1.0, np.arccos(np.clip(g_, -1, 1)) / np.pi)
    return (n - 1) * np.einsum("i,j,ij->", w * f, w * f, P)


@pytest.mark.parametrize("idx", [0, 1, 3])
def test_target_radius_gives_kbar_in_expectation(orc, idx):
    """Pin (independent): exact expected mean degree at the oracle's R is within
    1% of the requested kbar (Eq. 22 is 'a close approximation', PAPER.md:184;
    SURVEY.md E-1 finds <= 0.36%)."""
    c = gold("survey_radii.json")["configs"][idx]
    a = orc.alpha(c["gamma"])
    R = orc.target_radius(c["n"], c["kbar"], a)
    E = _exact_mean_degree(c["n"], a, R)
    assert E == pytest.approx(c["kbar"], rel=0.01)
    assert E == pytest.approx(c["Edeg"], rel=2e-3)


def test_target_radius_errors(orc):
    with pytest.raises(ValueError):
        orc.target_radius(1e4, 6, 0.5)          # gamma = 2 -> alpha = 1/2
    with pytest.raises(ValueError):
        orc.target_radius(1e4, 0.6e4, 1.0)      # above the formula peak
    with pytest.raises(ValueError):
        orc.target_radius(1e4, -1, 1.0)


def test_boundaries_spec_example(orc):
    e = gold("spec_examples.json")["boundaries_L4_p09_R10"]
    c = orc.boundaries(10.0, 4, 0.9)
    assert np.allclose(c, e["value"], atol=e["tol"])
    c = orc.boundaries(24.9, 24, 0.9)
    w = np.diff(c)
    assert c[0] == 0 and c[-1] == 24.9
    assert np.allclose(w[1:-1] / w[:-2], 0.9, rtol=1e-9)


# --------------------------------------------------------------------------- sampler
def test_sampler_spec_example(orc):
    e = gold("spec_examples.json")["sample_radial_alpha1_R10_u05"]
    assert orc.radius_from_uniform(0.5, 1.0, 10.0) == pytest.approx(e["value"], abs=e["tol"])


@pytest.mark.parametrize("a,R", [(1.0, 10.0), (0.6, 26.49), (0.85, 33.94), (0.5 + 1e-9, 15.0)])
def test_sampler_inverts_closed_form_cdf(orc, a, R):
    """Pin: F(r(u)) = u with F(r) = (cosh a r - 1)/(cosh a R - 1), the CDF of Eq. 1
    (PAPER.md:66), evaluated at 60 digits."""
    for u in [0.0, 1e-300, 1e-12, 1e-3, 0.25, 0.5, 0.9, 1 - 2**-40, 1 - 2**-53]:
        r = orc.radius_from_uniform(u, a, R)
        assert 0.0 <= r <= R
        F = (mp.cosh(a * mp.mpf(r)) - 1) / (mp.cosh(a * mp.mpf(R)) - 1)
        # |dF/dr| * ulp(r) bounds the attainable agreement
        dF = a * mp.sinh(a * mp.mpf(r)) / (mp.cosh(a * mp.mpf(R)) - 1)
        tol = 8e-16 * max(u, 1e-300) + float(dF) * 8 * 2.3e-16 * max(r, 1e-300)
        assert abs(float(F) - u) <= tol + 1e-300


@pytest.mark.parametrize("a,R", [(0.5, 10.0), (0.75, 15.0), (1.0, 10.0), (1.0, 15.0)])
def test_sampler_ks(orc, a, R):
    """KS test of 1e5 radial samples against F passes at 0.01;
    angular marginal uniform on [0, 2pi)."""
    th, r = orc.sample_points(100_000, a, R, seed=11)
    F = lambda x: (np.cosh(a * x) - 1.0) / (np.cosh(a * R) - 1.0)
    assert stats.kstest(r, F).pvalue > 0.01
    assert stats.kstest(th / (2 * np.pi), "uniform").pvalue > 0.01
    assert th.min() >= 0 and th.max() < 2 * np.pi and r.min() >= 0 and r.max() <= R


def test_sampler_theta_below_two_pi(orc):
    """Reading Z10: theta = fl(2pi) * u with u <= 1 - 2^-53 stays < fl(2pi)."""
    w = [0xFFFFFFFF, 0xFFFFFFFF, 0, 0]
    u1, _ = orc.uniforms(w)
    assert 2 * math.pi * u1 < 2 * math.pi


# --------------------------------------------------------------------------- predicate
def _S_mp(t1, r1, t2, r2):
    """(cosh d - 1)/2 from the LITERAL Eq. 3 at 60 digits."""
    t1, r1, t2, r2 = map(mp.mpf, (t1, r1, t2, r2))
    cd = mp.cosh(r1) * mp.cosh(r2) - mp.sinh(r1) * mp.sinh(r2) * mp.cos(abs(t1 - t2))
    return (cd - 1) / 2


def test_predicate_trivial_cases(orc):
    """d(p,p)=0; antipodal equal radii d=2r; collinear d=|a-b|."""
    assert orc.S(0.7, 3.2, 0.7, 3.2) == 0.0
    for r in [0.5, 3.0, 12.0]:
        assert orc.S(0.0, r, math.pi, r) == pytest.approx(math.sinh(r) ** 2, rel=1e-14)
    for a_, b_ in [(1.0, 4.0), (7.5, 2.25)]:
        assert orc.S(1.3, a_, 1.3, b_) == pytest.approx(math.sinh((a_ - b_) / 2) ** 2, rel=1e-14)


def test_predicate_vs_literal_eq3_mpmath(orc):
    """Pin: the cancellation-free S agrees with the literal Eq. 3 at 60 digits to
    ~1e-14 relative on random pairs, including seam-crossing ones."""
    rng = np.random.default_rng(5)
    worst = 0.0
    for _ in range(3000):
        R = rng.choice([10.0, 24.9, 33.9])
        r1, r2 = rng.uniform(0, R, 2)
        t1 = rng.uniform(0, 2 * np.pi)
        t2 = (t1 + rng.choice([1.0, -1.0]) * 10 ** rng.uniform(-9, 0.5)) % (2 * np.pi)
        s = orc.S(t1, r1, t2, r2)
        ref = _S_mp(t1, r1, t2, r2)
        worst = max(worst, abs(s - float(ref)) / float(ref))
    assert worst < 2e-14


def test_predicate_vs_literal_eq3_quad(orc):
    """The oracle's own __float128 literal Eq. 3 agrees with its stable S."""
    rng = np.random.default_rng(6)
    for _ in range(2000):
        r1, r2 = rng.uniform(0, 20, 2)
        t1, t2 = rng.uniform(0, 2 * np.pi, 2)
        cd, _ = orc.cosh_dist_literal_quad(t1, r1, t2, r2)
        assert (cd - 1) / 2 == pytest.approx(orc.S(t1, r1, t2, r2), rel=1e-13)


def test_angle_between_seam(orc):
    """Reading Z13: seam-crossing distance (2pi - max) + min at full precision."""
    for a_ in [1e-12, 3e-9, 1e-3]:
        for b_ in [0.0, 2e-12, 5e-9]:
            t1 = float(2 * mp.pi - a_)
            exact = (2 * mp.pi - mp.mpf(t1)) + b_
            got = orc.angle_between(t1, b_)
            assert abs(got - float(exact)) <= 4e-16 * float(exact)
            assert orc.angle_between(b_, t1) == got


def _near_pairs(R, n, seed):
    """Pairs built to sit at S = T (1 + eps) for tiny eps."""
    rng = np.random.default_rng(seed)
    T = mp.sinh(mp.mpf(R) / 2) ** 2
    out = []
    while len(out) < n:
        r1, r2 = rng.uniform(R / 3, R, 2)
        eps = rng.choice([0.0, 1e-15, -1e-15, 1e-13, -1e-13, 1e-11, -1e-11, 1e-9])
        rhs = (T * (1 + mp.mpf(eps)) - mp.sinh((mp.mpf(r1) - r2) / 2) ** 2) / (mp.sinh(r1) * mp.sinh(r2))
        if not (0 < rhs < 1):
            continue
        d = 2 * mp.asin(mp.sqrt(rhs))
        t1 = rng.uniform(0, 2 * np.pi)
        if rng.random() < 0.2:
            t1 = float(2 * mp.pi - d / 3)  # straddle the seam
        t2 = float(mp.mpf(t1) + d)
        if t2 >= 2 * np.pi:
            t2 = float(mp.mpf(t2) - 2 * mp.pi)
        out.append((t1, float(r1), t2, float(r2)))
    return out


@pytest.mark.parametrize("R", [16.7052678863, 24.8952454068, 33.9421594033])
def test_decision_on_near_threshold_pairs(orc, R):
    """Pin: oracle decisions == 60-digit literal Eq. 3 decisions on pairs built
    within 1e-9..0 of the threshold; the tie flag is raised exactly inside the
    north-star window |cosh d - cosh R| <= 1e-12 cosh R (plus margin)."""
    coshR = mp.cosh(mp.mpf(R))
    for (t1, r1, t2, r2) in _near_pairs(R, 400, seed=int(R * 1000)):
        S = _S_mp(t1, r1, t2, r2)
        truth = 2 * S + 1 <= coshR
        e, tie = orc.is_edge(t1, r1, t2, r2, R)
        assert e == truth
        rel = abs(2 * S + 1 - coshR) / coshR
        if rel <= 0.99e-12:
            assert tie
        if rel > 1.1e-12:
            assert not tie


# --------------------------------------------------------------------------- edge sets
def _mp_brute(theta, r, R):
    coshR = mp.cosh(mp.mpf(R))
    E = []
    for i in range(len(theta)):
        for j in range(i + 1, len(theta)):
            if 2 * _S_mp(theta[i], r[i], theta[j], r[j]) + 1 <= coshR:
                E.append((i, j))
    return np.array(E, dtype=np.uint32).reshape(-1, 2)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_brute_force_vs_mpmath_tiny(orc, seed):
    """Pin: brute force == pure-Python 60-digit literal Eq. 3 on tiny inputs."""
    mp.mp.dps = 40
    rng = np.random.default_rng(seed)
    for R in [4.0, 12.0, 16.7052678863]:
        n = 45
        th = rng.uniform(0, 2 * np.pi, n)
        th[:4] = [0.0, 2 * np.pi - 1e-9, 1e-9, np.nextafter(2 * np.pi, 0)]
        r = np.concatenate([rng.uniform(0, R, n // 2), R - rng.exponential(1.0, n - n // 2)])
        r = np.clip(r, 0, R)
        es = orc.brute_force(th, r, R)
        ref = _mp_brute(th, r, R)
        assert np.array_equal(es.pairs, ref)
    mp.mp.dps = 60


@pytest.mark.parametrize("gamma,kbar,n,seed", [(3.0, 6, 10_000, 1), (2.2, 8, 8_000, 7),
                                                (2.7, 16, 20_000, 9), (3.0, 40, 5_000, 4)])
def test_sweep_equals_brute_force(orc, gamma, kbar, n, seed):
    a = orc.alpha(gamma)
    R = orc.target_radius(n, kbar, a)
    th, r = orc.sample_points(n, a, R, seed)
    bf = orc.brute_force(th, r, R)
    sw = orc.sweep(th, r, R)
    assert np.array_equal(bf.pairs, sw.pairs)


def test_special_cases_complete_and_empty(orc):
    """huge R -> complete graph; R = 0 -> no edges."""
    rng = np.random.default_rng(0)
    n = 50
    th = rng.uniform(0, 2 * np.pi, n)
    R = 10 * math.log(n) + 50
    r = rng.uniform(0, R / 2.01, n)        # every pair has r1 + r2 < R  =>  d <= R
    es = orc.sweep(th, r, R)
    assert es.m == n * (n - 1) // 2
    es0 = orc.brute_force(th, rng.uniform(0, 1, n), 0.0)
    assert es0.m == 0


def test_rows_match_brute_force(orc):
    a = 1.0
    R = orc.target_radius(3000, 10, a)
    th, r = orc.sample_points(3000, a, R, 21)
    bf = orc.brute_force(th, r, R)
    q = np.array([0, 5, 17, 2999, int(np.argmin(r))], dtype=np.uint32)
    off, nbr, _ = orc.rows(th, r, R, q)
    for k, v in enumerate(q):
        ref = np.sort(np.concatenate([bf.pairs[bf.pairs[:, 0] == v, 1], bf.pairs[bf.pairs[:, 1] == v, 0]]))
        assert np.array_equal(nbr[off[k]:off[k + 1]], ref)


def test_invariants_mean_degree_and_tail(orc):
    """North star: no self-loops, each edge once, mean degree ~ kbar (Reading Z14:
    sigma-aware), tail exponent ~ gamma (SPEC.md:434-435 bands)."""
    for gamma, band in [(3.0, (2.7, 3.3)), (2.2, (1.9, 2.6))]:
        a = orc.alpha(gamma)
        n, kbar = 100_000, 10
        R = orc.target_radius(n, kbar, a)
        degs = []
        for seed in (1, 2, 3):
            th, r = orc.sample_points(n, a, R, seed)
            es = orc.sweep(th, r, R)
            p = es.pairs
            assert np.all(p[:, 0] < p[:, 1])
            key = p[:, 0].astype(np.uint64) * n + p[:, 1]
            assert len(np.unique(key)) == len(key)
            deg = np.bincount(p.ravel(), minlength=n)
            degs.append(deg)
        mean = np.mean([d.mean() for d in degs])
        E = _exact_mean_degree(n, a, R)
        assert mean == pytest.approx(E, rel=0.06)
        assert E == pytest.approx(kbar, rel=0.01)
        k = np.concatenate(degs)
        kmin = 2 * kbar
        tail = k[k >= kmin]
        mle = 1 + len(tail) / np.sum(np.log(tail / (kmin - 0.5)))
        assert band[0] <= mle <= band[1]


# ------------------------------------------------------------------ next rows (f1, f2)
def test_radius_from_C_closed_form(orc):
    """R = 2 ln n + C: n = e^5, C = 0 gives R = 10; C shifts R."""
    assert orc.radius_from_C(np.exp(5.0), 0.0) == pytest.approx(10.0, abs=1e-12)
    assert orc.radius_from_C(np.exp(5.0), -1.5) == pytest.approx(8.5, abs=1e-12)


def test_rotate_spec_example_and_range(orc):
    """rotated(phi, tau) = (phi + tau) mod 2pi."""
    assert orc.rotate(1.0, 0.0) == 1.0
    assert orc.rotate(6.0, 1.0) == pytest.approx(7.0 - 2 * np.pi, abs=1e-15)   # 0.7168
    assert orc.rotate(0.5, -1.0) == pytest.approx(2 * np.pi - 0.5, abs=1e-15)
    rng = np.random.default_rng(4)
    for phi, tau in zip(rng.uniform(0, 2 * np.pi, 2000), rng.uniform(-1, 1, 2000)):
        x = orc.rotate(phi, tau)
        assert 0.0 <= x < 2 * np.pi
        assert np.cos(x) == pytest.approx(np.cos(phi + tau), abs=1e-12)


def test_radial_step_algorithm2(orc):
    """Alg. 2: SPEC.md:356 example, identity for tau = 0, and the
    inverse move (r, tau) then (r', -tau) without reflection."""
    r1, t1 = orc.radial_step(1.0, 1.0, 10.0, 1.0)
    assert r1 == pytest.approx(1.5194, abs=1e-4) and t1 == 1.0
    assert r1 == pytest.approx(np.arcsinh(np.sinh(1.0) + 1.0), abs=1e-15)
    rng = np.random.default_rng(5)
    for a in (0.6, 1.0, 1.7):
        R = 20.0
        for r, tau in zip(rng.uniform(5, 19, 200), rng.uniform(-1, 1, 200)):  # no reflection
            assert orc.radial_step(r, 0.0, R, a) == (pytest.approx(r, rel=4e-15), 0.0)
            r2, t2 = orc.radial_step(r, tau, R, a)
            r3, t3 = orc.radial_step(r2, -t2, R, a)
            assert t2 == tau and r3 == pytest.approx(r, rel=1e-12)


def test_radial_step_reflection(orc):
    """Reflection: the result stays in [0, R]; tau flips iff the
    transformed coordinate left [0, sinh(alpha R)] (Reading D2, folded back)."""
    R, a = 10.0, 1.0
    S = np.sinh(a * R)
    r, t = orc.radial_step(0.5, -3.0, R, a)        # y = sinh(0.5) - 3 < 0 -> folded at 0
    assert t == 3.0 and r == pytest.approx(np.arcsinh(3.0 - np.sinh(0.5)), rel=1e-14)
    r, t = orc.radial_step(R - 1e-3, 1e3, R, a)    # y > S -> folded at S
    assert t == -1e3 and r == pytest.approx(np.arcsinh(2 * S - np.sinh(R - 1e-3) - 1e3), rel=1e-12)
    rng = np.random.default_rng(6)
    for r0, tau in zip(rng.uniform(0, R, 3000), rng.uniform(-50, 50, 3000)):
        r1, t1 = orc.radial_step(r0, tau, R, a)
        assert 0.0 <= r1 <= R
        y = np.sinh(a * r0) + tau
        assert (t1 == -tau) == (y < 0 or y > S)


def test_movement_init_ranges(orc):
    """Step values uniform on the Appendix B ranges, Philox
    counter (i, 1) so they are independent of the point sample (counter (i, 0))."""
    tp, tr = orc.movement_init(50_000, 3)
    assert tp.min() >= -1 and tp.max() < 1 and tr.min() >= -10 and tr.max() < 1
    assert stats.kstest((tp + 1) / 2, "uniform").pvalue > 1e-3
    assert stats.kstest((tr + 10) / 11, "uniform").pvalue > 1e-3
    w = orc.philox4x32_10([7, 0, 1, 0], [3, 0])
    u1 = (int(w[1]) << 32 | int(w[0])) >> 11
    assert tp[7] == pytest.approx(-1 + 2 * u1 * 2.0**-53, abs=0)


def test_theorem1_distribution_preserved(orc):
    """Theorem 1: 100 movement steps of 10^4 vertices keep the
    radial marginal at F(r) and the angular one uniform (KS at 0.01)."""
    n, a = 10_000, 1.0
    R = 2 * np.log(n) + 2
    th, r = orc.sample_points(n, a, R, 7)
    tp, tr = orc.movement_init(n, 9)
    F = lambda x: (np.cosh(a * x) - 1) / (np.cosh(a * R) - 1)
    crit = 1.628 / np.sqrt(n)
    for _ in range(100):
        th, r, tr = orc.move_points(th, r, tp, tr, R, a)
        assert stats.kstest(r, F).statistic < crit
    assert stats.kstest(th / (2 * np.pi), "uniform").statistic < crit


# ------------------------------------------------------------------ pins added in round 2
# orc_window, orc_sweep_count(_ordered), orc_row_ties, orc_sweep_csr, orc_sweep_digest,
# orc_mix64 (VERDICT r01 "Pin the rest of the oracle").
def _window_literal_mp(r, c, R):
    """Eqs. 6-9 as printed: the angular half-width at which a
    point at radius c is at distance R from a point at radius r,
    acos((cosh r cosh c - cosh R) / (sinh r sinh c)), at 50 digits; pi if the
    argument is <= -1 (whole circle) or sinh r sinh c = 0, 0 if it is >= 1."""
    with mp.workdps(50):
        r, c, R = mp.mpf(r), mp.mpf(c), mp.mpf(R)
        den = mp.sinh(r) * mp.sinh(c)
        if den == 0:
            return mp.pi
        g = (mp.cosh(r) * mp.cosh(c) - mp.cosh(R)) / den
        if g <= -1:
            return mp.pi
        if g >= 1:
            return mp.mpf(0)
        return mp.acos(g)


@pytest.mark.parametrize("R", [16.7052678863, 24.8952454068, 33.9421594033])
def test_window_vs_literal_eq6_9_mpmath(orc, R):
    """Pin orc_window (the stable asin form, Reading Z3) against the paper's literal
    acos form at 50 digits, over (r, c) spanning the disk (relative error 1e-12
    where the window is not tiny; absolute 1e-15 near 0), plus the special cases:
    c = 0 and r + c <= R are the full circle, |r - c| > R... cannot happen in the
    disk, r = c = R gives the single point (window 2 asin(sqrt(T/sinh^2 R)))."""
    rng = np.random.default_rng(int(R * 7))
    worst = 0.0
    for _ in range(600):
        r = float(rng.uniform(0, R))
        c = float(rng.uniform(0, R)) if rng.random() < 0.7 else float(R - rng.exponential(0.5))
        c = min(max(c, 0.0), R)
        got = orc.window(r, c, R)
        ref = float(_window_literal_mp(r, c, R))
        if ref > 1e-6:
            worst = max(worst, abs(got - ref) / ref)
        else:
            assert abs(got - ref) <= 1e-15
    assert worst < 1e-12
    # full circle: c = 0, and any pair with r + c <= R (then cosh(r + c) <= cosh R)
    assert orc.window(5.0, 0.0, R) == math.pi
    assert orc.window(R / 2 - 1e-6, R / 2 - 1e-6, R) == math.pi
    assert orc.window(0.0, 3.0, R) == math.pi
    # r = c = R: two boundary points at distance <= R iff the angle is <= this
    ref = float(_window_literal_mp(R, R, R))
    assert orc.window(R, R, R) == pytest.approx(ref, rel=1e-12)
    # monotone decreasing in c
    cs = np.linspace(0.1, R, 200)
    w = [orc.window(R * 0.9, c, R) for c in cs]
    assert all(a >= b for a, b in zip(w, w[1:]))


def _owner_filtered_count(th, r, pairs, lo, hi):
    """Edges whose smaller-(r, id) endpoint has id in [lo, hi)."""
    u, v = pairs[:, 0].astype(np.int64), pairs[:, 1].astype(np.int64)
    own = np.where((r[u] < r[v]) | ((r[u] == r[v]) & (u < v)), u, v)
    return int(np.count_nonzero((own >= lo) & (own < hi)))


@pytest.mark.parametrize("gamma,kbar,n,seed", [(3.0, 6, 10_000, 1), (2.2, 8, 8_000, 7),
                                                (2.7, 16, 20_000, 9)])
def test_sweep_count_equals_owner_filtered_brute_force(orc, gamma, kbar, n, seed):
    """Pin orc_sweep_count / orc_sweep_count_ordered (the CPU-baseline timer): for
    several id ranges, the count equals the number of brute-force edges owned by
    the range (owner = smaller (r, id) endpoint), and the
    full range counts every edge."""
    a = orc.alpha(gamma)
    R = orc.target_radius(n, kbar, a)
    th, r = orc.sample_points(n, a, R, seed)
    bf = orc.brute_force(th, r, R)
    order, pos = orc.angle_order(th)
    assert np.array_equal(order[pos], np.arange(n))
    assert np.all(np.diff(th[order]) >= 0)
    for lo, hi in [(0, n), (0, 1), (17, 4000), (n // 2, n), (n - 3, n), (5, 5)]:
        ref = _owner_filtered_count(th, r, bf.pairs, lo, hi)
        m, tests = orc.sweep_count(th, r, R, lo, hi)
        assert m == ref
        m2, tests2 = orc.sweep_count_ordered(th, r, R, order, pos, lo, hi)
        assert (m2, tests2) == (m, tests)
        assert tests >= m
    assert orc.sweep_count(th, r, R, 0, n)[0] == bf.m


@pytest.mark.parametrize("gamma,kbar,n,seed", [(3.0, 6, 10_000, 1), (2.2, 8, 8_000, 7),
                                                (2.7, 16, 20_000, 9), (3.0, 40, 5_000, 4)])
def test_sweep_csr_equals_brute_force(orc, gamma, kbar, n, seed):
    """Pin orc_sweep_csr: the CSR built from brute-force pairs (both directions,
    rows ascending) is identical, and so is the near-tie list."""
    a = orc.alpha(gamma)
    R = orc.target_radius(n, kbar, a)
    th, r = orc.sample_points(n, a, R, seed)
    bf = orc.brute_force(th, r, R)
    c = orc.sweep_csr(th, r, R)
    u = np.concatenate([bf.pairs[:, 0], bf.pairs[:, 1]]).astype(np.uint64)
    v = np.concatenate([bf.pairs[:, 1], bf.pairs[:, 0]]).astype(np.uint64)
    key = np.sort((u << np.uint64(32)) | v)
    deg = np.bincount(u.astype(np.int64), minlength=n)
    assert np.array_equal(c.row_ptr, np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64))
    assert np.array_equal(c.col, (key & np.uint64(0xFFFFFFFF)).astype(np.uint32))
    tk = lambda t: sorted(map(tuple, t.tolist()))
    assert tk(c.ties) == tk(bf.ties)


def _mix64_np(w):
    """SplitMix64 finaliser, retyped in numpy (wrapping uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        z = w.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x632BE59BD9B4E019)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def test_mix64_known_values(orc):
    """orc_mix64(w) = SplitMix64's output function of the state w * golden + inc.
    Pins: equality with the numpy retyping for w = 0..1999, and the finaliser's
    published first output of SplitMix64 from seed 0 (state = golden ratio
    constant) = 0xE220A8397B1DCDAF."""
    w = np.arange(2000, dtype=np.uint64)
    got = np.array([orc.mix64(int(x)) for x in w], dtype=np.uint64)
    assert np.array_equal(got, _mix64_np(w))
    with np.errstate(over="ignore"):
        z = np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    assert int(z) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("gamma,kbar,n,seed", [(2.7, 16, 20_000, 9), (2.2, 8, 8_000, 7)])
def test_sweep_digest_equals_brute_force(orc, gamma, kbar, n, seed):
    """Pin orc_sweep_digest: degrees and neighbour-set digests equal the ones
    computed in numpy from the brute-force pairs; a single moved edge changes the
    digest of both endpoints."""
    a = orc.alpha(gamma)
    R = orc.target_radius(n, kbar, a)
    th, r = orc.sample_points(n, a, R, seed)
    bf = orc.brute_force(th, r, R)
    m, deg, dig, ties, _ = orc.sweep_digest(th, r, R)
    assert m == bf.m
    u, v = bf.pairs[:, 0].astype(np.int64), bf.pairs[:, 1].astype(np.int64)
    assert np.array_equal(deg, np.bincount(np.concatenate([u, v]), minlength=n).astype(np.uint64))
    ref = np.zeros(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        np.add.at(ref, u, _mix64_np(v))
        np.add.at(ref, v, _mix64_np(u))
    assert np.array_equal(dig, ref)
    assert sorted(map(tuple, ties.tolist())) == sorted(map(tuple, bf.ties.tolist()))
    # sensitivity: replacing one neighbour changes the digest
    with np.errstate(over="ignore"):
        alt = ref[u[0]] - _mix64_np(v[:1])[0] + _mix64_np(np.array([v[0] + 1]))[0]
    assert alt != ref[u[0]]


def test_row_ties_equals_brute_force(orc):
    """Pin orc_row_ties: for vertices with planted near-threshold partners (pairs
    built at S = T (1 + eps), as SURVEY.md E-11), the tie list equals the set of w
    whose pair is flagged by orc_is_edge (itself pinned at 60 digits above), with
    the same quad decision, and equals brute force's tie list restricted to v."""
    R = 24.8952454068
    rng = np.random.default_rng(77)
    n0 = 3000
    th, r = orc.sample_points(n0, 1.0, R, 12)
    planted = _near_pairs(R, 40, seed=5)
    th = np.concatenate([th] + [[p[0], p[2]] for p in planted]).astype(np.float64)
    r = np.concatenate([r] + [[p[1], p[3]] for p in planted]).astype(np.float64)
    n = len(th)
    bf = orc.brute_force(th, r, R)
    assert len(bf.ties) > 0
    qs = list(range(n0, n, 7)) + [0, 1, 2]
    for v in qs:
        w, e = orc.row_ties(th, r, R, v)
        ref = []
        for x in range(n):
            if x == v:
                continue
            ee, tie = orc.is_edge(th[v], r[v], th[x], r[x], R)
            if tie:
                ref.append((x, ee))
        assert sorted(zip(w.tolist(), e.tolist())) == sorted(ref)
        bt = {(int(a_), int(b_)) for a_, b_ in bf.ties.tolist() if v in (a_, b_)}
        assert {(min(v, x), max(v, x)) for x in w.tolist()} == bt
    del rng
