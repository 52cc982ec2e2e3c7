"""Pins of the oracle's Eq. 1 (O2/O3) to things other than itself:
paper worked examples (tests/golden), closed forms, invariants, and an
independent brute-force K×K implementation (oracle/c)."""
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import oracle_c as oc
from oracle import ragb_oracle as o

A200 = Fraction(1, 200)


def f32hex(x):
    return hex(int(np.array(x, dtype=np.float32).view(np.uint32)))


def test_paper_motivation_example(golden):
    g = golden["eq1_motivation"]
    c = g["contexts"]
    a = Fraction(golden["alpha"]["num"], golden["alpha"]["den"])
    # printed: overlap-only metric is 0.5 for A-B, B-C, B-D
    for p, q in [("A", "B"), ("B", "C"), ("B", "D")]:
        s, _ = o.overlap(c[p], c[q])
        assert Fraction(s, 4) == Fraction(g["printed"]["naive_overlap_distance_AB_BC_BD"])
    # printed: B-D < A-B
    assert o.distance(c["B"], c["D"], a) < o.distance(c["A"], c["B"], a)
    for pair, v in g["derived"].items():
        p, q = pair[0], pair[1]
        s, D = o.overlap(c[p], c[q])
        assert (s, D) == (v["s"], v["D"])
        exact = o.distance_exact(c[p], c[q], a)
        assert exact == Fraction(v["d_num"], v["d_den"])
        if "f32_hex" in v:
            assert f32hex(o.distance(c[p], c[q], a)) == v["f32_hex"]


def test_fig4_distances(golden):
    g = golden["fig4_build"]
    C = g["contexts"]
    a = A200
    dv = g["derived"]
    assert o.distance_exact(C[0], C[1], a) == Fraction(dv["d01"]["d_num"], dv["d01"]["d_den"])
    assert f32hex(o.distance(C[0], C[1], a)) == dv["d01"]["f32_hex"]
    assert o.distance_exact(C[0], C[2], a) == Fraction(dv["d02"]["d_num"], dv["d02"]["d_den"])
    assert o.distance_exact(C[1], C[2], a) == Fraction(dv["d12"]["d_num"], dv["d12"]["d_den"])
    # printed: C1 and C2 have the smallest distance
    d01 = o.distance(C[0], C[1], a)
    assert d01 < o.distance(C[0], C[2], a) and d01 < o.distance(C[1], C[2], a)


@pytest.mark.parametrize("K", [1, 2, 3, 5, 10, 20, 33, 100])
def test_closed_forms(K):
    rng = np.random.default_rng(K)
    base = [int(x) for x in rng.permutation(1000)[:K]]
    # identical -> 0
    assert o.distance_exact(base, base, A200) == 0
    # disjoint -> exactly 1 (X3)
    other = [x + 5000 for x in base]
    assert o.distance(base, other, A200) == np.float32(1.0)
    # reversed list: alpha * floor(K^2/2) / K (Spearman footrule of the reversal)
    rev = base[::-1]
    assert o.distance_exact(base, rev, A200) == A200 * Fraction(K * K // 2, K)
    # arbitrary permutation sigma: alpha * F(sigma) / K with F = sum |i - sigma(i)|
    sigma = rng.permutation(K)
    perm = [base[int(i)] for i in sigma]
    F = sum(abs(int(sigma[i]) - i) for i in range(K))
    assert o.distance_exact(base, perm, A200) == A200 * Fraction(F, K)
    # one shared doc at positions (0, K-1): 1 - 1/K + alpha (K - 1)   (X16)
    if K >= 2:
        x = [1] + [100 + i for i in range(K - 1)]
        y = [200 + i for i in range(K - 1)] + [1]
        assert o.distance_exact(x, y, A200) == 1 - Fraction(1, K) + A200 * (K - 1)


def test_rn32_is_correct_rounding():
    # exact midpoints between consecutive floats round to even
    for f in [np.float32(0.3), np.float32(1.0), np.float32(0.51), np.float32(1.045)]:
        g = np.nextafter(f, np.float32(2))
        mid = (Fraction(float(f)) + Fraction(float(g))) / 2
        r = o.rn32(mid)
        even = f if (int(np.array(f).view(np.uint32)) & 1) == 0 else g
        assert r == even
        assert oc.rn32_ratio(mid.numerator, mid.denominator) == even
        # just above / below the midpoint
        eps = Fraction(1, 2 ** 60)
        assert o.rn32(mid + eps) == g and o.rn32(mid - eps) == f
        assert oc.rn32_ratio((mid + eps).numerator, (mid + eps).denominator) == g
    # exactly representable values are returned unchanged
    for v in [Fraction(1, 2), Fraction(3, 4), Fraction(1), Fraction(0)]:
        assert o.rn32(v) == np.float32(float(v))


def test_rn32_random_c_vs_python():
    rng = np.random.default_rng(7)
    for _ in range(3000):
        den = int(rng.integers(1, 2 ** 26))
        num = int(rng.integers(0, 4 * den))
        assert oc.rn32_ratio(num, den) == o.rn32(Fraction(num, den))


ctx_strategy = st.integers(1, 12).flatmap(
    lambda K: st.tuples(
        st.lists(st.integers(0, 20), min_size=1, max_size=K, unique=True),
        st.lists(st.integers(0, 20), min_size=1, max_size=K, unique=True)))


@settings(max_examples=400, deadline=None)
@given(ctx_strategy)
def test_properties(pair):
    ci, cj = pair
    d = o.distance_exact(ci, cj, A200)
    assert d == o.distance_exact(cj, ci, A200)  # symmetry
    s, D = o.overlap(ci, cj)
    assert s <= min(len(ci), len(cj))
    m = max(len(ci), len(cj))
    # bounds (X16): 0 <= d <= max(1, 1 - 1/m + alpha (m-1))
    assert 0 <= d <= max(Fraction(1), 1 - Fraction(1, m) + A200 * (m - 1))
    # brute-force K x K (independent C implementation) agrees on s, D, d
    K = max(len(ci), len(cj))
    ids = np.zeros((2, K), dtype=np.uint32)
    ids[0, :len(ci)] = ci
    ids[1, :len(cj)] = cj
    lens = np.array([len(ci), len(cj)], dtype=np.uint8)
    dd, ss, DD = oc.pairwise_rows(ids, lens, 1, 200, counts=True)
    assert (int(ss[0, 1]), int(DD[0, 1])) == (s, D)
    assert dd[0, 1] == o.rn32(d) and dd[1, 0] == dd[0, 1]
    assert dd[0, 0] == 0 and dd[1, 1] == 0


def test_pairwise_c_matches_python_on_workload():
    from synth.workload import config
    w = config("C1")
    ctxs = o.validate(w.ids)
    S, Dm, d = o.pairwise(ctxs, A200)
    dc, sc, Dc = oc.pairwise_rows(w.ids, None, 1, 200, counts=True)
    assert np.array_equal(S, sc) and np.array_equal(Dm, Dc)
    assert np.array_equal(d.view(np.uint32), dc.view(np.uint32))
    assert np.array_equal(d, d.T) and np.all(np.diag(d) == 0)
    # row nn: python definition vs C
    i1, v1 = o.row_nn(d)
    i2, v2 = oc.row_nn(dc)
    assert np.array_equal(i1, i2) and np.array_equal(v1, v2)


def test_variable_length_and_alpha_band():
    from synth.workload import generate
    w = generate(48, 8, 60, 11, len_min=3)
    ctxs = o.validate(w.ids, w.lens)
    for a in [Fraction(1, 1000), Fraction(1, 100), Fraction(3, 700)]:
        _, _, d = o.pairwise(ctxs, a)
        dc = oc.pairwise_rows(w.ids, w.lens, a.numerator, a.denominator)
        assert np.array_equal(d.view(np.uint32), dc.view(np.uint32))


def test_validate_rejects():
    with pytest.raises(o.OracleError):
        o.validate(np.array([[1, 2, 1]], dtype=np.uint32))
    with pytest.raises(o.OracleError):
        o.validate(np.array([[1, 0xFFFFFFFF]], dtype=np.uint32))
    with pytest.raises(o.OracleError):
        o.validate(np.array([[1, 2]], dtype=np.uint32), lens=np.array([0], dtype=np.uint8))
