"""Pins the CPU oracle (oracle/) against the reference.

(1) golden vectors produced by the reference's own gf2.hpp / rng.hpp
    (tests/golden/ref_gf2_rng.json, made by tests/golden/make_golden.py);
(2) the known-answer and property tests of proj/tests/test_gf2.cpp,
    test_fwht.cpp, test_kerdock.cpp (cited per test).
CPU only.
"""
import itertools
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ref_gf2_rng.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


# ----------------------------------------------------------- golden vectors --
def test_rng_stream_matches_reference_binary(orc, golden):
    for rec in golden["rng"]:
        seed = int(rec["seed"])
        u = orc.rng_u64(seed, len(rec["u64"]))
        assert [int(v) for v in u] == [int(v) for v in rec["u64"]]
        for bound, draws in rec["index"].items():
            got = orc.rng_index(seed, int(bound), len(draws))
            assert got.tolist() == draws, (seed, bound)
        assert orc.rng_gaussian(seed, len(rec["gaussian"])).tolist() == rec["gaussian"]
        assert orc.rng_unit_double(seed, len(rec["unit_double"])).tolist() == rec["unit_double"]
        assert orc.rng_coin(seed, len(rec["coin"])).tolist() == rec["coin"]
        assert orc.mix_seed(seed) == int(rec["mix_seed"])


def test_field_matches_reference_binary(orc, golden):
    for rec in golden["field"]:
        q = rec["q"]
        assert orc.modulus_for_degree(q) == int(rec["modulus"])
        assert orc.verify_irreducible(int(rec["modulus"]), q) == bool(rec["irreducible"])
        for a, b, p, t in zip(rec["a"], rec["b"], rec["mul"], rec["trace"]):
            assert orc.field_mul(q, int(a), int(b)) == int(p)
            assert orc.field_trace(q, int(a)) == int(t)


def test_coords_and_rank_match_reference_binary(orc, golden):
    for k, p, w in golden["coords"]:
        p &= (1 << k) - 1  # the generator masks p to k bits
        assert orc.coords_of_position(p, k) == w
        assert orc.position_of_coords(w, k) == p
    for rec in golden["rank"]:
        assert orc.gf2_rank([int(r) for r in rec["rows"]]) == rec["rank"]


# ------------------------------------------------------------- test_gf2.cpp --
def _naive_mul_mod(a, b, modulus, q):  # test_gf2.cpp:13-23
    prod = 0
    for i in range(q):
        for j in range(q):
            if (a >> i) & 1 and (b >> j) & 1:
                prod ^= 1 << (i + j)
    for d in range(2 * q - 2, q - 1, -1):
        if (prod >> d) & 1:
            prod ^= modulus << (d - q)
    return prod


def test_field_mul_fixed_values(orc):  # test_gf2.cpp:79-87
    assert orc.modulus_for_degree(3) == 0b1011
    assert orc.field_mul(3, 2, 4) == 3
    assert orc.field_mul(3, 1, 6) == 6
    assert orc.field_mul(3, 0, 5) == 0


def test_field_mul_exhaustive_vs_schoolbook(orc):  # test_gf2.cpp:89-97
    for q in (1, 3, 5):
        mod = orc.modulus_for_degree(q)
        for a, b in itertools.product(range(1 << q), repeat=2):
            assert orc.field_mul(q, a, b) == _naive_mul_mod(a, b, mod, q)
    q, mod = 7, orc.modulus_for_degree(7)
    rng = np.random.default_rng(1)
    for a, b in rng.integers(0, 128, size=(2000, 2)):
        assert orc.field_mul(q, int(a), int(b)) == _naive_mul_mod(int(a), int(b), mod, q)


def test_irreducibility(orc):  # test_gf2.cpp:60-77
    assert orc.verify_irreducible(0b111, 2)
    assert not orc.verify_irreducible(0b101, 2)
    assert orc.verify_irreducible(0b1011, 3)
    assert not orc.verify_irreducible(0b1111, 3)
    assert not orc.verify_irreducible(0b1001, 3)
    for q in (1, 3, 5, 7, 9, 11, 13, 15):
        assert orc.verify_irreducible(orc.modulus_for_degree(q), q)
    with pytest.raises(ValueError):
        orc.modulus_for_degree(4)


def test_trace_fixed_and_frobenius(orc):  # test_gf2.cpp:117-142
    assert orc.field_trace(3, 0) == 0
    assert orc.field_trace(3, 1) == 1
    assert orc.field_trace(3, 2) == 0
    for q in (1, 3, 5, 7):
        for a in range(1 << q):
            assert orc.field_trace(q, orc.field_mul(q, a, a)) == orc.field_trace(q, a)


def test_big_endian_map(orc):  # test_gf2.cpp:156-166
    for p in range(16):
        assert orc.position_of_coords(orc.coords_of_position(p, 4), 4) == p
    w = orc.coords_of_position(1, 4)
    assert (w >> 3) & 1 == 1 and w & 1 == 0


def test_rank_fixed(orc):  # test_gf2.cpp:29-40
    assert orc.gf2_rank([0, 0, 0, 0]) == 0
    assert orc.gf2_rank([1, 2, 4, 8]) == 4
    assert orc.gf2_rank([0b10, 0b01]) == 2


# ------------------------------------------------------------ test_fwht.cpp --
def _naive_walsh(v):  # test_fwht.cpp:15-28
    d = len(v)
    out = np.zeros(d)
    for q in range(d):
        out[q] = sum(-v[x] if bin(q & x).count("1") & 1 else v[x] for x in range(d))
    return out


def test_fwht_fixed_values(orc):  # test_fwht.cpp:32-64
    np.testing.assert_array_equal(orc.fwht_unnormalized([1, 0, 0, 0]), [1, 1, 1, 1])
    np.testing.assert_array_equal(orc.fwht_unnormalized([1, 2, 3, 4]), [10, -2, -4, 0])
    np.testing.assert_array_equal(orc.fwht_unnormalized([3, 5]), [8, -2])
    np.testing.assert_allclose(orc.fwht_normalized([1, 0, 0, 0]), [0.5] * 4)
    np.testing.assert_allclose(orc.fwht_normalized([1, 2, 3, 4]), [5, -1, -2, 0])
    with pytest.raises(ValueError):
        orc.fwht_unnormalized([0.0, 0.0, 0.0])


def test_fwht_vs_naive(orc):  # test_fwht.cpp:72-85
    rng = np.random.default_rng(123)
    for k in range(7):
        for _ in range(10):
            v = rng.standard_normal(1 << k)
            assert np.max(np.abs(orc.fwht_unnormalized(v) - _naive_walsh(v))) <= 1e-10


def test_fwht_involution_norm(orc):  # test_fwht.cpp:87-102
    rng = np.random.default_rng(321)
    for k in (1, 4, 9, 13, 16):
        v = rng.standard_normal(1 << k)
        n = np.linalg.norm(v)
        w = orc.fwht_normalized(v)
        assert abs(np.linalg.norm(w) - n) <= 1e-12 * n
        assert np.linalg.norm(orc.fwht_normalized(w) - v) <= 1e-12 * n


# --------------------------------------------------------- test_kerdock.cpp --
def _matrix_get(rows, i, j):
    return (int(rows[i]) >> j) & 1


def test_kerdock_k2(orc):  # test_kerdock.cpp:34-45
    assert orc.design_params(2) == (4, 12)
    assert orc.kerdock_matrix(2, 0).tolist() == [0, 0]
    assert orc.kerdock_matrix(2, 1).tolist() == [0b10, 0b01]


def test_design_params_rejects(orc):  # test_kerdock.cpp:47-51
    for k in (3, 0, 18):
        with pytest.raises(ValueError):
            orc.design_params(k)


def test_kerdock_skew_and_pairwise_full_rank(orc):  # test_kerdock.cpp:53-68
    for k in (2, 4, 6, 8):
        d, _ = orc.design_params(k)
        mats = [orc.kerdock_matrix(k, s) for s in range(d // 2)]
        for m in mats:
            for i in range(k):
                assert _matrix_get(m, i, i) == 0
                for j in range(k):
                    assert _matrix_get(m, i, j) == _matrix_get(m, j, i)
        for a in range(len(mats)):
            for b in range(a + 1, len(mats)):
                assert orc.gf2_rank(mats[a] ^ mats[b]) == k


def test_kerdock_k4_nonzero_full_rank(orc):  # test_kerdock.cpp:70-76
    for s in range(1, 8):
        assert orc.gf2_rank(orc.kerdock_matrix(4, s)) == 4


def test_quadratic_form_fixed(orc):  # test_kerdock.cpp:93-107
    swap2 = [0b10, 0b01]
    assert orc.quadratic_form(swap2, 0) == 0
    assert orc.quadratic_form(swap2, 0b11) == 1
    m = orc.kerdock_matrix(4, 5)
    for i in range(4):
        assert orc.quadratic_form(m, 1 << i) == 0
    assert orc.quadratic_form(m, 0) == 0


def test_polarization(orc):  # test_kerdock.cpp:109-123
    rng = np.random.default_rng(97)
    for k in (2, 4, 6, 8):
        d, _ = orc.design_params(k)
        for _ in range(100):
            m = orc.kerdock_matrix(k, int(rng.integers(0, d // 2)))
            x, y = (int(v) for v in rng.integers(0, 1 << k, size=2))
            bil = 0
            for i in range(k):
                if (x >> i) & 1:
                    bil ^= bin(int(m[i]) & y).count("1") & 1
            assert orc.quadratic_form(m, x ^ y) ^ orc.quadratic_form(m, x) ^ orc.quadratic_form(m, y) == bil


def test_linearization_bijection(orc):  # test_kerdock.cpp:125-133
    d, L = orc.design_params(4)
    seen = set()
    for ell in range(L):
        ident, s, w = orc.decode_index(4, ell)
        back = (d // 2) * d + w if ident else s * d + w
        assert back == ell
        seen.add((ident, s, w))
    assert len(seen) == L
    for bad in (L, -1):
        with pytest.raises(IndexError):
            orc.decode_index(4, bad)


def test_design_vector_fixed(orc):  # test_kerdock.cpp:135-162 / 164-198
    np.testing.assert_allclose(orc.projected_design_column(2, 4, 0), [1, 1, 1, 1])
    np.testing.assert_allclose(orc.projected_design_column(2, 4, 4), [1, 1, 1, -1])  # s=1, w=0
    assert not orc.projected_design_column(2, 2, 8 + 3).any()
    np.testing.assert_allclose(orc.projected_design_column(2, 2, 8 + 1), [0, 2])
    for bad_n in (0, 5):
        with pytest.raises(ValueError):
            orc.projected_design_column(2, bad_n, 8)


def test_resolution_of_identity(orc):  # test_kerdock.cpp:259-270
    d, L = orc.design_params(4)
    for n in (16, 13, 5):
        acc = np.zeros((n, n))
        for ell in range(L):
            s = orc.projected_design_column(4, n, ell)
            acc += np.outer(s, s)
        assert np.max(np.abs(acc / L - np.eye(n))) <= 1e-9
