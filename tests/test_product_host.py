"""CPU tests of the product's host-side logic (no GPU): the encoding layer is
backend-agnostic, so it is driven here over the float64 slot backend of the
oracle and must reproduce the reference's values and per-op ledgers
(hefit/encoding.py; pkg/tests/test_encoding.py:158-231 for the ledger
contracts); count_formula must equal the reference's closed forms."""

import numpy as np
import pytest

from oracle import slots as S
from paper_2403_14111_b200 import encoding as E
from paper_2403_14111_b200 import matmul as M
from paper_2403_14111_b200 import workloads as wl


def ctx():
    return S.SlotBackend(256, 16, max_level=12)


def test_encode_decode_roundtrip_and_tiling():
    c = ctx()
    rng = np.random.default_rng(0)
    for shape, tiling in [((10, 21), "none"), ((3, 40), "vertical"), ((37, 5), "horizontal"), ((16, 16), "none")]:
        A = rng.uniform(-1, 1, shape)
        enc = E.encode(c, A, tiling)
        np.testing.assert_array_equal(E.decode(enc, tol=1e-9), A)
        ref = S.encode(c, A, tiling)
        assert enc.grid == ref.grid and enc.period == ref.period
        for rb, gb in zip([b for r in ref.blocks for b in r], enc.flat()):
            np.testing.assert_array_equal(rb.slots, gb.slots)
    with pytest.raises(Exception):
        E.encode(c, np.zeros((17, 3)), "vertical")


@pytest.mark.parametrize("k", [1, 3, 7, 9])
def test_structural_ops_match_reference_ledgers(k):
    c = ctx()
    rng = np.random.default_rng(k)
    A = rng.uniform(-1, 1, (30, 40))
    enc = E.encode(c, A)
    full = E.padded_array(enc).real
    m, n = enc.grid
    s0, s1 = c.grid_rows, c.grid_cols

    b0 = c.ledger.snapshot()
    out = E.rot_up(enc, k)
    assert c.ledger.delta(b0)["Rot"] == m * n
    got = E.padded_array(out).real
    for p in range(m):
        blk = full[p * s0:(p + 1) * s0]
        np.testing.assert_array_equal(got[p * s0:(p + 1) * s0], np.roll(blk, -k, axis=0))

    b0 = c.ledger.snapshot()
    out = E.rot_left(enc, k)
    d = c.ledger.delta(b0)
    assert (d["Rot"], d["CMult"]) == (2 * m * n, m * n)
    got = E.padded_array(out).real
    for q in range(n):
        np.testing.assert_allclose(got[:, q * s1:(q + 1) * s1], np.roll(full[:, q * s1:(q + 1) * s1], -k, axis=1))

    b0 = c.ledger.snapshot()
    E.prot_up(enc, k)
    d = c.ledger.delta(b0)
    assert (d["Rot"], d["CMult"]) == (m * n, m * n)

    b0 = c.ledger.snapshot()
    cs = E.col_sums(enc)
    d = c.ledger.delta(b0)
    assert (d["Rot"], d["CMult"]) == (2 * m * int(np.log2(s1)), m)
    rowsum = full.sum(axis=1)                      # over all block columns
    got = E.padded_array(cs).real
    for j in (0, 5, s1 - 1):                       # broadcast to every column of the row
        np.testing.assert_allclose(got[:, j], rowsum, atol=1e-12)

    b0 = c.ledger.snapshot()
    E.row_sums(enc)
    d = c.ledger.delta(b0)
    assert (d["Rot"], d["CMult"]) == (n * int(np.log2(s0)), 0)


def test_masks_match_reference():
    c = ctx()
    for shift, mod, cplx, scale in [(0, 4, False, 1.0), (3, 8, True, 0.25), (-2, 16, True, 2.0)]:
        a = E.make_mask(c, shift, mod, complexified=cplx, scale=scale).blocks[0][0].slots
        b = S.make_mask(c, shift, mod, complexified=cplx, scale=scale).blocks[0][0].slots
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(E.col_range_mask(c, 5).blocks[0][0].slots,
                                  c.pack(S.keep_head_pattern(16, 16, 5).ravel()).slots)


def test_count_formula_equals_reference_closed_forms():
    rng = np.random.default_rng(3)
    for _ in range(50):
        a, b, cc = int(rng.integers(1, 3000)), int(rng.integers(1, 3000)), int(2 ** rng.integers(0, 5))
        s0 = int(2 ** rng.integers(3, 9))
        s1 = 32768 // s0
        for alg in ("diag_abt", "diag_atb_rl", "diag_atb_pru"):
            assert M.count_formula(alg, (a, b, cc), s0, s1) == S.count_formula(alg, (a, b, cc), s0, s1)
    # BASELINE configs (SURVEY.md §6 ledgers)
    assert M.count_formula("diag_abt", (128, 768, 16), 128, 256) == {"CMult": 16, "Mult": 24, "Rot": 152}
    assert M.count_formula("diag_atb_rl", (128, 768, 16), 128, 256) == {"CMult": 32, "Mult": 24, "Rot": 184}
    assert M.count_formula("diag_atb_pru", (128, 768, 16), 128, 256) == {"CMult": 46, "Mult": 24, "Rot": 198}


def test_workloads_are_deterministic_and_shaped():
    A, B = wl.config0()
    assert A.shape == (64, 64) and B.shape == (16, 64)
    X, W = wl.config1()
    assert X.shape == (128, 768) and W.shape == (10, 768)
    np.testing.assert_allclose(np.linalg.norm(X, axis=1), 1.0)
    PY, X2 = wl.config2()
    np.testing.assert_allclose(PY.sum(axis=1), 0.0, atol=1e-12)       # softmax rows minus one-hot
    Z = wl.config3()
    assert Z.shape == (128, 10) and np.abs(Z).max() <= 128
    X4, y4 = wl.config4()
    assert X4.shape == (1024, 768) and set(np.unique(y4)) <= set(range(10))
    np.testing.assert_array_equal(wl.config4()[0], X4)
