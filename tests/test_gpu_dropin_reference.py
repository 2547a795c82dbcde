"""The drop-in claim on the real reference: the UNMODIFIED hefit code
(baseline/_ref, the offline install of /root/reference/pkg) runs its own
hot-path functions -- ``matmul.diag_abt`` / ``diag_atb`` (matmul.py:74,113),
``approx.a_softmax`` and its building blocks (approx.py:205-344),
``training.nag_step`` (training.py:66) -- with ``CKKSContext`` passed where
it expects an ``EmulatorContext``.  Every op then runs as a B200 kernel
sequence through the C-ABI.  The result must equal the product's native
schedule bit for bit on the residues (per-op order: ``hoist=False``), and the
ledger must equal the reference's golden counts.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OPS = ("Add", "CMult", "Mult", "Rot", "Conj", "Bootstrap")


def _prod():
    import paper_2403_14111_b200 as P
    return P


def _led(ctx):
    c = ctx.ledger.counts()
    return [c[k] for k in OPS]


def _as_product(P, H):
    """The same ciphertext blocks behind the product's EncodedMatrix."""
    return P.EncodedMatrix(H.ctx, tuple(tuple(r) for r in H.blocks), tuple(H.shape), H.tiling, H.period)


def _same(a, b):
    assert a.grid == tuple(b.grid)
    for ra, rb in zip(a.blocks, b.blocks):
        for x, y in zip(ra, rb):
            assert x.level == y.level
            np.testing.assert_array_equal(x.residues(), y.residues())


def test_reference_diag_abt(hefit, golden):
    P = _prod()
    g = P.CKKSContext("small12", 16, seed=9, hoist=False)
    g.nonce = 0
    HA, HB = hefit.encode(g, golden["small_abt_A"]), hefit.encode(g, golden["small_abt_B"], "vertical")
    g.ledger.reset()
    ref = hefit.matmul.diag_abt(HA, HB, scale=0.25)
    assert _led(g) == list(golden["small_abt_led"])
    g.ledger.reset()
    nat = P.diag_abt(_as_product(P, HA), _as_product(P, HB), scale=0.25)
    assert _led(g) == list(golden["small_abt_led"])
    _same(nat, ref)
    assert np.max(np.abs(P.decode(_as_product(P, ref)) - golden["small_abt_out"])) < 1e-4


@pytest.mark.parametrize("branch,alev", [("rl", None), ("pru", 11)])
def test_reference_diag_atb(hefit, golden, branch, alev):
    P = _prod()
    g = P.CKKSContext("small12", 16, seed=6, hoist=False)
    g.nonce = 0
    HA = hefit.encode(g, golden["small_atb_A"], "horizontal", level=alev)
    HB = hefit.encode(g, golden["small_atb_B"])
    g.ledger.reset()
    ref = hefit.matmul.diag_atb(HA, HB, scale=2.0)
    assert _led(g) == list(golden[f"small_atb_{branch}_led"])
    nat = P.diag_atb(_as_product(P, HA), _as_product(P, HB), scale=2.0)
    _same(nat, ref)
    assert np.max(np.abs(P.decode(_as_product(P, ref)) - golden[f"small_atb_{branch}_out"])) < 1e-4


def test_reference_softmax(hefit, golden):
    P = _prod()
    g = P.CKKSContext("small12", 16, seed=8, auto_bootstrap=True, hoist=False)
    g.nonce = 0
    HM = hefit.encode(g, golden["small_sm_in"], "horizontal")
    g.nonce = 1000
    g.ledger.reset()
    ref = hefit.approx.a_softmax(HM)
    assert _led(g) == list(golden["small_sm_led"])
    n_ref = g.nonce
    g.nonce = 1000
    nat = P.a_softmax(_as_product(P, HM))
    assert g.nonce == n_ref
    _same(nat, ref)


def test_reference_softmax_building_blocks(hefit):
    """a_comp, a_max, domain_extend, _dep_compensation, a_exp, a_inv: the
    reference's functions over the B200 context == the exported native ones."""
    P = _prod()
    g = P.CKKSContext("small12", 16, seed=18, auto_bootstrap=True, hoist=False)
    rng = np.random.default_rng(3)
    cases = [
        ("a_comp", lambda H: (H(rng.uniform(-0.5, 0.5, (32, 4))), H(rng.uniform(-0.5, 0.5, (32, 4))))),
        ("a_max", lambda H: (H(rng.uniform(-60, 60, (32, 3)), "horizontal"),)),
        ("domain_extend", lambda H: (H(rng.uniform(-100, 0, (32, 4)), "horizontal"),)),
        ("_dep_compensation", lambda H: (H(rng.uniform(-8, 0, (32, 4)), "horizontal"),)),
        ("a_exp", lambda H: (H(rng.uniform(-8, 0, (32, 4)), "horizontal"),)),
        ("a_inv", lambda H: (H(rng.uniform(1, 10, (32, 4)), "horizontal"),)),
    ]
    native = {"a_comp": P.a_comp, "a_max": P.a_max, "domain_extend": P.domain_extend,
              "_dep_compensation": P.dep_compensation, "a_exp": P.a_exp, "a_inv": P.a_inv}
    for name, make in cases:
        g.nonce = 0
        args = make(lambda a, t="none": hefit.encode(g, a, t))
        fref = getattr(hefit.approx, name)
        g.nonce = 500
        g.ledger.reset()
        ref = fref(*args) if name != "_dep_compensation" else fref(args[0], hefit.DEFAULTS)
        led_ref, n_ref = _led(g), g.nonce
        g.nonce = 500
        g.ledger.reset()
        nat = native[name](*[_as_product(P, a) for a in args])
        assert _led(g) == led_ref, name
        assert g.nonce == n_ref, name
        _same(nat, ref)


def test_reference_nag_steps(hefit, golden):
    """hefit.training.nag_step on the B200 context (two steps, auto-bootstrap)
    == the product's nag_step: W and V residues, ledger."""
    P = _prod()
    x, y = golden["small_train_x"], golden["small_train_y"]
    Y = P.one_hot(y, 3)
    w0 = P.init_weights(3, x.shape[1], 7)
    g = P.CKKSContext("small12", 16, seed=10, auto_bootstrap=True, hoist=False)
    g.nonce = 0
    HW = hefit.encode(g, w0, "vertical")
    hs = hefit.training.TrainState(weights=HW, momentum=HW)
    ps = P.TrainState(_as_product(P, HW), _as_product(P, HW))
    for step in range(2):
        sl = slice(16 * step, 16 * step + 16)
        g.nonce = 100 * (step + 1)
        HX, HY = hefit.encode(g, x[sl]), hefit.encode(g, Y[sl], "horizontal")
        g.nonce = 1000 * (step + 1)
        hefit.training.nag_step(hs, HX, HY, 0.3, 16)
        n_ref = g.nonce
        g.nonce = 1000 * (step + 1)
        P.nag_step(ps, _as_product(P, HX), _as_product(P, HY), 0.3, 16)
        assert g.nonce == n_ref
        _same(ps.weights, hs.weights)
        _same(ps.momentum, hs.momentum)


@pytest.mark.slow
def test_reference_diag_abt_config1(hefit, golden):
    """BASELINE config 1 at N = 2^16 through the unmodified reference."""
    P = _prod()
    from paper_2403_14111_b200 import workloads as wl
    X, W = wl.config1()
    g = P.CKKSContext("cfg1", 128, seed=1, hoist=False)
    g.nonce = 0
    HX, HW = hefit.encode(g, X), hefit.encode(g, W, "vertical")
    g.ledger.reset()
    ref = hefit.matmul.diag_abt(HX, HW)
    assert _led(g) == list(golden["cfg1_led"])
    nat = P.diag_abt(_as_product(P, HX), _as_product(P, HW))
    _same(nat, ref)
    assert np.max(np.abs(P.decode(_as_product(P, ref), tol=1e-3) - X @ W.T)) < 1e-3
