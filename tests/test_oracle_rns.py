"""Known-answer tests pinning the C RNS-CKKS oracle (oracle/ckks_oracle.c).

Residue-level: NTT == schoolbook negacyclic product; NTT index j evaluates
at psi^(2 brv(j) + 1); mul_i is X^(N/2); automorphisms match coefficient
maps.  Slot-level: every op decrypts to the emulator's slot semantics
(emulator.py:195-273) within CKKS noise; restated schedules over the oracle
reproduce the reference's golden ledgers exactly and its values within the
stated tolerance.
"""

import numpy as np
import pytest

from oracle import rns as R
from oracle import slots as S
from paper_2403_14111_b200 import workloads as wl

OPS = S.OP_KINDS
TOL = 1e-6        # per-op decrypt tolerance (CKKS noise at Delta = 2^40..2^42)


@pytest.fixture(scope="module")
def tiny():
    return R.RnsParams("tiny", seed=7)


@pytest.fixture(scope="module")
def small():
    return R.RnsParams("small12", seed=11)


def brv(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2)


def negacyclic(a, b, q):
    n = len(a)
    out = [0] * n
    for i in range(n):
        if a[i] == 0:
            continue
        for j in range(n):
            k = i + j
            if k < n:
                out[k] = (out[k] + a[i] * b[j]) % q
            else:
                out[k - n] = (out[k - n] - a[i] * b[j]) % q
    return out


def test_primes_and_scales(tiny, small):
    for p in (tiny, small):
        q = [int(x) for x in p.moduli]
        assert len(set(q)) == len(q)
        assert all((x - 1) % (2 * p.N) == 0 for x in q)
        for x, psi in zip(q, p.psis):
            assert pow(int(psi), p.N, x) == x - 1
    assert [int(x).bit_length() for x in small.moduli] == [58] + [42] * 12 + [60] * 3
    assert small.scales[-1] == 2.0 ** 42


def test_ntt_matches_schoolbook(tiny):
    rng = np.random.default_rng(0)
    q = int(tiny.moduli[1])
    a = rng.integers(0, q, tiny.N, dtype=np.uint64)
    b = rng.integers(0, 5, tiny.N, dtype=np.uint64)
    fa, fb = tiny.ntt(1, a), tiny.ntt(1, b)
    prod = np.array([(int(x) * int(y)) % q for x, y in zip(fa, fb)], dtype=np.uint64)
    got = tiny.ntt(1, prod, inverse=True)
    want = negacyclic([int(x) for x in a], [int(x) for x in b], q)
    assert [int(x) for x in got] == want
    # evaluation-point convention of the spec
    psi = int(tiny.psis[1])
    for j in (0, 1, 5, tiny.N - 1):
        e = 2 * brv(j, tiny.logN) + 1
        val = sum(int(a[i]) * pow(psi, e * i, q) for i in range(tiny.N)) % q
        assert int(fa[j]) == val
    np.testing.assert_array_equal(tiny.ntt(1, fa, inverse=True), a)


def test_encode_decode_roundtrip(tiny):
    rng = np.random.default_rng(1)
    z = rng.uniform(-1, 1, tiny.slots) + 1j * rng.uniform(-1, 1, tiny.slots)
    ct = tiny.encrypt(z, tiny.L, nonce=3)
    got = tiny.decrypt(ct, tiny.L)
    assert np.max(np.abs(got - z)) < TOL
    # deterministic: same nonce, same residues
    np.testing.assert_array_equal(ct, tiny.encrypt(z, tiny.L, nonce=3))
    assert not np.array_equal(ct, tiny.encrypt(z, tiny.L, nonce=4))


def test_secret_is_ternary_hw(tiny):
    s = tiny.secret()
    assert set(np.unique(s)) <= {-1, 0, 1}
    assert int(np.count_nonzero(s)) == 32


def test_per_op_slot_semantics(small):
    rng = np.random.default_rng(2)
    n, L = small.slots, small.L
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    y = rng.uniform(-1, 1, n)
    cx, cy = small.encrypt(x, L, 0), small.encrypt(y, L, 1)
    dec = small.decrypt
    assert np.max(np.abs(dec(small.add(cx, cy, L), L) - (x + y))) < TOL
    assert np.max(np.abs(dec(small.add(cx, cy, L, negate=True), L) - (x - y))) < TOL
    assert np.max(np.abs(dec(small.mult(cx, cy, L), L - 1) - x * y)) < TOL
    assert np.max(np.abs(dec(small.mul_const(cx, L, 0.3 - 0.2j), L - 1) - x * (0.3 - 0.2j))) < TOL
    assert np.max(np.abs(dec(small.add_const(cx, L, 1.5 + 2j), L) - (x + 1.5 + 2j))) < TOL
    assert np.max(np.abs(dec(small.mul_i(cx, L), L) - 1j * x)) < TOL
    pt = small.encode_ntt(y, L)
    assert np.max(np.abs(dec(small.mul_pt(cx, pt, L), L - 1) - x * y)) < TOL
    for r in (1, 5, n - 3):
        got = dec(small.automorph(cx, L, small.galois(r)), L)
        assert np.max(np.abs(got - np.roll(x, -r))) < TOL
    got = dec(small.automorph(cx, L, 2 * small.N - 1), L)
    assert np.max(np.abs(got - np.conj(x))) < TOL
    lo = small.level_adjust(cx, L, 3)
    assert np.max(np.abs(dec(lo, 3) - x)) < TOL
    fresh = small.refresh(lo, 3, 99)
    assert np.max(np.abs(dec(fresh, L) - x)) < TOL
    c0 = small.level_adjust(cx, L, 0)
    assert np.max(np.abs(dec(small.refresh(c0, 0, 100), L) - x)) < TOL


def test_mul_i_is_monomial(tiny):
    # X^(N/2) encodes i in every slot: its NTT is (+I, ..., -I, ...)
    N = tiny.N
    q = int(tiny.moduli[0])
    m = np.zeros(N, np.uint64)
    m[N // 2] = 1
    f = tiny.ntt(0, m)
    I = pow(int(tiny.psis[0]), N // 2, q)
    assert all(int(v) == I for v in f[: N // 2])
    assert all(int(v) == q - I for v in f[N // 2:])


def test_restated_diag_abt_config0_over_oracle(golden):
    A, B = wl.config0()
    ctx = R.OracleCKKSContext("cfg0", 64, seed=5)
    r = S.diag_abt(S.encode(ctx, A), S.encode(ctx, B, "vertical"))
    led = np.array([ctx.ledger.counts()[k] for k in OPS])
    np.testing.assert_array_equal(led, golden["cfg0_led"])
    assert r.level == 1
    out = S.decode(r, tol=1e-4)
    assert np.max(np.abs(out - golden["cfg0_out"])) < 1e-4
    # key-switch pipelines run: 8 relinearisations (one per product sum), 8
    # hoisted rotations, 16 ladders of 6 doubling steps as 2 radix-8
    # rotate-and-sum stages each (96 of the ledger's 104 Rot), 1 conj
    assert ctx.extra["KeySwitch"] == 8 + 8 + 32 + 1


def test_restated_softmax_small12(golden):
    ctx = R.OracleCKKSContext("small12", 16, auto_bootstrap=True, seed=6)
    r = S.a_softmax(S.encode(ctx, golden["small_sm_in"], "horizontal"))
    led = np.array([ctx.ledger.counts()[k] for k in OPS])
    np.testing.assert_array_equal(led, golden["small_sm_led"])
    assert r.level == golden["small_sm_level"]
    out = S.decode(r, tol=1e-3)
    assert np.max(np.abs(out - golden["small_sm_out"])) < 1e-3


def test_restated_diag_atb_small12(golden):
    for branch, alev in (("rl", None), ("pru", 11)):
        ctx = R.OracleCKKSContext("small12", 16, seed=8)
        r = S.diag_atb(S.encode(ctx, golden["small_atb_A"], "horizontal", level=alev),
                       S.encode(ctx, golden["small_atb_B"]), scale=2.0)
        led = np.array([ctx.ledger.counts()[k] for k in OPS])
        np.testing.assert_array_equal(led, golden[f"small_atb_{branch}_led"])
        out = S.decode(r, tol=1e-4)
        assert np.max(np.abs(out - golden[f"small_atb_{branch}_out"])) < 1e-4


def test_restated_training_small12(golden):
    x, y = golden["small_train_x"], golden["small_train_y"]
    ctx = R.OracleCKKSContext("small12", 16, auto_bootstrap=True, seed=9)
    W = S.encode(ctx, S.init_weights(3, x.shape[1], 7), "vertical")
    st = S.State(W, W)
    Y = S.one_hot(y, 3)
    snaps = []
    for step in range(3):
        sl = slice((step % 2) * 16, (step % 2) * 16 + 16)
        S.nag_step(st, S.encode(ctx, x[sl]), S.encode(ctx, Y[sl], "horizontal"), 0.3, 16)
        snaps.append(S.decode(st.weights, tol=1e-3))
    led = np.array([ctx.ledger.counts()[k] for k in OPS])
    np.testing.assert_array_equal(led, golden["small_train_led"])
    assert np.max(np.abs(np.stack(snaps) - golden["small_train_snaps"])) < 1e-4


def test_hoisted_rotations_and_product_sums(small):
    """Fused forms: with the centred base conversion a digit's
    lift commutes with the automorphism (the centred range is symmetric), so a
    hoisted rotation equals the per-op rotation bit for bit; a product sum
    decrypts to the sum of products and equals orc_mult for a single pair."""
    rng = np.random.default_rng(3)
    n, L = small.slots, small.L
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    cx = small.encrypt(x, L, 0)
    rs = (1, 7, n - 2, n // 2)
    outs = small.rotate_hoisted(cx, L, [small.galois(r) for r in rs])
    for r, o in zip(rs, outs):
        assert np.max(np.abs(small.decrypt(o, L) - np.roll(x, -r))) < TOL
        np.testing.assert_array_equal(o, small.automorph(cx, L, small.galois(r)))
    ys = [rng.uniform(-1, 1, n) for _ in range(3)]
    xs = [rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n) for _ in range(3)]
    cxs = [small.encrypt(v, L, 10 + i) for i, v in enumerate(xs)]
    cys = [small.encrypt(v, L, 20 + i) for i, v in enumerate(ys)]
    s = small.mult_sum(cxs, cys, L)
    assert np.max(np.abs(small.decrypt(s, L - 1) - sum(a * b for a, b in zip(xs, ys)))) < TOL
    np.testing.assert_array_equal(small.mult_sum(cxs[:1], cys[:1], L), small.mult(cxs[0], cys[0], L))


def test_rotate_and_sum_stage(small):
    """Radix ladders: x + sum_r lrot(x, r) with one ModUp, the
    key products summed in the extended basis and one ModDown decrypts to the
    value of the doubling steps it replaces; with a single rotation it is the
    ordinary rotate-and-add up to the ModDown rounding of one pipeline, and
    the restated ladder keeps the reference ledger."""
    rng = np.random.default_rng(9)
    n, L = small.slots, small.L
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    cx = small.encrypt(x, L, 0)
    for rs in ((1, 2, 3), (n - 4, n - 8, n - 12), (5,), (16, 32, 48, 64, 80, 96, 112)):
        o = small.rotsum(cx, L, [small.galois(r) for r in rs])
        want = x + sum(np.roll(x, -r) for r in rs)
        assert np.max(np.abs(small.decrypt(o, L) - want)) < TOL
    one = small.rotsum(cx, L, [small.galois(5)])
    np.testing.assert_array_equal(one, small.add(cx, small.automorph(cx, L, small.galois(5)), L))
    for hoist in (True, False):
        ctx = R.OracleCKKSContext("small12", 16, seed=5, hoist=hoist)
        v = rng.uniform(-1, 1, ctx.slot_count)
        b = ctx.encrypt(v)
        got = S.ladder(ctx, b, 16, 4)            # row ladder: stride s1 = 16, 4 steps: two radix-4 stages
        got = S.ladder(ctx, got, -1, 3)          # 3 steps: one radix-8 stage
        want = v
        for t in range(4):
            want = want + np.roll(want, -16 * (1 << t))
        for t in range(3):
            want = want + np.roll(want, 1 << t)
        assert np.max(np.abs(got.slots - want)) < 1e-4
        assert ctx.ledger.counts()["Rot"] == 7 and ctx.ledger.counts()["Add"] == 7
        assert ctx.extra["KeySwitch"] == (3 if hoist else 7)
    assert [S.ladder_plan(n) for n in range(1, 9)] == [[1], [2], [3], [2, 2], [3, 2], [3, 3], [3, 2, 2], [3, 3, 2]]


@pytest.mark.parametrize("hoist", [True, False])
def test_fused_schedules_keep_the_reference_ledger(golden, hoist):
    """DiagABT with several block columns (product sums fuse) and DiagATB in
    both branches: the fused forms keep the reference ledger and values."""
    rng = np.random.default_rng(4)
    A, B = rng.uniform(-1, 1, (10, 40)), rng.uniform(-1, 1, (4, 40))
    ctx = R.OracleCKKSContext("small12", 16, seed=5, hoist=hoist)
    r = S.diag_abt(S.encode(ctx, A), S.encode(ctx, B, "vertical"), scale=0.5)
    slot = S.SlotBackend(256, 16, max_level=12)
    S.diag_abt(S.encode(slot, A), S.encode(slot, B, "vertical"), scale=0.5)
    assert ctx.ledger.counts() == slot.ledger.counts()
    assert np.max(np.abs(S.decode(r, tol=1e-3) - 0.5 * A @ B.T)) < 1e-4
    for branch, alev in (("rl", None), ("pru", 11)):
        ctx = R.OracleCKKSContext("small12", 16, seed=8, hoist=hoist)
        r = S.diag_atb(S.encode(ctx, golden["small_atb_A"], "horizontal", level=alev),
                       S.encode(ctx, golden["small_atb_B"]), scale=2.0)
        led = np.array([ctx.ledger.counts()[k] for k in OPS])
        np.testing.assert_array_equal(led, golden[f"small_atb_{branch}_led"])
        assert np.max(np.abs(S.decode(r, tol=1e-4) - golden[f"small_atb_{branch}_out"])) < 1e-4


def test_oracle_ckks_bootstrapping_boot10():
    """The restated CKKS bootstrapping (oracle/boot.py) on the 2^10 ring:
    a level-0 ciphertext refreshed to the application level 12 without the
    secret key, message within 1e-4."""
    from oracle import boot as B
    p = R.RnsParams("boot10", seed=5)
    p.set_app_level(12)
    bt = B.Bootstrapper(p, 12)
    rng = np.random.default_rng(1)
    w = rng.uniform(-1, 1, p.slots) + 1j * rng.uniform(-1, 1, p.slots)
    out = bt.bootstrap(p.encrypt(w, 0, 7), 0)
    assert out.shape == (2, 13, p.N)
    assert np.max(np.abs(p.decrypt(out, 12) - w)) < 1e-4
