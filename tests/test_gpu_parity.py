"""GPU parity: the CUDA path (through the C-ABI) against the C RNS-CKKS oracle.

Bit-exact on ciphertext residues (integer work), given the same seed and
nonce sequence; decrypted values against float64 within the CKKS tolerance.
"""

import numpy as np
import pytest

from oracle import rns as R
from oracle import slots as S

pytestmark = pytest.mark.gpu

OPS = S.OP_KINDS


def _prod():
    import paper_2403_14111_b200 as P
    return P


@pytest.fixture(scope="module", params=["tiny", "small12", "cfg0"])
def pair(request):
    P = _prod()
    name = request.param
    grid = {"tiny": 16, "small12": 16, "cfg0": 64}[name]
    return P.CKKSContext(name, grid, seed=77), R.OracleCKKSContext(name, grid, seed=77)


def test_moduli_and_scales(pair):
    g, o = pair
    np.testing.assert_array_equal(g.moduli, o.p.moduli)
    np.testing.assert_array_equal(g.scales, o.p.scales)


def test_encoder_bit_exact(pair):
    g, o = pair
    rng = np.random.default_rng(3)
    z = rng.uniform(-3, 3, g.slot_count) + 1j * rng.uniform(-3, 3, g.slot_count)
    for sc in (2.0 ** 40, g.scales[0], 12345.678):
        np.testing.assert_array_equal(g.encode_coef(z, sc), o.p.encode(z, sc))
    np.testing.assert_array_equal(g.encode_pt(z, g.max_level), o.p.encode_ntt(z, g.max_level))


def test_keys_bit_exact(pair):
    g, o = pair
    for gid in (0, g.galois_rot(1), g.galois_rot(-3), 2 * g.N - 1):
        np.testing.assert_array_equal(g.key(gid), o.p.key(gid))


def test_encrypt_decrypt(pair):
    g, o = pair
    rng = np.random.default_rng(4)
    z = rng.uniform(-1, 1, g.slot_count)
    for lv in (g.max_level, 1, 0):
        g.nonce, o.nonce = 10, 10
        a, b = g.encrypt(z, lv), o.encrypt(z, lv)
        np.testing.assert_array_equal(a.residues(), b.data)
        assert np.max(np.abs(a.slots - z)) < 1e-6


def test_per_op_residues(pair):
    g, o = pair
    rng = np.random.default_rng(5)
    n = g.slot_count
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    y = rng.uniform(-1, 1, n)
    mask = (np.arange(n) % 3 == 0) * 0.5 - 0.25j
    g.nonce, o.nonce = 0, 0
    gx, gy = g.encrypt(x), g.encrypt(y)
    ox, oy = o.encrypt(x), o.encrypt(y)

    def same(a, b, want=None, tol=1e-5):
        np.testing.assert_array_equal(a.residues(), b.data)
        assert a.level == b.level
        if want is not None:
            assert np.max(np.abs(a.slots - want)) < tol

    same(g.add(gx, gy), o.add(ox, oy), x + y)
    same(g.sub(gx, gy), o.sub(ox, oy), x - y)
    same(g.sub(0.75, gx), o.sub(0.75, ox), 0.75 - x)
    same(g.add(gx, 2.0 - 1j), o.add(ox, 2.0 - 1j), x + 2 - 1j)
    same(g.mult(gx, 0.3), o.mult(ox, 0.3), 0.3 * x)
    same(g.mult(gx, mask), o.mult(ox, mask), x * mask)
    same(g.add(gx, mask), o.add(ox, mask), x + mask)
    same(g.sub(mask, gx), o.sub(mask, ox), mask - x)
    gxy, oxy = g.mult(gx, gy), o.mult(ox, oy)
    same(gxy, oxy, x * y)
    same(g.add(gxy, gx), o.add(oxy, ox), x * y + x)          # level adjust 12 -> 11
    same(g.mult(gxy, gy), o.mult(oxy, oy), x * y * y)        # adjust + mult
    for r in (1, 7, n - 1, n // 2):
        same(g.lrot(gx, r), o.lrot(ox, r), np.roll(x, -r))
    same(g.conj(gx), o.conj(ox), np.conj(x))
    same(g.mul_i(gx), o.mul_i(ox), 1j * x)
    g.nonce, o.nonce = 500, 500
    same(g.bootstrap(gxy), o.bootstrap(oxy), x * y)
    lo_g, lo_o = g.level_adjust(gx, 0), o.p.level_adjust(ox.data, ox.level, 0)
    np.testing.assert_array_equal(lo_g.residues(), lo_o)
    g.auto_bootstrap = o.auto_bootstrap = True
    g.nonce, o.nonce = 900, 900
    same(g.mult(lo_g, lo_g), o.mult(R.RnsBlock(o, lo_o, 0), R.RnsBlock(o, lo_o, 0)), x * x)
    g.auto_bootstrap = o.auto_bootstrap = False
    rs = g.rescale(gx)
    np.testing.assert_array_equal(rs.residues(), o.p.rescale(ox.data, ox.level))


def _fused_ops(g, o, seed, tol=1e-5):
    """hoisted rotations and product sums: residues, levels, ledgers"""
    rng = np.random.default_rng(seed)
    n = g.slot_count
    xs = [rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n) for _ in range(3)]
    ys = [rng.uniform(-1, 1, n) for _ in range(3)]
    g.nonce, o.nonce = 0, 0
    gx, gy = [g.encrypt(v) for v in xs], [g.encrypt(v) for v in ys]
    ox, oy = [o.encrypt(v) for v in xs], [o.encrypt(v) for v in ys]
    g.ledger.reset()
    o.ledger.reset()
    rs = (1, 5, 0, n - 3, n // 2)
    for r, a, b in zip(rs, g.lrot_hoisted(gx[0], rs), o.lrot_hoisted(ox[0], rs)):
        np.testing.assert_array_equal(a.residues(), b.data)
        assert np.max(np.abs(a.slots - np.roll(xs[0], -r))) < tol
        if r == 0:
            assert a is gx[0]
    gs, os_ = g.mult_sum(gx, gy), o.mult_sum(ox, oy)
    np.testing.assert_array_equal(gs.residues(), os_.data)
    assert gs.level == os_.level == g.max_level - 1
    assert np.max(np.abs(gs.slots - sum(a * b for a, b in zip(xs, ys)))) < tol
    assert _ledger(g) == _ledger(o) == [2, 0, 3, 4, 0, 0]
    # centred base conversion: a hoisted rotation is the per-op key switch bit for bit
    for r, a in zip(rs, g.lrot_hoisted(gx[0], rs)):
        if r:
            np.testing.assert_array_equal(a.residues(), g.lrot(gx[0], r).residues())
    # doubling ladders as radix-4 / radix-8 rotate-and-sum stages (one ModUp /
    # ModDown per two or three steps): residues vs the oracle's stages, the
    # reference's ledger
    g.ledger.reset()
    o.ledger.reset()
    ks0 = g.extra["KeySwitch"], o.extra["KeySwitch"]
    for stride, steps, lv in ((1, 4, None), (-1, 3, None), (g.grid_cols, 2, 2), (-2, 1, 1), (1, 5, None)):
        z = rng.uniform(-1, 1, n) * 2.0 ** -steps
        g.nonce, o.nonce = 50, 50
        a = g.encrypt(z) if lv is None else g.encrypt(z, lv)
        b = o.encrypt(z) if lv is None else o.encrypt(z, lv)
        la, lb = S.ladder(g, a, stride, steps), S.ladder(o, b, stride, steps)
        np.testing.assert_array_equal(la.residues(), lb.data)
        want = z
        for t in range(steps):
            want = want + np.roll(want, -stride * (1 << t))
        assert np.max(np.abs(la.slots - want)) < tol
    assert _ledger(g) == _ledger(o) == [15, 0, 0, 15, 0, 0]
    assert g.extra["KeySwitch"] - ks0[0] == o.extra["KeySwitch"] - ks0[1] == 2 + 1 + 1 + 1 + 2


def test_fused_ops_residues(pair):
    _fused_ops(*pair, seed=6)


@pytest.mark.slow
def test_fused_ops_residues_cfg1():
    """the same through the fused N = 2^16 pipeline (keyswitch_hoisted, batched relinearisation)"""
    P = _prod()
    # key-switch noise at cfg1: the first digit's modulus (58 + 3 x 42 bits)
    # exceeds P (3 x 60 bits), so one switch leaves ~1e-4 in the worst slot
    _fused_ops(P.CKKSContext("cfg1", 128, seed=3), R.OracleCKKSContext("cfg1", 128, seed=3), seed=7, tol=1e-3)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["n14", "n15", "n17"])
def test_fused_pipeline_other_rings(name):
    """The fused key-switch / rescale pipeline's column-pass geometries for
    N = 2^14, 2^15 and 2^17 (keyswitch.cu ColCfg; cfg1 covers 2^16): rotation,
    conjugation, ct x ct (relinearisation + rescale in one pass), ct x pt
    (fused rescale), hoisted rotations and a radix-8 + radix-4 ladder,
    residues against the oracle with alpha = 2, 3, 1 digits."""
    P = _prod()
    g = P.CKKSContext(name, 128, seed=21)
    o = R.OracleCKKSContext(name, 128, seed=21)
    rng = np.random.default_rng(12)
    n = g.slot_count
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    y = rng.uniform(-1, 1, n)
    g.nonce, o.nonce = 0, 0
    gx, gy, ox, oy = g.encrypt(x), g.encrypt(y), o.encrypt(x), o.encrypt(y)
    np.testing.assert_array_equal(gx.residues(), ox.data)
    for r in (1, n - 5):
        a, b = g.lrot(gx, r), o.lrot(ox, r)
        np.testing.assert_array_equal(a.residues(), b.data)
        assert np.max(np.abs(a.slots - np.roll(x, -r))) < 1e-4
    np.testing.assert_array_equal(g.conj(gx).residues(), o.conj(ox).data)
    gm, om = g.mult(gx, gy), o.mult(ox, oy)
    np.testing.assert_array_equal(gm.residues(), om.data)
    assert gm.level == g.max_level - 1 and np.max(np.abs(gm.slots - x * y)) < 1e-4
    gp, op = g.cmult(gm, y), o.cmult(om, y)
    np.testing.assert_array_equal(gp.residues(), op.data)
    for a, b in zip(g.lrot_hoisted(gp, (3, 0, n - 1)), o.lrot_hoisted(op, (3, 0, n - 1))):
        np.testing.assert_array_equal(a.residues(), b.data if hasattr(b, "data") else b)
    z = rng.uniform(-1, 1, n) / 32
    gz, oz = g.encrypt(z, 2), o.encrypt(z, 2)
    la, lb = S.ladder(g, gz, -3, 5), S.ladder(o, oz, -3, 5)
    np.testing.assert_array_equal(la.residues(), lb.data)
    want = z
    for t in range(5):
        want = want + np.roll(want, 3 << t)
    assert np.max(np.abs(la.slots - want)) < 1e-4
    data = _adversarial(g.moduli, g.max_level + 1, g.N, "max", rng)
    gb, ob = g.from_residues(data, g.max_level), R.RnsBlock(o, data, g.max_level)
    np.testing.assert_array_equal(g.mult(gb, gb).residues(), o.mult(ob, ob).data)
    np.testing.assert_array_equal(S.ladder(g, gb, 1, 3).residues(), S.ladder(o, ob, 1, 3).data)


@pytest.mark.parametrize("hoist,cols", [(True, 40), (False, 40), (True, 200)])
def test_native_multi_column_diag_abt_small12(hoist, cols):
    """DiagABT with 3 (and 13: more than one 8-product group of the fused
    tensor sum) block columns (the product sums fuse when hoist is on):
    native schedule == restated schedule over the oracle in the same mode."""
    P = _prod()
    rng = np.random.default_rng(4)
    A, B = rng.uniform(-1, 1, (10, cols)) / np.sqrt(cols / 40), rng.uniform(-1, 1, (4, cols))
    g = P.CKKSContext("small12", 16, seed=5, hoist=hoist)
    o = R.OracleCKKSContext("small12", 16, seed=5, hoist=hoist)
    GA, OA = _enc_pair(g, o, A)
    g.nonce = o.nonce = 40
    GB, OB = P.encode(g, B, "vertical"), S.encode(o, B, "vertical")
    out = P.diag_abt(GA, GB, scale=0.5)
    ref = S.diag_abt(OA, OB, scale=0.5)
    _same_grid(out, ref)
    assert _ledger(g) == _ledger(o)
    assert np.max(np.abs(P.decode(out, tol=1e-3) - 0.5 * A @ B.T)) < 1e-4


def _enc_pair(g, o, arr, tiling="none", level=None):
    from paper_2403_14111_b200 import encode
    g.nonce = o.nonce = 0
    return encode(g, arr, tiling, level=level), S.encode(o, arr, tiling, level=level)


def _same_grid(G, O):
    assert G.grid == O.grid
    for rg, ro in zip(G.blocks, O.blocks):
        for bg, bo in zip(rg, ro):
            np.testing.assert_array_equal(bg.residues(), bo.data)


def _ledger(ctx):
    c = ctx.ledger.counts()
    return [c[k] for k in OPS]


def test_native_diag_abt_config0(golden):
    P = _prod()
    from paper_2403_14111_b200 import workloads as wl
    A, B = wl.config0()
    g, o = P.CKKSContext("cfg0", 64, seed=5), R.OracleCKKSContext("cfg0", 64, seed=5)
    GA, OA = _enc_pair(g, o, A)
    g.nonce = o.nonce = 100
    GB, OB = P.encode(g, B, "vertical"), S.encode(o, B, "vertical")
    out = P.diag_abt(GA, GB)
    ref = S.diag_abt(OA, OB)
    _same_grid(out, ref)
    assert _ledger(g) == list(golden["cfg0_led"]) == _ledger(o)
    assert out.level == 1
    assert np.max(np.abs(P.decode(out) - A @ B.T)) < 1e-4


@pytest.mark.parametrize("alev", [None, 11])
def test_native_diag_atb_small12(golden, alev):
    P = _prod()
    g, o = P.CKKSContext("small12", 16, seed=6), R.OracleCKKSContext("small12", 16, seed=6)
    GA, OA = _enc_pair(g, o, golden["small_atb_A"], "horizontal", level=alev)
    g.nonce = o.nonce = 50
    GB, OB = P.encode(g, golden["small_atb_B"]), S.encode(o, golden["small_atb_B"])
    out = P.diag_atb(GA, GB, scale=2.0)
    ref = S.diag_atb(OA, OB, scale=2.0)
    _same_grid(out, ref)
    branch = "rl" if alev is None else "pru"
    assert _ledger(g) == list(golden[f"small_atb_{branch}_led"])
    assert np.max(np.abs(P.decode(out) - golden[f"small_atb_{branch}_out"])) < 1e-4


def test_native_softmax_small12(golden):
    P = _prod()
    g = P.CKKSContext("small12", 16, seed=8, auto_bootstrap=True)
    o = R.OracleCKKSContext("small12", 16, seed=8, auto_bootstrap=True)
    GM, OM = _enc_pair(g, o, golden["small_sm_in"], "horizontal")
    out = P.a_softmax(GM)
    ref = S.a_softmax(OM)
    _same_grid(out, ref)
    assert g.nonce == o.nonce
    assert _ledger(g) == list(golden["small_sm_led"])
    assert np.max(np.abs(P.decode(out, tol=1e-3) - golden["small_sm_out"])) < 1e-3


def test_backend_interface_semantics():
    """EmulatorContext semantics the reference's callers rely on
    (emulator.py:160-273, errors.py): error codes, lrot-by-0 identity,
    plaintext pass-through, per-operand auto-bootstrap counting."""
    P = _prod()
    g = P.CKKSContext("small12", 16, seed=15)
    z = np.linspace(-1, 1, g.slot_count)
    x = g.encrypt(z)
    assert g.lrot(x, 0) is x and g.lrot(x, g.slot_count) is x
    pt = g.pack(z)
    assert g.bootstrap(pt) is pt and not pt.encrypted and pt.level == float("inf")
    with pytest.raises(TypeError):
        g.cmult(x, x)
    with pytest.raises(P.SlotCountMismatch):
        g.encrypt(np.zeros(3))
    with pytest.raises(ValueError):
        g.encrypt(z, level=g.max_level + 1)
    low = g.encrypt(z, level=0)
    with pytest.raises(P.DepthExhausted) as ei:
        g.mult(low, low)
    assert ei.value.code == "emulator.depth"
    g.auto_bootstrap = True
    before = g.ledger.snapshot()
    y = g.mult(low, low)                                  # both operands refreshed: 2 Bootstraps
    d = g.ledger.delta(before)
    assert d["Bootstrap"] == 2 and d["Mult"] == 1 and y.level == g.max_level - 1
    assert np.max(np.abs(y.slots - z * z)) < 1e-5
    before = g.ledger.snapshot()
    s = g.add(pt, pt)                                     # plaintext op: unledgered
    assert not s.encrypted and g.ledger.delta(before)["Add"] == 0
    a = g.add(x, 2.5)
    b = g.sub(2.5, x)
    assert np.max(np.abs(a.slots - (z + 2.5))) < 1e-6 and np.max(np.abs(b.slots - (2.5 - z))) < 1e-6
    assert g.ledger.delta(before)["Add"] == 2
    e = P.encode(g, np.ones((3, 5)))
    with pytest.raises(P.ResidualImaginary):
        P.decode(e.map_blocks(g.mul_i))
    assert g.decodes_by("observer") == [("observer", None)]      # audited before the check (encoding.py:216-218)
    P.decode(e, role="client", tag="t")
    assert g.decodes_by("client") == [("client", "t")]


def test_table4_baselines_small12(golden):
    """col_major_abt / row_major_atb (matmul.py:160-237) natively: residues vs
    the oracle, ledgers and values vs the reference's golden vectors."""
    P = _prod()
    g, o = P.CKKSContext("small12", 16, seed=14), R.OracleCKKSContext("small12", 16, seed=14)
    GA, OA = _enc_pair(g, o, golden["small_cm_A"])
    g.nonce = o.nonce = 40
    GB, OB = P.encode(g, golden["small_cm_B"]), S.encode(o, golden["small_cm_B"])
    out, ref = P.col_major_abt(GA, GB, scale=-1.0), S.col_major_abt(OA, OB, scale=-1.0)
    _same_grid(out, ref)
    assert _ledger(g) == list(golden["small_cm_led"])
    assert np.max(np.abs(P.decode(out) - golden["small_cm_out"])) < 1e-4
    g.ledger.reset()
    GA, OA = _enc_pair(g, o, golden["small_rm_A"])
    g.nonce = o.nonce = 80
    GB, OB = P.encode(g, golden["small_rm_B"]), S.encode(o, golden["small_rm_B"])
    out, ref = P.row_major_atb(GA, GB, scale=0.5), S.row_major_atb(OA, OB, scale=0.5)
    _same_grid(out, ref)
    assert _ledger(g) == list(golden["small_rm_led"])
    assert np.max(np.abs(P.decode(out) - golden["small_rm_out"])) < 1e-4


def test_block_parallel_softmax_matches_sequential_oracle():
    """4 block rows run as concurrent branches with the nonce plan: residues and
    the nonce counter equal the oracle's sequential (block-interleaved) run."""
    P = _prod()
    rng = np.random.default_rng(9)
    Z = rng.uniform(-60, 60, (64, 5))
    g = P.CKKSContext("small12", 16, seed=13, auto_bootstrap=True)
    o = R.OracleCKKSContext("small12", 16, seed=13, auto_bootstrap=True)
    GZ, OZ = _enc_pair(g, o, Z, "horizontal")
    out = P.a_softmax(GZ)
    ref = S.a_softmax(OZ)
    _same_grid(out, ref)
    assert g.nonce == o.nonce
    assert _ledger(g) == [o.ledger.counts()[k] for k in OPS]


def test_dropin_per_op_equals_native(golden):
    """The reference op sequence (restated in oracle/slots.py) issued op by op
    through the product's EmulatorContext interface == the native schedule."""
    P = _prod()
    g = P.CKKSContext("small12", 16, seed=9)
    A, B = golden["small_abt_A"], golden["small_abt_B"]
    g.nonce = 0
    GA, GB = P.encode(g, A), P.encode(g, B, "vertical")
    native = P.diag_abt(GA, GB, scale=0.25)
    led_native = _ledger(g)
    g.ledger.reset()
    per_op = S.diag_abt(S.Grid(g, GA.blocks, GA.shape, GA.tiling, GA.period),
                        S.Grid(g, GB.blocks, GB.shape, GB.tiling, GB.period), scale=0.25)
    assert _ledger(g) == led_native == list(golden["small_abt_led"])
    for bn, bp in zip(native.flat(), [b for r in per_op.blocks for b in r]):
        np.testing.assert_array_equal(bn.residues(), bp.residues())


def test_nag_steps_small12(golden):
    P = _prod()
    x, y = golden["small_train_x"], golden["small_train_y"]
    g = P.CKKSContext("small12", 16, seed=10, auto_bootstrap=True)
    o = R.OracleCKKSContext("small12", 16, seed=10, auto_bootstrap=True)
    w0 = S.init_weights(3, x.shape[1], 7)
    Y = S.one_hot(y, 3)
    GW, OW = _enc_pair(g, o, w0, "vertical")
    gs, os_ = P.TrainState(GW, GW), S.State(OW, OW)
    for step in range(3):
        sl = slice((step % 2) * 16, (step % 2) * 16 + 16)
        g.nonce = o.nonce = 1000 * (step + 1)
        GX, GY = P.encode(g, x[sl]), P.encode(g, Y[sl], "horizontal")
        OX, OY = S.encode(o, x[sl]), S.encode(o, Y[sl], "horizontal")
        P.nag_step(gs, GX, GY, 0.3, 16)
        S.nag_step(os_, OX, OY, 0.3, 16)
        _same_grid(gs.weights, os_.weights)
        _same_grid(gs.momentum, os_.momentum)
    assert _ledger(g) == list(golden["small_train_led"])
    w = P.decode(gs.weights, tol=1e-3)
    assert np.max(np.abs(w - golden["small_train_snaps"][-1])) < 1e-4


def test_nccl_reducer_plumbing(golden):
    """diag_atb with the multi-GPU reducer on a 1-rank NCCL group: the device
    residue view, the all-reduce and hc_mod_reduce leave the result unchanged."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2403_14111_b200 import sharding
    P = _prod()
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    g = P.CKKSContext("small12", 16, seed=12)
    rng = np.random.default_rng(1)
    A, B = rng.uniform(-1, 1, (64, 4)), rng.uniform(-1, 1, (64, 21))
    GA, GB = P.encode(g, A, "horizontal"), P.encode(g, B)
    plain = P.diag_atb(GA, GB, scale=0.5)
    red = P.diag_atb(GA, GB, scale=0.5, reducer=sharding.NcclModReducer())
    for a, b in zip(plain.flat(), red.flat()):
        np.testing.assert_array_equal(a.residues(), b.residues())
    assert np.max(np.abs(P.decode(red) - 0.5 * A.T @ B)) < 1e-3
    dist.destroy_process_group()


@pytest.mark.slow
def test_config1_diag_abt_full_size(golden):
    """BASELINE config 1 at N=2^16: residues vs the oracle, values vs float64."""
    P = _prod()
    from paper_2403_14111_b200 import workloads as wl
    X, W = wl.config1()
    g, o = P.CKKSContext("cfg1", 128, seed=1), R.OracleCKKSContext("cfg1", 128, seed=1)
    GX, OX = _enc_pair(g, o, X)
    g.nonce = o.nonce = 10
    GW, OW = P.encode(g, W, "vertical"), S.encode(o, W, "vertical")
    out = P.diag_abt(GX, GW)
    ref = S.diag_abt(OX, OW)
    _same_grid(out, ref)
    assert _ledger(g) == list(golden["cfg1_led"])
    assert out.level == 9
    # CKKS noise of the 2 x 8-step rotation ladders at Delta = 2^42, dnum = 4
    assert np.max(np.abs(P.decode(out, tol=1e-3) - X @ W.T)) < 1e-3


@pytest.mark.slow
@pytest.mark.parametrize("branch,alev", [("rl", None), ("pru", 11)])
def test_config2_diag_atb_full_size(golden, branch, alev):
    """BASELINE config 2: (P-Y)^T X at N=2^16, both alignment branches."""
    P = _prod()
    from paper_2403_14111_b200 import workloads as wl
    PY, X = wl.config2()
    g, o = P.CKKSContext("cfg1", 128, seed=2), R.OracleCKKSContext("cfg1", 128, seed=2)
    GA, OA = _enc_pair(g, o, PY, "horizontal", level=alev)
    g.nonce = o.nonce = 10
    GX, OX = P.encode(g, X), S.encode(o, X)
    out = P.diag_atb(GA, GX)
    ref = S.diag_atb(OA, OX)
    _same_grid(out, ref)
    assert _ledger(g) == list(golden[f"cfg2_{branch}_led"])
    assert out.level == golden[f"cfg2_{branch}_level"]
    assert np.max(np.abs(P.decode(out, tol=1e-3) - PY.T @ X)) < 1e-3


@pytest.mark.slow
def test_config3_softmax_full_size(golden):
    """BASELINE config 3: 128x10 logits in [-128, 128] at N=2^16; residues vs the
    oracle, max error vs float64 softmax within the paper's Table-5 bound."""
    P = _prod()
    from paper_2403_14111_b200 import workloads as wl
    Z = wl.config3()
    g = P.CKKSContext("cfg1", 128, seed=3, auto_bootstrap=True)
    o = R.OracleCKKSContext("cfg1", 128, seed=3, auto_bootstrap=True)
    GZ, OZ = _enc_pair(g, o, Z, "horizontal")
    out = P.a_softmax(GZ)
    ref = S.a_softmax(OZ)
    _same_grid(out, ref)
    assert _ledger(g) == list(golden["cfg3_led"])
    got = P.decode(out, tol=1e-3)
    # vs the reference emulator (noise-free): CKKS noise through the inverse's
    # ~1/y^2 conditioning; over key / encryption seeds 3..8 the worst of the
    # 1280 outputs measured 4.5e-4 .. 1.3e-3 at an rms of 4..7e-5
    # (scripts/softmax_noise.py), so 2e-3 bounds the tail, 2e-4 the rms
    diff = np.abs(got - golden["cfg3_out"])
    assert diff.max() < 2e-3 and np.sqrt((diff ** 2).mean()) < 2e-4
    assert np.max(np.abs(got - S.exact_softmax(Z))) < 0.0097         # PAPER.md:1071 (c=10)


@pytest.mark.slow
def test_config4_data_parallel_step_1024_rows():
    """The 1024-row batch as one NAG step (8 block rows; the multi-GPU
    data-parallel form run on one GPU): weights vs the float64 slot emulator
    running the reference op sequence on the same batch."""
    P = _prod()
    from paper_2403_14111_b200 import workloads as wl
    X, y = wl.config4()
    Y = S.one_hot(y, wl.CLASSES)
    w0 = S.init_weights(wl.CLASSES, X.shape[1], wl.INIT_SEED)
    g = P.CKKSContext("cfg1", 128, seed=4, auto_bootstrap=True)
    W = P.encode(g, w0, "vertical")
    st = P.TrainState(W, W)
    P.nag_step(st, P.encode(g, X), P.encode(g, Y, "horizontal"), wl.LEARNING_RATE, X.shape[0])
    e = S.SlotBackend(32768, 128, max_level=12, auto_bootstrap=True)
    EW = S.encode(e, w0, "vertical")
    es = S.State(EW, EW)
    S.nag_step(es, S.encode(e, X), S.encode(e, Y, "horizontal"), wl.LEARNING_RATE, X.shape[0])
    assert _ledger(g) == [e.ledger.counts()[k] for k in OPS]
    assert np.max(np.abs(P.decode(st.weights, tol=1e-3) - S.decode(es.weights))) < 1e-3


@pytest.mark.slow
def test_config4_training_step_full_size(golden):
    """BASELINE config 4: the first 128-row NAG step at N=2^16 (ledger per step
    164/101/382/518/4/54), weights vs the reference emulator's first snapshot."""
    P = _prod()
    from paper_2403_14111_b200 import workloads as wl
    X, y = wl.config4()
    Y = S.one_hot(y, wl.CLASSES)
    g = P.CKKSContext("cfg1", 128, seed=4, auto_bootstrap=True)
    w0 = S.init_weights(wl.CLASSES, X.shape[1], wl.INIT_SEED)
    W = P.encode(g, w0, "vertical")
    st = P.TrainState(W, W)
    P.nag_step(st, P.encode(g, X[:128]), P.encode(g, Y[:128], "horizontal"), wl.LEARNING_RATE, 128)
    assert _ledger(g) == [518, 101, 164, 382, 4, 54]
    w1 = P.decode(st.weights, tol=1e-3)
    assert np.max(np.abs(w1 - golden["cfg4_snaps"][0])) < 1e-3


def _adversarial(moduli, nl, N, kind, rng):
    """[2][nl][N] residues that push the lazy-reduction bounds: every word at
    q - 1, alternating 0 / q - 1, or uniform."""
    q = np.asarray(moduli[:nl], dtype=np.uint64)[None, :, None]
    if kind == "max":
        return np.broadcast_to(q - np.uint64(1), (2, nl, N)).copy()
    if kind == "alt":
        pat = (np.arange(N) % 2).astype(np.uint64)[None, None, :]
        return (pat * (q - np.uint64(1))).astype(np.uint64) + np.zeros((2, nl, N), np.uint64)
    return (rng.integers(0, 2 ** 63, (2, nl, N), dtype=np.uint64) % q).astype(np.uint64)


@pytest.mark.parametrize("name,grid", [("small12", 16), ("cfg1", 128)])
def test_adversarial_residues(name, grid):
    """Rescale, rotation, conjugation and ct x ct on extreme residues: the
    integer and FP64 lazy-bound paths (ntt_pass.cuh) must stay bit-exact."""
    P = _prod()
    g = P.CKKSContext(name, grid, seed=91)
    o = R.OracleCKKSContext(name, grid, seed=91)
    rng = np.random.default_rng(8)
    lv = g.max_level
    for kind in ("max", "alt", "rand"):
        data = _adversarial(g.moduli, lv + 1, g.N, kind, rng)
        gb, ob = g.from_residues(data, lv), R.RnsBlock(o, data, lv)
        np.testing.assert_array_equal(g.rescale(gb).residues(), o.p.rescale(data, lv))
        for r in (1, 5):
            np.testing.assert_array_equal(g.lrot(gb, r).residues(), o.lrot(ob, r).data)
        np.testing.assert_array_equal(S.ladder(g, gb, 3, 3).residues(), S.ladder(o, ob, 3, 3).data)
        np.testing.assert_array_equal(g.conj(gb).residues(), o.conj(ob).data)
        np.testing.assert_array_equal(g.mult(gb, gb).residues(), o.mult(ob, ob).data)
