"""GPU tests of the multi-rank path.

* ``hc_mod_reduce`` on genuinely unreduced sums of R canonical residues
  (R = 2, 4, 8; words up to R * q), against numpy ``%`` and the library's
  own modular adds.
* The config-4 data-parallel NAG step (training.py:66-100 on a batch of 8
  block rows) run as R simulated ranks on one GPU: one context per shard
  (``set_shard``), each thread driving its context, the DiagATB block-row
  pre-sums (encoding.py:375-377) exchanged by ``LocalModReducer`` and
  finished by ``hc_mod_reduce``.  Every rank's W and V residues must equal
  the single-context run over all 8 block rows bit for bit.
* ``NcclModReducer`` on a 1-rank NCCL group (stream handoff plumbing) is in
  test_gpu_parity.py.
"""

import gc
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _prod():
    import paper_2403_14111_b200 as P
    return P


@pytest.mark.parametrize("name,grid", [("small12", 16), ("cfg1", 128)])
@pytest.mark.parametrize("R", [2, 4, 8])
def test_mod_reduce_unreduced_sums(name, grid, R):
    P = _prod()
    g = P.CKKSContext(name, grid, seed=31)
    lv = g.max_level
    q = g.moduli[: lv + 1].astype(np.uint64)[None, :, None]
    rng = np.random.default_rng(R)
    parts = [(rng.integers(0, 2 ** 63, (2, lv + 1, g.N), dtype=np.uint64) % q).astype(np.uint64)
             for _ in range(R - 1)]
    parts.append(np.broadcast_to(q - np.uint64(1), (2, lv + 1, g.N)).copy())   # extreme words
    raw = np.zeros_like(parts[0])
    for p in parts:
        raw += p                                    # uint64, no wrap: R * q < 2^64
    assert raw.max() >= q.max()                     # the input is genuinely unreduced
    ct = g.from_residues(raw, lv)
    g.mod_reduce(ct)
    np.testing.assert_array_equal(ct.residues(), raw % q)
    # and the library's own modular adds of the parts
    acc = g.from_residues(parts[0], lv)
    for p in parts[1:]:
        acc = g.add(acc, g.from_residues(p, lv))
    np.testing.assert_array_equal(ct.residues(), acc.residues())


def _step_inputs(name):
    from paper_2403_14111_b200 import workloads as wl
    if name == "cfg1":
        X, y = wl.config4()
        return X, y, wl.CLASSES, wl.LEARNING_RATE, 128, wl.INIT_SEED
    rng = np.random.default_rng(44)
    X = rng.standard_normal((128, 32))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    return X, rng.integers(0, 3, 128), 3, 0.5, 16, 7


def _grid(ctx, res, shape, tiling, period):
    P = _prod()
    blocks = tuple(tuple(ctx.from_residues(r, r.shape[1] - 1) for r in row) for row in res)
    return P.EncodedMatrix(ctx, blocks, shape, tiling, period)


def _residues(M):
    return [[b.residues() for b in row] for row in M.blocks]


def _sharded_vs_single(name, worlds):
    P = _prod()
    from paper_2403_14111_b200 import sharding
    X, y, classes, lr, grid, wseed = _step_inputs(name)
    Y = P.one_hot(y, classes)
    w0 = P.init_weights(classes, X.shape[1], wseed)
    g = P.CKKSContext(name, grid, seed=4, auto_bootstrap=True)
    g.nonce = 100
    W, EX, EY = P.encode(g, w0, "vertical"), P.encode(g, X), P.encode(g, Y, "horizontal")
    m = EX.grid[0]
    assert m == 8
    wres, xres, yres = _residues(W), _residues(EX), _residues(EY)
    st = P.TrainState(W, W)
    g.nonce = 5000
    P.nag_step(st, EX, EY, lr, X.shape[0])
    ref_w, ref_v, ref_nonce = _residues(st.weights), _residues(st.momentum), g.nonce
    ref_led = g.ledger.counts()
    boots = ref_led["Bootstrap"]
    assert boots > 0                                   # the step refreshes (softmax and W / V)
    for R in worlds:
        red = sharding.LocalModReducer(R)
        ctxs = [P.CKKSContext(name, grid, seed=4, auto_bootstrap=True) for _ in range(R)]
        out, errs = [None] * R, []

        def run(r):
            try:
                c = ctxs[r]
                part = sharding.partition(m, R, r)
                c.set_shard(m, part.start)
                rows = slice(part.start * grid, part.stop * grid)
                Wr = _grid(c, wres, W.shape, "vertical", W.period)
                Xr = _grid(c, xres[part.start:part.stop], X[rows].shape, "none", None)
                Yr = _grid(c, yres[part.start:part.stop], Y[rows].shape, "horizontal", EY.period)
                s = P.TrainState(Wr, Wr)
                c.nonce = 5000
                P.nag_step(s, Xr, Yr, lr, X.shape[0], reducer=red.rank(r))
                out[r] = (_residues(s.weights), _residues(s.momentum), c.nonce)
            except Exception as e:     # surfaced below
                errs.append(e)
                red._bar.abort()

        th = [threading.Thread(target=run, args=(r,)) for r in range(R)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        for r in range(R):
            w, v, nonce = out[r]
            assert nonce == ref_nonce
            for a, b in zip(w, ref_w):
                for x, z in zip(a, b):
                    np.testing.assert_array_equal(x, z)
            for a, b in zip(v, ref_v):
                for x, z in zip(a, b):
                    np.testing.assert_array_equal(x, z)


def test_sharded_nag_step_bit_exact_small12():
    """8 block rows of 16 as 2, 3, 4 and 8 simulated ranks == 1 context."""
    _sharded_vs_single("small12", [2, 3, 4, 8])


@pytest.mark.slow
def test_sharded_nag_step_bit_exact_config4():
    """BASELINE config 4: the 1024-row step as 2 and 4 simulated ranks at
    N = 2^16 == the single-GPU run over all 8 block rows, bit for bit."""
    _sharded_vs_single("cfg1", [2, 4])


@pytest.mark.slow
def test_config4_step1_residues_vs_oracle():
    """The first 128-row config-4 NAG step: W and V residues equal the C
    RNS-CKKS oracle running the restated reference step (same seed, nonces)."""
    P = _prod()
    from oracle import rns as R
    from oracle import slots as S
    from paper_2403_14111_b200 import workloads as wl
    X, y = wl.config4()
    Y = S.one_hot(y, wl.CLASSES)
    w0 = S.init_weights(wl.CLASSES, X.shape[1], wl.INIT_SEED)
    g = P.CKKSContext("cfg1", 128, seed=4, auto_bootstrap=True)
    o = R.OracleCKKSContext("cfg1", 128, seed=4, auto_bootstrap=True)
    g.nonce = o.nonce = 0
    GW, OW = P.encode(g, w0, "vertical"), S.encode(o, w0, "vertical")
    GX, OX = P.encode(g, X[:128]), S.encode(o, X[:128])
    GY, OY = P.encode(g, Y[:128], "horizontal"), S.encode(o, Y[:128], "horizontal")
    gs, os_ = P.TrainState(GW, GW), S.State(OW, OW)
    P.nag_step(gs, GX, GY, wl.LEARNING_RATE, 128)
    S.nag_step(os_, OX, OY, wl.LEARNING_RATE, 128)
    for G, O in ((gs.weights, os_.weights), (gs.momentum, os_.momentum)):
        for gb, ob in zip(G.flat(), [b for r in O.blocks for b in r]):
            np.testing.assert_array_equal(gb.residues(), ob.data)
    assert g.nonce == o.nonce
    assert [g.ledger.counts()[k] for k in P.OP_KINDS] == [518, 101, 164, 382, 4, 54]


@pytest.mark.slow
def test_config4_epoch_vs_reference_snapshots(golden):
    """The reference's run_steps (training.py:340-375) with its own signature on
    the B200 context: 8 steps of 128 rows (one config-4 epoch); every decoded
    W against the reference emulator's snapshot, and the exact ledger."""
    P = _prod()
    from paper_2403_14111_b200 import workloads as wl
    X, y = wl.config4()
    g = P.CKKSContext("cfg1", 128, seed=4, auto_bootstrap=True)
    snaps = P.run_steps(X, y, wl.CLASSES, 8, ctx=g, batch_size=128, lr=wl.LEARNING_RATE, seed=wl.INIT_SEED)
    assert len(snaps) == 8
    for k, (got, ref) in enumerate(zip(snaps, golden["cfg4_snaps"])):
        assert np.max(np.abs(got - ref)) < 2e-3, k
    assert [g.ledger.counts()[k] for k in P.OP_KINDS] == list(golden["cfg4_led"])


def _pass_sharded(name, grid, fn, worlds):
    """DiagABT / DiagATB with the c/2 diagonal passes split over R simulated
    ranks (hc_set_pass_shard) == the single-context schedule, bit for bit."""
    P = _prod()
    from paper_2403_14111_b200 import sharding
    from paper_2403_14111_b200 import workloads as wl
    if name == "cfg1":
        X, W = wl.config1()
        PY, _ = wl.config2()
    else:
        rng = np.random.default_rng(12)
        X, W = rng.uniform(-1, 1, (32, 40)), rng.uniform(-1, 1, (4, 40))
        PY = rng.uniform(-1, 1, (32, 4))
    g = P.CKKSContext(name, grid, seed=2)
    g.nonce = 0
    EX, EW, EP = P.encode(g, X), P.encode(g, W, "vertical"), P.encode(g, PY, "horizontal")
    args = (EX, EW) if fn == "abt" else (EP, EX)
    run1 = P.diag_abt if fn == "abt" else P.diag_atb
    ref = run1(*args)
    res = [_residues(a) for a in args]
    ref_res = _residues(ref)
    for R in worlds:
        red = sharding.LocalModReducer(R)
        out, errs = [None] * R, []

        def run(r):
            try:
                c = P.CKKSContext(name, grid, seed=2)
                c.set_pass_shard(R, r, red.rank(r))
                mats = [_grid(c, rr, a.shape, a.tiling, a.period) for rr, a in zip(res, args)]
                out[r] = _residues(run1(*mats))
            except Exception as e:
                errs.append(e)
                red._bar.abort()

        th = [threading.Thread(target=run, args=(r,)) for r in range(R)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        for r in range(R):
            for a, b in zip(out[r], ref_res):
                for x, z in zip(a, b):
                    np.testing.assert_array_equal(x, z)
        del th, red
        gc.collect()   # the R shard contexts (keys + reserved pool each) before the next world


@pytest.mark.parametrize("fn", ["abt", "atb"])
def test_pass_sharded_small12(fn):
    _pass_sharded("small12", 16, fn, [2])


@pytest.mark.slow
@pytest.mark.parametrize("fn", ["abt", "atb"])
def test_pass_sharded_config1(fn):
    """The bench pair's multi-GPU form: 8 passes over 2, 4 and 8 ranks."""
    _pass_sharded("cfg1", 128, fn, [2, 4, 8])
