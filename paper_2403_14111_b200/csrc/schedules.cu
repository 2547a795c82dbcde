// Native schedules: the reference's layer-1/2 op sequences issued straight
// to the device evaluator.  Grid operations are applied block by block in
// the order the reference's EncodedMatrix.map_blocks / _zip evaluate them,
// and every composite expression is split into explicit steps so the op
// order (and therefore the refresh-nonce sequence) is the reference's.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <map>

#include "schedules.h"

namespace hc {

using G = std::vector<CtP>;
using cd = std::complex<double>;

// Fork/join of independent schedule branches (the c/2 diagonal passes) onto
// side streams.  Branch k runs on side stream k % S after waiting for
// everything the main stream issued before the fork; join() makes the main
// stream wait for all branches.  Temporaries of a branch are allocated and
// freed on its stream; branch results outlive the join and are freed on the
// main stream afterwards.  The op sequence (and therefore every residue) is
// unchanged: only the host-side issue order interleaves.
//
// Forks nest: a fork at nesting depth d draws its streams from pool d
// (FORK_POOL streams each), records its fork event on the stream that was
// current when it was created (the parent branch's stream) and joins back
// onto that stream.
constexpr int FORK_POOL = 32, FORK_DEPTHS = 3;

struct Fork {
    Ctx& c;
    int S, base;
    cudaStream_t parent;
    cudaEvent_t ev;
    std::vector<char> used;
    Fork(Ctx& ctx, int nstreams) : c(ctx), used(FORK_POOL, 0) {
        const int depth = c.fork_depth++;
        if (depth >= FORK_DEPTHS) {
            S = 0;                                  // too deep: run inline on the parent stream
            base = 0;
        } else {
            S = std::max(1, std::min(nstreams, FORK_POOL));
            // nested forks of sibling branches rotate through their pool so
            // they do not serialise on the same streams
            int off = 0;
            if (depth > 0) {
                off = c.fork_rot[depth];
                if (off + S > FORK_POOL) off = 0;
                c.fork_rot[depth] = off + S;
            }
            base = depth * FORK_POOL + off;
        }
        while ((int)c.side.size() < FORK_POOL * FORK_DEPTHS) {
            cudaStream_t s;
            HC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            c.side.push_back(s);
            cudaEvent_t e;
            HC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c.side_ev.push_back(e);
        }
        parent = c.stream;
        if (c.fork_evs.size() <= (size_t)depth) {
            cudaEvent_t e;
            HC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c.fork_evs.push_back(e);
        }
        ev = c.fork_evs[depth];
        if (S) HC_CUDA(cudaEventRecord(ev, parent));
    }
    void enter(int k) {
        if (!S) return;
        const int s = k % S;
        if (!used[s]) {
            HC_CUDA(cudaStreamWaitEvent(c.side[base + s], ev, 0));
            used[s] = 1;
        }
        c.stream = c.side[base + s];
    }
    void leave() { c.stream = parent; }
    void join() {
        c.stream = parent;
        for (int s = 0; s < S; s++) {
            if (!used[s]) continue;
            HC_CUDA(cudaEventRecord(c.side_ev[base + s], c.side[base + s]));
            HC_CUDA(cudaStreamWaitEvent(parent, c.side_ev[base + s], 0));
            used[s] = 0;
        }
    }
    ~Fork() {
        c.stream = parent;
        for (int s = 0; s < S; s++)
            if (used[s]) {
                cudaEventRecord(c.side_ev[base + s], c.side[base + s]);
                cudaStreamWaitEvent(parent, c.side_ev[base + s], 0);
            }
        c.fork_depth--;
    }
};

// run fn(i) for i < count as concurrent branches (width capped by the context)
template <class F>
static void par_for(Ctx& c, int count, int width, F&& fn) {
    if (count <= 1 || std::min(width, c.fork_cap) <= 1) {
        for (int i = 0; i < count; i++) fn(i);
        return;
    }
    Fork fork(c, std::min(width, c.fork_cap));
    for (int i = 0; i < count; i++) {
        fork.enter(i);
        fn(i);
        fork.leave();
    }
    fork.join();
}

static int fork_width(const Ctx& c, int branches) { return std::max(1, std::min(branches, c.fork_cap)); }

static int ilog2(int n) {
    int l = 0;
    while ((1 << l) < n) l++;
    return l;
}

// ---- slot patterns (encoding.py:231-278, approx.py:149-163) ---------------

struct Geo {
    int s0, s1, S;
};

static Geo geo(const Eval& ev, int s0) { return Geo{s0, (ev.c.N / 2) / s0, ev.c.N / 2}; }

static std::string dkey(double v) {
    char b[32];
    std::snprintf(b, sizeof b, "%a", v);
    return b;
}

// make_mask: 1 at (i, j) with j = i + shift (mod modulus); complexified:
// 0.5 M(shift) - 0.5i M(shift + modulus/2); times scale
static Pattern diag_mask(const Geo& g, int shift, int modulus, bool cplx, double scale) {
    shift = ((shift % modulus) + modulus) % modulus;
    Pattern p;
    p.key = "diag:" + std::to_string(g.s0) + ":" + std::to_string(shift) + ":" + std::to_string(modulus) + ":" +
            (cplx ? "c" : "r") + ":" + dkey(scale);
    p.gen = [g, shift, modulus, cplx, scale](std::vector<cd>& vals) {
        for (int i = 0; i < g.s0; i++)
            for (int j = 0; j < g.s1; j++) {
                const double main = ((((j - i - shift) % modulus) + modulus) % modulus == 0) ? 1.0 : 0.0;
                cd v;
                if (cplx) {
                    const double twin =
                        ((((j - i - shift - modulus / 2) % modulus) + modulus) % modulus == 0) ? 1.0 : 0.0;
                    v = cd(0.5 * main, 0.0) - cd(0.0, 0.5 * twin);
                } else {
                    v = cd(main, 0.0);
                }
                vals[(size_t)i * g.s1 + j] = cd(v.real() * scale, v.imag() * scale);
            }
    };
    return p;
}

template <class F>
static Pattern col_pattern(const Geo& g, const std::string& key, F f) {
    Pattern p;
    p.key = key + ":" + std::to_string(g.s0);
    p.gen = [g, f](std::vector<cd>& vals) {
        for (int i = 0; i < g.s0; i++)
            for (int j = 0; j < g.s1; j++) vals[(size_t)i * g.s1 + j] = cd(f(j), 0.0);
    };
    return p;
}

static Pattern keep_head(const Geo& g, int stop) {
    return col_pattern(g, "head:" + std::to_string(stop), [stop](int j) { return j < stop ? 1.0 : 0.0; });
}
static Pattern col0(const Geo& g) {
    return col_pattern(g, "col0", [](int j) { return j == 0 ? 1.0 : 0.0; });
}

// ---- structural ops (encoding.py:284-381) ----------------------------------

// rot_up on a block row / column: lrot(k * s1) per block; k == 0 returns the input
static G rot_up(Eval& ev, const G& E, int k, const Geo& g) {
    k %= g.s0;
    if (k == 0) return E;
    G o(E.size());
    for (size_t i = 0; i < E.size(); i++) o[i] = ev.lrot(E[i], (int64_t)k * g.s1);
    return o;
}

static G rot_left(Eval& ev, const G& E, int k, const Geo& g) {
    k %= g.s1;
    if (k == 0) return E;
    const Pattern keep = keep_head(g, g.s1 - k);
    G o(E.size());
    for (size_t i = 0; i < E.size(); i++) {
        CtP a1 = ev.lrot(E[i], k);
        CtP head = ev.mult_p(a1, keep);
        CtP tail = ev.sub(a1, head);
        CtP back = ev.rrot(tail, g.s1);
        o[i] = ev.add(head, back);
    }
    return o;
}

static G prot_up(Eval& ev, const G& E, int k, const Geo& g) {
    k %= g.s1;
    if (k == 0) return E;
    const Pattern keep = keep_head(g, g.s1 - k);
    G o(E.size());
    for (size_t i = 0; i < E.size(); i++) {
        CtP head = ev.mult_p(E[i], keep);
        CtP tail = ev.sub(E[i], head);
        CtP up = ev.lrot(tail, g.s1);
        o[i] = ev.add(head, up);
    }
    return o;
}

// col_sums over an r x cols grid -> r blocks
static G col_sums(Eval& ev, const G& E, int r, int cols, const Geo& g, int width = 1) {
    const Pattern c0 = col0(g);
    G out(r);
    par_for(ev.c, r, width, [&](int p) {
        CtP acc = E[(size_t)p * cols];
        for (int q = 1; q < cols; q++) acc = ev.add(acc, E[(size_t)p * cols + q]);
        acc = ev.ladder(acc, 1, ilog2(g.s1));
        acc = ev.mult_p(acc, c0);
        acc = ev.ladder(acc, -1, ilog2(g.s1));
        out[p] = acc;
    });
    return out;
}

// row_sums over an r x cols grid -> cols blocks; the block-row pre-add is the
// cross-rank reduction point (encoding.py:375-377)
static G row_sums(Eval& ev, const G& E, int r, int cols, const Geo& g, const Reducer& red) {
    G pre(cols);
    for (int q = 0; q < cols; q++) {
        CtP acc = E[q];
        for (int p = 1; p < r; p++) acc = ev.add(acc, E[(size_t)p * cols + q]);
        pre[q] = acc;
    }
    if (red) red(pre);
    for (int q = 0; q < cols; q++) {
        pre[q] = ev.ladder(pre[q], g.s1, ilog2(g.s0));
    }
    return pre;
}

static int grid_level(const G& E) {
    int l = 1 << 30;
    for (auto& b : E) l = std::min(l, b->level);
    return l;
}

static int geo_rows(const Eval& ev) {
    if (ev.c.grid_rows <= 0) throw Error(-1, "grid_rows not set (hc_set_grid_rows)");
    return ev.c.grid_rows;
}

// ---- key-switch throughput probe (measurement only) ------------------------
// `streams` independent chains of `reps` rotations each (chain i rotates by
// i + 1, so every chain uses its own key), issued through the same fork/join
// machinery as the schedules.  Returns the number of key switches issued.
int64_t probe_rotations(Eval& ev, const CtP& x, int streams, int reps, int batch) {
    for (int i = 0; i < streams; i++) get_key(ev.c, (int)galois_rot(ev.c, i + 1));
    par_for(ev.c, streams, streams, [&](int i) {
        if (batch <= 1) {
            CtP a = x;
            for (int r = 0; r < reps; r++) a = ev.lrot(a, i + 1);
            return;
        }
        G a(batch);
        for (int b = 0; b < batch; b++) a[b] = ev.add(x, x);   // distinct operands
        for (int r = 0; r < reps; r++) a = ev.lrot_batch(a, i + 1);
    });
    return (int64_t)streams * reps * std::max(1, batch);
}

// `streams` independent branches, each running `reps` ladders (stride, steps)
// over its own batch of `batch` ciphertexts (measurement only).
void probe_ladders(Eval& ev, const CtP& x, int streams, int batch, int64_t stride, int steps, int reps) {
    par_for(ev.c, streams, streams, [&](int) {
        G a(batch);
        for (int b = 0; b < batch; b++) a[b] = ev.add(x, x);   // distinct operands
        for (int r = 0; r < reps; r++) a = ev.ladder(a, stride, steps);
    });
}

// ---- lockstep (batched) forms ----------------------------------------------
// When no auto-bootstrap can fire, the independent diagonal passes run in
// lockstep: every op that the passes (and blocks) apply with the same Galois
// element becomes one batched key-switch pipeline (the ladders of all c/2
// passes, the products of all passes, the RU/RL rotations of all blocks).
// Each ciphertext sees exactly the op sequence of the reference (residues
// unchanged); only the issue order across independent branches differs.

// A batched op over many independent operands: sub-batches of at most
// C.batch run as concurrent branches, so one sub-batch's pipeline tails
// overlap another's kernels.
static G rot_many(Eval& ev, const G& xs, int64_t r, bool add_self = false) {
    Ctx& C = ev.c;
    const int SB = std::max(1, C.batch), nsub = ((int)xs.size() + SB - 1) / SB;
    if (nsub <= 1) return ev.lrot_batch(xs, r, add_self);
    G out(xs.size());
    par_for(C, nsub, fork_width(C, nsub), [&](int i) {
        const size_t lo = (size_t)i * SB, hi = std::min(xs.size(), lo + SB);
        G part = ev.lrot_batch(G(xs.begin() + lo, xs.begin() + hi), r, add_self);
        std::copy(part.begin(), part.end(), out.begin() + lo);
    });
    return out;
}

// the doubling ladder of many independent operands (Eval::ladder), in
// sub-batches on concurrent branches like rot_many
static G ladder_many(Eval& ev, const G& xs, int64_t stride, int steps) {
    Ctx& C = ev.c;
    const int SB = std::max(1, C.batch);
    // sub-batches of one level each (a batched pipeline needs one level; DiagATB's
    // passes end one level apart), in first-appearance order
    std::vector<std::vector<size_t>> subs;
    {
        std::vector<std::pair<int, std::vector<size_t>>> by_level;
        for (size_t i = 0; i < xs.size(); i++) {
            size_t u = 0;
            while (u < by_level.size() && by_level[u].first != xs[i]->level) u++;
            if (u == by_level.size()) by_level.emplace_back(xs[i]->level, std::vector<size_t>());
            by_level[u].second.push_back(i);
        }
        for (auto& lv : by_level)
            for (size_t lo = 0; lo < lv.second.size(); lo += SB)
                subs.emplace_back(lv.second.begin() + lo, lv.second.begin() + std::min(lv.second.size(), lo + (size_t)SB));
    }
    const int nsub = (int)subs.size();
    if (nsub <= 1) return ev.ladder(xs, stride, steps);
    G out(xs.size());
    par_for(C, nsub, fork_width(C, nsub), [&](int i) {
        G in;
        for (size_t j : subs[i]) in.push_back(xs[j]);
        G part = ev.ladder(in, stride, steps);
        for (size_t u = 0; u < subs[i].size(); u++) out[subs[i][u]] = part[u];
    });
    return out;
}

static G mult_many(Eval& ev, const G& xs_in, const G& ys_in) {
    Ctx& C = ev.c;
    const int SB = std::max(1, C.batch), nsub = ((int)xs_in.size() + SB - 1) / SB;
    if (nsub <= 1) return ev.mult_batch(xs_in, ys_in);
    // operands shared across sub-batches (DiagATB's B blocks, one use per
    // pass) are level-adjusted once here, before the fan-out; residues are
    // those of the per-product adjustment (deterministic)
    G xs = xs_in, ys = ys_in;
    bool boot = false;
    for (size_t i = 0; i < xs.size(); i++) boot |= xs[i]->level < 1 || ys[i]->level < 1;
    if (!boot) {
        // one batch per (source level, target level), shared operands once
        std::vector<int> ls(xs.size());
        for (size_t i = 0; i < xs.size(); i++) ls[i] = std::min(xs[i]->level, ys[i]->level);
        ev.at_batch(xs, ls);
        ev.at_batch(ys, ls);
    }
    G out(xs.size());
    par_for(C, nsub, fork_width(C, nsub), [&](int i) {
        const size_t lo = (size_t)i * SB, hi = std::min(xs.size(), lo + SB);
        G part = ev.mult_batch(G(xs.begin() + lo, xs.begin() + hi), G(ys.begin() + lo, ys.begin() + hi));
        std::copy(part.begin(), part.end(), out.begin() + lo);
    });
    return out;
}

static G concat(const std::vector<G>& parts) {
    G o;
    for (auto& p : parts) o.insert(o.end(), p.begin(), p.end());
    return o;
}

// Diagonal-pass sharding (hc_set_pass_shard): the c/2 passes
// are independent; this context runs passes k = rank, rank + world, ...,
// hands its partial accumulator (the sum of its passes' terms) to the pass
// reducer, which replaces it by the modular sum over ranks, and every rank
// finishes the replicated conj epilogue.  Modular sums are exact, so the
// result equals the single-context schedule bit for bit.
static std::vector<int> local_passes(const Ctx& C, int K) {
    std::vector<int> ks;
    for (int k = C.pass_rank; k < K; k += std::max(1, C.pass_world)) ks.push_back(k);
    if (ks.empty()) throw Error(-4, "pass sharding: more ranks than diagonal passes");
    return ks;
}

// `lstar` is the level every pass's term reaches in the unsharded schedule's
// sum (its lowest): a partial above it is adjusted first, which is the same
// adjustment the unsharded sum applies to the higher-level pass (k = 0) when
// the next pass is added, so the modular sum over ranks matches bit for bit.
static G reduce_passes(Eval& ev, G out, int lstar) {
    if (ev.c.pass_world > 1) {
        if (!ev.c.pass_reducer) throw Error(-4, "pass sharding without a pass reducer");
        for (auto& x : out) {
            if (x->level < lstar) throw Error(-4, "pass sharding: partial below the common level");
            x = ev.at(x, lstar);
        }
        ev.c.pass_reducer(out);
    }
    return out;
}

static std::vector<CtP> diag_abt_lockstep(Eval& ev, const G& A, int m, int n, const G& B, int c, double scale,
                                          const Geo& g) {
    const std::vector<int> ks = local_passes(ev.c, c / 2);
    const int K = (int)ks.size();
    // packing prologue: B + i * RU(B, c/2), all block columns in one batch
    const int kk0 = (c / 2) % g.s0;
    G rolled = kk0 ? ev.lrot_batch(B, (int64_t)kk0 * g.s1) : B;
    G ri(n);
    for (int q = 0; q < n; q++) ri[q] = ev.mul_i(rolled[q]);
    G packed = ev.add_batch(B, ri);
    std::vector<G> shifted(K);
    G acc((size_t)K * m);
    if (ev.c.hoist) {
        // fused form (oracle/slots.py diag_abt): RU(packed, k)
        // of every pass with one ModUp per block column, and each (pass, block
        // row) product sum -- the col_sums pre-add of the rowwise products --
        // relinearised and rescaled once
        std::vector<int64_t> amounts(K);
        for (int u = 0; u < K; u++) amounts[u] = (int64_t)(ks[u] % g.s0) * g.s1;
        std::vector<G> H = ev.lrot_hoisted(packed, amounts);
        std::vector<G> as, bs;
        for (int k = 0; k < K; k++)
            for (int p = 0; p < m; p++) {
                as.emplace_back(A.begin() + (size_t)p * n, A.begin() + (size_t)(p + 1) * n);
                G b(n);
                for (int q = 0; q < n; q++) b[q] = H[q][k];
                bs.push_back(b);
            }
        acc = ev.mult_sum_batch(as, bs);
    } else {
        // RU(packed, k) per pass (one batch per k: its own Galois element)
        for (int k = 0; k < K; k++) {
            const int kk = ks[k] % g.s0;
            shifted[k] = kk ? ev.lrot_batch(packed, (int64_t)kk * g.s1) : packed;
        }
        // all passes' products in one batch
        G xs, ys;
        for (int k = 0; k < K; k++)
            for (int p = 0; p < m; p++)
                for (int q = 0; q < n; q++) {
                    xs.push_back(A[(size_t)p * n + q]);
                    ys.push_back(shifted[k][q]);
                }
        G prod = mult_many(ev, xs, ys);
        // col_sums of every (pass, block row): pre-add, then the ladders in lockstep
        for (int k = 0; k < K; k++)
            for (int p = 0; p < m; p++) {
                const size_t base = ((size_t)k * m + p) * n;
                CtP a = prod[base];
                for (int q = 1; q < n; q++) a = ev.add(a, prod[base + q]);
                acc[(size_t)k * m + p] = a;
            }
    }
    acc = ladder_many(ev, acc, 1, ilog2(g.s1));
    const Pattern c0 = col0(g);
    acc = ev.mult_p_batch(acc, std::vector<const Pattern*>(acc.size(), &c0));
    acc = ladder_many(ev, acc, -1, ilog2(g.s1));
    std::vector<G> terms(K, G(m));
    {
        std::vector<Pattern> masks;
        for (int k = 0; k < K; k++) masks.push_back(diag_mask(g, ks[k], c, true, scale));
        std::vector<const Pattern*> ps;
        for (int k = 0; k < K; k++)
            for (int p = 0; p < m; p++) ps.push_back(&masks[k]);
        G t = ev.mult_p_batch(acc, ps);
        for (int k = 0; k < K; k++)
            for (int p = 0; p < m; p++) terms[k][p] = t[(size_t)k * m + p];
    }
    G out = terms[0];
    for (int k = 1; k < K; k++) out = ev.add_batch(out, terms[k]);
    out = reduce_passes(ev, out, out[0]->level);   // every pass's term at one level
    G cj = ev.conj_batch(out);
    return ev.add_batch(out, cj);
}

// rot_left of every block of E by k (encoding.py:291-311); the rrot(s1) of
// several calls can be gathered by the caller: returns (head, tail) pairs.
// `first`, when given, holds lrot(E, k) already (hoisted by the caller).
static void rot_left_split(Eval& ev, const G& E, int k, const Geo& g, G& head, G& tail, const G* first = nullptr) {
    const Pattern keep = keep_head(g, g.s1 - k);
    G a1 = first ? *first : ev.lrot_batch(E, k);
    head = ev.mult_p_batch(a1, std::vector<const Pattern*>(a1.size(), &keep));
    tail = ev.add_batch(a1, head, true);
}

static std::vector<CtP> diag_atb_lockstep(Eval& ev, const G& A, int m, const G& B, int n, int c, double scale,
                                          const Geo& g, const Reducer& red) {
    const std::vector<int> ks = local_passes(ev.c, c / 2);
    const int K = (int)ks.size();
    const int s1 = g.s1;
    const bool partial = grid_level(A) < grid_level(B);
    // packing prologue: A + i * RL(A, c/2)
    G packed(m);
    {
        const int k = (c / 2) % s1;
        G one = A;
        if (k) {
            G head, tail;
            rot_left_split(ev, A, k, g, head, tail);
            G back = ev.lrot_batch(tail, -(int64_t)s1);
            one = ev.add_batch(head, back);
        }
        G oi(m);
        for (int p = 0; p < m; p++) oi[p] = ev.mul_i(one[p]);
        packed = ev.add_batch(A, oi);
    }
    // the level of pass k's term (all passes, for pass sharding): RL / PRU of
    // a non-zero k costs the rotated operand one level, then the product and
    // the mask one each
    int lstar = 1 << 30;
    for (int k = 0; k < c / 2; k++) {
        int ll = grid_level(packed), lr = grid_level(B);
        if (k % s1) (partial ? lr : ll) -= 1;
        lstar = std::min(lstar, std::min(ll, lr) - 2);
    }
    // left operands of every pass; fused form (oracle/slots.py
    // diag_atb): the leading rotations lrot(packed, k) share one ModUp per block
    std::vector<G> left(K);
    std::vector<G> first(K);
    if (ev.c.hoist) {
        std::vector<int64_t> amounts(K);
        for (int k = 0; k < K; k++) amounts[k] = partial ? ks[k] : ks[k] % s1;
        std::vector<G> H = ev.lrot_hoisted(packed, amounts);
        for (int k = 0; k < K; k++) {
            first[k].resize(m);
            for (int p = 0; p < m; p++) first[k][p] = H[p][k];
        }
    }
    if (partial) {
        for (int k = 0; k < K; k++) left[k] = ev.c.hoist ? first[k] : ev.lrot_batch(packed, ks[k]);
    } else {
        // RL per pass (encoding.py:291-311): head = lrot(packed, k) * keep_k,
        // tail = lrot - head, left = head + rrot(tail, s1); the keep masks of
        // every pass in one batch, the rrot(s1) of every tail in one batch
        std::vector<int> moving;
        for (int k = 0; k < K; k++) {
            if (ks[k] % s1 == 0) left[k] = packed;
            else moving.push_back(k);
        }
        std::vector<Pattern> keeps;
        for (int k : moving) keeps.push_back(keep_head(g, s1 - ks[k] % s1));
        G a1s;
        std::vector<const Pattern*> ps;
        for (size_t u = 0; u < moving.size(); u++) {
            const int k = moving[u];
            const G a1 = ev.c.hoist ? first[k] : ev.lrot_batch(packed, ks[k] % s1);
            for (int p = 0; p < m; p++) {
                a1s.push_back(a1[p]);
                ps.push_back(&keeps[u]);
            }
        }
        G heads = ev.mult_p_batch(a1s, ps);
        G tails = ev.add_batch(a1s, heads, true);   // one batch; a shared a1 is level-adjusted once
        G back = rot_many(ev, tails, -(int64_t)s1);
        G lefts = ev.add_batch(heads, back);
        size_t o = 0;
        for (int k : moving) {
            left[k].resize(m);
            for (int p = 0; p < m; p++, o++) left[k][p] = lefts[o];
        }
    }
    // right operands: B, or PRU(B, k) on the partial branch (all lrot(s1) in one batch)
    std::vector<G> right(K, B);
    if (partial) {
        // the keep masks of every (pass, block) in one batch, the tails in one
        // batch (B's blocks are level-adjusted once for all passes), the
        // lrot(s1) of every tail in one batch, the sums in one batch
        std::vector<int> moving;
        for (int k = 0; k < K; k++)
            if (ks[k] % s1) moving.push_back(k);
        std::vector<Pattern> keeps;
        keeps.reserve(moving.size());
        G src;
        std::vector<const Pattern*> ps;
        for (int k : moving) {
            keeps.push_back(keep_head(g, s1 - ks[k] % s1));
            for (size_t i = 0; i < B.size(); i++) {
                src.push_back(B[i]);
                ps.push_back(&keeps.back());
            }
        }
        if (!src.empty()) {
            G hd = ev.mult_p_batch(src, ps);
            G tl = ev.add_batch(src, hd, true);
            G up = rot_many(ev, tl, (int64_t)s1);
            G rt = ev.add_batch(hd, up);
            size_t o = 0;
            for (int k : moving)
                for (size_t i = 0; i < B.size(); i++) right[k][i] = rt[o++];
        }
    }
    // all passes' products in one batch
    G xs, ys;
    for (int k = 0; k < K; k++)
        for (int p = 0; p < m; p++)
            for (int q = 0; q < n; q++) {
                xs.push_back(left[k][p]);
                ys.push_back(right[k][(size_t)p * n + q]);
            }
    G prod = mult_many(ev, xs, ys);
    // row_sums: block-row pre-adds (cross-rank reduction point, in pass order),
    // then the ladders of every (pass, block column) in lockstep
    G acc((size_t)K * n);
    for (int k = 0; k < K; k++)
        for (int q = 0; q < n; q++) acc[(size_t)k * n + q] = prod[((size_t)k * m) * n + q];
    for (int p = 1; p < m; p++) {   // one batched add per block row, every (pass, column) at once
        G rhs((size_t)K * n);
        for (int k = 0; k < K; k++)
            for (int q = 0; q < n; q++) rhs[(size_t)k * n + q] = prod[((size_t)k * m + p) * n + q];
        acc = ev.add_batch(acc, rhs);
    }
    if (red)
        for (int k = 0; k < K; k++) {
            G pre(acc.begin() + (size_t)k * n, acc.begin() + (size_t)(k + 1) * n);
            red(pre);
            for (int q = 0; q < n; q++) acc[(size_t)k * n + q] = pre[q];
        }
    acc = ladder_many(ev, acc, s1, ilog2(g.s0));
    std::vector<G> terms(K, G(n));
    {
        std::vector<Pattern> masks;
        for (int k = 0; k < K; k++) masks.push_back(diag_mask(g, -ks[k], c, true, scale));
        std::vector<const Pattern*> ps;
        for (int k = 0; k < K; k++)
            for (int q = 0; q < n; q++) ps.push_back(&masks[k]);
        G t = ev.mult_p_batch(acc, ps);
        for (int k = 0; k < K; k++)
            for (int q = 0; q < n; q++) terms[k][q] = t[(size_t)k * n + q];
    }
    G out = terms[0];
    for (int k = 1; k < K; k++) out = ev.add_batch(out, terms[k]);
    out = reduce_passes(ev, out, lstar);
    G cj = ev.conj_batch(out);
    return ev.add_batch(out, cj);
}

// ---- DiagABT (matmul.py:74-110) --------------------------------------------

std::vector<CtP> sched_diag_abt(Eval& ev, const std::vector<CtP>& A, int m, int n, const std::vector<CtP>& B, int c,
                                double scale) {
    const Geo g = geo(ev, geo_rows(ev));
    if (c < 1 || c > g.s1 || (c & (c - 1))) throw Error(-4, "diag_abt: bad period");
    if ((int)A.size() != m * n || (int)B.size() != n) throw Error(-4, "diag_abt: grid mismatch");
    if (c == 1) {
        G prod((size_t)m * n);
        for (int p = 0; p < m; p++)
            for (int q = 0; q < n; q++) prod[(size_t)p * n + q] = ev.mult(A[(size_t)p * n + q], B[q]);
        G sums = col_sums(ev, prod, m, n, g);
        const Pattern ones = diag_mask(g, 0, 1, false, scale);
        for (int p = 0; p < m; p++) sums[p] = ev.mult_p(sums[p], ones);
        return sums;
    }
    Ctx& C = ev.c;
    // Branches may run concurrently (or in lockstep) only when no
    // auto-bootstrap can fire inside (DiagABT consumes 3 levels), so the
    // refresh-nonce order is the reference's sequential one.
    const bool par = !ev.auto_boot || std::min(grid_level(A), grid_level(B)) >= 4;
    // the fused forms exist only in lockstep form: hoist implies lockstep
    if (par && (C.lockstep || C.hoist)) return diag_abt_lockstep(ev, A, m, n, B, c, scale, g);
    if (C.pass_world > 1) throw Error(-4, "pass sharding needs the lockstep schedule (no refresh inside)");
    auto W = [&](int w) { return par ? w : 1; };
    // packing prologue, one branch per block column: B + i * RU(B, c/2)
    G packed(n);
    par_for(C, n, W(n), [&](int q) {
        const int kk = (c / 2) % g.s0;
        CtP rolled = kk ? ev.lrot(B[q], (int64_t)kk * g.s1) : B[q];
        CtP mi = ev.mul_i(rolled);
        packed[q] = ev.add(B[q], mi);
    });
    // the c/2 diagonal passes are independent: one branch each, and inside a
    // pass the per-block-column rotation + products run as nested branches
    std::vector<G> terms(c / 2);
    par_for(C, c / 2, W(fork_width(C, c / 2)), [&](int k) {
        G prod((size_t)m * n);
        par_for(C, n, W(n), [&](int q) {
            const int kk = k % g.s0;
            CtP shifted = kk ? ev.lrot(packed[q], (int64_t)kk * g.s1) : packed[q];
            for (int p = 0; p < m; p++) prod[(size_t)p * n + q] = ev.mult(A[(size_t)p * n + q], shifted);
        });
        G sums = col_sums(ev, prod, m, n, g, W(m));
        const Pattern mask = diag_mask(g, k, c, true, scale);
        terms[k].resize(m);
        for (int p = 0; p < m; p++) terms[k][p] = ev.mult_p(sums[p], mask);
    });
    G acc = terms[0];
    for (int k = 1; k < c / 2; k++)
        for (int p = 0; p < m; p++) acc[p] = ev.add(acc[p], terms[k][p]);
    par_for(C, m, W(m), [&](int p) {
        CtP cj = ev.conj(acc[p]);
        acc[p] = ev.add(acc[p], cj);
    });
    return acc;
}

// ---- DiagATB (matmul.py:113-154) -------------------------------------------

std::vector<CtP> sched_diag_atb(Eval& ev, const std::vector<CtP>& A, int m, const std::vector<CtP>& B, int n, int c,
                                double scale, const Reducer& red) {
    const Geo g = geo(ev, geo_rows(ev));
    if (c < 1 || c > g.s0 || g.s0 % c) throw Error(-4, "diag_atb: bad period");
    if ((int)A.size() != m || (int)B.size() != m * n) throw Error(-4, "diag_atb: grid mismatch");
    auto colwise = [&](const G& C, const G& Bm) {
        G prod((size_t)m * n);
        for (int p = 0; p < m; p++)
            for (int q = 0; q < n; q++) prod[(size_t)p * n + q] = ev.mult(C[p], Bm[(size_t)p * n + q]);
        return prod;
    };
    if (c == 1) {
        G sums = row_sums(ev, colwise(A, B), m, n, g, red);
        const Pattern ones = diag_mask(g, 0, 1, false, scale);
        for (int q = 0; q < n; q++) sums[q] = ev.mult_p(sums[q], ones);
        return sums;
    }
    const bool partial = grid_level(A) < grid_level(B);
    Ctx& C = ev.c;
    const int s1 = g.s1;
    // Serial when an auto-bootstrap could fire inside (DiagATB consumes 4
    // levels): concurrent branches would reorder the refresh nonces.  A
    // cross-rank reducer is fine: the host still reaches the k-th pre-sum's
    // collective in k order on every rank, and only that branch waits for it.
    const bool ser = ev.auto_boot && std::min(grid_level(A), grid_level(B)) < 5;
    if (!ser && (C.lockstep || C.hoist)) return diag_atb_lockstep(ev, A, m, B, n, c, scale, g, red);
    if (C.pass_world > 1) throw Error(-4, "pass sharding needs the lockstep schedule (no refresh inside)");
    const int width = ser ? 1 : fork_width(C, c / 2);
    // packing prologue per block row: A + i * RL(A, c/2)
    G packed(m);
    par_for(C, m, ser ? 1 :m, [&](int p) {
        G one = rot_left(ev, G{A[p]}, c / 2, g);
        CtP mi = ev.mul_i(one[0]);
        packed[p] = ev.add(A[p], mi);
    });
    std::vector<G> terms(c / 2);
    par_for(C, c / 2, width, [&](int k) {
        G left(m);
        G right = B;
        if (partial) {
            for (int p = 0; p < m; p++) left[p] = ev.lrot(packed[p], k);
        } else {
            for (int p = 0; p < m; p++) left[p] = rot_left(ev, G{packed[p]}, k, g)[0];
        }
        // products (and, on the PRU branch, the partial row rotation of B) per block column
        G prod((size_t)m * n);
        par_for(C, n, ser ? 1 :n, [&](int q) {
            for (int p = 0; p < m; p++) {
                CtP r = B[(size_t)p * n + q];
                if (partial) r = prot_up(ev, G{r}, k, g)[0];
                prod[(size_t)p * n + q] = ev.mult(left[p], r);
            }
        });
        // row_sums: block-row pre-add (cross-rank reduction point), then per column the ladder
        G pre(n);
        for (int q = 0; q < n; q++) {
            CtP a = prod[q];
            for (int p = 1; p < m; p++) a = ev.add(a, prod[(size_t)p * n + q]);
            pre[q] = a;
        }
        if (red) red(pre);
        const Pattern mask = diag_mask(g, -k, c, true, scale);
        terms[k].resize(n);
        par_for(C, n, ser ? 1 :n, [&](int q) {
            CtP a = ev.ladder(pre[q], s1, ilog2(g.s0));
            terms[k][q] = ev.mult_p(a, mask);
        });
    });
    G acc = terms[0];
    for (int k = 1; k < c / 2; k++)
        for (int q = 0; q < n; q++) acc[q] = ev.add(acc[q], terms[k][q]);
    par_for(C, n, ser ? 1 :n, [&](int q) {
        CtP cj = ev.conj(acc[q]);
        acc[q] = ev.add(acc[q], cj);
    });
    return acc;
}

// ---- Table-4 baselines (matmul.py:160-237) ---------------------------------

static Pattern row_select(const Geo& g, int j, double v) {
    Pattern p;
    p.key = "rowsel:" + std::to_string(g.s0) + ":" + std::to_string(j) + ":" + dkey(v);
    p.gen = [g, j, v](std::vector<cd>& vals) {
        for (int i = 0; i < g.s0; i++)
            for (int k = 0; k < g.s1; k++) vals[(size_t)i * g.s1 + k] = cd(i == j ? v : 0.0, 0.0);
    };
    return p;
}

static Pattern col0_scaled(const Geo& g, double v) {
    return col_pattern(g, "col0s:" + dkey(v), [v](int j) { return j == 0 ? v : 0.0; });
}

// col_major_abt: A (m x n grid, untiled), B (1 x n, untiled, c rows); out m blocks
std::vector<CtP> sched_col_major_abt(Eval& ev, const std::vector<CtP>& A, int m, int n, const std::vector<CtP>& B,
                                     int c, double scale) {
    const Geo g = geo(ev, geo_rows(ev));
    if (c < 1 || c > g.s1) throw Error(-4, "col_major_abt: B rows must fit one block");
    if ((int)A.size() != m * n || (int)B.size() != n) throw Error(-4, "col_major_abt: grid mismatch");
    const bool par = !ev.auto_boot || std::min(grid_level(A), grid_level(B)) >= 4;
    const Pattern c0 = col0_scaled(g, scale);
    std::vector<G> terms(c);
    par_for(ev.c, c, par ? fork_width(ev.c, c) : 1, [&](int j) {
        const Pattern rowj = row_select(g, j, 1.0);
        G picked(n);
        for (int q = 0; q < n; q++) picked[q] = ev.mult_p(B[q], rowj);
        for (int q = 0; q < n; q++) picked[q] = ev.ladder(picked[q], g.s1, ilog2(g.s0));
        G prod((size_t)m * n);
        for (int p = 0; p < m; p++)
            for (int q = 0; q < n; q++) prod[(size_t)p * n + q] = ev.mult(A[(size_t)p * n + q], picked[q]);
        terms[j].resize(m);
        for (int p = 0; p < m; p++) {
            CtP blk = prod[(size_t)p * n];
            for (int q = 1; q < n; q++) blk = ev.add(blk, prod[(size_t)p * n + q]);
            blk = ev.ladder(blk, 1, ilog2(g.s1));
            blk = ev.mult_p(blk, c0);
            terms[j][p] = ev.rrot(blk, j);
        }
    });
    G acc = terms[0];
    for (int j = 1; j < c; j++)
        for (int p = 0; p < m; p++) acc[p] = ev.add(acc[p], terms[j][p]);
    return acc;
}

// row_major_atb: A (m x 1 grid, untiled, c columns), B (m x n); out n blocks
std::vector<CtP> sched_row_major_atb(Eval& ev, const std::vector<CtP>& A, int m, const std::vector<CtP>& B, int n,
                                     int c, double scale) {
    const Geo g = geo(ev, geo_rows(ev));
    if (c < 1 || c > g.s0) throw Error(-4, "row_major_atb: A columns must fit one block");
    if ((int)A.size() != m || (int)B.size() != m * n) throw Error(-4, "row_major_atb: grid mismatch");
    const bool par = !ev.auto_boot || std::min(grid_level(A), grid_level(B)) >= 4;
    const Pattern c0 = col0(g);
    std::vector<G> terms(c);
    par_for(ev.c, c, par ? fork_width(ev.c, c) : 1, [&](int j) {
        G picked(m);
        for (int p = 0; p < m; p++) picked[p] = ev.lrot(A[p], j);
        for (int p = 0; p < m; p++) picked[p] = ev.mult_p(picked[p], c0);
        for (int p = 0; p < m; p++) picked[p] = ev.ladder(picked[p], -1, ilog2(g.s1));
        G prod((size_t)m * n);
        for (int p = 0; p < m; p++)
            for (int q = 0; q < n; q++) prod[(size_t)p * n + q] = ev.mult(picked[p], B[(size_t)p * n + q]);
        G sums = row_sums(ev, prod, m, n, g, Reducer());
        const Pattern rowj = row_select(g, j, scale);
        terms[j].resize(n);
        for (int q = 0; q < n; q++) terms[j][q] = ev.mult_p(sums[q], rowj);
    });
    G acc = terms[0];
    for (int j = 1; j < c; j++)
        for (int q = 0; q < n; q++) acc[q] = ev.add(acc[q], terms[j][q]);
    return acc;
}

// ---- approximate softmax (approx.py:195-344), encrypted carrier ------------

namespace {

const double EXP_POLY[13] = {0.9999999999999948,     0.9999999999996788,    0.5000000000004744,
                             0.1666666666766445,     0.04166666666019774,   0.00833333324592319,
                             0.0013888889188354027,  0.00019841302319140728, 2.4801530417934142e-05,
                             2.7551504280360845e-06, 2.7561173628426655e-07, 2.5547752396936175e-08,
                             2.0934824859870782e-09};
const double COMP_F[4] = {35.0 / 16, -35.0 / 16, 21.0 / 16, -5.0 / 16};
const double COMP_G[4] = {4589.0 / 1024, -16577.0 / 1024, 25614.0 / 1024, -12860.0 / 1024};

struct SM {
    Eval& ev;
    Geo g;
    int classes, period;

    // the products run as batches over the blocks (one key-switch /
    // rescale pipeline per op); refreshes keep the block-by-block order
    G scale(const G& x, double t) { return ev.mult_c_batch(x, t); }
    G addc(const G& x, double s) { return ev.add_c_batch(x, s); }
    G rsubc(const G& x, double s) { return ev.add_c_batch(x, s, false, true); }   // s - x
    G add(const G& x, const G& y) { return ev.add_batch(x, y); }
    G sub(const G& x, const G& y) { return ev.add_batch(x, y, true); }
    G subp(const G& x, const Pattern& p) { return ev.add_p_batch(x, p, true, false); }
    G mul(const G& x, const G& y) { return ev.mult_batch(x, y); }
    G mulp(const G& x, const Pattern& p) { return ev.mult_p_batch(x, std::vector<const Pattern*>(x.size(), &p)); }
    G lrot(const G& x, int r) { return ev.lrot_batch(x, r); }
    G rrot(const G& x, int r) {
        G o(x.size());
        for (size_t i = 0; i < x.size(); i++) o[i] = ev.rrot(x[i], r);
        return o;
    }

    G odd7(const G& x, const double* a) {
        G y = mul(x, x);
        G acc = scale(y, a[3]);
        acc = addc(acc, a[2]);
        G t = mul(acc, y);
        acc = addc(t, a[1]);
        t = mul(acc, y);
        acc = addc(t, a[0]);
        return mul(acc, x);
    }
    G comp(const G& x, const G& y) {
        G d = sub(x, y);
        G u = odd7(d, COMP_G);
        u = odd7(u, COMP_G);
        u = odd7(u, COMP_F);
        G v = addc(u, 1.0);
        return scale(v, 0.5);
    }
    G amax(const G& M, const SoftmaxCfg& cfg, int max_range) {
        const double two_r = 2.0 * max_range;
        G work = scale(M, 1.0 / two_r);
        if (classes < period) {
            const int c = classes, cp = period;
            work = subp(work, col_pattern(g, "padhalf:" + std::to_string(c) + ":" + std::to_string(cp),
                                          [c, cp](int j) { return (j % cp) >= c ? 0.5 : 0.0; }));
        }
        G best = work;
        for (int t = 0; t < ilog2(period); t++) {
            G rival = lrot(best, 1 << t);
            G w = comp(best, rival);
            G x2 = rsubc(w, 1.0);
            // best * w and rival * (1 - w) are independent: one batch, the
            // first product's blocks before the second's (the reference order)
            G xy = mul(cat(best, rival), cat(w, x2));
            best = add(G(xy.begin(), xy.begin() + best.size()), G(xy.begin() + best.size(), xy.end()));
        }
        best = mulp(best, col0(g));
        best = ev.ladder(best, -1, ilog2(g.s1));
        return scale(best, two_r);
    }
    G domain_extend(G M, const SoftmaxCfg& cfg) {
        const double delta = 4.0 / (27.0 * std::pow(cfg.base_range, 2.0));
        for (int i = cfg.extension_steps - 1; i >= 0; i--) {
            const double di = delta * std::pow(cfg.extension_base, (double)(-2 * i));
            // the square and the scaling are independent: two branches on
            // side streams, issued in the reference's order (nonces unchanged)
            G sq, sc;
            par_for(ev.c, 2, 2, [&](int i) {
                if (i == 0) sq = mul(M, M);
                else sc = scale(M, di);
            });
            G pr = mul(sq, sc);
            M = sub(M, pr);
        }
        return M;
    }
    G dep_comp(const G& M, const SoftmaxCfg& cfg) {
        const double L2 = std::pow(cfg.extension_base, 2.0);
        const double Ln = std::pow(L2, (double)cfg.extension_steps);
        const double K = L2 * (Ln - 1.0) / (Ln * (L2 - 1.0));
        const double R = cfg.base_range;
        const double c3 = 1.0 * (4.0 / 27.0) * K / std::pow(R, 2.0);
        const double c5 = 1.0 * (4.0 / 27.0) * K / std::pow(R, 4.0);
        G sq = mul(M, M);
        G cube = mul(sq, M);
        G fifth, t3;
        par_for(ev.c, 2, 2, [&](int i) {   // independent: side streams, reference issue order
            if (i == 0) fifth = mul(cube, sq);
            else t3 = scale(cube, c3);
        });
        G t5 = scale(fifth, c5);
        G d = sub(t3, t5);
        return add(M, d);
    }
    G exp(const G& M, const SoftmaxCfg& cfg) {
        const int B = cfg.exp_range;
        G z = scale(M, 1.0 / B);
        G acc = scale(z, EXP_POLY[12]);
        acc = addc(acc, EXP_POLY[11]);
        for (int k = 10; k >= 0; k--) {
            G t = mul(acc, z);
            acc = addc(t, EXP_POLY[k]);
        }
        for (int i = 0; i < ilog2(B); i++) acc = mul(acc, acc);
        return acc;
    }
    G inv(const G& M, const SoftmaxCfg& cfg) {
        G y = scale(M, 1.0 / cfg.inv_range);
        G a = rsubc(y, 2.0);
        G b = rsubc(y, 1.0);
        // Goldschmidt: b_{i+1} = b_i^2, a_{i+1} = a_i (b_{i+1} + 1).  The
        // update of a in iteration i and the squaring of iteration i + 1 both
        // need only b_{i+1}: one batch (a's products first, as in the
        // reference's op order), so the chain is iters + 1 products long
        const size_t n = M.size();
        if (cfg.inv_iters < 1) return scale(a, 1.0 / cfg.inv_range);
        b = mul(b, b);
        G t = addc(b, 1.0);
        for (int i = 0; i < cfg.inv_iters; i++) {
            if (i + 1 < cfg.inv_iters) {
                G r = mul(cat(a, b), cat(t, b));
                a = G(r.begin(), r.begin() + n);
                b = G(r.begin() + n, r.end());
                t = addc(b, 1.0);
            } else {
                a = mul(a, t);
            }
        }
        return scale(a, 1.0 / cfg.inv_range);
    }
    static G cat(const G& x, const G& y) {
        G o = x;
        o.insert(o.end(), y.begin(), y.end());
        return o;
    }
};

}  // namespace

static std::vector<CtP> softmax_serial(Eval& ev, const std::vector<CtP>& M, int classes, int period,
                                       const SoftmaxCfg& cfg);

std::vector<CtP> sched_softmax(Eval& ev, const std::vector<CtP>& M, int classes, int period, const SoftmaxCfg& cfg) {
    const Geo g = geo(ev, geo_rows(ev));
    if (period < classes || period > g.s1 || (period & (period - 1))) throw Error(-4, "softmax: bad period");
    if (cfg.exp_range < 1 || (cfg.exp_range & (cfg.exp_range - 1))) throw Error(-4, "exp_range must be a power of two");
    const int m = (int)M.size();
    Ctx& C = ev.c;
    if (C.shard_total > 0 && !ev.plan.on) {
        // block-row shard of a larger batch: lockstep over the local blocks with
        // the whole batch's nonce layout, so every refresh (and the context
        // nonce afterwards) equals the single-context run of all block rows
        if (C.shard_first + m > C.shard_total) throw Error(-4, "softmax: shard exceeds the batch");
        Eval sev(C, ev.auto_boot);
        {
            std::lock_guard<std::mutex> lk(C.mu);
            sev.plan.base = C.nonce;
        }
        sev.plan.on = true;
        sev.plan.m = C.shard_total;
        sev.plan.p = C.shard_first;
        sev.plan.mloc = m;
        std::vector<CtP> out = softmax_serial(sev, M, classes, period, cfg);
        std::lock_guard<std::mutex> lk(C.mu);
        C.nonce = sev.plan.base + (u64)C.shard_total * sev.plan.events;
        return out;
    }
    bool uniform = m > 1 && !ev.plan.on;
    for (auto& b : M) uniform = uniform && b->level == M[0]->level;
    // lockstep (default): the blocks advance op by op, each op one batch --
    // the reference's own order, so refreshes draw the sequential nonces
    if (!uniform || ev.c.fork_cap <= 1 || ev.c.lockstep) return softmax_serial(ev, M, classes, period, cfg);
    // Block rows are independent: one branch per block row, each with the
    // nonce plan that reproduces the sequential (block-interleaved) order.
    u64 base;
    {
        std::lock_guard<std::mutex> lk(ev.c.mu);
        base = ev.c.nonce;
    }
    std::vector<CtP> out(m);
    u64 events = 0;
    par_for(ev.c, m, m, [&](int p) {
        Eval bev(ev.c, ev.auto_boot);
        bev.plan.on = true;
        bev.plan.base = base;
        bev.plan.m = m;
        bev.plan.p = p;
        out[p] = softmax_serial(bev, std::vector<CtP>{M[p]}, classes, period, cfg)[0];
        events = bev.plan.events;
    });
    std::lock_guard<std::mutex> lk(ev.c.mu);
    ev.c.nonce = base + (u64)m * events;
    return out;
}

static std::vector<CtP> softmax_serial(Eval& ev, const std::vector<CtP>& M, int classes, int period,
                                       const SoftmaxCfg& cfg) {
    const Geo g = geo(ev, geo_rows(ev));
    SM sm{ev, g, classes, period};
    const double full = cfg.base_range * std::pow(cfg.extension_base, (double)cfg.extension_steps);
    const int max_range = (int)std::ceil(full / 2);
    G best = sm.amax(M, cfg, max_range);
    const int c = classes;
    const Pattern keep = col_pattern(g, "keep:" + std::to_string(c), [c](int j) { return j < c ? 1.0 : 0.0; });
    G d = sm.sub(M, best);
    G norm = sm.mulp(d, keep);
    norm = sm.domain_extend(norm, cfg);
    if (cfg.precise) norm = sm.dep_comp(norm, cfg);
    G e = sm.exp(norm, cfg);
    G expd = sm.mulp(e, keep);
    // col_sums of every block (encoding.py:335-360) in lockstep
    G total = expd;
    total = ev.ladder(total, 1, ilog2(g.s1));
    total = sm.mulp(total, col0(g));
    total = ev.ladder(total, -1, ilog2(g.s1));
    G recip = sm.inv(total, cfg);
    G out = sm.mul(expd, recip);
    const int reps = g.s1 / period;
    return ev.ladder(out, -(int64_t)period, ilog2(reps));
}

std::vector<CtP> sched_approx(Eval& ev, int fn, const std::vector<CtP>& X, const std::vector<CtP>& Y, int classes,
                              int period, const SoftmaxCfg& cfg) {
    const Geo g = geo(ev, geo_rows(ev));
    SM sm{ev, g, classes, period};
    switch (fn) {
        case APPROX_COMP:
            if (Y.size() != X.size()) throw Error(-4, "a_comp: operand grids differ");
            return sm.comp(X, Y);
        case APPROX_MAX: {
            if (period < classes || period > g.s1 || (period & (period - 1))) throw Error(-4, "a_max: bad period");
            const double full = cfg.base_range * std::pow(cfg.extension_base, (double)cfg.extension_steps);
            return sm.amax(X, cfg, (int)std::ceil(full / 2));
        }
        case APPROX_DOMAIN_EXTEND: return sm.domain_extend(X, cfg);
        case APPROX_DEP_COMP: return sm.dep_comp(X, cfg);
        case APPROX_EXP:
            if (cfg.exp_range < 1 || (cfg.exp_range & (cfg.exp_range - 1)))
                throw Error(-4, "exp_range must be a power of two");
            return sm.exp(X, cfg);
        case APPROX_INV: return sm.inv(X, cfg);
        default: throw Error(-1, "unknown approximation");
    }
}

}  // namespace hc
