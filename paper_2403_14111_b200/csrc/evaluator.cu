// Exact RNS-CKKS ciphertext operations on the device, and the
// reference-semantics policy layer (Eval) shared by the per-op C-ABI and the
// native schedules.
//
// Hybrid key switching (K5):
//   INTT(d) -> ModUp fast base conversion per digit -> NTT of new limbs ->
//   key inner product (128-bit lazy accumulation, one Barrett reduction) ->
//   INTT of the P limbs -> ModDown conversion -> NTT -> (acc - conv) * P^-1
//   with the automorphism's c0 / the tensor's (d0, d1) added in the same pass.
#include <cstdlib>
#include <cmath>
#include <map>

#include "evaluator.h"
#include "kernels.cuh"

namespace hc {

typedef unsigned __int128 u128;

static u64 mulm(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 shoup_of(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static u64 from_i64_h(int64_t v, u64 q) {
    if (v >= 0) return (u64)v % q;
    u64 m = (u64)(-(v + 1)) % q;
    return q - 1 - m;
}

static void check_same(const Ct& a, const Ct& b) {
    if (a.level != b.level) throw Error(-4, "level mismatch in low-level op");
}

// (cr + ci I, cr - ci I) per limb with Shoup companions
static void const_pairs(const Ctx& c, int64_t cr, int64_t ci, int nl, ConstTab& t) {
    for (int i = 0; i < nl; i++) {
        const u64 q = c.pr[i].q;
        const u64 r = from_i64_h(cr, q), im = mulm(from_i64_h(ci, q), c.pr[i].I, q);
        const u64 lo = (r + im) % q, hi = (r + q - im) % q;
        t.v[4 * i] = lo;
        t.v[4 * i + 1] = shoup_of(lo, q);
        t.v[4 * i + 2] = hi;
        t.v[4 * i + 3] = shoup_of(hi, q);
    }
}

CtP ev_add(Ctx& c, const Ct& a, const Ct& b, bool sub) {
    check_same(a, b);
    CtP o = new_ct(c, a.level);
    k_elementwise(c, sub ? EWP_SUB : EWP_ADD, o->d, a.d, b.d, nullptr, a.level + 1, 2, 2);
    return o;
}

CtP ev_neg(Ctx& c, const Ct& a) {
    CtP o = new_ct(c, a.level);
    k_elementwise(c, EWP_NEG, o->d, a.d, nullptr, nullptr, a.level + 1, 2, 0);
    return o;
}

CtP ev_add_pt(Ctx& c, const Ct& a, const Pt& p, bool sub, bool pt_minus_ct) {
    if (p.level < a.level) throw Error(-4, "plaintext level too low");
    CtP o = new_ct(c, a.level);
    int op = pt_minus_ct ? EWP_PT_RSUB : (sub ? EWP_PT_SUB : EWP_PT_ADD);
    k_elementwise(c, op, o->d, a.d, p.d, nullptr, a.level + 1, 2, 1);
    return o;
}

CtP ev_add_const(Ctx& c, const Ct& a, double re, double im, bool negate_ct) {
    const double s = c.scale[a.level];
    ConstTab t;
    const_pairs(c, std::llrint(re * s), std::llrint(im * s), a.level + 1, t);
    CtP o = new_ct(c, a.level);
    k_elementwise(c, negate_ct ? EWP_CONST_RADD : EWP_CONST_ADD, o->d, a.d, nullptr, &t, a.level + 1, 2, 0);
    return o;
}

// rescale [npoly][level+1][N] at `a` into [npoly][level][N] at `out`
static void rescale_raw(Ctx& c, const u64* a, int level, int npoly, u64* out) {
    if (rescale_fused(c, a, level, npoly, out)) return;
    const int N = c.N;
    u64* X = c.alloc((size_t)npoly * N);
    JobList j;
    j.n = npoly;
    for (int s = 0; s < npoly; s++) {
        j.prime[s] = level;
        j.ptr[s] = X + (size_t)s * N;
        j.src[s] = a + ((size_t)s * (level + 1) + level) * N;
    }
    ntt_inverse(c, j);
    u64* Y = c.alloc((size_t)npoly * level * N);
    k_rescale_bcast(c, Y, X, level, npoly);
    JobList f;
    f.n = 0;
    for (int s = 0; s < npoly; s++)
        for (int i = 0; i < level; i++) {
            f.prime[f.n] = i;
            f.ptr[f.n] = Y + ((size_t)s * level + i) * N;
            f.src[f.n] = nullptr;
            f.n++;
        }
    ntt_forward(c, f);
    k_rescale_combine(c, out, a, Y, level, npoly);
    c.free(X);
    c.free(Y);
}

// out[b] = rescale of the 2-poly input T + 2 * poly * b (level -> level - 1)
static void rescale_many(Ctx& c, const u64* T, size_t poly, int level, std::vector<CtP>& out) {
    const size_t B = out.size();
    std::vector<const u64*> a(B);
    std::vector<u64*> o(B);
    for (size_t b = 0; b < B; b++) {
        out[b] = new_ct(c, level - 1);
        a[b] = T + 2 * poly * b;
        o[b] = out[b]->d;
    }
    if (rescale_fused_batch(c, (int)B, a.data(), level, 2, o.data())) return;
    for (size_t b = 0; b < B; b++) rescale_raw(c, a[b], level, 2, o[b]);
}

CtP ev_rescale(Ctx& c, const Ct& a) {
    if (a.level < 1) throw Error(-3, "rescale at level 0");
    CtP o = new_ct(c, a.level - 1);
    rescale_raw(c, a.d, a.level, 2, o->d);
    return o;
}

static CtP mul_int_rescale(Ctx& c, const u64* a, int level, int64_t cr, int64_t ci) {
    ConstTab t;
    const_pairs(c, cr, ci, level + 1, t);
    u64* T = c.alloc((size_t)2 * (level + 1) * c.N);
    k_elementwise(c, EWP_CONST_MUL, T, a, nullptr, &t, level + 1, 2, 0);
    CtP o = new_ct(c, level - 1);
    rescale_raw(c, T, level, 2, o->d);
    c.free(T);
    return o;
}

CtP ev_mul_const(Ctx& c, const Ct& a, double re, double im) {
    if (a.level < 1) throw Error(-3, "multiply at level 0");
    const double s = c.scale[a.level];
    return mul_int_rescale(c, a.d, a.level, std::llrint(re * s), std::llrint(im * s));
}

CtP ev_mul_pt(Ctx& c, const Ct& a, const Pt& p) {
    if (a.level < 1) throw Error(-3, "multiply at level 0");
    if (p.level != a.level) throw Error(-4, "plaintext level must equal ciphertext level");
    u64* T = c.alloc((size_t)2 * (a.level + 1) * c.N);
    k_elementwise(c, EWP_PT_MUL, T, a.d, p.d, nullptr, a.level + 1, 2, 1);
    CtP o = new_ct(c, a.level - 1);
    rescale_raw(c, T, a.level, 2, o->d);
    c.free(T);
    return o;
}

CtP ev_mul_i(Ctx& c, const Ct& a) {
    ConstTab t;
    const_pairs(c, 0, 1, a.level + 1, t);
    CtP o = new_ct(c, a.level);
    k_elementwise(c, EWP_CONST_MUL, o->d, a.d, nullptr, &t, a.level + 1, 2, 0);
    return o;
}

CtP ev_drop(Ctx& c, const Ct& a, int to) {
    if (to > a.level) throw Error(-4, "drop to a higher level");
    CtP o = new_ct(c, to);
    for (int s = 0; s < 2; s++)
        HC_CUDA(cudaMemcpyAsync(o->poly(s), a.poly(s), sizeof(u64) * (size_t)(to + 1) * c.N,
                                cudaMemcpyDeviceToDevice, c.stream));
    return o;
}

static void rescale_many(Ctx& c, const u64* T, size_t poly, int level, std::vector<CtP>& out);

// Level adjustment of several ciphertexts from one level to `to`: the first
// to + 2 limbs of each poly times llrint(Δ_{to+1}²/Δ_from) (read in place, one
// launch), then one batched rescale
std::vector<CtP> ev_level_adjust_batch(Ctx& c, const std::vector<const Ct*>& xs, int to) {
    std::vector<CtP> out(xs.size());
    if (xs.empty()) return out;
    const int from = xs[0]->level;
    for (auto* x : xs)
        if (x->level != from || to >= from) throw Error(-4, "level adjust needs one source level above the target");
    const int nl2 = to + 2;
    const double s1 = c.scale[to + 1];
    const int64_t cst = std::llrint(s1 * (s1 / c.scale[from]));
    ConstTab t;
    const_pairs(c, cst, 0, nl2, t);
    const size_t poly = (size_t)nl2 * c.N;
    Scratch sc(c);
    u64* T = sc.take(2 * poly * xs.size());
    std::vector<u64*> o(2 * xs.size());
    std::vector<const u64*> a(2 * xs.size());
    for (size_t b = 0; b < xs.size(); b++)
        for (int s = 0; s < 2; s++) {
            o[2 * b + s] = T + (2 * b + s) * poly;
            a[2 * b + s] = xs[b]->poly(s);
        }
    k_elementwise_batch(c, EWP_CONST_MUL, (int)o.size(), o.data(), a.data(), nullptr, &t, nl2, 1, 0);
    rescale_many(c, T, poly, to + 1, out);
    return out;
}

CtP ev_level_adjust(Ctx& c, const Ct& a, int to) {
    if (to >= a.level) throw Error(-4, "level adjust needs a lower target");
    return ev_level_adjust_batch(c, {&a}, to)[0];
}

// ---------------------------------------------------------------------------
// hybrid key switching
// ---------------------------------------------------------------------------

static inline int tprime(const Ctx& c, int level, int t) { return t <= level ? t : c.L + 1 + (t - level - 1); }

// ModUp of d ([level+1][N], NTT) -> UP [beta][nt][N] (NTT form, allocated here)
static u64* ks_modup(Ctx& c, const u64* d, int level) {
    const int N = c.N, nl = level + 1, K = c.K, nt = nl + K;
    const int beta = (nl + c.alpha - 1) / c.alpha;
    u64* X = c.alloc((size_t)nl * N);
    ntt_limbs(c, X, 0, nl, true, d);
    u64* UP = c.alloc((size_t)beta * nt * N);
    k_modup(c, UP, X, d, level, beta);
    {
        JobList j;
        j.n = 0;
        for (int dj = 0; dj < beta; dj++) {
            const int lo = dj * c.alpha, hi = std::min(lo + c.alpha, nl);
            for (int t = 0; t < nt; t++) {
                if (t >= lo && t < hi) continue;
                if (j.n == MAXJ) { ntt_forward(c, j); j.n = 0; }
                j.prime[j.n] = tprime(c, level, t);
                j.ptr[j.n] = UP + ((size_t)dj * nt + t) * N;
                j.src[j.n] = nullptr;
                j.n++;
            }
        }
        ntt_forward(c, j);
    }
    c.free(X);
    return UP;
}

// ModDown of the key products ACC [2][nt][N] (its dropped limbs are
// overwritten), + addend; merged: ModDown + rescale by q_l P, out at level - 1
static void ks_tail_acc(Ctx& c, u64* ACC, int level, u64* out, const u64* addend, int add_npoly, bool merged = false) {
    const int N = c.N, nl = level + 1, K = c.K, nt = nl + K;
    const int nout = merged ? nl - 1 : nl;
    {
        JobList j;
        j.n = 0;
        for (int s = 0; s < 2; s++)
            for (int t = merged ? nl - 1 : nl; t < nt; t++) {
                j.prime[j.n] = tprime(c, level, t);
                j.ptr[j.n] = ACC + ((size_t)s * nt + t) * N;
                j.src[j.n] = nullptr;
                j.n++;
            }
        ntt_inverse(c, j);
    }
    u64* W = c.alloc((size_t)2 * nout * N);
    k_moddown_conv(c, W, ACC, level, merged);
    ntt_limbs(c, W, 0, nout, false);
    ntt_limbs(c, W + (size_t)nout * N, 0, nout, false);
    k_moddown_combine(c, out, ACC, W, addend, add_npoly, level, merged);
    c.free(W);
    c.counts[OP_KS]++;
}

// Relinearisation + rescale of B tensors D + 3 * poly * b = (d0, d1, d2) at
// `level` in one pass: [P]_q (d0, d1) joins the key products of
// ModUp(d2) in the extended basis and one ModDown divides by q_l P.
static void rescale_many(Ctx& c, const u64* T, size_t poly, int level, std::vector<CtP>& out);
static void relin_rescale_many(Ctx& c, const u64* D, size_t poly, int level, std::vector<CtP>& out) {
    const size_t B = out.size();
    if (level < 1) throw Error(-3, "multiply at level 0");
    const Key& key = get_key(c, 0);
    if (level > c.app_L) {
        // bootstrapping levels keep ModDown and the exact centred rescale apart:
        // EvalMod's precision is bound by the rescale rounding, which the merged
        // conversion makes ~2.3x larger (a sum of K + 1 centred terms)
        Scratch sc(c);
        u64* T = sc.take(2 * poly * B);
        std::vector<KsIn> in(B);
        for (size_t b = 0; b < B; b++) {
            const u64* Db = D + 3 * poly * b;
            in[b] = KsIn{Db + 2 * poly, T + 2 * poly * b, Db, nullptr, key.d};
        }
        if (keyswitch_fused_batch(c, (int)B, in.data(), 0, level, 2, 0)) c.counts[OP_KS] += (int64_t)B;
        else
            for (size_t b = 0; b < B; b++) keyswitch(c, in[b].d, level, key, in[b].out, in[b].add, 2);
        rescale_many(c, T, poly, level, out);
        return;
    }
    std::vector<const u64*> ds(B);
    std::vector<u64*> o(B);
    for (size_t b = 0; b < B; b++) {
        out[b] = new_ct(c, level - 1);
        ds[b] = D + 3 * poly * b;
        o[b] = out[b]->d;
    }
    if (keyswitch_relin_rescale(c, (int)B, ds.data(), o.data(), level, key.d)) {
        c.counts[OP_KS] += (int64_t)B;
        return;
    }
    const int nl = level + 1, nt = nl + c.K, beta = (nl + c.alpha - 1) / c.alpha;
    for (size_t b = 0; b < B; b++) {
        u64* UP = ks_modup(c, ds[b] + 2 * poly, level);
        u64* ACC = c.alloc((size_t)2 * nt * c.N);
        k_keyprod(c, ACC, UP, key.d, level, beta);
        k_fold_p(c, ACC, ds[b], level);
        ks_tail_acc(c, ACC, level, o[b], nullptr, 0, true);
        c.free(ACC);
        c.free(UP);
    }
}

// key product of the ModUp digits UP with `key`, ModDown, + addend
static void ks_tail(Ctx& c, const u64* UP, int level, const Key& key, u64* out, const u64* addend, int add_npoly) {
    const int nl = level + 1, nt = nl + c.K;
    const int beta = (nl + c.alpha - 1) / c.alpha;
    u64* ACC = c.alloc((size_t)2 * nt * c.N);
    k_keyprod(c, ACC, UP, key.d, level, beta);
    ks_tail_acc(c, ACC, level, out, addend, add_npoly);
    c.free(ACC);
}

// d: [level+1][N] (NTT).  out [2][level+1][N] = KS(d) + addend (first add_npoly polys)
void keyswitch(Ctx& c, const u64* d, int level, const Key& key, u64* out, const u64* addend, int add_npoly) {
    u64* UP = ks_modup(c, d, level);
    ks_tail(c, UP, level, key, out, addend, add_npoly);
    c.free(UP);
}

CtP ev_automorph(Ctx& c, const Ct& a, u64 g) {
    const Key& key = get_key(c, (int)g);
    const int nl = a.level + 1;
    {
        CtP o = new_ct(c, a.level);
        if (keyswitch_fused(c, a.poly(1), g, a.level, key, o->d, a.poly(0), 1, g)) {
            c.counts[OP_KS]++;
            return o;
        }
    }
    u64* S = c.alloc((size_t)2 * nl * c.N);
    k_automorph(c, S, a.d, 2 * nl, g);
    CtP o = new_ct(c, a.level);
    keyswitch(c, S + (size_t)nl * c.N, a.level, key, o->d, S, 1);
    c.free(S);
    return o;
}

bool ev_automorph_add(Ctx& c, const Ct& a, u64 g, CtP& out) {
    if (c.logN < 14) return false;
    const Key& key = get_key(c, (int)g);
    CtP o = new_ct(c, a.level);
    if (!keyswitch_fused(c, a.poly(1), g, a.level, key, o->d, a.poly(0), 1, g, a.d)) return false;
    c.counts[OP_KS]++;
    out = o;
    return true;
}

// Batched rotations / conjugations (all inputs at one level): one fused
// key-switch pipeline for the whole batch.  add_self: out_b = sigma(a_b) + a_b.
std::vector<CtP> ev_automorph_batch(Ctx& c, const std::vector<const Ct*>& a, u64 g, bool add_self) {
    const size_t B = a.size();
    std::vector<CtP> out(B);
    if (B == 0) return out;
    bool uniform = c.logN >= 14;
    for (auto* x : a) uniform &= x->level == a[0]->level;
    if (uniform && B > 1) {
        const Key& key = get_key(c, (int)g);
        std::vector<KsIn> in(B);
        for (size_t b = 0; b < B; b++) {
            out[b] = new_ct(c, a[b]->level);
            in[b] = KsIn{a[b]->poly(1), out[b]->d, a[b]->poly(0), add_self ? a[b]->d : nullptr, key.d};
        }
        if (keyswitch_fused_batch(c, (int)B, in.data(), g, a[0]->level, 1, g)) {
            c.counts[OP_KS] += (int64_t)B;
            return out;
        }
    }
    for (size_t b = 0; b < B; b++) {
        if (!add_self) { out[b] = ev_automorph(c, *a[b], g); continue; }
        if (ev_automorph_add(c, *a[b], g, out[b])) continue;
        CtP r = ev_automorph(c, *a[b], g);
        out[b] = ev_add(c, *a[b], *r, false);
    }
    return out;
}

// Batched ct x ct products (pairs at one level): tensor per pair, one fused
// relinearisation pipeline, rescale per pair.
std::vector<CtP> ev_mult_batch(Ctx& c, const std::vector<std::pair<const Ct*, const Ct*>>& ab) {
    const size_t B = ab.size();
    std::vector<CtP> out(B);
    if (B == 0) return out;
    bool uniform = c.logN >= 14;
    for (auto& pr : ab) {
        check_same(*pr.first, *pr.second);
        uniform &= pr.first->level == ab[0].first->level;
    }
    if (!uniform || B == 1) {
        for (size_t b = 0; b < B; b++) out[b] = ev_mult(c, *ab[b].first, *ab[b].second);
        return out;
    }
    const int level = ab[0].first->level;
    if (level < 1) throw Error(-3, "multiply at level 0");
    const int nl = level + 1;
    const size_t poly = (size_t)nl * c.N;
    Scratch sc(c);
    u64* D = sc.take(3 * poly * B);
    std::vector<u64*> dd(B);
    std::vector<const u64*> aa(B), bb(B);
    for (size_t b = 0; b < B; b++) {
        dd[b] = D + 3 * poly * b;
        aa[b] = ab[b].first->d;
        bb[b] = ab[b].second->d;
    }
    k_tensor_batch(c, (int)B, dd.data(), aa.data(), bb.data(), nl);
    relin_rescale_many(c, D, poly, level, out);
    return out;
}

// Hoisted rotations: rotation r of input i shares the ModUp
// of c1(i) with every other rotation of it; the digits are permuted by each
// Galois element inside the key product.  All inputs at one level.
// out[i][r] = sigma_{g_r}(x_i) with the hoisted key switch.
std::vector<std::vector<CtP>> ev_rot_hoisted(Ctx& c, const std::vector<const Ct*>& xs, const std::vector<u64>& gals) {
    const size_t nx = xs.size(), ng = gals.size();
    std::vector<std::vector<CtP>> out(nx, std::vector<CtP>(ng));
    if (nx == 0 || ng == 0) return out;
    const int level = xs[0]->level;
    for (auto* x : xs)
        if (x->level != level) throw Error(-4, "hoisted rotation: inputs at different levels");
    std::vector<const Key*> keys(ng);
    for (size_t r = 0; r < ng; r++) keys[r] = &get_key(c, (int)gals[r]);
    for (size_t i = 0; i < nx; i++)
        for (size_t r = 0; r < ng; r++) out[i][r] = new_ct(c, level);
    if (c.logN >= 14) {
        std::vector<const u64*> c0s(nx), c1s(nx);
        for (size_t i = 0; i < nx; i++) { c0s[i] = xs[i]->poly(0); c1s[i] = xs[i]->poly(1); }
        std::vector<KsHoist> e;
        for (size_t i = 0; i < nx; i++)
            for (size_t r = 0; r < ng; r++) e.push_back(KsHoist{(int)i, gals[r], keys[r]->d, out[i][r]->d});
        if (!keyswitch_hoisted(c, c0s.data(), c1s.data(), level, (int)e.size(), e.data()))
            throw Error(-2, "hoisted rotation");
        c.counts[OP_KS] += (int64_t)e.size();
        return out;
    }
    // small rings: the unfused pipeline, digits permuted by an explicit automorphism
    const int nl = level + 1, nt = nl + c.K, beta = (nl + c.alpha - 1) / c.alpha;
    for (size_t i = 0; i < nx; i++) {
        u64* UP = ks_modup(c, xs[i]->poly(1), level);
        u64* UPg = c.alloc((size_t)beta * nt * c.N);
        u64* S0 = c.alloc((size_t)nl * c.N);
        for (size_t r = 0; r < ng; r++) {
            k_automorph(c, UPg, UP, beta * nt, gals[r]);
            k_automorph(c, S0, xs[i]->poly(0), nl, gals[r]);
            ks_tail(c, UPg, level, *keys[r], out[i][r]->d, S0, 1);
        }
        c.free(S0);
        c.free(UPg);
        c.free(UP);
    }
    return out;
}

// Rotate-and-sum stage (radix ladders): out_i = x_i + sum_r
// sigma_{g_r}(x_i); one ModUp of c1(i), the rotations' key products summed in
// the extended basis, one ModDown.  All inputs at one level.
std::vector<CtP> ev_rotsum_batch(Ctx& c, const std::vector<const Ct*>& xs, const std::vector<u64>& gals) {
    const size_t nx = xs.size(), ng = gals.size();
    std::vector<CtP> out(nx);
    if (nx == 0) return out;
    const int level = xs[0]->level;
    for (auto* x : xs)
        if (x->level != level) throw Error(-4, "rotate-and-sum: inputs at different levels");
    std::vector<const u64*> keys(ng);
    for (size_t r = 0; r < ng; r++) keys[r] = get_key(c, (int)gals[r]).d;
    for (size_t i = 0; i < nx; i++) out[i] = new_ct(c, level);
    if (c.logN >= 14) {
        std::vector<const u64*> in(nx);
        std::vector<u64*> o(nx);
        for (size_t i = 0; i < nx; i++) { in[i] = xs[i]->d; o[i] = out[i]->d; }
        if (!keyswitch_rotsum(c, (int)nx, in.data(), o.data(), level, (int)ng, gals.data(), keys.data()))
            throw Error(-2, "rotate-and-sum stage");
        c.counts[OP_KS] += (int64_t)nx;
        return out;
    }
    // small rings: the unfused pipeline, digits permuted by an explicit automorphism
    const int nl = level + 1, nt = nl + c.K, beta = (nl + c.alpha - 1) / c.alpha;
    for (size_t i = 0; i < nx; i++) {
        u64* UP = ks_modup(c, xs[i]->poly(1), level);
        u64* UPg = c.alloc((size_t)beta * nt * c.N);
        u64* ACC = c.alloc((size_t)2 * nt * c.N);
        u64* S = c.alloc((size_t)2 * nl * c.N);    // addend: x + (sum_r sigma_r(c0), 0)
        u64* T = c.alloc((size_t)nl * c.N);
        HC_CUDA(cudaMemcpyAsync(S, xs[i]->d, sizeof(u64) * 2 * nl * c.N, cudaMemcpyDeviceToDevice, c.stream));
        for (size_t r = 0; r < ng; r++) {
            k_automorph(c, UPg, UP, beta * nt, gals[r]);
            k_keyprod(c, ACC, UPg, keys[r], level, beta, r > 0);
            k_automorph(c, T, xs[i]->poly(0), nl, gals[r]);
            k_elementwise(c, EWP_ADD, S, S, T, nullptr, nl, 1, 1);
        }
        ks_tail_acc(c, ACC, level, out[i]->d, S, 2);
        c.free(T);
        c.free(S);
        c.free(ACC);
        c.free(UPg);
        c.free(UP);
    }
    return out;
}

// Product sums with one relinearisation each:
// out_b = rescale(d0 + KS(d2)_0, d1 + KS(d2)_1), d = sum_q tensor(a_bq, b_bq).
// Every operand of every group at one level >= 1.
std::vector<CtP> ev_mult_sum_batch(Ctx& c, const std::vector<std::vector<std::pair<const Ct*, const Ct*>>>& groups) {
    const size_t B = groups.size();
    std::vector<CtP> out(B);
    if (B == 0) return out;
    const int level = groups[0][0].first->level;
    for (auto& gr : groups)
        for (auto& pr : gr)
            if (pr.first->level != level || pr.second->level != level) throw Error(-4, "product sum: level mismatch");
    if (level < 1) throw Error(-3, "multiply at level 0");
    const int nl = level + 1;
    const size_t poly = (size_t)nl * c.N;
    Scratch sc(c);
    u64* D = sc.take(3 * poly * B);
    for (size_t b = 0; b < B; b++) {
        u64* Db = D + 3 * poly * b;
        std::vector<const u64*> as, bs;
        for (auto& pr : groups[b]) { as.push_back(pr.first->d); bs.push_back(pr.second->d); }
        k_tensor_sum(c, Db, as.data(), bs.data(), (int)as.size(), nl);
    }
    relin_rescale_many(c, D, poly, level, out);
    return out;
}

CtP ev_mult(Ctx& c, const Ct& a, const Ct& b) {
    check_same(a, b);
    if (a.level < 1) throw Error(-3, "multiply at level 0");
    const int nl = a.level + 1;
    const size_t poly = (size_t)nl * c.N;
    Scratch sc(c);
    u64* D = sc.take(3 * poly);
    k_tensor(c, D, a.d, b.d, nl);
    std::vector<CtP> o(1);
    relin_rescale_many(c, D, poly, a.level, o);
    return o[0];
}

// ---------------------------------------------------------------------------
// Eval: the reference backend semantics (emulator.py:160-273) over CKKS
// ---------------------------------------------------------------------------

void Eval::rec(int k, int n) {
    std::lock_guard<std::mutex> g(c.mu);
    c.counts[k] += n;
}

double model_limbs(const Ctx& c, int kind, int variant, int level) {
    const double Lq = level + 1, d = (level + c.alpha) / c.alpha;
    switch (kind) {
        case OP_ADD: return variant == MV_CT ? 6 * Lq : (variant == MV_PT ? 5 * Lq : 4 * Lq);
        case OP_CMULT: return variant == MV_PT ? 5 * Lq - 2 : 4 * Lq - 2;
        case OP_MULT: return 4 * Lq + 2 * d * (Lq + c.K) + 2 * (Lq - 1);
        case OP_ROT:
        case OP_CONJ: return 4 * Lq + 2 * d * (Lq + c.K);
        case MODEL_MULI: return 4 * Lq;
        default: return 0;
    }
}

void Eval::model(int kind, int variant, int level, int n) {
    const double b = n * model_limbs(c, kind, variant, level) * 8.0 * c.N;
    std::lock_guard<std::mutex> g(c.mu);
    c.model_bytes += b;
}

u64 Eval::next_nonce() {
    std::lock_guard<std::mutex> g(c.mu);
    return c.nonce++;
}

CtP Eval::at(const CtP& a, int level) {
    if (a->level == level) return a;
    rec(OP_ADJUST);
    return ev_level_adjust(c, *a, level);
}

u64 Eval::boot_nonce(int j, int r) {
    if (plan.on && plan.mloc > 1) throw Error(-4, "single-operand refresh inside a multi-block nonce plan");
    rec(OP_BOOT);
    return plan.on ? plan.base + (u64)plan.m * plan.events + (u64)plan.p * r + j : next_nonce();
}

std::vector<u64> Eval::batch_nonces(const std::vector<int>& r) {
    std::vector<u64> out;
    const size_t n = r.size();
    const size_t ml = plan.on ? (size_t)std::max(plan.mloc, 1) : 1;
    if (n % ml) throw Error(-4, "sharded batch: items are not whole rounds over the shard's blocks");
    for (size_t s0 = 0; s0 < n; s0 += ml) {
        const int rs = r[s0];
        for (size_t i = s0; i < s0 + ml; i++) {
            if (r[i] != rs) throw Error(-4, "sharded batch: blocks of one op at different levels");
            for (int j = 0; j < rs; j++) {
                rec(OP_BOOT);
                out.push_back(plan.on ? plan.base + (u64)plan.m * plan.events + (u64)(plan.p + (int)(i - s0)) * rs + j
                                      : next_nonce());
            }
        }
        plan.events += rs;
    }
    return out;
}

// the reference's bootstrap (emulator.py:267-273): the refresh surrogate, or
// with c.boot_mode real CKKS bootstrapping (bootstrap.cu; the nonce is drawn
// either way, so both modes keep one nonce sequence)
static CtP do_refresh(Ctx& c, const CtP& a, u64 nonce) {
    return c.boot_mode ? ev_bootstrap(c, a) : refresh(c, *a, nonce);
}

CtP Eval::refresh_planned(const CtP& a, int j, int r) { return do_refresh(c, a, boot_nonce(j, r)); }

// refresh the given operands with their nonces, batched per level
static void refresh_many(Ctx& c, std::vector<CtP*>& slots, const std::vector<u64>& nonces) {
    if (c.boot_mode) {   // CKKS bootstrapping of all of them together (per level)
        std::map<int, std::vector<size_t>> lv;
        for (size_t u = 0; u < slots.size(); u++) lv[(*slots[u])->level].push_back(u);
        for (auto& kv : lv) {
            std::vector<CtP> in;
            for (size_t u : kv.second) in.push_back(*slots[u]);
            std::vector<CtP> out = ev_bootstrap_batch(c, in);
            for (size_t t = 0; t < kv.second.size(); t++) *slots[kv.second[t]] = out[t];
        }
        return;
    }
    std::map<int, std::vector<size_t>> by_level;
    for (size_t u = 0; u < slots.size(); u++) by_level[(*slots[u])->level].push_back(u);
    for (auto& kv : by_level) {
        std::vector<const Ct*> a;
        std::vector<u64> n;
        for (size_t u : kv.second) {
            a.push_back(slots[u]->get());
            n.push_back(nonces[u]);
        }
        std::vector<CtP> r = refresh_batch(c, a, n);
        for (size_t t = 0; t < kv.second.size(); t++) *slots[kv.second[t]] = r[t];
    }
}

void Eval::ready_batch(std::vector<CtP>& xs) {
    std::vector<CtP*> slots;
    std::vector<int> r(xs.size(), 0);
    for (size_t i = 0; i < xs.size(); i++) {
        if (xs[i]->level >= 1) continue;
        if (!auto_boot) throw Error(-3, "mult: operand at level 0 cannot be multiplied");
        r[i] = 1;
        slots.push_back(&xs[i]);
    }
    if (slots.empty()) return;
    std::vector<u64> nonces = batch_nonces(r);
    refresh_many(c, slots, nonces);
}

CtP Eval::ready(const CtP& a) {
    if (a->level >= 1) return a;
    if (!auto_boot) throw Error(-3, "mult: operand at level 0 cannot be multiplied");
    CtP o = refresh_planned(a, 0, 1);
    plan.events += 1;
    return o;
}

CtP Eval::add(const CtP& a, const CtP& b, bool sub) {
    rec(OP_ADD);
    const int l = std::min(a->level, b->level);
    model(OP_ADD, MV_CT, l);
    return ev_add(c, *at(a, l), *at(b, l), sub);
}

CtP Eval::add_c(const CtP& a, std::complex<double> s, bool sub, bool reversed) {
    rec(OP_ADD);
    model(OP_ADD, MV_SCALAR, a->level);
    // ct + s, ct - s, s - ct
    if (reversed) return ev_add_const(c, *a, s.real(), s.imag(), true);
    if (sub) s = -s;
    return ev_add_const(c, *a, s.real(), s.imag(), false);
}

CtP Eval::add_p(const CtP& a, const Pattern& p, bool sub, bool reversed) {
    rec(OP_ADD);
    model(OP_ADD, MV_PT, a->level);
    PtP pt = encoded(p, a->level);
    return ev_add_pt(c, *a, *pt, sub, reversed);
}

CtP Eval::mult(const CtP& x, const CtP& y) {
    // per-operand auto-bootstrap, x before y (emulator.py:218-221)
    const int r = (x->level < 1 ? 1 : 0) + (y->level < 1 ? 1 : 0);
    if (r && !auto_boot) throw Error(-3, "mult: operand at level 0 cannot be multiplied");
    CtP a = x, b = y;
    int j = 0;
    if (x->level < 1) a = refresh_planned(x, j++, r);
    if (y->level < 1) b = refresh_planned(y, j++, r);
    plan.events += r;
    rec(OP_MULT);
    const int l = std::min(a->level, b->level);
    model(OP_MULT, MV_CT, l);
    return ev_mult(c, *at(a, l), *at(b, l));
}

CtP Eval::mult_c(const CtP& x, std::complex<double> s) {
    CtP a = ready(x);
    rec(OP_CMULT);
    model(OP_CMULT, MV_SCALAR, a->level);
    return ev_mul_const(c, *a, s.real(), s.imag());
}

CtP Eval::mult_p(const CtP& x, const Pattern& p) {
    CtP a = ready(x);
    rec(OP_CMULT);
    model(OP_CMULT, MV_PT, a->level);
    PtP pt = encoded(p, a->level);
    return ev_mul_pt(c, *a, *pt);
}

CtP Eval::lrot(const CtP& a, int64_t r) {
    const int64_t S = c.N / 2;
    r = ((r % S) + S) % S;
    if (r == 0) return a;
    rec(OP_ROT);
    model(OP_ROT, MV_CT, a->level);
    return ev_automorph(c, *a, galois_rot(c, r));
}

CtP Eval::add_lrot(const CtP& a, int64_t r) {
    const int64_t S = c.N / 2;
    r = ((r % S) + S) % S;
    if (r == 0) return add(a, a);
    rec(OP_ROT);
    rec(OP_ADD);
    model(OP_ROT, MV_CT, a->level);
    model(OP_ADD, MV_CT, a->level);
    CtP o;
    if (ev_automorph_add(c, *a, galois_rot(c, r), o)) return o;
    CtP rot = ev_automorph(c, *a, galois_rot(c, r));
    return ev_add(c, *a, *rot, false);
}

std::vector<CtP> Eval::lrot_batch(const std::vector<CtP>& xs, int64_t r, bool add_self) {
    const int64_t S = c.N / 2;
    r = ((r % S) + S) % S;
    std::vector<CtP> out(xs.size());
    if (r == 0) {
        for (size_t i = 0; i < xs.size(); i++) out[i] = add_self ? add(xs[i], xs[i]) : xs[i];
        return out;
    }
    rec(OP_ROT, (int)xs.size());
    if (add_self) rec(OP_ADD, (int)xs.size());
    for (auto& x : xs) {
        model(OP_ROT, MV_CT, x->level);
        if (add_self) model(OP_ADD, MV_CT, x->level);
    }
    std::vector<const Ct*> a(xs.size());
    for (size_t i = 0; i < xs.size(); i++) a[i] = xs[i].get();
    return ev_automorph_batch(c, a, galois_rot(c, r), add_self);
}

// doubling steps of the next rotate-and-sum stage when `rem` remain (oracle/slots.py
// ladder_plan): radix 8 while >= 5 remain or exactly 3, else radix 4, else one step
static int ladder_width(int rem) { return (rem >= 5 || rem == 3) ? 3 : std::min(2, rem); }

std::vector<CtP> Eval::ladder(const std::vector<CtP>& xs_in, int64_t stride, int steps) {
    std::vector<CtP> xs = xs_in;
    if (!c.hoist) {
        for (int t = 0; t < steps; t++) xs = lrot_batch(xs, stride * ((int64_t)1 << t), true);
        return xs;
    }
    const int64_t S = c.N / 2;
    for (int t = 0; t < steps;) {
        const int w = ladder_width(steps - t);
        const int64_t base = stride * ((int64_t)1 << t);
        t += w;
        std::vector<u64> gals;
        bool zero = false;
        for (int u = 1; u < (1 << w); u++) {
            const int64_t r = (((base * u) % S) + S) % S;
            zero |= r == 0;
            gals.push_back(galois_rot(c, r));
        }
        if (zero) throw Error(-4, "ladder: rotation by a multiple of the slot count");
        // the ledger and the §8(d) model record the w doubling steps this stage stands for
        rec(OP_ROT, w * (int)xs.size());
        rec(OP_ADD, w * (int)xs.size());
        for (auto& x : xs) {
            model(OP_ROT, MV_CT, x->level, w);
            model(OP_ADD, MV_CT, x->level, w);
        }
        // one stage per level present
        std::vector<CtP> out(xs.size());
        std::vector<char> done(xs.size(), 0);
        for (size_t i = 0; i < xs.size(); i++) {
            if (done[i]) continue;
            std::vector<size_t> idx;
            std::vector<const Ct*> a;
            for (size_t j = i; j < xs.size(); j++)
                if (!done[j] && xs[j]->level == xs[i]->level) {
                    idx.push_back(j);
                    a.push_back(xs[j].get());
                    done[j] = 1;
                }
            std::vector<CtP> r = ev_rotsum_batch(c, a, gals);
            for (size_t k = 0; k < idx.size(); k++) out[idx[k]] = r[k];
        }
        xs = out;
    }
    return xs;
}

std::vector<CtP> Eval::conj_batch(const std::vector<CtP>& xs) {
    rec(OP_CONJ, (int)xs.size());
    for (auto& x : xs) model(OP_CONJ, MV_CT, x->level);
    std::vector<const Ct*> a(xs.size());
    for (size_t i = 0; i < xs.size(); i++) a[i] = xs[i].get();
    return ev_automorph_batch(c, a, 2 * (u64)c.N - 1, false);
}

std::vector<CtP> Eval::mult_batch(const std::vector<CtP>& xs_in, const std::vector<CtP>& ys_in) {
    std::vector<CtP> xs = xs_in, ys = ys_in;
    std::vector<CtP> out(xs.size());
    // per-operand auto-bootstrap (emulator.py:218-221) in the reference's
    // op-by-op order -- x before y, product by product -- so every refresh
    // draws the nonce the sequential order gives it; then one batch
    std::vector<CtP*> slots;
    std::vector<int> rs(xs.size(), 0);
    for (size_t i = 0; i < xs.size(); i++) {
        const int r = (xs[i]->level < 1 ? 1 : 0) + (ys[i]->level < 1 ? 1 : 0);
        if (!r) continue;
        if (!auto_boot) throw Error(-3, "mult: operand at level 0 cannot be multiplied");
        rs[i] = r;
        if (xs[i]->level < 1) slots.push_back(&xs[i]);
        if (ys[i]->level < 1) slots.push_back(&ys[i]);
    }
    if (!slots.empty()) {
        std::vector<u64> nonces = batch_nonces(rs);
        refresh_many(c, slots, nonces);
    }
    rec(OP_MULT, (int)xs.size());
    for (size_t i = 0; i < xs.size(); i++) model(OP_MULT, MV_CT, std::min(xs[i]->level, ys[i]->level));
    // level adjustments in batches; an operand shared by several products
    // (DiagATB's B blocks, one per pass) is adjusted once (deterministic)
    std::vector<int> ls(xs.size());
    for (size_t i = 0; i < xs.size(); i++) ls[i] = std::min(xs[i]->level, ys[i]->level);
    std::vector<CtP> ax = xs, ay = ys;
    at_batch(ax, ls);
    at_batch(ay, ls);
    // one fused pipeline per level present
    std::vector<char> done(xs.size(), 0);
    for (size_t i = 0; i < xs.size(); i++) {
        if (done[i]) continue;
        std::vector<size_t> idx;
        std::vector<std::pair<const Ct*, const Ct*>> ab;
        for (size_t j = i; j < xs.size(); j++)
            if (!done[j] && ax[j]->level == ax[i]->level) {
                idx.push_back(j);
                ab.emplace_back(ax[j].get(), ay[j].get());
                done[j] = 1;
            }
        std::vector<CtP> r = ev_mult_batch(c, ab);
        for (size_t k = 0; k < idx.size(); k++) out[idx[k]] = r[k];
    }
    return out;
}

std::vector<std::vector<CtP>> Eval::lrot_hoisted(const std::vector<CtP>& xs, const std::vector<int64_t>& rs) {
    const int64_t S = c.N / 2;
    std::vector<int64_t> rr(rs.size());
    std::vector<u64> gals;
    std::vector<int> slot(rs.size(), -1);
    for (size_t k = 0; k < rs.size(); k++) {
        rr[k] = ((rs[k] % S) + S) % S;
        if (!rr[k]) continue;
        for (size_t j = 0; j < k; j++)
            if (rr[j] == rr[k]) slot[k] = slot[j];
        if (slot[k] < 0) { slot[k] = (int)gals.size(); gals.push_back(galois_rot(c, rr[k])); }
    }
    std::vector<std::vector<CtP>> out(xs.size(), std::vector<CtP>(rs.size()));
    int moving = 0;
    for (auto v : rr) moving += v != 0;
    rec(OP_ROT, moving * (int)xs.size());
    for (auto& x : xs) model(OP_ROT, MV_CT, x->level, moving);
    // one hoisted pipeline per level present
    std::vector<char> done(xs.size(), 0);
    for (size_t i = 0; i < xs.size(); i++) {
        if (done[i]) continue;
        std::vector<size_t> idx;
        std::vector<const Ct*> a;
        for (size_t j = i; j < xs.size(); j++)
            if (!done[j] && xs[j]->level == xs[i]->level) {
                idx.push_back(j);
                a.push_back(xs[j].get());
                done[j] = 1;
            }
        std::vector<std::vector<CtP>> h = ev_rot_hoisted(c, a, gals);
        for (size_t t = 0; t < idx.size(); t++)
            for (size_t k = 0; k < rs.size(); k++) out[idx[t]][k] = rr[k] ? h[t][slot[k]] : xs[idx[t]];
    }
    return out;
}

std::vector<CtP> Eval::mult_sum_batch(const std::vector<std::vector<CtP>>& as, const std::vector<std::vector<CtP>>& bs) {
    std::vector<CtP> out(as.size());
    std::vector<size_t> fused;
    for (size_t i = 0; i < as.size(); i++) {
        const size_t n = as[i].size();
        bool ok = n >= 2 && bs[i].size() == n;
        const int l = as[i][0]->level;
        for (size_t q = 0; ok && q < n; q++) ok = as[i][q]->level == l && bs[i][q]->level == l;
        ok = ok && l >= 1;
        if (ok) { fused.push_back(i); continue; }
        // the separate ops, in the reference's order
        CtP acc = mult(as[i][0], bs[i][0]);
        for (size_t q = 1; q < n; q++) acc = add(acc, mult(as[i][q], bs[i][q]));
        out[i] = acc;
    }
    // one batched relinearisation per level present
    std::vector<char> done(fused.size(), 0);
    for (size_t u = 0; u < fused.size(); u++) {
        if (done[u]) continue;
        std::vector<size_t> idx;
        std::vector<std::vector<std::pair<const Ct*, const Ct*>>> groups;
        const int l = as[fused[u]][0]->level;
        for (size_t v = u; v < fused.size(); v++) {
            const size_t i = fused[v];
            if (done[v] || as[i][0]->level != l) continue;
            done[v] = 1;
            idx.push_back(i);
            std::vector<std::pair<const Ct*, const Ct*>> gr;
            for (size_t q = 0; q < as[i].size(); q++) gr.emplace_back(as[i][q].get(), bs[i][q].get());
            groups.push_back(gr);
            rec(OP_MULT, (int)as[i].size());
            rec(OP_ADD, (int)as[i].size() - 1);
            model(OP_MULT, MV_CT, l, (int)as[i].size());
            model(OP_ADD, MV_CT, l - 1, (int)as[i].size() - 1);
        }
        std::vector<CtP> r = ev_mult_sum_batch(c, groups);
        for (size_t t = 0; t < idx.size(); t++) out[idx[t]] = r[t];
    }
    return out;
}

// ---- batched element-wise ops (one launch over the blocks of a lockstep op)

std::vector<CtP> Eval::at_batch(std::vector<CtP>& xs, const std::vector<int>& ls) {
    // group the needed adjustments by (source level, target): one batch each;
    // a ciphertext needed by several slots is adjusted once (deterministic)
    std::map<std::pair<int, int>, std::vector<const Ct*>> groups;
    std::map<std::pair<const Ct*, int>, CtP> done;
    for (size_t i = 0; i < xs.size(); i++) {
        if (xs[i]->level == ls[i]) continue;
        auto key = std::make_pair((const Ct*)xs[i].get(), ls[i]);
        if (done.count(key)) continue;
        done[key] = nullptr;
        groups[{xs[i]->level, ls[i]}].push_back(xs[i].get());
    }
    for (auto& kv : groups) {
        rec(OP_ADJUST, (int)kv.second.size());
        std::vector<CtP> r = ev_level_adjust_batch(c, kv.second, kv.first.second);
        for (size_t u = 0; u < r.size(); u++) done[{kv.second[u], kv.first.second}] = r[u];
    }
    for (size_t i = 0; i < xs.size(); i++)
        if (xs[i]->level != ls[i]) xs[i] = done[{xs[i].get(), ls[i]}];
    return xs;
}

std::vector<CtP> Eval::add_batch(const std::vector<CtP>& xs_in, const std::vector<CtP>& ys_in, bool sub) {
    std::vector<CtP> out(xs_in.size());
    std::vector<CtP> xs = xs_in, ys = ys_in;
    bool ok = xs.size() > 1;
    int lmin = ok ? xs[0]->level : 0;
    for (size_t i = 0; ok && i < xs.size(); i++) lmin = std::min(lmin, std::min(xs[i]->level, ys[i]->level));
    if (ok) {
        // result level min(levels) per pair (emulator.py:195-210); one batch
        // when every pair lands on one level
        std::vector<int> ls(xs.size());
        for (size_t i = 0; i < xs.size(); i++) {
            ls[i] = std::min(xs[i]->level, ys[i]->level);
            ok = ok && ls[i] == lmin;
        }
        if (ok) {
            at_batch(xs, ls);
            at_batch(ys, ls);
        }
    }
    if (!ok) {
        for (size_t i = 0; i < xs.size(); i++) out[i] = add(xs[i], ys[i], sub);
        return out;
    }
    rec(OP_ADD, (int)xs.size());
    const int level = xs[0]->level;
    model(OP_ADD, MV_CT, level, (int)xs.size());
    std::vector<u64*> o(xs.size());
    std::vector<const u64*> a(xs.size()), b(xs.size());
    for (size_t i = 0; i < xs.size(); i++) {
        out[i] = new_ct(c, level);
        o[i] = out[i]->d;
        a[i] = xs[i]->d;
        b[i] = ys[i]->d;
    }
    k_elementwise_batch(c, sub ? EWP_SUB : EWP_ADD, (int)xs.size(), o.data(), a.data(), b.data(), nullptr, level + 1,
                        2, 2);
    return out;
}

std::vector<CtP> Eval::add_c_batch(const std::vector<CtP>& xs, std::complex<double> s, bool sub, bool reversed) {
    std::vector<CtP> out(xs.size());
    bool ok = xs.size() > 1;
    for (auto& x : xs) ok = ok && x->level == xs[0]->level;
    if (!ok) {
        for (size_t i = 0; i < xs.size(); i++) out[i] = add_c(xs[i], s, sub, reversed);
        return out;
    }
    rec(OP_ADD, (int)xs.size());
    const int level = xs[0]->level;
    model(OP_ADD, MV_SCALAR, level, (int)xs.size());
    if (!reversed && sub) s = -s;
    const double sc = c.scale[level];
    ConstTab t;
    const_pairs(c, std::llrint(s.real() * sc), std::llrint(s.imag() * sc), level + 1, t);
    std::vector<u64*> o(xs.size());
    std::vector<const u64*> a(xs.size());
    for (size_t i = 0; i < xs.size(); i++) {
        out[i] = new_ct(c, level);
        o[i] = out[i]->d;
        a[i] = xs[i]->d;
    }
    k_elementwise_batch(c, reversed ? EWP_CONST_RADD : EWP_CONST_ADD, (int)xs.size(), o.data(), a.data(), nullptr,
                        &t, level + 1, 2, 0);
    return out;
}

std::vector<CtP> Eval::add_p_batch(const std::vector<CtP>& xs, const Pattern& p, bool sub, bool reversed) {
    std::vector<CtP> out(xs.size());
    bool ok = xs.size() > 1;
    for (auto& x : xs) ok = ok && x->level == xs[0]->level;
    if (!ok) {
        for (size_t i = 0; i < xs.size(); i++) out[i] = add_p(xs[i], p, sub, reversed);
        return out;
    }
    rec(OP_ADD, (int)xs.size());
    const int level = xs[0]->level;
    model(OP_ADD, MV_PT, level, (int)xs.size());
    PtP pt = encoded(p, level);
    std::vector<u64*> o(xs.size());
    std::vector<const u64*> a(xs.size()), b(xs.size(), pt->d);
    for (size_t i = 0; i < xs.size(); i++) {
        out[i] = new_ct(c, level);
        o[i] = out[i]->d;
        a[i] = xs[i]->d;
    }
    const int op = reversed ? EWP_PT_RSUB : (sub ? EWP_PT_SUB : EWP_PT_ADD);
    k_elementwise_batch(c, op, (int)xs.size(), o.data(), a.data(), b.data(), nullptr, level + 1, 2, 1);
    return out;
}

std::vector<CtP> Eval::mult_c_batch(const std::vector<CtP>& xs_in, std::complex<double> s) {
    std::vector<CtP> xs = xs_in;
    if (xs.size() > 1) ready_batch(xs);   // refreshes in block order, batched
    std::vector<CtP> out(xs.size());
    bool ok = c.logN >= 14 && xs.size() > 1;
    for (auto& x : xs) ok = ok && x->level >= 1 && x->level == xs[0]->level;
    if (!ok) {
        for (size_t i = 0; i < xs.size(); i++) out[i] = mult_c(xs[i], s);
        return out;
    }
    rec(OP_CMULT, (int)xs.size());
    const int level = xs[0]->level;
    model(OP_CMULT, MV_SCALAR, level, (int)xs.size());
    const size_t poly = (size_t)(level + 1) * c.N;
    const double sc = c.scale[level];
    ConstTab t;
    const_pairs(c, std::llrint(s.real() * sc), std::llrint(s.imag() * sc), level + 1, t);
    Scratch scr(c);
    u64* T = scr.take(2 * poly * xs.size());
    {   // the products of the batch in one launch
        std::vector<u64*> o(xs.size());
        std::vector<const u64*> a(xs.size());
        for (size_t i = 0; i < xs.size(); i++) {
            o[i] = T + 2 * poly * i;
            a[i] = xs[i]->d;
        }
        k_elementwise_batch(c, EWP_CONST_MUL, (int)xs.size(), o.data(), a.data(), nullptr, &t, level + 1, 2, 0);
    }
    rescale_many(c, T, poly, level, out);
    return out;
}

std::vector<CtP> Eval::mult_p_batch(const std::vector<CtP>& xs_in, const std::vector<const Pattern*>& ps) {
    std::vector<CtP> xs = xs_in;
    if (xs.size() > 1) ready_batch(xs);   // refreshes in block order, batched
    std::vector<CtP> out(xs.size());
    bool ok = c.logN >= 14 && xs.size() > 1;
    for (auto& x : xs) ok = ok && x->level >= 1;
    if (!ok) {
        for (size_t i = 0; i < xs.size(); i++) out[i] = mult_p(xs[i], *ps[i]);
        return out;
    }
    // one batch per level present (DiagATB's passes end one level apart): the
    // products in one launch, then one batched rescale
    std::map<int, std::vector<size_t>> groups;
    for (size_t i = 0; i < xs.size(); i++) groups[xs[i]->level].push_back(i);
    for (auto it = groups.rbegin(); it != groups.rend(); ++it) {
        const int level = it->first;
        const std::vector<size_t>& idx = it->second;
        const size_t n = idx.size();
        rec(OP_CMULT, (int)n);
        model(OP_CMULT, MV_PT, level, (int)n);
        const size_t poly = (size_t)(level + 1) * c.N;
        Scratch sc(c);
        u64* T = sc.take(2 * poly * n);
        std::vector<PtP> pts(n);
        std::vector<u64*> o(n);
        std::vector<const u64*> a(n), b(n);
        for (size_t u = 0; u < n; u++) {
            pts[u] = encoded(*ps[idx[u]], level);
            o[u] = T + 2 * poly * u;
            a[u] = xs[idx[u]]->d;
            b[u] = pts[u]->d;
        }
        k_elementwise_batch(c, EWP_PT_MUL, (int)n, o.data(), a.data(), b.data(), nullptr, level + 1, 2, 1);
        std::vector<CtP> r(n);
        rescale_many(c, T, poly, level, r);
        for (size_t u = 0; u < n; u++) out[idx[u]] = r[u];
    }
    return out;
}

CtP Eval::conj(const CtP& a) {
    rec(OP_CONJ);
    model(OP_CONJ, MV_CT, a->level);
    return ev_automorph(c, *a, 2 * (u64)c.N - 1);
}

CtP Eval::mul_i(const CtP& a) {
    model(MODEL_MULI, MV_CT, a->level);   // unledgered (emulator.py:259-265) but charged by §8(d)
    return ev_mul_i(c, *a);
}

CtP Eval::bootstrap(const CtP& a) {
    CtP o = refresh_planned(a, 0, 1);
    plan.events += 1;
    return o;
}

PtP Eval::encoded(const Pattern& p, int level) {
    std::string key = p.key + "@" + std::to_string(level);
    {
        std::lock_guard<std::mutex> g(c.mu);
        auto it = c.pt_cache.find(key);
        if (it != c.pt_cache.end()) {
            it->second.used = ++c.pt_clock;
            return it->second.pt;
        }
    }
    std::vector<std::complex<double>> generated;
    const std::vector<std::complex<double>>* vals = &p.vals;
    if (p.vals.empty() && p.gen) {
        generated.resize(c.N / 2);
        p.gen(generated);
        vals = &generated;
    }
    std::vector<double> zr(vals->size()), zi(vals->size());
    for (size_t i = 0; i < vals->size(); i++) { zr[i] = (*vals)[i].real(); zi[i] = (*vals)[i].imag(); }
    PtP pt = encode_pt(c, zr.data(), zi.data(), level, c.scale[level]);
    std::lock_guard<std::mutex> g(c.mu);
    if (!c.pt_cache_cap) {
        const char* e = std::getenv("HC_PT_CACHE_MB");
        c.pt_cache_cap = (size_t)(e ? std::atoll(e) : 4096) << 20;
    }
    const size_t bytes = (size_t)(level + 1) * c.N * 8;
    auto ins = c.pt_cache.emplace(key, Ctx::PtEntry{pt, ++c.pt_clock});
    if (!ins.second) return ins.first->second.pt;
    c.pt_cache_bytes += bytes;
    // evict least-recently-used entries (never the one just inserted); a
    // schedule still holding an evicted plaintext keeps it alive (shared_ptr)
    while (c.pt_cache_bytes > c.pt_cache_cap && c.pt_cache.size() > 1) {
        auto lru = c.pt_cache.end();
        for (auto it = c.pt_cache.begin(); it != c.pt_cache.end(); ++it)
            if (it != ins.first && (lru == c.pt_cache.end() || it->second.used < lru->second.used)) lru = it;
        c.pt_cache_bytes -= (size_t)(lru->second.pt->level + 1) * c.N * 8;
        c.pt_cache.erase(lru);
    }
    return pt;
}

}  // namespace hc
