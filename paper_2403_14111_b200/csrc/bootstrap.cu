// CKKS bootstrapping: ModRaise, CoeffToSlot, EvalMod,
// SlotToCoeff on the library's exact primitives.  Stands in for the
// reference's level reset (`bootstrap`, emulator.py:267-273; the paper ran
// HEaaN's) without the secret key: the server refreshes
// ciphertexts by homomorphic evaluation alone.  The C oracle's restatement
// (oracle/boot.py) performs the same exact operations, so the residues match
// bit for bit (tests/test_gpu_bootstrap.py).
//
//   ModRaise      level-0 coefficients, centred mod q0, lifted to q_0..q_L:
//                 the ciphertext decrypts to T = m + q0 I (I small)
//   CoeffToSlot   V^-1 (V_jk = zeta^(5^j k)) as log2(n) butterfly levels in
//                 three merged groups, each a set of diagonals applied by
//                 baby-step giant-step (babies lrot(x, b s), per giant the
//                 raw ct x pt products summed, one rescale, lrot by g n1 s);
//                 then one scalar product by Delta_L / (2 K q0)
//   EvalMod       u + conj(u) and -i (u - conj(u)); each a degree-27
//                 Chebyshev series of cos(2 pi (K u - 1/4) / 16) and four
//                 double angles -> sin(2 pi x), x = T / q0
//   SlotToCoeff   exact integer gain 2^15, re + i im, the forward groups
//                 (innermost first, 1/(2 pi) and q0 / Delta_0 folded in)
//                 landing at the application's top level
//
// Every matrix entry is +-2^-r zeta^E with an exact integer exponent; the
// values f * (cos(pi E / N), sin(pi E / N)) and the Chebyshev table are
// computed by the same expressions as the oracle's, so the encoded
// plaintexts are bit-identical.
#include <cmath>
#include <map>

#include "evaluator.h"
#include "kernels.cuh"

namespace hc {

namespace {

constexpr int K_RANGE = 16;
constexpr int DOUBLINGS = 4;
constexpr u64 INT_GAIN = 1ull << 15;
const double CHEB[28] = {
    0.21921621501751104,     -0.04163425650808503,    0.5729882897213429,     -0.005706988408963243,
    0.6283207584137114,      0.07308641363683221,     -0.5527025194229122,    -0.030879541430194817,
    0.14588477734714397,     0.005709279677339937,    -0.020179274144300055,  -0.0006170816570300078,
    0.0017582253584081749,   4.4379335769130696e-05,  -0.0001063328757854582, -2.291335574193446e-06,
    4.746072353514685e-06,   8.935411073699164e-08,   -1.6317891342227947e-07, -2.730062564463901e-09,
    4.461227928980592e-09,   6.71974137060941e-11,    -9.940233410834453e-11, -1.3618179787512087e-12,
    1.840671891504253e-12,   2.3454661363066562e-14,  -2.95837563102632e-14,  -5.269516377095246e-16};
constexpr int CHEB_DEG = 27;

// one merged group of butterfly levels, baby-step giant-step form
struct Group {
    int s = 1, n1 = 1, level = -1;
    std::vector<int> babies;                                  // baby indices b (rotation b * s)
    std::vector<std::pair<int, std::vector<std::pair<int, PtP>>>> giants;   // g -> [(b, pre-rotated diagonal)]
    // host values before encoding: g -> b -> slots
    std::map<int, std::map<int, std::vector<std::complex<double>>>> vals;
};

}  // namespace

struct BootState {
    std::vector<Group> cts, stc;
    double c_cts = 0;
};

namespace {

std::vector<std::vector<int>> level_groups(int L, int ng = 3) {
    std::vector<std::vector<int>> out;
    const int base = L / ng, extra = L % ng;
    int lo = 1;
    for (int g = 0; g < ng; g++) {
        const int sz = base + (g < extra ? 1 : 0);
        std::vector<int> v;
        for (int i = 0; i < sz; i++) v.push_back(lo + i);
        out.push_back(v);
        lo += sz;
    }
    return out;
}

u64 powm(u64 b, u64 e, u64 m) {
    unsigned __int128 r = 1, x = b % m;
    while (e) {
        if (e & 1) r = (r * x) % m;
        x = (x * x) % m;
        e >>= 1;
    }
    return (u64)r;
}

// the diagonals of one merged group: rows propagate through the levels
// (inverse: B_last^-1 first ... B_first^-1 last; forward: B_first ... B_last)
Group make_group(const Ctx& c, const std::vector<int>& levels, bool inverse, double factor,
                 const std::vector<double>& zre, const std::vector<double>& zim) {
    const int N = c.N, n = N / 2;
    const int64_t twoN = 2 * (int64_t)N;
    const int r = (int)levels.size();
    std::vector<int> order = levels;
    if (inverse) std::reverse(order.begin(), order.end());
    std::vector<int64_t> cols(n), exps(n, 0);
    for (int j = 0; j < n; j++) cols[j] = j;
    int width = 1;
    for (int lv : order) {
        const int bs = n >> (lv - 1), h = bs / 2;
        std::vector<int64_t> E5(h);
        for (int v = 0; v < h; v++) E5[v] = (int64_t)powm(5, (u64)v, (u64)twoN);
        std::vector<int64_t> nc((size_t)n * 2 * width), ne((size_t)n * 2 * width);
        for (int j = 0; j < n; j++)
            for (int w = 0; w < width; w++) {
                const int64_t col = cols[(size_t)j * width + w], ex = exps[(size_t)j * width + w];
                const int64_t cin = col % bs;
                const bool top = cin < h;
                const int64_t jj = top ? cin : cin - h;
                const int64_t E = (E5[jj] * ((int64_t)1 << (lv - 1))) % twoN;
                int64_t c1 = top ? col : col - h, c2 = top ? col + h : col, e1, e2;
                if (inverse) {
                    e1 = top ? 0 : -E;
                    e2 = top ? 0 : N - E;
                } else {
                    e1 = 0;
                    e2 = top ? E : E + N;
                }
                const size_t o = (size_t)j * 2 * width;
                nc[o + w] = c1;
                ne[o + w] = (((ex + e1) % twoN) + twoN) % twoN;
                nc[o + width + w] = c2;
                ne[o + width + w] = (((ex + e2) % twoN) + twoN) % twoN;
            }
        cols.swap(nc);
        exps.swap(ne);
        width *= 2;
    }
    const double f = inverse ? std::ldexp(1.0, -r) * factor : factor;
    std::map<int, std::vector<std::complex<double>>> diags;
    for (int j = 0; j < n; j++)
        for (int w = 0; w < width; w++) {
            const int64_t col = cols[(size_t)j * width + w], e = exps[(size_t)j * width + w];
            const int d = (int)(((col - j) % n + n) % n);
            auto& v = diags[d];
            if (v.empty()) v.assign(n, std::complex<double>(0.0, 0.0));
            v[j] = std::complex<double>(f * zre[e], f * zim[e]);
        }
    Group g;
    g.s = n >> levels.back();
    std::map<int, const std::vector<std::complex<double>>*> ks;
    const int span = n / g.s;
    for (auto& kv : diags) {
        int k = kv.first / g.s;
        if (k >= span / 2) k -= span;
        ks[k] = &kv.second;
    }
    g.n1 = 1;
    while ((size_t)g.n1 * g.n1 < ks.size()) g.n1 *= 2;
    for (auto& kv : ks) {
        const int k = kv.first;
        const int gg = (k >= 0) ? k / g.n1 : -((-k + g.n1 - 1) / g.n1);   // floor division
        const int b = k - gg * g.n1;
        const int G = (int)((((int64_t)gg * g.n1 * g.s) % n + n) % n);
        std::vector<std::complex<double>> rolled(n);
        for (int j = 0; j < n; j++) rolled[j] = (*kv.second)[((j - G) % n + n) % n];
        g.vals[gg][b] = std::move(rolled);
    }
    std::map<int, int> bset;
    for (auto& gv : g.vals)
        for (auto& bv : gv.second) bset[bv.first] = 1;
    for (auto& kv : bset) g.babies.push_back(kv.first);
    return g;
}

// encode a group's diagonals at `level` (scale Delta_level) on first use
void encode_group(Ctx& c, Group& g, int level) {
    if (g.level == level) return;
    if (g.level >= 0) throw Error(-4, "bootstrap group applied at a different level");
    const int n = c.N / 2;
    std::vector<double> re(n), im(n);
    for (auto& gv : g.vals) {
        std::vector<std::pair<int, PtP>> row;
        for (auto& bv : gv.second) {
            for (int j = 0; j < n; j++) { re[j] = bv.second[j].real(); im[j] = bv.second[j].imag(); }
            row.emplace_back(bv.first, encode_pt(c, re.data(), im.data(), level, c.scale[level]));
        }
        g.giants.emplace_back(gv.first, std::move(row));
    }
    g.level = level;
    g.vals.clear();
}

BootState& boot_state(Ctx& c) {
    std::lock_guard<std::mutex> lk(c.mu);
    if (c.boot) return *c.boot;
    // CoeffToSlot 3 + scaling 1 + EvalMod 10 + SlotToCoeff 3 levels
    if (c.L - 17 != c.app_L) throw Error(-4, "bootstrapping needs exactly 17 levels above the application's");
    auto st = std::make_shared<BootState>();
    const int N = c.N;
    std::vector<double> zre(2 * (size_t)N), zim(2 * (size_t)N);
    for (int e = 0; e < 2 * N; e++) {
        zre[e] = std::cos(M_PI * (double)e / (double)N);
        zim[e] = std::sin(M_PI * (double)e / (double)N);
    }
    int lg = 0;
    while ((1 << lg) < N / 2) lg++;
    auto groups = level_groups(lg);
    const double q0 = (double)c.pr[0].q;
    st->c_cts = c.scale[c.L] / (2.0 * K_RANGE * q0);
    const double c_stc = q0 / (2.0 * M_PI * c.scale[0] * (double)INT_GAIN);
    for (auto& g : groups) st->cts.push_back(make_group(c, g, true, 1.0, zre, zim));
    for (int i = (int)groups.size() - 1; i >= 0; i--)
        st->stc.push_back(make_group(c, groups[i], false, i == (int)groups.size() - 1 ? c_stc : 1.0, zre, zim));
    c.boot = st;
    return *c.boot;
}

// ---- batched forms: every step over the vector of ciphertexts being
// bootstrapped together (the blocks of one lockstep op), each a batched key
// switch / rescale / product where the library has one; residues are those
// of the per-ciphertext ops

using V = std::vector<CtP>;

std::vector<const Ct*> ptrs(const V& v) {
    std::vector<const Ct*> p(v.size());
    for (size_t i = 0; i < v.size(); i++) p[i] = v[i].get();
    return p;
}

V rot(Ctx& c, const V& a, int64_t r) {
    const int64_t n = c.N / 2;
    r = ((r % n) + n) % n;
    if (r == 0) return a;
    return ev_automorph_batch(c, ptrs(a), galois_rot(c, r), false);
}

V adj(Ctx& c, const V& a, int to) {
    bool same = true;
    for (auto& x : a) same = same && x->level == a[0]->level;
    if (same && a[0]->level > to) return ev_level_adjust_batch(c, ptrs(a), to);
    V o(a.size());
    for (size_t i = 0; i < a.size(); i++) o[i] = a[i]->level == to ? a[i] : ev_level_adjust(c, *a[i], to);
    return o;
}

V rescale(Ctx& c, const V& a) {
    const int l = a[0]->level;
    V o(a.size());
    std::vector<const u64*> in(a.size());
    std::vector<u64*> out(a.size());
    for (size_t i = 0; i < a.size(); i++) {
        o[i] = new_ct(c, l - 1);
        in[i] = a[i]->d;
        out[i] = o[i]->d;
    }
    if (!rescale_fused_batch(c, (int)a.size(), in.data(), l, 2, out.data()))
        for (size_t i = 0; i < a.size(); i++) o[i] = ev_rescale(c, *a[i]);
    return o;
}

V add(Ctx& c, const V& a, const V& b, bool sub = false) {
    V o(a.size());
    for (size_t i = 0; i < a.size(); i++) o[i] = ev_add(c, *a[i], *b[i], sub);
    return o;
}

V add_const(Ctx& c, const V& a, double v) {
    V o(a.size());
    for (size_t i = 0; i < a.size(); i++) o[i] = ev_add_const(c, *a[i], v, 0.0, false);
    return o;
}

V mul_const(Ctx& c, const V& a, double v) {
    V o(a.size());
    for (size_t i = 0; i < a.size(); i++) o[i] = ev_mul_const(c, *a[i], v, 0.0);
    return o;
}

V mul_i(Ctx& c, const V& a) {
    V o(a.size());
    for (size_t i = 0; i < a.size(); i++) o[i] = ev_mul_i(c, *a[i]);
    return o;
}

V mult(Ctx& c, const V& a, const V& b) {
    std::vector<std::pair<const Ct*, const Ct*>> ab(a.size());
    for (size_t i = 0; i < a.size(); i++) ab[i] = {a[i].get(), b[i].get()};
    return ev_mult_batch(c, ab);
}

V conj(Ctx& c, const V& a) { return ev_automorph_batch(c, ptrs(a), 2 * (u64)c.N - 1, false); }

// y = M x for one merged group (baby-step giant-step), level l -> l - 1
V linear(Ctx& c, const V& x, Group& g) {
    const int l = x[0]->level;
    encode_group(c, g, l);
    std::map<int, V> baby;
    for (int b : g.babies) baby[b] = rot(c, x, (int64_t)b * g.s);
    const int nl = l + 1;
    V outer;
    for (auto& gv : g.giants) {
        // sum_b baby_b (x) pdiag_(g, b): one dot-product kernel per ciphertext
        V acc(x.size());
        for (size_t i = 0; i < x.size(); i++) {
            std::vector<const u64*> as, ps;
            for (auto& bp : gv.second) {
                as.push_back(baby[bp.first][i]->d);
                ps.push_back(bp.second->d);
            }
            acc[i] = new_ct(c, l);
            k_pt_dot(c, acc[i]->d, as.data(), ps.data(), (int)as.size(), nl);
        }
        V inner = rot(c, rescale(c, acc), (int64_t)gv.first * g.n1 * g.s);
        outer = outer.empty() ? inner : add(c, outer, inner);
    }
    return outer;
}

V mul_int(Ctx& c, const V& a, u64 k) {
    ConstTab t;
    const int nl = a[0]->level + 1;
    for (int i = 0; i < nl; i++) {
        const u64 q = c.pr[i].q, v = k % q;
        t.v[4 * i] = v;
        t.v[4 * i + 1] = (u64)(((unsigned __int128)v << 64) / q);
        t.v[4 * i + 2] = v;
        t.v[4 * i + 3] = t.v[4 * i + 1];
    }
    V o(a.size());
    for (size_t i = 0; i < a.size(); i++) {
        o[i] = new_ct(c, a[i]->level);
        k_elementwise(c, EWP_CONST_MUL, o[i]->d, a[i]->d, nullptr, &t, nl, 2, 0);
    }
    return o;
}

V evalmod(Ctx& c, const V& u) {
    std::vector<V> T(CHEB_DEG + 1);
    T[1] = u;
    for (int k = 2; k <= CHEB_DEG; k++) {
        int a = 1;
        while (a * 2 <= k) a *= 2;
        const int b = k - a;
        V t;
        if (b == 0) {
            t = mult(c, T[k / 2], T[k / 2]);
        } else {
            const int lm = std::min(T[a][0]->level, T[b][0]->level);
            t = mult(c, adj(c, T[a], lm), adj(c, T[b], lm));
        }
        t = add(c, t, t);
        T[k] = (b == 0) ? add_const(c, t, -1.0) : add(c, t, adj(c, T[a - b], t[0]->level), true);
    }
    int lmin = 1 << 30;
    for (int k = 1; k <= CHEB_DEG; k++) lmin = std::min(lmin, T[k][0]->level);
    V acc;
    for (int k = 1; k <= CHEB_DEG; k++) {
        V term = mul_const(c, adj(c, T[k], lmin), CHEB[k]);
        acc = acc.empty() ? term : add(c, acc, term);
    }
    acc = add_const(c, acc, CHEB[0]);
    for (int i = 0; i < DOUBLINGS; i++) {
        V t = mult(c, acc, acc);
        t = add(c, t, t);
        acc = add_const(c, t, -1.0);
    }
    return acc;
}

}  // namespace

// ModRaise of a level-0 ciphertext to level `to` (kernels.cu k_mod_raise)
CtP ev_mod_raise(Ctx& c, const Ct& a, int to) {
    if (a.level != 0) throw Error(-4, "mod raise needs a level-0 ciphertext");
    Scratch sc(c);
    u64* X = sc.take(2 * (size_t)c.N);
    {
        JobList j;
        j.n = 2;
        for (int s = 0; s < 2; s++) {
            j.prime[s] = 0;
            j.ptr[s] = X + (size_t)s * c.N;
            j.src[s] = a.poly(s);
        }
        ntt_inverse(c, j);
    }
    CtP o = new_ct(c, to);
    k_mod_raise(c, o->d, X, to + 1);
    const int nl = to + 1;
    for (int base = 0; base < 2 * nl; base += MAXJ) {
        JobList j;
        j.n = std::min(MAXJ, 2 * nl - base);
        for (int u = 0; u < j.n; u++) {
            const int s = (base + u) / nl, i = (base + u) % nl;
            j.prime[u] = i;
            j.ptr[u] = o->poly(s) + (size_t)i * c.N;
            j.src[u] = nullptr;
        }
        ntt_forward(c, j);
    }
    return o;
}

std::vector<CtP> ev_bootstrap_batch(Ctx& c, const std::vector<CtP>& in) {
    if (in.empty()) return {};
    BootState& st = boot_state(c);
    // one level per batch (the blocks of a lockstep op share their level history)
    for (auto& x : in)
        if (x->level != in[0]->level) {
            std::vector<CtP> o;
            for (auto& y : in) o.push_back(ev_bootstrap_batch(c, {y})[0]);
            return o;
        }
    V a = adj(c, in, 0);
    V x(a.size());
    for (size_t i = 0; i < a.size(); i++) x[i] = ev_mod_raise(c, *a[i], c.L);
    for (auto& g : st.cts) x = linear(c, x, g);
    x = mul_const(c, x, st.c_cts);
    V cj = conj(c, x);
    V ure = add(c, x, cj);
    V uim = mul_i(c, add(c, cj, x, true));
    // the real and imaginary parts through EvalMod together
    V both = ure;
    both.insert(both.end(), uim.begin(), uim.end());
    V s = evalmod(c, both);
    const size_t m = in.size();
    V sre(s.begin(), s.begin() + m), sim(s.begin() + m, s.end());
    V y = add(c, mul_int(c, sre, INT_GAIN), mul_i(c, mul_int(c, sim, INT_GAIN)));
    for (auto& g : st.stc) y = linear(c, y, g);
    if (y[0]->level != c.app_L) throw Error(-4, "bootstrap landed off the application's top level");
    return y;
}

CtP ev_bootstrap(Ctx& c, const CtP& a) { return ev_bootstrap_batch(c, {a})[0]; }

}  // namespace hc
