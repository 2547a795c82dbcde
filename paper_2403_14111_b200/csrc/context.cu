// Context setup (parameters, primes, device tables), key generation,
// encoding, encryption, decryption and the refresh surrogate.
//
// Every choice follows the CKKS spec in DESIGN.md §3; the host encoder is
// compiled with -ffp-contract=off so its double arithmetic is bit-identical
// to the oracle's (oracle/ckks_oracle.c) on the same machine.
#include <set>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"

namespace hc {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------------------
// host number theory
// ---------------------------------------------------------------------------

static u64 powmod(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = (u64)(((u128)r * b) % q);
        b = (u64)(((u128)b * b) % q);
        e >>= 1;
    }
    return r;
}
static u64 invmod(u64 a, u64 q) { return powmod(a % q, q - 2, q); }
static u64 mulm(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 shoup_of(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }

static bool is_prime(u64 n) {
    static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (u64 b : bases)
        if (n % b == 0) return n == b;
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    for (u64 b : bases) {
        u64 x = powmod(b, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; r++) {
            x = mulm(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

static unsigned brv(unsigned x, int bits) {
    unsigned r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

double host_trace_threshold_ms() {
    static const double t = [] {
        const char* e = std::getenv("HC_HOST_TRACE");
        return e ? std::atof(e) : -1.0;
    }();
    return t;
}
static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
HostTrace::HostTrace(const char* w) : what(w) {
    if (host_trace_threshold_ms() >= 0) t0 = now_ms();
}
HostTrace::~HostTrace() {
    if (host_trace_threshold_ms() < 0) return;
    const double dt = now_ms() - t0;
    if (dt > host_trace_threshold_ms()) std::fprintf(stderr, "[hc host] %s blocked %.1f ms\n", what, dt);
}

u64* Ctx::alloc(size_t words) {
    HostTrace tr("alloc");
    void* p = nullptr;
    HC_CUDA(cudaMallocFromPoolAsync(&p, words * sizeof(u64), pool, stream));
    return (u64*)p;
}
void Ctx::free(u64* p) {
    HostTrace tr("free");
    if (p) HC_CUDA(cudaFreeAsync(p, stream));
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("HC_PDL");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

Scratch::Scratch(Ctx& ctx) : c(ctx) {
    a = &c.arenas[c.stream];
    mark = a->top;
}
Scratch::~Scratch() { a->top = mark; }
u64* Scratch::take(size_t words) {
    words = (words + 31) & ~(size_t)31;   // 256-byte alignment
    if (a->top + words > a->cap) {
        // grow: the old buffer may still be read by queued work on this
        // stream, so it is retired, not freed; live data below `top` in it is
        // not moved (outer scopes keep their pointers), only new takes go to
        // the new buffer
        HostTrace tr("scratch grow");
        const size_t need = std::max(a->cap * 2, a->top + words + ((size_t)64 << 20) / 8);
        void* p = nullptr;
        HC_CUDA(cudaMalloc(&p, need * sizeof(u64)));
        if (a->base) c.arena_graveyard.push_back(a->base);
        a->base = (u64*)p;
        a->cap = need;
        // outer scopes' marks index the old buffer; restart this scope at 0 of the new one
        a->top = 0;
        mark = 0;
    }
    u64* p = a->base + a->top;
    a->top += words;
    return p;
}

cudaEvent_t Ctx::get_event() {
    if (!ev_free.empty()) {
        cudaEvent_t e = ev_free.back();
        ev_free.pop_back();
        return e;
    }
    cudaEvent_t e;
    HC_CUDA(cudaEventCreate(&e));
    return e;
}

Launch::Launch(Ctx& ctx, const char* name, double bytes) : c(ctx), trace(name) {
    c.launches++;
    if (!c.prof) return;
    Ctx::ProfRec r{name, c.get_event(), c.get_event(), bytes};
    HC_CUDA(cudaEventRecord(r.a, c.stream));
    idx = (int)c.prof_recs.size();
    c.prof_recs.push_back(r);
}

Launch::~Launch() {
    if (idx >= 0) cudaEventRecord(c.prof_recs[idx].b, c.stream);
}

size_t Ct::words() const { return (size_t)npoly * (level + 1) * ctx->N; }
u64* Ct::poly(int s) const { return d + (size_t)s * (level + 1) * ctx->N; }

static void ct_deleter(Ct* c) {
    if (c->d && c->ctx) {
        try { c->ctx->free(c->d); } catch (...) {}
    }
    delete c;
}
static void pt_deleter(Pt* p) {
    if (p->d && p->ctx) {
        try { p->ctx->free(p->d); } catch (...) {}
    }
    delete p;
}

CtP new_ct(Ctx& c, int level, int npoly) {
    Ct* x = new Ct();
    x->ctx = &c;
    x->level = level;
    x->npoly = npoly;
    x->d = c.alloc((size_t)npoly * (level + 1) * c.N);
    return CtP(x, ct_deleter);
}

PtP new_pt(Ctx& c, int level) {
    Pt* x = new Pt();
    x->ctx = &c;
    x->level = level;
    x->d = c.alloc((size_t)(level + 1) * c.N);
    return PtP(x, pt_deleter);
}

void ntt_limbs(Ctx& c, u64* d, int p0, int n, bool inverse, const u64* src) {
    for (int base = 0; base < n; base += MAXJ) {
        JobList j;
        j.n = std::min(MAXJ, n - base);
        for (int i = 0; i < j.n; i++) {
            j.prime[i] = p0 + base + i;
            j.ptr[i] = d + (size_t)(base + i) * c.N;
            j.src[i] = src ? src + (size_t)(base + i) * c.N : nullptr;
        }
        if (inverse) ntt_inverse(c, j); else ntt_forward(c, j);
    }
}

template <class T>
static T* upload(Ctx& c, const std::vector<T>& v) {
    T* d = nullptr;
    HC_CUDA(cudaMalloc(&d, sizeof(T) * v.size()));
    HC_CUDA(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return d;
}

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------

Ctx* ctx_create(int logN, int nq, const int* qbits, int np, const int* pbits, int alpha, int log_scale, int hw,
                double sigma, u64 seed, int device) {
    if (logN < 4 || logN > 17 || nq < 1 || np < 1 || nq + np > MAXP || alpha < 1 || alpha > 8 || np > 8)
        throw Error(-1, "bad parameters");
    Ctx* c = new Ctx();
    c->logN = logN; c->N = 1 << logN; c->L = nq - 1; c->K = np; c->alpha = alpha; c->app_L = nq - 1;
    c->dnum = (nq + alpha - 1) / alpha; c->nall = nq + np; c->hw = hw; c->sigma = sigma; c->seed = seed;
    c->device = device;
    const int N = c->N, M = N / 2, nall = c->nall, L = c->L, K = c->K;
    HC_CUDA(cudaSetDevice(device));
    HC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->main_stream = c->stream;
    if (const char* e = std::getenv("HC_STREAMS")) c->fork_cap = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("HC_NTT_FP")) c->ntt_fp = std::atoi(e) != 0;
    if (const char* e = std::getenv("HC_LOCKSTEP")) c->lockstep = std::atoi(e) != 0;
    if (const char* e = std::getenv("HC_HOIST")) c->hoist = std::atoi(e) != 0;
    if (const char* e = std::getenv("HC_BATCH")) c->batch = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("HC_RUNAHEAD")) c->ra_depth = std::max(1, std::atoi(e));
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    HC_CUDA(cudaMemPoolCreate(&c->pool, &props));
    uint64_t thr = UINT64_MAX;
    HC_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // Reserve the pool's working set up front (one allocation, freed back to the
    // pool, which keeps it): growing the pool mid-schedule maps memory through
    // the driver and showed up as ~2x step-time spikes.
    {
        const size_t reserve = (size_t)512 * (size_t)(nq + np) * ((size_t)8 << logN);
        void* p = nullptr;
        HC_CUDA(cudaMallocFromPoolAsync(&p, reserve, c->pool, c->stream));
        HC_CUDA(cudaFreeAsync(p, c->stream));
        HC_CUDA(cudaStreamSynchronize(c->stream));
    }
    // Cross-stream reuse of freed blocks (the pool's event tracking) stays on by
    // default: stream-local reuse (HC_POOL_XSTREAM=0) issues ~25% faster on the
    // host but lets every side stream grow its own cache, and the resulting
    // pool growth measured as multi-x step-time spikes.
    {
        const char* e = std::getenv("HC_POOL_XSTREAM");
        int on = (e && !std::atoi(e)) ? 0 : 1;
        HC_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseFollowEventDependencies, &on));
        HC_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowOpportunistic, &on));
        HC_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowInternalDependencies, &on));
    }

    // primes: below 2^b, q = 2^b - t*2N + 1, first unused prime in order
    std::vector<u64> used;
    for (int i = 0; i < nall; i++) {
        const int b = i < nq ? qbits[i] : pbits[i - nq];
        // q < 2^60: the forward NTT keeps lazy values below 16q in one word (ntt_pass.cuh)
        if (b < 20 || b > 60) throw Error(-1, "prime bits out of range (20..60)");
        for (u64 t = 1;; t++) {
            const u64 q = ((u64)1 << b) - t * 2 * (u64)N + 1;
            bool dup = false;
            for (u64 u : used) dup |= (u == q);
            if (!dup && is_prime(q)) { used.push_back(q); break; }
        }
    }
    std::vector<PrimeDev> pd(nall);
    std::vector<u64> tw((size_t)2 * nall * N), itw((size_t)2 * nall * N);
    for (int i = 0; i < nall; i++) {
        PrimeHost& p = c->pr[i];
        const u64 q = used[i];
        p.q = q;
        const u128 mu = (~(u128)0) / q;
        p.mu_hi = (u64)(mu >> 64);
        p.mu_lo = (u64)mu;
        for (u64 g = 2;; g++) {
            const u64 x = powmod(g, (q - 1) / (2 * (u64)N), q);
            if (powmod(x, (u64)N, q) == q - 1) { p.psi = x; break; }
        }
        p.ipsi = invmod(p.psi, q);
        p.ninv = invmod((u64)N, q);
        p.I = powmod(p.psi, (u64)N / 2, q);
        const bool fp = c->ntt_fp && q < ((u64)1 << FP_MAXBITS);
        pd[i] = PrimeDev{q, 2 * q, p.mu_hi, p.mu_lo, p.I, shoup_of(p.I, q), p.ninv, shoup_of(p.ninv, q),
                         (double)q, 1.0 / (double)q, fp ? 1 : 0};
        std::vector<u64> pw(N), ipw(N);
        pw[0] = ipw[0] = 1;
        for (int k = 1; k < N; k++) { pw[k] = mulm(pw[k - 1], p.psi, q); ipw[k] = mulm(ipw[k - 1], p.ipsi, q); }
        for (int k = 0; k < N; k++) {
            const unsigned r = brv((unsigned)k, logN);
            // (w, w_shoup) pairs: one 16-byte load per twiddle in the NTT passes;
            // FP64 primes hold (w, w/q) as doubles instead (ntt_pass.cuh ArFp)
            auto pair = [&](u64 w, u64* dst) {
                if (fp) {
                    const double wd = (double)w, wq = wd / (double)q;
                    std::memcpy(dst, &wd, 8);
                    std::memcpy(dst + 1, &wq, 8);
                } else {
                    dst[0] = w;
                    dst[1] = shoup_of(w, q);
                }
            };
            pair(pw[r], &tw[2 * ((size_t)i * N + k)]);
            pair(ipw[r], &itw[2 * ((size_t)i * N + k)]);
        }
    }
    c->d_primes = upload(*c, pd);
    c->d_tw = upload(*c, tw);
    c->d_itw = upload(*c, itw);

    // canonical scales
    c->scale[L] = std::ldexp(1.0, log_scale);
    for (int l = L; l >= 1; l--) c->scale[l - 1] = (c->scale[l] * c->scale[l]) / (double)c->pr[l].q;

    // ModUp tables: [level][digit][a][target prime] (value, shoup) and [level][digit][a] inverses
    std::vector<u64> mu_tab((size_t)(L + 1) * c->dnum * alpha * nall * 2, 0);
    std::vector<u64> mu_inv((size_t)(L + 1) * c->dnum * alpha * 2, 0);
    for (int l = 0; l <= L; l++)
        for (int j = 0; j < c->dnum; j++) {
            const int lo = j * alpha;
            if (lo > l) continue;
            const int hi = std::min(lo + alpha, l + 1);
            for (int a = lo; a < hi; a++) {
                const u64 qa = c->pr[a].q;
                u64 qh = 1;
                for (int b = lo; b < hi; b++) if (b != a) qh = mulm(qh, c->pr[b].q % qa, qa);
                const u64 inv = invmod(qh, qa);
                const size_t ii = ((size_t)(l * c->dnum + j) * alpha + (a - lo)) * 2;
                mu_inv[ii] = inv;
                mu_inv[ii + 1] = shoup_of(inv, qa);
                for (int t = 0; t < nall; t++) {
                    const u64 pt = c->pr[t].q;
                    u64 v = 1;
                    for (int b = lo; b < hi; b++) if (b != a) v = mulm(v, c->pr[b].q % pt, pt);
                    const size_t ti = (((size_t)(l * c->dnum + j) * alpha + (a - lo)) * nall + t) * 2;
                    mu_tab[ti] = v;
                    mu_tab[ti + 1] = shoup_of(v, pt);
                }
            }
        }
    c->d_modup = upload(*c, mu_tab);
    c->d_modup_inv = upload(*c, mu_inv);
    std::vector<u64> mu_negq((size_t)(L + 1) * c->dnum * nall, 0);
    for (int l = 0; l <= L; l++)
        for (int j = 0; j < c->dnum; j++) {
            const int lo = j * alpha;
            if (lo > l) continue;
            const int hi = std::min(lo + alpha, l + 1);
            for (int t = 0; t < nall; t++) {
                const u64 pt = c->pr[t].q;
                u64 v = 1;
                for (int b = lo; b < hi; b++) v = mulm(v, c->pr[b].q % pt, pt);
                mu_negq[(size_t)(l * c->dnum + j) * nall + t] = v ? pt - v : 0;
            }
        }
    c->d_modup_negq = upload(*c, mu_negq);
    std::vector<u64> mu_cc((size_t)(L + 1) * c->dnum * nall, 0);
    for (int l = 0; l <= L; l++)
        for (int j = 0; j < c->dnum; j++) {
            const int lo = j * alpha;
            if (lo > l) continue;
            const int hi = std::min(lo + alpha, l + 1);
            for (int t = 0; t < nall; t++) {
                const u64 pt = c->pr[t].q;
                u64 sacc = 0;
                for (int a = lo; a < hi; a++) {
                    const size_t ti = (((size_t)(l * c->dnum + j) * alpha + (a - lo)) * nall + t) * 2;
                    sacc = (sacc + mulm(((c->pr[a].q - 1) / 2) % pt, mu_tab[ti], pt)) % pt;
                }
                mu_cc[(size_t)(l * c->dnum + j) * nall + t] = sacc ? pt - sacc : 0;
            }
        }
    c->d_modup_cc = upload(*c, mu_cc);

    // ModDown tables
    std::vector<u64> md_tab((size_t)K * nall * 2), md_inv((size_t)K * 2), pinv((size_t)nall * 2), pm(nall);
    for (int t = 0; t < K; t++) {
        const u64 pt = c->pr[L + 1 + t].q;
        u64 ph = 1;
        for (int b = 0; b < K; b++) if (b != t) ph = mulm(ph, c->pr[L + 1 + b].q % pt, pt);
        const u64 inv = invmod(ph, pt);
        md_inv[2 * t] = inv;
        md_inv[2 * t + 1] = shoup_of(inv, pt);
        for (int i = 0; i < nall; i++) {
            const u64 qi = c->pr[i].q;
            u64 v = 1;
            for (int b = 0; b < K; b++) if (b != t) v = mulm(v, c->pr[L + 1 + b].q % qi, qi);
            md_tab[((size_t)t * nall + i) * 2] = v;
            md_tab[((size_t)t * nall + i) * 2 + 1] = shoup_of(v, qi);
        }
    }
    for (int i = 0; i < nall; i++) {
        const u64 qi = c->pr[i].q;
        u64 P = 1;
        for (int t = 0; t < K; t++) P = mulm(P, c->pr[L + 1 + t].q % qi, qi);
        pm[i] = P;
        const u64 inv = (i <= L) ? invmod(P, qi) : 0;
        pinv[2 * i] = inv;
        pinv[2 * i + 1] = (i <= L) ? shoup_of(inv, qi) : 0;
    }
    c->d_moddown = upload(*c, md_tab);
    c->d_moddown_inv = upload(*c, md_inv);
    std::vector<u64> md_negp(nall);
    for (int i = 0; i < nall; i++) md_negp[i] = pm[i] ? c->pr[i].q - pm[i] : 0;
    c->d_moddown_negp = upload(*c, md_negp);
    std::vector<u64> md_cc(nall, 0);
    for (int i = 0; i < nall; i++) {
        const u64 qi = c->pr[i].q;
        u64 sacc = 0;
        for (int t = 0; t < K; t++)
            sacc = (sacc + mulm(((c->pr[L + 1 + t].q - 1) / 2) % qi, md_tab[((size_t)t * nall + i) * 2], qi)) % qi;
        md_cc[i] = sacc ? qi - sacc : 0;
    }
    c->d_moddown_cc = upload(*c, md_cc);
    c->d_pinv = upload(*c, pinv);
    // merged ModDown + rescale: per level l >= 1 the dropped
    // basis is B = (q_l, p_1..p_K), D = q_l * P
    {
        const int nb = K + 1;
        std::vector<u64> inv((size_t)(L + 1) * nb * 2, 0), tab((size_t)(L + 1) * nb * nall * 2, 0),
            negd((size_t)(L + 1) * nall, 0), cc((size_t)(L + 1) * nall, 0), dinv((size_t)(L + 1) * nall * 2, 0);
        for (int l = 1; l <= L; l++) {
            std::vector<int> bp(nb);
            bp[0] = l;
            for (int t = 0; t < K; t++) bp[1 + t] = L + 1 + t;
            for (int t = 0; t < nb; t++) {
                const u64 bt = c->pr[bp[t]].q;
                u64 dh = 1;
                for (int b = 0; b < nb; b++) if (b != t) dh = mulm(dh, c->pr[bp[b]].q % bt, bt);
                const u64 iv = invmod(dh, bt);
                inv[((size_t)l * nb + t) * 2] = iv;
                inv[((size_t)l * nb + t) * 2 + 1] = shoup_of(iv, bt);
            }
            for (int i = 0; i < l; i++) {
                const u64 qi = c->pr[i].q;
                u64 Dm = 1, sacc = 0;
                for (int t = 0; t < nb; t++) {
                    u64 v = 1;
                    for (int b = 0; b < nb; b++) if (b != t) v = mulm(v, c->pr[bp[b]].q % qi, qi);
                    tab[(((size_t)l * nb + t) * nall + i) * 2] = v;
                    tab[(((size_t)l * nb + t) * nall + i) * 2 + 1] = shoup_of(v, qi);
                    Dm = mulm(Dm, c->pr[bp[t]].q % qi, qi);
                    sacc = (sacc + mulm(((c->pr[bp[t]].q - 1) / 2) % qi, v, qi)) % qi;
                }
                negd[(size_t)l * nall + i] = Dm ? qi - Dm : 0;
                cc[(size_t)l * nall + i] = sacc ? qi - sacc : 0;
                const u64 di = invmod(Dm, qi);
                dinv[((size_t)l * nall + i) * 2] = di;
                dinv[((size_t)l * nall + i) * 2 + 1] = shoup_of(di, qi);
            }
        }
        c->d_md2_inv = upload(*c, inv);
        c->d_md2_tab = upload(*c, tab);
        c->d_md2_negd = upload(*c, negd);
        c->d_md2_cc = upload(*c, cc);
        c->d_md2_dinv = upload(*c, dinv);
    }
    // P mod q_i for key generation lives right after the rescale table
    std::vector<u64> rs((size_t)(L + 1) * nall * 3 + nall, 0);
    for (int l = 1; l <= L; l++) {
        const u64 ql = c->pr[l].q;
        for (int i = 0; i < l; i++) {
            const u64 qi = c->pr[i].q;
            const u64 inv = invmod(ql % qi, qi);
            rs[((size_t)l * nall + i) * 3] = inv;
            rs[((size_t)l * nall + i) * 3 + 1] = shoup_of(inv, qi);
            rs[((size_t)l * nall + i) * 3 + 2] = ql % qi;
        }
    }
    for (int i = 0; i < nall; i++) rs[(size_t)(L + 1) * nall * 3 + i] = pm[i];
    c->d_rescale = upload(*c, rs);

    // encoder tables
    c->tw_re.resize(M); c->tw_im.resize(M); c->zt_re.resize(M); c->zt_im.resize(M); c->slot_t.resize(M);
    for (int k = 0; k < M; k++) {
        const double a = 2.0 * M_PI * (double)k / (double)M;
        c->tw_re[k] = std::cos(a); c->tw_im[k] = std::sin(a);
        const double b = M_PI * (double)k / (double)N;
        c->zt_re[k] = std::cos(b); c->zt_im[k] = std::sin(b);
    }
    u64 e = 1;
    for (int j = 0; j < M; j++) { c->slot_t[j] = (int)((e - 1) / 4); e = (e * 5) % (2 * (u64)N); }

    // CDT discrete Gaussian over [-B, B]
    const int B = (int)std::ceil(sigma * 12.0);
    if (2 * B > 128) throw Error(-1, "sigma too large");
    double tot = 0.0;
    for (int x = -B; x <= B; x++) tot += std::exp(-(double)x * (double)x / (2.0 * sigma * sigma));
    double acc = 0.0;
    c->cdt_b = B; c->cdt_n = 2 * B;
    for (int i = 0; i < 2 * B; i++) {
        const int x = -B + i;
        acc += std::exp(-(double)x * (double)x / (2.0 * sigma * sigma));
        const double v = (acc / tot) * 18446744073709551616.0;
        c->cdt_host[i] = v >= 18446744073709551615.0 ? ~(u64)0 : (u64)v;
    }
    c->d_cdt = upload(*c, std::vector<u64>(c->cdt_host, c->cdt_host + c->cdt_n));

    // ternary secret with Hamming weight hw
    c->sk_coef.assign(N, 0);
    const u64 skey = rng_key(seed, stream_id(DOM_SK, 0, 0));
    u64 ctr = 0;
    for (int i = 0; i < hw; i++) {
        u64 pos;
        for (;;) {
            pos = (u64)(((u128)rng_at(skey, ctr++) * (u64)N) >> 64);
            if (!c->sk_coef[pos]) break;
        }
        c->sk_coef[pos] = (rng_at(skey, ctr++) & 1) ? 1 : -1;
    }
    i64* d_s = (i64*)c->alloc(N);
    HC_CUDA(cudaMemcpyAsync(d_s, c->sk_coef.data(), sizeof(i64) * N, cudaMemcpyHostToDevice, c->stream));
    HC_CUDA(cudaMalloc(&c->d_sk, sizeof(u64) * (size_t)nall * N));
    k_coef_to_rns(*c, c->d_sk, d_s, nullptr, 0, nall);
    ntt_limbs(*c, c->d_sk, 0, nall, false);
    c->free((u64*)d_s);
    HC_CUDA(cudaStreamSynchronize(c->stream));
    return c;
}

void ctx_destroy(Ctx* c) {
    if (!c) return;
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    if (c->d2h_stream) cudaStreamSynchronize(c->d2h_stream);
    c->io_pending.clear();
    cudaStreamSynchronize(c->stream);
    for (auto& kv : c->arenas) cudaFree(kv.second.base);
    for (auto* p : c->arena_graveyard) cudaFree(p);
    if (std::getenv("HC_POOL_STATS")) {
        uint64_t v[4] = {0, 0, 0, 0};
        cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrReservedMemCurrent, &v[0]);
        cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrReservedMemHigh, &v[1]);
        cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrUsedMemCurrent, &v[2]);
        cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrUsedMemHigh, &v[3]);
        std::fprintf(stderr, "[hc pool] reserved %.2f GB (high %.2f GB), used %.2f GB (high %.2f GB)\n", v[0] / 1e9,
                     v[1] / 1e9, v[2] / 1e9, v[3] / 1e9);
    }
    c->pt_cache.clear();
    c->pt_cache_bytes = 0;
    c->boot.reset();   // bootstrapping plaintexts return to the pool while it exists
    for (auto& kv : c->keys) cudaFree(kv.second.d);
    cudaFree(c->d_primes); cudaFree(c->d_tw); cudaFree(c->d_itw);
    cudaFree(c->d_cdt); cudaFree(c->d_sk); cudaFree(c->d_modup); cudaFree(c->d_modup_inv);
    cudaFree(c->d_moddown); cudaFree(c->d_moddown_inv); cudaFree(c->d_modup_negq); cudaFree(c->d_moddown_negp); cudaFree(c->d_modup_cc); cudaFree(c->d_moddown_cc); cudaFree(c->d_pinv); cudaFree(c->d_rescale);
    cudaFree(c->d_md2_inv); cudaFree(c->d_md2_tab); cudaFree(c->d_md2_negd); cudaFree(c->d_md2_cc); cudaFree(c->d_md2_dinv);
    cudaStreamSynchronize(c->stream);
    for (auto s : c->side) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    for (auto e : c->side_ev) cudaEventDestroy(e);
    if (c->fork_ev) cudaEventDestroy(c->fork_ev);
    for (auto e : c->fork_evs) cudaEventDestroy(e);
    for (auto e : c->ra_ev) if (e) cudaEventDestroy(e);
    cudaMemPoolDestroy(c->pool);
    cudaStreamDestroy(c->main_stream);
    delete c;
}

u64 galois_rot(const Ctx& c, int64_t r) {
    const int64_t M = c.N / 2;
    const u64 rr = (u64)(((r % M) + M) % M);
    return powmod(5, rr, 2 * (u64)c.N);
}

// ---------------------------------------------------------------------------
// switching keys: b_j = -a_j s + e_j + [limb in digit j] P s'
// ---------------------------------------------------------------------------

Key& get_key(Ctx& c, int gid) {
    auto it = c.keys.find(gid);
    if (it != c.keys.end()) return it->second;
    const int N = c.N, nall = c.nall;
    const size_t poly = (size_t)nall * N;
    Key k;
    k.id = gid;
    HC_CUDA(cudaMalloc(&k.d, sizeof(u64) * (size_t)c.dnum * 2 * poly));
    u64* sp = c.alloc(poly);
    if (gid == 0) k_square(c, sp, c.d_sk, nall);
    else k_automorph(c, sp, c.d_sk, nall, (u64)gid);
    i64* e = (i64*)c.alloc(N);
    const u64* pm = c.d_rescale + (size_t)(c.L + 1) * nall * 3;
    for (int j = 0; j < c.dnum; j++) {
        u64* b = k.d + (size_t)(2 * j) * poly;
        u64* a = b + poly;
        k_uniform(c, a, 0, nall, stream_id(DOM_KEY_A, (u64)gid, (u64)j));
        k_cdt(c, e, stream_id(DOM_KEY_E, (u64)gid, (u64)j));
        k_coef_to_rns(c, b, e, nullptr, 0, nall);
        ntt_limbs(c, b, 0, nall, false);
        const int lo = j * c.alpha, hi = std::min(lo + c.alpha, c.L + 1);
        k_key_combine(c, b, a, c.d_sk, sp, pm, nall, lo, hi);
    }
    c.free((u64*)e);
    c.free(sp);
    // other streams may use the key right after this returns
    HC_CUDA(cudaStreamSynchronize(c.stream));
    return c.keys.emplace(gid, k).first->second;
}

// ---------------------------------------------------------------------------
// host encoder: slot j <-> zeta^(5^j); size N/2 radix-2 FFT
// ---------------------------------------------------------------------------

static void fft(const Ctx& c, double* re, double* im, bool inverse) {
    const int M = c.N / 2, logM = c.logN - 1;
    for (int i = 0; i < M; i++) {
        const int r = (int)brv((unsigned)i, logM);
        if (r > i) { std::swap(re[i], re[r]); std::swap(im[i], im[r]); }
    }
    for (int len = 2; len <= M; len <<= 1) {
        const int half = len >> 1, step = M / len;
        for (int i = 0; i < M; i += len)
            for (int j = 0; j < half; j++) {
                const double wr = c.tw_re[j * step];
                const double wi = inverse ? -c.tw_im[j * step] : c.tw_im[j * step];
                const double vr0 = re[i + j + half], vi0 = im[i + j + half];
                const double vr = vr0 * wr - vi0 * wi;
                const double vi = vr0 * wi + vi0 * wr;
                const double ur = re[i + j], ui = im[i + j];
                re[i + j] = ur + vr; im[i + j] = ui + vi;
                re[i + j + half] = ur - vr; im[i + j + half] = ui - vi;
            }
    }
}

int encode_host(const Ctx& c, const double* zr, const double* zi, double scale, int64_t* coef) {
    const int M = c.N / 2;
    std::vector<double> re(M), im(M);
    for (int j = 0; j < M; j++) { re[c.slot_t[j]] = zr[j]; im[c.slot_t[j]] = zi ? zi[j] : 0.0; }
    fft(c, re.data(), im.data(), true);
    const double inv = 1.0 / (double)M;
    bool bad = false;
    for (int k = 0; k < M; k++) {
        const double wr = re[k] * inv, wi = im[k] * inv;
        const double ur = wr * c.zt_re[k] + wi * c.zt_im[k];
        const double ui = wi * c.zt_re[k] - wr * c.zt_im[k];
        const double a = ur * scale, b = ui * scale;
        if (!(std::fabs(a) < 9.2e18) || !(std::fabs(b) < 9.2e18)) bad = true;
        coef[k] = bad ? 0 : std::llrint(a);
        coef[k + M] = bad ? 0 : std::llrint(b);
    }
    return bad ? -1 : 0;
}

void decode_host(const Ctx& c, const double* m, double* zr, double* zi) {
    const int M = c.N / 2;
    std::vector<double> re(M), im(M);
    for (int k = 0; k < M; k++) {
        const double ur = m[k], ui = m[k + M];
        re[k] = ur * c.zt_re[k] - ui * c.zt_im[k];
        im[k] = ur * c.zt_im[k] + ui * c.zt_re[k];
    }
    fft(c, re.data(), im.data(), false);
    for (int j = 0; j < M; j++) { zr[j] = re[c.slot_t[j]]; zi[j] = im[c.slot_t[j]]; }
}

PtP encode_pt(Ctx& c, const double* zr, const double* zi, int level, double scale) {
    std::vector<int64_t> m(c.N);
    if (encode_host(c, zr, zi, scale, m.data())) throw Error(-5, "encode overflow");
    i64* dm = (i64*)c.alloc(c.N);
    HC_CUDA(cudaMemcpyAsync(dm, m.data(), sizeof(i64) * c.N, cudaMemcpyHostToDevice, c.stream));
    PtP p = new_pt(c, level);
    k_coef_to_rns(c, p->d, dm, nullptr, 0, level + 1);
    ntt_limbs(c, p->d, 0, level + 1, false);
    c.free((u64*)dm);
    HC_CUDA(cudaStreamSynchronize(c.stream));   // host vector m goes out of scope
    return p;
}

// ---------------------------------------------------------------------------
// encryption (secret key), decryption, refresh surrogate
// ---------------------------------------------------------------------------

CtP encrypt_coef_dev(Ctx& c, const int64_t* d_m, int level, u64 nonce) {
    const int nl = level + 1;
    CtP ct = new_ct(c, level);
    k_uniform(c, ct->poly(1), 0, nl, stream_id(DOM_ENC_A, nonce, 0));
    i64* e = (i64*)c.alloc(c.N);
    k_cdt(c, e, stream_id(DOM_ENC_E, nonce, 0));
    k_coef_to_rns(c, ct->poly(0), d_m, e, 0, nl);
    ntt_limbs(c, ct->poly(0), 0, nl, false);
    k_enc_combine(c, ct->poly(0), ct->poly(1), nl);
    c.free((u64*)e);
    return ct;
}

CtP encrypt(Ctx& c, const double* zr, const double* zi, int level, u64 nonce) {
    std::vector<int64_t> m(c.N);
    if (encode_host(c, zr, zi, c.scale[level], m.data())) throw Error(-5, "encode overflow");
    i64* dm = (i64*)c.alloc(c.N);
    HC_CUDA(cudaMemcpyAsync(dm, m.data(), sizeof(i64) * c.N, cudaMemcpyHostToDevice, c.stream));
    CtP ct = encrypt_coef_dev(c, dm, level, nonce);
    c.free((u64*)dm);
    HC_CUDA(cudaStreamSynchronize(c.stream));
    return ct;
}

// x = INTT(c0 + c1 s) over the first nl limbs
static u64* dec_limbs(Ctx& c, const Ct& a, int nl) {
    u64* x = c.alloc((size_t)nl * c.N);
    k_dec(c, x, a.poly(0), a.poly(1), nl);
    ntt_limbs(c, x, 0, nl, true);
    return x;
}

void decrypt(Ctx& c, const Ct& a, double* zr, double* zi) {
    const int N = c.N, nl = a.level >= 1 ? 2 : 1;
    u64* x = dec_limbs(c, a, nl);
    std::vector<u64> h((size_t)nl * N);
    HC_CUDA(cudaMemcpyAsync(h.data(), x, sizeof(u64) * h.size(), cudaMemcpyDeviceToHost, c.stream));
    c.free(x);
    HC_CUDA(cudaStreamSynchronize(c.stream));
    const u64 q0 = c.pr[0].q;
    std::vector<double> md(N);
    for (int k = 0; k < N; k++) {
        const u64 v0 = h[k];
        const i64 x0 = v0 > (q0 - 1) / 2 ? (i64)v0 - (i64)q0 : (i64)v0;
        if (nl == 1) { md[k] = (double)x0; continue; }
        const u64 q1 = c.pr[1].q;
        const u64 xm = x0 >= 0 ? (u64)x0 % q1 : (q1 - 1 - ((u64)(-(x0 + 1)) % q1));
        const u64 d = h[N + k] >= xm ? h[N + k] - xm : h[N + k] + q1 - xm;
        const u64 kk = mulm(d, invmod(q0 % q1, q1), q1);
        const i64 kc = kk > (q1 - 1) / 2 ? (i64)kk - (i64)q1 : (i64)kk;
        md[k] = (double)x0 + (double)q0 * (double)kc;
    }
    const double s = c.scale[a.level];
    for (int k = 0; k < N; k++) md[k] = md[k] / s;
    decode_host(c, md.data(), zr, zi);
}

// B refreshes of ciphertexts at one level (the surrogate above, batched)
std::vector<CtP> refresh_batch(Ctx& c, const std::vector<const Ct*>& a, const std::vector<u64>& nonces) {
    std::vector<CtP> out(a.size());
    for (size_t b0 = 0; b0 < a.size(); b0 += KS_MAXB) {
        const int B = (int)std::min<size_t>(KS_MAXB, a.size() - b0);
        const int level = a[b0]->level;
        for (int b = 0; b < B; b++)
            if (a[b0 + b]->level != level) throw Error(-4, "batched refresh needs one level");
        const int two = level >= 1 ? 1 : 0, nl = c.app_L + 1;
        Scratch sc(c);
        u64* X = sc.take((size_t)B * (1 + two) * c.N);
        std::vector<const u64*> c0(B), c1(B);
        std::vector<u64*> xb(B), o(B);
        for (int b = 0; b < B; b++) {
            c0[b] = a[b0 + b]->poly(0);
            c1[b] = a[b0 + b]->poly(1);
            xb[b] = X + (size_t)b * (1 + two) * c.N;
            out[b0 + b] = new_ct(c, c.app_L);
            o[b] = out[b0 + b]->d;
        }
        const u64* nn = nonces.data() + b0;
        k_refresh_batch(c, B, c0.data(), c1.data(), xb.data(), nullptr, nn, 0, two, 0, 0);
        {
            JobList j;
            j.n = B * (1 + two);
            for (int b = 0; b < B; b++)
                for (int i = 0; i <= two; i++) {
                    j.prime[b * (1 + two) + i] = i;
                    j.ptr[b * (1 + two) + i] = xb[b] + (size_t)i * c.N;
                    j.src[b * (1 + two) + i] = nullptr;
                }
            ntt_inverse(c, j);
        }
        const u64 inv01 = two ? invmod(c.pr[0].q % c.pr[1].q, c.pr[1].q) : 0;
        k_refresh_batch(c, B, nullptr, nullptr, xb.data(), o.data(), nn, 1, two, inv01, c.scale[c.app_L] / c.scale[level]);
        for (int base = 0; base < B * nl; base += MAXJ) {
            JobList j;
            j.n = std::min(MAXJ, B * nl - base);
            for (int u = 0; u < j.n; u++) {
                const int b = (base + u) / nl, i = (base + u) % nl;
                j.prime[u] = i;
                j.ptr[u] = o[b] + (size_t)i * c.N;
                j.src[u] = nullptr;
            }
            ntt_forward(c, j);
        }
        k_refresh_batch(c, B, nullptr, nullptr, xb.data(), o.data(), nn, 2, two, 0, 0);
    }
    return out;
}

CtP refresh(Ctx& c, const Ct& a, u64 nonce) {
    const int two = a.level >= 1 ? 1 : 0;
    u64* x = dec_limbs(c, a, 1 + two);
    i64* m = (i64*)c.alloc(c.N);
    const u64 inv01 = two ? invmod(c.pr[0].q % c.pr[1].q, c.pr[1].q) : 0;
    k_refresh_msg(c, m, x, two, inv01, c.scale[c.app_L] / c.scale[a.level]);
    c.free(x);
    CtP out = encrypt_coef_dev(c, m, c.app_L, nonce);
    c.free((u64*)m);
    return out;
}

void set_smem_attr(const void* kern, size_t bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    HC_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if (done.insert({kern, dev}).second)
        HC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace hc
