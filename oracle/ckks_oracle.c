/*
 * TEST INFRASTRUCTURE ONLY — CPU RNS-CKKS oracle (plain C, gcc, OpenMP).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product (the CUDA
 * library under paper_2403_14111_b200/csrc) never links or calls it.
 *
 * What it restates.  The reference (hefit, /root/reference/pkg/src/hefit)
 * models a ciphertext as a complex128 slot vector with a level
 * (emulator.py:49-67) and its ops as exact slot arithmetic
 * (emulator.py:195-273).  The RNS-CKKS scheme the paper runs on (HEaaN,
 * PAPER.md:509-513) is not in /root/reference, so this file restates the
 * published RNS-CKKS algorithms (Cheon-Kim-Kim-Song 2017; Cheon-Han-Kim-Kim-
 * Song RNS variant 2018; Han-Ki hybrid key switching 2020) with every free
 * choice pinned in DESIGN.md §3 ("the CKKS spec"), so that the CUDA product
 * and this oracle are bit-exact on residues:
 *   - primes below 2^b, q = 2^b - t*2N + 1, t = 1, 2, ...; psi from the
 *     smallest generator g with g^((q-1)/2N) of order 2N
 *   - negacyclic NTT, Cooley-Tukey, natural in / bit-reversed out; slot of
 *     NTT index j is evaluation at psi^(2*brv(j)+1)
 *   - encoder: slot j <-> zeta^(5^j); size-N/2 radix-2 complex FFT with a
 *     libm twiddle table, -ffp-contract=off, llrint rounding
 *   - per-level canonical scales D_L = 2^logD, D_{l-1} = D_l^2 / q_l
 *   - centred rescale; hybrid key switch with alpha primes per digit
 *   - splitmix64 counter PRNG; CDT discrete Gaussian; HW-h ternary secret
 *   - refresh surrogate = decrypt mod q0 (q0*q1 CRT when l >= 1) + re-encrypt
 *     (labelled: it is NOT CKKS bootstrapping; emulator.py:267-273 semantics)
 * Parity status: slot values pinned to the reference's golden vectors
 * (tests/golden); residues pinned only to internal mathematical KATs
 * (NTT == schoolbook negacyclic product, CRT == bigint), since no reference
 * residues exist.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned __int128 u128;

#define MAXP 48

typedef struct {
    u64 q, mu_hi, mu_lo;   /* Barrett: mu = floor(2^128 / q) */
    u64 psi, ipsi, ninv, I;
    u64 *w, *ws;           /* psi^brv(k), Shoup companion */
    u64 *iw, *iws;         /* psi^-brv(k) */
} prime_t;

typedef struct key_s {
    int id;                /* galois element, 0 = relinearisation */
    u64 *data;             /* [dnum][2][nall][N] */
    struct key_s *next;
} swkey_t;

typedef struct {
    int logN, N, L, K, alpha, dnum, nall, hw;
    int app_L;            /* application top level: refreshes land here */
    double sigma;
    u64 seed;
    prime_t pr[MAXP];
    double scale[MAXP];    /* canonical scale per level */
    double *tw_re, *tw_im; /* exp(2 pi i k / M), k < M */
    double *zt_re, *zt_im; /* zeta^k = exp(pi i k / N), k < M */
    int *slot_t;           /* t_j = (5^j mod 2N - 1)/4 */
    u64 cdt[128];
    int cdt_n, cdt_b;
    i64 *sk;               /* ternary secret, coefficient form */
    u64 *sk_ntt;           /* [nall][N] */
    swkey_t *keys;
} orc_ctx;

/* ------------------------------------------------------------------ */
/* modular arithmetic                                                  */
/* ------------------------------------------------------------------ */

static inline u64 mulhi(u64 a, u64 b) { return (u64)(((u128)a * b) >> 64); }

static inline u64 reduce128(u128 x, const prime_t *p) {
    u64 xh = (u64)(x >> 64), xl = (u64)x;
    u64 qh = xh * p->mu_hi + mulhi(xh, p->mu_lo) + mulhi(xl, p->mu_hi);
    u64 r = xl - qh * p->q;
    while (r >= p->q) r -= p->q;
    return r;
}
static inline u64 mulmod(u64 a, u64 b, const prime_t *p) { return reduce128((u128)a * b, p); }
static inline u64 addmod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
static inline u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
static inline u64 shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static inline u64 mul_shoup(u64 x, u64 w, u64 ws, u64 q) {
    u64 r = x * w - mulhi(x, ws) * q;
    return r >= q ? r - q : r;
}
static u64 powmod(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) { if (e & 1) r = (u64)(((u128)r * b) % q); b = (u64)(((u128)b * b) % q); e >>= 1; }
    return r;
}
static u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }
static inline u64 from_i64(i64 v, u64 q) {
    if (v >= 0) return (u64)v % q;
    u64 m = (u64)(-(v + 1)) % q;          /* -(v) - 1 without overflow */
    return q - 1 - m;
}

static int is_prime(u64 n) {
    static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) { if (n % bases[i] == 0) return n == bases[i]; }
    u64 d = n - 1; int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        u64 x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) {
            x = (u64)(((u128)x * x) % n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

static inline unsigned brv(unsigned x, int bits) {
    unsigned r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* ------------------------------------------------------------------ */
/* PRNG (splitmix64 counter mode) and samplers                         */
/* ------------------------------------------------------------------ */

static inline u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline u64 rng(u64 seed, u64 stream, u64 ctr) {
    return mix64(mix64(seed ^ mix64(stream + 0x9E3779B97F4A7C15ULL)) + ctr * 0x9E3779B97F4A7C15ULL);
}
static inline u64 stream_id(u64 domain, u64 id, u64 sub) { return (domain << 48) ^ (id << 16) ^ sub; }
enum { DOM_SK = 1, DOM_KEY_A = 2, DOM_KEY_E = 3, DOM_ENC_A = 4, DOM_ENC_E = 5 };

static inline i64 cdt_sample(const orc_ctx *c, u64 r) {
    int cnt = 0;
    for (int i = 0; i < c->cdt_n; i++) cnt += (c->cdt[i] <= r);
    return (i64)cnt - c->cdt_b;
}

/* ------------------------------------------------------------------ */
/* NTT                                                                 */
/* ------------------------------------------------------------------ */

static void ntt(const orc_ctx *c, const prime_t *p, u64 *a) {
    int N = c->N;
    u64 q = p->q;
    int t = N;
    for (int m = 1; m < N; m <<= 1) {
        t >>= 1;
        for (int i = 0; i < m; i++) {
            u64 W = p->w[m + i], Ws = p->ws[m + i];
            int j1 = 2 * i * t;
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = mul_shoup(a[j + t], W, Ws, q);
                a[j] = addmod(U, V, q);
                a[j + t] = submod(U, V, q);
            }
        }
    }
}

static void intt(const orc_ctx *c, const prime_t *p, u64 *a) {
    int N = c->N;
    u64 q = p->q;
    int t = 1;
    for (int m = N >> 1; m >= 1; m >>= 1) {
        for (int i = 0; i < m; i++) {
            u64 W = p->iw[m + i], Ws = p->iws[m + i];
            int j1 = 2 * i * t;
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = a[j + t];
                a[j] = addmod(U, V, q);
                a[j + t] = mul_shoup(submod(U, V, q), W, Ws, q);
            }
        }
        t <<= 1;
    }
    u64 ns = shoup(p->ninv, q);
    for (int j = 0; j < N; j++) a[j] = mul_shoup(a[j], p->ninv, ns, q);
}

/* ------------------------------------------------------------------ */
/* context                                                             */
/* ------------------------------------------------------------------ */

static void setup_prime(orc_ctx *c, prime_t *p, u64 q) {
    int N = c->N;
    p->q = q;
    u128 mu = (~(u128)0) / q;   /* floor((2^128 - 1)/q) == floor(2^128/q) for q not a power of 2 */
    p->mu_hi = (u64)(mu >> 64);
    p->mu_lo = (u64)mu;
    for (u64 g = 2;; g++) {
        u64 x = powmod(g, (q - 1) / (2 * (u64)N), q);
        if (powmod(x, (u64)N, q) == q - 1) { p->psi = x; break; }
    }
    p->ipsi = invmod(p->psi, q);
    p->ninv = invmod((u64)N, q);
    p->I = powmod(p->psi, (u64)N / 2, q);
    p->w = malloc(sizeof(u64) * N); p->ws = malloc(sizeof(u64) * N);
    p->iw = malloc(sizeof(u64) * N); p->iws = malloc(sizeof(u64) * N);
    u64 *pw = malloc(sizeof(u64) * N), *ipw = malloc(sizeof(u64) * N);
    pw[0] = 1; ipw[0] = 1;
    for (int i = 1; i < N; i++) {
        pw[i] = (u64)(((u128)pw[i - 1] * p->psi) % q);
        ipw[i] = (u64)(((u128)ipw[i - 1] * p->ipsi) % q);
    }
    for (int k = 0; k < N; k++) {
        unsigned r = brv((unsigned)k, c->logN);
        p->w[k] = pw[r]; p->ws[k] = shoup(pw[r], q);
        p->iw[k] = ipw[r]; p->iws[k] = shoup(ipw[r], q);
    }
    free(pw); free(ipw);
}

static u64 find_prime(int bits, int N, const u64 *used, int nused) {
    for (u64 t = 1;; t++) {
        u64 q = ((u64)1 << bits) - t * 2 * (u64)N + 1;
        int dup = 0;
        for (int i = 0; i < nused; i++) dup |= (used[i] == q);
        if (!dup && is_prime(q)) return q;
    }
}

orc_ctx *orc_create(int logN, int nq, const int *qbits, int np, const int *pbits, int alpha,
                    int log_scale, int hw, double sigma, u64 seed) {
    orc_ctx *c = calloc(1, sizeof(orc_ctx));
    c->logN = logN; c->N = 1 << logN; c->L = nq - 1; c->app_L = nq - 1; c->K = np; c->alpha = alpha;
    c->dnum = (nq + alpha - 1) / alpha; c->nall = nq + np; c->hw = hw; c->sigma = sigma;
    c->seed = seed;
    int N = c->N, M = N / 2;
    u64 used[MAXP];
    for (int i = 0; i < c->nall; i++) {
        int b = i < nq ? qbits[i] : pbits[i - nq];
        used[i] = find_prime(b, N, used, i);
        setup_prime(c, &c->pr[i], used[i]);
    }
    c->scale[c->L] = ldexp(1.0, log_scale);
    for (int l = c->L; l >= 1; l--) c->scale[l - 1] = (c->scale[l] * c->scale[l]) / (double)c->pr[l].q;
    c->tw_re = malloc(sizeof(double) * M); c->tw_im = malloc(sizeof(double) * M);
    c->zt_re = malloc(sizeof(double) * M); c->zt_im = malloc(sizeof(double) * M);
    for (int k = 0; k < M; k++) {
        double a = 2.0 * M_PI * (double)k / (double)M;
        c->tw_re[k] = cos(a); c->tw_im[k] = sin(a);
        double b = M_PI * (double)k / (double)N;
        c->zt_re[k] = cos(b); c->zt_im[k] = sin(b);
    }
    c->slot_t = malloc(sizeof(int) * M);
    u64 e = 1;
    for (int j = 0; j < M; j++) { c->slot_t[j] = (int)((e - 1) / 4); e = (e * 5) % (2 * (u64)N); }
    /* CDT over [-B, B] */
    int B = (int)ceil(sigma * 12.0);
    double tot = 0.0;
    for (int x = -B; x <= B; x++) tot += exp(-(double)x * (double)x / (2.0 * sigma * sigma));
    double acc = 0.0;
    c->cdt_b = B; c->cdt_n = 2 * B;
    for (int i = 0; i < 2 * B; i++) {
        int x = -B + i;
        acc += exp(-(double)x * (double)x / (2.0 * sigma * sigma));
        double v = (acc / tot) * 18446744073709551616.0;
        c->cdt[i] = v >= 18446744073709551615.0 ? ~(u64)0 : (u64)v;
    }
    /* secret */
    c->sk = calloc(N, sizeof(i64));
    u64 ctr = 0;
    for (int i = 0; i < hw; i++) {
        u64 pos;
        for (;;) { pos = mulhi(rng(seed, stream_id(DOM_SK, 0, 0), ctr++), (u64)N); if (!c->sk[pos]) break; }
        c->sk[pos] = (rng(seed, stream_id(DOM_SK, 0, 0), ctr++) & 1) ? 1 : -1;
    }
    c->sk_ntt = malloc(sizeof(u64) * (size_t)c->nall * N);
    for (int i = 0; i < c->nall; i++) {
        u64 *d = c->sk_ntt + (size_t)i * N;
        for (int k = 0; k < N; k++) d[k] = from_i64(c->sk[k], c->pr[i].q);
        ntt(c, &c->pr[i], d);
    }
    return c;
}

void orc_set_app_level(orc_ctx *c, int level) { c->app_L = level; }

void orc_destroy(orc_ctx *c) {
    if (!c) return;
    for (int i = 0; i < c->nall; i++) { free(c->pr[i].w); free(c->pr[i].ws); free(c->pr[i].iw); free(c->pr[i].iws); }
    free(c->tw_re); free(c->tw_im); free(c->zt_re); free(c->zt_im); free(c->slot_t);
    free(c->sk); free(c->sk_ntt);
    swkey_t *k = c->keys;
    while (k) { swkey_t *n = k->next; free(k->data); free(k); k = n; }
    free(c);
}

void orc_info(const orc_ctx *c, u64 *moduli, double *scales, u64 *psis) {
    for (int i = 0; i < c->nall; i++) { moduli[i] = c->pr[i].q; if (psis) psis[i] = c->pr[i].psi; }
    for (int l = 0; l <= c->L; l++) scales[l] = c->scale[l];
}

void orc_secret(const orc_ctx *c, i64 *out) { memcpy(out, c->sk, sizeof(i64) * c->N); }
int orc_cdt(const orc_ctx *c, u64 *out) { memcpy(out, c->cdt, sizeof(u64) * c->cdt_n); return c->cdt_n; }

/* ------------------------------------------------------------------ */
/* encoder (host, double; see header)                                  */
/* ------------------------------------------------------------------ */

static void fft(const orc_ctx *c, double *re, double *im, int inverse) {
    int M = c->N / 2, logM = c->logN - 1;
    for (int i = 0; i < M; i++) {
        int r = (int)brv((unsigned)i, logM);
        if (r > i) { double t = re[i]; re[i] = re[r]; re[r] = t; t = im[i]; im[i] = im[r]; im[r] = t; }
    }
    for (int len = 2; len <= M; len <<= 1) {
        int half = len >> 1, step = M / len;
        for (int i = 0; i < M; i += len) {
            for (int j = 0; j < half; j++) {
                double wr = c->tw_re[j * step];
                double wi = inverse ? -c->tw_im[j * step] : c->tw_im[j * step];
                double vr0 = re[i + j + half], vi0 = im[i + j + half];
                double vr = vr0 * wr - vi0 * wi;
                double vi = vr0 * wi + vi0 * wr;
                double ur = re[i + j], ui = im[i + j];
                re[i + j] = ur + vr; im[i + j] = ui + vi;
                re[i + j + half] = ur - vr; im[i + j + half] = ui - vi;
            }
        }
    }
}

/* slots (M complex) -> N integer coefficients at `scale`; returns 0 or -1 on overflow */
int orc_encode(const orc_ctx *c, const double *zr, const double *zi, double scale, i64 *coef) {
    int M = c->N / 2;
    double *re = malloc(sizeof(double) * M), *im = malloc(sizeof(double) * M);
    for (int j = 0; j < M; j++) { re[c->slot_t[j]] = zr[j]; im[c->slot_t[j]] = zi ? zi[j] : 0.0; }
    fft(c, re, im, 1);
    double inv = 1.0 / (double)M;
    int bad = 0;
    for (int k = 0; k < M; k++) {
        double wr = re[k] * inv, wi = im[k] * inv;
        /* u = w * conj(zeta^k) */
        double ur = wr * c->zt_re[k] + wi * c->zt_im[k];
        double ui = wi * c->zt_re[k] - wr * c->zt_im[k];
        double a = ur * scale, b = ui * scale;
        if (!(fabs(a) < 9.2e18) || !(fabs(b) < 9.2e18)) bad = 1;
        coef[k] = bad ? 0 : llrint(a);
        coef[k + M] = bad ? 0 : llrint(b);
    }
    free(re); free(im);
    return bad ? -1 : 0;
}

/* N real coefficients (already divided by scale) -> M complex slots */
void orc_decode_real(const orc_ctx *c, const double *m, double *zr, double *zi) {
    int M = c->N / 2;
    double *re = malloc(sizeof(double) * M), *im = malloc(sizeof(double) * M);
    for (int k = 0; k < M; k++) {
        double ur = m[k], ui = m[k + M];
        re[k] = ur * c->zt_re[k] - ui * c->zt_im[k];
        im[k] = ur * c->zt_im[k] + ui * c->zt_re[k];
    }
    fft(c, re, im, 0);
    for (int j = 0; j < M; j++) { zr[j] = re[c->slot_t[j]]; zi[j] = im[c->slot_t[j]]; }
    free(re); free(im);
}

/* ------------------------------------------------------------------ */
/* polynomial helpers (limb-major [nl][N])                             */
/* ------------------------------------------------------------------ */

static void coef_to_ntt(const orc_ctx *c, const i64 *coef, int nl, const int *limbs, u64 *out) {
    int N = c->N;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nl; i++) {
        const prime_t *p = &c->pr[limbs ? limbs[i] : i];
        u64 *d = out + (size_t)i * N;
        for (int k = 0; k < N; k++) d[k] = from_i64(coef[k], p->q);
        ntt(c, p, d);
    }
}

/* sample a uniform polynomial directly in NTT form over basis limbs `limbs` */
static void sample_uniform(const orc_ctx *c, u64 stream, int nl, const int *limbs, u64 *out) {
    int N = c->N;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nl; i++) {
        int li = limbs ? limbs[i] : i;
        u64 q = c->pr[li].q;
        u64 *d = out + (size_t)i * N;
        for (int k = 0; k < N; k++) d[k] = mulhi(rng(c->seed, stream, (u64)li * N + k), q);
    }
}

static void sample_error(const orc_ctx *c, u64 stream, i64 *e) {
    for (int k = 0; k < c->N; k++) e[k] = cdt_sample(c, rng(c->seed, stream, (u64)k));
}

/* ------------------------------------------------------------------ */
/* keys                                                                */
/* ------------------------------------------------------------------ */

static void automorph_coef_i64(int N, const i64 *in, u64 g, i64 *out) {
    for (int i = 0; i < N; i++) {
        u64 j = ((u64)i * g) % (2 * (u64)N);
        if (j < (u64)N) out[j] = in[i]; else out[j - N] = -in[i];
    }
}

static swkey_t *get_key(orc_ctx *c, int id) {
    for (swkey_t *k = c->keys; k; k = k->next) if (k->id == id) return k;
    int N = c->N, nall = c->nall, L = c->L;
    size_t limb = (size_t)N, poly = (size_t)nall * N;
    swkey_t *k = calloc(1, sizeof(swkey_t));
    k->id = id;
    k->data = malloc(sizeof(u64) * (size_t)c->dnum * 2 * poly);
    /* target secret s' in NTT form over all limbs */
    u64 *sp = malloc(sizeof(u64) * poly);
    if (id == 0) {
#pragma omp parallel for
        for (int i = 0; i < nall; i++)
            for (int j = 0; j < N; j++) sp[i * limb + j] = mulmod(c->sk_ntt[i * limb + j], c->sk_ntt[i * limb + j], &c->pr[i]);
    } else {
        i64 *t = malloc(sizeof(i64) * N);
        automorph_coef_i64(N, c->sk, (u64)id, t);
        coef_to_ntt(c, t, nall, NULL, sp);
        free(t);
    }
    i64 *e = malloc(sizeof(i64) * N);
    u64 *en = malloc(sizeof(u64) * poly);
    for (int j = 0; j < c->dnum; j++) {
        u64 *b = k->data + (size_t)(2 * j) * poly, *a = b + poly;
        sample_uniform(c, stream_id(DOM_KEY_A, (u64)id, (u64)j), nall, NULL, a);
        sample_error(c, stream_id(DOM_KEY_E, (u64)id, (u64)j), e);
        coef_to_ntt(c, e, nall, NULL, en);
        int lo = j * c->alpha, hi = lo + c->alpha;
        if (hi > L + 1) hi = L + 1;
#pragma omp parallel for
        for (int i = 0; i < nall; i++) {
            const prime_t *p = &c->pr[i];
            u64 Pm = 1;
            for (int t = 0; t < c->K; t++) Pm = mulmod(Pm, c->pr[L + 1 + t].q % p->q, p);
            int in_digit = (i >= lo && i < hi);
            for (int x = 0; x < N; x++) {
                size_t o = i * limb + x;
                u64 v = submod(en[o], mulmod(a[o], c->sk_ntt[o], p), p->q);
                if (in_digit) v = addmod(v, mulmod(Pm, sp[o], p), p->q);
                b[o] = v;
            }
        }
    }
    free(e); free(en); free(sp);
    k->next = c->keys;
    c->keys = k;
    return k;
}

/* debug accessor: copy key `id` ([dnum][2][nall][N]) */
void orc_key(orc_ctx *c, int id, u64 *out) {
    swkey_t *k = get_key(c, id);
    memcpy(out, k->data, sizeof(u64) * (size_t)c->dnum * 2 * c->nall * c->N);
}

/* ------------------------------------------------------------------ */
/* encryption                                                          */
/* ------------------------------------------------------------------ */

/* encrypt integer coefficients m at `level` with nonce; ct [2][level+1][N] */
void orc_encrypt_coef(const orc_ctx *c, const i64 *m, int level, u64 nonce, u64 *ct) {
    int N = c->N, nl = level + 1;
    size_t poly = (size_t)nl * N;
    u64 *c0 = ct, *c1 = ct + poly;
    sample_uniform(c, stream_id(DOM_ENC_A, nonce, 0), nl, NULL, c1);
    i64 *e = malloc(sizeof(i64) * N);
    sample_error(c, stream_id(DOM_ENC_E, nonce, 0), e);
    i64 *me = malloc(sizeof(i64) * N);
    for (int k = 0; k < N; k++) me[k] = m[k] + e[k];
    coef_to_ntt(c, me, nl, NULL, c0);
#pragma omp parallel for
    for (int i = 0; i < nl; i++) {
        const prime_t *p = &c->pr[i];
        for (int k = 0; k < N; k++) {
            size_t o = (size_t)i * N + k;
            c0[o] = submod(c0[o], mulmod(c1[o], c->sk_ntt[o], p), p->q);
        }
    }
    free(e); free(me);
}

int orc_encrypt(const orc_ctx *c, const double *zr, const double *zi, int level, u64 nonce, u64 *ct) {
    i64 *m = malloc(sizeof(i64) * c->N);
    int rc = orc_encode(c, zr, zi, c->scale[level], m);
    if (rc == 0) orc_encrypt_coef(c, m, level, nonce, ct);
    free(m);
    return rc;
}

/* plaintext residues (NTT form) of slots at `scale` over limbs 0..level */
int orc_encode_ntt(const orc_ctx *c, const double *zr, const double *zi, int level, double scale, u64 *pt) {
    i64 *m = malloc(sizeof(i64) * c->N);
    int rc = orc_encode(c, zr, zi, scale, m);
    if (rc == 0) coef_to_ntt(c, m, level + 1, NULL, pt);
    free(m);
    return rc;
}

/* decrypt to centred coefficients as doubles (two-prime CRT when level >= 1) */
static void decrypt_coef(const orc_ctx *c, const u64 *ct, int level, double *md) {
    int N = c->N, nl = level >= 1 ? 2 : 1;
    size_t poly = (size_t)(level + 1) * N;
    u64 *x = malloc(sizeof(u64) * nl * N);
    for (int i = 0; i < nl; i++) {
        const prime_t *p = &c->pr[i];
        for (int k = 0; k < N; k++) {
            size_t o = (size_t)i * N + k;
            x[o] = addmod(ct[o], mulmod(ct[poly + o], c->sk_ntt[o], p), p->q);
        }
        intt(c, p, x + (size_t)i * N);
    }
    u64 q0 = c->pr[0].q;
    for (int k = 0; k < N; k++) {
        u64 v0 = x[k];
        i64 x0 = v0 > (q0 - 1) / 2 ? (i64)v0 - (i64)q0 : (i64)v0;
        if (nl == 1) { md[k] = (double)x0; continue; }
        const prime_t *p1 = &c->pr[1];
        u64 q1 = p1->q;
        u64 d = submod(x[N + k], from_i64(x0, q1), q1);
        u64 kk = mulmod(d, invmod(q0 % q1, q1), p1);
        i64 kc = kk > (q1 - 1) / 2 ? (i64)kk - (i64)q1 : (i64)kk;
        md[k] = (double)x0 + (double)q0 * (double)kc;
    }
    free(x);
}

void orc_decrypt(const orc_ctx *c, const u64 *ct, int level, double *zr, double *zi) {
    int N = c->N;
    double *md = malloc(sizeof(double) * N);
    decrypt_coef(c, ct, level, md);
    double s = c->scale[level];
    for (int k = 0; k < N; k++) md[k] = md[k] / s;
    orc_decode_real(c, md, zr, zi);
    free(md);
}

/* refresh surrogate: decrypt (mod q0 / q0q1), rescale the message to the top
 * scale, re-encrypt at max level with `nonce`.  emulator.py:267-273 semantics. */
void orc_refresh(const orc_ctx *c, const u64 *ct, int level, u64 nonce, u64 *out) {
    int N = c->N;
    double *md = malloc(sizeof(double) * N);
    decrypt_coef(c, ct, level, md);
    double ratio = c->scale[c->app_L] / c->scale[level];
    i64 *m = malloc(sizeof(i64) * N);
    for (int k = 0; k < N; k++) m[k] = llrint(md[k] * ratio);
    orc_encrypt_coef(c, m, c->app_L, nonce, out);
    free(md); free(m);
}

/* ------------------------------------------------------------------ */
/* elementwise ops (ct layout [2][nl][N])                              */
/* ------------------------------------------------------------------ */

void orc_add(const orc_ctx *c, const u64 *a, const u64 *b, int level, int npoly_b, int negate_b, u64 *out) {
    int N = c->N, nl = level + 1;
    for (int s = 0; s < 2; s++)
        for (int i = 0; i < nl; i++) {
            u64 q = c->pr[i].q;
            for (int k = 0; k < N; k++) {
                size_t o = ((size_t)s * nl + i) * N + k;
                u64 y = (s < npoly_b) ? b[o] : 0;
                out[o] = negate_b ? submod(a[o], y, q) : addmod(a[o], y, q);
            }
        }
}

void orc_neg(const orc_ctx *c, const u64 *a, int level, u64 *out) {
    int N = c->N, nl = level + 1;
    for (int s = 0; s < 2; s++)
        for (int i = 0; i < nl; i++) {
            u64 q = c->pr[i].q;
            for (int k = 0; k < N; k++) {
                size_t o = ((size_t)s * nl + i) * N + k;
                out[o] = a[o] ? q - a[o] : 0;
            }
        }
}

/* constant pair per limb: first half of NTT slots gets cr + ci*I, second cr - ci*I */
static void const_pair(const orc_ctx *c, i64 cr, i64 ci, int i, u64 *lo, u64 *hi) {
    const prime_t *p = &c->pr[i];
    u64 r = from_i64(cr, p->q), im = mulmod(from_i64(ci, p->q), p->I, p);
    *lo = addmod(r, im, p->q);
    *hi = submod(r, im, p->q);
}

void orc_add_const(const orc_ctx *c, const u64 *a, int level, double re, double im, u64 *out) {
    int N = c->N, nl = level + 1;
    double s = c->scale[level];
    i64 cr = llrint(re * s), ci = llrint(im * s);
    memcpy(out, a, sizeof(u64) * 2 * nl * N);
    for (int i = 0; i < nl; i++) {
        u64 lo, hi;
        const_pair(c, cr, ci, i, &lo, &hi);
        u64 q = c->pr[i].q;
        for (int k = 0; k < N; k++) out[(size_t)i * N + k] = addmod(a[(size_t)i * N + k], k < N / 2 ? lo : hi, q);
    }
}

/* multiply by the integer pair (cr, ci) (no rescale) */
static void mul_int_pair(const orc_ctx *c, const u64 *a, int level, i64 cr, i64 ci, u64 *out) {
    int N = c->N, nl = level + 1;
    for (int i = 0; i < nl; i++) {
        u64 lo, hi;
        const_pair(c, cr, ci, i, &lo, &hi);
        const prime_t *p = &c->pr[i];
        for (int s = 0; s < 2; s++)
            for (int k = 0; k < N; k++) {
                size_t o = ((size_t)s * nl + i) * N + k;
                out[o] = mulmod(a[o], k < N / 2 ? lo : hi, p);
            }
    }
}

void orc_mul_i(const orc_ctx *c, const u64 *a, int level, u64 *out) { mul_int_pair(c, a, level, 0, 1, out); }

/* centred rescale of a [npoly][level+1][N] ciphertext to level-1 */
void orc_rescale(const orc_ctx *c, const u64 *a, int level, int npoly, u64 *out) {
    int N = c->N, nl = level + 1;
    const prime_t *pl = &c->pr[level];
    u64 ql = pl->q;
    u64 *x = malloc(sizeof(u64) * N);
    for (int s = 0; s < npoly; s++) {
        memcpy(x, a + ((size_t)s * nl + level) * N, sizeof(u64) * N);
        intt(c, pl, x);
#pragma omp parallel for
        for (int i = 0; i < level; i++) {
            const prime_t *p = &c->pr[i];
            u64 *y = malloc(sizeof(u64) * N);
            for (int k = 0; k < N; k++) {
                u64 v = x[k];
                y[k] = v > (ql - 1) / 2 ? submod(v % p->q, ql % p->q, p->q) : v % p->q;
            }
            ntt(c, p, y);
            u64 inv = invmod(ql % p->q, p->q);
            for (int k = 0; k < N; k++) {
                size_t i_in = ((size_t)s * nl + i) * N + k, i_out = ((size_t)s * level + i) * N + k;
                out[i_out] = mulmod(submod(a[i_in], y[k], p->q), inv, p);
            }
            free(y);
        }
    }
    free(x);
}

void orc_mul_const(const orc_ctx *c, const u64 *a, int level, double re, double im, u64 *out) {
    int nl = level + 1;
    double s = c->scale[level];
    u64 *t = malloc(sizeof(u64) * 2 * nl * c->N);
    mul_int_pair(c, a, level, llrint(re * s), llrint(im * s), t);
    orc_rescale(c, t, level, 2, out);
    free(t);
}

/* pt: [level+1][N] NTT residues encoded at scale[level] */
void orc_mul_pt(const orc_ctx *c, const u64 *a, const u64 *pt, int level, u64 *out) {
    int N = c->N, nl = level + 1;
    u64 *t = malloc(sizeof(u64) * 2 * nl * N);
    for (int s = 0; s < 2; s++)
#pragma omp parallel for
        for (int i = 0; i < nl; i++)
            for (int k = 0; k < N; k++) {
                size_t o = ((size_t)s * nl + i) * N + k;
                t[o] = mulmod(a[o], pt[(size_t)i * N + k], &c->pr[i]);
            }
    orc_rescale(c, t, level, 2, out);
    free(t);
}

/* ct x pt without the rescale: [2][level+1][N] at scale scale[level]^2 */
void orc_mul_pt_raw(const orc_ctx *c, const u64 *a, const u64 *pt, int level, u64 *out) {
    int N = c->N, nl = level + 1;
    for (int s = 0; s < 2; s++)
#pragma omp parallel for
        for (int i = 0; i < nl; i++)
            for (int k = 0; k < N; k++) {
                size_t o = ((size_t)s * nl + i) * N + k;
                out[o] = mulmod(a[o], pt[(size_t)i * N + k], &c->pr[i]);
            }
}

/* exact multiplication by a non-negative integer k (no rescale, no level) */
void orc_mul_int(const orc_ctx *c, const u64 *a, int level, u64 k, u64 *out) {
    int N = c->N, nl = level + 1;
    for (int s = 0; s < 2; s++)
        for (int i = 0; i < nl; i++) {
            const prime_t *p = &c->pr[i];
            u64 kk = k % p->q;
            for (int j = 0; j < N; j++) {
                size_t o = ((size_t)s * nl + i) * N + j;
                out[o] = mulmod(a[o], kk, p);
            }
        }
}

/* ModRaise (bootstrapping): a level-0 ciphertext [2][1][N]
 * -> [2][to+1][N]: each polynomial's coefficients, centred mod q0, lifted to
 * every prime q_0..q_to; the result decrypts to m + q0 * I(X), I small */
void orc_mod_raise(const orc_ctx *c, const u64 *a, int to, u64 *out) {
    int N = c->N, nl = to + 1;
    const prime_t *p0 = &c->pr[0];
    u64 q0 = p0->q;
    u64 *x = malloc(sizeof(u64) * N);
    for (int s = 0; s < 2; s++) {
        memcpy(x, a + (size_t)s * N, sizeof(u64) * N);
        intt(c, p0, x);
#pragma omp parallel for
        for (int i = 0; i < nl; i++) {
            const prime_t *p = &c->pr[i];
            u64 *y = out + ((size_t)s * nl + i) * N;
            for (int k = 0; k < N; k++) {
                u64 v = x[k];
                y[k] = v > (q0 - 1) / 2 ? submod(v % p->q, q0 % p->q, p->q) : v % p->q;
            }
            ntt(c, p, y);
        }
    }
    free(x);
}

void orc_add_pt(const orc_ctx *c, const u64 *a, const u64 *pt, int level, int negate, u64 *out) {
    orc_add(c, a, pt, level, 1, negate, out);
}

/* drop limbs: [2][from+1][N] -> [2][to+1][N] */
void orc_drop(const orc_ctx *c, const u64 *a, int from, int to, u64 *out) {
    size_t N = c->N;
    for (int s = 0; s < 2; s++)
        memcpy(out + (size_t)s * (to + 1) * N, a + (size_t)s * (from + 1) * N, sizeof(u64) * (to + 1) * N);
}

/* bring a level-`from` ciphertext to level `to` < from with canonical scale */
void orc_level_adjust(const orc_ctx *c, const u64 *a, int from, int to, u64 *out) {
    int N = c->N;
    u64 *d = malloc(sizeof(u64) * 2 * (to + 2) * N);
    orc_drop(c, a, from, to + 1, d);
    double s1 = c->scale[to + 1];
    i64 cst = llrint(s1 * (s1 / c->scale[from]));
    u64 *t = malloc(sizeof(u64) * 2 * (to + 2) * N);
    mul_int_pair(c, d, to + 1, cst, 0, t);
    orc_rescale(c, t, to + 1, 2, out);
    free(d); free(t);
}

/* ------------------------------------------------------------------ */
/* key switching                                                       */
/* ------------------------------------------------------------------ */

/* ModUp of d ([level+1][N], NTT form): up [beta][nt][N] in NTT form over
 * the target basis (Q_l then P); for target limbs inside digit j the value is
 * d itself.  Centred fast base conversion of the digit's INTT, scaled by
 * [(Q'/q_i)^-1]_{q_i}: each term y_a is taken in (-q_a/2, q_a/2], i.e.
 * sum_a y_a [Q'/q_a]_p - #{a : y_a > (q_a-1)/2} [Q']_p, so the lifted digit
 * has no constant bias (an uncentred digit's mean Q'/2 is amplified ~N-fold
 * in the slots by the key-switching error); then the forward
 * NTT on every non-digit target. */
static void ks_modup(orc_ctx *c, const u64 *d, int level, u64 *up) {
    int N = c->N, L = c->L, K = c->K, nl = level + 1;
    int nt = nl + K;
    int *tl = malloc(sizeof(int) * nt);
    for (int i = 0; i < nl; i++) tl[i] = i;
    for (int t = 0; t < K; t++) tl[nl + t] = L + 1 + t;
    int beta = (nl + c->alpha - 1) / c->alpha;
    u64 *x = malloc(sizeof(u64) * (size_t)c->alpha * N);
    for (int j = 0; j < beta; j++) {
        int lo = j * c->alpha, hi = lo + c->alpha;
        if (hi > nl) hi = nl;
        int na = hi - lo;
        /* y_i = INTT(d_i) * [(Q'/q_i)^-1]_{q_i} */
        for (int a = 0; a < na; a++) {
            int i = lo + a;
            const prime_t *p = &c->pr[i];
            memcpy(x + (size_t)a * N, d + (size_t)i * N, sizeof(u64) * N);
            intt(c, p, x + (size_t)a * N);
            u64 qh = 1;
            for (int b = lo; b < hi; b++) if (b != i) qh = mulmod(qh, c->pr[b].q % p->q, p);
            u64 inv = invmod(qh, p->q);
            for (int k = 0; k < N; k++) x[(size_t)a * N + k] = mulmod(x[(size_t)a * N + k], inv, p);
        }
        u64 *upj = up + (size_t)j * nt * N;
#pragma omp parallel for schedule(dynamic)
        for (int t = 0; t < nt; t++) {
            int li = tl[t];
            const prime_t *p = &c->pr[li];
            u64 *o = upj + (size_t)t * N;
            if (li >= lo && li < hi) { memcpy(o, d + (size_t)li * N, sizeof(u64) * N); continue; }
            u64 cf[MAXP], Qd = 1;
            for (int a = 0; a < na; a++) {
                u64 v = 1;
                for (int b = lo; b < hi; b++) if (b != lo + a) v = mulmod(v, c->pr[b].q % p->q, p);
                cf[a] = v;
                Qd = mulmod(Qd, c->pr[lo + a].q % p->q, p);
            }
            for (int k = 0; k < N; k++) {
                u128 s = 0;
                u64 cnt = 0;
                for (int a = 0; a < na; a++) {
                    const u64 y = x[(size_t)a * N + k];
                    s += (u128)y * cf[a];
                    cnt += y > (c->pr[lo + a].q - 1) / 2;
                }
                o[k] = submod(reduce128(s, p), mulmod(cnt, Qd, p), p->q);
            }
            ntt(c, p, o);
        }
    }
    free(x); free(tl);
}

/* Key inner product of the ModUp digits `up` with `key`, accumulated into
 * acc [2][nt][N] (extended basis Q_l P, NTT form; the caller zeroes it). */
static void ks_keyprod_acc(orc_ctx *c, const u64 *up, int level, swkey_t *key, u64 *acc) {
    int N = c->N, L = c->L, K = c->K, nall = c->nall, nl = level + 1;
    int nt = nl + K;
    int *tl = malloc(sizeof(int) * nt);
    for (int i = 0; i < nl; i++) tl[i] = i;
    for (int t = 0; t < K; t++) tl[nl + t] = L + 1 + t;
    int beta = (nl + c->alpha - 1) / c->alpha;
    size_t poly = (size_t)nt * N;
    for (int j = 0; j < beta; j++) {
        const u64 *upj = up + (size_t)j * poly;
        /* inner product with digit j of the key */
        const u64 *kb = key->data + (size_t)(2 * j) * nall * N, *ka = kb + (size_t)nall * N;
#pragma omp parallel for
        for (int t = 0; t < nt; t++) {
            int li = tl[t];
            const prime_t *p = &c->pr[li];
            for (int k = 0; k < N; k++) {
                size_t o = (size_t)t * N + k, ko = (size_t)li * N + k;
                acc[o] = addmod(acc[o], mulmod(upj[o], kb[ko], p), p->q);
                acc[poly + o] = addmod(acc[poly + o], mulmod(upj[o], ka[ko], p), p->q);
            }
        }
    }
    free(tl);
}

/* ModDown by P of acc [2][nt][N] (NTT form): out [2][level+1][N]. */
static void ks_moddown(orc_ctx *c, const u64 *acc, int level, u64 *out) {
    int N = c->N, L = c->L, K = c->K, nl = level + 1;
    int nt = nl + K;
    size_t poly = (size_t)nt * N;
    for (int s = 0; s < 2; s++) {
        const u64 *A = acc + (size_t)s * poly;
        u64 *y = malloc(sizeof(u64) * (size_t)K * N);
        for (int t = 0; t < K; t++) {
            const prime_t *p = &c->pr[L + 1 + t];
            memcpy(y + (size_t)t * N, A + (size_t)(nl + t) * N, sizeof(u64) * N);
            intt(c, p, y + (size_t)t * N);
            u64 ph = 1;
            for (int b = 0; b < K; b++) if (b != t) ph = mulmod(ph, c->pr[L + 1 + b].q % p->q, p);
            u64 inv = invmod(ph, p->q);
            for (int k = 0; k < N; k++) y[(size_t)t * N + k] = mulmod(y[(size_t)t * N + k], inv, p);
        }
#pragma omp parallel for
        for (int i = 0; i < nl; i++) {
            const prime_t *p = &c->pr[i];
            u64 cf[MAXP], Pm = 1;
            for (int t = 0; t < K; t++) {
                u64 v = 1;
                for (int b = 0; b < K; b++) if (b != t) v = mulmod(v, c->pr[L + 1 + b].q % p->q, p);
                cf[t] = v;
                Pm = mulmod(Pm, c->pr[L + 1 + t].q % p->q, p);
            }
            u64 pinv = invmod(Pm, p->q);
            u64 *w = malloc(sizeof(u64) * N);
            /* centred conversion of the P part (as in ks_modup) */
            for (int k = 0; k < N; k++) {
                u128 sacc = 0;
                u64 cnt = 0;
                for (int t = 0; t < K; t++) {
                    const u64 v = y[(size_t)t * N + k];
                    sacc += (u128)v * cf[t];
                    cnt += v > (c->pr[L + 1 + t].q - 1) / 2;
                }
                w[k] = submod(reduce128(sacc, p), mulmod(cnt, Pm, p), p->q);
            }
            ntt(c, p, w);
            for (int k = 0; k < N; k++)
                out[((size_t)s * nl + i) * N + k] = mulmod(submod(A[(size_t)i * N + k], w[k], p->q), pinv, p);
            free(w);
        }
        free(y);
    }
}

static size_t modup_words(const orc_ctx *c, int level);

/* Merged ModDown + rescale: acc [2][nt][N] (NTT form) holds
 * X over q_0..q_l and P; out [2][level][N] = (X - [X]_D) / D at level - 1,
 * D = q_l * P, with [X]_D lifted from the basis B = (q_l, p_1, .., p_K) by the
 * centred fast base conversion of ks_moddown.  B's limbs are acc's limbs
 * level .. level + K (contiguous).  One rounding instead of ModDown's and the
 * rescale's two. */
static void ks_moddown_rescale(orc_ctx *c, const u64 *acc, int level, u64 *out) {
    int N = c->N, L = c->L, K = c->K, nl = level + 1;
    int nt = nl + K, nb = K + 1;
    size_t poly = (size_t)nt * N;
    int bp[MAXP];
    bp[0] = level;
    for (int t = 0; t < K; t++) bp[1 + t] = L + 1 + t;
    for (int s = 0; s < 2; s++) {
        const u64 *A = acc + (size_t)s * poly;
        u64 *y = malloc(sizeof(u64) * (size_t)nb * N);
        for (int t = 0; t < nb; t++) {
            const prime_t *p = &c->pr[bp[t]];
            memcpy(y + (size_t)t * N, A + (size_t)(level + t) * N, sizeof(u64) * N);
            intt(c, p, y + (size_t)t * N);
            u64 dh = 1;
            for (int b = 0; b < nb; b++) if (b != t) dh = mulmod(dh, c->pr[bp[b]].q % p->q, p);
            u64 inv = invmod(dh, p->q);
            for (int k = 0; k < N; k++) y[(size_t)t * N + k] = mulmod(y[(size_t)t * N + k], inv, p);
        }
#pragma omp parallel for
        for (int i = 0; i < level; i++) {
            const prime_t *p = &c->pr[i];
            u64 cf[MAXP], Dm = 1;
            for (int t = 0; t < nb; t++) {
                u64 v = 1;
                for (int b = 0; b < nb; b++) if (b != t) v = mulmod(v, c->pr[bp[b]].q % p->q, p);
                cf[t] = v;
                Dm = mulmod(Dm, c->pr[bp[t]].q % p->q, p);
            }
            u64 dinv = invmod(Dm, p->q);
            u64 *w = malloc(sizeof(u64) * N);
            for (int k = 0; k < N; k++) {
                u128 sacc = 0;
                u64 cnt = 0;
                for (int t = 0; t < nb; t++) {
                    const u64 v = y[(size_t)t * N + k];
                    sacc += (u128)v * cf[t];
                    cnt += v > (c->pr[bp[t]].q - 1) / 2;
                }
                w[k] = submod(reduce128(sacc, p), mulmod(cnt, Dm, p), p->q);
            }
            ntt(c, p, w);
            for (int k = 0; k < N; k++)
                out[((size_t)s * level + i) * N + k] = mulmod(submod(A[(size_t)i * N + k], w[k], p->q), dinv, p);
            free(w);
        }
        free(y);
    }
}

/* Relinearisation + rescale of a tensor d = (d0, d1, d2) at `level` in one
 * pass: X = P * (d0, d1) + <ModUp(d2), relin key> in the
 * extended basis, then the merged ModDown + rescale: out at level - 1.
 * Application levels only (level <= app_L). */
static void keyswitch(orc_ctx *c, const u64 *d, int level, swkey_t *key, u64 *out);

static void relin_rescale(orc_ctx *c, const u64 *d, int level, u64 *out) {
    int N = c->N, L = c->L, K = c->K, nl = level + 1, nt = nl + K;
    size_t poly = (size_t)nl * N, epoly = (size_t)nt * N;
    swkey_t *key = get_key(c, 0);
    if (level > c->app_L) {
        /* bootstrapping levels keep ModDown and the exact centred rescale apart:
         * the merged conversion's rounding (a sum of K + 1 centred terms
         * instead of one) is ~2.3x larger, and EvalMod's precision is bound by
         * exactly that rounding (measured: 5.4e-4 -> 1.1e-3 per bootstrap) */
        u64 *t = malloc(sizeof(u64) * 2 * poly), *ks = malloc(sizeof(u64) * 2 * poly);
        keyswitch(c, d + 2 * poly, level, key, ks);
        for (size_t o = 0; o < 2 * poly; o++) t[o] = addmod(d[o], ks[o], c->pr[(o % poly) / N].q);
        orc_rescale(c, t, level, 2, out);
        free(t); free(ks);
        return;
    }
    u64 *up = malloc(sizeof(u64) * modup_words(c, level));
    ks_modup(c, d + 2 * poly, level, up);
    u64 *acc = calloc(2 * epoly, sizeof(u64));
    ks_keyprod_acc(c, up, level, key, acc);
    for (int i = 0; i < nl; i++) {
        const prime_t *p = &c->pr[i];
        u64 Pm = 1;
        for (int t = 0; t < K; t++) Pm = mulmod(Pm, c->pr[L + 1 + t].q % p->q, p);
        for (int k = 0; k < N; k++) {
            size_t o = (size_t)i * N + k;
            acc[o] = addmod(acc[o], mulmod(d[o], Pm, p), p->q);
            acc[epoly + o] = addmod(acc[epoly + o], mulmod(d[poly + o], Pm, p), p->q);
        }
    }
    ks_moddown_rescale(c, acc, level, out);
    free(up); free(acc);
}

/* Key inner product of the ModUp digits `up` with `key`, then ModDown by P:
 * out [2][level+1][N] = (k0, k1). */
static void ks_keyprod_moddown(orc_ctx *c, const u64 *up, int level, swkey_t *key, u64 *out) {
    size_t poly = (size_t)(level + 1 + c->K) * c->N;
    u64 *acc = calloc(2 * poly, sizeof(u64));
    ks_keyprod_acc(c, up, level, key, acc);
    ks_moddown(c, acc, level, out);
    free(acc);
}

static size_t modup_words(const orc_ctx *c, int level) {
    int nl = level + 1, beta = (nl + c->alpha - 1) / c->alpha;
    return (size_t)beta * (nl + c->K) * c->N;
}

/* d: [level+1][N] NTT; out: [2][level+1][N] with (k0, k1) */
static void keyswitch(orc_ctx *c, const u64 *d, int level, swkey_t *key, u64 *out) {
    u64 *up = malloc(sizeof(u64) * modup_words(c, level));
    ks_modup(c, d, level, up);
    ks_keyprod_moddown(c, up, level, key, out);
    free(up);
}

static void automorph_ntt(const orc_ctx *c, const u64 *in, u64 g, int nl, u64 *out) {
    int N = c->N, logN = c->logN;
    u64 twoN = 2 * (u64)N;
    for (int j = 0; j < N; j++) {
        u64 e = 2 * (u64)brv((unsigned)j, logN) + 1;
        u64 e2 = (e * g) % twoN;
        unsigned src = brv((unsigned)((e2 - 1) / 2), logN);
        for (int i = 0; i < nl; i++) out[(size_t)i * N + j] = in[(size_t)i * N + src];
    }
}

/* rotate / conjugate by galois element g; ct [2][level+1][N] */
void orc_automorph(orc_ctx *c, const u64 *a, int level, u64 g, u64 *out) {
    int N = c->N, nl = level + 1;
    size_t poly = (size_t)nl * N;
    swkey_t *key = get_key(c, (int)g);
    u64 *s = malloc(sizeof(u64) * 2 * poly);
    automorph_ntt(c, a, g, nl, s);
    automorph_ntt(c, a + poly, g, nl, s + poly);
    u64 *ks = malloc(sizeof(u64) * 2 * poly);
    keyswitch(c, s + poly, level, key, ks);
    for (int i = 0; i < nl; i++) {
        u64 q = c->pr[i].q;
        for (int k = 0; k < N; k++) {
            size_t o = (size_t)i * N + k;
            out[o] = addmod(s[o], ks[o], q);
            out[poly + o] = ks[poly + o];
        }
    }
    free(s); free(ks);
}

u64 orc_galois_rot(const orc_ctx *c, i64 r) {
    u64 M = (u64)c->N / 2, twoN = 2 * (u64)c->N;
    u64 rr = (u64)(((r % (i64)M) + (i64)M) % (i64)M);
    return powmod(5, rr, twoN);
}

/* tensor, then relinearisation + rescale in one pass (relin_rescale); a, b at the same level */
void orc_mult(orc_ctx *c, const u64 *a, const u64 *b, int level, u64 *out) {
    int N = c->N, nl = level + 1;
    size_t poly = (size_t)nl * N;
    u64 *d = malloc(sizeof(u64) * 3 * poly);
#pragma omp parallel for
    for (int i = 0; i < nl; i++) {
        const prime_t *p = &c->pr[i];
        for (int k = 0; k < N; k++) {
            size_t o = (size_t)i * N + k;
            u64 a0 = a[o], a1 = a[poly + o], b0 = b[o], b1 = b[poly + o];
            d[o] = mulmod(a0, b0, p);
            d[poly + o] = reduce128((u128)a0 * b1 + (u128)a1 * b0, p);
            d[2 * poly + o] = mulmod(a1, b1, p);
        }
    }
    relin_rescale(c, d, level, out);
    free(d);
}

/* Hoisted rotations: one ModUp of c1 shared by every
 * Galois element g_r.  The automorphism is a permutation of NTT indices on
 * every limb, so sigma_g applied to the extended-basis digits is a valid
 * ModUp of sigma_g(c1) (the base-conversion overflow u*D_j becomes
 * sigma_g(u)*D_j); the result is a different, equally valid key switch, so
 * residues differ from orc_automorph.  out_r = (sigma(c0) + KS0, KS1). */
void orc_rotate_hoisted(orc_ctx *c, const u64 *a, int level, const u64 *gs, int ng, u64 *outs) {
    int N = c->N, nl = level + 1, nt = nl + c->K;
    int beta = (nl + c->alpha - 1) / c->alpha;
    size_t poly = (size_t)nl * N, mw = modup_words(c, level);
    u64 *up = malloc(sizeof(u64) * mw);
    ks_modup(c, a + poly, level, up);
    u64 *ups = malloc(sizeof(u64) * mw);
    u64 *c0 = malloc(sizeof(u64) * poly);
    u64 *ks = malloc(sizeof(u64) * 2 * poly);
    for (int r = 0; r < ng; r++) {
        swkey_t *key = get_key(c, (int)gs[r]);
        for (int j = 0; j < beta; j++)
            automorph_ntt(c, up + (size_t)j * nt * N, gs[r], nt, ups + (size_t)j * nt * N);
        ks_keyprod_moddown(c, ups, level, key, ks);
        automorph_ntt(c, a, gs[r], nl, c0);
        u64 *o = outs + (size_t)r * 2 * poly;
        for (int i = 0; i < nl; i++) {
            u64 q = c->pr[i].q;
            for (int k = 0; k < N; k++) {
                size_t e = (size_t)i * N + k;
                o[e] = addmod(c0[e], ks[e], q);
                o[poly + e] = ks[poly + e];
            }
        }
    }
    free(up); free(ups); free(c0); free(ks);
}

/* Rotate-and-sum stage (radix ladders): out = a + sum_r
 * sigma_{g_r}(a) with one ModUp of c1 (digits permuted per Galois element, as
 * in orc_rotate_hoisted), the key inner products of all ng rotations summed
 * in the extended basis Q_l P and one ModDown:
 *   out0 = c0 + sum_r sigma_r(c0) + ModDown(sum_r <sigma_r(up), key_r>)_0
 *   out1 = c1 +                     ModDown(sum_r <sigma_r(up), key_r>)_1 */
void orc_rotsum(orc_ctx *c, const u64 *a, int level, const u64 *gs, int ng, u64 *out) {
    int N = c->N, nl = level + 1, nt = nl + c->K;
    int beta = (nl + c->alpha - 1) / c->alpha;
    size_t poly = (size_t)nl * N, mw = modup_words(c, level);
    u64 *up = malloc(sizeof(u64) * mw);
    ks_modup(c, a + poly, level, up);
    u64 *ups = malloc(sizeof(u64) * mw);
    u64 *c0 = malloc(sizeof(u64) * poly);
    u64 *acc = calloc(2 * (size_t)nt * N, sizeof(u64));
    u64 *s0 = malloc(sizeof(u64) * poly);
    memcpy(s0, a, sizeof(u64) * poly);
    for (int r = 0; r < ng; r++) {
        swkey_t *key = get_key(c, (int)gs[r]);
        for (int j = 0; j < beta; j++)
            automorph_ntt(c, up + (size_t)j * nt * N, gs[r], nt, ups + (size_t)j * nt * N);
        ks_keyprod_acc(c, ups, level, key, acc);
        automorph_ntt(c, a, gs[r], nl, c0);
        for (int i = 0; i < nl; i++) {
            u64 q = c->pr[i].q;
            for (int k = 0; k < N; k++) {
                size_t e = (size_t)i * N + k;
                s0[e] = addmod(s0[e], c0[e], q);
            }
        }
    }
    u64 *ks = malloc(sizeof(u64) * 2 * poly);
    ks_moddown(c, acc, level, ks);
    for (int i = 0; i < nl; i++) {
        u64 q = c->pr[i].q;
        for (int k = 0; k < N; k++) {
            size_t e = (size_t)i * N + k;
            out[e] = addmod(s0[e], ks[e], q);
            out[poly + e] = addmod(a[poly + e], ks[poly + e], q);
        }
    }
    free(up); free(ups); free(c0); free(acc); free(s0); free(ks);
}

/* Sum of n ct x ct products with one relinearisation and one rescale:
 * d = sum_q tensor(a_q, b_q) (component-wise mod q), then relin_rescale.  as / bs: n ciphertexts [2][level+1][N] each,
 * contiguous. */
void orc_mult_sum(orc_ctx *c, const u64 *as, const u64 *bs, int n, int level, u64 *out) {
    int N = c->N, nl = level + 1;
    size_t poly = (size_t)nl * N;
    u64 *d = calloc(3 * poly, sizeof(u64));
    for (int q = 0; q < n; q++) {
        const u64 *a = as + (size_t)q * 2 * poly, *b = bs + (size_t)q * 2 * poly;
#pragma omp parallel for
        for (int i = 0; i < nl; i++) {
            const prime_t *p = &c->pr[i];
            for (int k = 0; k < N; k++) {
                size_t o = (size_t)i * N + k;
                u64 a0 = a[o], a1 = a[poly + o], b0 = b[o], b1 = b[poly + o];
                d[o] = addmod(d[o], mulmod(a0, b0, p), p->q);
                d[poly + o] = addmod(d[poly + o], reduce128((u128)a0 * b1 + (u128)a1 * b0, p), p->q);
                d[2 * poly + o] = addmod(d[2 * poly + o], mulmod(a1, b1, p), p->q);
            }
        }
    }
    relin_rescale(c, d, level, out);
    free(d);
}

/* ------------------------------------------------------------------ */
/* raw KATs                                                            */
/* ------------------------------------------------------------------ */

void orc_ntt_limb(const orc_ctx *c, int limb, u64 *a, int inverse) {
    if (inverse) intt(c, &c->pr[limb], a); else ntt(c, &c->pr[limb], a);
}
u64 orc_mulmod(const orc_ctx *c, int limb, u64 a, u64 b) { return mulmod(a, b, &c->pr[limb]); }
u64 orc_rng(u64 seed, u64 stream, u64 ctr) { return rng(seed, stream, ctr); }
