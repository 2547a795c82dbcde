// Fused hybrid key switching and rescale for split-pass rings (N >= 2^14).
//
// Per key switch of d = sigma(c1) at level l (nl = l+1 limbs, nt = nl + K,
// beta digits of alpha primes), the unfused pipeline makes ~15 launches and
// round-trips every ModUp / ModDown limb through HBM three times.  Here:
//
//   1. INTT of d, gathering sigma on the fly, final scale N^-1 * (Q'/q_i)^-1
//      folded into one Shoup constant             -> Y    (2 launches)
//   2. A: column pass of the forward NTT of every non-digit limb, whose
//      first-round loads compute the fast base conversion
//      sum_a Y_a * [Q'/q_a]_{p_t} on the fly          -> I    (1 launch)
//   3. B: chunk pass of those NTTs (batched, lazy outputs), then the
//      streaming key product: one thread per coefficient (pair) of target
//      limb t reads every digit's NTT output (or, for t inside the digit,
//      sigma(d) itself), multiplies with the key words held in registers and
//      accumulates (128-bit integer or exact FP64); one reduction per output.
//      (A form with the key product inside the chunk pass's stores was
//      measured slower and removed.)               -> ACC  (2 launches)
//   4. INTT of ACC's P limbs, final scale N^-1 * (P/p)^-1  (2 launches)
//   5. D: column pass of the ModDown NTT with the P->Q conversion in its
//      loads                                           -> Wt   (1 launch)
//   6. E: chunk pass whose stores compute (ACC - W) * P^-1 + addend, the
//      addend being sigma(c0) (gathered) or the tensor's (d0, d1)
//                                                      -> out  (1 launch)
//
// Every step is exact modular arithmetic, so the residues equal the
// unfused path and the oracle bit for bit.
#include <cstdlib>
#include <type_traits>

#include "evaluator.h"
#include "kernels.cuh"
#include "ntt_pass.cuh"

namespace hc {

#ifndef HC_CH_SUBS
#define HC_CH_SUBS 2   // 128-thread CTAs: finer last wave (measured 4 -> 2: -3 % kernel time)
#endif
constexpr int CH_LOG = 9, CH_SUBS = HC_CH_SUBS;   // chunk pass: 512-point, CH_SUBS per CTA

constexpr int KS_MAXJOBS = 256;   // (digit, target) column-pass jobs of one ModUp (dnum <= 8)
struct KsJobs {
    int n;
    unsigned char digit[KS_MAXJOBS];
    unsigned char t[KS_MAXJOBS];
};

struct KsGeo {
    int level, nl, nt, L, K, alpha, dnum, nall, beta, logN, N1;
    // ModDown: the dropped basis is ACC's limbs mdf .. mdf + nk - 1 and the
    // result has nout limbs: (nl, K, nl) for the division by P; (nl - 1, K + 1,
    // nl - 1) for the merged ModDown + rescale by q_l P of a ct x ct product
    int mdf, nk, nout;
    __host__ __device__ int prime(int t) const { return t <= level ? t : L + 1 + (t - level - 1); }
    // per-key-switch strides of the batched intermediates (words)
    __host__ __device__ size_t y_stride() const { return (size_t)nl << logN; }            // Y   [nl][N]
    __host__ __device__ size_t i_stride() const { return (size_t)beta * nt << logN; }     // I   [beta][nt][N]
    __host__ __device__ size_t acc_stride() const { return (size_t)2 * nt << logN; }      // ACC [2][nt][N]
    __host__ __device__ size_t w_stride() const { return (size_t)2 * nl << logN; }        // Wt  [2][nl][N]
};

// The key switches of one batched pipeline: all at the same level and read
// through the same Galois element; each has its own input, output, addends
// and switching key (equal keys are read once by the key product).
//
// Hoisted form (several Galois elements applied to one input): the ModUp
// stage runs once per distinct input (no gather), and entry b of the tail
// reads its input's digits and c1 through its own element ugal[b].
struct KsBatch {
    int nb;
    const u64* d[KS_MAXB];      // c1 source (NTT form), read through ugal[b] or the pipeline's gal
    const u64* up[KS_MAXB];     // ModUp digits of this entry's input ([beta][nt][N])
    u64* out[KS_MAXB];          // [2][nl][N]
    const u64* add[KS_MAXB];    // [add_npoly][nl][N] addend (read through agal[b]) or null
    const u64* add2[KS_MAXB];   // [2][nl][N] second addend (ladder step) or null
    const u64* key[KS_MAXB];    // [dnum][2][nall][N]
    u64 ugal[KS_MAXB];          // hoisted: Galois element gathered over up[b] and d[b] (0 = none)
    u64 agal[KS_MAXB];          // Galois element the addend is read through (0 = none)
};

// ---- A: ModUp conversion fused into the column pass --------------------------

// Conversion constants live in registers and the per-limb base pointers are
// formed once, so each converted element costs NA Shoup products and loads.
// Centred conversion: the inputs arrive shifted, y'' = y + h_a
// mod q_a with h_a = (q_a - 1) / 2 (the producing INTT's store adds it), so the
// centred value is y'' - h_a and sum_a (y''_a - h_a) [Q'/q_a]_p starts from
// the per-(digit, target) constant cc = [-sum_a h_a [Q'/q_a]_p]_p: no
// per-term comparison.
template <int NA>
struct LdModup {
    const u64* __restrict__ y[NA];   // shifted Y limbs of the digit, coefficient form, pre-scaled by (Q'/q_a)^-1
    u64 w[NA], ws[NA];               // [Q'/q_a]_p and Shoup companions (0 for an inert term)
    u64 cc;                          // [-sum_a h_a [Q'/q_a]_p]_p
    int na;
    u64 p;
    // Terms a >= na are inert (w = ws = 0) and their pointer is a valid
    // limb, so every load is unconditional: the NA loads of an element issue
    // together instead of one load -> use chain per term.
    __device__ __forceinline__ u64 operator()(size_t k) const {
        u64 v[NA];
#pragma unroll
        for (int a = 0; a < NA; a++) v[a] = __ldg(y[a] + k);
        u64 acc = cc;
#pragma unroll
        for (int a = 0; a < NA; a++) acc += mul_shoup_lazy(v[a], w[a], ws[a], p);
        return acc;   // < (2 * NA + 1) * p: the pass's input bound
    }
    __device__ __forceinline__ void load8(size_t k, u64* x) const {
#pragma unroll
        for (int e = 0; e < 8; e++) x[e] = (*this)(k + e);
    }
};

#ifndef KS_PMB_CHAIN
#define KS_PMB_CHAIN PASS_MIN_BLOCKS   // register budget of the column passes of a lone key switch (grid z = 1)
#endif
#ifndef KS_COLS_PMB
#define KS_COLS_PMB PASS_MIN_BLOCKS    // register budget of the batched conversion column passes
#endif
template <int LOGSZ, int SUBS, int NA, int PMB = KS_COLS_PMB>
__global__ void __launch_bounds__(PassGeo<LOGSZ, MODE_COLS, SUBS>::THREADS, PMB)
    ks_modup_cols(KsJobs jobs, KsGeo g, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ Y, const u64* __restrict__ modup_tab,
                  const u64* __restrict__ cc_tab, u64* __restrict__ I) {
    pdl_trigger();
    extern __shared__ u64 sm[];
    const int job = blockIdx.y;
    const int j = jobs.digit[job], t = jobs.t[job];
    const int pi = g.prime(t);
    const size_t N = (size_t)1 << g.logN;
    const int lo = j * g.alpha;
    const int hi = min(lo + g.alpha, g.nl);
    const PrimeDev P = primes[pi];
    const u64 p = P.q;
    Y += blockIdx.z * g.y_stride();
    I += blockIdx.z * g.i_stride();
    LdModup<NA> ld;
    ld.na = hi - lo;
    ld.p = p;
    const u64* cf = modup_tab + (((size_t)(g.level * g.dnum + j) * g.alpha) * g.nall + pi) * 2;
    ld.cc = cc_tab[(size_t)(g.level * g.dnum + j) * g.nall + pi];
#pragma unroll
    for (int a = 0; a < NA; a++) {
        const bool on = a < ld.na;
        const int aa = on ? a : 0;
        ld.y[a] = Y + (size_t)(lo + aa) * N;
        ld.w[a] = on ? cf[(size_t)aa * g.nall * 2] : 0;
        ld.ws[a] = on ? cf[(size_t)aa * g.nall * 2 + 1] : 0;
    }
    StPlain<false, false> st{I + ((size_t)j * g.nt + t) * N, p, 0, 0};
    PassGeo<LOGSZ, MODE_COLS, SUBS> G;
    G.init(g.N1);
    const ulonglong2* TW = tw + ((size_t)pi << g.logN);
    ulonglong2* twsm = PassGeo<LOGSZ, MODE_COLS, SUBS>::twsm_of(sm);
    stage_twiddles(G, twsm, TW, g.N1);
    pdl_wait();   // everything above reads context-lifetime tables only
    ntt_pass<LOGSZ, MODE_COLS, SUBS, false, 2 * NA + 1, BOUND_LIM>(G, sm, TW, P, ld, st, twsm, true);
}

constexpr int KP_MAXB = 8;   // digits handled by the key product (dnum <= 8; instantiated for 4 and 8)
#ifndef KP_PAIRB
#define KP_PAIRB 2           // batches of at least this many key switches take coefficient pairs
#endif
#ifndef KP_MINB
#define KP_MINB 3            // resident 256-thread CTAs per SM the key product is register-budgeted for (2: 30.95, 3: 30.82, 4: 31.10 ms/pair)
#endif

// ---- B (split form): streaming key inner product over NTT-form digits -----
// UP[j][t] holds NTT(conv_j(t)) for t outside digit j; inside the digit the
// value is sigma(d)[t] itself, gathered on the fly.  Grid y = target limb t
// (prime constants and the digit layout uniform per CTA); each thread owns
// a pair of coefficients (16-byte accesses) for every key switch of the
// batch, with the key words held in registers while the key does not change.

// E coefficients per thread (1 or 2; pairs use 16-byte accesses)
template <int E>
__device__ __forceinline__ void kp_load(const u64* __restrict__ base, size_t k, u64 gal_or_zero, int logN, u64* v) {
    if (gal_or_zero) {
#pragma unroll
        for (int e = 0; e < E; e++) v[e] = base[galois_src((unsigned)(k + e), logN, gal_or_zero)];
    } else if (E == 2) {
        const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(base + k);
        v[0] = w.x;
        v[E - 1] = w.y;
    } else {
        v[0] = base[k];
    }
}

// The batch loop for one arithmetic (FP64 for primes below 2^46, else 128-bit
// integer MACs; uniform per CTA): key words converted once per key, not per
// batch entry.  (Prefetching entry b + 1's digits needs 127 registers; at two
// resident CTAs it measured slower, 5.8 -> 6.6 ms per pair.)
template <int E, bool FP, int MB>
__device__ __forceinline__ void kp_run(const KsGeo& g, const PrimeDev& P, int t, int pi, int dig, size_t k, u64 gal,
                                       const KsBatch& kb, u64* __restrict__ acc) {
    using KW = typename std::conditional<FP, double, u64>::type;
    const size_t N = (size_t)1 << g.logN;
    const size_t kstride = (size_t)g.nall * N;
    KW kbv[MB][E], kav[MB][E];
    auto load_x = [&](int b, u64 (&x)[MB][E]) {
        const u64* up = kb.up[b];
        const u64 ug = kb.ugal[b];
#pragma unroll
        for (int j = 0; j < MB; j++) {
            if (j >= g.beta) break;
            if (j == dig) kp_load<E>(kb.d[b] + (size_t)t * N, k, ug ? ug : gal, g.logN, x[j]);
            else kp_load<E>(up + ((size_t)j * g.nt + t) * N, k, ug, g.logN, x[j]);
        }
    };
    const u64* kprev = nullptr;
    for (int b = 0; b < kb.nb; b++) {
        if (kb.key[b] != kprev) {
            kprev = kb.key[b];
#pragma unroll
            for (int j = 0; j < MB; j++) {
                if (j >= g.beta) break;
                const u64* kp = kprev + ((size_t)(2 * j) * g.nall + pi) * N;
                u64 wb[E], wa[E];
                kp_load<E>(kp, k, 0, g.logN, wb);
                kp_load<E>(kp + kstride, k, 0, g.logN, wa);
#pragma unroll
                for (int e = 0; e < E; e++) {
                    if constexpr (FP) {
                        kbv[j][e] = fp_word(wb[e]);
                        kav[j][e] = fp_word(wa[e]);
                    } else {
                        kbv[j][e] = wb[e];
                        kav[j][e] = wa[e];
                    }
                }
            }
        }
        u64 xc[MB][E];
        load_x(b, xc);
        u64 ob[E], oa[E];
#pragma unroll
        for (int e = 0; e < E; e++) {
            if constexpr (FP) {
                // each term exact and centered (|r| < 0.6q), the sum of <= 4
                // reduced once; digits are lazy words below 16q < 2^50
                double sb = 0, sa = 0;
#pragma unroll
                for (int j = 0; j < MB; j++) {
                    if (j >= g.beta) break;
                    const double y = fp_word(xc[j][e]);
                    sb = __dadd_rn(sb, fp_mulmod(y, kbv[j][e], P.qd, P.qinv));
                    sa = __dadd_rn(sa, fp_mulmod(y, kav[j][e], P.qd, P.qinv));
                }
                ob[e] = fp_canon(sb, P.qd, P.qinv);
                oa[e] = fp_canon(sa, P.qd, P.qinv);
            } else {
                U128 b0 = {0, 0}, a0 = {0, 0};
#pragma unroll
                for (int j = 0; j < MB; j++) {
                    if (j >= g.beta) break;
                    mac128(b0, xc[j][e], kbv[j][e]);
                    mac128(a0, xc[j][e], kav[j][e]);
                }
                ob[e] = reduce128(b0.hi, b0.lo, P);
                oa[e] = reduce128(a0.hi, a0.lo, P);
            }
        }
        u64* ab = acc + b * g.acc_stride();
        if (E == 2) {
            *reinterpret_cast<ulonglong2*>(ab + (size_t)t * N + k) = make_ulonglong2(ob[0], ob[E - 1]);
            *reinterpret_cast<ulonglong2*>(ab + ((size_t)g.nt + t) * N + k) = make_ulonglong2(oa[0], oa[E - 1]);
        } else {
            ab[(size_t)t * N + k] = ob[0];
            ab[((size_t)g.nt + t) * N + k] = oa[0];
        }
    }
}

template <int E, int MB = 4>
__global__ void __launch_bounds__(256, E == 2 ? KP_MINB : (MB > 4 ? 2 : 3)) ks_keyprod_stream(KsGeo g, const PrimeDev* __restrict__ primes,
                                                                      u64 gal, KsBatch kb,
                                                                      u64* __restrict__ acc, int tlimit) {
    pdl_enter();
    const size_t N = (size_t)1 << g.logN;
    const int t = blockIdx.y;
    const int pi = g.prime(t);
    const PrimeDev P = primes[pi];
    const size_t k = E * ((size_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (k >= N) return;
    const int dig = t < g.nl ? t / g.alpha : -1;   // the digit that contains limb t (uniform), or -1 for a P limb
    if (P.fp) kp_run<E, true, MB>(g, P, t, pi, dig, k, gal, kb, acc);
    else kp_run<E, false, MB>(g, P, t, pi, dig, k, gal, kb, acc);
}

// ---- B (rotate-and-sum form): key products of several rotations of one input,
// summed in the extended basis -------------------------------------------------
// out = x + sum_r sigma_r(x) (radix ladders): entry b's digits
// UP_b are read through each Galois element g_r and multiplied with key_r;
// the 2 * R * beta products of a coefficient accumulate in registers, and
// [P]_q * sigma_r(c0) joins poly 0's Q limbs, so the single ModDown that
// follows (exact division by P) returns sum_r sigma_r(c0) + the key-switched
// part; x itself is the ModDown store's second addend.  A thread owns one
// coefficient pair of target limb t for up to RS_NBT entries: the key words
// of rotation r are loaded once and reused by the entries.  Aligned index
// pairs map to aligned pairs under every Galois element (src(k + 1) =
// src(k) ^ 1), so each gather is one 16-byte load.
constexpr int RS_MAXR = 7;   // rotations per stage (radix 8)
struct KsRotsum {
    int nb, nrot;
    const u64* c0[KS_MAXB];    // x_b poly 0 [nl][N]
    const u64* c1[KS_MAXB];    // x_b poly 1 [nl][N]
    const u64* up[KS_MAXB];    // ModUp digits of c1_b [beta][nt][N]
    u64 gal[RS_MAXR];
    const u64* key[RS_MAXR];   // [dnum][2][nall][N]
};

// E words of index pair / word k read through a Galois permutation: aligned
// pairs map to aligned pairs, possibly swapped (src(k + 1) = src(k) ^ 1)
template <int E>
__device__ __forceinline__ void rs_gather(const u64* __restrict__ base, unsigned src, u64* v) {
    if (E == 2) {
        const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(base + (src & ~1u));
        const bool sw = src & 1u;
        v[0] = sw ? w.y : w.x;
        v[E - 1] = sw ? w.x : w.y;
    } else {
        v[0] = base[src];
    }
}
template <int E>
__device__ __forceinline__ void rs_load(const u64* __restrict__ p, u64* v) {
    if (E == 2) {
        const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(p);
        v[0] = w.x;
        v[E - 1] = w.y;
    } else {
        v[0] = p[0];
    }
}

// NBT entries per pass over the rotations (register budget)
template <bool FP, int MB, int NBT, int E>
__device__ __forceinline__ void rs_run(const KsGeo& g, const PrimeDev& P, int t, int pi, int dig, unsigned k, int b0,
                                       int nb, const KsRotsum& rb, u64 pq, u64* __restrict__ acc) {
    using KW = typename std::conditional<FP, double, u64>::type;
    const size_t N = (size_t)1 << g.logN;
    const size_t kstride = (size_t)g.nall * N;
    double fb[NBT][E], fa[NBT][E];
    U128 ib[NBT][E], ia[NBT][E];
#pragma unroll
    for (int i = 0; i < NBT; i++)
#pragma unroll
        for (int e = 0; e < E; e++) {
            if constexpr (FP) { fb[i][e] = 0; fa[i][e] = 0; }
            else { ib[i][e] = U128{0, 0}; ia[i][e] = U128{0, 0}; }
        }
    const bool qlimb = t < g.nl;
    const double pqd = FP ? fp_word(pq) : 0.0;
    // 128-bit sums hold 15 products of a lazy digit (< 16q) and a key word
    // (q < 2^60); deeper sums (8 digits) are folded after each rotation
    const bool fold = !FP && (g.beta + 1) * rb.nrot > 15;
    for (int r = 0; r < rb.nrot; r++) {
        const unsigned src = galois_src(k, g.logN, rb.gal[r]);
        // every load of this rotation is issued before the first use: the key
        // words, then each entry's digits and c0
        u64 kw[MB][2][E];
#pragma unroll
        for (int j = 0; j < MB; j++) {
            if (j >= g.beta) break;
            const u64* kp = rb.key[r] + ((size_t)(2 * j) * g.nall + pi) * N + k;
            rs_load<E>(kp, kw[j][0]);
            rs_load<E>(kp + kstride, kw[j][1]);
        }
        u64 x[NBT][MB + 1][E];
#pragma unroll
        for (int i = 0; i < NBT; i++) {
            if (i >= nb) break;
            const int b = b0 + i;
#pragma unroll
            for (int j = 0; j < MB; j++) {
                if (j >= g.beta) break;
                const u64* bp = (j == dig) ? rb.c1[b] + (size_t)t * N : rb.up[b] + ((size_t)j * g.nt + t) * N;
                rs_gather<E>(bp, src, x[i][j]);
            }
            if (qlimb) rs_gather<E>(rb.c0[b] + (size_t)t * N, src, x[i][MB]);
        }
        KW kbv[MB][E], kav[MB][E];
#pragma unroll
        for (int j = 0; j < MB; j++) {
            if (j >= g.beta) break;
#pragma unroll
            for (int e = 0; e < E; e++) {
                if constexpr (FP) { kbv[j][e] = fp_word(kw[j][0][e]); kav[j][e] = fp_word(kw[j][1][e]); }
                else { kbv[j][e] = kw[j][0][e]; kav[j][e] = kw[j][1][e]; }
            }
        }
#pragma unroll
        for (int i = 0; i < NBT; i++) {
            if (i >= nb) break;
#pragma unroll
            for (int e = 0; e < E; e++) {
                if constexpr (FP) {
                    double sb = fb[i][e], sa = fa[i][e];
#pragma unroll
                    for (int j = 0; j < MB; j++) {
                        if (j >= g.beta) break;
                        const double y = fp_word(x[i][j][e]);
                        sb = __dadd_rn(sb, fp_mulmod(y, kbv[j][e], P.qd, P.qinv));
                        sa = __dadd_rn(sa, fp_mulmod(y, kav[j][e], P.qd, P.qinv));
                    }
                    if (qlimb) sb = __dadd_rn(sb, fp_mulmod(fp_word(x[i][MB][e]), pqd, P.qd, P.qinv));
                    fb[i][e] = sb;
                    fa[i][e] = sa;
                } else {
#pragma unroll
                    for (int j = 0; j < MB; j++) {
                        if (j >= g.beta) break;
                        mac128(ib[i][e], x[i][j][e], kbv[j][e]);
                        mac128(ia[i][e], x[i][j][e], kav[j][e]);
                    }
                    if (qlimb) mac128(ib[i][e], x[i][MB][e], pq);
                    if (fold && r + 1 < rb.nrot) {
                        ib[i][e] = U128{reduce128(ib[i][e].hi, ib[i][e].lo, P), 0};
                        ia[i][e] = U128{reduce128(ia[i][e].hi, ia[i][e].lo, P), 0};
                    }
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NBT; i++) {
        if (i >= nb) break;
        u64 ob[E], oa[E];
#pragma unroll
        for (int e = 0; e < E; e++) {
            if constexpr (FP) {
                ob[e] = fp_canon(fb[i][e], P.qd, P.qinv);
                oa[e] = fp_canon(fa[i][e], P.qd, P.qinv);
            } else {
                ob[e] = reduce128(ib[i][e].hi, ib[i][e].lo, P);
                oa[e] = reduce128(ia[i][e].hi, ia[i][e].lo, P);
            }
        }
        u64* ab = acc + (size_t)(b0 + i) * g.acc_stride();
        if (E == 2) {
            *reinterpret_cast<ulonglong2*>(ab + (size_t)t * N + k) = make_ulonglong2(ob[0], ob[E - 1]);
            *reinterpret_cast<ulonglong2*>(ab + ((size_t)g.nt + t) * N + k) = make_ulonglong2(oa[0], oa[E - 1]);
        } else {
            ab[(size_t)t * N + k] = ob[0];
            ab[((size_t)g.nt + t) * N + k] = oa[0];
        }
    }
}

// knobs (measured with scripts/ladder_probe.py, 3 streams x batches of 3
// radix-4 stages at level 11, us per stage): coefficients per thread, entries
// per pass over the rotations for FP64 / integer limbs, entries per thread
// group, resident 256-thread CTAs per SM.  One coefficient of one entry per
// thread at 5 CTAs per SM (48 registers; the entries of a coefficient block
// run side by side and share its key words through L2) measured best: 99.5;
// 2 entries per thread 112.8, 4 entries 111.0, coefficient pairs 117-132,
// 4 / 6 CTAs per SM 102.7 / 109.5
#ifndef RS_E
#define RS_E 1
#endif
#ifndef RS_NF
#define RS_NF 1
#endif
#ifndef RS_NI
#define RS_NI 1
#endif
#ifndef RS_GROUP
#define RS_GROUP 1
#endif
#ifndef RS_MINB
#define RS_MINB 5
#endif
constexpr int RS_NBT = RS_GROUP;   // entries per thread
// grid x = (coefficient block, entry group) with the group fastest, so the
// groups sharing a block's key words run together (second read from L2)
template <int MB = 4>
__global__ void __launch_bounds__(256, MB > 4 ? 2 : RS_MINB) ks_keyprod_rotsum(KsGeo g, const PrimeDev* __restrict__ primes,
                                                                  KsRotsum rb, const u64* __restrict__ pmodq,
                                                                  u64* __restrict__ acc, int ngroups) {
    pdl_enter();
    const size_t N = (size_t)1 << g.logN;
    const int t = blockIdx.y;
    const int pi = g.prime(t);
    const PrimeDev P = primes[pi];
    const int grp = blockIdx.x % ngroups;
    const unsigned k = (unsigned)RS_E * ((blockIdx.x / ngroups) * blockDim.x + threadIdx.x);
    if (k >= N) return;
    const int b0 = grp * RS_NBT;
    const int nb = min(RS_NBT, rb.nb - b0);
    const int dig = t < g.nl ? t / g.alpha : -1;
    const u64 pq = t < g.nl ? pmodq[pi] : 0;
    // entries per pass over the rotations, by register budget: the later
    // passes re-read the key words from L1 / L2
    constexpr int NF = MB > 4 ? 1 : RS_NF, NI = MB > 4 ? 1 : RS_NI;
    if (P.fp) {
        for (int o = 0; o < nb; o += NF) rs_run<true, MB, NF, RS_E>(g, P, t, pi, dig, k, b0 + o, min(NF, nb - o), rb, pq, acc);
    } else {
        for (int o = 0; o < nb; o += NI) rs_run<false, MB, NI, RS_E>(g, P, t, pi, dig, k, b0 + o, min(NI, nb - o), rb, pq, acc);
    }
}

// The stage kernel proper: digit count and rotation count are compile-time,
// so every loop is unrolled, the (rotation, digit) bases are scalar offsets of
// one per-thread index and the parameter arrays are read at constant offsets
// (the generic form above spent 88 % of its issue slots on loop control and
// 64-bit address arithmetic: 1031 instructions per thread against ~400 here).
// Grid (entry, coefficient block, target limb): the entries of a coefficient
// block run side by side and share its key words through L2.
// MODE 0: rotate-and-sum (digits, c1 and c0 read through gal[r]; [P]_q c0 joins poly 0).
// MODE 1: relinearisation (NR = 1, no permutation): [P]_q (d0, d1) join both
// polys, c0 -> the tensor's d0 with d1 right behind it ([nl][N] each), so the
// merged ModDown + rescale that follows returns rescale(d + KS(d2)).
template <int BETA, int NR, int MODE = 0>
__global__ void __launch_bounds__(256, BETA > 4 ? 3 : RS_MINB) ks_keyprod_rotsum_t(KsGeo g, const PrimeDev* __restrict__ primes,
                                                                    KsRotsum rb, const u64* __restrict__ pmodq,
                                                                    u64* __restrict__ acc) {
    pdl_enter();
    const int t = blockIdx.z;
    const int pi = g.prime(t);
    const PrimeDev P = primes[pi];
    const int b = blockIdx.x;
    const unsigned k = blockIdx.y * 256u + threadIdx.x;
    const unsigned N = 1u << g.logN;
    const bool qlimb = t < g.nl;
    const int dig = qlimb ? t / g.alpha : -1;
    const size_t toff = (size_t)t * N;
    const u64* __restrict__ c1 = rb.c1[b] + toff;
    const u64* __restrict__ c0 = rb.c0[b] + toff;
    const u64* __restrict__ up = rb.up[b] + toff;
    const size_t dstride = (size_t)g.nt * N;            // digit stride of UP
    const size_t kstride = (size_t)g.nall * N;          // (b, a) stride of a key digit
    const size_t koff = (size_t)pi * N + k;
    const size_t pstride = (size_t)g.nl * N;            // MODE 1: d0 -> d1
    const u64 pq = qlimb ? pmodq[pi] : 0;
    u64 ob, oa;
    if (P.fp) {
        const double q = P.qd, qinv = P.qinv, pqd = fp_word(pq);
        double sb = 0, sa = 0;
#pragma unroll
        for (int r = 0; r < NR; r++) {
            const unsigned src = MODE == 0 ? galois_src(k, g.logN, rb.gal[r]) : k;
            const u64* __restrict__ kp = rb.key[r] + koff;
            u64 kb[BETA], ka[BETA], x[BETA], z = 0, z1 = 0;
#pragma unroll
            for (int j = 0; j < BETA; j++) {
                kb[j] = __ldg(kp + (size_t)(2 * j) * kstride);
                ka[j] = __ldg(kp + (size_t)(2 * j + 1) * kstride);
                x[j] = (j == dig ? c1 : up + j * dstride)[src];
            }
            if (qlimb) z = c0[src];
            if (MODE == 1 && qlimb) z1 = c0[pstride + src];
#pragma unroll
            for (int j = 0; j < BETA; j++) {
                const double y = fp_word(x[j]);
                sb = __dadd_rn(sb, fp_mulmod(y, fp_word(kb[j]), q, qinv));
                sa = __dadd_rn(sa, fp_mulmod(y, fp_word(ka[j]), q, qinv));
            }
            if (qlimb) sb = __dadd_rn(sb, fp_mulmod(fp_word(z), pqd, q, qinv));
            if (MODE == 1 && qlimb) sa = __dadd_rn(sa, fp_mulmod(fp_word(z1), pqd, q, qinv));
        }
        ob = fp_canon(sb, q, qinv);
        oa = fp_canon(sa, q, qinv);
    } else {
        // 128-bit sums hold 15 products of a lazy digit (< 16q) and a key
        // word (q < 2^60): folded to one word whenever the next rotation's
        // BETA + 1 products would pass that
        constexpr int FOLD = 15 / (BETA + 1);   // rotations between folds
        U128 ib = {0, 0}, ia = {0, 0};
#pragma unroll
        for (int r = 0; r < NR; r++) {
            const unsigned src = MODE == 0 ? galois_src(k, g.logN, rb.gal[r]) : k;
            const u64* __restrict__ kp = rb.key[r] + koff;
            u64 kb[BETA], ka[BETA], x[BETA], z = 0, z1 = 0;
#pragma unroll
            for (int j = 0; j < BETA; j++) {
                kb[j] = __ldg(kp + (size_t)(2 * j) * kstride);
                ka[j] = __ldg(kp + (size_t)(2 * j + 1) * kstride);
                x[j] = (j == dig ? c1 : up + j * dstride)[src];
            }
            if (qlimb) z = c0[src];
            if (MODE == 1 && qlimb) z1 = c0[pstride + src];
#pragma unroll
            for (int j = 0; j < BETA; j++) {
                mac128(ib, x[j], kb[j]);
                mac128(ia, x[j], ka[j]);
            }
            if (qlimb) mac128(ib, z, pq);
            if (MODE == 1 && qlimb) mac128(ia, z1, pq);
            if ((r + 1) % FOLD == 0 && r + 1 < NR) {
                ib = U128{reduce128(ib.hi, ib.lo, P), 0};
                ia = U128{reduce128(ia.hi, ia.lo, P), 0};
            }
        }
        ob = reduce128(ib.hi, ib.lo, P);
        oa = reduce128(ia.hi, ia.lo, P);
    }
    static_assert(BETA + 1 <= 15 && NR <= RS_MAXR, "128-bit key-product sum bound");
    // FP64 sums: NR * (BETA + 1) <= 63 terms below 0.6q, q < 2^46: exact integers below 2^53
    u64* __restrict__ ab = acc + (size_t)b * g.acc_stride() + toff + k;
    ab[0] = ob;
    ab[dstride] = oa;
}

// The plain key product in the stage kernel's form: one coefficient of one
// entry per thread, the digit count compile-time, grid (entry, coefficient
// block, target limb) so the entries of a coefficient block run side by side
// and equal keys are read once from HBM (the rest from L2).  Entry b reads its
// c1 through ugal[b] (hoisted) or the pipeline's element, its ModUp digits
// through ugal[b] only (a plain pipeline's digits are already permuted).
template <int BETA>
__global__ void __launch_bounds__(256, BETA > 4 ? 3 : RS_MINB) ks_keyprod_plain_t(KsGeo g, const PrimeDev* __restrict__ primes, u64 gal,
                                                                    KsBatch kb, u64* __restrict__ acc) {
    pdl_enter();
    const int t = blockIdx.z;
    const int pi = g.prime(t);
    const PrimeDev P = primes[pi];
    const int b = blockIdx.x;
    const unsigned k = blockIdx.y * 256u + threadIdx.x;
    const unsigned N = 1u << g.logN;
    const int dig = t < g.nl ? t / g.alpha : -1;
    const size_t toff = (size_t)t * N;
    const u64 ug = kb.ugal[b], gd = ug ? ug : gal;
    const unsigned src_d = gd ? galois_src(k, g.logN, gd) : k;
    const unsigned src_u = ug ? src_d : k;
    const u64* __restrict__ c1 = kb.d[b] + toff;
    const u64* __restrict__ up = kb.up[b] + toff;
    const size_t dstride = (size_t)g.nt * N;
    const size_t kstride = (size_t)g.nall * N;
    const u64* __restrict__ kp = kb.key[b] + (size_t)pi * N + k;
    u64 kbw[BETA], kaw[BETA], x[BETA];
#pragma unroll
    for (int j = 0; j < BETA; j++) {
        kbw[j] = __ldg(kp + (size_t)(2 * j) * kstride);
        kaw[j] = __ldg(kp + (size_t)(2 * j + 1) * kstride);
        x[j] = j == dig ? c1[src_d] : up[j * dstride + src_u];
    }
    u64 ob, oa;
    if (P.fp) {
        const double q = P.qd, qinv = P.qinv;
        double sb = 0, sa = 0;
#pragma unroll
        for (int j = 0; j < BETA; j++) {
            const double y = fp_word(x[j]);
            sb = __dadd_rn(sb, fp_mulmod(y, fp_word(kbw[j]), q, qinv));
            sa = __dadd_rn(sa, fp_mulmod(y, fp_word(kaw[j]), q, qinv));
        }
        ob = fp_canon(sb, q, qinv);
        oa = fp_canon(sa, q, qinv);
    } else {
        U128 ib = {0, 0}, ia = {0, 0};
#pragma unroll
        for (int j = 0; j < BETA; j++) {
            mac128(ib, x[j], kbw[j]);
            mac128(ia, x[j], kaw[j]);
        }
        ob = reduce128(ib.hi, ib.lo, P);
        oa = reduce128(ia.hi, ia.lo, P);
    }
    u64* __restrict__ ab = acc + (size_t)b * g.acc_stride() + toff + k;
    ab[0] = ob;
    ab[dstride] = oa;
}

// ---- D: ModDown conversion fused into the column pass ----------------------

// (the P -> Q conversion has the ModUp loader's shape: K inputs, one target)
template <int LOGSZ, int SUBS, int NK, int PMB = KS_COLS_PMB>
__global__ void __launch_bounds__(PassGeo<LOGSZ, MODE_COLS, SUBS>::THREADS, PMB)
    ks_moddown_cols(KsGeo g, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ acc, const u64* __restrict__ md_tab,
                    const u64* __restrict__ cc_tab, u64* __restrict__ Wt) {
    pdl_trigger();
    extern __shared__ u64 sm[];
    const int s = blockIdx.y / g.nout, i = blockIdx.y % g.nout;
    const size_t N = (size_t)1 << g.logN;
    const PrimeDev P = primes[i];
    const u64 q = P.q;
    acc += blockIdx.z * g.acc_stride();
    Wt += blockIdx.z * g.w_stride();
    LdModup<NK> ld;
    ld.na = g.nk;
    ld.p = q;
    ld.cc = cc_tab[i];
#pragma unroll
    for (int t = 0; t < NK; t++) {
        const bool on = t < g.nk;
        const int tt = on ? t : 0;
        ld.y[t] = acc + ((size_t)s * g.nt + g.mdf + tt) * N;
        ld.w[t] = on ? md_tab[((size_t)tt * g.nall + i) * 2] : 0;
        ld.ws[t] = on ? md_tab[((size_t)tt * g.nall + i) * 2 + 1] : 0;
    }
    StPlain<false, false> st{Wt + ((size_t)s * g.nout + i) * N, q, 0, 0};
    PassGeo<LOGSZ, MODE_COLS, SUBS> G;
    G.init(g.N1);
    const ulonglong2* TW = tw + ((size_t)i << g.logN);
    ulonglong2* twsm = PassGeo<LOGSZ, MODE_COLS, SUBS>::twsm_of(sm);
    stage_twiddles(G, twsm, TW, g.N1);
    pdl_wait();   // everything above reads context-lifetime tables only
    ntt_pass<LOGSZ, MODE_COLS, SUBS, false, 2 * NK + 1, BOUND_LIM>(G, sm, TW, P, ld, st, twsm, true);
}

// ---- E: chunk pass with the ModDown combine in its stores ------------------

struct StModdown {
    u64* __restrict__ out;           // [nl][N] of this poly
    const u64* __restrict__ accq;    // ACC Q limb i of this poly (full limb base)
    const u64* __restrict__ add;     // addend limb base or nullptr (read through gal)
    u64 q, pinv, pinv_s, gal;
    int logN;
    const u64* __restrict__ add2;    // second addend limb (not permuted) or nullptr: rotate-and-add ladders
    // w < MD_OUTB * q (the chunk pass's output bound), accq canonical: the
    // Shoup product takes the unreduced difference (< 15q < 2^64)
    static constexpr int MD_OUTB = 14;
    __device__ __forceinline__ u64 one(size_t k, u64 w) const {
        u64 v = mul_shoup(accq[k] + MD_OUTB * q - w, pinv, pinv_s, q);
        if (add) {
            const u64 a = gal ? add[galois_src((unsigned)k, logN, gal)] : add[k];
            v = add_mod(v, a, q);
        }
        if (add2) v = add_mod(v, add2[k], q);
        return v;
    }
    __device__ __forceinline__ void operator()(size_t k, u64 w) const { out[k] = one(k, w); }
    // 8 consecutive words: every operand load (ACC, the gathered addend, the
    // ladder addend) is issued before the first use, so the gathers overlap
    // instead of forming a load -> use chain per element
    __device__ __forceinline__ void store8(size_t k, const u64* w) const {
        u64 A[8], D[8], E[8];
        const ulonglong2* ap = reinterpret_cast<const ulonglong2*>(accq + k);
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const ulonglong2 t = ap[v];
            A[2 * v] = t.x;
            A[2 * v + 1] = t.y;
        }
        if (add) {
            if (gal) {
#pragma unroll
                for (int e = 0; e < 8; e++) D[e] = add[galois_src((unsigned)(k + e), logN, gal)];
            } else {
                const ulonglong2* dp = reinterpret_cast<const ulonglong2*>(add + k);
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    const ulonglong2 t = dp[v];
                    D[2 * v] = t.x;
                    D[2 * v + 1] = t.y;
                }
            }
        }
        if (add2) {
            const ulonglong2* ep = reinterpret_cast<const ulonglong2*>(add2 + k);
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const ulonglong2 t = ep[v];
                E[2 * v] = t.x;
                E[2 * v + 1] = t.y;
            }
        }
        u64 r[8];
#pragma unroll
        for (int e = 0; e < 8; e++) {
            u64 v = mul_shoup(A[e] + MD_OUTB * q - w[e], pinv, pinv_s, q);
            if (add) v = add_mod(v, D[e], q);
            if (add2) v = add_mod(v, E[e], q);
            r[e] = v;
        }
        ulonglong2* o = reinterpret_cast<ulonglong2*>(out + k);
#pragma unroll
        for (int v = 0; v < 4; v++) o[v] = make_ulonglong2(r[2 * v], r[2 * v + 1]);
    }
};

// ModDown chunk pass: 5 resident 128-thread CTAs per SM (96 registers) instead
// of the passes' 8 (64): its stores read three operands per word and the
// extra registers let them issue early (kernel 6.71 -> 6.42 ms per pair,
// 42 -> 44 % of the HBM peak; 6 CTAs: 6.65 ms)
#ifndef MD_MINB
#define MD_MINB (5 * 128 / PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::THREADS)
#endif
#ifndef MD_MINB_CHAIN
#define MD_MINB_CHAIN MD_MINB   // the same for a lone key switch (grid z = 1)
#endif
template <int MINB = MD_MINB>
__global__ void __launch_bounds__(PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::THREADS, MINB)
    ks_moddown_chunks(KsGeo g, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ Wt, const u64* __restrict__ acc,
                      const u64* __restrict__ pinv, int add_npoly, KsBatch kb) {
    pdl_trigger();
    extern __shared__ u64 sm[];
    const int s = blockIdx.y / g.nout, i = blockIdx.y % g.nout;
    const size_t N = (size_t)1 << g.logN;
    const int b = blockIdx.z;
    Wt += b * g.w_stride();
    acc += b * g.acc_stride();
    const u64* __restrict__ addend = kb.add[b];
    const u64* __restrict__ addend2 = kb.add2[b];
    u64* __restrict__ out = kb.out[b];
    const PrimeDev P = primes[i];
    const u64 q = P.q;
    LdPlain ld{Wt + ((size_t)s * g.nout + i) * N};
    StModdown st{out + ((size_t)s * g.nout + i) * N, acc + ((size_t)s * g.nt + i) * N,
                 (s < add_npoly && addend) ? addend + ((size_t)s * g.nl + i) * N : nullptr, q, pinv[2 * i], pinv[2 * i + 1],
                 kb.agal[b], g.logN, addend2 ? addend2 + ((size_t)s * g.nl + i) * N : nullptr};
    PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS> G;
    G.init(g.N1);
    const ulonglong2* TW = tw + ((size_t)i << g.logN);
    ulonglong2* twsm = PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::twsm_of(sm);
    stage_twiddles(G, twsm, TW, g.N1);
    pdl_wait();   // everything above reads context-lifetime tables only
    ntt_pass<CH_LOG, MODE_CHUNKS, CH_SUBS, false, BOUND_LIM, StModdown::MD_OUTB>(G, sm, TW, P, ld, st, twsm, true);
}

// ---- fused rescale (R1: bcast in the column pass, R2: combine in the chunk pass)

struct LdBcast {
    const u64* __restrict__ X;   // INTT of the dropped limb
    u64 ql, q, qlm;
    u64 r1;                      // floor(2^64 / q): Shoup companion of 1 (= PrimeDev::mu_hi)
    __device__ __forceinline__ u64 operator()(size_t k) const {
        const u64 v = X[k], vm = mul_shoup(v, 1, r1, q);   // v mod q without a 64-bit division
        return v > (ql - 1) / 2 ? sub_mod(vm, qlm, q) : vm;
    }
    __device__ __forceinline__ void load8(size_t k, u64* x) const {
        for (int e = 0; e < 8; e++) x[e] = (*this)(k + e);
    }
};

// batched rescales (grid z = ciphertext): inputs / outputs per ciphertext
struct RsBatch {
    const u64* a[KS_MAXB];
    u64* out[KS_MAXB];
};

#ifndef RS_PMB
#define RS_PMB PASS_MIN_BLOCKS   // register budget of the rescale passes (as PASS_MIN_BLOCKS)
#endif
template <int LOGSZ, int SUBS>
__global__ void __launch_bounds__(PassGeo<LOGSZ, MODE_COLS, SUBS>::THREADS, RS_PMB)
    rs_cols(int level, int logN, int N1, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ X, const u64* __restrict__ tab,
            u64* __restrict__ Yt, int npoly) {
    pdl_trigger();
    extern __shared__ u64 sm[];
    const int s = blockIdx.y / level, i = blockIdx.y % level;
    const size_t N = (size_t)1 << logN;
    X += (size_t)blockIdx.z * npoly * N;
    Yt += (size_t)blockIdx.z * npoly * level * N;
    const PrimeDev P = primes[i];
    const u64 q = P.q;
    LdBcast ld{X + (size_t)s * N, primes[level].q, q, tab[3 * i + 2], P.mu_hi};
    StPlain<false, false> st{Yt + ((size_t)s * level + i) * N, q, 0, 0};
    PassGeo<LOGSZ, MODE_COLS, SUBS> G;
    G.init(N1);
    const ulonglong2* TW = tw + ((size_t)i << logN);
    ulonglong2* twsm = PassGeo<LOGSZ, MODE_COLS, SUBS>::twsm_of(sm);
    stage_twiddles(G, twsm, TW, N1);
    pdl_wait();   // everything above reads context-lifetime tables only
    ntt_pass<LOGSZ, MODE_COLS, SUBS, false, 2, BOUND_LIM>(G, sm, TW, P, ld, st, twsm, true);
}

struct StRescale {
    u64* __restrict__ out;
    const u64* __restrict__ a;
    u64 q, c, cs;
    static constexpr int RS_OUTB = 14;   // y < 14q, a canonical: a + 14q - y < 15q
    __device__ __forceinline__ u64 one(size_t k, u64 y) const {
        return mul_shoup(a[k] + RS_OUTB * q - y, c, cs, q);
    }
    __device__ __forceinline__ void operator()(size_t k, u64 y) const { out[k] = one(k, y); }
    __device__ __forceinline__ void store8(size_t k, const u64* y) const {
        u64 A[8];   // all operand loads before the first use
        const ulonglong2* ap = reinterpret_cast<const ulonglong2*>(a + k);
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const ulonglong2 t = ap[v];
            A[2 * v] = t.x;
            A[2 * v + 1] = t.y;
        }
        ulonglong2* o = reinterpret_cast<ulonglong2*>(out + k);
#pragma unroll
        for (int v = 0; v < 4; v++)
            o[v] = make_ulonglong2(mul_shoup(A[2 * v] + RS_OUTB * q - y[2 * v], c, cs, q),
                                   mul_shoup(A[2 * v + 1] + RS_OUTB * q - y[2 * v + 1], c, cs, q));
    }
};

__global__ void __launch_bounds__(PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::THREADS,
                                  PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::MIN_BLOCKS * RS_PMB / PASS_MIN_BLOCKS)
    rs_chunks(int level, int logN, int N1, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ Yt, RsBatch rb,
              const u64* __restrict__ tab, int npoly) {
    pdl_trigger();
    extern __shared__ u64 sm[];
    const int s = blockIdx.y / level, i = blockIdx.y % level;
    const size_t N = (size_t)1 << logN;
    Yt += (size_t)blockIdx.z * npoly * level * N;
    const u64* __restrict__ a = rb.a[blockIdx.z];
    u64* __restrict__ out = rb.out[blockIdx.z];
    const PrimeDev P = primes[i];
    const u64 q = P.q;
    LdPlain ld{Yt + ((size_t)s * level + i) * N};
    StRescale st{out + ((size_t)s * level + i) * N, a + ((size_t)s * (level + 1) + i) * N, q, tab[3 * i],
                 tab[3 * i + 1]};
    PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS> G;
    G.init(N1);
    const ulonglong2* TW = tw + ((size_t)i << logN);
    ulonglong2* twsm = PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::twsm_of(sm);
    stage_twiddles(G, twsm, TW, N1);
    pdl_wait();   // everything above reads context-lifetime tables only
    ntt_pass<CH_LOG, MODE_CHUNKS, CH_SUBS, false, BOUND_LIM, StRescale::RS_OUTB>(G, sm, TW, P, ld, st, twsm, true);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

typedef unsigned __int128 u128;
static u64 mulm(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 shoup_of(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static u64 powm(u64 b, u64 e, u64 q) {
    u64 r = 1;
    b %= q;
    while (e) { if (e & 1) r = mulm(r, b, q); b = mulm(b, b, q); e >>= 1; }
    return r;
}

// column-pass geometry per ring degree
template <int LOGN>
struct ColCfg;
template <> struct ColCfg<14> { static constexpr int LOGSZ = 5, SUBS = 64; };
template <> struct ColCfg<15> { static constexpr int LOGSZ = 6, SUBS = 32; };
#ifndef HC_COL_SUBS16
#define HC_COL_SUBS16 16
#endif
template <> struct ColCfg<16> { static constexpr int LOGSZ = 7, SUBS = HC_COL_SUBS16; };
template <> struct ColCfg<17> { static constexpr int LOGSZ = 8, SUBS = 8; };

// One key-switch tail entry: which ModUp input it consumes and, hoisted, the
// Galois element applied to that input's digits.
struct KsTail {
    int src;
    u64 ugal;
    const u64* d;   // c1 of the input (NTT form)
    u64* out;
    const u64* add;
    const u64* add2;
    const u64* key;
    u64 agal;
};

// The fused pipeline: ModUp stage over `nin` inputs din[] (read through gal),
// then key product + ModDown over `B` tail entries.
// Rotate-and-sum stage (ks_keyprod_rotsum): tail entry b sums the rotations
// gal[0..nrot) of input b (c0[b], its c1 = din[b]) with keys key[].
struct KsRotsumSpec {
    int nrot;
    u64 gal[RS_MAXR];
    const u64* key[RS_MAXR];
    const u64* const* c0;
    // relinearisation + rescale in one pass: nrot = 1, no
    // permutation, c0[b] -> the tensor's (d0, d1), din[b] = d2; [P]_q (d0, d1)
    // joins the key product and the ModDown divides by q_l P (outputs at level - 1)
    bool relin = false;
};

// HC_KP_PLAIN: 0 = the plain pipelines keep ks_keyprod_stream, 1 = ks_keyprod_plain_t
// for up to 4 digits, 2 (default) = for up to 8 (the bootstrapping chains: 58.1 -> 53.9 ms)
static int kp_plain_t() {
    static const int v = [] { const char* e = std::getenv("HC_KP_PLAIN"); return e ? std::atoi(e) : 2; }();
    return v;
}

template <int LOGN>
static void ks_pipeline_t(Ctx& c, int nin, const u64* const* din, u64 gal, int level, int B, const KsTail* in,
                          int add_npoly, const KsRotsumSpec* rsum = nullptr) {
    constexpr int CL = ColCfg<LOGN>::LOGSZ, CS = ColCfg<LOGN>::SUBS;
    using CG = PassGeo<CL, MODE_COLS, CS>;
    using HG = PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>;
    const int N = c.N, nl = level + 1, K = c.K, nt = nl + K;
    const bool merged = rsum && rsum->relin;
    if (merged && level < 1) throw Error(-3, "relinearise + rescale at level 0");
    KsGeo g{level, nl, nt, c.L, K, c.alpha, c.dnum, c.nall, (nl + c.alpha - 1) / c.alpha, c.logN, N >> CH_LOG,
            merged ? nl - 1 : nl, merged ? K + 1 : K, merged ? nl - 1 : nl};
    const size_t csm = CG::smem_bytes(), hsm = HG::smem_bytes();
    KsBatch kb;
    kb.nb = B;

    Scratch sc(c);
    // 1. Y = INTT(sigma(d)) * (Q'/q_i)^-1
    u64* Y = sc.take((size_t)nin * g.y_stride());
    {
        JobList j;
        j.n = nl;
        j.custom = 1;
        j.center = 1;   // shifted outputs for the centred conversion (LdModup)
        j.galois = gal;
        j.nb = nin;
        for (int b = 0; b < nin; b++) {
            j.boff[b] = (long long)(b * g.y_stride());
            j.sboff[b] = (long long)(din[b] - din[0]);
        }
        for (int i = 0; i < nl; i++) {
            const int dj = i / c.alpha, lo = dj * c.alpha, hi = std::min(lo + c.alpha, nl);
            const u64 qi = c.pr[i].q;
            u64 qh = 1;
            for (int b = lo; b < hi; b++) if (b != i) qh = mulm(qh, c.pr[b].q % qi, qi);
            const u64 sc = mulm(c.pr[i].ninv, powm(qh, qi - 2, qi), qi);
            j.prime[i] = i;
            j.ptr[i] = Y + (size_t)i * N;
            j.src[i] = din[0] + (size_t)i * N;
            j.scale[i] = sc;
            j.scale_s[i] = shoup_of(sc, qi);
        }
        ntt_inverse(c, j);
    }
    // 2. A: conversion + column pass for every (digit, non-digit target)
    u64* I = sc.take((size_t)nin * g.i_stride());
    {
        KsJobs jobs;
        jobs.n = 0;
        for (int dj = 0; dj < g.beta; dj++) {
            const int lo = dj * c.alpha, hi = std::min(lo + c.alpha, nl);
            for (int t = 0; t < nt; t++) {
                if (t >= lo && t < hi) continue;
                jobs.digit[jobs.n] = (unsigned char)dj;
                jobs.t[jobs.n] = (unsigned char)t;
                jobs.n++;
            }
        }
        // algorithmic: the digit limbs Y read once, one intermediate limb written per job
        Launch scope(c, "ks_modup_cols", 8.0 * N * nin * (nl + (double)jobs.n));
        dim3 grid((N >> CL) / CS, jobs.n, nin);
        auto go = [&](auto kern) {
            set_smem(kern, csm);
            launch_k(c, kern, grid, CG::THREADS, csm, jobs, g, c.d_primes, c.twp(0, false), Y, c.d_modup,
                     c.d_modup_cc, I);
        };
        switch (c.alpha) {
            case 1: if (nin == 1) go(ks_modup_cols<CL, CS, 1, KS_PMB_CHAIN>); else go(ks_modup_cols<CL, CS, 1>); break;
            case 2: if (nin == 1) go(ks_modup_cols<CL, CS, 2, KS_PMB_CHAIN>); else go(ks_modup_cols<CL, CS, 2>); break;
            case 3: if (nin == 1) go(ks_modup_cols<CL, CS, 3, KS_PMB_CHAIN>); else go(ks_modup_cols<CL, CS, 3>); break;
            default: if (nin == 1) go(ks_modup_cols<CL, CS, 4, KS_PMB_CHAIN>); else go(ks_modup_cols<CL, CS, 4>); break;
        }
        HC_CUDA(cudaGetLastError());
    }
    // 3. B: chunk pass of every (digit, target) limb, then the streaming key
    //    product -> ACC [2][nt][N] per key switch
    u64* ACC = sc.take((size_t)B * g.acc_stride());
    {
        JobList j;
        j.n = 0;
        j.nb = nin;
        for (int b = 0; b < nin; b++) j.boff[b] = (long long)(b * g.i_stride());
        for (int dj = 0; dj < g.beta; dj++) {
            const int lo = dj * c.alpha, hi = std::min(lo + c.alpha, nl);
            for (int t = 0; t < nt; t++) {
                if (t >= lo && t < hi) continue;
                if (j.n == MAXJ) { ntt_forward_chunks(c, j); j.n = 0; }
                j.prime[j.n] = g.prime(t);
                j.ptr[j.n] = I + ((size_t)dj * nt + t) * N;
                j.src[j.n] = nullptr;
                j.n++;
            }
        }
        ntt_forward_chunks(c, j);
        for (int b = 0; b < B; b++) {
            kb.d[b] = in[b].d;
            kb.up[b] = I + (size_t)in[b].src * g.i_stride();
            kb.out[b] = in[b].out;
            kb.add[b] = in[b].add;
            kb.add2[b] = in[b].add2;
            kb.key[b] = in[b].key;
            kb.ugal[b] = in[b].ugal;
            kb.agal[b] = in[b].agal;
        }
        int nkeys = 1;
        for (int b = 1; b < B; b++) nkeys += in[b].key != in[b - 1].key;
        // algorithmic: the digit limbs (once per input) and ACC per key switch, each distinct key run once
        if (rsum) nkeys = rsum->nrot;
        Launch scope(c, rsum ? "ks_keyprod_rotsum" : "ks_keyprod_stream",
                     8.0 * N * ((double)nin * g.beta * nt + 2.0 * B * nt + 2.0 * nkeys * g.beta * nt +
                                (rsum ? (double)B * nl : 0.0)));
        if (rsum) {
            // rotate-and-sum: digits (once per input, re-read per rotation from L2),
            // c0, ACC and every rotation's key
            KsRotsum rb;
            rb.nb = B;
            rb.nrot = rsum->nrot;
            for (int r = 0; r < rsum->nrot; r++) { rb.gal[r] = rsum->gal[r]; rb.key[r] = rsum->key[r]; }
            for (int b = 0; b < B; b++) {
                rb.c0[b] = rsum->c0[b];
                rb.c1[b] = din[b];
                rb.up[b] = I + (size_t)b * g.i_stride();
            }
            const int ngroups = (B + RS_NBT - 1) / RS_NBT;
            const u64* pmodq = c.d_rescale + (size_t)(c.L + 1) * c.nall * 3;
            dim3 grid((unsigned)((N / RS_E + 255) / 256) * ngroups, nt);
            dim3 tgrid((unsigned)B, (unsigned)(N / 256), (unsigned)nt);
            const int nr = rsum->nrot;
            auto go = [&](auto kern) { launch_k(c, kern, tgrid, 256, 0, g, c.d_primes, rb, pmodq, ACC); };
            if (merged && g.beta == 4) go(ks_keyprod_rotsum_t<4, 1, 1>);
            else if (merged && g.beta == 3) go(ks_keyprod_rotsum_t<3, 1, 1>);
            else if (merged && g.beta == 2) go(ks_keyprod_rotsum_t<2, 1, 1>);
            else if (merged && g.beta == 1) go(ks_keyprod_rotsum_t<1, 1, 1>);
            else if (merged && g.beta == 5) go(ks_keyprod_rotsum_t<5, 1, 1>);
            else if (merged && g.beta == 6) go(ks_keyprod_rotsum_t<6, 1, 1>);
            else if (merged && g.beta == 7) go(ks_keyprod_rotsum_t<7, 1, 1>);
            else if (merged && g.beta == 8) go(ks_keyprod_rotsum_t<8, 1, 1>);
            else if (merged) throw Error(-2, "relinearise + rescale: more than 8 digits");
            else if (nr == 3 && g.beta == 4) go(ks_keyprod_rotsum_t<4, 3>);
            else if (nr == 3 && g.beta == 3) go(ks_keyprod_rotsum_t<3, 3>);
            else if (nr == 3 && g.beta == 2) go(ks_keyprod_rotsum_t<2, 3>);
            else if (nr == 3 && g.beta == 1) go(ks_keyprod_rotsum_t<1, 3>);
            else if (nr == 7 && g.beta == 4) go(ks_keyprod_rotsum_t<4, 7>);
            else if (nr == 7 && g.beta == 3) go(ks_keyprod_rotsum_t<3, 7>);
            else if (nr == 7 && g.beta == 2) go(ks_keyprod_rotsum_t<2, 7>);
            else if (nr == 7 && g.beta == 1) go(ks_keyprod_rotsum_t<1, 7>);
            else if (nr == 1 && g.beta == 4) go(ks_keyprod_rotsum_t<4, 1>);
            else if (nr == 1 && g.beta == 3) go(ks_keyprod_rotsum_t<3, 1>);
            else if (nr == 1 && g.beta == 2) go(ks_keyprod_rotsum_t<2, 1>);
            else if (nr == 1 && g.beta == 1) go(ks_keyprod_rotsum_t<1, 1>);
            else if (g.beta > 4) launch_k(c, ks_keyprod_rotsum<8>, grid, 256, 0, g, c.d_primes, rb, pmodq, ACC, ngroups);
            else launch_k(c, ks_keyprod_rotsum<4>, grid, 256, 0, g, c.d_primes, rb, pmodq, ACC, ngroups);
        } else
        // a lone key switch (chains) takes one coefficient per thread for
        // parallelism; batches take pairs (16-byte accesses, fewer index ops)
        // entries per distinct key: the stage-form kernel re-reads a shared key from L2
        // once per entry, the streaming form keeps its words in registers across the
        // entries -- better from 4 entries per key up (16 same-key rotations at
        // level 12: 11,700/s against 11,400/s)
        if (kp_plain_t() && g.beta <= (kp_plain_t() > 1 ? 8 : 4) && B < 4 * nkeys) {
            dim3 tgrid((unsigned)B, (unsigned)(N / 256), (unsigned)nt);
            auto go = [&](auto kern) { launch_k(c, kern, tgrid, 256, 0, g, c.d_primes, gal, kb, ACC); };
            switch (g.beta) {
                case 1: go(ks_keyprod_plain_t<1>); break;
                case 2: go(ks_keyprod_plain_t<2>); break;
                case 3: go(ks_keyprod_plain_t<3>); break;
                case 4: go(ks_keyprod_plain_t<4>); break;
                case 5: go(ks_keyprod_plain_t<5>); break;
                case 6: go(ks_keyprod_plain_t<6>); break;
                case 7: go(ks_keyprod_plain_t<7>); break;
                default: go(ks_keyprod_plain_t<8>); break;
            }
        } else if (g.beta > 4) {   // deep chains (bootstrapping): 8 digits, one coefficient per thread
            dim3 grid((unsigned)((N + 255) / 256), nt);
            launch_k(c, ks_keyprod_stream<1, 8>, grid, 256, 0, g, c.d_primes, gal, kb, ACC, nt);
        } else if (B >= KP_PAIRB) {
            dim3 grid((unsigned)((N / 2 + 255) / 256), nt);
            launch_k(c, ks_keyprod_stream<2>, grid, 256, 0, g, c.d_primes, gal, kb, ACC, nt);
        } else {
            dim3 grid((unsigned)((N + 255) / 256), nt);
            launch_k(c, ks_keyprod_stream<1>, grid, 256, 0, g, c.d_primes, gal, kb, ACC, nt);
        }
        HC_CUDA(cudaGetLastError());
    }
    // 4. INTT of the P limbs, final scale N^-1 (P/p_t)^-1 (in place)
    {
        JobList j;
        j.n = 0;
        j.custom = 1;
        j.center = 1;   // shifted outputs for the centred P -> Q conversion
        j.nb = B;
        for (int b = 0; b < B; b++) j.boff[b] = (long long)(b * g.acc_stride());
        for (int s = 0; s < 2; s++)
            for (int t = 0; t < g.nk; t++) {
                // the dropped basis: ACC limbs mdf .. mdf + nk - 1 (P, or q_l and P)
                const int pi = g.prime(g.mdf + t);
                const u64 p = c.pr[pi].q;
                u64 ph = 1;
                for (int b = 0; b < g.nk; b++) if (b != t) ph = mulm(ph, c.pr[g.prime(g.mdf + b)].q % p, p);
                const u64 sc = mulm(c.pr[pi].ninv, powm(ph, p - 2, p), p);
                j.prime[j.n] = pi;
                j.ptr[j.n] = ACC + ((size_t)s * nt + g.mdf + t) * N;
                j.src[j.n] = nullptr;
                j.scale[j.n] = sc;
                j.scale_s[j.n] = shoup_of(sc, p);
                j.n++;
            }
        ntt_inverse(c, j);
    }
    // 5. D: P -> Q conversion + column pass
    u64* Wt = sc.take((size_t)B * g.w_stride());
    {
        Launch scope(c, "ks_moddown_cols", 8.0 * N * B * (2.0 * g.nk + 2.0 * g.nout));
        dim3 grid((N >> CL) / CS, 2 * g.nout, B);
        const u64* md_tab = merged ? c.d_md2_tab + (size_t)level * (K + 1) * c.nall * 2 : c.d_moddown;
        const u64* md_cc = merged ? c.d_md2_cc + (size_t)level * c.nall : c.d_moddown_cc;
        auto go = [&](auto kern) {
            set_smem(kern, csm);
            launch_k(c, kern, grid, CG::THREADS, csm, g, c.d_primes, c.twp(0, false), ACC, md_tab, md_cc, Wt);
        };
        switch (g.nk) {
            case 1: if (B == 1) go(ks_moddown_cols<CL, CS, 1, KS_PMB_CHAIN>); else go(ks_moddown_cols<CL, CS, 1>); break;
            case 2: if (B == 1) go(ks_moddown_cols<CL, CS, 2, KS_PMB_CHAIN>); else go(ks_moddown_cols<CL, CS, 2>); break;
            case 3: if (B == 1) go(ks_moddown_cols<CL, CS, 3, KS_PMB_CHAIN>); else go(ks_moddown_cols<CL, CS, 3>); break;
            case 4: if (B == 1) go(ks_moddown_cols<CL, CS, 4, KS_PMB_CHAIN>); else go(ks_moddown_cols<CL, CS, 4>); break;
            default: if (B == 1) go(ks_moddown_cols<CL, CS, 5, KS_PMB_CHAIN>); else go(ks_moddown_cols<CL, CS, 5>); break;
        }
        HC_CUDA(cudaGetLastError());
    }
    // 6. E: chunk pass + (ACC - W) P^-1 + addend
    {
        set_smem(ks_moddown_chunks<>, hsm);
        set_smem(ks_moddown_chunks<MD_MINB_CHAIN>, hsm);
        int nadd2 = 0;
        for (int b = 0; b < B; b++) nadd2 += in[b].add2 != nullptr;
        Launch scope(c, "ks_moddown_chunks",
                     8.0 * N * (B * (2.0 * g.nout * 3 + (double)add_npoly * nl) + 2.0 * nl * nadd2));
        dim3 grid((N >> CH_LOG) / CH_SUBS, 2 * g.nout, B);
        // (ACC - W) / P, or / (q_l P) for the merged ModDown + rescale
        const u64* dinv = merged ? c.d_md2_dinv + (size_t)level * c.nall * 2 : c.d_pinv;
        if (B == 1)
            launch_k(c, ks_moddown_chunks<MD_MINB_CHAIN>, grid, HG::THREADS, hsm, g, c.d_primes, c.twp(0, false), Wt,
                     ACC, dinv, add_npoly, kb);
        else
            launch_k(c, ks_moddown_chunks<>, grid, HG::THREADS, hsm, g, c.d_primes, c.twp(0, false), Wt, ACC,
                     dinv, add_npoly, kb);
        HC_CUDA(cudaGetLastError());
    }
}

static bool fusable(const Ctx& c, int level) {
    return (level + c.alpha) / c.alpha <= KP_MAXB && c.K <= 4 && c.alpha <= 4 && c.logN >= 14 && c.logN <= 17;
}

static void ks_pipeline(Ctx& c, int nin, const u64* const* din, u64 gal, int level, int B, const KsTail* in,
                        int add_npoly, const KsRotsumSpec* rsum = nullptr) {
    switch (c.logN) {
        case 14: ks_pipeline_t<14>(c, nin, din, gal, level, B, in, add_npoly, rsum); break;
        case 15: ks_pipeline_t<15>(c, nin, din, gal, level, B, in, add_npoly, rsum); break;
        case 16: ks_pipeline_t<16>(c, nin, din, gal, level, B, in, add_npoly, rsum); break;
        default: ks_pipeline_t<17>(c, nin, din, gal, level, B, in, add_npoly, rsum); break;
    }
}

// out_b = x_b + sum_r sigma_{gals[r]}(x_b) for B inputs at one level (x_b = [c0 | c1] at xs[b])
bool keyswitch_rotsum(Ctx& c, int B, const u64* const* xs, u64* const* outs, int level, int nrot, const u64* gals,
                      const u64* const* keys) {
    if (!fusable(c, level) || nrot < 1 || nrot > RS_MAXR) return false;
    const size_t poly = (size_t)(level + 1) * c.N;
    KsRotsumSpec rs;
    rs.nrot = nrot;
    for (int r = 0; r < nrot; r++) { rs.gal[r] = gals[r]; rs.key[r] = keys[r]; }
    for (int b0 = 0; b0 < B; b0 += KS_MAXB) {
        const int nb = std::min(KS_MAXB, B - b0);
        const u64* din[KS_MAXB];
        const u64* c0s[KS_MAXB];
        KsTail tl[KS_MAXB];
        for (int b = 0; b < nb; b++) {
            const u64* x = xs[b0 + b];
            c0s[b] = x;
            din[b] = x + poly;
            tl[b] = KsTail{b, 0, x + poly, outs[b0 + b], nullptr, x, nullptr, 0};
        }
        rs.c0 = c0s;
        ks_pipeline(c, nb, din, 0, level, nb, tl, 0, &rs);
    }
    return true;
}

bool keyswitch_fused_batch(Ctx& c, int B, const KsIn* in, u64 gal, int level, int add_npoly, u64 add_gal) {
    if (!fusable(c, level)) return false;
    for (int b0 = 0; b0 < B; b0 += KS_MAXB) {
        const int nb = std::min(KS_MAXB, B - b0);
        const u64* din[KS_MAXB];
        KsTail tl[KS_MAXB];
        for (int b = 0; b < nb; b++) {
            const KsIn& x = in[b0 + b];
            din[b] = x.d;
            tl[b] = KsTail{b, 0, x.d, x.out, x.add, x.add2, x.key, add_gal};
        }
        ks_pipeline(c, nb, din, gal, level, nb, tl, add_npoly);
    }
    return true;
}

// Relinearisation + rescale of B tensors at one level >= 1:
// ds[b] = (d0, d1, d2) [3][level+1][N]; outs[b] [2][level][N] at level - 1.
bool keyswitch_relin_rescale(Ctx& c, int B, const u64* const* ds, u64* const* outs, int level, const u64* key) {
    if (!fusable(c, level)) return false;
    const size_t poly = (size_t)(level + 1) * c.N;
    KsRotsumSpec rs;
    rs.nrot = 1;
    rs.gal[0] = 0;
    rs.key[0] = key;
    rs.relin = true;
    for (int b0 = 0; b0 < B; b0 += KS_MAXB) {
        const int nb = std::min(KS_MAXB, B - b0);
        const u64* din[KS_MAXB];
        const u64* d0s[KS_MAXB];
        KsTail tl[KS_MAXB];
        for (int b = 0; b < nb; b++) {
            const u64* d = ds[b0 + b];
            d0s[b] = d;
            din[b] = d + 2 * poly;
            tl[b] = KsTail{b, 0, d + 2 * poly, outs[b0 + b], nullptr, nullptr, key, 0};
        }
        rs.c0 = d0s;
        ks_pipeline(c, nb, din, 0, level, nb, tl, 0, &rs);
    }
    return true;
}

bool keyswitch_hoisted(Ctx& c, const u64* const* c0s, const u64* const* c1s, int level, int B, const KsHoist* e) {
    if (!fusable(c, level)) return false;
    for (int b0 = 0; b0 < B; b0 += KS_MAXB) {
        const int nb = std::min(KS_MAXB, B - b0);
        // this chunk's distinct inputs, in first-use order
        int srcs[KS_MAXB], nsrc = 0;
        const u64* din[KS_MAXB];
        KsTail tl[KS_MAXB];
        for (int b = 0; b < nb; b++) {
            const KsHoist& x = e[b0 + b];
            int m = -1;
            for (int i = 0; i < nsrc; i++) if (srcs[i] == x.src) m = i;
            if (m < 0) { m = nsrc; srcs[nsrc] = x.src; din[nsrc++] = c1s[x.src]; }
            tl[b] = KsTail{m, x.gal, c1s[x.src], x.out, c0s[x.src], nullptr, x.key, x.gal};
        }
        ks_pipeline(c, nsrc, din, 0, level, nb, tl, 1);
    }
    return true;
}

bool keyswitch_fused(Ctx& c, const u64* d, u64 gal, int level, const Key& key, u64* out, const u64* addend,
                     int add_npoly, u64 add_gal, const u64* addend2) {
    const KsIn in{d, out, addend, addend2, key.d};
    return keyswitch_fused_batch(c, 1, &in, gal, level, add_npoly, add_gal);
}

template <int LOGN>
static void rescale_fused_t(Ctx& c, int B, const u64* const* a, int level, int npoly, u64* const* out) {
    constexpr int CL = ColCfg<LOGN>::LOGSZ, CS = ColCfg<LOGN>::SUBS;
    using CG = PassGeo<CL, MODE_COLS, CS>;
    using HG = PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>;
    const int N = c.N;
    Scratch sc(c);
    u64* X = sc.take((size_t)B * npoly * N);
    JobList j;
    j.n = B * npoly;
    for (int b = 0; b < B; b++)
        for (int s = 0; s < npoly; s++) {
            j.prime[b * npoly + s] = level;
            j.ptr[b * npoly + s] = X + ((size_t)b * npoly + s) * N;
            j.src[b * npoly + s] = a[b] + ((size_t)s * (level + 1) + level) * N;
        }
    ntt_inverse(c, j);
    u64* Yt = sc.take((size_t)B * npoly * level * N);
    const u64* tab = c.d_rescale + (size_t)level * c.nall * 3;
    const size_t csm = CG::smem_bytes(), hsm = HG::smem_bytes();
    const int N1 = N >> CH_LOG;
    {
        set_smem(rs_cols<CL, CS>, csm);
        Launch scope(c, "rs_cols", 8.0 * N * B * npoly * (1.0 + level));
        dim3 grid((N >> CL) / CS, npoly * level, B);
        launch_k(c, rs_cols<CL, CS>, grid, CG::THREADS, csm, level, c.logN, N1, c.d_primes, c.twp(0, false), X,
                                                              tab, Yt, npoly);
        HC_CUDA(cudaGetLastError());
    }
    {
        set_smem(rs_chunks, hsm);
        RsBatch rb;
        for (int b = 0; b < B; b++) { rb.a[b] = a[b]; rb.out[b] = out[b]; }
        Launch scope(c, "rs_chunks", 8.0 * N * B * npoly * 3.0 * level);
        dim3 grid((N >> CH_LOG) / CH_SUBS, npoly * level, B);
        launch_k(c, rs_chunks, grid, HG::THREADS, hsm, level, c.logN, N1, c.d_primes, c.twp(0, false), Yt, rb, tab,
                                                        npoly);
        HC_CUDA(cudaGetLastError());
    }
}

bool rescale_fused_batch(Ctx& c, int B, const u64* const* a, int level, int npoly, u64* const* out) {
    if (c.logN < 14 || c.logN > 17) return false;
    for (int b0 = 0; b0 < B; b0 += KS_MAXB) {
        const int nb = std::min(KS_MAXB, B - b0);
        switch (c.logN) {
            case 14: rescale_fused_t<14>(c, nb, a + b0, level, npoly, out + b0); break;
            case 15: rescale_fused_t<15>(c, nb, a + b0, level, npoly, out + b0); break;
            case 16: rescale_fused_t<16>(c, nb, a + b0, level, npoly, out + b0); break;
            default: rescale_fused_t<17>(c, nb, a + b0, level, npoly, out + b0); break;
        }
    }
    return true;
}

bool rescale_fused(Ctx& c, const u64* a, int level, int npoly, u64* out) {
    return rescale_fused_batch(c, 1, &a, level, npoly, &out);
}

}  // namespace hc
