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
//   3. B: chunk pass of those NTTs, one CTA per (chunk tile, target limb t),
//      looping over the digits: each digit's NTT output (or, for t inside
//      the digit, sigma(d) itself) is multiplied with the key in registers
//      and accumulated in 128 bits; one Barrett reduction per output
//                                                      -> ACC  (1 launch)
//   4. INTT of ACC's P limbs, final scale N^-1 * (P/p)^-1  (2 launches)
//   5. D: column pass of the ModDown NTT with the P->Q conversion in its
//      loads                                           -> Wt   (1 launch)
//   6. E: chunk pass whose stores compute (ACC - W) * P^-1 + addend, the
//      addend being sigma(c0) (gathered) or the tensor's (d0, d1)
//                                                      -> out  (1 launch)
//
// Every step is exact modular arithmetic, so the residues equal the
// unfused path and the oracle bit for bit.
#include "evaluator.h"
#include "kernels.cuh"
#include "ntt_pass.cuh"

namespace hc {

constexpr int CH_LOG = 9, CH_SUBS = 4;       // chunk pass: 512-point, 4 per CTA

struct KsJobs {
    int n;
    unsigned char digit[MAXJ];
    unsigned char t[MAXJ];
};

struct KsGeo {
    int level, nl, nt, L, K, alpha, dnum, nall, beta, logN, N1;
    __host__ __device__ int prime(int t) const { return t <= level ? t : L + 1 + (t - level - 1); }
};

// ---- A: ModUp conversion fused into the column pass --------------------------

// Conversion constants live in registers and the per-limb base pointers are
// formed once, so each converted element costs NA Shoup products and loads.
template <int NA>
struct LdModup {
    const u64* __restrict__ y[NA];   // Y limbs of the digit, coefficient form, pre-scaled by (Q'/q_a)^-1
    u64 w[NA], ws[NA];               // [Q'/q_a]_p and Shoup companions
    int na;
    u64 p;
    __device__ __forceinline__ u64 operator()(size_t k) const {
        u64 acc = 0;
#pragma unroll
        for (int a = 0; a < NA; a++)
            if (a < na) acc += mul_shoup_lazy(y[a][k], w[a], ws[a], p);
        return acc;   // < 2 * NA * p: the pass's input bound (INB = 2 * NA)
    }
    __device__ __forceinline__ void load8(size_t k, u64* x) const {
#pragma unroll
        for (int e = 0; e < 8; e++) x[e] = (*this)(k + e);
    }
};

template <int LOGSZ, int SUBS, int NA>
__global__ void __launch_bounds__(PassGeo<LOGSZ, MODE_COLS, SUBS>::THREADS, PASS_MIN_BLOCKS)
    ks_modup_cols(KsJobs jobs, KsGeo g, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ Y, const u64* __restrict__ modup_tab,
                  u64* __restrict__ I) {
    extern __shared__ u64 sm[];
    const int job = blockIdx.y;
    const int j = jobs.digit[job], t = jobs.t[job];
    const int pi = g.prime(t);
    const size_t N = (size_t)1 << g.logN;
    const int lo = j * g.alpha;
    const int hi = min(lo + g.alpha, g.nl);
    const PrimeDev P = primes[pi];
    const u64 p = P.q;
    LdModup<NA> ld;
    ld.na = hi - lo;
    ld.p = p;
    const u64* cf = modup_tab + (((size_t)(g.level * g.dnum + j) * g.alpha) * g.nall + pi) * 2;
#pragma unroll
    for (int a = 0; a < NA; a++) {
        const int aa = a < ld.na ? a : 0;
        ld.y[a] = Y + (size_t)(lo + aa) * N;
        ld.w[a] = cf[(size_t)aa * g.nall * 2];
        ld.ws[a] = cf[(size_t)aa * g.nall * 2 + 1];
    }
    StPlain<false, false> st{I + ((size_t)j * g.nt + t) * N, p, 0, 0};
    PassGeo<LOGSZ, MODE_COLS, SUBS> G;
    G.init(g.N1);
    const ulonglong2* TW = tw + ((size_t)pi << g.logN);
    ulonglong2* twsm = PassGeo<LOGSZ, MODE_COLS, SUBS>::twsm_of(sm);
    stage_twiddles(G, twsm, TW, g.N1);
    ntt_pass<LOGSZ, MODE_COLS, SUBS, false, 2 * NA, BOUND_LIM>(G, sm, TW, P, ld, st, twsm, true);
}

// ---- B: chunk pass + key inner product ------------------------------------

struct StCapture {
    u64* x;
    __device__ __forceinline__ void operator()(size_t, u64) const {}   // unused: chunk edge is contiguous
    __device__ __forceinline__ void store8(size_t, const u64* v) const {
#pragma unroll
        for (int e = 0; e < 8; e++) x[e] = v[e];
    }
};

constexpr int KP_MAXB = 4;   // digits handled by the fused key product (dnum <= 4)
#ifndef KP_MIN_BLOCKS
#define KP_MIN_BLOCKS 2
#endif

__global__ void __launch_bounds__(PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::THREADS, KP_MIN_BLOCKS)
    ks_chunks_keyprod(KsGeo g, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ I, const u64* __restrict__ d, u64 gal,
                      const u64* __restrict__ key, u64* __restrict__ acc) {
    using PG = PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>;
    extern __shared__ u64 sm[];
    const int t = blockIdx.y;
    const int pi = g.prime(t);
    const size_t N = (size_t)1 << g.logN;
    const PrimeDev P = primes[pi];
    PG G;
    G.init(g.N1);
    const ulonglong2* TW = tw + ((size_t)pi << g.logN);
    ulonglong2* twsm = PG::twsm_of(sm);
    stage_twiddles(G, twsm, TW, g.N1);
    cp_async_wait_all();
    __syncthreads();
    const size_t k0 = G.gidx(G.lt * 8);     // this thread's 8 consecutive output coefficients
    // digit values staged in registers; the 128-bit accumulators are then
    // short-lived (one pair of outputs at a time), which keeps the kernel at
    // 3 CTAs per SM
    u64 xs[KP_MAXB][8];
#pragma unroll
    for (int j = 0; j < KP_MAXB; j++) {
        if (j >= g.beta) break;
        const int lo = j * g.alpha, hi = min(lo + g.alpha, g.nl);
        if (t >= lo && t < hi) {
            if (gal) {
                LdGalois ld{d + (size_t)t * N, g.logN, gal};
                ld.load8(k0, xs[j]);
            } else {
                LdPlain ld{d + (size_t)t * N};
                ld.load8(k0, xs[j]);
            }
        } else {
            __syncthreads();
            LdPlain ld{I + ((size_t)j * g.nt + t) * N};
            StCapture st{xs[j]};
            ntt_pass<CH_LOG, MODE_CHUNKS, CH_SUBS, false, BOUND_LIM, BOUND_LIM>(G, sm, TW, P, ld, st, twsm, false);
        }
    }
    ulonglong2* o0 = reinterpret_cast<ulonglong2*>(acc + (size_t)t * N + k0);
    ulonglong2* o1 = reinterpret_cast<ulonglong2*>(acc + ((size_t)g.nt + t) * N + k0);
    const size_t kstride = (size_t)g.nall * N;
#pragma unroll
    for (int v = 0; v < 4; v++) {
        U128 b0 = {0, 0}, b1 = {0, 0}, a0 = {0, 0}, a1 = {0, 0};
#pragma unroll
        for (int j = 0; j < KP_MAXB; j++) {
            if (j >= g.beta) break;
            const u64* kb = key + ((size_t)(2 * j) * g.nall + pi) * N + k0 + 2 * v;
            const ulonglong2 kbv = *reinterpret_cast<const ulonglong2*>(kb);
            const ulonglong2 kav = *reinterpret_cast<const ulonglong2*>(kb + kstride);
            mac128(b0, xs[j][2 * v], kbv.x);
            mac128(b1, xs[j][2 * v + 1], kbv.y);
            mac128(a0, xs[j][2 * v], kav.x);
            mac128(a1, xs[j][2 * v + 1], kav.y);
        }
        o0[v] = make_ulonglong2(reduce128(b0.hi, b0.lo, P), reduce128(b1.hi, b1.lo, P));
        o1[v] = make_ulonglong2(reduce128(a0.hi, a0.lo, P), reduce128(a1.hi, a1.lo, P));
    }
}

// ---- B (split form): streaming key inner product over NTT-form digits -----
// UP[j][t] holds NTT(conv_j(t)) for t outside digit j; inside the digit the
// value is sigma(d)[t] itself, gathered on the fly.  Two coefficients per
// thread, 16-byte accesses, one Barrett reduction per output.

__global__ void __launch_bounds__(256) ks_keyprod_stream(KsGeo g, const PrimeDev* __restrict__ primes,
                                                         const u64* __restrict__ UP, const u64* __restrict__ d,
                                                         u64 gal, const u64* __restrict__ key,
                                                         u64* __restrict__ acc, int tlimit) {
    const size_t N = (size_t)1 << g.logN;
    const size_t total = (size_t)tlimit << (g.logN - 1);
    const size_t kstride = (size_t)g.nall * N;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < total; v += (size_t)gridDim.x * blockDim.x) {
        const int t = (int)(v >> (g.logN - 1));
        const size_t k = (v & ((N >> 1) - 1)) * 2;
        const int pi = g.prime(t);
        const PrimeDev P = primes[pi];
        // issue every load of the (up to KP_MAXB) digits before the first MAC
        u64 x0[KP_MAXB], x1[KP_MAXB];
        ulonglong2 kbv[KP_MAXB], kav[KP_MAXB];
#pragma unroll
        for (int j = 0; j < KP_MAXB; j++) {
            if (j >= g.beta) break;
            const int lo = j * g.alpha, hi = min(lo + g.alpha, g.nl);
            if (t >= lo && t < hi) {
                const u64* src = d + (size_t)t * N;
                if (gal) {
                    x0[j] = src[galois_src((unsigned)k, g.logN, gal)];
                    x1[j] = src[galois_src((unsigned)k + 1, g.logN, gal)];
                } else {
                    const ulonglong2 xv = *reinterpret_cast<const ulonglong2*>(src + k);
                    x0[j] = xv.x;
                    x1[j] = xv.y;
                }
            } else {
                const ulonglong2 xv = *reinterpret_cast<const ulonglong2*>(UP + ((size_t)j * g.nt + t) * N + k);
                x0[j] = xv.x;
                x1[j] = xv.y;
            }
            const u64* kb = key + ((size_t)(2 * j) * g.nall + pi) * N + k;
            kbv[j] = *reinterpret_cast<const ulonglong2*>(kb);
            kav[j] = *reinterpret_cast<const ulonglong2*>(kb + kstride);
        }
        ulonglong2 ob, oa;
        if (P.fp) {
            // FP64 products (q < 2^46): each term exact and centered (|r| < 0.6q),
            // the sum of <= 4 reduced once; digits are lazy words below 2q
            double sb0 = 0, sb1 = 0, sa0 = 0, sa1 = 0;
#pragma unroll
            for (int j = 0; j < KP_MAXB; j++) {
                if (j >= g.beta) break;
                const double y0 = fp_word(x0[j]), y1 = fp_word(x1[j]);
                sb0 = __dadd_rn(sb0, fp_mulmod(y0, fp_word(kbv[j].x), P.qd, P.qinv));
                sb1 = __dadd_rn(sb1, fp_mulmod(y1, fp_word(kbv[j].y), P.qd, P.qinv));
                sa0 = __dadd_rn(sa0, fp_mulmod(y0, fp_word(kav[j].x), P.qd, P.qinv));
                sa1 = __dadd_rn(sa1, fp_mulmod(y1, fp_word(kav[j].y), P.qd, P.qinv));
            }
            ob = make_ulonglong2(fp_canon(sb0, P.qd, P.qinv), fp_canon(sb1, P.qd, P.qinv));
            oa = make_ulonglong2(fp_canon(sa0, P.qd, P.qinv), fp_canon(sa1, P.qd, P.qinv));
        } else {
            U128 b0 = {0, 0}, b1 = {0, 0}, a0 = {0, 0}, a1 = {0, 0};
#pragma unroll
            for (int j = 0; j < KP_MAXB; j++) {
                if (j >= g.beta) break;
                mac128(b0, x0[j], kbv[j].x);
                mac128(b1, x1[j], kbv[j].y);
                mac128(a0, x0[j], kav[j].x);
                mac128(a1, x1[j], kav[j].y);
            }
            ob = make_ulonglong2(reduce128(b0.hi, b0.lo, P), reduce128(b1.hi, b1.lo, P));
            oa = make_ulonglong2(reduce128(a0.hi, a0.lo, P), reduce128(a1.hi, a1.lo, P));
        }
        *reinterpret_cast<ulonglong2*>(acc + (size_t)t * N + k) = ob;
        *reinterpret_cast<ulonglong2*>(acc + ((size_t)g.nt + t) * N + k) = oa;
    }
}

// ---- B2 for the P limbs: key product + the first (chunk) pass of their INTT --
// Each thread owns 8 consecutive coefficients, which are exactly the
// elements the inverse chunk pass's first round needs, so the products never
// leave registers before the transform.

struct LdRegs {
    const u64* x;
    __device__ __forceinline__ u64 operator()(size_t) const { return 0; }   // unused: edge is contiguous
    __device__ __forceinline__ void load8(size_t, u64* o) const {
#pragma unroll
        for (int e = 0; e < 8; e++) o[e] = x[e];
    }
};

__global__ void __launch_bounds__(PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::THREADS, PASS_MIN_BLOCKS)
    ks_keyprod_p_intt(KsGeo g, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ itw,
                      const u64* __restrict__ UP, const u64* __restrict__ key, u64* __restrict__ acc) {
    using PG = PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>;
    extern __shared__ u64 sm[];
    const int t = g.nl + blockIdx.y;            // P limb (never inside a Q digit)
    const int pi = g.prime(t);
    const size_t N = (size_t)1 << g.logN;
    const PrimeDev P = primes[pi];
    PG G;
    G.init(g.N1);
    const size_t k0 = G.gidx(G.lt * 8);
    const size_t kstride = (size_t)g.nall * N;
    u64 r0[8], r1[8];
#pragma unroll
    for (int v = 0; v < 4; v++) {
        U128 b0 = {0, 0}, b1 = {0, 0}, a0 = {0, 0}, a1 = {0, 0};
#pragma unroll
        for (int j = 0; j < KP_MAXB; j++) {
            if (j >= g.beta) break;
            const ulonglong2 xv =
                *reinterpret_cast<const ulonglong2*>(UP + ((size_t)j * g.nt + t) * N + k0 + 2 * v);
            const u64* kb = key + ((size_t)(2 * j) * g.nall + pi) * N + k0 + 2 * v;
            const ulonglong2 kbv = *reinterpret_cast<const ulonglong2*>(kb);
            const ulonglong2 kav = *reinterpret_cast<const ulonglong2*>(kb + kstride);
            mac128(b0, xv.x, kbv.x);
            mac128(b1, xv.y, kbv.y);
            mac128(a0, xv.x, kav.x);
            mac128(a1, xv.y, kav.y);
        }
        r0[2 * v] = reduce128(b0.hi, b0.lo, P);
        r0[2 * v + 1] = reduce128(b1.hi, b1.lo, P);
        r1[2 * v] = reduce128(a0.hi, a0.lo, P);
        r1[2 * v + 1] = reduce128(a1.hi, a1.lo, P);
    }
    const ulonglong2* TW = itw + ((size_t)pi << g.logN);
    {
        LdRegs ld{r0};
        StPlain<true, false> st{acc + (size_t)t * N, P.q, 0, 0};
        ntt_pass<CH_LOG, MODE_CHUNKS, CH_SUBS, true, 2, 2>(G, sm, TW, P, ld, st);
    }
    __syncthreads();
    {
        LdRegs ld{r1};
        StPlain<true, false> st{acc + ((size_t)g.nt + t) * N, P.q, 0, 0};
        ntt_pass<CH_LOG, MODE_CHUNKS, CH_SUBS, true, 2, 2>(G, sm, TW, P, ld, st);
    }
}

// ---- D: ModDown conversion fused into the column pass ----------------------

// (the P -> Q conversion has the ModUp loader's shape: K inputs, one target)
template <int LOGSZ, int SUBS, int NK>
__global__ void __launch_bounds__(PassGeo<LOGSZ, MODE_COLS, SUBS>::THREADS, PASS_MIN_BLOCKS)
    ks_moddown_cols(KsGeo g, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ acc, const u64* __restrict__ md_tab,
                    u64* __restrict__ Wt) {
    extern __shared__ u64 sm[];
    const int s = blockIdx.y / g.nl, i = blockIdx.y % g.nl;
    const size_t N = (size_t)1 << g.logN;
    const PrimeDev P = primes[i];
    const u64 q = P.q;
    LdModup<NK> ld;
    ld.na = g.K;
    ld.p = q;
#pragma unroll
    for (int t = 0; t < NK; t++) {
        const int tt = t < g.K ? t : 0;
        ld.y[t] = acc + ((size_t)s * g.nt + g.nl + tt) * N;
        ld.w[t] = md_tab[((size_t)tt * g.nall + i) * 2];
        ld.ws[t] = md_tab[((size_t)tt * g.nall + i) * 2 + 1];
    }
    StPlain<false, false> st{Wt + ((size_t)s * g.nl + i) * N, q, 0, 0};
    PassGeo<LOGSZ, MODE_COLS, SUBS> G;
    G.init(g.N1);
    const ulonglong2* TW = tw + ((size_t)i << g.logN);
    ulonglong2* twsm = PassGeo<LOGSZ, MODE_COLS, SUBS>::twsm_of(sm);
    stage_twiddles(G, twsm, TW, g.N1);
    ntt_pass<LOGSZ, MODE_COLS, SUBS, false, 2 * NK, BOUND_LIM>(G, sm, TW, P, ld, st, twsm, true);
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
    __device__ __forceinline__ void store8(size_t k, const u64* w) const {
        ulonglong2* o = reinterpret_cast<ulonglong2*>(out + k);
#pragma unroll
        for (int v = 0; v < 4; v++) o[v] = make_ulonglong2(one(k + 2 * v, w[2 * v]), one(k + 2 * v + 1, w[2 * v + 1]));
    }
};

__global__ void __launch_bounds__(PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::THREADS, PASS_MIN_BLOCKS)
    ks_moddown_chunks(KsGeo g, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ Wt, const u64* __restrict__ acc,
                      const u64* __restrict__ pinv, const u64* __restrict__ addend, int add_npoly, u64 add_gal,
                      const u64* __restrict__ addend2, u64* __restrict__ out) {
    extern __shared__ u64 sm[];
    const int s = blockIdx.y / g.nl, i = blockIdx.y % g.nl;
    const size_t N = (size_t)1 << g.logN;
    const PrimeDev P = primes[i];
    const u64 q = P.q;
    LdPlain ld{Wt + ((size_t)s * g.nl + i) * N};
    StModdown st{out + ((size_t)s * g.nl + i) * N, acc + ((size_t)s * g.nt + i) * N,
                 (s < add_npoly) ? addend + ((size_t)s * g.nl + i) * N : nullptr, q, pinv[2 * i], pinv[2 * i + 1],
                 add_gal, g.logN, addend2 ? addend2 + ((size_t)s * g.nl + i) * N : nullptr};
    PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS> G;
    G.init(g.N1);
    const ulonglong2* TW = tw + ((size_t)i << g.logN);
    ulonglong2* twsm = PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::twsm_of(sm);
    stage_twiddles(G, twsm, TW, g.N1);
    ntt_pass<CH_LOG, MODE_CHUNKS, CH_SUBS, false, BOUND_LIM, StModdown::MD_OUTB>(G, sm, TW, P, ld, st, twsm, true);
}

// ---- fused rescale (R1: bcast in the column pass, R2: combine in the chunk pass)

struct LdBcast {
    const u64* __restrict__ X;   // INTT of the dropped limb
    u64 ql, q, qlm;
    __device__ __forceinline__ u64 operator()(size_t k) const {
        const u64 v = X[k], vm = v % q;
        return v > (ql - 1) / 2 ? sub_mod(vm, qlm, q) : vm;
    }
    __device__ __forceinline__ void load8(size_t k, u64* x) const {
        for (int e = 0; e < 8; e++) x[e] = (*this)(k + e);
    }
};

template <int LOGSZ, int SUBS>
__global__ void __launch_bounds__(PassGeo<LOGSZ, MODE_COLS, SUBS>::THREADS, PASS_MIN_BLOCKS)
    rs_cols(int level, int logN, int N1, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ X, const u64* __restrict__ tab,
            u64* __restrict__ Yt) {
    extern __shared__ u64 sm[];
    const int s = blockIdx.y / level, i = blockIdx.y % level;
    const size_t N = (size_t)1 << logN;
    const PrimeDev P = primes[i];
    const u64 q = P.q;
    LdBcast ld{X + (size_t)s * N, primes[level].q, q, tab[3 * i + 2]};
    StPlain<false, false> st{Yt + ((size_t)s * level + i) * N, q, 0, 0};
    PassGeo<LOGSZ, MODE_COLS, SUBS> G;
    G.init(N1);
    const ulonglong2* TW = tw + ((size_t)i << logN);
    ulonglong2* twsm = PassGeo<LOGSZ, MODE_COLS, SUBS>::twsm_of(sm);
    stage_twiddles(G, twsm, TW, N1);
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
        ulonglong2* o = reinterpret_cast<ulonglong2*>(out + k);
#pragma unroll
        for (int v = 0; v < 4; v++) o[v] = make_ulonglong2(one(k + 2 * v, y[2 * v]), one(k + 2 * v + 1, y[2 * v + 1]));
    }
};

__global__ void __launch_bounds__(PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>::THREADS, PASS_MIN_BLOCKS)
    rs_chunks(int level, int logN, int N1, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, const u64* __restrict__ Yt, const u64* __restrict__ a,
              const u64* __restrict__ tab, u64* __restrict__ out) {
    extern __shared__ u64 sm[];
    const int s = blockIdx.y / level, i = blockIdx.y % level;
    const size_t N = (size_t)1 << logN;
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

template <class K>
static void set_smem(K kern, size_t bytes, bool& done) {
    if (!done) {
        HC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        done = true;
    }
}

// column-pass geometry per ring degree
template <int LOGN>
struct ColCfg;
template <> struct ColCfg<14> { static constexpr int LOGSZ = 5, SUBS = 64; };
template <> struct ColCfg<15> { static constexpr int LOGSZ = 6, SUBS = 32; };
template <> struct ColCfg<16> { static constexpr int LOGSZ = 7, SUBS = 16; };
template <> struct ColCfg<17> { static constexpr int LOGSZ = 8, SUBS = 8; };

template <int LOGN>
static void keyswitch_fused_t(Ctx& c, const u64* d, u64 gal, int level, const Key& key, u64* out,
                              const u64* addend, int add_npoly, u64 add_gal, const u64* addend2) {
    constexpr int CL = ColCfg<LOGN>::LOGSZ, CS = ColCfg<LOGN>::SUBS;
    using CG = PassGeo<CL, MODE_COLS, CS>;
    using HG = PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>;
    const int N = c.N, nl = level + 1, K = c.K, nt = nl + K;
    KsGeo g{level, nl, nt, c.L, K, c.alpha, c.dnum, c.nall, (nl + c.alpha - 1) / c.alpha, c.logN, N >> CH_LOG};
    const size_t csm = CG::smem_bytes(), hsm = HG::smem_bytes();

    // 1. Y = INTT(sigma(d)) * (Q'/q_i)^-1
    u64* Y = c.alloc((size_t)nl * N);
    {
        JobList j;
        j.n = nl;
        j.custom = 1;
        j.galois = gal;
        for (int i = 0; i < nl; i++) {
            const int dj = i / c.alpha, lo = dj * c.alpha, hi = std::min(lo + c.alpha, nl);
            const u64 qi = c.pr[i].q;
            u64 qh = 1;
            for (int b = lo; b < hi; b++) if (b != i) qh = mulm(qh, c.pr[b].q % qi, qi);
            const u64 sc = mulm(c.pr[i].ninv, powm(qh, qi - 2, qi), qi);
            j.prime[i] = i;
            j.ptr[i] = Y + (size_t)i * N;
            j.src[i] = d + (size_t)i * N;
            j.scale[i] = sc;
            j.scale_s[i] = shoup_of(sc, qi);
        }
        ntt_inverse(c, j);
    }
    // 2. A: conversion + column pass for every (digit, non-digit target)
    u64* I = c.alloc((size_t)g.beta * nt * N);
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
        static bool at = false;
        // algorithmic: the digit limbs Y read once, one intermediate limb written per job
        Launch scope(c, "ks_modup_cols", 8.0 * N * (nl + (double)jobs.n));
        dim3 grid((N >> CL) / CS, jobs.n);
        auto go = [&](auto kern) {
            set_smem(kern, csm, at);
            kern<<<grid, CG::THREADS, csm, c.stream>>>(jobs, g, c.d_primes, c.twp(0, false), Y, c.d_modup, I);
        };
        switch (c.alpha) {
            case 1: go(ks_modup_cols<CL, CS, 1>); break;
            case 2: go(ks_modup_cols<CL, CS, 2>); break;
            case 3: go(ks_modup_cols<CL, CS, 3>); break;
            default: go(ks_modup_cols<CL, CS, 4>); break;
        }
        HC_CUDA(cudaGetLastError());
    }
    c.free(Y);
    // 3. B: chunk pass + key inner product -> ACC [2][nt][N]
    u64* ACC = c.alloc((size_t)2 * nt * N);
    if (c.ks_split) {
        // split form: finish the NTTs of all (digit, target) limbs in one
        // launch, then stream the key product
        JobList j;
        j.n = 0;
        for (int dj = 0; dj < g.beta; dj++) {
            const int lo = dj * c.alpha, hi = std::min(lo + c.alpha, nl);
            for (int t = 0; t < nt; t++) {
                if (t >= lo && t < hi) continue;
                j.prime[j.n] = g.prime(t);
                j.ptr[j.n] = I + ((size_t)dj * nt + t) * N;
                j.src[j.n] = nullptr;
                j.n++;
            }
        }
        ntt_forward_chunks(c, j);
        // ks_split == 2: P limbs take the fused key-product + INTT-chunk kernel
        // (measured slower: a 96-CTA grid; kept as an option)
        const int tq = c.ks_split == 2 ? nl : nt;
        {
            const size_t work = (size_t)tq * (N / 2);
            Launch scope(c, "ks_keyprod_stream", 8.0 * N * ((double)g.beta * tq + 2.0 * g.beta * tq + 2.0 * tq));
            int blocks = (int)std::min<size_t>((work + 255) / 256, 148 * 16);
            ks_keyprod_stream<<<blocks, 256, 0, c.stream>>>(g, c.d_primes, I, d, gal, key.d, ACC, tq);
            HC_CUDA(cudaGetLastError());
        }
        if (c.ks_split == 2) {
            Launch scope(c, "ks_keyprod_p_intt", 8.0 * N * ((double)g.beta * K + 2.0 * g.beta * K + 2.0 * K));
            dim3 grid((N >> CH_LOG) / CH_SUBS, K);
            ks_keyprod_p_intt<<<grid, HG::THREADS, hsm, c.stream>>>(g, c.d_primes, c.twp(0, true), I, key.d, ACC);
            HC_CUDA(cudaGetLastError());
        }
    } else {
        static bool at = false;
        set_smem(ks_chunks_keyprod, hsm, at);
        const double inb = (double)g.beta * nt - nl + nl;      // I limbs + in-digit d limbs
        Launch scope(c, "ks_chunks_keyprod", 8.0 * N * (inb + 2.0 * g.beta * nt + 2.0 * nt));
        dim3 grid((N >> CH_LOG) / CH_SUBS, nt);
        ks_chunks_keyprod<<<grid, HG::THREADS, hsm, c.stream>>>(g, c.d_primes, c.twp(0, false), I, d, gal, key.d,
                                                                ACC);
        HC_CUDA(cudaGetLastError());
    }
    c.free(I);
    // 4. INTT of the P limbs, final scale N^-1 (P/p_t)^-1 (in place)
    {
        JobList j;
        j.n = 0;
        j.custom = 1;
        for (int s = 0; s < 2; s++)
            for (int t = 0; t < K; t++) {
                const int pi = c.L + 1 + t;
                const u64 p = c.pr[pi].q;
                u64 ph = 1;
                for (int b = 0; b < K; b++) if (b != t) ph = mulm(ph, c.pr[c.L + 1 + b].q % p, p);
                const u64 sc = mulm(c.pr[pi].ninv, powm(ph, p - 2, p), p);
                j.prime[j.n] = pi;
                j.ptr[j.n] = ACC + ((size_t)s * nt + nl + t) * N;
                j.src[j.n] = nullptr;
                j.scale[j.n] = sc;
                j.scale_s[j.n] = shoup_of(sc, p);
                j.n++;
            }
        if (c.ks_split == 2) ntt_inverse_cols(c, j);     // chunk pass already done in ks_keyprod_p_intt
        else ntt_inverse(c, j);
    }
    // 5. D: P -> Q conversion + column pass
    u64* Wt = c.alloc((size_t)2 * nl * N);
    {
        static bool at = false;
        Launch scope(c, "ks_moddown_cols", 8.0 * N * (2.0 * K + 2.0 * nl));
        dim3 grid((N >> CL) / CS, 2 * nl);
        auto go = [&](auto kern) {
            set_smem(kern, csm, at);
            kern<<<grid, CG::THREADS, csm, c.stream>>>(g, c.d_primes, c.twp(0, false), ACC, c.d_moddown, Wt);
        };
        switch (K) {
            case 1: go(ks_moddown_cols<CL, CS, 1>); break;
            case 2: go(ks_moddown_cols<CL, CS, 2>); break;
            case 3: go(ks_moddown_cols<CL, CS, 3>); break;
            default: go(ks_moddown_cols<CL, CS, 4>); break;
        }
        HC_CUDA(cudaGetLastError());
    }
    // 6. E: chunk pass + (ACC - W) P^-1 + addend
    {
        static bool at = false;
        set_smem(ks_moddown_chunks, hsm, at);
        Launch scope(c, "ks_moddown_chunks", 8.0 * N * (2.0 * nl * 3 + (double)add_npoly * nl));
        dim3 grid((N >> CH_LOG) / CH_SUBS, 2 * nl);
        ks_moddown_chunks<<<grid, HG::THREADS, hsm, c.stream>>>(g, c.d_primes, c.twp(0, false), Wt, ACC, c.d_pinv,
                                                                addend, add_npoly, add_gal, addend2, out);
        HC_CUDA(cudaGetLastError());
    }
    c.free(Wt);
    c.free(ACC);
}

bool keyswitch_fused(Ctx& c, const u64* d, u64 gal, int level, const Key& key, u64* out, const u64* addend,
                     int add_npoly, u64 add_gal, const u64* addend2) {
    if ((level + c.alpha) / c.alpha > KP_MAXB || c.K > 4 || c.alpha > 4) return false;
    switch (c.logN) {
        case 14: keyswitch_fused_t<14>(c, d, gal, level, key, out, addend, add_npoly, add_gal, addend2); return true;
        case 15: keyswitch_fused_t<15>(c, d, gal, level, key, out, addend, add_npoly, add_gal, addend2); return true;
        case 16: keyswitch_fused_t<16>(c, d, gal, level, key, out, addend, add_npoly, add_gal, addend2); return true;
        case 17: keyswitch_fused_t<17>(c, d, gal, level, key, out, addend, add_npoly, add_gal, addend2); return true;
        default: return false;
    }
}

template <int LOGN>
static void rescale_fused_t(Ctx& c, const u64* a, int level, int npoly, u64* out) {
    constexpr int CL = ColCfg<LOGN>::LOGSZ, CS = ColCfg<LOGN>::SUBS;
    using CG = PassGeo<CL, MODE_COLS, CS>;
    using HG = PassGeo<CH_LOG, MODE_CHUNKS, CH_SUBS>;
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
    u64* Yt = c.alloc((size_t)npoly * level * N);
    const u64* tab = c.d_rescale + (size_t)level * c.nall * 3;
    const size_t csm = CG::smem_bytes(), hsm = HG::smem_bytes();
    const int N1 = N >> CH_LOG;
    {
        static bool at = false;
        set_smem(rs_cols<CL, CS>, csm, at);
        Launch scope(c, "rs_cols", 8.0 * N * npoly * (1.0 + level));
        dim3 grid((N >> CL) / CS, npoly * level);
        rs_cols<CL, CS><<<grid, CG::THREADS, csm, c.stream>>>(level, c.logN, N1, c.d_primes, c.twp(0, false), X,
                                                              tab, Yt);
        HC_CUDA(cudaGetLastError());
    }
    {
        static bool at = false;
        set_smem(rs_chunks, hsm, at);
        Launch scope(c, "rs_chunks", 8.0 * N * npoly * 3.0 * level);
        dim3 grid((N >> CH_LOG) / CH_SUBS, npoly * level);
        rs_chunks<<<grid, HG::THREADS, hsm, c.stream>>>(level, c.logN, N1, c.d_primes, c.twp(0, false), Yt, a, tab,
                                                        out);
        HC_CUDA(cudaGetLastError());
    }
    c.free(X);
    c.free(Yt);
}

bool rescale_fused(Ctx& c, const u64* a, int level, int npoly, u64* out) {
    switch (c.logN) {
        case 14: rescale_fused_t<14>(c, a, level, npoly, out); return true;
        case 15: rescale_fused_t<15>(c, a, level, npoly, out); return true;
        case 16: rescale_fused_t<16>(c, a, level, npoly, out); return true;
        case 17: rescale_fused_t<17>(c, a, level, npoly, out); return true;
        default: return false;
    }
}

}  // namespace hc
