// One NTT pass as a device template with load / store hooks, so producers
// (base conversion, rescale broadcast, automorphism gather) run inside the
// first round's loads and consumers (key inner product, ModDown combine,
// rescale combine) inside the last round's stores.  See ntt.cu for the
// decomposition and conventions.
//
// Instruction economy (the pass is issue-bound on sm_100a): twiddles are
// stored as (w, w_shoup) pairs and fetched with one 16-byte load; every
// per-element address inside a butterfly group is base + m * stride with a
// compile-time stride (column stride 2^9, shared-memory padding of one word
// per 8 that stays linear inside a group), so the unrolled loops use
// immediate offsets.
#pragma once
#include "hc_internal.h"

namespace hc {

enum { MODE_FULL = 0, MODE_COLS = 1, MODE_CHUNKS = 2 };
constexpr int CHUNK_LOG = 9;   // chunk-pass size for split rings; = log2(column stride)
// resident 256-thread CTAs per SM the pass kernels are register-budgeted for
#ifndef PASS_MIN_BLOCKS
#define PASS_MIN_BLOCKS 4
#endif

template <int LOGSZ, int MODE, int SUBS>
struct PassGeo {
    static constexpr int SZ = 1 << LOGSZ;
    static constexpr int TPS = SZ / 8;
    static constexpr int NR = (LOGSZ + 2) / 3;
    static constexpr int PADSZ = SZ + SZ / 8;
    static constexpr int THREADS = SUBS * TPS;
    // split passes keep the 64-register budget at any CTA size; a full-ring
    // pass is bounded by its shared memory instead
    static constexpr int MIN_BLOCKS = (MODE != MODE_FULL || THREADS >= 256) ? PASS_MIN_BLOCKS * 256 / THREADS : 1;
    static constexpr size_t N2 = (size_t)1 << CHUNK_LOG;   // column stride (MODE_COLS)
    static constexpr size_t smem_words() { return (size_t)SUBS * (MODE == MODE_COLS ? SZ : PADSZ); }
    // data + staged twiddles.  Only column passes stage (their whole twiddle
    // set is SZ pairs, 2 KiB); a chunk pass needs ~one pair per element, and
    // front-loading 32 KiB per CTA measured slower than streaming them from L2.
    static constexpr bool STAGE_TW = (MODE == MODE_COLS);
    static constexpr size_t smem_bytes() { return smem_words() * 8 + (STAGE_TW ? (size_t)SZ * 16 : 0); }
    static __device__ __forceinline__ ulonglong2* twsm_of(u64* sm) {
        return STAGE_TW ? reinterpret_cast<ulonglong2*>(sm + smem_words()) : nullptr;
    }
    static constexpr bool EDGE_CONTIG = (MODE != MODE_COLS) && (LOGSZ % 3 == 0);
    int sub, lt, first_sub, R;
    __device__ __forceinline__ void init(int N1) {
        const int tid = threadIdx.x;
        if (MODE == MODE_COLS) { sub = tid % SUBS; lt = tid / SUBS; }
        else { sub = tid / TPS; lt = tid % TPS; }
        first_sub = blockIdx.x * SUBS;
        R = (MODE == MODE_CHUNKS) ? (N1 + first_sub + sub) : 1;
    }
    __device__ __forceinline__ size_t gidx(int pos) const {
        if (MODE == MODE_COLS) return (size_t)(first_sub + sub) + (size_t)pos * N2;
        return ((size_t)(first_sub + sub) << LOGSZ) + pos;
    }
    __device__ __forceinline__ int sidx(int pos) const {
        if (MODE == MODE_COLS) return pos * SUBS + sub;
        return sub * PADSZ + pos + (pos >> 3);
    }
    // twiddles staged in shared memory: the CTA's (w, w_shoup) pairs, per stage
    //   COLS / FULL (R = 1): entry widx = 2^s + i for widx < SZ
    //   CHUNKS: stage s holds SUBS * 2^s entries for this CTA's chunks
    static constexpr int TW_ENTRIES = (MODE == MODE_CHUNKS) ? SUBS * SZ : SZ;
    __device__ __forceinline__ int twl(int s, int i) const {   // i = index inside the stage for this sub
        if (MODE == MODE_CHUNKS) return SUBS * ((1 << s) - 1) + (sub << s) + i;
        return (1 << s) + i;
    }
    // strides of element m inside a group whose elements are u apart
    static constexpr size_t gstep(int u) { return MODE == MODE_COLS ? (size_t)u * N2 : (size_t)u; }
    static constexpr bool slinear(int u) { return MODE == MODE_COLS || u == 1 || u >= 8; }
    static constexpr int sstep(int u) { return MODE == MODE_COLS ? u * SUBS : (u == 1 ? 1 : u + u / 8); }
};

// ---- forward-pass reduction plan --------------------------------------------
// Every prime is below 2^60 (ctx_create enforces it), so a word holds any
// value below 16q.  A Cooley-Tukey butterfly maps operand bounds (X < Bq,
// any Y) to outputs below (B + 2)q, because the Shoup product is < 2q for any
// 64-bit Y.  Instead of Harvey's "reduce X below 2q in every stage" the plan
// lets the bound grow by 2q per stage and reduces X only when the next stage
// would pass 16q (one conditional subtraction of 8q: X < 8q, outputs < 10q).
// The pass's last stage reduces further when its consumer needs outputs below
// OUTB * q.  Bounds are uniform over the elements of a stage and known at
// compile time; the plan decides, per stage, how X is reduced:
//   RED_NONE, RED_8 (X < 8q), RED_2 (X < 2q via 8q / 4q / 2q subtractions).
enum { RED_NONE = 0, RED_8 = 1, RED_2 = 2 };
constexpr int BOUND_LIM = 16;
__host__ __device__ constexpr int fwd_red(int B, bool last, int outb) {
    const int lim = last && outb < BOUND_LIM ? outb : BOUND_LIM;
    return B + 2 <= lim ? RED_NONE : (10 <= lim ? RED_8 : RED_2);
}
__host__ __device__ constexpr int fwd_after(int B, int red) {
    return red == RED_NONE ? B + 2 : (red == RED_8 ? 10 : 4);
}
// bound (in units of q) before stage s of an nst-stage pass; s = nst gives the output bound
__host__ __device__ constexpr int fwd_bound(int inb, int nst, int outb, int s) {
    int B = inb;
    for (int i = 0; i < s; i++) B = fwd_after(B, fwd_red(B, i == nst - 1, outb));
    return B;
}
// x < B q (B <= 16)  ->  x < T q (T in {1, 2, 4, 8}) by conditional subtractions of 8q, 4q, 2q, q
__device__ __forceinline__ u64 reduce_to(u64 x, u64 q, int B, int T) {
    if (B > 8 && T <= 8) x = x >= 8 * q ? x - 8 * q : x;
    if (B > 4 && T <= 4) x = x >= 4 * q ? x - 4 * q : x;
    if (B > 2 && T <= 2) x = x >= 2 * q ? x - 2 * q : x;
    if (B > 1 && T <= 1) x = x >= q ? x - q : x;
    return x;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Issue the asynchronous copy of this CTA's twiddles into shared memory
// (completed by cp_async_wait_all + __syncthreads, which ntt_pass does after
// its first-round data loads when tw_pending is set).
template <int LOGSZ, int MODE, int SUBS>
__device__ __forceinline__ void stage_twiddles(const PassGeo<LOGSZ, MODE, SUBS>& G, ulonglong2* twsm,
                                               const ulonglong2* __restrict__ TW, int N1) {
    using PG = PassGeo<LOGSZ, MODE, SUBS>;
    const int tid = threadIdx.x;
    if (!twsm) return;
    if (MODE == MODE_CHUNKS) {
#pragma unroll 1
        for (int s = 0; s < LOGSZ; s++) {
            const int cnt = SUBS << s;
            const ulonglong2* src = TW + ((size_t)(N1 + G.first_sub) << s);
            ulonglong2* dst = twsm + SUBS * ((1 << s) - 1);
            for (int i = tid; i < cnt; i += PG::THREADS) cp_async16(dst + i, src + i);
        }
    } else {
        for (int i = tid; i < PG::SZ; i += PG::THREADS) cp_async16(twsm + i, TW + i);
    }
}

// ---- butterfly arithmetic policies ------------------------------------------
//
// ArInt: 64-bit words, Shoup products, the reduction plan above (any prime
// below 2^60).
//
// ArFp: primes below 2^46 run in FP64 (the B200 FP64 pipe issues DFMA at the
// IMAD rate, and one butterfly is 8 FP64 instructions instead of ~30 integer
// ones).  Residues are integers held exactly in doubles, signed and lazy.  The
// product of x (|x| < 32q) by a twiddle w is exact as h + l (h = x*w rounded,
// l = fma(x, w, -h)); the quotient is rint(x * w/q) with w/q precomputed, off
// the true x*w/q by at most 0.75, so T = (h - qt*q) + l is exact with
// |T| <= 0.75q.  Forward outputs grow by 0.75q per stage (no reduction in a
// pass of <= 13 stages from inputs below 16q); inverse sums double per stage
// and are reduced (|v| <= q/2) when they would pass 16q.  Pass boundaries
// stay integer: words in, lazy words in [0, 2q) out, so every load / store
// hook is shared with the integer path and results are bit-identical.
template <int LOGSZ, int INB, int OUTB>
struct ArInt {
    using V = u64;
    using W = ulonglong2;
    static constexpr bool IS_FP = false;
    u64 q, twoq;
    __device__ __forceinline__ ArInt(const PrimeDev& P) : q(P.q), twoq(2 * P.q) {}
    __device__ __forceinline__ V in(u64 u) const { return u; }
    __device__ __forceinline__ u64 out(V v) const { return v; }
    __device__ __forceinline__ void fwd(V& a, V& b, const W& w, int st) const {
        const int B = fwd_bound(INB, LOGSZ, OUTB, st);
        const int red = fwd_red(B, st == LOGSZ - 1, OUTB);
        u64 X = a;
        if (red == RED_8) X = reduce_to(X, q, B, 8);
        else if (red == RED_2) X = reduce_to(X, q, B, 2);
        const u64 T = mul_shoup_lazy(b, w.x, w.y, q);
        a = X + T;
        b = X + twoq - T;
    }
    __device__ __forceinline__ void inv(V& a, V& b, const W& w, int) const {
        const u64 X = a + b;
        const u64 D = a + twoq - b;
        a = X >= twoq ? X - twoq : X;
        b = mul_shoup_lazy(D, w.x, w.y, q);
    }
};


// inverse: reduce the sums of executed stage e (bounds in units of q; inputs below 2q)
__host__ __device__ constexpr bool fp_inv_red(int e) {
    int B = 2;
    for (int i = 0; i < e; i++) B = (2 * B > 16) ? 1 : 2 * B;
    return 2 * B > 16;
}

template <int LOGSZ, int INB, int OUTB>
struct ArFp {
    using V = double;
    using W = double2;   // (w, w / q)
    static constexpr bool IS_FP = true;
    double q, qinv, qp52;
    static_assert(4 * INB + 3 * LOGSZ <= 4 * 32, "FP forward pass bound");
    __device__ __forceinline__ ArFp(const PrimeDev& P) : q(P.qd), qinv(P.qinv), qp52(P.qd + FP_P52) {}
    __device__ __forceinline__ V in(u64 u) const { return fp_word(u); }
    // |v| < 32q -> centered remainder (|r| <= q/2) -> word in [0, 2q)
    __device__ __forceinline__ double red(double v) const {
        const double qt = __dsub_rn(__fma_rn(v, qinv, FP_MAGIC), FP_MAGIC);
        return __fma_rn(-qt, q, v);
    }
    __device__ __forceinline__ u64 out(V v) const {
        return (u64)__double_as_longlong(__dadd_rn(red(v), qp52)) & FP_MANT;
    }
    __device__ __forceinline__ double mm(double x, const W& w) const {
        const double h = __dmul_rn(x, w.x);
        const double l = __fma_rn(x, w.x, -h);
        const double qt = __dsub_rn(__fma_rn(x, w.y, FP_MAGIC), FP_MAGIC);
        return __dadd_rn(__fma_rn(-qt, q, h), l);
    }
    __device__ __forceinline__ void fwd(V& a, V& b, const W& w, int) const {
        const double T = mm(b, w);
        const double X = a;
        a = __dadd_rn(X, T);
        b = __dsub_rn(X, T);
    }
    __device__ __forceinline__ void inv(V& a, V& b, const W& w, int st) const {
        const double X = __dadd_rn(a, b);
        const double D = __dsub_rn(a, b);
        a = fp_inv_red(LOGSZ - 1 - st) ? red(X) : X;
        b = mm(D, w);
    }
};

enum { TW_JIT = 0, TW_ROUND = 1, TW_PREFETCH = 2 };
#ifndef FP_CHUNK_TW
#define FP_CHUNK_TW TW_PREFETCH
#endif

// Runs the pass.  LD: u64 operator()(size_t gidx) and void load8(size_t gidx, u64* x)
// (8 consecutive words, only used when EDGE_CONTIG).  ST: void operator()(size_t gidx, u64 v)
// and store8(size_t gidx, const u64* x).  Forward: LD words are below INB * q and the
// words handed to ST below OUTB * q (integer: the reduction plan above; FP64: [0, 2q)).
// Inverse: LD words below 2q, ST words below 2q.  TW: the prime's twiddle pairs,
// (w, w_shoup) words or, for FP64 primes, (w, w/q) doubles.
template <class AR, int LOGSZ, int MODE, int SUBS, bool INV, class LD, class ST>
__device__ __forceinline__ void ntt_pass_ar(const AR& ar, const PassGeo<LOGSZ, MODE, SUBS>& G, u64* smw,
                                            const ulonglong2* __restrict__ TWw, LD& ld, ST& st,
                                            const ulonglong2* twsmw, bool tw_pending) {
    using PG = PassGeo<LOGSZ, MODE, SUBS>;
    using V = typename AR::V;
    using W = typename AR::W;
    V* sm = reinterpret_cast<V*>(smw);
    const W* __restrict__ TW = reinterpret_cast<const W*>(TWw);
    const W* twsm = reinterpret_cast<const W*>(twsmw);
    V x[8];
    // one 16-byte load per twiddle pair; round rdx's pairs in stage order
    auto twload = [&](int rdx, W* out) {
        const int fr = INV ? (PG::NR - 1 - rdx) : rdx;
        const int s0 = 3 * fr;
        const int r = (LOGSZ - s0) < 3 ? (LOGSZ - s0) : 3;
        const int logu = LOGSZ - s0 - r;
        const int NG = 8 >> r;
        int n = 0;
#pragma unroll
        for (int j = 0; j < NG; j++) {
            const int blk = (G.lt + j * PG::TPS) >> logu;
            const int B0 = G.R * (1 << s0) + blk;
#pragma unroll
            for (int qq = 0; qq < r; qq++) {
                if (twsm) {
                    const W* tp = twsm + G.twl(s0 + qq, blk << qq);
#pragma unroll
                    for (int sb = 0; sb < (1 << qq); sb++) out[n++] = tp[sb];
                } else {
                    const W* tp = TW + (B0 << qq);
#pragma unroll
                    for (int sb = 0; sb < (1 << qq); sb++) out[n++] = tp[sb];
                }
            }
        }
    };
    // the (1 << qq) pairs of group j, stage qq of round rdx (just-in-time loads)
    auto twgroup = [&](int rdx, int j, int qq, W* out) {
        const int fr = INV ? (PG::NR - 1 - rdx) : rdx;
        const int s0 = 3 * fr;
        const int r = (LOGSZ - s0) < 3 ? (LOGSZ - s0) : 3;
        const int logu = LOGSZ - s0 - r;
        const int blk = (G.lt + j * PG::TPS) >> logu;
        const W* tp = twsm ? twsm + G.twl(s0 + qq, blk << qq) : TW + ((G.R * (1 << s0) + blk) << qq);
#pragma unroll
        for (int sb = 0; sb < (1 << qq); sb++) out[sb] = tp[sb];
    };
    // twiddle schedule: TW_PREFETCH issues the next round's pairs before the
    // shared-memory exchange (integer path; FP64 chunk passes, whose pairs come
    // from L2); TW_ROUND loads a round's pairs at its start; TW_JIT loads each
    // stage's pairs just before it (FP64 column passes: staged in shared
    // memory, and the register budget has no room for two rounds of pairs)
    constexpr int TWM = !AR::IS_FP ? TW_PREFETCH : (MODE == MODE_COLS ? TW_JIT : FP_CHUNK_TW);
    W tw_r[7], tw_n[7];
#pragma unroll
    for (int rd = 0; rd < PG::NR; rd++) {
        const int fr = INV ? (PG::NR - 1 - rd) : rd;
        const int s0 = 3 * fr;
        const int r = (LOGSZ - s0) < 3 ? (LOGSZ - s0) : 3;
        const int logu = LOGSZ - s0 - r;
        const int u = 1 << logu;
        const int NG = 8 >> r;
        const int GS = 1 << r;
        // ---- load ----
#pragma unroll
        for (int j = 0; j < NG; j++) {
            const int g = G.lt + j * PG::TPS;
            const int base = ((g >> logu) << (logu + r)) + (g & (u - 1));
            if (rd == 0) {
                const size_t gb = G.gidx(base);
                if (PG::EDGE_CONTIG && logu == 0 && r == 3) {
                    u64 w8[8];
                    ld.load8(gb, w8);
#pragma unroll
                    for (int m = 0; m < 8; m++) x[8 * j + m] = ar.in(w8[m]);
                } else {
#pragma unroll
                    for (int m = 0; m < GS; m++) x[j * GS + m] = ar.in(ld(gb + m * PG::gstep(u)));
                }
            } else if (PG::slinear(u)) {
                const V* sp = sm + G.sidx(base);
#pragma unroll
                for (int m = 0; m < GS; m++) x[j * GS + m] = sp[m * PG::sstep(u)];
            } else {
#pragma unroll
                for (int m = 0; m < GS; m++) x[j * GS + m] = sm[G.sidx(base + (m << logu))];
            }
        }
        if (rd == 0 && tw_pending) {
            cp_async_wait_all();
            __syncthreads();
        }
        // ---- twiddles: round 0's now; with PREFETCH_TW every later round's were
        // issued at the end of the previous round, ahead of its shared-memory exchange ----
        if ((rd == 0 && TWM == TW_PREFETCH) || TWM == TW_ROUND) twload(rd, tw_r);
        // ---- butterflies ----
#pragma unroll
        for (int j = 0; j < NG; j++) {
            V* y = x + j * GS;
            const int gbase = j * (GS - 1);
            if (!INV) {
#pragma unroll
                for (int qq = 0; qq < r; qq++) {
                    const int half = 1 << (r - 1 - qq);
                    W ts[4];
                    if (TWM == TW_JIT) twgroup(rd, j, qq, ts);
#pragma unroll
                    for (int m1 = 0; m1 < GS; m1++) {
                        if (m1 & half) continue;
                        const W& w = TWM != TW_JIT ? tw_r[gbase + ((1 << qq) - 1) + (m1 >> (r - qq))]
                                                     : ts[m1 >> (r - qq)];
                        ar.fwd(y[m1], y[m1 + half], w, s0 + qq);
                    }
                }
            } else {
#pragma unroll
                for (int qq = r - 1; qq >= 0; qq--) {
                    const int half = 1 << (r - 1 - qq);
                    W ts[4];
                    if (TWM == TW_JIT) twgroup(rd, j, qq, ts);
#pragma unroll
                    for (int m1 = 0; m1 < GS; m1++) {
                        if (m1 & half) continue;
                        const W& w = TWM != TW_JIT ? tw_r[gbase + ((1 << qq) - 1) + (m1 >> (r - qq))]
                                                     : ts[m1 >> (r - qq)];
                        ar.inv(y[m1], y[m1 + half], w, s0 + qq);
                    }
                }
            }
        }
        // ---- next round's twiddles in flight during the exchange below ----
        if (TWM == TW_PREFETCH && rd + 1 < PG::NR) twload(rd + 1, tw_n);
        // ---- store ----
        const bool last = (rd == PG::NR - 1);
#pragma unroll
        for (int j = 0; j < NG; j++) {
            const int g = G.lt + j * PG::TPS;
            const int base = ((g >> logu) << (logu + r)) + (g & (u - 1));
            if (last) {
                const size_t gb = G.gidx(base);
                if (PG::EDGE_CONTIG && logu == 0 && r == 3) {
                    u64 w8[8];
#pragma unroll
                    for (int m = 0; m < 8; m++) w8[m] = ar.out(x[8 * j + m]);
                    st.store8(gb, w8);
                } else {
#pragma unroll
                    for (int m = 0; m < GS; m++) st(gb + m * PG::gstep(u), ar.out(x[j * GS + m]));
                }
            } else if (PG::slinear(u)) {
                V* sp = sm + G.sidx(base);
#pragma unroll
                for (int m = 0; m < GS; m++) sp[m * PG::sstep(u)] = x[j * GS + m];
            } else {
#pragma unroll
                for (int m = 0; m < GS; m++) sm[G.sidx(base + (m << logu))] = x[j * GS + m];
            }
        }
        if (!last) {
            __syncthreads();
            if (TWM == TW_PREFETCH) {
#pragma unroll
                for (int e = 0; e < 7; e++) tw_r[e] = tw_n[e];
            }
        }
    }
}

// The pass on prime P: FP64 arithmetic for primes below 2^FP_MAXBITS (P.fp),
// integer otherwise (branch uniform per CTA).
template <int LOGSZ, int MODE, int SUBS, bool INV, int INB, int OUTB, class LD, class ST>
__device__ __forceinline__ void ntt_pass(const PassGeo<LOGSZ, MODE, SUBS>& G, u64* sm,
                                         const ulonglong2* __restrict__ TW, const PrimeDev& P, LD& ld, ST& st,
                                         const ulonglong2* twsm = nullptr, bool tw_pending = false) {
#if defined(HC_ONLY_INT)
    if (false) {
#elif defined(HC_ONLY_FP)
    if (true) {
#else
    if (P.fp) {
#endif
        const ArFp<LOGSZ, INB, OUTB> ar(P);
        ntt_pass_ar<ArFp<LOGSZ, INB, OUTB>, LOGSZ, MODE, SUBS, INV>(ar, G, sm, TW, ld, st, twsm, tw_pending);
    } else {
        const ArInt<LOGSZ, INB, OUTB> ar(P);
        ntt_pass_ar<ArInt<LOGSZ, INB, OUTB>, LOGSZ, MODE, SUBS, INV>(ar, G, sm, TW, ld, st, twsm, tw_pending);
    }
}

// ---- compact pass (sub-wave launches) ------------------------------------------
//
// The radix-8 pass above is straight-line code: ~1000 instructions (16-20 KB)
// per arithmetic path, executed once per warp.  In a launch that does not
// fill the machine (the INTTs of a lone ciphertext in the softmax /
// inversion chains, the 6 special-prime limbs of a ModDown) every SM streams
// that code from L2 for a handful of warps, and ncu shows instruction fetch
// (`no_instruction`) as the top stall: 12-15 us per pass for work that moves
// 3 MB.  The compact pass is the same transform as a loop: four words per
// thread and two stages (radix 4) per iteration, every iteration through
// shared memory (one barrier each), the CTA's twiddle pairs staged once by
// cp.async, loads and stores coalesced through the shared tile.  ~300
// instructions per arithmetic path, twice the threads per sub-transform; same
// load / store hooks, same twiddle tables, bit-identical residues.  Lazy
// bounds are uniform instead of planned: integer forward values stay below 4q
// (Harvey), FP64 values follow the growth rules above with the inverse
// reductions on a compile-time mask.  An odd stage count runs stage 0 alone.
template <int LOGSZ, int MODE, int SUBS>
struct SmallGeo {
    static constexpr int SZ = 1 << LOGSZ;
    static constexpr int Q = SZ / 4;
    static constexpr int THREADS = SUBS * Q;
    static constexpr size_t N2 = (size_t)1 << CHUNK_LOG;
    static constexpr int TW_ENTRIES = (MODE == MODE_CHUNKS) ? SUBS * SZ : SZ;
    // padding (bank conflicts of the stride-4^k groups): columns interleave
    // SUBS sub-transforms per position, chunks lay them out one after another
    static constexpr int PADSZ = (MODE == MODE_COLS) ? (SUBS >= 16 ? SZ : SZ + SZ / 4) : SZ + 3 * (SZ / 16);
    static constexpr size_t smem_words() { return (size_t)SUBS * PADSZ; }
    static constexpr size_t smem_bytes() { return smem_words() * 8 + (size_t)TW_ENTRIES * 16; }
    static __device__ __forceinline__ ulonglong2* twsm_of(u64* sm) {
        return reinterpret_cast<ulonglong2*>(sm + smem_words());
    }
    int sub, g, first_sub, R;
    __device__ __forceinline__ void init(int N1) {
        const int tid = threadIdx.x;
        if (MODE == MODE_COLS) { sub = tid % SUBS; g = tid / SUBS; }
        else { sub = tid / Q; g = tid % Q; }
        first_sub = blockIdx.x * SUBS;
        R = (MODE == MODE_CHUNKS) ? (N1 + first_sub + sub) : 1;
    }
    __device__ __forceinline__ size_t gidx(int pos) const {
        if (MODE == MODE_COLS) return (size_t)(first_sub + sub) + (size_t)pos * N2;
        return ((size_t)(first_sub + sub) << LOGSZ) + pos;
    }
    __device__ __forceinline__ int sidx(int pos) const {
        if (MODE == MODE_COLS) return (SUBS >= 16 ? pos : pos + (pos >> 2)) * SUBS + sub;
        return sub * PADSZ + pos + 3 * (pos >> 4);
    }
    __device__ __forceinline__ int twl(int s, int i) const {
        if (MODE == MODE_CHUNKS) return SUBS * ((1 << s) - 1) + (sub << s) + i;
        return (1 << s) + i;
    }
};

template <int LOGSZ, int MODE, int SUBS>
__device__ __forceinline__ void stage_twiddles_small(const SmallGeo<LOGSZ, MODE, SUBS>& G, ulonglong2* twsm,
                                                     const ulonglong2* __restrict__ TW, int N1) {
    using SG = SmallGeo<LOGSZ, MODE, SUBS>;
    const int tid = threadIdx.x;
    if (MODE == MODE_CHUNKS) {
#pragma unroll 1
        for (int s = 0; s < LOGSZ; s++) {
            const int cnt = SUBS << s;
            const ulonglong2* src = TW + ((size_t)(N1 + G.first_sub) << s);
            ulonglong2* dst = twsm + SUBS * ((1 << s) - 1);
            for (int i = tid; i < cnt; i += SG::THREADS) cp_async16(dst + i, src + i);
        }
    } else {
        for (int i = tid; i < SG::SZ; i += SG::THREADS) cp_async16(twsm + i, TW + i);
    }
}

// uniform-bound butterflies for the looped stages
template <int INB>
struct SmInt {
    using V = u64;
    using W = ulonglong2;
    u64 q, twoq;
    __device__ __forceinline__ SmInt(const PrimeDev& P) : q(P.q), twoq(2 * P.q) {}
    // forward input below INB q -> below 4q; inverse inputs are below 2q already
    __device__ __forceinline__ V in(u64 u, bool inv) const { return inv ? u : reduce_to(u, q, INB, 4); }
    __device__ __forceinline__ u64 out(V v) const { return v; }   // fwd < 4q, inv < 2q
    __device__ __forceinline__ void fwd(V& a, V& b, const W& w) const {
        const u64 X = a >= twoq ? a - twoq : a;
        const u64 T = mul_shoup_lazy(b, w.x, w.y, q);
        a = X + T;
        b = X + twoq - T;
    }
    __device__ __forceinline__ void inv(V& a, V& b, const W& w, int) const {
        const u64 X = a + b;
        const u64 D = a + twoq - b;
        a = X >= twoq ? X - twoq : X;
        b = mul_shoup_lazy(D, w.x, w.y, q);
    }
};
template <int LOGSZ>
__host__ __device__ constexpr unsigned fp_inv_red_mask() {
    unsigned m = 0;
    for (int e = 0; e < LOGSZ; e++) m |= fp_inv_red(e) ? (1u << e) : 0u;
    return m;
}
template <int LOGSZ, int INB>
struct SmFp {
    using V = double;
    using W = double2;
    double q, qinv, qp52;
    static_assert(4 * INB + 3 * LOGSZ <= 4 * 32, "FP forward pass bound");
    __device__ __forceinline__ SmFp(const PrimeDev& P) : q(P.qd), qinv(P.qinv), qp52(P.qd + FP_P52) {}
    __device__ __forceinline__ V in(u64 u, bool) const { return fp_word(u); }
    __device__ __forceinline__ double red(double v) const {
        const double qt = __dsub_rn(__fma_rn(v, qinv, FP_MAGIC), FP_MAGIC);
        return __fma_rn(-qt, q, v);
    }
    __device__ __forceinline__ u64 out(V v) const {
        return (u64)__double_as_longlong(__dadd_rn(red(v), qp52)) & FP_MANT;
    }
    __device__ __forceinline__ double mm(double x, const W& w) const {
        const double h = __dmul_rn(x, w.x);
        const double l = __fma_rn(x, w.x, -h);
        const double qt = __dsub_rn(__fma_rn(x, w.y, FP_MAGIC), FP_MAGIC);
        return __dadd_rn(__fma_rn(-qt, q, h), l);
    }
    __device__ __forceinline__ void fwd(V& a, V& b, const W& w) const {
        const double T = mm(b, w);
        const double X = a;
        a = __dadd_rn(X, T);
        b = __dsub_rn(X, T);
    }
    // e = ordinal of the executed inverse stage (0 first)
    __device__ __forceinline__ void inv(V& a, V& b, const W& w, int e) const {
        const double X = __dadd_rn(a, b);
        const double D = __dsub_rn(a, b);
        a = ((fp_inv_red_mask<LOGSZ>() >> e) & 1u) ? red(X) : X;
        b = mm(D, w);
    }
};

template <class AR, int LOGSZ, int MODE, int SUBS, bool INV, class LD, class ST>
__device__ __forceinline__ void ntt_pass_small_ar(const AR& ar, const SmallGeo<LOGSZ, MODE, SUBS>& G, u64* smw,
                                                  LD& ld, ST& st) {
    using SG = SmallGeo<LOGSZ, MODE, SUBS>;
    using V = typename AR::V;
    using W = typename AR::W;
    V* sm = reinterpret_cast<V*>(smw);
    const W* twsm = reinterpret_cast<const W*>(SG::twsm_of(smw));
    const int g = G.g;
    constexpr int ODD = LOGSZ & 1;
    // coalesced loads of positions g + m SZ/4 into the shared tile
    {
        u64 w[4];
#pragma unroll
        for (int m = 0; m < 4; m++) w[m] = ld(G.gidx(g + m * SG::Q));
#pragma unroll
        for (int m = 0; m < 4; m++) sm[G.sidx(g + m * SG::Q)] = ar.in(w[m], INV);
    }
    cp_async_wait_all();
    __syncthreads();
    // stage 0 alone (odd stage counts): pairs (g + m SZ/4, g + (m + 2) SZ/4), one twiddle
    auto lone_stage = [&]() {
        V x[4];
        int ix[4];
#pragma unroll
        for (int m = 0; m < 4; m++) { ix[m] = G.sidx(g + m * SG::Q); x[m] = sm[ix[m]]; }
        const W w = twsm[G.twl(0, 0)];
        if (INV) { ar.inv(x[0], x[2], w, LOGSZ - 1); ar.inv(x[1], x[3], w, LOGSZ - 1); }
        else { ar.fwd(x[0], x[2], w); ar.fwd(x[1], x[3], w); }
#pragma unroll
        for (int m = 0; m < 4; m++) sm[ix[m]] = x[m];
        __syncthreads();
    };
    if (!INV && ODD) lone_stage();
    // stages (s, s + 1) per iteration: words base + m u2, u2 = SZ >> (s + 2)
#pragma unroll 1
    for (int it = 0; it < LOGSZ / 2; it++) {
        const int s = INV ? (LOGSZ - 2 - 2 * it) : (ODD + 2 * it);
        const int logu2 = LOGSZ - 2 - s;
        const int blk = g >> logu2;
        const int base = (blk << (logu2 + 2)) + (g & ((1 << logu2) - 1));
        V x[4];
        int ix[4];
#pragma unroll
        for (int m = 0; m < 4; m++) { ix[m] = G.sidx(base + (m << logu2)); x[m] = sm[ix[m]]; }
        const W wa = twsm[G.twl(s, blk)];
        const W* tb = twsm + G.twl(s + 1, 2 * blk);
        const W wb0 = tb[0], wb1 = tb[1];
        if (INV) {
            ar.inv(x[0], x[1], wb0, 2 * it);
            ar.inv(x[2], x[3], wb1, 2 * it);
            ar.inv(x[0], x[2], wa, 2 * it + 1);
            ar.inv(x[1], x[3], wa, 2 * it + 1);
        } else {
            ar.fwd(x[0], x[2], wa);
            ar.fwd(x[1], x[3], wa);
            ar.fwd(x[0], x[1], wb0);
            ar.fwd(x[2], x[3], wb1);
        }
#pragma unroll
        for (int m = 0; m < 4; m++) sm[ix[m]] = x[m];
        __syncthreads();
    }
    if (INV && ODD) lone_stage();
#pragma unroll
    for (int m = 0; m < 4; m++) st(G.gidx(g + m * SG::Q), ar.out(sm[G.sidx(g + m * SG::Q)]));
}

// The compact pass on prime P.  INB as for ntt_pass; forward outputs are
// below 4q (integer) / 2q (FP64), inverse outputs below 2q.  The caller has
// issued stage_twiddles_small before its pdl_wait.
template <int LOGSZ, int MODE, int SUBS, bool INV, int INB, class LD, class ST>
__device__ __forceinline__ void ntt_pass_small(const SmallGeo<LOGSZ, MODE, SUBS>& G, u64* sm, const PrimeDev& P,
                                               LD& ld, ST& st) {
    if (P.fp) {
        const SmFp<LOGSZ, INB> ar(P);
        ntt_pass_small_ar<SmFp<LOGSZ, INB>, LOGSZ, MODE, SUBS, INV>(ar, G, sm, ld, st);
    } else {
        const SmInt<INB> ar(P);
        ntt_pass_small_ar<SmInt<INB>, LOGSZ, MODE, SUBS, INV>(ar, G, sm, ld, st);
    }
}

// One compact pass inside a multi-phase (cooperative) kernel: the shared tile
// is reused from phase to phase, so the CTA synchronises, stages this
// sub-transform's twiddles and runs the pass.
template <int LOGSZ, int MODE, int SUBS, bool INV, int INB, class LD, class ST>
__device__ __forceinline__ void small_pass_run(int N1, int xblock, u64* sm, const ulonglong2* __restrict__ TW,
                                               const PrimeDev& P, LD& ld, ST& st) {
    using SG = SmallGeo<LOGSZ, MODE, SUBS>;
    SG G;
    G.init(N1);
    G.first_sub = xblock * SUBS;
    if (MODE == MODE_CHUNKS) G.R = N1 + G.first_sub + G.sub;
    __syncthreads();
    stage_twiddles_small<LOGSZ, MODE, SUBS>(G, SG::twsm_of(sm), TW, N1);
    ntt_pass_small<LOGSZ, MODE, SUBS, INV, INB>(G, sm, P, ld, st);
}

// L2 loads for words written earlier in the same kernel by other CTAs
struct LdCg {
    const u64* p;
    __device__ __forceinline__ u64 operator()(size_t i) const { return __ldcg(p + i); }
};

// ---- common hooks ----

struct LdPlain {
    const u64* __restrict__ p;
    __device__ __forceinline__ u64 operator()(size_t i) const { return p[i]; }
    __device__ __forceinline__ void load8(size_t i, u64* x) const {
        const ulonglong2* v = reinterpret_cast<const ulonglong2*>(p + i);
#pragma unroll
        for (int k = 0; k < 4; k++) { ulonglong2 t = v[k]; x[2 * k] = t.x; x[2 * k + 1] = t.y; }
    }
};

// final store: fwd reduce [0,4q) -> [0,q); inv multiply by a per-limb constant (N^-1 [* c])
template <bool INV, bool FINAL>
struct StPlain {
    u64* __restrict__ p;
    u64 q, c, cs;
    u64 off = 0;   // inverse final store: + off mod q (the centred base conversion's shift)
    __device__ __forceinline__ u64 fin(u64 v) const {
        if (!FINAL) return v;
        if (INV) return csub(mul_shoup(v, c, cs, q) + off, q);
        v = v >= 2 * q ? v - 2 * q : v;
        return v >= q ? v - q : v;
    }
    __device__ __forceinline__ void operator()(size_t i, u64 v) const { p[i] = fin(v); }
    __device__ __forceinline__ void store8(size_t i, const u64* x) const {
        ulonglong2* v = reinterpret_cast<ulonglong2*>(p + i);
#pragma unroll
        for (int k = 0; k < 4; k++) v[k] = make_ulonglong2(fin(x[2 * k]), fin(x[2 * k + 1]));
    }
};

// NTT-domain Galois permutation: out[j] = in[src(j)]
__device__ __forceinline__ unsigned galois_src(unsigned j, int logN, u64 g) {
    // only the low logN + 1 bits of the product matter: 32-bit arithmetic
    const unsigned mask = (2u << logN) - 1;
    const unsigned ex = 2 * (__brev(j) >> (32 - logN)) + 1;
    const unsigned e2 = (ex * (unsigned)g) & mask;
    return __brev((e2 - 1) >> 1) >> (32 - logN);
}

// gather loader for the automorphism fused into a pass
struct LdGalois {
    const u64* __restrict__ p;
    int logN;
    u64 g;
    __device__ __forceinline__ u64 operator()(size_t i) const {
        const size_t mask = ((size_t)1 << logN) - 1;
        return p[(i & ~mask) + galois_src((unsigned)(i & mask), logN, g)];
    }
    __device__ __forceinline__ void load8(size_t i, u64* x) const {
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = (*this)(i + k);
    }
};

}  // namespace hc
