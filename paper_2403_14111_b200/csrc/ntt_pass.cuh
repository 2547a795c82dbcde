// One NTT pass as a device template with load / store hooks, so producers
// (base conversion, rescale broadcast, automorphism gather) run inside the
// first round's loads and consumers (key inner product, ModDown combine,
// rescale combine) inside the last round's stores.  See ntt.cu for the
// decomposition and conventions.
#pragma once
#include "hc_internal.h"

namespace hc {

enum { MODE_FULL = 0, MODE_COLS = 1, MODE_CHUNKS = 2 };

// Geometry of one pass: SUBS sub-transforms of 2^LOGSZ points per CTA.
//   MODE_COLS  : sub-transform = column c (element pos at c + pos * N2), root R = 1
//   MODE_CHUNKS: sub-transform = chunk h (element pos at (h << LOGSZ) + pos), root R = N1 + h
//   MODE_FULL  : the whole limb, root R = 1
template <int LOGSZ, int MODE, int SUBS>
struct PassGeo {
    static constexpr int SZ = 1 << LOGSZ;
    static constexpr int TPS = SZ / 8;
    static constexpr int NR = (LOGSZ + 2) / 3;
    static constexpr int PADSZ = SZ + SZ / 16;
    static constexpr int THREADS = SUBS * TPS;
    static constexpr size_t smem_words() { return (size_t)SUBS * (MODE == MODE_COLS ? SZ : PADSZ); }
    int sub, lt, first_sub, R;
    size_t N2;
    __device__ __forceinline__ void init(int logN, int N1) {
        const int tid = threadIdx.x;
        if (MODE == MODE_COLS) { sub = tid % SUBS; lt = tid / SUBS; }
        else { sub = tid / TPS; lt = tid % TPS; }
        first_sub = blockIdx.x * SUBS;
        N2 = ((size_t)1 << logN) >> (MODE == MODE_COLS ? LOGSZ : 0);
        R = (MODE == MODE_CHUNKS) ? (N1 + first_sub + sub) : 1;
    }
    __device__ __forceinline__ size_t gidx(int pos) const {
        if (MODE == MODE_COLS) return (size_t)(first_sub + sub) + (size_t)pos * N2;
        return ((size_t)(first_sub + sub) << LOGSZ) + pos;
    }
    __device__ __forceinline__ int sidx(int pos) const {
        if (MODE == MODE_COLS) return pos * SUBS + sub;
        return sub * PADSZ + pos + (pos >> 4);
    }
    // positions owned by this thread in the last round (forward) / first round (inverse)
    static constexpr bool EDGE_CONTIG = (MODE != MODE_COLS) && (LOGSZ % 3 == 0);
};

// Runs the pass.  LD: u64 operator()(size_t gidx) and void load8(size_t gidx, u64* x)
// (8 consecutive words, only used when EDGE_CONTIG).  ST: void operator()(size_t gidx, u64 v)
// and store8(size_t gidx, const u64* x).  Values handed to ST are lazy: [0, 4q) forward,
// [0, 2q) inverse.
template <int LOGSZ, int MODE, int SUBS, bool INV, class LD, class ST>
__device__ __forceinline__ void ntt_pass(const PassGeo<LOGSZ, MODE, SUBS>& G, u64* sm, const u64* __restrict__ W,
                                         const u64* __restrict__ Ws, u64 q, LD& ld, ST& st) {
    using PG = PassGeo<LOGSZ, MODE, SUBS>;
    const u64 twoq = 2 * q;
    u64 x[8];
#pragma unroll
    for (int rd = 0; rd < PG::NR; rd++) {
        const int fr = INV ? (PG::NR - 1 - rd) : rd;
        const int s0 = 3 * fr;
        const int r = (LOGSZ - s0) < 3 ? (LOGSZ - s0) : 3;
        const int logu = LOGSZ - s0 - r;
        const int NG = 8 >> r;
        const int GS = 1 << r;
        // ---- load ----
#pragma unroll
        for (int j = 0; j < NG; j++) {
            const int g = G.lt + j * PG::TPS;
            const int blk = g >> logu, o = g & ((1 << logu) - 1);
            const int base = (blk << (logu + r)) + o;
            if (rd == 0 && PG::EDGE_CONTIG && logu == 0 && r == 3) {
                ld.load8(G.gidx(base), x + 8 * j);
            } else {
#pragma unroll
                for (int m = 0; m < GS; m++) {
                    const int pos = base + (m << logu);
                    x[j * GS + m] = (rd == 0) ? ld(G.gidx(pos)) : sm[G.sidx(pos)];
                }
            }
        }
        // ---- twiddles for the round, loaded up front ----
        u64 tw_r[7], tws_r[7];
        {
            int n = 0;
#pragma unroll
            for (int j = 0; j < NG; j++) {
                const int blk = (G.lt + j * PG::TPS) >> logu;
#pragma unroll
                for (int qq = 0; qq < r; qq++) {
#pragma unroll
                    for (int sb = 0; sb < (1 << qq); sb++) {
                        const int widx = G.R * (1 << (s0 + qq)) + (blk << qq) + sb;
                        tw_r[n] = __ldg(W + widx);
                        tws_r[n] = __ldg(Ws + widx);
                        n++;
                    }
                }
            }
        }
        // ---- butterflies (Harvey lazy) ----
#pragma unroll
        for (int j = 0; j < NG; j++) {
            u64* y = x + j * GS;
            const int gbase = j * (GS - 1);
            if (!INV) {
#pragma unroll
                for (int qq = 0; qq < r; qq++) {
                    const int half = 1 << (r - 1 - qq);
#pragma unroll
                    for (int m1 = 0; m1 < GS; m1++) {
                        if (m1 & half) continue;
                        const int k = gbase + ((1 << qq) - 1) + (m1 >> (r - qq));
                        u64 X = y[m1];
                        X = X >= twoq ? X - twoq : X;
                        const u64 T = mul_shoup_lazy(y[m1 + half], tw_r[k], tws_r[k], q);
                        y[m1] = X + T;
                        y[m1 + half] = X + twoq - T;
                    }
                }
            } else {
#pragma unroll
                for (int qq = r - 1; qq >= 0; qq--) {
                    const int half = 1 << (r - 1 - qq);
#pragma unroll
                    for (int m1 = 0; m1 < GS; m1++) {
                        if (m1 & half) continue;
                        const int k = gbase + ((1 << qq) - 1) + (m1 >> (r - qq));
                        const u64 U = y[m1], V = y[m1 + half];
                        const u64 X = U + V;
                        y[m1] = X >= twoq ? X - twoq : X;
                        y[m1 + half] = mul_shoup_lazy(U + twoq - V, tw_r[k], tws_r[k], q);
                    }
                }
            }
        }
        // ---- store ----
        const bool last = (rd == PG::NR - 1);
#pragma unroll
        for (int j = 0; j < NG; j++) {
            const int g = G.lt + j * PG::TPS;
            const int blk = g >> logu, o = g & ((1 << logu) - 1);
            const int base = (blk << (logu + r)) + o;
            if (last && PG::EDGE_CONTIG && logu == 0 && r == 3) {
                st.store8(G.gidx(base), x + 8 * j);
            } else {
#pragma unroll
                for (int m = 0; m < GS; m++) {
                    const int pos = base + (m << logu);
                    if (last) st(G.gidx(pos), x[j * GS + m]);
                    else sm[G.sidx(pos)] = x[j * GS + m];
                }
            }
        }
        if (!last) __syncthreads();
    }
}

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
    __device__ __forceinline__ u64 fin(u64 v) const {
        if (!FINAL) return v;
        if (INV) return mul_shoup(v, c, cs, q);
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
    const u64 mask = (2ull << logN) - 1;
    const u64 ex = 2 * (u64)(__brev(j) >> (32 - logN)) + 1;
    const u64 e2 = (ex * g) & mask;
    return __brev((unsigned)((e2 - 1) >> 1)) >> (32 - logN);
}

// gather loader for the automorphism fused into a pass (g == 0: identity)
struct LdGalois {
    const u64* __restrict__ p;
    int logN;
    u64 g;
    __device__ __forceinline__ u64 operator()(size_t i) const {
        if (!g) return p[i];
        const size_t mask = ((size_t)1 << logN) - 1;
        return p[(i & ~mask) + galois_src((unsigned)(i & mask), logN, g)];
    }
    __device__ __forceinline__ void load8(size_t i, u64* x) const {
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = (*this)(i + k);
    }
};

}  // namespace hc
