// Batched negacyclic NTT / INTT over word-size RNS primes (sm_100a).
//
// Convention: forward is Cooley-Tukey, natural order in,
// bit-reversed order out; NTT index j holds the evaluation at
// psi^(2 brv(j) + 1).  Inverse is Gentleman-Sande with the N^-1 scaling
// fused into the final store.  Twiddles psi^brv(k) carry Shoup companions.
// Harvey lazy butterflies: forward values live in [0, 4q), inverse in
// [0, 2q); the final store reduces to [0, q), so results are canonical
// residues, bit-exact with the oracle's plain NTT.
//
// Decomposition.  N = N1 * N2.  Forward = pass "cols" (N2 independent
// N1-point sub-transforms on elements c + r*N2, root index R = 1) then pass
// "chunks" (N1 independent N2-point sub-transforms on contiguous chunk h,
// root index R = N1 + h); inverse runs them in the opposite order.  Stage
// s' of a sub-transform with root index R uses twiddle tw[R*2^s' + i'].
// For N <= 2^13 one "full" pass keeps the whole limb in shared memory.
//
// Inside a pass every thread owns 8 words in registers and runs up to 3
// butterfly stages (radix 8) per round; rounds exchange through shared
// memory (one barrier per round).  The first round loads straight from HBM
// and the last round stores straight to HBM, so a pass reads and writes
// each word exactly once.  Chunk-mode shared memory is padded by one word
// every 16 to keep the stride-8 rounds bank-conflict free; column mode
// keeps consecutive threads on consecutive columns (coalesced HBM access,
// conflict-free shared memory).  All index math is shifts and masks.
#include "hc_internal.h"

namespace hc {

enum { MODE_FULL = 0, MODE_COLS = 1, MODE_CHUNKS = 2 };

template <int LOGSZ, int MODE, int SUBS, bool INV>
__global__ void __launch_bounds__(SUBS*(1 << LOGSZ) / 8) ntt_kernel(JobList jobs, const PrimeDev* __restrict__ primes,
                                                                    const u64* __restrict__ tw,
                                                                    const u64* __restrict__ tws, int logN, int N1,
                                                                    int use_src, int last) {
    constexpr int SZ = 1 << LOGSZ;
    constexpr int TPS = SZ / 8;                 // threads per sub-transform
    constexpr int NR = (LOGSZ + 2) / 3;         // rounds of <= 3 stages
    constexpr int PADSZ = SZ + SZ / 16;
    extern __shared__ u64 sm[];

    const int job = blockIdx.y;
    const int pidx = jobs.prime[job];
    const u64* __restrict__ src = (use_src && jobs.src[job]) ? jobs.src[job] : jobs.ptr[job];
    u64* __restrict__ dst = jobs.ptr[job];
    const u64 q = primes[pidx].q, twoq = 2 * q;
    const size_t N = (size_t)1 << logN;
    const u64* __restrict__ W = tw + (size_t)pidx * N;
    const u64* __restrict__ Ws = tws + (size_t)pidx * N;
    const int tid = threadIdx.x;
    int sub, lt;
    if (MODE == MODE_COLS) { sub = tid % SUBS; lt = tid / SUBS; }
    else { sub = tid / TPS; lt = tid % TPS; }
    const int first_sub = blockIdx.x * SUBS;
    const size_t N2 = N >> (MODE == MODE_COLS ? LOGSZ : 0);
    const int R = (MODE == MODE_CHUNKS) ? (N1 + first_sub + sub) : 1;

    auto gidx = [&](int pos) -> size_t {
        if (MODE == MODE_COLS) return (size_t)(first_sub + sub) + (size_t)pos * N2;
        return ((size_t)(first_sub + sub) << LOGSZ) + pos;
    };
    auto sidx = [&](int pos) -> int {
        if (MODE == MODE_COLS) return pos * SUBS + sub;
        return sub * PADSZ + pos + (pos >> 4);
    };

    u64 x[8];
#pragma unroll
    for (int rd = 0; rd < NR; rd++) {
        const int fr = INV ? (NR - 1 - rd) : rd;           // forward round index of this round
        const int s0 = 3 * fr;
        const int r = (LOGSZ - s0) < 3 ? (LOGSZ - s0) : 3;  // stages in this round
        const int logu = LOGSZ - s0 - r;
        const int G = 8 >> r;                               // groups per thread
        const int GS = 1 << r;                              // elements per group
        // ---- load ----
#pragma unroll
        for (int j = 0; j < G; j++) {
            const int g = lt + j * TPS;
            const int blk = g >> logu, o = g & ((1 << logu) - 1);
            const int base = (blk << (logu + r)) + o;
            if (rd == 0 && MODE != MODE_COLS && logu == 0 && r == 3) {
                const ulonglong2* p = reinterpret_cast<const ulonglong2*>(src + gidx(base));
#pragma unroll
                for (int v = 0; v < 4; v++) { ulonglong2 t = p[v]; x[8 * j + 2 * v] = t.x; x[8 * j + 2 * v + 1] = t.y; }
            } else {
#pragma unroll
                for (int m = 0; m < GS; m++) {
                    const int pos = base + (m << logu);
                    x[j * GS + m] = (rd == 0) ? src[gidx(pos)] : sm[sidx(pos)];
                }
            }
        }
        // ---- twiddles: issue every load of the round up front (latency overlap) ----
        u64 tw_r[7], tws_r[7];
        {
            int n = 0;
#pragma unroll
            for (int j = 0; j < G; j++) {
                const int blk = (lt + j * TPS) >> logu;
#pragma unroll
                for (int qq = 0; qq < r; qq++) {
                    const int half = 1 << (r - 1 - qq);
#pragma unroll
                    for (int m1 = 0; m1 < GS; m1++) {
                        if (m1 & half) continue;
                        if ((m1 & ((half << 1) - 1)) != 0) continue;      // one twiddle per sub-block
                        const int widx = R * (1 << (s0 + qq)) + (blk << qq) + (m1 >> (r - qq));
                        tw_r[n] = __ldg(W + widx);
                        tws_r[n] = __ldg(Ws + widx);
                        n++;
                    }
                }
            }
        }
        // ---- butterflies ----
        int tn = 0;
#pragma unroll
        for (int j = 0; j < G; j++) {
            u64* y = x + j * GS;
            if (!INV) {
#pragma unroll
                for (int qq = 0; qq < r; qq++) {
                    const int half = 1 << (r - 1 - qq);
                    const int tbase = tn;
#pragma unroll
                    for (int m1 = 0; m1 < GS; m1++) {
                        if (m1 & half) continue;
                        const int k = tbase + (m1 >> (r - qq));
                        if ((m1 & ((half << 1) - 1)) == 0) tn++;
                        const u64 w = tw_r[k], ws = tws_r[k];
                        u64 X = y[m1];
                        X = X >= twoq ? X - twoq : X;
                        const u64 T = mul_shoup_lazy(y[m1 + half], w, ws, q);
                        y[m1] = X + T;
                        y[m1 + half] = X + twoq - T;
                    }
                }
            } else {
                // twiddles were loaded in forward stage order: stage qq's block
                // starts at offset (2^qq - 1) within this group's 2^r - 1 entries
                const int gbase = tn;
                tn += GS - 1;
#pragma unroll
                for (int qq = r - 1; qq >= 0; qq--) {
                    const int half = 1 << (r - 1 - qq);
#pragma unroll
                    for (int m1 = 0; m1 < GS; m1++) {
                        if (m1 & half) continue;
                        const int k = gbase + ((1 << qq) - 1) + (m1 >> (r - qq));
                        const u64 w = tw_r[k], ws = tws_r[k];
                        const u64 U = y[m1], V = y[m1 + half];
                        u64 X = U + V;
                        y[m1] = X >= twoq ? X - twoq : X;
                        y[m1 + half] = mul_shoup_lazy(U + twoq - V, w, ws, q);
                    }
                }
            }
        }
        // ---- store ----
        const bool to_global = (rd == NR - 1);
        if (to_global && last) {
            const PrimeDev P = primes[pidx];
#pragma unroll
            for (int e = 0; e < 8; e++) {
                u64 v = x[e];
                if (INV) v = mul_shoup(v, P.ninv, P.ninv_s, q);
                else { v = v >= twoq ? v - twoq : v; v = v >= q ? v - q : v; }
                x[e] = v;
            }
        }
#pragma unroll
        for (int j = 0; j < G; j++) {
            const int g = lt + j * TPS;
            const int blk = g >> logu, o = g & ((1 << logu) - 1);
            const int base = (blk << (logu + r)) + o;
            if (to_global && MODE != MODE_COLS && logu == 0 && r == 3) {
                ulonglong2* p = reinterpret_cast<ulonglong2*>(dst + gidx(base));
#pragma unroll
                for (int v = 0; v < 4; v++) p[v] = make_ulonglong2(x[8 * j + 2 * v], x[8 * j + 2 * v + 1]);
            } else {
#pragma unroll
                for (int m = 0; m < GS; m++) {
                    const int pos = base + (m << logu);
                    if (to_global) dst[gidx(pos)] = x[j * GS + m];
                    else sm[sidx(pos)] = x[j * GS + m];
                }
            }
        }
        if (!to_global) __syncthreads();
    }
}

template <int LOGSZ, int MODE, int SUBS>
static void launch_t(Ctx& c, const JobList& jobs, bool inv, int N1, int use_src, int last) {
    constexpr int SZ = 1 << LOGSZ;
    constexpr int threads = SUBS * SZ / 8;
    const size_t smem = sizeof(u64) * (size_t)SUBS * (MODE == MODE_COLS ? SZ : SZ + SZ / 16);
    const int nsub = (MODE == MODE_COLS) ? (c.N >> LOGSZ) : (MODE == MODE_CHUNKS ? N1 : 1);
    dim3 grid(nsub / SUBS, jobs.n);
    static const char* names[2][3] = {{"ntt_fwd_full", "ntt_fwd_cols", "ntt_fwd_chunks"},
                                      {"ntt_inv_full", "ntt_inv_cols", "ntt_inv_chunks"}};
    static bool attr[2] = {false, false};
    if (!attr[inv ? 1 : 0]) {
        if (inv) HC_CUDA(cudaFuncSetAttribute(ntt_kernel<LOGSZ, MODE, SUBS, true>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        else HC_CUDA(cudaFuncSetAttribute(ntt_kernel<LOGSZ, MODE, SUBS, false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[inv ? 1 : 0] = true;
    }
    Launch scope(c, names[inv ? 1 : 0][MODE], 16.0 * c.N * jobs.n);
    if (inv)
        ntt_kernel<LOGSZ, MODE, SUBS, true><<<grid, threads, smem, c.stream>>>(jobs, c.d_primes, c.d_itw, c.d_itws,
                                                                              c.logN, N1, use_src, last);
    else
        ntt_kernel<LOGSZ, MODE, SUBS, false><<<grid, threads, smem, c.stream>>>(jobs, c.d_primes, c.d_tw, c.d_tws,
                                                                               c.logN, N1, use_src, last);
    HC_CUDA(cudaGetLastError());
}

static void full_pass(Ctx& c, const JobList& jobs, bool inv) {
    switch (c.logN) {
        case 9: launch_t<9, MODE_FULL, 1>(c, jobs, inv, 1, 1, 1); break;
        case 10: launch_t<10, MODE_FULL, 1>(c, jobs, inv, 1, 1, 1); break;
        case 11: launch_t<11, MODE_FULL, 1>(c, jobs, inv, 1, 1, 1); break;
        case 12: launch_t<12, MODE_FULL, 1>(c, jobs, inv, 1, 1, 1); break;
        case 13: launch_t<13, MODE_FULL, 1>(c, jobs, inv, 1, 1, 1); break;
        default: throw Error(-1, "unsupported ring degree");
    }
}

// split passes for 2^14 .. 2^17: chunks of 2^9, columns of 2^(logN-9)
static void cols_pass(Ctx& c, const JobList& jobs, bool inv, int N1, int use_src, int last) {
    switch (c.logN) {
        case 14: launch_t<5, MODE_COLS, 64>(c, jobs, inv, N1, use_src, last); break;
        case 15: launch_t<6, MODE_COLS, 32>(c, jobs, inv, N1, use_src, last); break;
        case 16: launch_t<7, MODE_COLS, 16>(c, jobs, inv, N1, use_src, last); break;
        case 17: launch_t<8, MODE_COLS, 8>(c, jobs, inv, N1, use_src, last); break;
        default: throw Error(-1, "unsupported ring degree");
    }
}

static void chunks_pass(Ctx& c, const JobList& jobs, bool inv, int N1, int use_src, int last) {
    launch_t<9, MODE_CHUNKS, 4>(c, jobs, inv, N1, use_src, last);
}

constexpr int FULL_MAX_LOG = 13;
constexpr int CHUNK_LOG = 9;

void ntt_forward(Ctx& c, const JobList& jobs) {
    if (jobs.n == 0) return;
    if (c.logN <= FULL_MAX_LOG) { full_pass(c, jobs, false); return; }
    const int N1 = 1 << (c.logN - CHUNK_LOG);
    cols_pass(c, jobs, false, N1, 1, 0);
    chunks_pass(c, jobs, false, N1, 0, 1);
}

void ntt_inverse(Ctx& c, const JobList& jobs) {
    if (jobs.n == 0) return;
    if (c.logN <= FULL_MAX_LOG) { full_pass(c, jobs, true); return; }
    const int N1 = 1 << (c.logN - CHUNK_LOG);
    chunks_pass(c, jobs, true, N1, 1, 0);
    cols_pass(c, jobs, true, N1, 0, 1);
}

}  // namespace hc
