// Batched negacyclic NTT / INTT over word-size RNS primes (sm_100a).
//
// Convention: forward is Cooley-Tukey, natural order in,
// bit-reversed order out; NTT index j holds the evaluation at
// psi^(2 brv(j) + 1).  Inverse is Gentleman-Sande with the N^-1 scaling
// fused into the final store.  Twiddles psi^brv(k) carry Shoup companions;
// butterflies keep values lazily in [0, 2q) and the final pass reduces to
// [0, q), so results are canonical residues (bit-exact with the oracle).
//
// Decomposition.  N = N1 * N2.  A transform of size N splits into
//   pass "columns": N2 independent N1-point sub-transforms on elements
//                   c + r*N2 (stride N2), all with root index R = 1;
//   pass "chunks" : N1 independent N2-point sub-transforms on contiguous
//                   chunks h, root index R = N1 + h.
// Stage s' of a sub-transform with root index R uses twiddle tw[R*2^s' + i'].
// For N <= 2^13 a single "full" pass keeps the whole limb in shared memory.
// Each CTA stages a tile of TE words in shared memory; one launch covers a
// JobList of limbs (blockIdx.y), each with its own prime and optional
// out-of-place source.
#include "hc_internal.h"

namespace hc {

enum { MODE_FULL = 0, MODE_COLS = 1, MODE_CHUNKS = 2 };

template <bool INV>
__global__ void __launch_bounds__(1024) ntt_tile_kernel(JobList jobs, const PrimeDev* __restrict__ primes,
                                                        const u64* __restrict__ tw, const u64* __restrict__ tws,
                                                        int N, int logSZ, int mode, int log_te, int N1,
                                                        int use_src, int last) {
    extern __shared__ u64 sm[];
    const int job = blockIdx.y;
    const int pidx = jobs.prime[job];
    const u64* src = (use_src && jobs.src[job]) ? jobs.src[job] : jobs.ptr[job];
    u64* dst = jobs.ptr[job];
    const PrimeDev P = primes[pidx];
    const u64 q = P.q, twoq = P.twoq;
    const u64* W = tw + (size_t)pidx * N;
    const u64* Ws = tws + (size_t)pidx * N;
    const int TE = 1 << log_te;
    const int SZ = 1 << logSZ;
    const int tile = blockIdx.x;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int N2 = N / N1;

    // ---- load ----
    if (mode == MODE_COLS) {
        const int cols = TE >> logSZ;          // sub-transforms per tile
        const int c0 = tile * cols;
        for (int e = tid; e < TE; e += nth) {
            int r = e / cols, c = e - r * cols;
            sm[e] = src[(size_t)(c0 + c) + (size_t)r * N2];
        }
    } else {
        const size_t base = (size_t)tile * TE;
        for (int e = tid; e < TE; e += nth) sm[e] = src[base + e];
    }
    __syncthreads();

    const int half = SZ >> 1;
    const int nb = TE >> 1;                    // butterflies per stage in the tile
    const int cols = TE >> logSZ;
    for (int st = 0; st < logSZ; st++) {
        const int s = INV ? (logSZ - 1 - st) : st;     // local stage index
        const int t = SZ >> (s + 1);
        const int m = 1 << s;
        for (int b = tid; b < nb; b += nth) {
            int sub, k;
            if (mode == MODE_COLS) { sub = b % cols; k = b / cols; }
            else { sub = b / half; k = b - sub * half; }
            const int i = k / t, j = k - i * t;
            const int p1 = i * 2 * t + j, p2 = p1 + t;
            int a1, a2, R;
            if (mode == MODE_COLS) { a1 = p1 * cols + sub; a2 = p2 * cols + sub; R = 1; }
            else { a1 = sub * SZ + p1; a2 = sub * SZ + p2; R = (mode == MODE_CHUNKS) ? (N1 + tile * cols + sub) : 1; }
            const int widx = R * m + i;
            const u64 w = W[widx], ws = Ws[widx];
            u64 U = sm[a1], V = sm[a2];
            if (!INV) {
                V = mul_shoup_lazy(V, w, ws, q);
                u64 X = U + V, Y = U + twoq - V;
                sm[a1] = X >= twoq ? X - twoq : X;
                sm[a2] = Y >= twoq ? Y - twoq : Y;
            } else {
                u64 X = U + V;
                sm[a1] = X >= twoq ? X - twoq : X;
                sm[a2] = mul_shoup_lazy(U + twoq - V, w, ws, q);
            }
        }
        __syncthreads();
    }

    // ---- store ----
    auto fin = [&](u64 v) -> u64 {
        if (!last) return v;
        if (INV) return mul_shoup(v, P.ninv, P.ninv_s, q);
        return v >= q ? v - q : v;
    };
    if (mode == MODE_COLS) {
        const int c0 = tile * cols;
        for (int e = tid; e < TE; e += nth) {
            int r = e / cols, c = e - r * cols;
            dst[(size_t)(c0 + c) + (size_t)r * N2] = fin(sm[e]);
        }
    } else {
        const size_t base = (size_t)tile * TE;
        for (int e = tid; e < TE; e += nth) dst[base + e] = fin(sm[e]);
    }
}

static void launch_pass(Ctx& c, const JobList& jobs, bool inv, int logSZ, int mode, int log_te, int N1,
                        int use_src, int last) {
    if (jobs.n == 0) return;
    const int TE = 1 << log_te;
    int threads = TE / 4;
    if (threads > 1024) threads = 1024;
    if (threads < 32) threads = 32;
    dim3 grid(c.N / TE, jobs.n);
    size_t smem = sizeof(u64) * TE;
    static const char* names[2][3] = {{"ntt_fwd_full", "ntt_fwd_cols", "ntt_fwd_chunks"},
                                      {"ntt_inv_full", "ntt_inv_cols", "ntt_inv_chunks"}};
    Launch scope(c, names[inv ? 1 : 0][mode], 16.0 * c.N * jobs.n);
    if (inv) {
        ntt_tile_kernel<true><<<grid, threads, smem, c.stream>>>(jobs, c.d_primes, c.d_itw, c.d_itws, c.N, logSZ,
                                                                 mode, log_te, N1, use_src, last);
    } else {
        ntt_tile_kernel<false><<<grid, threads, smem, c.stream>>>(jobs, c.d_primes, c.d_tw, c.d_tws, c.N, logSZ,
                                                                  mode, log_te, N1, use_src, last);
    }
    HC_CUDA(cudaGetLastError());
}

static void ensure_attrs() {
    static bool done = false;
    if (done) return;
    HC_CUDA(cudaFuncSetAttribute(ntt_tile_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    HC_CUDA(cudaFuncSetAttribute(ntt_tile_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    done = true;
}

constexpr int FULL_MAX_LOG = 13;   // whole limb in shared memory up to 64 KiB
constexpr int CHUNK_LOG = 9;       // N2 = 512 for the chunk pass when split
constexpr int TILE_LOG = 11;       // 2048 words (16 KiB) per CTA when split

void ntt_forward(Ctx& c, const JobList& jobs) {
    ensure_attrs();
    if (c.logN <= FULL_MAX_LOG) {
        launch_pass(c, jobs, false, c.logN, MODE_FULL, c.logN, 1, 1, 1);
        return;
    }
    const int k1 = c.logN - CHUNK_LOG, N1 = 1 << k1;
    launch_pass(c, jobs, false, k1, MODE_COLS, TILE_LOG, N1, 1, 0);
    launch_pass(c, jobs, false, CHUNK_LOG, MODE_CHUNKS, TILE_LOG, N1, 0, 1);
}

void ntt_inverse(Ctx& c, const JobList& jobs) {
    ensure_attrs();
    if (c.logN <= FULL_MAX_LOG) {
        launch_pass(c, jobs, true, c.logN, MODE_FULL, c.logN, 1, 1, 1);
        return;
    }
    const int k1 = c.logN - CHUNK_LOG, N1 = 1 << k1;
    launch_pass(c, jobs, true, CHUNK_LOG, MODE_CHUNKS, TILE_LOG, N1, 1, 0);
    launch_pass(c, jobs, true, k1, MODE_COLS, TILE_LOG, N1, 0, 1);
}

}  // namespace hc
