// Batched negacyclic NTT / INTT over word-size RNS primes (sm_100a).
//
// Convention: forward is Cooley-Tukey, natural order in,
// bit-reversed order out; NTT index j holds the evaluation at
// psi^(2 brv(j) + 1).  Inverse is Gentleman-Sande with the N^-1 scaling
// (or a per-limb constant that folds N^-1 with the next base-conversion
// factor) applied in the final store.  Twiddles psi^brv(k) carry Shoup
// companions.  Lazy butterflies: inverse values live in [0, 2q) (Harvey);
// forward values grow by 2q per stage up to 16q and are reduced on the plan
// in ntt_pass.cuh (primes < 2^60); the final store reduces to [0, q), so
// results are canonical residues, bit-exact with the oracle's plain NTT.
//
// Decomposition.  N = N1 * N2.  Forward = pass "cols" (N2 independent
// N1-point sub-transforms on elements c + r*N2, root index R = 1) then pass
// "chunks" (N1 independent N2-point sub-transforms on contiguous chunk h,
// root index R = N1 + h); inverse runs them in the opposite order.  Stage
// s' of a sub-transform with root index R uses twiddle tw[R*2^s' + i'].
// For N <= 2^13 one "full" pass keeps the whole limb in shared memory.
//
// Inside a pass (ntt_pass.cuh) every thread owns 8 words in registers and
// runs up to 3 butterfly stages (radix 8) per round; rounds exchange through
// shared memory (one barrier per round).  The first round loads straight
// from HBM and the last round stores straight to HBM, so a pass reads and
// writes each word exactly once.  All index math is shifts and masks.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "ntt_pass.cuh"

namespace hc {

#ifndef NTT_PMB
#define NTT_PMB PASS_MIN_BLOCKS   // register budget of the generic NTT kernel (as PASS_MIN_BLOCKS)
#endif
#ifndef NTT_PMB_SMALL
#define NTT_PMB_SMALL 2           // register budget of the sub-wave chain launches of the split passes
#endif
template <int LOGSZ, int MODE, int SUBS, bool INV, int PMB = NTT_PMB>
__global__ void __launch_bounds__(PassGeo<LOGSZ, MODE, SUBS>::THREADS,
                                  (PassGeo<LOGSZ, MODE, SUBS>::MIN_BLOCKS * PMB / PASS_MIN_BLOCKS) > 0
                                      ? PassGeo<LOGSZ, MODE, SUBS>::MIN_BLOCKS * PMB / PASS_MIN_BLOCKS : 1)
    ntt_kernel(JobList jobs, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, int logN,
               int N1, int use_src, int last) {
    pdl_trigger();
    extern __shared__ u64 sm[];
    const int job = blockIdx.y, b = blockIdx.z;
    const int pidx = jobs.prime[job];
    u64* dst = jobs.ptr[job] + (b ? jobs.boff[b] : 0);
    const u64* src = (use_src && jobs.src[job]) ? jobs.src[job] + (b ? jobs.sboff[b] : 0) : dst;
    const PrimeDev P = primes[pidx];
    const ulonglong2* TW = tw + ((size_t)pidx << logN);
    using PG = PassGeo<LOGSZ, MODE, SUBS>;
    PG G;
    G.init(N1);
    ulonglong2* twsm = PG::twsm_of(sm);
    if (twsm) stage_twiddles<LOGSZ, MODE, SUBS>(G, twsm, TW, N1);
    const bool pend = twsm != nullptr;
    pdl_wait();   // above: context-lifetime tables (primes, twiddles) only
    const u64 gal = use_src ? jobs.galois : 0;
    u64 c = P.ninv, cs = P.ninv_s;
    if (INV && jobs.custom) { c = jobs.scale[job]; cs = jobs.scale_s[job]; }
    const u64 off = (INV && jobs.center) ? (P.q - 1) / 2 : 0;
    // forward input bounds: canonical (or < 2q) residues for the first pass,
    // the column pass's lazy output (< 16q) for the chunk pass; final stores
    // need < 4q, lazy stores < 16q
    constexpr int INB = (MODE == MODE_CHUNKS) ? BOUND_LIM : 2;
    if (gal) {
        LdGalois ld{src, logN, gal};
        if (last) { StPlain<INV, true> st{dst, P.q, c, cs, off}; ntt_pass<LOGSZ, MODE, SUBS, INV, INB, 4>(G, sm, TW, P, ld, st, twsm, pend); }
        else { StPlain<INV, false> st{dst, P.q, 0, 0}; ntt_pass<LOGSZ, MODE, SUBS, INV, INB, BOUND_LIM>(G, sm, TW, P, ld, st, twsm, pend); }
    } else {
        LdPlain ld{src};
        if (last) { StPlain<INV, true> st{dst, P.q, c, cs, off}; ntt_pass<LOGSZ, MODE, SUBS, INV, INB, 4>(G, sm, TW, P, ld, st, twsm, pend); }
        else { StPlain<INV, false> st{dst, P.q, 0, 0}; ntt_pass<LOGSZ, MODE, SUBS, INV, INB, BOUND_LIM>(G, sm, TW, P, ld, st, twsm, pend); }
    }
}

template <int LOGSZ, int MODE, int SUBS, int PMB = NTT_PMB>
static void launch_t(Ctx& c, const JobList& jobs, bool inv, int N1, int use_src, int last) {
    using PG = PassGeo<LOGSZ, MODE, SUBS>;
    const size_t smem = PG::smem_bytes();
    const int nsub = (MODE == MODE_COLS) ? (c.N >> LOGSZ) : (MODE == MODE_CHUNKS ? N1 : 1);
    dim3 grid(nsub / SUBS, jobs.n, jobs.nb);
    static const char* names[2][3] = {{"ntt_fwd_full", "ntt_fwd_cols", "ntt_fwd_chunks"},
                                      {"ntt_inv_full", "ntt_inv_cols", "ntt_inv_chunks"}};
    if (inv) set_smem(ntt_kernel<LOGSZ, MODE, SUBS, true, PMB>, smem);
    else set_smem(ntt_kernel<LOGSZ, MODE, SUBS, false, PMB>, smem);
    Launch scope(c, names[inv ? 1 : 0][MODE], 16.0 * c.N * jobs.n * jobs.nb);
    if (inv)
        launch_k(c, ntt_kernel<LOGSZ, MODE, SUBS, true, PMB>, grid, PG::THREADS, smem, jobs, c.d_primes, c.twp(0, true),
                                                                                  c.logN, N1, use_src, last);
    else
        launch_k(c, ntt_kernel<LOGSZ, MODE, SUBS, false, PMB>, grid, PG::THREADS, smem, jobs, c.d_primes,
                                                                                   c.twp(0, false), c.logN, N1,
                                                                                   use_src, last);
    HC_CUDA(cudaGetLastError());
}

// Compact (looped, one butterfly per thread) variant for sub-wave launches:
// see ntt_pass.cuh.  Same arguments and hooks as ntt_kernel.
template <int LOGSZ, int MODE, int SUBS, bool INV>
__global__ void __launch_bounds__(SmallGeo<LOGSZ, MODE, SUBS>::THREADS)
    ntt_small_kernel(JobList jobs, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, int logN,
                     int N1, int use_src, int last) {
    pdl_trigger();
    extern __shared__ u64 sm[];
    const int job = blockIdx.y, b = blockIdx.z;
    const int pidx = jobs.prime[job];
    u64* dst = jobs.ptr[job] + (b ? jobs.boff[b] : 0);
    const u64* src = (use_src && jobs.src[job]) ? jobs.src[job] + (b ? jobs.sboff[b] : 0) : dst;
    const PrimeDev P = primes[pidx];
    const ulonglong2* TW = tw + ((size_t)pidx << logN);
    using SG = SmallGeo<LOGSZ, MODE, SUBS>;
    SG G;
    G.init(N1);
    stage_twiddles_small<LOGSZ, MODE, SUBS>(G, SG::twsm_of(sm), TW, N1);
    pdl_wait();   // above: context-lifetime tables (primes, twiddles) only
    const u64 gal = use_src ? jobs.galois : 0;
    u64 c = P.ninv, cs = P.ninv_s;
    if (INV && jobs.custom) { c = jobs.scale[job]; cs = jobs.scale_s[job]; }
    const u64 off = (INV && jobs.center) ? (P.q - 1) / 2 : 0;
    constexpr int INB = (MODE == MODE_CHUNKS) ? BOUND_LIM : 2;
    if (gal) {
        LdGalois ld{src, logN, gal};
        if (last) { StPlain<INV, true> st{dst, P.q, c, cs, off}; ntt_pass_small<LOGSZ, MODE, SUBS, INV, INB>(G, sm, P, ld, st); }
        else { StPlain<INV, false> st{dst, P.q, 0, 0}; ntt_pass_small<LOGSZ, MODE, SUBS, INV, INB>(G, sm, P, ld, st); }
    } else {
        LdPlain ld{src};
        if (last) { StPlain<INV, true> st{dst, P.q, c, cs, off}; ntt_pass_small<LOGSZ, MODE, SUBS, INV, INB>(G, sm, P, ld, st); }
        else { StPlain<INV, false> st{dst, P.q, 0, 0}; ntt_pass_small<LOGSZ, MODE, SUBS, INV, INB>(G, sm, P, ld, st); }
    }
}

template <int LOGSZ, int MODE, int SUBS>
static void launch_small(Ctx& c, const JobList& jobs, bool inv, int N1, int use_src, int last) {
    using SG = SmallGeo<LOGSZ, MODE, SUBS>;
    const size_t smem = SG::smem_bytes();
    const int nsub = (MODE == MODE_COLS) ? (c.N >> LOGSZ) : N1;
    dim3 grid(nsub / SUBS, jobs.n, jobs.nb);
    static const char* names[2][3] = {{"ntt_fwd_full", "ntt_fwd_cols", "ntt_fwd_chunks"},
                                      {"ntt_inv_full", "ntt_inv_cols", "ntt_inv_chunks"}};
    Launch scope(c, names[inv ? 1 : 0][MODE], 16.0 * c.N * jobs.n * jobs.nb);
    if (inv)
        launch_k(c, ntt_small_kernel<LOGSZ, MODE, SUBS, true>, grid, SG::THREADS, smem, jobs, c.d_primes,
                 c.twp(0, true), c.logN, N1, use_src, last);
    else
        launch_k(c, ntt_small_kernel<LOGSZ, MODE, SUBS, false>, grid, SG::THREADS, smem, jobs, c.d_primes,
                 c.twp(0, false), c.logN, N1, use_src, last);
    HC_CUDA(cudaGetLastError());
}

// HC_NTT_SMALL: 0 = never, 1 = lone sub-wave launches (chains), 2 = every sub-wave launch, 3 = every launch
static int small_policy() {
    static const int v = [] {
        const char* e = std::getenv("HC_NTT_SMALL");
        return e ? std::atoi(e) : 1;
    }();
    return v;
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

// split passes for 2^14 .. 2^17: chunks of 2^9, columns of 2^(logN-9).
// A launch that would not fill one wave of 256-thread CTAs (148 SMs x 4, e.g.
// the 13 limbs of a key switch's first INTT or its 6 special-prime limbs)
// takes the 64-thread variant: 4x the CTAs for the same work, so latency and
// instruction fetch are spread over every SM.
static bool small_grid(const JobList& jobs, int ctas_per_job) { return ctas_per_job * jobs.n * jobs.nb < 148 * 4; }
// a sub-wave launch of a lone ciphertext (grid z = 1: the chains of softmax /
// inversion) is latency-bound, so it takes a larger register budget
// (NTT_PMB_SMALL=2: softmax 22.70 -> 22.16 ms); batched sub-wave launches keep
// NTT_PMB (the larger budget measured +0.3 % per pair there)
static bool chain_grid(const JobList& jobs, int ctas_per_job) { return jobs.nb == 1 && small_grid(jobs, ctas_per_job); }

static void cols_pass(Ctx& c, const JobList& jobs, bool inv, int N1, int use_src, int last) {
    const int big_subs = 1 << (20 - c.logN);   // 64, 32, 16, 8 columns per CTA for 2^14 .. 2^17
    const bool sm = small_grid(jobs, 512 / big_subs), ch = sm && jobs.nb == 1;
    if ((small_policy() == 1 && ch) || (small_policy() == 2 && sm) || small_policy() == 3) {
        switch (c.logN) {
            case 14: launch_small<5, MODE_COLS, 16>(c, jobs, inv, N1, use_src, last); return;
            case 15: launch_small<6, MODE_COLS, 8>(c, jobs, inv, N1, use_src, last); return;
            case 16: launch_small<7, MODE_COLS, 4>(c, jobs, inv, N1, use_src, last); return;
            case 17: launch_small<8, MODE_COLS, 2>(c, jobs, inv, N1, use_src, last); return;
            default: throw Error(-1, "unsupported ring degree");
        }
    }
    switch (c.logN) {
        case 14: if (ch) launch_t<5, MODE_COLS, 16, NTT_PMB_SMALL>(c, jobs, inv, N1, use_src, last);
                 else if (sm) launch_t<5, MODE_COLS, 16>(c, jobs, inv, N1, use_src, last);
                 else launch_t<5, MODE_COLS, 64>(c, jobs, inv, N1, use_src, last); break;
        case 15: if (ch) launch_t<6, MODE_COLS, 8, NTT_PMB_SMALL>(c, jobs, inv, N1, use_src, last);
                 else if (sm) launch_t<6, MODE_COLS, 8>(c, jobs, inv, N1, use_src, last);
                 else launch_t<6, MODE_COLS, 32>(c, jobs, inv, N1, use_src, last); break;
        case 16: if (ch) launch_t<7, MODE_COLS, 4, NTT_PMB_SMALL>(c, jobs, inv, N1, use_src, last);
                 else if (sm) launch_t<7, MODE_COLS, 4>(c, jobs, inv, N1, use_src, last);
                 else launch_t<7, MODE_COLS, 16>(c, jobs, inv, N1, use_src, last); break;
        case 17: if (ch) launch_t<8, MODE_COLS, 2, NTT_PMB_SMALL>(c, jobs, inv, N1, use_src, last);
                 else if (sm) launch_t<8, MODE_COLS, 2>(c, jobs, inv, N1, use_src, last);
                 else launch_t<8, MODE_COLS, 8>(c, jobs, inv, N1, use_src, last); break;
        default: throw Error(-1, "unsupported ring degree");
    }
}

#ifndef HC_NTT_CH_SUBS
#define HC_NTT_CH_SUBS 2   // 128-thread CTAs (measured 4 -> 2: -0.8 % per pair)
#endif
static void chunks_pass(Ctx& c, const JobList& jobs, bool inv, int N1, int use_src, int last) {
    const bool smg = small_grid(jobs, N1 / HC_NTT_CH_SUBS);
    if ((small_policy() == 1 && smg && jobs.nb == 1) || (small_policy() == 2 && smg) || small_policy() == 3) {
        launch_small<9, MODE_CHUNKS, 1>(c, jobs, inv, N1, use_src, last);
        return;
    }
    if (chain_grid(jobs, N1 / HC_NTT_CH_SUBS)) launch_t<9, MODE_CHUNKS, 1, NTT_PMB_SMALL>(c, jobs, inv, N1, use_src, last);
    else if (small_grid(jobs, N1 / HC_NTT_CH_SUBS)) launch_t<9, MODE_CHUNKS, 1>(c, jobs, inv, N1, use_src, last);
    else launch_t<9, MODE_CHUNKS, HC_NTT_CH_SUBS>(c, jobs, inv, N1, use_src, last);
}

// second half of a split forward NTT (in place), for callers that ran the
// column pass themselves with a fused producer
// Output stays lazy below 16q < 2^64: the only consumer (the key product)
// takes any 64-bit input into its 128-bit accumulation.
void ntt_forward_chunks(Ctx& c, const JobList& jobs) {
    if (jobs.n == 0) return;
    chunks_pass(c, jobs, false, 1 << (c.logN - 9), 0, 0);
}

void ntt_forward(Ctx& c, const JobList& jobs) {
    if (jobs.n == 0) return;
    if (c.logN <= 13) { full_pass(c, jobs, false); return; }
    const int N1 = 1 << (c.logN - 9);
    cols_pass(c, jobs, false, N1, 1, 0);
    chunks_pass(c, jobs, false, N1, 0, 1);
}

// ---- both inverse passes of a lone sub-wave INTT in one cooperative launch ----
//
// In the chains a launch costs more than its work (ncu: 9-10 us per compact
// pass of 6-13 limbs, ~5 us of it fixed), so the two passes of an INTT run as
// one kernel: every CTA runs the compact chunk pass of chunk x of its limb,
// the grid synchronises (cooperative launch: all CTAs are co-resident, so the
// barrier cannot deadlock whatever runs on the other streams), then the same
// CTA runs the compact column pass of column block x.  Chunk CTAs and column
// blocks are both N1 per limb, both passes use 128 threads.  The column pass
// reads words other CTAs wrote in this kernel: L2 loads (ld.global.cg).
template <int CL, int CS>
__global__ void __launch_bounds__(128)
    intt_fused_kernel(JobList jobs, const PrimeDev* __restrict__ primes, const ulonglong2* __restrict__ tw, int logN,
                      int N1) {
    pdl_trigger();
    extern __shared__ u64 sm[];
    static_assert(SmallGeo<9, MODE_CHUNKS, 1>::THREADS == 128 && SmallGeo<CL, MODE_COLS, CS>::THREADS == 128,
                  "fused INTT: 128-thread passes");
    pdl_wait();
    // grid y strides over the limb jobs (the grid is capped at the co-residency bound)
    for (int job = blockIdx.y; job < jobs.n; job += gridDim.y) {
        const int pidx = jobs.prime[job];
        u64* dst = jobs.ptr[job];
        const u64* src = jobs.src[job] ? jobs.src[job] : dst;
        const PrimeDev P = primes[pidx];
        const ulonglong2* TW = tw + ((size_t)pidx << logN);
        StPlain<true, false> st{dst, P.q, 0, 0};
        if (jobs.galois) {
            LdGalois ld{src, logN, jobs.galois};
            small_pass_run<9, MODE_CHUNKS, 1, true, 2>(N1, blockIdx.x, sm, TW, P, ld, st);
        } else {
            LdPlain ld{src};
            small_pass_run<9, MODE_CHUNKS, 1, true, 2>(N1, blockIdx.x, sm, TW, P, ld, st);
        }
    }
    cooperative_groups::this_grid().sync();
    for (int job = blockIdx.y; job < jobs.n; job += gridDim.y) {
        const int pidx = jobs.prime[job];
        u64* dst = jobs.ptr[job];
        const PrimeDev P = primes[pidx];
        const ulonglong2* TW = tw + ((size_t)pidx << logN);
        u64 c = P.ninv, cs = P.ninv_s;
        if (jobs.custom) { c = jobs.scale[job]; cs = jobs.scale_s[job]; }
        const u64 off = jobs.center ? (P.q - 1) / 2 : 0;
        LdCg ld{dst};
        StPlain<true, true> st{dst, P.q, c, cs, off};
        small_pass_run<CL, MODE_COLS, CS, true, 2>(N1, blockIdx.x, sm, TW, P, ld, st);
    }
}

// HC_INTT_FUSE: the most limbs a lone INTT may have to take the one-launch form (0 = never)
static int intt_fuse_max() {
    static const int v = [] { const char* e = std::getenv("HC_INTT_FUSE"); return e ? std::atoi(e) : 9; }();
    return v;
}
template <int CL, int CS>
static bool launch_intt_fused(Ctx& c, const JobList& jobs, int N1) {
    using S1 = SmallGeo<9, MODE_CHUNKS, 1>;
    using S2 = SmallGeo<CL, MODE_COLS, CS>;
    const size_t smem = S1::smem_bytes() > S2::smem_bytes() ? S1::smem_bytes() : S2::smem_bytes();
    auto kern = intt_fused_kernel<CL, CS>;
    // co-residency bound of the cooperative launch, once per device
    static int cap[64] = {0};
    int dev = 0;
    HC_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return false;
    if (!cap[dev]) {
        int per_sm = 0, sms = 0;
        HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
        HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        cap[dev] = per_sm * sms > 0 ? per_sm * sms : -1;
    }
    const int gy = std::min(jobs.n, cap[dev] / N1);
    if (gy < 1) return false;
    Launch scope(c, "ntt_inv_fused", 32.0 * c.N * jobs.n);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(N1, gy, 1);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, jobs, (const PrimeDev*)c.d_primes,
                                             (const ulonglong2*)c.twp(0, true), c.logN, N1);
    if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported) {
        // fewer SMs than the occupancy query promised (MPS partition, green context):
        // nothing was launched; this device keeps the two-launch form from now on
        (void)cudaGetLastError();
        cap[dev] = -1;
        return false;
    }
    HC_CUDA(e);
    return true;
}

void ntt_inverse(Ctx& c, const JobList& jobs) {
    if (jobs.n == 0) return;
    if (c.logN <= 13) { full_pass(c, jobs, true); return; }
    const int N1 = 1 << (c.logN - 9);
    if (small_policy() >= 1 && jobs.nb == 1 && jobs.n <= intt_fuse_max()) {
        bool done = false;
        switch (c.logN) {
            case 14: done = launch_intt_fused<5, 16>(c, jobs, N1); break;
            case 15: done = launch_intt_fused<6, 8>(c, jobs, N1); break;
            case 16: done = launch_intt_fused<7, 4>(c, jobs, N1); break;
            case 17: done = launch_intt_fused<8, 2>(c, jobs, N1); break;
            default: break;
        }
        if (done) return;
    }
    chunks_pass(c, jobs, true, N1, 1, 0);
    cols_pass(c, jobs, true, N1, 0, 1);
}

}  // namespace hc
