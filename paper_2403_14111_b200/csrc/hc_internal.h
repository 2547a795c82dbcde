// Internal declarations of the B200 RNS-CKKS library (not part of the C-ABI).
#pragma once
#include <utility>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "modarith.cuh"

namespace hc {

constexpr int MAXP = 48;       // max primes in Q u P
constexpr int MAXJ = 96;       // max limb jobs in one batched launch
constexpr int KS_MAXB = 24;    // max key switches in one batched pipeline (keyswitch.cu)

#define HC_CUDA(x)                                                                     \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            throw hc::Error(-2, std::string("CUDA: ") + cudaGetErrorString(e_) + " at " \
                                    + __FILE__ + ":" + std::to_string(__LINE__));      \
    } while (0)

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// one limb job for a batched launch: a pointer to N words and its prime
struct JobList {
    int n = 0;
    int custom = 0;          // inverse only: final multiplier scale[] instead of N^-1
    int center = 0;          // inverse only: outputs shifted by (q-1)/2 mod q (centred base conversion input)
    u64 galois = 0;          // first pass gathers the source through this automorphism
    int prime[MAXJ];
    u64* ptr[MAXJ];
    const u64* src[MAXJ];   // optional out-of-place source (nullptr = in place)
    u64 scale[MAXJ], scale_s[MAXJ];
    // batch dimension (grid z): copy b of job i works on ptr[i] + boff[b] and
    // reads src[i] + sboff[b] (element offsets; copy 0 has offset 0)
    int nb = 1;
    long long boff[KS_MAXB], sboff[KS_MAXB];
};

// host-side view of one prime with its precomputation
struct PrimeHost {
    u64 q, mu_hi, mu_lo, psi, ipsi, ninv, I;
};

struct Ctx;

// device ciphertext: residues [npoly][level+1][N] in NTT form
struct Ct {
    Ctx* ctx = nullptr;
    u64* d = nullptr;
    int level = 0;
    int npoly = 2;
    size_t words() const;
    u64* poly(int s) const;
};
using CtP = std::shared_ptr<Ct>;

// device plaintext: residues [level+1][N] in NTT form, encoded at scale[level]
struct Pt {
    Ctx* ctx = nullptr;
    u64* d = nullptr;
    int level = 0;
};
using PtP = std::shared_ptr<Pt>;

struct Key {
    int id;                       // galois element, 0 = relinearisation
    u64* d;                       // [dnum][2][nall][N]
};

enum OpKind { OP_ADD = 0, OP_CMULT, OP_MULT, OP_ROT, OP_CONJ, OP_BOOT, OP_ADJUST, OP_KS, OP_NKIND };

struct Ctx {
    int logN, N, L, K, alpha, dnum, nall, hw;
    // the application's top level (EmulatorContext.max_level): fresh
    // encryptions default to it and the refresh / bootstrap land on it; below
    // L when the chain carries bootstrapping levels above
    int app_L = 0;
    int boot_mode = 0;            // 0: refresh surrogate, 1: CKKS bootstrapping (hc_set_bootstrap)
    std::shared_ptr<struct BootState> boot;   // bootstrapping plan and plaintexts (bootstrap.cu)
    double sigma;
    u64 seed;
    int device;
    int grid_rows = 0;            // s0 of the slot grid (EmulatorContext.grid_rows)
    // block-row sharding (hc_set_shard): this context holds block rows
    // [shard_first, shard_first + m) of a batch of shard_total; refresh nonces
    // follow the whole batch's sequential order (evaluator.h NoncePlan)
    int shard_total = 0, shard_first = 0;
    // diagonal-pass sharding (hc_set_pass_shard): this context runs passes
    // k = pass_rank (mod pass_world) of DiagABT / DiagATB and pass_reducer
    // replaces the partial accumulators by their modular sum over ranks
    int pass_world = 1, pass_rank = 0;
    std::function<void(std::vector<std::shared_ptr<struct Ct>>&)> pass_reducer;
    // `stream` is the stream every launch / allocation goes to.  It is the
    // context's main stream except inside a schedule's fork region, where it
    // temporarily names one of the side streams (see schedules.cu Fork).
    cudaStream_t stream = nullptr;
    cudaStream_t main_stream = nullptr;
    std::vector<cudaStream_t> side;
    std::vector<cudaEvent_t> side_ev;
    cudaEvent_t fork_ev = nullptr;
    std::vector<cudaEvent_t> fork_evs;   // one fork event per nesting depth
    int fork_depth = 0;
    int fork_rot[4] = {0, 0, 0, 0};
    int fork_cap = 8;             // max side streams a schedule fans out to (hc_set_streams)
    bool ntt_fp = true;           // FP64 NTT passes for primes below 2^46 (HC_NTT_FP=0 disables)
    bool lockstep = true;         // batched (lockstep) diagonal passes when no refresh can fire (HC_LOCKSTEP)
    bool hoist = true;            // fused schedule forms: hoisted rotations, one relinearisation per product sum (HC_HOIST, hc_set_hoist)
    int batch = 6;                // key switches per batched pipeline in the lockstep schedules (HC_BATCH; 3 -> 6: training step -2 %)
    std::vector<cudaEvent_t> ra_ev;   // schedule run-ahead throttle (capi.cu): a schedule call
    int ra_idx = 0;                   // waits for the one ra_depth calls back to finish
    int ra_depth = 8;                 // HC_RUNAHEAD (2 measured host-jitter-bound steps)
    cudaMemPool_t pool = nullptr;
    // host <-> device transfers of the asynchronous C-ABI (hc_ct_upload_async /
    // hc_ct_download_async) run on their own stream, overlapping compute;
    // ciphertexts being downloaded stay alive until hc_sync / hc_timer_end
    cudaStream_t copy_stream = nullptr;   // uploads
    cudaStream_t d2h_stream = nullptr;    // downloads (a download waits for compute; uploads must not queue behind it)
    std::vector<std::shared_ptr<struct Ct>> io_pending;
    PrimeHost pr[MAXP];
    double scale[MAXP];
    // device tables
    PrimeDev* d_primes = nullptr;
    u64 *d_tw = nullptr, *d_itw = nullptr;   // [nall][N][2]: (psi^brv(k), shoup) and inverse
    const ulonglong2* twp(int prime, bool inv) const {
        return reinterpret_cast<const ulonglong2*>(inv ? d_itw : d_tw) + (size_t)prime * N;
    }
    u64* d_cdt = nullptr;
    int cdt_n = 0, cdt_b = 0;
    u64 cdt_host[128];
    u64* d_sk = nullptr;          // [nall][N] NTT form
    std::vector<int64_t> sk_coef;
    // host encoder tables
    std::vector<double> tw_re, tw_im, zt_re, zt_im;
    std::vector<int> slot_t;
    // keys (lazy, by galois element)
    std::map<int, Key> keys;
    // base-conversion tables (device), see context.cu
    u64* d_modup = nullptr;       // [L+1 levels][dnum][alpha][nall] (value, shoup) pairs
    u64* d_modup_inv = nullptr;   // [L+1][dnum][alpha] (value, shoup)
    u64* d_moddown = nullptr;     // [K][nall] (value, shoup) phat_{p->i}
    u64* d_moddown_inv = nullptr; // [K] (value, shoup)
    // centred base conversion: [-Q'_j]_{p} per (level, digit,
    // target prime) and [-P]_{q_i} per prime -- added once per term taken
    // from the upper half of its prime
    u64* d_modup_negq = nullptr;  // [L+1][dnum][nall]
    u64* d_moddown_negp = nullptr;   // [nall]
    // the fused passes read inputs shifted by h_a = (q_a-1)/2 (y'' = y + h_a
    // mod q_a, so the centred value is y'' - h_a) and start from the constant
    // [-sum_a h_a [Q'/q_a]_p]_p (ModUp) / [-sum_t h_t [P/p_t]_{q_i}]_{q_i} (ModDown)
    u64* d_modup_cc = nullptr;    // [L+1][dnum][nall]
    u64* d_moddown_cc = nullptr;  // [nall]
    u64* d_pinv = nullptr;        // [nall] (value, shoup) P^-1 mod q_i
    u64* d_rescale = nullptr;     // [L+1 (dropped prime l)][nall] (q_l^-1 mod q_i, shoup, q_l mod q_i)
    // merged ModDown + rescale of a ct x ct product at level l:
    // the dropped basis B_l = (q_l, p_1..p_K), D_l = q_l P
    u64* d_md2_inv = nullptr;     // [L+1][K+1] (value, shoup) (D/b_t)^-1 mod b_t
    u64* d_md2_tab = nullptr;     // [L+1][K+1][nall] (value, shoup) D/b_t mod q_i
    u64* d_md2_negd = nullptr;    // [L+1][nall] [-D]_{q_i}
    u64* d_md2_cc = nullptr;      // [L+1][nall] [-sum_t h_t D/b_t]_{q_i}, h_t = (b_t - 1) / 2
    u64* d_md2_dinv = nullptr;    // [L+1][nall] (value, shoup) D^-1 mod q_i
    const u64* pmodq() const { return d_rescale + (size_t)(L + 1) * nall * 3; }   // [nall] P mod q_i
    // counters
    uint64_t nonce = 0;
    int64_t counts[OP_NKIND] = {0};
    double model_bytes = 0;       // SURVEY §8(d) per-op HBM model of the ledgered ops (Eval::model)
    std::mutex mu;
    // encoded-mask cache used by the native schedules and content-addressed
    // Python operands: least-recently-used eviction above pt_cache_cap bytes
    // (HC_PT_CACHE_MB, default 4096)
    struct PtEntry {
        PtP pt;
        uint64_t used;
    };
    std::map<std::string, PtEntry> pt_cache;
    size_t pt_cache_bytes = 0, pt_cache_cap = 0;
    uint64_t pt_clock = 0;

    // the C-ABI's owning handle; every ciphertext/plaintext handle holds a
    // strong reference, so the context outlives all of them in any
    // destruction order (e.g. Python's cyclic garbage collection)
    std::weak_ptr<Ctx> self;

    // launch accounting and the optional per-kernel event profiler
    int64_t launches = 0;
    bool prof = false;
    struct ProfRec {
        const char* name;
        cudaEvent_t a, b;
        double bytes;
    };
    std::vector<ProfRec> prof_recs;
    std::vector<cudaEvent_t> ev_free;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    cudaEvent_t get_event();

    // workspace stream-ordered allocation
    u64* alloc(size_t words);
    void free(u64* p);

    // Per-stream scratch arenas for the temporaries of one pipeline (key
    // switch, rescale, tensor).  Work on one stream is ordered, so a scope can
    // reuse the bytes the previous scope on that stream released; no pool
    // bookkeeping on the hot path (the pool occasionally blocked the issuing
    // thread for 100+ ms while it remapped memory).  Scopes nest (stack).
    struct Arena {
        u64* base = nullptr;
        size_t cap = 0, top = 0;
    };
    std::map<cudaStream_t, Arena> arenas;
    std::vector<u64*> arena_graveyard;   // outgrown buffers (may still be in use by queued work)
};

// RAII scratch scope on the context's current stream
struct Scratch {
    Ctx& c;
    Ctx::Arena* a;
    size_t mark;
    explicit Scratch(Ctx& ctx);
    ~Scratch();
    u64* take(size_t words);
};

// Diagnosis of host-side stalls: with HC_HOST_TRACE=<ms>, any traced scope
// (allocation, free, launch, run-ahead wait) that blocks the issuing thread
// longer than that is reported on stderr.
double host_trace_threshold_ms();
struct HostTrace {
    const char* what;
    double t0 = 0;
    explicit HostTrace(const char* w);
    ~HostTrace();
};

// Programmatic dependent launch (sm_90+): every kernel is launched with
// programmatic stream serialisation and starts with pdl_enter(): it lets the
// next kernel of the stream begin launching, then waits until the previous
// kernel has completed and its writes are visible -- ordering identical to
// plain stream order, minus the launch gap.  HC_PDL=0 launches plainly.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
    pdl_trigger();
    pdl_wait();
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_k(Ctx& c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    HC_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// cudaFuncAttributeMaxDynamicSharedMemorySize once per (kernel, device);
// thread-safe (contexts may be driven from several host threads)
void set_smem_attr(const void* kern, size_t bytes);
template <class K>
inline void set_smem(K kern, size_t bytes) {
    set_smem_attr(reinterpret_cast<const void*>(kern), bytes);
}

// RAII scope around one kernel launch: counts it and, when profiling,
// brackets it with CUDA events on the context stream.  `bytes` is the
// launch's algorithmic HBM traffic (inputs read once + outputs written once).
struct Launch {
    Ctx& c;
    int idx = -1;
    HostTrace trace;
    Launch(Ctx& ctx, const char* name, double bytes);
    ~Launch();
};

// ---- kernels / launchers (ntt.cu, kernels.cu) ----
void ntt_forward(Ctx& c, const JobList& jobs);
void ntt_inverse(Ctx& c, const JobList& jobs);
void ntt_forward_chunks(Ctx& c, const JobList& jobs);

// ---- context (context.cu) ----
Ctx* ctx_create(int logN, int nq, const int* qbits, int np, const int* pbits, int alpha,
                int log_scale, int hw, double sigma, u64 seed, int device);
void ctx_destroy(Ctx* c);
Key& get_key(Ctx& c, int gid);
int encode_host(const Ctx& c, const double* zr, const double* zi, double scale, int64_t* coef);
void decode_host(const Ctx& c, const double* m, double* zr, double* zi);
CtP new_ct(Ctx& c, int level, int npoly = 2);
PtP new_pt(Ctx& c, int level);
PtP encode_pt(Ctx& c, const double* zr, const double* zi, int level, double scale);
CtP encrypt_coef_dev(Ctx& c, const int64_t* d_m, int level, u64 nonce);
CtP encrypt(Ctx& c, const double* zr, const double* zi, int level, u64 nonce);
void decrypt(Ctx& c, const Ct& a, double* zr, double* zi);
CtP refresh(Ctx& c, const Ct& a, u64 nonce);
std::vector<CtP> refresh_batch(Ctx& c, const std::vector<const Ct*>& a, const std::vector<u64>& nonces);
u64 galois_rot(const Ctx& c, int64_t r);

// ---- evaluator (evaluator.cu): exact CKKS ops, DESIGN.md §3 ----
CtP ev_add(Ctx& c, const Ct& a, const Ct& b, bool sub);
CtP ev_add_pt(Ctx& c, const Ct& a, const Pt& p, bool sub, bool pt_minus_ct);
CtP ev_add_const(Ctx& c, const Ct& a, double re, double im, bool negate_ct);
CtP ev_neg(Ctx& c, const Ct& a);
CtP ev_mul_pt(Ctx& c, const Ct& a, const Pt& p);
CtP ev_mul_const(Ctx& c, const Ct& a, double re, double im);
CtP ev_mult(Ctx& c, const Ct& a, const Ct& b);
CtP ev_automorph(Ctx& c, const Ct& a, u64 g);
CtP ev_mul_i(Ctx& c, const Ct& a);
CtP ev_rescale(Ctx& c, const Ct& a);
CtP ev_level_adjust(Ctx& c, const Ct& a, int to);
CtP ev_drop(Ctx& c, const Ct& a, int to);

}  // namespace hc
