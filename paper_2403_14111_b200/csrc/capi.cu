// extern "C" boundary (include/hc.h): handle wrappers, error mapping.
#include <array>
#include <cstdio>
#include <cstring>
#include <map>

#include <cstdlib>
#include "../../include/hc.h"
#include "evaluator.h"
#include "kernels.cuh"
#include "schedules.h"

struct hc_ctx {
    hc::Ctx* c;
    bool auto_boot = false;
    std::shared_ptr<hc::Ctx> sp;      // released by hc_ctx_destroy; the context dies with its last handle
};
// members are destroyed in reverse order: the residues (p) go back to the
// context's pool before the owner reference can drop the context itself
struct hc_ct {
    std::shared_ptr<hc::Ctx> owner;
    hc::CtP p;
};
struct hc_pt {
    std::shared_ptr<hc::Ctx> owner;
    hc::PtP p;
};

static thread_local std::string g_err;

template <class F>
static int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const hc::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

static hc_ct* wrap(hc::CtP p) {
    std::shared_ptr<hc::Ctx> owner = p->ctx->self.lock();
    return new hc_ct{std::move(owner), std::move(p)};
}

extern "C" {

const char* hc_last_error(void) { return g_err.c_str(); }

int hc_ctx_create(int log_n, int nq, const int* qbits, int np, const int* pbits, int alpha, int log_scale,
                  int hamming_weight, double sigma, uint64_t seed, int device, hc_ctx** out) {
    return guard([&] {
        hc::Ctx* c = hc::ctx_create(log_n, nq, qbits, np, pbits, alpha, log_scale, hamming_weight, sigma, seed,
                                    device);
        std::shared_ptr<hc::Ctx> sp(c, [](hc::Ctx* p) { hc::ctx_destroy(p); });
        c->self = sp;
        *out = new hc_ctx{c, false, sp};
    });
}

int hc_ctx_destroy(hc_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        delete ctx;    // the context itself is destroyed once no handle references it
    });
}

int hc_ctx_info(hc_ctx* ctx, uint64_t* moduli, double* scales) {
    return guard([&] {
        for (int i = 0; i < ctx->c->nall; i++) moduli[i] = ctx->c->pr[i].q;
        for (int l = 0; l <= ctx->c->L; l++) scales[l] = ctx->c->scale[l];
    });
}

int hc_set_grid_rows(hc_ctx* ctx, int grid_rows) {
    const int S = ctx->c->N / 2;
    if (grid_rows < 1 || grid_rows > S || (grid_rows & (grid_rows - 1))) {
        g_err = "grid_rows must be a power of two <= slot count";
        return HC_EPARAM;
    }
    ctx->c->grid_rows = grid_rows;
    return 0;
}

int hc_set_streams(hc_ctx* ctx, int n) {
    if (n < 1 || n > 64) {
        g_err = "stream count must be in [1, 64]";
        return HC_EPARAM;
    }
    ctx->c->fork_cap = n;
    return 0;
}

int hc_set_auto_bootstrap(hc_ctx* ctx, int on) {
    ctx->auto_boot = on != 0;
    return 0;
}

int hc_set_hoist(hc_ctx* ctx, int on) {
    ctx->c->hoist = on != 0;
    return 0;
}

int hc_ctx_counts(hc_ctx* ctx, int64_t* counts, int reset) {
    std::lock_guard<std::mutex> g(ctx->c->mu);
    for (int i = 0; i < HC_NCOUNTS; i++) {
        if (counts) counts[i] = ctx->c->counts[i];
        if (reset) ctx->c->counts[i] = 0;
    }
    return 0;
}

int hc_ctx_nonce(hc_ctx* ctx, uint64_t* get, const uint64_t* set) {
    std::lock_guard<std::mutex> g(ctx->c->mu);
    if (get) *get = ctx->c->nonce;
    if (set) ctx->c->nonce = *set;
    return 0;
}

static void io_drain(hc::Ctx& c) {
    if (!c.copy_stream) return;
    HC_CUDA(cudaStreamSynchronize(c.copy_stream));
    HC_CUDA(cudaStreamSynchronize(c.d2h_stream));
    c.io_pending.clear();
}

// make the context stream wait for every transfer issued so far
static void io_join(hc::Ctx& c) {
    if (!c.copy_stream) return;
    for (cudaStream_t s : {c.copy_stream, c.d2h_stream}) {
        cudaEvent_t e = c.get_event();
        HC_CUDA(cudaEventRecord(e, s));
        HC_CUDA(cudaStreamWaitEvent(c.stream, e, 0));
        c.ev_free.push_back(e);
    }
}

static void io_stream(hc::Ctx& c) {
    if (!c.copy_stream) {
        HC_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
        HC_CUDA(cudaStreamCreateWithFlags(&c.d2h_stream, cudaStreamNonBlocking));
    }
}

int hc_sync(hc_ctx* ctx) {
    return guard([&] {
        io_join(*ctx->c);
        HC_CUDA(cudaStreamSynchronize(ctx->c->stream));
        io_drain(*ctx->c);
    });
}

int hc_keygen(hc_ctx* ctx, int g) { return guard([&] { hc::get_key(*ctx->c, g); }); }

int hc_key_download(hc_ctx* ctx, int g, uint64_t* out) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        const hc::Key& k = hc::get_key(c, g);
        const size_t words = (size_t)c.dnum * 2 * c.nall * c.N;
        HC_CUDA(cudaMemcpyAsync(out, k.d, words * 8, cudaMemcpyDeviceToHost, c.stream));
        HC_CUDA(cudaStreamSynchronize(c.stream));
    });
}

uint64_t hc_galois_rot(hc_ctx* ctx, int64_t r) { return hc::galois_rot(*ctx->c, r); }

int hc_ct_free(hc_ct* ct) {
    hc::HostTrace tr("hc_ct_free");
    return guard([&] { delete ct; });
}
int hc_ct_level(const hc_ct* ct) { return ct->p->level; }

int hc_ct_download(const hc_ct* ct, uint64_t* out) {
    return guard([&] {
        hc::Ctx& c = *ct->p->ctx;
        HC_CUDA(cudaMemcpyAsync(out, ct->p->d, ct->p->words() * 8, cudaMemcpyDeviceToHost, c.stream));
        HC_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int hc_ct_upload(hc_ctx* ctx, const uint64_t* in, int level, hc_ct** out) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        if (level < 0 || level > c.L) throw hc::Error(HC_EPARAM, "level out of range");
        hc::CtP p = hc::new_ct(c, level);
        HC_CUDA(cudaMemcpyAsync(p->d, in, p->words() * 8, cudaMemcpyHostToDevice, c.stream));
        HC_CUDA(cudaStreamSynchronize(c.stream));
        *out = wrap(p);
    });
}

int hc_ct_upload_async(hc_ctx* ctx, const uint64_t* in, int level, hc_ct** out) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        if (level < 0 || level > c.L) throw hc::Error(HC_EPARAM, "level out of range");
        io_stream(c);
        // allocated on the copy stream, so the copy does not queue behind compute
        cudaStream_t saved = c.stream;
        c.stream = c.copy_stream;
        hc::CtP p;
        try {
            p = hc::new_ct(c, level);
        } catch (...) {
            c.stream = saved;
            throw;
        }
        c.stream = saved;
        HC_CUDA(cudaMemcpyAsync(p->d, in, p->words() * 8, cudaMemcpyHostToDevice, c.copy_stream));
        cudaEvent_t e = c.get_event();
        HC_CUDA(cudaEventRecord(e, c.copy_stream));
        HC_CUDA(cudaStreamWaitEvent(c.stream, e, 0));
        c.ev_free.push_back(e);
        *out = wrap(p);
    });
}

int hc_ct_download_async(const hc_ct* ct, uint64_t* out) {
    return guard([&] {
        hc::Ctx& c = *ct->p->ctx;
        io_stream(c);
        cudaEvent_t e = c.get_event();
        HC_CUDA(cudaEventRecord(e, c.stream));
        HC_CUDA(cudaStreamWaitEvent(c.d2h_stream, e, 0));
        c.ev_free.push_back(e);
        HC_CUDA(cudaMemcpyAsync(out, ct->p->d, ct->p->words() * 8, cudaMemcpyDeviceToHost, c.d2h_stream));
        c.io_pending.push_back(ct->p);
    });
}

int hc_ct_device_ptr(const hc_ct* ct, uint64_t** dptr) {
    *dptr = ct->p->d;
    return 0;
}

int hc_pt_free(hc_pt* pt) {
    return guard([&] { delete pt; });
}

int hc_encode_pt(hc_ctx* ctx, const double* re, const double* im, int level, hc_pt** out) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        if (level < 0 || level > c.L) throw hc::Error(HC_EPARAM, "level out of range");
        *out = new hc_pt{ctx->sp, hc::encode_pt(c, re, im, level, c.scale[level])};
    });
}

int hc_pt_download(const hc_pt* pt, uint64_t* out) {
    return guard([&] {
        hc::Ctx& c = *pt->p->ctx;
        HC_CUDA(cudaMemcpyAsync(out, pt->p->d, (size_t)(pt->p->level + 1) * c.N * 8, cudaMemcpyDeviceToHost,
                                c.stream));
        HC_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int hc_encode_coef(hc_ctx* ctx, const double* re, const double* im, double scale, int64_t* coef) {
    return guard([&] {
        if (hc::encode_host(*ctx->c, re, im, scale, coef)) throw hc::Error(HC_EENCODE, "encode overflow");
    });
}

int hc_encrypt(hc_ctx* ctx, const double* re, const double* im, int level, uint64_t nonce, hc_ct** out) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        if (level < 0 || level > c.L) throw hc::Error(HC_EPARAM, "level out of range");
        *out = wrap(hc::encrypt(c, re, im, level, nonce));
    });
}

int hc_decrypt(hc_ctx* ctx, const hc_ct* ct, double* re, double* im) {
    return guard([&] { hc::decrypt(*ctx->c, *ct->p, re, im); });
}

static hc::Pattern pattern_of(hc_ctx* ctx, const double* re, const double* im, const char* key) {
    hc::Pattern p;
    p.key = std::string("py:") + (key ? key : "");
    const int S = ctx->c->N / 2;
    p.vals.resize(S);
    for (int i = 0; i < S; i++) p.vals[i] = {re[i], im ? im[i] : 0.0};
    return p;
}

int hc_op_add(hc_ctx* ctx, const hc_ct* a, const hc_ct* b, int sub, hc_ct** out) {
    return guard([&] { *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).add(a->p, b->p, sub != 0)); });
}

int hc_op_add_scalar(hc_ctx* ctx, const hc_ct* a, double re, double im, int mode, hc_ct** out) {
    return guard([&] {
        *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).add_c(a->p, {re, im}, mode == 1, mode == 2));
    });
}

int hc_op_add_plain(hc_ctx* ctx, const hc_ct* a, const double* re, const double* im, const char* key, int mode,
                    hc_ct** out) {
    return guard([&] {
        hc::Pattern p = pattern_of(ctx, re, im, key);
        *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).add_p(a->p, p, mode == 1, mode == 2));
    });
}

int hc_op_mult(hc_ctx* ctx, const hc_ct* a, const hc_ct* b, hc_ct** out) {
    return guard([&] { *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).mult(a->p, b->p)); });
}

int hc_op_mult_scalar(hc_ctx* ctx, const hc_ct* a, double re, double im, hc_ct** out) {
    return guard([&] { *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).mult_c(a->p, {re, im})); });
}

int hc_op_mult_plain(hc_ctx* ctx, const hc_ct* a, const double* re, const double* im, const char* key,
                     hc_ct** out) {
    return guard([&] {
        hc::Pattern p = pattern_of(ctx, re, im, key);
        *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).mult_p(a->p, p));
    });
}

int hc_op_lrot(hc_ctx* ctx, const hc_ct* a, int64_t r, hc_ct** out) {
    return guard([&] { *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).lrot(a->p, r)); });
}

int hc_op_lrot_hoisted(hc_ctx* ctx, const hc_ct* a, const int64_t* rs, int n, hc_ct** outs) {
    return guard([&] {
        if (n < 0) throw hc::Error(HC_EPARAM, "negative rotation count");
        std::vector<int64_t> r(rs, rs + n);
        auto o = hc::Eval(*ctx->c, ctx->auto_boot).lrot_hoisted({a->p}, r);
        for (int k = 0; k < n; k++) outs[k] = wrap(o[0][k]);
    });
}

int hc_op_ladder(hc_ctx* ctx, const hc_ct* a, int64_t stride, int steps, hc_ct** out) {
    return guard([&] {
        if (steps < 0 || steps > 30) throw hc::Error(HC_EPARAM, "ladder: bad step count");
        *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).ladder(a->p, stride, steps));
    });
}

int hc_op_mult_sum(hc_ctx* ctx, const hc_ct* const* a, const hc_ct* const* b, int n, hc_ct** out) {
    return guard([&] {
        if (n < 1) throw hc::Error(HC_EPARAM, "empty product sum");
        std::vector<hc::CtP> xs(n), ys(n);
        for (int q = 0; q < n; q++) { xs[q] = a[q]->p; ys[q] = b[q]->p; }
        *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).mult_sum_batch({xs}, {ys})[0]);
    });
}

int hc_op_conj(hc_ctx* ctx, const hc_ct* a, hc_ct** out) {
    return guard([&] { *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).conj(a->p)); });
}

int hc_op_mul_i(hc_ctx* ctx, const hc_ct* a, hc_ct** out) {
    return guard([&] { *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).mul_i(a->p)); });
}

int hc_op_bootstrap(hc_ctx* ctx, const hc_ct* a, hc_ct** out) {
    return guard([&] { *out = wrap(hc::Eval(*ctx->c, ctx->auto_boot).bootstrap(a->p)); });
}

int hc_rescale(hc_ctx* ctx, const hc_ct* a, hc_ct** out) {
    return guard([&] { *out = wrap(hc::ev_rescale(*ctx->c, *a->p)); });
}

int hc_level_adjust(hc_ctx* ctx, const hc_ct* a, int level, hc_ct** out) {
    return guard([&] { *out = wrap(hc::ev_level_adjust(*ctx->c, *a->p, level)); });
}

int hc_ctx_model_bytes(hc_ctx* ctx, double* bytes, int reset) {
    return guard([&] {
        std::lock_guard<std::mutex> g(ctx->c->mu);
        if (bytes) *bytes = ctx->c->model_bytes;
        if (reset) ctx->c->model_bytes = 0;
    });
}

int hc_set_app_level(hc_ctx* ctx, int level) {
    return guard([&] {
        if (level < 1 || level > ctx->c->L) throw hc::Error(HC_EPARAM, "application level out of range");
        ctx->c->app_L = level;
    });
}

int hc_set_bootstrap(hc_ctx* ctx, int mode) {
    return guard([&] {
        if (mode < 0 || mode > 1) throw hc::Error(HC_EPARAM, "bootstrap mode is 0 (surrogate) or 1 (CKKS)");
        if (mode == 1 && ctx->c->L - 17 != ctx->c->app_L)
            throw hc::Error(HC_EPARAM, "CKKS bootstrapping needs 17 chain levels above the application's");
        ctx->c->boot_mode = mode;
    });
}

int hc_bootstrap_ct(hc_ctx* ctx, const hc_ct* a, hc_ct** out) {
    return guard([&] { *out = wrap(hc::ev_bootstrap(*ctx->c, a->p)); });
}

int hc_set_shard(hc_ctx* ctx, int total_blocks, int first_block) {
    return guard([&] {
        if (total_blocks < 0 || first_block < 0 || (total_blocks && first_block >= total_blocks))
            throw hc::Error(HC_EPARAM, "bad shard");
        ctx->c->shard_total = total_blocks;
        ctx->c->shard_first = first_block;
    });
}

int hc_set_pass_shard(hc_ctx* ctx, int world, int rank, hc_reduce_fn reduce_fn, void* user) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) throw hc::Error(HC_EPARAM, "bad pass shard");
        if (world > 1 && !reduce_fn) throw hc::Error(HC_EPARAM, "pass sharding needs a reducer");
        hc::Ctx& c = *ctx->c;
        c.pass_world = world;
        c.pass_rank = rank;
        if (world == 1) {
            c.pass_reducer = nullptr;
            return;
        }
        c.pass_reducer = [reduce_fn, user](std::vector<hc::CtP>& cts) {
            std::vector<hc_ct*> hs(cts.size());
            for (size_t i = 0; i < cts.size(); i++) hs[i] = wrap(cts[i]);
            const int rc = reduce_fn(user, hs.data(), (int)hs.size());
            for (size_t i = 0; i < cts.size(); i++) { cts[i] = hs[i]->p; delete hs[i]; }
            if (rc) throw hc::Error(HC_ECUDA, "cross-rank pass reduction failed");
        };
    });
}

int hc_ctx_stream(hc_ctx* ctx, void** stream) {
    return guard([&] { *stream = (void*)ctx->c->stream; });
}

int hc_mod_reduce(hc_ctx* ctx, hc_ct* ct) {
    return guard([&] { hc::k_mod_reduce(*ctx->c, ct->p->d, ct->p->level + 1, ct->p->npoly); });
}

// ---- measurement ----

int hc_timer_begin(hc_ctx* ctx) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        if (!c.t0) { HC_CUDA(cudaEventCreate(&c.t0)); HC_CUDA(cudaEventCreate(&c.t1)); }
        HC_CUDA(cudaEventRecord(c.t0, c.stream));
    });
}

int hc_timer_end(hc_ctx* ctx, float* ms) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        io_join(c);   // pending downloads are inside the timed region
        HC_CUDA(cudaEventRecord(c.t1, c.stream));
        HC_CUDA(cudaEventSynchronize(c.t1));
        HC_CUDA(cudaEventElapsedTime(ms, c.t0, c.t1));
        io_drain(c);
    });
}

int64_t hc_launch_count(hc_ctx* ctx) { return ctx->c->launches; }

int hc_bench_ntt(hc_ctx* ctx, int nlimbs, int reps, int inverse, float* ms) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        if (nlimbs < 1 || reps < 1) throw hc::Error(HC_EPARAM, "bad sizes");
        u64* buf = c.alloc((size_t)nlimbs * c.N);
        HC_CUDA(cudaMemsetAsync(buf, 0, (size_t)nlimbs * c.N * 8, c.stream));
        // HC_BENCH_PRIME=i pins every limb to prime i (default: primes in turn)
        const char* pe = std::getenv("HC_BENCH_PRIME");
        const int pin = pe ? std::atoi(pe) : -1;
        if (pin >= c.nall) throw hc::Error(HC_EPARAM, "HC_BENCH_PRIME out of range");
        auto run = [&] {
            for (int base = 0; base < nlimbs; base += hc::MAXJ) {
                hc::JobList j;
                j.n = std::min(hc::MAXJ, nlimbs - base);
                for (int i = 0; i < j.n; i++) {
                    j.prime[i] = pin >= 0 ? pin : (base + i) % c.nall;
                    j.ptr[i] = buf + (size_t)(base + i) * c.N;
                    j.src[i] = nullptr;
                }
                if (inverse) hc::ntt_inverse(c, j);
                else hc::ntt_forward(c, j);
            }
        };
        run();
        if (!c.t0) { HC_CUDA(cudaEventCreate(&c.t0)); HC_CUDA(cudaEventCreate(&c.t1)); }
        HC_CUDA(cudaEventRecord(c.t0, c.stream));
        for (int r = 0; r < reps; r++) run();
        HC_CUDA(cudaEventRecord(c.t1, c.stream));
        HC_CUDA(cudaEventSynchronize(c.t1));
        HC_CUDA(cudaEventElapsedTime(ms, c.t0, c.t1));
        c.free(buf);
    });
}

static void snap(hc_ctx* ctx, int64_t* b);

int hc_bench_keyswitch(hc_ctx* ctx, const hc_ct* a, int streams, int reps, float* ms) {
    return hc_bench_keyswitch_batch(ctx, a, streams, 1, reps, ms);
}

int hc_bench_keyswitch_batch(hc_ctx* ctx, const hc_ct* a, int streams, int batch, int reps, float* ms) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        if (streams < 1 || batch < 1 || reps < 1) throw hc::Error(HC_EPARAM, "bad sizes");
        int64_t saved[HC_NCOUNTS];
        snap(ctx, saved);
        hc::Eval ev(c, false);
        hc::probe_rotations(ev, a->p, streams, 1, batch);     // warm keys and pool
        HC_CUDA(cudaStreamSynchronize(c.stream));
        if (!c.t0) { HC_CUDA(cudaEventCreate(&c.t0)); HC_CUDA(cudaEventCreate(&c.t1)); }
        HC_CUDA(cudaEventRecord(c.t0, c.stream));
        hc::probe_rotations(ev, a->p, streams, reps, batch);
        HC_CUDA(cudaEventRecord(c.t1, c.stream));
        HC_CUDA(cudaEventSynchronize(c.t1));
        HC_CUDA(cudaEventElapsedTime(ms, c.t0, c.t1));
        std::lock_guard<std::mutex> g(c.mu);
        for (int i = 0; i < HC_NCOUNTS; i++) c.counts[i] = saved[i];
    });
}

int hc_bench_ladder(hc_ctx* ctx, const hc_ct* a, int streams, int batch, int64_t stride, int steps, int reps,
                    float* ms) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        if (streams < 1 || batch < 1 || reps < 1 || steps < 1) throw hc::Error(HC_EPARAM, "bad sizes");
        int64_t saved[HC_NCOUNTS];
        snap(ctx, saved);
        const double model = c.model_bytes;
        hc::Eval ev(c, false);
        hc::probe_ladders(ev, a->p, streams, batch, stride, steps, 1);   // warm keys and pool
        HC_CUDA(cudaStreamSynchronize(c.stream));
        if (!c.t0) { HC_CUDA(cudaEventCreate(&c.t0)); HC_CUDA(cudaEventCreate(&c.t1)); }
        HC_CUDA(cudaEventRecord(c.t0, c.stream));
        hc::probe_ladders(ev, a->p, streams, batch, stride, steps, reps);
        HC_CUDA(cudaEventRecord(c.t1, c.stream));
        HC_CUDA(cudaEventSynchronize(c.t1));
        HC_CUDA(cudaEventElapsedTime(ms, c.t0, c.t1));
        std::lock_guard<std::mutex> g(c.mu);
        for (int i = 0; i < HC_NCOUNTS; i++) c.counts[i] = saved[i];
        c.model_bytes = model;
    });
}

int hc_prof_begin(hc_ctx* ctx) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        HC_CUDA(cudaStreamSynchronize(c.stream));
        for (auto& r : c.prof_recs) { c.ev_free.push_back(r.a); c.ev_free.push_back(r.b); }
        c.prof_recs.clear();
        c.prof = true;
    });
}

int hc_prof_end(hc_ctx* ctx, char* json, int len) {
    return guard([&] {
        hc::Ctx& c = *ctx->c;
        HC_CUDA(cudaStreamSynchronize(c.stream));
        c.prof = false;
        std::map<std::string, std::array<double, 3>> agg;
        for (auto& r : c.prof_recs) {
            float ms = 0;
            HC_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
            auto& a = agg[r.name];
            a[0] += 1;
            a[1] += ms;
            a[2] += r.bytes;
            c.ev_free.push_back(r.a);
            c.ev_free.push_back(r.b);
        }
        c.prof_recs.clear();
        std::string s = "{";
        for (auto& kv : agg) {
            if (s.size() > 1) s += ",";
            char b[256];
            std::snprintf(b, sizeof b, "\"%s\":[%.0f,%.6f,%.0f]", kv.first.c_str(), kv.second[0], kv.second[1],
                          kv.second[2]);
            s += b;
        }
        s += "}";
        if ((int)s.size() + 1 > len) throw hc::Error(HC_EPARAM, "profile buffer too small");
        std::memcpy(json, s.c_str(), s.size() + 1);
    });
}

// ---- schedules ----

static std::vector<hc::CtP> unwrap(const hc_ct* const* a, int n) {
    std::vector<hc::CtP> v(n);
    for (int i = 0; i < n; i++) v[i] = a[i]->p;
    return v;
}

static void add_counts(hc_ctx* ctx, const int64_t* before, int64_t* counts) {
    if (!counts) return;
    std::lock_guard<std::mutex> g(ctx->c->mu);
    for (int i = 0; i < HC_NCOUNTS; i++) counts[i] += ctx->c->counts[i] - before[i];
}

static void snap(hc_ctx* ctx, int64_t* b) {
    std::lock_guard<std::mutex> g(ctx->c->mu);
    for (int i = 0; i < HC_NCOUNTS; i++) b[i] = ctx->c->counts[i];
}

// Bound how far the host runs ahead of the device: a schedule may start
// issuing only once the schedule before the previous one has finished.  Each
// schedule issues thousands of launches and allocations; unbounded run-ahead
// piles up stream-ordered frees the pool cannot recycle yet and forces it to
// grow mid-run.
struct RunAhead {
    hc::Ctx& c;
    explicit RunAhead(hc::Ctx& ctx) : c(ctx) {
        if (c.ra_ev.empty()) {
            c.ra_ev.resize(c.ra_depth);
            for (auto& e : c.ra_ev) {
                HC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                HC_CUDA(cudaEventRecord(e, c.main_stream));
            }
        }
        hc::HostTrace tr("run-ahead wait");
        HC_CUDA(cudaEventSynchronize(c.ra_ev[c.ra_idx]));
    }
    ~RunAhead() {
        cudaEventRecord(c.ra_ev[c.ra_idx], c.main_stream);
        c.ra_idx = (c.ra_idx + 1) % (int)c.ra_ev.size();
    }
};

int hc_diag_abt(hc_ctx* ctx, const hc_ct* const* A, int m, int n, const hc_ct* const* B, int c, double scale,
                hc_ct** out, int64_t* counts) {
    hc::HostTrace tr("hc_diag_abt");
    return guard([&] {
        int64_t before[HC_NCOUNTS];
        snap(ctx, before);
        RunAhead throttle(*ctx->c);
        hc::Eval ev(*ctx->c, ctx->auto_boot);
        std::vector<hc::CtP> res = hc::sched_diag_abt(ev, unwrap(A, m * n), m, n, unwrap(B, n), c, scale);
        for (int i = 0; i < m; i++) out[i] = wrap(res[i]);
        add_counts(ctx, before, counts);
    });
}

int hc_diag_atb(hc_ctx* ctx, const hc_ct* const* A, int m, const hc_ct* const* B, int n, int c, double scale,
                hc_ct** out, int64_t* counts, hc_reduce_fn reduce_fn, void* user) {
    hc::HostTrace tr("hc_diag_atb");
    return guard([&] {
        int64_t before[HC_NCOUNTS];
        snap(ctx, before);
        RunAhead throttle(*ctx->c);
        hc::Eval ev(*ctx->c, ctx->auto_boot);
        hc::Reducer red;
        if (reduce_fn) {
            red = [&](std::vector<hc::CtP>& cts) {
                std::vector<hc_ct*> hs(cts.size());
                for (size_t i = 0; i < cts.size(); i++) hs[i] = wrap(cts[i]);
                // no host synchronisation: the reducer orders its collective
                // after the pre-sums on hc_ctx_stream() (stream handoff)
                const int rc = reduce_fn(user, hs.data(), (int)hs.size());
                for (size_t i = 0; i < cts.size(); i++) { cts[i] = hs[i]->p; delete hs[i]; }
                if (rc) throw hc::Error(HC_ECUDA, "cross-rank reduction failed");
            };
        }
        std::vector<hc::CtP> res = hc::sched_diag_atb(ev, unwrap(A, m), m, unwrap(B, m * n), n, c, scale, red);
        for (int i = 0; i < n; i++) out[i] = wrap(res[i]);
        add_counts(ctx, before, counts);
    });
}

int hc_col_major_abt(hc_ctx* ctx, const hc_ct* const* A, int m, int n, const hc_ct* const* B, int c, double scale,
                     hc_ct** out, int64_t* counts) {
    return guard([&] {
        int64_t before[HC_NCOUNTS];
        snap(ctx, before);
        RunAhead throttle(*ctx->c);
        hc::Eval ev(*ctx->c, ctx->auto_boot);
        std::vector<hc::CtP> res = hc::sched_col_major_abt(ev, unwrap(A, m * n), m, n, unwrap(B, n), c, scale);
        for (int i = 0; i < m; i++) out[i] = wrap(res[i]);
        add_counts(ctx, before, counts);
    });
}

int hc_row_major_atb(hc_ctx* ctx, const hc_ct* const* A, int m, const hc_ct* const* B, int n, int c, double scale,
                     hc_ct** out, int64_t* counts) {
    return guard([&] {
        int64_t before[HC_NCOUNTS];
        snap(ctx, before);
        RunAhead throttle(*ctx->c);
        hc::Eval ev(*ctx->c, ctx->auto_boot);
        std::vector<hc::CtP> res = hc::sched_row_major_atb(ev, unwrap(A, m), m, unwrap(B, m * n), n, c, scale);
        for (int i = 0; i < n; i++) out[i] = wrap(res[i]);
        add_counts(ctx, before, counts);
    });
}

int hc_softmax(hc_ctx* ctx, const hc_ct* const* A, int m, int classes, int period, const double* cfg, hc_ct** out,
               int64_t* counts) {
    return guard([&] {
        int64_t before[HC_NCOUNTS];
        snap(ctx, before);
        RunAhead throttle(*ctx->c);
        hc::Eval ev(*ctx->c, ctx->auto_boot);
        hc::SoftmaxCfg sc;
        if (cfg) sc = hc::SoftmaxCfg::from(cfg);
        std::vector<hc::CtP> res = hc::sched_softmax(ev, unwrap(A, m), classes, period, sc);
        for (int i = 0; i < m; i++) out[i] = wrap(res[i]);
        add_counts(ctx, before, counts);
    });
}

int hc_approx(hc_ctx* ctx, int fn, const hc_ct* const* A, const hc_ct* const* B, int m, int classes, int period,
              const double* cfg, hc_ct** out, int64_t* counts) {
    return guard([&] {
        int64_t before[HC_NCOUNTS];
        snap(ctx, before);
        RunAhead throttle(*ctx->c);
        hc::Eval ev(*ctx->c, ctx->auto_boot);
        hc::SoftmaxCfg sc;
        if (cfg) sc = hc::SoftmaxCfg::from(cfg);
        std::vector<hc::CtP> y;
        if (fn == hc::APPROX_COMP) y = unwrap(B, m);
        std::vector<hc::CtP> res = hc::sched_approx(ev, fn, unwrap(A, m), y, classes, period, sc);
        for (int i = 0; i < m; i++) out[i] = wrap(res[i]);
        add_counts(ctx, before, counts);
    });
}

}  // extern "C"
