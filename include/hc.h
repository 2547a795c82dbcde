/*
 * hc.h — C-ABI of the B200-native RNS-CKKS backend for the HETAL hot path.
 *
 * The reference (hefit) ships no FFI: its backend seam is the Python
 * `EmulatorContext` duck type (pkg/src/hefit/emulator.py:111-281), declared
 * as "a backend interface a real HE library could later satisfy"
 * (SPEC.md:19).  Each entry point below replaces one method of that
 * interface (or one layer-2 schedule built on it); the comment names the
 * reference line it stands in for.  Plain pointers and sizes only: no torch
 * types cross this boundary.
 *
 * Conventions
 *   - Every function returns 0 on success or a negative status:
 *       HC_EPARAM (-1) bad argument        HC_ECUDA  (-2) CUDA failure
 *       HC_EDEPTH (-3) level exhausted     -> hefit.errors.DepthExhausted (errors.py:14-17)
 *       HC_ELEVEL (-4) layout/level misuse HC_EENCODE (-5) encoding overflow
 *     hc_last_error() returns the message of the last failure on this thread.
 *   - Ciphertext residues are [2][level+1][N] uint64 in NTT form.
 *   - Slot vectors are N/2 complex values passed as separate re/im doubles.
 *   - Handles are owned by the caller and released with hc_*_free.
 *   - Ops are asynchronous on the context's CUDA stream; download / decrypt
 *     and hc_sync synchronise.
 */
#ifndef HC_H
#define HC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HC_EPARAM -1
#define HC_ECUDA -2
#define HC_EDEPTH -3
#define HC_ELEVEL -4
#define HC_EENCODE -5

typedef struct hc_ctx hc_ctx;
typedef struct hc_ct hc_ct;
typedef struct hc_pt hc_pt;

/* ledger slots of hc_ctx_counts: the reference's OP_KINDS (emulator.py:29)
 * followed by two CKKS-only counters that the reference ledger never sees */
enum { HC_ADD = 0, HC_CMULT, HC_MULT, HC_ROT, HC_CONJ, HC_BOOTSTRAP, HC_LEVEL_ADJUST, HC_KEYSWITCH, HC_NCOUNTS };

const char *hc_last_error(void);

/* EmulatorContext.__init__ (emulator.py:124-148): ring, modulus chain and keys.
 * qbits[nq] (q0 first), pbits[np]; alpha primes per key-switching digit. */
int hc_ctx_create(int log_n, int nq, const int *qbits, int np, const int *pbits, int alpha, int log_scale,
                  int hamming_weight, double sigma, uint64_t seed, int device, hc_ctx **out);
int hc_ctx_destroy(hc_ctx *ctx);
/* moduli[nq+np]; scales[nq] canonical scale per level */
int hc_ctx_info(hc_ctx *ctx, uint64_t *moduli, double *scales);
/* EmulatorContext.grid_rows (emulator.py:144): s0 of the s0 x s1 slot grid */
int hc_set_grid_rows(hc_ctx *ctx, int grid_rows);
/* width of the fork/join over independent diagonal passes (1 = one stream) */
int hc_set_streams(hc_ctx *ctx, int n);
/* EmulatorContext.auto_bootstrap (emulator.py:132) */
int hc_set_auto_bootstrap(hc_ctx *ctx, int on);
/* fused schedule forms on (default) / off: hoisted rotations and one
 * relinearisation per product sum; residues follow the
 * oracle's matching mode, the ledger is the reference's either way */
int hc_set_hoist(hc_ctx *ctx, int on);
/* OpLedger.counts / reset (emulator.py:88-108); counts[HC_NCOUNTS] */
int hc_ctx_counts(hc_ctx *ctx, int64_t *counts, int reset);
/* encryption-randomness counter (shared with the oracle's nonce sequence) */
int hc_ctx_nonce(hc_ctx *ctx, uint64_t *get, const uint64_t *set);
int hc_sync(hc_ctx *ctx);
/* pre-generate the switching key of galois element g (0 = relinearisation) */
int hc_keygen(hc_ctx *ctx, int g);
int hc_key_download(hc_ctx *ctx, int g, uint64_t *out); /* [dnum][2][nq+np][N] */
uint64_t hc_galois_rot(hc_ctx *ctx, int64_t r);

/* ciphertext handles (CipherBlock, emulator.py:49-67) */
int hc_ct_free(hc_ct *ct);
int hc_ct_level(const hc_ct *ct);
int hc_ct_download(const hc_ct *ct, uint64_t *out);
int hc_ct_upload(hc_ctx *ctx, const uint64_t *in, int level, hc_ct **out);
int hc_ct_device_ptr(const hc_ct *ct, uint64_t **dptr);
/* Asynchronous transfers for serving loops: the copy runs on the context's
 * copy stream and overlaps compute.  An upload returns at once; every op
 * issued afterwards sees the data (the context stream waits for the copy).
 * A download is ordered after all work issued so far and completes by the
 * next hc_sync / hc_timer_end; `in` / `out` must stay valid (pinned host
 * memory for full overlap) until then. */
int hc_ct_upload_async(hc_ctx *ctx, const uint64_t *in, int level, hc_ct **out);
int hc_ct_download_async(const hc_ct *ct, uint64_t *out);

/* plaintexts: encoded at scales[level] in NTT form */
int hc_pt_free(hc_pt *pt);
int hc_encode_pt(hc_ctx *ctx, const double *re, const double *im, int level, hc_pt **out);
int hc_pt_download(const hc_pt *pt, uint64_t *out);
/* host encoder KAT: slots -> N integer coefficients at `scale` */
int hc_encode_coef(hc_ctx *ctx, const double *re, const double *im, double scale, int64_t *coef);

/* EmulatorContext.encrypt (emulator.py:160-164) with an explicit nonce */
int hc_encrypt(hc_ctx *ctx, const double *re, const double *im, int level, uint64_t nonce, hc_ct **out);
/* CipherBlock.slots read by encoding.decode (encoding.py:202): audited client decrypt */
int hc_decrypt(hc_ctx *ctx, const hc_ct *ct, double *re, double *im);

/* ---- EmulatorContext ops with the reference's ledger / level semantics ---- */
/* add / sub (emulator.py:195-210): ct +- ct */
int hc_op_add(hc_ctx *ctx, const hc_ct *a, const hc_ct *b, int sub, hc_ct **out);
/* ct + s (mode 0), ct - s (mode 1), s - ct (mode 2) for a complex scalar */
int hc_op_add_scalar(hc_ctx *ctx, const hc_ct *a, double re, double im, int mode, hc_ct **out);
/* same with a slot-vector plaintext; `key` content-addresses the encoding cache */
int hc_op_add_plain(hc_ctx *ctx, const hc_ct *a, const double *re, const double *im, const char *key, int mode,
                    hc_ct **out);
/* mult (emulator.py:212-229): ct x ct -> Mult (+ per-operand auto-bootstrap) */
int hc_op_mult(hc_ctx *ctx, const hc_ct *a, const hc_ct *b, hc_ct **out);
/* cmult (emulator.py:231-235): ct x scalar / ct x plaintext -> CMult */
int hc_op_mult_scalar(hc_ctx *ctx, const hc_ct *a, double re, double im, hc_ct **out);
int hc_op_mult_plain(hc_ctx *ctx, const hc_ct *a, const double *re, const double *im, const char *key, hc_ct **out);
/* lrot (emulator.py:237-247); r mod slots must be non-zero (r == 0 is the caller's no-op) */
int hc_op_lrot(hc_ctx *ctx, const hc_ct *a, int64_t r, hc_ct **out);
/* lrot(a, rs[k]) for k < n with one shared ModUp (hoisted; Rot per non-zero
 * r, r == 0 yields a handle to a itself); outs[n] */
int hc_op_lrot_hoisted(hc_ctx *ctx, const hc_ct *a, const int64_t *rs, int n, hc_ct **outs);
/* the doubling ladder of encoding.py:354-359 / 378-379 and approx.py:165-189,
 *   for t < steps: a = add(a, lrot(a, stride * 2^t))      (stride < 0: rrot),
 * steps Rot + steps Add on the ledger.  With the fused schedule forms on
 * (hc_set_hoist) two steps run as one radix-4 rotate-and-sum stage
 * a + lrot(a, s) + lrot(a, 2s) + lrot(a, 3s) with one ModUp and one ModDown. */
int hc_op_ladder(hc_ctx *ctx, const hc_ct *a, int64_t stride, int steps, hc_ct **out);
/* add(...add(mult(a0, b0), mult(a1, b1))...) over n pairs with one
 * relinearisation + rescale (n Mult, n-1 Add); the separate ops unless all
 * operands share one level >= 1 and n >= 2 */
int hc_op_mult_sum(hc_ctx *ctx, const hc_ct *const *a, const hc_ct *const *b, int n, hc_ct **out);
/* conj (emulator.py:253-257), mul_i (emulator.py:259-265, unledgered) */
int hc_op_conj(hc_ctx *ctx, const hc_ct *a, hc_ct **out);
int hc_op_mul_i(hc_ctx *ctx, const hc_ct *a, hc_ct **out);
/* bootstrap (emulator.py:267-273): the refresh surrogate (decrypt /
 * re-encrypt, needs the secret key) or, after hc_set_bootstrap(ctx, 1), real
 * CKKS bootstrapping (ModRaise, CoeffToSlot, EvalMod, SlotToCoeff; no secret
 * key); the result lands on the application level */
int hc_op_bootstrap(hc_ctx *ctx, const hc_ct *a, hc_ct **out);
/* EmulatorContext.max_level when the chain carries bootstrapping levels
 * above it: fresh encryptions default to it, refreshes land on it */
int hc_set_app_level(hc_ctx *ctx, int level);
/* 0: refresh surrogate (default), 1: CKKS bootstrapping (needs a chain with
 * 17 levels above the application level, e.g. the boot16 parameter set) */
int hc_set_bootstrap(hc_ctx *ctx, int mode);
/* one CKKS bootstrapping of a (any level) regardless of the mode, unledgered */
int hc_bootstrap_ct(hc_ctx *ctx, const hc_ct *a, hc_ct **out);

/* ---- exact CKKS primitives (no ledger), for residue-level parity ---- */
int hc_rescale(hc_ctx *ctx, const hc_ct *a, hc_ct **out);
int hc_level_adjust(hc_ctx *ctx, const hc_ct *a, int level, hc_ct **out);

/* ---- layer-2 schedules (native, same op order and ledger as the reference) ---- */
/* diag_abt (matmul.py:74-110): A[m][n] untiled blocks (row-major handles),
 * B[n] the single block row of the vertically tiled operand, period c.
 * out[m]: the horizontally tiled result column.  counts[HC_NCOUNTS] += delta. */
int hc_diag_abt(hc_ctx *ctx, const hc_ct *const *A, int m, int n, const hc_ct *const *B, int c, double scale,
                hc_ct **out, int64_t *counts);
/* diag_atb (matmul.py:113-154): A[m] (one block column, horizontally tiled,
 * period c), B[m][n]; out[n].  The row_sums pre-add (encoding.py:375-377) is
 * the cross-rank reduction point: with nranks > 1 the caller provides
 * `reduce_fn(user, cts, count)` which must replace each ciphertext's residues
 * by the modular sum over ranks (see hc_mod_reduce). */
typedef int (*hc_reduce_fn)(void *user, hc_ct **cts, int count);
int hc_diag_atb(hc_ctx *ctx, const hc_ct *const *A, int m, const hc_ct *const *B, int n, int c, double scale,
                hc_ct **out, int64_t *counts, hc_reduce_fn reduce_fn, void *user);
/* Table-4 baselines: col_major_abt (matmul.py:160-198), A[m][n] and B[n] untiled
 * (B's c <= s1 rows in one block row), out[m]; row_major_atb (matmul.py:201-237),
 * A[m] untiled (c <= s0 columns), B[m][n], out[n] */
int hc_col_major_abt(hc_ctx *ctx, const hc_ct *const *A, int m, int n, const hc_ct *const *B, int c, double scale,
                     hc_ct **out, int64_t *counts);
int hc_row_major_atb(hc_ctx *ctx, const hc_ct *const *A, int m, const hc_ct *const *B, int n, int c, double scale,
                     hc_ct **out, int64_t *counts);
/* a_softmax (approx.py:312-344) on one horizontally tiled block column A[m] */
int hc_softmax(hc_ctx *ctx, const hc_ct *const *A, int m, int classes, int period, const double *cfg, hc_ct **out,
               int64_t *counts);

/* building blocks of the softmax (hefit/__init__.py:22-28 exports them):
 * fn = HC_APPROX_COMP a_comp(A, B) (approx.py:205-213), HC_APPROX_MAX
 * a_max (approx.py:216-238; A one horizontally tiled block column of period
 * `period`, `classes` active), HC_APPROX_DOMAIN_EXTEND (approx.py:241-253),
 * HC_APPROX_DEP_COMP (approx.py:256-273), HC_APPROX_EXP (approx.py:276-292),
 * HC_APPROX_INV (approx.py:295-309).  A[m] (and B[m]) any blocks; out[m];
 * cfg as for hc_softmax; op order, ledger and refresh points as the reference */
enum { HC_APPROX_COMP = 0, HC_APPROX_MAX, HC_APPROX_DOMAIN_EXTEND, HC_APPROX_DEP_COMP, HC_APPROX_EXP, HC_APPROX_INV };
int hc_approx(hc_ctx *ctx, int fn, const hc_ct *const *A, const hc_ct *const *B, int m, int classes, int period,
              const double *cfg, hc_ct **out, int64_t *counts);

/* finish a cross-rank uint64 sum: residues mod q_i in place (K8); any
 * 64-bit word is accepted (a sum of R canonical residues with R * q < 2^64) */
int hc_mod_reduce(hc_ctx *ctx, hc_ct *ct);
/* block-row sharding: this context holds block rows
 * [first_block, first_block + m) of a batch of total_blocks (0 = off).  The
 * batched softmax then draws every refresh nonce the single-context run of
 * the whole batch would draw (training.py:66-100 data-parallel form), so the
 * replicated weights stay bit-identical across ranks. */
int hc_set_shard(hc_ctx *ctx, int total_blocks, int first_block);
/* diagonal-pass sharding of hc_diag_abt / hc_diag_atb: the
 * c/2 independent passes of matmul.py:102-108 / 141-152 are split round-robin
 * (k = rank mod world); before the conj epilogue each context calls
 * reduce_fn(user, acc, count) on its partial accumulators, which must replace
 * them by the modular sum over ranks (all-reduce + hc_mod_reduce).  The result
 * equals the unsharded schedule's residues.  world = 1 turns it off. */
int hc_set_pass_shard(hc_ctx *ctx, int world, int rank, hc_reduce_fn reduce_fn, void *user);
/* the CUDA stream (cudaStream_t) the context issues on right now; a
 * hc_reduce_fn orders its collective and hc_mod_reduce after the pre-sums on
 * it (stream handoff, no host synchronisation) */
int hc_ctx_stream(hc_ctx *ctx, void **stream);

/* ---- measurement (no reference counterpart) ---- */
/* algorithmic HBM bytes of the ledgered ops issued so far under SURVEY §8(d)'s
 * per-op model (inputs read once, output written once, key-switch
 * intermediates on chip; Add 6/5/4 Lq, CMult 5Lq-2 / 4Lq-2, Mult
 * 4Lq + 2d(Lq+K) + 2(Lq-1), Rot/Conj 4Lq + 2d(Lq+K) limbs of 8N bytes) */
int hc_ctx_model_bytes(hc_ctx *ctx, double *bytes, int reset);
/* CUDA events on the context stream around a region */
int hc_timer_begin(hc_ctx *ctx);
int hc_timer_end(hc_ctx *ctx, float *ms);
/* kernels launched by this context so far */
int64_t hc_launch_count(hc_ctx *ctx);
/* key-switch throughput: `streams` concurrent chains of `reps` rotations of ct
 * (device time in ms over all streams*reps key switches; ledger untouched) */
int hc_bench_keyswitch(hc_ctx *ctx, const hc_ct *ct, int streams, int reps, float *ms);
/* same with `batch` rotations per step of each chain issued as one batched pipeline
 * (device time in ms over all streams*batch*reps key switches) */
int hc_bench_keyswitch_batch(hc_ctx *ctx, const hc_ct *ct, int streams, int batch, int reps, float *ms);
/* ladder throughput: `streams` concurrent branches, each `reps` doubling
 * ladders (hc_op_ladder's stride / steps) over its own batch of `batch`
 * copies of ct (device time in ms; ledger and model untouched) */
int hc_bench_ladder(hc_ctx *ctx, const hc_ct *ct, int streams, int batch, int64_t stride, int steps, int reps,
                    float *ms);
/* batched NTT throughput: `reps` forward (or inverse) transforms of `nlimbs` limbs */
int hc_bench_ntt(hc_ctx *ctx, int nlimbs, int reps, int inverse, float *ms);
/* per-kernel event profiler: JSON {"kernel": [launches, total_ms, algorithmic_bytes], ...} */
int hc_prof_begin(hc_ctx *ctx);
int hc_prof_end(hc_ctx *ctx, char *json, int len);

#ifdef __cplusplus
}
#endif
#endif
