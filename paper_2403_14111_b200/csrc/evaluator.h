// Policy layer with the reference backend's semantics (emulator.py:160-273):
// ledger increments, per-operand auto-bootstrap at level 0, result level =
// min(levels) (- 1 for products), lrot by 0 is free and returns its input.
// CKKS-specific: operands at different levels are first brought to the
// lower level by an unledgered level adjustment (counted under OP_ADJUST).
#pragma once
#include <complex>
#include <functional>
#include <string>
#include <vector>

#include "hc_internal.h"

namespace hc {

void keyswitch(Ctx& c, const u64* d, int level, const Key& key, u64* out, const u64* addend, int add_npoly);
// fused pipeline (keyswitch.cu) for split-pass rings; false when N < 2^14.
// d and the addend are read through the galois permutation gal / add_gal (0 = none).
bool keyswitch_fused(Ctx& c, const u64* d, u64 gal, int level, const Key& key, u64* out, const u64* addend,
                     int add_npoly, u64 add_gal, const u64* addend2 = nullptr);
// one key switch of a batched pipeline (keyswitch.cu): d is read through the
// batch's Galois element, add (add_npoly polys) through add_gal, add2 as is
struct KsIn {
    const u64* d;
    u64* out;
    const u64* add;
    const u64* add2;
    const u64* key;
};
bool keyswitch_fused_batch(Ctx& c, int B, const KsIn* in, u64 gal, int level, int add_npoly, u64 add_gal);
// hoisted key switches (keyswitch.cu): entry b rotates input src (c0s / c1s)
// by Galois element gal with `key` into out; one ModUp per distinct input
struct KsHoist {
    int src;
    u64 gal;
    const u64* key;
    u64* out;
};
bool keyswitch_hoisted(Ctx& c, const u64* const* c0s, const u64* const* c1s, int level, int B, const KsHoist* e);
// rotate-and-sum stage (keyswitch.cu, DESIGN.md §3 radix ladders): out_b = x_b +
// sum_r sigma_{gals[r]}(x_b), one ModUp and one ModDown per input; nrot <= 7
bool keyswitch_rotsum(Ctx& c, int B, const u64* const* xs, u64* const* outs, int level, int nrot, const u64* gals,
                      const u64* const* keys);
// relinearisation + rescale in one pass (keyswitch.cu): ds[b] = the
// tensor (d0, d1, d2) at `level`, outs[b] at level - 1; false when not fusable
bool keyswitch_relin_rescale(Ctx& c, int B, const u64* const* ds, u64* const* outs, int level, const u64* key);
std::vector<CtP> ev_rotsum_batch(Ctx& c, const std::vector<const Ct*>& xs, const std::vector<u64>& gals);
// CKKS bootstrapping (bootstrap.cu): any level -> app_L
CtP ev_mod_raise(Ctx& c, const Ct& a, int to);
CtP ev_bootstrap(Ctx& c, const CtP& a);
// several ciphertexts bootstrapped together: every step batched (same residues)
std::vector<CtP> ev_bootstrap_batch(Ctx& c, const std::vector<CtP>& a);
// batched primitives (evaluator.cu)
std::vector<CtP> ev_level_adjust_batch(Ctx& c, const std::vector<const Ct*>& xs, int to);
std::vector<CtP> ev_automorph_batch(Ctx& c, const std::vector<const Ct*>& a, u64 g, bool add_self);
std::vector<CtP> ev_mult_batch(Ctx& c, const std::vector<std::pair<const Ct*, const Ct*>>& ab);

// out = sigma_g(a) + a in one key switch (rotate-and-add ladder step); false if not fusable
bool ev_automorph_add(Ctx& c, const Ct& a, u64 g, CtP& out);
bool rescale_fused(Ctx& c, const u64* a, int level, int npoly, u64* out);
// B rescales of npoly-poly inputs at one level in one pipeline (4 launches)
bool rescale_fused_batch(Ctx& c, int B, const u64* const* a, int level, int npoly, u64* const* out);

// a plaintext slot pattern with a cache key (content-addressed by the caller).
// Values are either given (vals) or produced by gen() only on a cache miss,
// so steady-state schedules never rebuild 2^15-slot masks on the host.
struct Pattern {
    std::string key;
    std::vector<std::complex<double>> vals;
    std::function<void(std::vector<std::complex<double>>&)> gen;
};

// Deterministic refresh nonces for a block-parallel run: block p of m, whose
// ops would be interleaved block by block in the reference's sequential order,
// takes for the j-th of r refreshes in an op the nonce
//   base + m * (refreshes in its earlier ops) + p * r + j,
// exactly the nonce the sequential order assigns (all blocks share one level
// history, so every block refreshes the same operands in the same ops).
//
// A shard holding mloc consecutive blocks p .. p + mloc - 1 of m runs them in
// lockstep: a batched op lists its items [sub-op][block] (mloc blocks per
// sub-op), and item i of a sub-op drawing r refreshes takes
//   base + m * events + (p + i) * r + j,
// then events += r -- again the nonces of the whole batch's sequential run.
struct NoncePlan {
    bool on = false;
    u64 base = 0;
    int m = 1, p = 0, mloc = 1;
    u64 events = 0;
};

// operand kinds of the per-op HBM model: ct (op) ct, ct (op) plaintext, ct (op) scalar
enum { MV_CT = 0, MV_PT, MV_SCALAR };
constexpr int MODEL_MULI = 100;   // model kind of mul_i (not a ledger slot)
// limbs (8N bytes each) the §8(d) model charges one op at `level`
double model_limbs(const Ctx& c, int kind, int variant, int level);

struct Eval {
    Ctx& c;
    bool auto_boot;
    NoncePlan plan;
    Eval(Ctx& ctx, bool ab) : c(ctx), auto_boot(ab) {}
    CtP refresh_planned(const CtP& a, int j, int r);
    // records a Bootstrap and returns the nonce of the j-th of r refreshes of an op
    u64 boot_nonce(int j, int r);
    // ready() over a vector: level-0 operands refreshed (block order, batched)
    void ready_batch(std::vector<CtP>& xs);
    // nonces of a batched op whose item i draws r[i] refreshes (records the
    // Bootstraps); sequential draws, or the plan's layout above
    std::vector<u64> batch_nonces(const std::vector<int>& r);

    void rec(int kind, int n = 1);
    // SURVEY §8(d) per-op HBM model of a ledgered op at `level` (operand
    // kind MV_*), accumulated in Ctx::model_bytes (hc_ctx_model_bytes)
    void model(int kind, int variant, int level, int n = 1);
    u64 next_nonce();
    CtP at(const CtP& a, int level);
    // at() over a vector (in place, slot i to level ls[i]), batched per (source, target) level
    std::vector<CtP> at_batch(std::vector<CtP>& xs, const std::vector<int>& ls);
    CtP ready(const CtP& a);

    CtP add(const CtP& a, const CtP& b, bool sub = false);
    CtP sub(const CtP& a, const CtP& b) { return add(a, b, true); }
    CtP add_c(const CtP& a, std::complex<double> s, bool sub = false, bool reversed = false);
    CtP add_p(const CtP& a, const Pattern& p, bool sub = false, bool reversed = false);
    CtP mult(const CtP& a, const CtP& b);
    CtP mult_c(const CtP& a, std::complex<double> s);
    CtP mult_p(const CtP& a, const Pattern& p);
    CtP lrot(const CtP& a, int64_t r);
    CtP rrot(const CtP& a, int64_t r) { return lrot(a, -r); }
    // add(a, lrot(a, r)): one Rot + one Add on the ledger, fused into the key switch
    CtP add_lrot(const CtP& a, int64_t r);
    CtP add_rrot(const CtP& a, int64_t r) { return add_lrot(a, -r); }
    CtP conj(const CtP& a);
    // batched forms (same ledger entries as the per-op calls; one fused
    // key-switch pipeline per level): lrot (add_self: add(a, lrot(a, r))),
    // conj and ct x ct over vectors of independent operands
    std::vector<CtP> lrot_batch(const std::vector<CtP>& xs, int64_t r, bool add_self = false);
    // the reference's doubling ladder over independent operands,
    //   for t < steps: x = add(x, lrot(x, stride * 2^t))      (stride < 0: rrot)
    // (encoding.py:354-359, 378-379, approx.py:165-189).  With the fused
    // schedule forms (Ctx::hoist) two or three steps run as one radix-4 / radix-8
    // rotate-and-sum stage x + sum_u lrot(x, u s) (8 steps -> 3 + 3 + 2): same
    // slot values and ledger (steps Rot + steps Add), one ModUp / ModDown per stage
    std::vector<CtP> ladder(const std::vector<CtP>& xs, int64_t stride, int steps);
    CtP ladder(const CtP& x, int64_t stride, int steps) { return ladder(std::vector<CtP>{x}, stride, steps)[0]; }
    std::vector<CtP> conj_batch(const std::vector<CtP>& xs);
    std::vector<CtP> mult_batch(const std::vector<CtP>& xs, const std::vector<CtP>& ys);
    // fused forms (residues differ from the separate ops, the
    // ledger does not): lrot of every x by every r with one ModUp per x
    // (out[x][r]; r = 0 returns x), and add(...add(mult(a0, b0), mult(a1, b1))...)
    // with one relinearisation and rescale per group (separate ops unless
    // every operand is at one level >= 1 and the group has >= 2 products)
    // mult_p over independent operands (pattern ps[i] for xs[i]) with one
    // batched rescale; same ledger and residues as the separate calls
    std::vector<CtP> mult_p_batch(const std::vector<CtP>& xs, const std::vector<const Pattern*>& ps);
    // add / sub, + - scalar, + - plaintext over independent operands at one
    // level: one launch (the separate ops otherwise); same ledger and residues
    std::vector<CtP> add_batch(const std::vector<CtP>& xs, const std::vector<CtP>& ys, bool sub = false);
    std::vector<CtP> add_c_batch(const std::vector<CtP>& xs, std::complex<double> s, bool sub = false,
                                 bool reversed = false);
    std::vector<CtP> add_p_batch(const std::vector<CtP>& xs, const Pattern& p, bool sub = false,
                                 bool reversed = false);
    // mult_c over independent operands by one scalar, one batched rescale
    std::vector<CtP> mult_c_batch(const std::vector<CtP>& xs, std::complex<double> s);
    std::vector<std::vector<CtP>> lrot_hoisted(const std::vector<CtP>& xs, const std::vector<int64_t>& rs);
    std::vector<CtP> mult_sum_batch(const std::vector<std::vector<CtP>>& as, const std::vector<std::vector<CtP>>& bs);
    CtP mul_i(const CtP& a);
    CtP bootstrap(const CtP& a);
    PtP encoded(const Pattern& p, int level);
};

}  // namespace hc
