#pragma once
#include "hc_internal.h"

namespace hc {

enum EwOpPublic { EWP_ADD = 0, EWP_SUB, EWP_NEG, EWP_PT_ADD, EWP_PT_SUB, EWP_PT_RSUB, EWP_PT_MUL, EWP_CONST_MUL,
                  EWP_CONST_ADD, EWP_CONST_RADD };

// per-limb constant pair (first half / second half of the NTT slots), with Shoup companions
struct ConstTab {
    u64 v[4 * MAXP];
};
void k_elementwise(Ctx& c, int op, u64* out, const u64* a, const u64* b, const ConstTab* consts, int nl, int npoly,
                   int bpoly);
void k_tensor(Ctx& c, u64* d, const u64* a, const u64* b, int nl);
void k_tensor_batch(Ctx& c, int B, u64* const* d, const u64* const* a, const u64* const* b, int nl);
// the element-wise op over B ciphertexts (b may be null when unused)
void k_elementwise_batch(Ctx& c, int op, int B, u64* const* out, const u64* const* a, const u64* const* b,
                         const ConstTab* consts, int nl, int npoly, int bpoly);
// d = sum_q tensor(a[q], b[q]), n <= 8
void k_tensor_sum(Ctx& c, u64* d, const u64* const* a, const u64* const* b, int n, int nl);
void k_automorph(Ctx& c, u64* out, const u64* in, int nlimbs, u64 g);
// ModRaise lift of [2][N] level-0 coefficients to [2][nl][N] (bootstrap.cu)
void k_mod_raise(Ctx& c, u64* out, const u64* X, int nl);
// out [2][nl][N] = sum_t a_t (x) p_t (ciphertexts times NTT plaintexts, no rescale), T <= 16
void k_pt_dot(Ctx& c, u64* out, const u64* const* a, const u64* const* p, int T, int nl);
void k_modup(Ctx& c, u64* up, const u64* X, const u64* D, int level, int beta);
// accumulate: acc += the products (rotate-and-sum stages)
void k_keyprod(Ctx& c, u64* acc, const u64* up, const u64* key, int level, int beta, bool accumulate = false);
// merged: the ModDown + rescale by q_l P of a ct x ct product (W / out have `level` limbs)
void k_moddown_conv(Ctx& c, u64* W, const u64* acc, int level, bool merged = false);
void k_moddown_combine(Ctx& c, u64* out, const u64* acc, const u64* W, const u64* addend, int add_npoly, int level,
                       bool merged = false);
// ACC [2][nt][N] Q limbs += [P]_q d, d = (d0, d1) [2][level+1][N]
void k_fold_p(Ctx& c, u64* acc, const u64* d, int level);
void k_rescale_bcast(Ctx& c, u64* Y, const u64* X, int level, int npoly);
void k_rescale_combine(Ctx& c, u64* out, const u64* a, const u64* Y, int level, int npoly);
void k_uniform(Ctx& c, u64* out, int first_prime, int nl, u64 stream);
void k_cdt(Ctx& c, i64* e, u64 stream);
void k_coef_to_rns(Ctx& c, u64* out, const i64* m, const i64* e, int first_prime, int nl);
void k_key_combine(Ctx& c, u64* b, const u64* a, const u64* s, const u64* s2, const u64* pm, int nl, int dlo,
                   int dhi);
void k_square(Ctx& c, u64* out, const u64* a, int nl);
void k_dec(Ctx& c, u64* x, const u64* c0, const u64* c1, int nl);
void k_refresh_msg(Ctx& c, i64* m, const u64* x, int two, u64 inv01, double ratio);
void k_enc_combine(Ctx& c, u64* c0, const u64* c1, int nl);
void k_mod_reduce(Ctx& c, u64* x, int nl, int npoly);
// batched refresh surrogate stages (B <= KS_MAXB): 0 = decryption limbs into
// xbuf, 1 = message + error + mask into out (c0 in coefficient form), 2 = c0 -= c1 s
void k_refresh_batch(Ctx& c, int B, const u64* const* c0, const u64* const* c1, u64* const* xbuf, u64* const* out,
                     const u64* nonces, int stage, int two, u64 inv01, double ratio);

// batched NTT helpers over contiguous limbs with primes [p0, p0 + n)
void ntt_limbs(Ctx& c, u64* d, int p0, int n, bool inverse, const u64* src = nullptr);

}  // namespace hc
