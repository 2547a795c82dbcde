// Element-wise, base-conversion, key-product and sampling kernels (sm_100a).
//
// All kernels work on limb-major residue arrays [poly][limb][N] (uint64) in
// HBM.  Element-wise kernels move two words per thread (16-byte vector
// accesses) and use a grid sized in multiples of the SM count; they are
// HBM-bound by construction.  Base conversion (ModUp / ModDown) and the key
// inner product are the integer-heavy parts of key switching.
#include <algorithm>

#include "kernels.cuh"

namespace hc {

static inline int nblocks(size_t work, int threads) {
    size_t b = (work + threads - 1) / threads;
    const size_t cap = 148 * 16;
    return (int)(b < cap ? b : cap);
}

// ---------------------------------------------------------------------------
// element-wise ciphertext ops; prime of limb i is i (Q basis)
// ---------------------------------------------------------------------------

enum EwOp { EW_ADD, EW_SUB, EW_NEG, EW_PT_ADD, EW_PT_SUB, EW_PT_RSUB, EW_PT_MUL, EW_CONST_MUL, EW_CONST_ADD,
            EW_CONST_RADD };

// consts: per limb {lo, lo_shoup, hi, hi_shoup}; grid z = ciphertext of a batch
struct EwPtrs {
    u64* out[KS_MAXB];
    const u64* a[KS_MAXB];
    const u64* b[KS_MAXB];
};
// EW_U index pairs (16 bytes each) per thread: every operand load is issued
// before the first use (one pair per thread ran at ~2.2 TB/s, latency-bound)
constexpr int EW_U = 4;
__global__ void __launch_bounds__(256) ew_kernel(int op, EwPtrs ptr, const ConstTab consts,
                                                 const PrimeDev* __restrict__ primes, int nl, int npoly, int N,
                                                 int bpoly) {
    pdl_enter();
    // grid.y = poly * nl + limb: no integer division on the hot path
    u64* __restrict__ out = ptr.out[blockIdx.z];
    const u64* __restrict__ a = ptr.a[blockIdx.z];
    const u64* __restrict__ b = ptr.b[blockIdx.z];
    const int half = N / 2;
    const int limb = blockIdx.y % nl;
    const int s = blockIdx.y / nl;
    const PrimeDev P = primes[limb];
    const u64 q = P.q;
    // second operand: a ciphertext poly (add / sub, polys below bpoly), a
    // plaintext limb (poly 0 only, except the product), or none
    const bool ctb = op <= EW_SUB, ptb = op >= EW_PT_ADD && op <= EW_PT_MUL;
    const bool hasb = ctb ? s < bpoly : (ptb && (op == EW_PT_MUL || s == 0));
    const u64* __restrict__ bb = ctb ? b + (size_t)blockIdx.y * N : (ptb ? b + (size_t)limb * N : nullptr);
    const u64* __restrict__ aa = a + (size_t)blockIdx.y * N;
    u64* __restrict__ oo = out + (size_t)blockIdx.y * N;
    const int v0 = (blockIdx.x * blockDim.x) * EW_U + threadIdx.x;
    ulonglong2 x[EW_U], y[EW_U];
#pragma unroll
    for (int u = 0; u < EW_U; u++) {
        const int v = v0 + u * (int)blockDim.x;
        if (v < half) x[u] = *reinterpret_cast<const ulonglong2*>(aa + 2 * v);
    }
#pragma unroll
    for (int u = 0; u < EW_U; u++) {
        const int v = v0 + u * (int)blockDim.x;
        y[u] = make_ulonglong2(0, 0);
        if (hasb && v < half) y[u] = *reinterpret_cast<const ulonglong2*>(bb + 2 * v);
    }
#pragma unroll
    for (int u = 0; u < EW_U; u++) {
        const int v = v0 + u * (int)blockDim.x;
        if (v >= half) continue;
        const int k = 2 * v;
        u64 r0, r1;
        switch (op) {
            case EW_ADD:
            case EW_PT_ADD: r0 = add_mod(x[u].x, y[u].x, q); r1 = add_mod(x[u].y, y[u].y, q); break;
            case EW_SUB:
            case EW_PT_SUB: r0 = sub_mod(x[u].x, y[u].x, q); r1 = sub_mod(x[u].y, y[u].y, q); break;
            case EW_PT_RSUB: r0 = sub_mod(y[u].x, x[u].x, q); r1 = sub_mod(y[u].y, x[u].y, q); break;
            case EW_NEG: r0 = neg_mod(x[u].x, q); r1 = neg_mod(x[u].y, q); break;
            case EW_PT_MUL: r0 = mul_mod(x[u].x, y[u].x, P); r1 = mul_mod(x[u].y, y[u].y, P); break;
            case EW_CONST_MUL: {
                const u64* cc = consts.v + 4 * limb + (k < half ? 0 : 2);
                r0 = mul_shoup(x[u].x, cc[0], cc[1], q);
                r1 = mul_shoup(x[u].y, cc[0], cc[1], q);
                break;
            }
            case EW_CONST_ADD:
            case EW_CONST_RADD: {
                const u64 cv = (s == 0) ? consts.v[4 * limb + (k < half ? 0 : 2)] : 0;
                u64 x0 = x[u].x, x1 = x[u].y;
                if (op == EW_CONST_RADD) { x0 = neg_mod(x0, q); x1 = neg_mod(x1, q); }
                r0 = add_mod(x0, cv, q);
                r1 = add_mod(x1, cv, q);
                break;
            }
            default: r0 = r1 = 0;
        }
        *reinterpret_cast<ulonglong2*>(oo + k) = make_ulonglong2(r0, r1);
    }
}

void k_elementwise_batch(Ctx& c, int op, int B, u64* const* out, const u64* const* a, const u64* const* b,
                         const ConstTab* consts, int nl, int npoly, int bpoly) {
    static const ConstTab zero = {};
    const bool pt_b = op >= EW_PT_ADD && op <= EW_PT_MUL;
    const double rd = (double)npoly * nl + (pt_b ? nl : (op <= EW_SUB ? bpoly * nl : 0));
    for (int b0 = 0; b0 < B; b0 += KS_MAXB) {
        const int nb = std::min(KS_MAXB, B - b0);
        EwPtrs p;
        for (int i = 0; i < nb; i++) {
            p.out[i] = out[b0 + i];
            p.a[i] = a[b0 + i];
            p.b[i] = b ? b[b0 + i] : nullptr;
        }
        Launch scope(c, "elementwise", 8.0 * c.N * nb * (rd + (double)npoly * nl));
        dim3 grid((unsigned)((c.N / 2 + 256 * EW_U - 1) / (256 * EW_U)), (unsigned)(npoly * nl), nb);
        launch_k(c, ew_kernel, grid, 256, 0, op, p, consts ? *consts : zero, c.d_primes, nl, npoly, c.N, bpoly);
        HC_CUDA(cudaGetLastError());
    }
}

void k_elementwise(Ctx& c, int op, u64* out, const u64* a, const u64* b, const ConstTab* consts, int nl, int npoly,
                   int bpoly) {
    k_elementwise_batch(c, op, 1, &out, &a, b ? &b : nullptr, consts, nl, npoly, bpoly);
}

// ---------------------------------------------------------------------------
// tensor product: d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1
// ---------------------------------------------------------------------------

// grid (x, limb, ciphertext of the batch): the prime is uniform per CTA and
// every access moves two words (16 bytes)
__global__ void tensor_kernel(EwPtrs ptr, const PrimeDev* __restrict__ primes, int nl, int N) {
    pdl_enter();
    u64* __restrict__ d = ptr.out[blockIdx.z];
    const u64* __restrict__ a = ptr.a[blockIdx.z];
    const u64* __restrict__ b = ptr.b[blockIdx.z];
    const size_t poly = (size_t)nl * N, off = (size_t)blockIdx.y * N;
    const PrimeDev P = primes[blockIdx.y];
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < (size_t)N / 2; v += (size_t)gridDim.x * blockDim.x) {
        const size_t e = off + 2 * v;
        const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(a + e), a1 = *reinterpret_cast<const ulonglong2*>(a + poly + e);
        const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(b + e), b1 = *reinterpret_cast<const ulonglong2*>(b + poly + e);
        U128 x0 = {0, 0}, x1 = {0, 0};
        mac128(x0, a0.x, b1.x);
        mac128(x0, a1.x, b0.x);
        mac128(x1, a0.y, b1.y);
        mac128(x1, a1.y, b0.y);
        *reinterpret_cast<ulonglong2*>(d + e) = make_ulonglong2(mul_mod(a0.x, b0.x, P), mul_mod(a0.y, b0.y, P));
        *reinterpret_cast<ulonglong2*>(d + poly + e) =
            make_ulonglong2(reduce128(x0.hi, x0.lo, P), reduce128(x1.hi, x1.lo, P));
        *reinterpret_cast<ulonglong2*>(d + 2 * poly + e) = make_ulonglong2(mul_mod(a1.x, b1.x, P), mul_mod(a1.y, b1.y, P));
    }
}

void k_tensor_batch(Ctx& c, int B, u64* const* d, const u64* const* a, const u64* const* b, int nl) {
    for (int b0 = 0; b0 < B; b0 += KS_MAXB) {
        const int nb = std::min(KS_MAXB, B - b0);
        EwPtrs p;
        for (int i = 0; i < nb; i++) {
            p.out[i] = d[b0 + i];
            p.a[i] = a[b0 + i];
            p.b[i] = b[b0 + i];
        }
        Launch scope(c, "tensor", 8.0 * c.N * 7 * nl * nb);
        dim3 grid((unsigned)std::max(1, std::min((c.N / 2 + 255) / 256, 2 * 148 * 8 / std::max(1, nl * nb))), nl, nb);
        launch_k(c, tensor_kernel, grid, 256, 0, p, c.d_primes, nl, c.N);
        HC_CUDA(cudaGetLastError());
    }
}

void k_tensor(Ctx& c, u64* d, const u64* a, const u64* b, int nl) { k_tensor_batch(c, 1, &d, &a, &b, nl); }

// sum of n tensor products (fused product sums): each
// component accumulated in 128 bits (at most 2 * TS_MAXN products of
// 61-bit residues) and reduced once
constexpr int TS_MAXN = 8;
struct TensorSrc {
    const u64* a[TS_MAXN];
    const u64* b[TS_MAXN];
};
__global__ void tensor_sum_kernel(u64* __restrict__ d, TensorSrc src, int n, const PrimeDev* __restrict__ primes,
                                  int nl, int N, int accumulate) {
    pdl_enter();
    const size_t poly = (size_t)nl * N;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < poly; e += (size_t)gridDim.x * blockDim.x) {
        const PrimeDev P = primes[e / N];
        // accumulate: continue a longer sum from the previous group's canonical words
        U128 s0 = {accumulate ? d[e] : 0, 0}, s1 = {accumulate ? d[poly + e] : 0, 0},
             s2 = {accumulate ? d[2 * poly + e] : 0, 0};
        for (int q = 0; q < n; q++) {
            const u64 a0 = src.a[q][e], a1 = src.a[q][poly + e], b0 = src.b[q][e], b1 = src.b[q][poly + e];
            mac128(s0, a0, b0);
            mac128(s1, a0, b1);
            mac128(s1, a1, b0);
            mac128(s2, a1, b1);
        }
        d[e] = reduce128(s0.hi, s0.lo, P);
        d[poly + e] = reduce128(s1.hi, s1.lo, P);
        d[2 * poly + e] = reduce128(s2.hi, s2.lo, P);
    }
}

// sums of more than TS_MAXN products run in groups, each continuing the
// previous group's reduced words (exact: the result is the same integer mod q)
void k_tensor_sum(Ctx& c, u64* d, const u64* const* a, const u64* const* b, int n, int nl) {
    if (n < 1 || n > 64) throw Error(-1, "tensor sum: bad operand count");
    for (int q0 = 0; q0 < n; q0 += TS_MAXN) {
        const int m = std::min(TS_MAXN, n - q0);
        TensorSrc src;
        for (int q = 0; q < m; q++) { src.a[q] = a[q0 + q]; src.b[q] = b[q0 + q]; }
        Launch scope(c, "tensor", 8.0 * c.N * (4.0 * m + (q0 ? 6 : 3)) * nl);
        launch_k(c, tensor_sum_kernel, nblocks((size_t)nl * c.N, 256), 256, 0, d, src, m, c.d_primes, nl, c.N,
                 q0 ? 1 : 0);
        HC_CUDA(cudaGetLastError());
    }
}

// ---------------------------------------------------------------------------
// Galois automorphism in the NTT domain: out[j] = in[src(j)]
// ---------------------------------------------------------------------------

__global__ void automorph_kernel(u64* __restrict__ out, const u64* __restrict__ in, int nlimbs, int logN, u64 g) {
    pdl_enter();
    const int N = 1 << logN;
    const u64 mask = 2 * (u64)N - 1;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)nlimbs * N;
         e += (size_t)gridDim.x * blockDim.x) {
        const unsigned j = (unsigned)(e & (N - 1));
        const size_t base = e - j;
        const u64 ex = 2 * (u64)(__brev(j) >> (32 - logN)) + 1;
        const u64 e2 = (ex * g) & mask;
        const unsigned src = __brev((unsigned)((e2 - 1) >> 1)) >> (32 - logN);
        out[e] = in[base + src];
    }
}

void k_automorph(Ctx& c, u64* out, const u64* in, int nlimbs, u64 g) {
    Launch scope(c, "automorph", 16.0 * c.N * nlimbs);
    launch_k(c, automorph_kernel, nblocks((size_t)nlimbs * c.N, 256), 256, 0, out, in, nlimbs, c.logN, g);
    HC_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// ModUp fast base conversion for all active digits of a level.
//   X   : [level+1][N] coefficient form of the input (INTT of d)
//   D   : [level+1][N] NTT form of the input (copied into in-digit limbs)
//   UP  : [beta][nt][N], nt = level+1+K; limb t <-> prime (t <= level ? t : L+1+t-(level+1))
// Non-digit limbs are written in coefficient form (NTT'd afterwards).
// ---------------------------------------------------------------------------

__global__ void modup_kernel(u64* __restrict__ up, const u64* __restrict__ X, const u64* __restrict__ D,
                             const u64* __restrict__ tab, const u64* __restrict__ tab_inv,
                             const u64* __restrict__ negq_tab, const PrimeDev* __restrict__ primes, int level, int L,
                             int K, int alpha, int dnum, int nall, int N) {
    pdl_enter();
    const int j = blockIdx.y;
    const int lo = j * alpha;
    int hi = lo + alpha;
    if (hi > level + 1) hi = level + 1;
    const int na = hi - lo;
    const int nt = level + 1 + K;
    const u64* inv = tab_inv + ((size_t)(level * dnum + j) * alpha) * 2;
    const u64* cf = tab + ((size_t)(level * dnum + j) * alpha) * nall * 2;
    const u64* negq = negq_tab + (size_t)(level * dnum + j) * nall;
    u64* out = up + (size_t)j * nt * N;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        u64 y[8];
        u64 cnt = 0;   // centred conversion: terms from the upper half of their prime
        for (int a = 0; a < na; a++) {
            const u64 q = primes[lo + a].q;
            y[a] = mul_shoup(X[(size_t)(lo + a) * N + k], inv[2 * a], inv[2 * a + 1], q);
            cnt += y[a] > (q - 1) / 2;
        }
        for (int t = 0; t < nt; t++) {
            const int pi = t <= level ? t : L + 1 + (t - level - 1);
            if (t >= lo && t < hi) {
                out[(size_t)t * N + k] = D[(size_t)t * N + k];
                continue;
            }
            const u64 p = primes[pi].q;
            u64 acc = cnt * negq[pi];
            for (int a = 0; a < na; a++) {
                const u64* c2 = cf + ((size_t)a * nall + pi) * 2;
                acc += mul_shoup_lazy(y[a], c2[0], c2[1], p);
                if (acc >= 8 * p) acc -= 8 * p;   // < 8p for any alpha <= 8 (p < 2^60)
            }
            if (acc >= 4 * p) acc -= 4 * p;
            if (acc >= 2 * p) acc -= 2 * p;
            if (acc >= p) acc -= p;
            out[(size_t)t * N + k] = acc;
        }
    }
}

void k_modup(Ctx& c, u64* up, const u64* X, const u64* D, int level, int beta) {
    dim3 grid((c.N + 255) / 256, beta);
    const int nl = level + 1, nt = nl + c.K;
    Launch scope(c, "modup", 8.0 * c.N * (2.0 * nl + (double)beta * nt));
    launch_k(c, modup_kernel, grid, 256, 0, up, X, D, c.d_modup, c.d_modup_inv, c.d_modup_negq, c.d_primes, level,
             c.L, c.K, c.alpha, c.dnum, c.nall, c.N);
    HC_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// key inner product: acc[s][t] = sum_j UP[j][t] * key[j][s][prime(t)]
// ---------------------------------------------------------------------------

__global__ void keyprod_kernel(u64* __restrict__ acc, const u64* __restrict__ up, const u64* __restrict__ key,
                               const PrimeDev* __restrict__ primes, int level, int L, int K, int beta, int nall,
                               int N, int accumulate) {
    pdl_enter();
    const int nt = level + 1 + K;
    const size_t poly = (size_t)nt * N;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < poly; e += (size_t)gridDim.x * blockDim.x) {
        const int t = (int)(e / N);
        const size_t k = e - (size_t)t * N;
        const int pi = t <= level ? t : L + 1 + (t - level - 1);
        const PrimeDev P = primes[pi];
        U128 s0 = {0, 0}, s1 = {0, 0};
        for (int j = 0; j < beta; j++) {
            const u64 u = up[(size_t)j * poly + e];
            const u64* kb = key + ((size_t)(2 * j) * nall + pi) * N + k;
            const u64* ka = kb + (size_t)nall * N;
            mac128(s0, u, *kb);
            mac128(s1, u, *ka);
        }
        u64 r0 = reduce128(s0.hi, s0.lo, P), r1 = reduce128(s1.hi, s1.lo, P);
        if (accumulate) {
            r0 = add_mod(r0, acc[e], P.q);
            r1 = add_mod(r1, acc[poly + e], P.q);
        }
        acc[e] = r0;
        acc[poly + e] = r1;
    }
}

void k_keyprod(Ctx& c, u64* acc, const u64* up, const u64* key, int level, int beta, bool accumulate) {
    const size_t poly = (size_t)(level + 1 + c.K) * c.N;
    const double nt = level + 1 + c.K;
    Launch scope(c, "keyprod", 8.0 * c.N * (3.0 * beta * nt + 2.0 * nt));
    launch_k(c, keyprod_kernel, nblocks(poly, 256), 256, 0, acc, up, key, c.d_primes, level, c.L, c.K, beta,
                                                              c.nall, c.N, accumulate ? 1 : 0);
    HC_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// ModDown: W[s][i] = sum_t [ACC_p_t * (P/p_t)^-1]_{p_t} * [P/p_t]_{q_i}   (coefficient form)
//   ACC: [2][nt][N]; its P limbs (t >= level+1) are already in coefficient form
// ---------------------------------------------------------------------------

// The dropped basis is ACC's limbs mdf .. mdf + nk - 1 (P, or q_l and P for the
// merged ModDown + rescale); W and out have nout limbs per poly.
__global__ void moddown_conv_kernel(u64* __restrict__ W, const u64* __restrict__ acc, const u64* __restrict__ tab,
                                    const u64* __restrict__ tab_inv, const u64* __restrict__ negp,
                                    const PrimeDev* __restrict__ primes, int level, int L, int K, int nall, int N,
                                    int mdf, int nk, int nout) {
    pdl_enter();
    const int s = blockIdx.y;
    const int nt = level + 1 + K;
    const u64* A = acc + (size_t)s * nt * N;
    u64* out = W + (size_t)s * nout * N;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        u64 y[8];
        u64 cnt = 0;   // centred conversion (as in modup_kernel)
        for (int t = 0; t < nk; t++) {
            const int li = mdf + t;
            const u64 p = primes[li <= level ? li : L + 1 + (li - level - 1)].q;
            y[t] = mul_shoup(A[(size_t)li * N + k], tab_inv[2 * t], tab_inv[2 * t + 1], p);
            cnt += y[t] > (p - 1) / 2;
        }
        for (int i = 0; i < nout; i++) {
            const u64 q = primes[i].q;
            u64 v = cnt * negp[i];
            for (int t = 0; t < nk; t++) {
                const u64* c2 = tab + ((size_t)t * nall + i) * 2;
                v += mul_shoup_lazy(y[t], c2[0], c2[1], q);
                if (v >= 8 * q) v -= 8 * q;   // < 8q for any nk <= 8 (q < 2^60)
            }
            if (v >= 4 * q) v -= 4 * q;
            if (v >= 2 * q) v -= 2 * q;
            if (v >= q) v -= q;
            out[(size_t)i * N + k] = v;
        }
    }
}

void k_moddown_conv(Ctx& c, u64* W, const u64* acc, int level, bool merged) {
    dim3 grid((c.N + 255) / 256, 2);
    const int nk = merged ? c.K + 1 : c.K, nout = merged ? level : level + 1, mdf = merged ? level : level + 1;
    Launch scope(c, "moddown_conv", 8.0 * c.N * (2.0 * nk + 2.0 * nout));
    if (merged)
        launch_k(c, moddown_conv_kernel, grid, 256, 0, W, acc, c.d_md2_tab + (size_t)level * (c.K + 1) * c.nall * 2,
                 c.d_md2_inv + (size_t)level * (c.K + 1) * 2, c.d_md2_negd + (size_t)level * c.nall, c.d_primes, level,
                 c.L, c.K, c.nall, c.N, mdf, nk, nout);
    else
        launch_k(c, moddown_conv_kernel, grid, 256, 0, W, acc, c.d_moddown, c.d_moddown_inv, c.d_moddown_negp,
                 c.d_primes, level, c.L, c.K, c.nall, c.N, mdf, nk, nout);
    HC_CUDA(cudaGetLastError());
}

// out[s][i] = (ACC[s][i] - W[s][i]) * P^-1 (+ addend[s][i] when s < add_npoly), i < nout
__global__ void moddown_combine_kernel(u64* __restrict__ out, const u64* __restrict__ acc, const u64* __restrict__ W,
                                       const u64* __restrict__ pinv, const u64* __restrict__ addend, int add_npoly,
                                       const PrimeDev* __restrict__ primes, int level, int K, int N, int nout) {
    pdl_enter();
    const int nl = level + 1, nt = nl + K;
    const size_t poly = (size_t)nout * N;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < 2 * poly; e += (size_t)gridDim.x * blockDim.x) {
        const int s = (int)(e / poly);
        const size_t r = e - (size_t)s * poly;
        const int i = (int)(r / N);
        const u64 q = primes[i].q;
        const u64 a = acc[(size_t)s * nt * N + r];
        u64 v = mul_shoup(a + q - W[e], pinv[2 * i], pinv[2 * i + 1], q);
        if (s < add_npoly) v = add_mod(v, addend[e], q);
        out[e] = v;
    }
}

void k_moddown_combine(Ctx& c, u64* out, const u64* acc, const u64* W, const u64* addend, int add_npoly,
                       int level, bool merged) {
    const int nout = merged ? level : level + 1;
    const size_t work = 2 * (size_t)nout * c.N;
    Launch scope(c, "moddown_combine", 8.0 * c.N * nout * (6.0 + add_npoly));
    launch_k(c, moddown_combine_kernel, nblocks(work, 256), 256, 0, out, acc, W,
             merged ? c.d_md2_dinv + (size_t)level * c.nall * 2 : c.d_pinv, addend, add_npoly, c.d_primes, level, c.K,
             c.N, nout);
    HC_CUDA(cudaGetLastError());
}

// ACC's Q limbs += [P]_q (d0, d1): the tensor's first two polys join the key
// products in the extended basis (relinearisation + rescale in one pass)
__global__ void fold_p_kernel(u64* __restrict__ acc, const u64* __restrict__ d, const u64* __restrict__ pmodq,
                              const PrimeDev* __restrict__ primes, int nl, int nt, int N) {
    pdl_enter();
    const size_t poly = (size_t)nl * N;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < 2 * poly; e += (size_t)gridDim.x * blockDim.x) {
        const int s = (int)(e / poly);
        const size_t r = e - (size_t)s * poly;
        const int i = (int)(r / N);
        const PrimeDev P = primes[i];
        u64* a = acc + (size_t)s * nt * N + r;
        *a = add_mod(*a, mul_mod(d[e], pmodq[i], P), P.q);
    }
}

void k_fold_p(Ctx& c, u64* acc, const u64* d, int level) {
    const int nl = level + 1;
    Launch scope(c, "fold_p", 8.0 * c.N * nl * 6.0);
    launch_k(c, fold_p_kernel, nblocks(2 * (size_t)nl * c.N, 256), 256, 0, acc, d, c.pmodq(), c.d_primes, nl,
             nl + c.K, c.N);
    HC_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// rescale by q_l: Y[s][i] = centred(X[s]) mod q_i; out = (a - NTT(Y)) * q_l^-1
// ---------------------------------------------------------------------------

__global__ void rescale_bcast_kernel(u64* __restrict__ Y, const u64* __restrict__ X, const u64* __restrict__ tab,
                                     const PrimeDev* __restrict__ primes, int level, int npoly, int N) {
    pdl_enter();
    const u64 ql = primes[level].q;
    const size_t per = (size_t)level * N;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < npoly * per; e += (size_t)gridDim.x * blockDim.x) {
        const int s = (int)(e / per);
        const size_t r = e - s * per;
        const int i = (int)(r / N);
        const size_t k = r - (size_t)i * N;
        const u64 q = primes[i].q;
        const u64 v = X[(size_t)s * N + k];
        const u64 qlm = tab[3 * i + 2];
        const u64 vm = mul_shoup(v, 1, primes[i].mu_hi, q);   // v mod q without a 64-bit division
        Y[e] = v > (ql - 1) / 2 ? sub_mod(vm, qlm, q) : vm;
    }
}

__global__ void rescale_combine_kernel(u64* __restrict__ out, const u64* __restrict__ a, const u64* __restrict__ Y,
                                       const u64* __restrict__ tab, const PrimeDev* __restrict__ primes, int level,
                                       int npoly, int N) {
    pdl_enter();
    const size_t per = (size_t)level * N;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < npoly * per; e += (size_t)gridDim.x * blockDim.x) {
        const int s = (int)(e / per);
        const size_t r = e - s * per;
        const int i = (int)(r / N);
        const u64 q = primes[i].q;
        const u64 x = a[(size_t)s * (level + 1) * N + r];
        out[e] = mul_shoup(x + q - Y[e], tab[3 * i], tab[3 * i + 1], q);
    }
}

void k_rescale_bcast(Ctx& c, u64* Y, const u64* X, int level, int npoly) {
    const u64* tab = c.d_rescale + (size_t)level * c.nall * 3;
    Launch scope(c, "rescale_bcast", 8.0 * c.N * npoly * (1.0 + level));
    launch_k(c, rescale_bcast_kernel, nblocks((size_t)npoly * level * c.N, 256), 256, 0, Y, X, tab, c.d_primes,
                                                                                          level, npoly, c.N);
    HC_CUDA(cudaGetLastError());
}

void k_rescale_combine(Ctx& c, u64* out, const u64* a, const u64* Y, int level, int npoly) {
    const u64* tab = c.d_rescale + (size_t)level * c.nall * 3;
    Launch scope(c, "rescale_combine", 8.0 * c.N * npoly * 3.0 * level);
    launch_k(c, rescale_combine_kernel, nblocks((size_t)npoly * level * c.N, 256), 256, 0, out, a, Y, tab,
                                                                                            c.d_primes, level, npoly,
                                                                                            c.N);
    HC_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// sampling, encryption, decryption, refresh
// ---------------------------------------------------------------------------

// out[i][k] = uniform mod prime(first + i), counter (prime index)*N + k
__global__ void uniform_kernel(u64* __restrict__ out, const PrimeDev* __restrict__ primes, int first, int nl, int N,
                               u64 key) {
    pdl_enter();
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)nl * N; e += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / N);
        const int pi = first + i;
        const size_t k = e - (size_t)i * N;
        out[e] = __umul64hi(rng_at(key, (u64)pi * N + k), primes[pi].q);
    }
}

void k_uniform(Ctx& c, u64* out, int first_prime, int nl, u64 stream) {
    Launch scope(c, "sample_uniform", 8.0 * c.N * nl);
    launch_k(c, uniform_kernel, nblocks((size_t)nl * c.N, 256), 256, 0, out, c.d_primes, first_prime, nl, c.N,
                                                                          rng_key(c.seed, stream));
    HC_CUDA(cudaGetLastError());
}

__global__ void cdt_kernel(i64* __restrict__ e, const u64* __restrict__ cdt, int n, int b, int N, u64 key) {
    pdl_enter();
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const u64 r = rng_at(key, (u64)k);
        int cnt = 0;
        for (int i = 0; i < n; i++) cnt += (cdt[i] <= r);
        e[k] = (i64)cnt - b;
    }
}

void k_cdt(Ctx& c, i64* e, u64 stream) {
    Launch scope(c, "sample_gauss", 8.0 * c.N);
    launch_k(c, cdt_kernel, nblocks(c.N, 256), 256, 0, e, c.d_cdt, c.cdt_n, c.cdt_b, c.N, rng_key(c.seed, stream));
    HC_CUDA(cudaGetLastError());
}

// out[i][k] = (m[k] + e[k]) mod q_i for primes 0..nl-1 (e optional)
__global__ void coef_to_rns_kernel(u64* __restrict__ out, const i64* __restrict__ m, const i64* __restrict__ e,
                                   const PrimeDev* __restrict__ primes, int first, int nl, int N) {
    pdl_enter();
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < (size_t)nl * N; x += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(x / N);
        const size_t k = x - (size_t)i * N;
        i64 v = m ? m[k] : 0;
        if (e) v += e[k];
        out[x] = from_i64(v, primes[first + i].q);
    }
}

void k_coef_to_rns(Ctx& c, u64* out, const i64* m, const i64* e, int first_prime, int nl) {
    Launch scope(c, "coef_to_rns", 8.0 * c.N * (2.0 + nl));
    launch_k(c, coef_to_rns_kernel, nblocks((size_t)nl * c.N, 256), 256, 0, out, m, e, c.d_primes, first_prime, nl,
                                                                              c.N);
    HC_CUDA(cudaGetLastError());
}

// b = b_in - a*s (+ pm_i * s2 for limbs in [dlo, dhi)); all prime-indexed from 0 over nl limbs
__global__ void key_combine_kernel(u64* __restrict__ b, const u64* __restrict__ a, const u64* __restrict__ s,
                                   const u64* __restrict__ s2, const u64* __restrict__ pm,
                                   const PrimeDev* __restrict__ primes, int nl, int dlo, int dhi, int N) {
    pdl_enter();
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < (size_t)nl * N; x += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(x / N);
        const PrimeDev P = primes[i];
        u64 v = sub_mod(b[x], mul_mod(a[x], s[x], P), P.q);
        if (s2 && i >= dlo && i < dhi) v = add_mod(v, mul_mod(pm[i], s2[x], P), P.q);
        b[x] = v;
    }
}

void k_key_combine(Ctx& c, u64* b, const u64* a, const u64* s, const u64* s2, const u64* pm, int nl, int dlo,
                   int dhi) {
    launch_k(c, key_combine_kernel, nblocks((size_t)nl * c.N, 256), 256, 0, b, a, s, s2, pm, c.d_primes, nl, dlo,
                                                                              dhi, c.N);
    HC_CUDA(cudaGetLastError());
}

__global__ void square_kernel(u64* __restrict__ out, const u64* __restrict__ a, const PrimeDev* __restrict__ primes,
                              int nl, int N) {
    pdl_enter();
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < (size_t)nl * N; x += (size_t)gridDim.x * blockDim.x)
        out[x] = mul_mod(a[x], a[x], primes[x / N]);
}

void k_square(Ctx& c, u64* out, const u64* a, int nl) {
    launch_k(c, square_kernel, nblocks((size_t)nl * c.N, 256), 256, 0, out, a, c.d_primes, nl, c.N);
    HC_CUDA(cudaGetLastError());
}

// x[i] = c0[i] + c1[i] * s[i] for limbs 0..nl-1
__global__ void dec_kernel(u64* __restrict__ x, const u64* __restrict__ c0, const u64* __restrict__ c1,
                           const u64* __restrict__ s, const PrimeDev* __restrict__ primes, int nl, int N) {
    pdl_enter();
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)nl * N; e += (size_t)gridDim.x * blockDim.x) {
        const PrimeDev P = primes[e / N];
        x[e] = add_mod(c0[e], mul_mod(c1[e], s[e], P), P.q);
    }
}

void k_dec(Ctx& c, u64* x, const u64* c0, const u64* c1, int nl) {
    Launch scope(c, "decrypt_limbs", 8.0 * c.N * 4 * nl);
    launch_k(c, dec_kernel, nblocks((size_t)nl * c.N, 256), 256, 0, x, c0, c1, c.d_sk, c.d_primes, nl, c.N);
    HC_CUDA(cudaGetLastError());
}

// refresh surrogate message: m'[k] = rint(m_d * ratio), m_d = x0c + q0 * kc
__global__ void refresh_msg_kernel(i64* __restrict__ m, const u64* __restrict__ x, const PrimeDev* __restrict__ primes,
                                   int two, u64 inv_q0_mod_q1, double ratio, int N) {
    pdl_enter();
    const PrimeDev P0 = primes[0];
    const PrimeDev P1 = primes[1];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const u64 v0 = x[k];
        const i64 x0 = v0 > (P0.q - 1) / 2 ? (i64)v0 - (i64)P0.q : (i64)v0;
        double md;
        if (!two) {
            md = __ll2double_rn(x0);
        } else {
            const u64 d = sub_mod(x[N + k], from_i64(x0, P1.q), P1.q);
            const u64 kk = mul_mod(d, inv_q0_mod_q1, P1);
            const i64 kc = kk > (P1.q - 1) / 2 ? (i64)kk - (i64)P1.q : (i64)kk;
            md = __dadd_rn(__ll2double_rn(x0), __dmul_rn(__ull2double_rn(P0.q), __ll2double_rn(kc)));
        }
        m[k] = __double2ll_rn(__dmul_rn(md, ratio));
    }
}

void k_refresh_msg(Ctx& c, i64* m, const u64* x, int two, u64 inv01, double ratio) {
    Launch scope(c, "refresh_msg", 8.0 * c.N * 3);
    launch_k(c, refresh_msg_kernel, nblocks(c.N, 256), 256, 0, m, x, c.d_primes, two, inv01, ratio, c.N);
    HC_CUDA(cudaGetLastError());
}

// ---- batched refresh surrogate (grid y = ciphertext): the same words as
// dec_kernel / refresh_msg_kernel / cdt_kernel / coef_to_rns_kernel /
// uniform_kernel / enc_combine_kernel applied one ciphertext at a time
struct RefreshBatch {
    const u64* c0[KS_MAXB];
    const u64* c1[KS_MAXB];
    u64* x[KS_MAXB];        // [1 + two][N] decryption limbs
    u64* out[KS_MAXB];      // [2][nl][N]
    u64 key_a[KS_MAXB], key_e[KS_MAXB];
};

__global__ void dec_batch_kernel(RefreshBatch rb, const u64* __restrict__ s, const PrimeDev* __restrict__ primes,
                                 int nl, int N) {
    pdl_enter();
    const int b = blockIdx.y;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)nl * N; e += (size_t)gridDim.x * blockDim.x) {
        const PrimeDev P = primes[e / N];
        rb.x[b][e] = add_mod(rb.c0[b][e], mul_mod(rb.c1[b][e], s[e], P), P.q);
    }
}

// message (refresh_msg_kernel), error (cdt_kernel), residues of m + e
// (coef_to_rns_kernel) and the uniform mask a (uniform_kernel), per coefficient
__global__ void refresh_encode_kernel(RefreshBatch rb, const PrimeDev* __restrict__ primes, const u64* __restrict__ cdt,
                                      int cdt_n, int cdt_b, int two, u64 inv_q0_mod_q1, double ratio, int nl, int N) {
    pdl_enter();
    const int b = blockIdx.y;
    const PrimeDev P0 = primes[0];
    const PrimeDev P1 = primes[1];
    const u64* x = rb.x[b];
    u64* c0 = rb.out[b];
    u64* c1 = rb.out[b] + (size_t)nl * N;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const u64 v0 = x[k];
        const i64 x0 = v0 > (P0.q - 1) / 2 ? (i64)v0 - (i64)P0.q : (i64)v0;
        double md;
        if (!two) {
            md = __ll2double_rn(x0);
        } else {
            const u64 d = sub_mod(x[N + k], from_i64(x0, P1.q), P1.q);
            const u64 kk = mul_mod(d, inv_q0_mod_q1, P1);
            const i64 kc = kk > (P1.q - 1) / 2 ? (i64)kk - (i64)P1.q : (i64)kk;
            md = __dadd_rn(__ll2double_rn(x0), __dmul_rn(__ull2double_rn(P0.q), __ll2double_rn(kc)));
        }
        const i64 m = __double2ll_rn(__dmul_rn(md, ratio));
        const u64 r = rng_at(rb.key_e[b], (u64)k);
        int cnt = 0;
        for (int i = 0; i < cdt_n; i++) cnt += (cdt[i] <= r);
        const i64 v = m + ((i64)cnt - cdt_b);
        for (int i = 0; i < nl; i++) {
            const u64 q = primes[i].q;
            c0[(size_t)i * N + k] = from_i64(v, q);
            c1[(size_t)i * N + k] = __umul64hi(rng_at(rb.key_a[b], (u64)i * N + k), q);
        }
    }
}

__global__ void enc_combine_batch_kernel(RefreshBatch rb, const u64* __restrict__ s, const PrimeDev* __restrict__ primes,
                                         int nl, int N) {
    pdl_enter();
    const int b = blockIdx.y;
    u64* c0 = rb.out[b];
    const u64* c1 = rb.out[b] + (size_t)nl * N;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)nl * N; e += (size_t)gridDim.x * blockDim.x) {
        const PrimeDev P = primes[e / N];
        c0[e] = sub_mod(c0[e], mul_mod(c1[e], s[e], P), P.q);
    }
}

void k_refresh_batch(Ctx& c, int B, const u64* const* c0, const u64* const* c1, u64* const* xbuf, u64* const* out,
                     const u64* nonces, int stage, int two, u64 inv01, double ratio) {
    RefreshBatch rb;
    for (int b = 0; b < B; b++) {
        rb.c0[b] = c0 ? c0[b] : nullptr;
        rb.c1[b] = c1 ? c1[b] : nullptr;
        rb.x[b] = xbuf[b];
        rb.out[b] = out ? out[b] : nullptr;
        rb.key_a[b] = rng_key(c.seed, stream_id(DOM_ENC_A, nonces[b], 0));
        rb.key_e[b] = rng_key(c.seed, stream_id(DOM_ENC_E, nonces[b], 0));
    }
    const int nl = c.app_L + 1;
    if (stage == 0) {
        Launch scope(c, "decrypt_limbs", 8.0 * c.N * 4 * (1 + two) * B);
        dim3 grid((unsigned)std::max(1, nblocks((size_t)(1 + two) * c.N, 256) / B), B);
        launch_k(c, dec_batch_kernel, grid, 256, 0, rb, c.d_sk, c.d_primes, 1 + two, c.N);
    } else if (stage == 1) {
        Launch scope(c, "refresh_encode", 8.0 * c.N * (1.0 + two + 2.0 * nl) * B);
        dim3 grid((unsigned)((c.N + 255) / 256), B);
        launch_k(c, refresh_encode_kernel, grid, 256, 0, rb, c.d_primes, c.d_cdt, c.cdt_n, c.cdt_b, two, inv01, ratio,
                                                          nl, c.N);
    } else {
        Launch scope(c, "enc_combine", 8.0 * c.N * 4 * nl * B);
        dim3 grid((unsigned)std::max(1, nblocks((size_t)nl * c.N, 256) / B), B);
        launch_k(c, enc_combine_batch_kernel, grid, 256, 0, rb, c.d_sk, c.d_primes, nl, c.N);
    }
    HC_CUDA(cudaGetLastError());
}

// c0 = c0 - c1 * s (c0 holds NTT(m + e) on entry)
__global__ void enc_combine_kernel(u64* __restrict__ c0, const u64* __restrict__ c1, const u64* __restrict__ s,
                                   const PrimeDev* __restrict__ primes, int nl, int N) {
    pdl_enter();
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)nl * N; e += (size_t)gridDim.x * blockDim.x) {
        const PrimeDev P = primes[e / N];
        c0[e] = sub_mod(c0[e], mul_mod(c1[e], s[e], P), P.q);
    }
}

void k_enc_combine(Ctx& c, u64* c0, const u64* c1, int nl) {
    Launch scope(c, "enc_combine", 8.0 * c.N * 4 * nl);
    launch_k(c, enc_combine_kernel, nblocks((size_t)nl * c.N, 256), 256, 0, c0, c1, c.d_sk, c.d_primes, nl, c.N);
    HC_CUDA(cudaGetLastError());
}

// cross-rank reduction finish: x mod q_i for any 64-bit word x (a sum of R
// residues, R * q < 2^64): a Shoup product by 1 with the Barrett word
// floor(2^64 / q) (= PrimeDev::mu_hi) lands in [0, 2q), one conditional
// subtraction finishes; grid y = limb, 16-byte accesses
__global__ void mod_reduce_kernel(u64* __restrict__ x, const PrimeDev* __restrict__ primes, int nl, int N) {
    pdl_enter();
    const int limb = blockIdx.y;
    const PrimeDev P = primes[limb % nl];
    ulonglong2* v = reinterpret_cast<ulonglong2*>(x + (size_t)limb * N);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N / 2; e += gridDim.x * blockDim.x) {
        ulonglong2 w = v[e];
        w.x = csub(mul_shoup_lazy(w.x, 1, P.mu_hi, P.q), P.q);
        w.y = csub(mul_shoup_lazy(w.y, 1, P.mu_hi, P.q), P.q);
        v[e] = w;
    }
}

void k_mod_reduce(Ctx& c, u64* x, int nl, int npoly) {
    Launch scope(c, "mod_reduce", 16.0 * c.N * npoly * nl);
    dim3 grid((unsigned)std::min<size_t>((c.N / 2 + 255) / 256, 64), npoly * nl);
    launch_k(c, mod_reduce_kernel, grid, 256, 0, x, c.d_primes, nl, c.N);
    HC_CUDA(cudaGetLastError());
}

// ModRaise lift (bootstrap.cu): X [2][N] coefficients mod q0 (canonical),
// centred, reduced into every prime q_0 .. q_{nl-1}: out [2][nl][N]
// (coefficient form; the caller runs the forward NTT).  grid (x, limb, poly)
__global__ void mod_raise_kernel(u64* __restrict__ out, const u64* __restrict__ X, const PrimeDev* __restrict__ primes,
                                 int nl, int N) {
    pdl_enter();
    const int i = blockIdx.y, s = blockIdx.z;
    const PrimeDev P = primes[i];
    const u64 q0 = primes[0].q, half = (q0 - 1) / 2;
    const u64 q0m = csub(mul_shoup_lazy(q0, 1, P.mu_hi, P.q), P.q);
    const u64* x = X + (size_t)s * N;
    u64* o = out + ((size_t)s * nl + i) * N;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const u64 v = x[k];
        const u64 r = csub(mul_shoup_lazy(v, 1, P.mu_hi, P.q), P.q);
        o[k] = v > half ? sub_mod(r, q0m, P.q) : r;
    }
}

void k_mod_raise(Ctx& c, u64* out, const u64* X, int nl) {
    Launch scope(c, "mod_raise", 8.0 * c.N * 2 * (1.0 + nl));
    dim3 grid((unsigned)std::min((c.N + 255) / 256, 64), nl, 2);
    launch_k(c, mod_raise_kernel, grid, 256, 0, out, X, c.d_primes, nl, c.N);
    HC_CUDA(cudaGetLastError());
}

// Plaintext dot product (bootstrapping's baby-step giant-step inner sums,
// bootstrap.cu): out[s][i] = sum_t a_t[s][i] * p_t[i] mod q_i over T <= 16
// terms, 128-bit accumulation and one reduction (the same words as the
// separate products and modular adds); grid y = poly * nl + limb
struct DotSrc {
    const u64* a[16];
    const u64* p[16];
};
__global__ void pt_dot_kernel(u64* __restrict__ out, DotSrc src, int T, const PrimeDev* __restrict__ primes, int nl,
                              int N) {
    pdl_enter();
    const int limb = blockIdx.y % nl;
    const PrimeDev P = primes[limb];
    const size_t off = (size_t)blockIdx.y * N, poff = (size_t)limb * N;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < (size_t)N / 2; v += (size_t)gridDim.x * blockDim.x) {
        const size_t k = 2 * v;
        U128 s0 = {0, 0}, s1 = {0, 0};
        for (int t = 0; t < T; t++) {
            const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(src.a[t] + off + k);
            const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(src.p[t] + poff + k);
            mac128(s0, x.x, w.x);
            mac128(s1, x.y, w.y);
        }
        *reinterpret_cast<ulonglong2*>(out + off + k) =
            make_ulonglong2(reduce128(s0.hi, s0.lo, P), reduce128(s1.hi, s1.lo, P));
    }
}

void k_pt_dot(Ctx& c, u64* out, const u64* const* a, const u64* const* p, int T, int nl) {
    if (T < 1 || T > 16) throw Error(-1, "pt_dot: 1..16 terms");
    DotSrc src;
    for (int t = 0; t < T; t++) { src.a[t] = a[t]; src.p[t] = p[t]; }
    Launch scope(c, "pt_dot", 8.0 * c.N * nl * (3.0 * T + 2));
    dim3 grid((unsigned)std::min((c.N / 2 + 255) / 256, 64), 2 * nl);
    launch_k(c, pt_dot_kernel, grid, 256, 0, out, src, T, c.d_primes, nl, c.N);
    HC_CUDA(cudaGetLastError());
}

}  // namespace hc
