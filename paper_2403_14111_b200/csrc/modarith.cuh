// Word-size modular arithmetic for the sm_100a kernels (primes < 2^61).
//
// * Shoup multiplication by a fixed operand (twiddles, base-conversion
//   constants): one __umul64hi + two low products, result in [0, 2q).
// * Barrett reduction of a 128-bit value with mu = floor(2^128 / q) split in
//   two words; the estimate is off by at most 3, so r < 4q fits 64 bits.
//   Used for ct x ct products and 128-bit lazy accumulations (key inner
//   product, tensor cross term).
#pragma once
#include <cstdint>

typedef uint64_t u64;
typedef int64_t i64;

constexpr int FP_MAXBITS = 46;   // NTT passes run in FP64 for primes below 2^46 (ntt_pass.cuh)

struct PrimeDev {
    u64 q, twoq, mu_hi, mu_lo;   // Barrett constants
    u64 I, I_s;                  // psi^(N/2) and its Shoup companion
    u64 ninv, ninv_s;            // N^-1 (INTT scaling)
    double qd, qinv;             // q and 1/q as doubles (FP64 NTT path)
    int fp;                      // NTT passes on this prime run in FP64 (q < 2^46, ntt_pass.cuh)
};

__device__ __forceinline__ u64 mulhi64(u64 a, u64 b) { return __umul64hi(a, b); }

// x * w mod q, result in [0, 2q); valid for any x < 2^64, w < q
__device__ __forceinline__ u64 mul_shoup_lazy(u64 x, u64 w, u64 ws, u64 q) {
    return x * w - __umul64hi(x, ws) * q;
}
__device__ __forceinline__ u64 mul_shoup(u64 x, u64 w, u64 ws, u64 q) {
    u64 r = mul_shoup_lazy(x, w, ws, q);
    return r >= q ? r - q : r;
}
__device__ __forceinline__ u64 csub(u64 a, u64 q) { return a >= q ? a - q : a; }
__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
__device__ __forceinline__ u64 neg_mod(u64 a, u64 q) { return a ? q - a : 0; }

// 128-bit value (hi, lo) mod q, fully reduced
__device__ __forceinline__ u64 reduce128(u64 hi, u64 lo, const PrimeDev& p) {
    u64 qh = hi * p.mu_hi + __umul64hi(hi, p.mu_lo) + __umul64hi(lo, p.mu_hi);
    u64 r = lo - qh * p.q;
    r = r >= p.twoq ? r - p.twoq : r;
    return r >= p.q ? r - p.q : r;
}

struct U128 {
    u64 lo, hi;
};
__device__ __forceinline__ void mac128(U128& acc, u64 a, u64 b) {
    u64 lo = a * b, hi = __umul64hi(a, b);
    acc.lo += lo;
    acc.hi += hi + (acc.lo < lo ? 1 : 0);
}
__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, const PrimeDev& p) {
    return reduce128(__umul64hi(a, b), a * b, p);
}

// ---- FP64 residue arithmetic for primes below 2^FP_MAXBITS ----
// Residues are integers held exactly in doubles.  x * y mod q for |x| < 2^50,
// 0 <= y < q: h + l is the exact product (h rounded, l = fma(x, y, -h)), the
// quotient rint(h / q) is within 0.6 of the true one, so the result
// (h - qt q) + l is exact with |r| < 0.6q.  Used by the NTT passes
// (ntt_pass.cuh, constant twiddles with w/q precomputed) and the key product.
constexpr double FP_MAGIC = 6755399441055744.0;   // 1.5 * 2^52: fma(x, c, M) - M = rint(x * c)
constexpr double FP_P52 = 4503599627370496.0;     // 2^52
constexpr u64 FP_EXP52 = 0x4330000000000000ull;   // bits of 2^52
constexpr u64 FP_MANT = (1ull << 52) - 1;
// exact word -> double for words below 2^52
__device__ __forceinline__ double fp_word(u64 u) {
    return __dsub_rn(__longlong_as_double((long long)(u | FP_EXP52)), FP_P52);
}
__device__ __forceinline__ double fp_mulmod(double x, double y, double q, double qinv) {
    const double h = __dmul_rn(x, y);
    const double l = __fma_rn(x, y, -h);
    const double qt = __dsub_rn(__fma_rn(h, qinv, FP_MAGIC), FP_MAGIC);
    return __dadd_rn(__fma_rn(-qt, q, h), l);
}
// |v| < 2^52 (an exact integer; v / q < 2^51) -> canonical word in [0, q)
__device__ __forceinline__ u64 fp_canon(double v, double q, double qinv) {
    const double qt = __dsub_rn(__fma_rn(v, qinv, FP_MAGIC), FP_MAGIC);
    double r = __fma_rn(-qt, q, v);   // exact, |r| <= q/2
    r = r < 0 ? __dadd_rn(r, q) : r;
    return (u64)__double_as_longlong(__dadd_rn(r, FP_P52)) & FP_MANT;
}

// int64 -> residue mod q
__device__ __forceinline__ u64 from_i64(i64 v, u64 q) {
    if (v >= 0) return (u64)v % q;
    u64 m = (u64)(-(v + 1)) % q;
    return q - 1 - m;
}

// splitmix64 counter PRNG (spec in DESIGN.md §3; identical to the oracle)
__host__ __device__ __forceinline__ u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ u64 rng_key(u64 seed, u64 stream) {
    return mix64(seed ^ mix64(stream + 0x9E3779B97F4A7C15ULL));
}
__host__ __device__ __forceinline__ u64 rng_at(u64 key, u64 ctr) {
    return mix64(key + ctr * 0x9E3779B97F4A7C15ULL);
}
__host__ __device__ __forceinline__ u64 stream_id(u64 domain, u64 id, u64 sub) {
    return (domain << 48) ^ (id << 16) ^ sub;
}
enum { DOM_SK = 1, DOM_KEY_A = 2, DOM_KEY_E = 3, DOM_ENC_A = 4, DOM_ENC_E = 5 };
