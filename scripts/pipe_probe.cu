// Integer pipe throughput probe (B200): warp-instructions per cycle per SM for
// the multiply forms the NTT butterfly is built from.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe scripts/pipe_probe.cu
// Each kernel runs ACC independent chains of ITER operations per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITER = 4096;
constexpr int ACC = 8;

#define KERNEL(NAME, TYPE, BODY)                                              \
    __global__ void NAME(TYPE* out, uint32_t m0, uint32_t m1) {               \
        TYPE a[ACC];                                                          \
        _Pragma("unroll") for (int j = 0; j < ACC; j++) a[j] = threadIdx.x + j; \
        for (int i = 0; i < ITER; i++) {                                      \
            _Pragma("unroll") for (int j = 0; j < ACC; j++) { BODY; }         \
        }                                                                     \
        TYPE s = 0;                                                           \
        _Pragma("unroll") for (int j = 0; j < ACC; j++) s += a[j];            \
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;                       \
    }

// IMAD.WIDE.U32: 32x32+64 -> 64
KERNEL(k_wide, uint64_t, asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[j]) : "r"(m0 + j), "r"(m1)))
// IMAD: 32x32+32 low
KERNEL(k_lo, uint32_t, asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(m0), "r"(m1)))
// IMAD.HI.U32
KERNEL(k_hi, uint32_t, asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(m0), "r"(m1)))
// IADD3
KERNEL(k_add, uint32_t, asm volatile("add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(m0)))
// mul.lo.u64 (3 IMAD incl one WIDE)
KERNEL(k_mul64, uint64_t, a[j] = a[j] * ((uint64_t)m0 << 20 | m1))
// mul.hi.u64
KERNEL(k_mulhi64, uint64_t, a[j] = __umul64hi(a[j], ((uint64_t)m0 << 32 | m1)) + a[j])

// one IMAD.WIDE.U32 and one IADD3 per step (pipe overlap)
KERNEL(k_mix, uint64_t, asm volatile("{.reg .u32 t; mad.wide.u32 %0, %1, %2, %0; cvt.u32.u64 t, %0; add.u32 t, t, %2; mov.b64 %0, {t, t};}" : "+l"(a[j]) : "r"(m0 + j), "r"(m1)))
// IMAD (lo) and IADD3 alternating
KERNEL(k_mix2, uint32_t, asm volatile("mad.lo.u32 %0, %0, %1, %2; add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(m0), "r"(m1)))

// lazy Shoup product x*w mod q in [0,2q): exact 64x64 high word (4 wide products)
__device__ __forceinline__ uint64_t shoup(uint64_t x, uint64_t w, uint64_t ws, uint64_t q) {
    return x * w - __umul64hi(x, ws) * q;
}
// same with the high word estimated from three 32x32 products (deficit <= 2, result in [0,4q))
__device__ __forceinline__ uint64_t shoup3(uint64_t x, uint64_t w, uint64_t ws, uint64_t q) {
    uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32), yl = (uint32_t)ws, yh = (uint32_t)(ws >> 32);
    uint64_t h = (uint64_t)__umulhi(xh, yl) + __umulhi(xl, yh);
    h += (uint64_t)xh * yh;
    return x * w - h * q;
}
KERNEL(k_shoup, uint64_t, a[j] = shoup(a[j], (uint64_t)m0 << 28 | m1, (uint64_t)m1 << 40 | m0, ((uint64_t)m0 << 40) + 1))
KERNEL(k_shoup3, uint64_t, a[j] = shoup3(a[j], (uint64_t)m0 << 28 | m1, (uint64_t)m1 << 40 | m0, ((uint64_t)m0 << 40) + 1))

// FP64 pipe: dependent-free DFMA chains
KERNEL(k_dfma, double, asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[j]) : "d"((double)m0), "d"((double)m1)))
// FP64 modular product of integers held in doubles (q < 2^50): h + l = x*w exactly,
// quotient by rint(h * qinv), remainder in (-2q, 2q)
__device__ __forceinline__ double fmodmul(double x, double w, double q, double qinv) {
    const double h = x * w;
    const double l = fma(x, w, -h);
    const double qt = rint(h * qinv);
    return fma(-qt, q, h) + l;
}
// same with the rounding by the 1.5 * 2^52 magic constant (no FRND)
__device__ __forceinline__ double fmodmul2(double x, double w, double q, double qinv) {
    const double h = x * w;
    const double l = fma(x, w, -h);
    const double qt = fma(h, qinv, 6755399441055744.0) - 6755399441055744.0;
    return fma(-qt, q, h) + l;
}
KERNEL(k_fmodmul2, double, a[j] = fmodmul2(a[j], (double)m0 * 1e6, 4398046511093.0, 1.0 / 4398046511093.0))
KERNEL(k_fbfly2, double, { double t = fmodmul2(a[(j + 1) % ACC], (double)m1 * 1e6, 4398046511093.0, 1.0 / 4398046511093.0); double x = a[j]; a[j] = x + t; a[(j + 1) % ACC] = x - t; })
KERNEL(k_fmodmul, double, a[j] = fmodmul(a[j], (double)m0 * 1e6, 4398046511093.0, 1.0 / 4398046511093.0))
// FP64 CT butterfly pair (X + T, X - T) on signed lazy values
KERNEL(k_fbfly, double, { double t = fmodmul(a[(j + 1) % ACC], (double)m1 * 1e6, 4398046511093.0, 1.0 / 4398046511093.0); double x = a[j]; a[j] = x + t; a[(j + 1) % ACC] = x - t; })
// integer Harvey CT butterfly pair for comparison
KERNEL(k_ibfly, uint64_t, { uint64_t q = ((uint64_t)m0 << 40) + 1; uint64_t X = a[j]; X = X >= 2 * q ? X - 2 * q : X; uint64_t T = shoup(a[(j + 1) % ACC], (uint64_t)m0 << 28 | m1, (uint64_t)m1 << 40 | m0, q); a[j] = X + T; a[(j + 1) % ACC] = X + 2 * q - T; })

int main() {
    int blocks = 148 * 8, threads = 256;
    uint64_t* out;
    cudaMalloc(&out, (size_t)blocks * threads * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int clk_khz;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    struct { const char* name; void (*launch)(uint64_t*); } ks[] = {
        {"IMAD.WIDE.U32", [](uint64_t* o) { k_wide<<<148 * 8, 256>>>(o, 3, 5); }},
        {"IMAD (lo)", [](uint64_t* o) { k_lo<<<148 * 8, 256>>>((uint32_t*)o, 3, 5); }},
        {"IMAD.HI", [](uint64_t* o) { k_hi<<<148 * 8, 256>>>((uint32_t*)o, 3, 5); }},
        {"IADD3", [](uint64_t* o) { k_add<<<148 * 8, 256>>>((uint32_t*)o, 3, 5); }},
        {"WIDE+IADD3", [](uint64_t* o) { k_mix<<<148 * 8, 256>>>(o, 3, 5); }},
        {"IMAD+IADD3", [](uint64_t* o) { k_mix2<<<148 * 8, 256>>>((uint32_t*)o, 3, 5); }},
        {"shoup (exact hi)", [](uint64_t* o) { k_shoup<<<148 * 8, 256>>>(o, 3, 5); }},
        {"shoup3 (approx hi)", [](uint64_t* o) { k_shoup3<<<148 * 8, 256>>>(o, 3, 5); }},
        {"DFMA", [](uint64_t* o) { k_dfma<<<148 * 8, 256>>>((double*)o, 3, 5); }},
        {"fp64 modmul", [](uint64_t* o) { k_fmodmul<<<148 * 8, 256>>>((double*)o, 3, 5); }},
        {"fp64 butterfly", [](uint64_t* o) { k_fbfly<<<148 * 8, 256>>>((double*)o, 3, 5); }},
        {"fp64 modmul (magic rint)", [](uint64_t* o) { k_fmodmul2<<<148 * 8, 256>>>((double*)o, 3, 5); }},
        {"fp64 butterfly (magic rint)", [](uint64_t* o) { k_fbfly2<<<148 * 8, 256>>>((double*)o, 3, 5); }},
        {"int butterfly", [](uint64_t* o) { k_ibfly<<<148 * 8, 256>>>(o, 3, 5); }},
        {"mul.lo.u64", [](uint64_t* o) { k_mul64<<<148 * 8, 256>>>(o, 3, 5); }},
        {"mul.hi.u64", [](uint64_t* o) { k_mulhi64<<<148 * 8, 256>>>(o, 3, 5); }},
    };
    for (auto& k : ks) {
        k.launch(out);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; r++) k.launch(out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = 5.0 * blocks * threads / 32.0 * ITER * ACC;   // warp-level ops
        double per_s = ops / (ms * 1e-3);
        printf("{\"op\": \"%s\", \"warp_ops_per_s\": %.4e, \"per_sm_per_clk_at_%d_mhz\": %.3f, \"ms\": %.3f}\n",
               k.name, per_s, clk_khz / 1000, per_s / 148 / (clk_khz * 1e3), ms);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
