// pipe_rate.cu -- issue throughput of the integer/FP instructions Philox and
// the SR code path use, on one B200 (thread-ops per clock per SM at the
// measured SM clock).  Guides the K3 instruction mix: which of
// IMAD.WIDE / IMAD.HI / IMAD / LOP3 / IADD3 / FFMA / FFMA2 / PRMT are full rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8;  // independent chains per thread

#define KERNEL(NAME, ...)                                                            \
    __global__ void NAME(uint32_t iters, uint32_t seed, uint32_t* out) {              \
        uint32_t a[CH], b[CH];                                                        \
        _Pragma("unroll") for (int i = 0; i < CH; ++i) {                              \
            a[i] = threadIdx.x * 7919u + i * 104729u + seed;                          \
            b[i] = a[i] ^ 0x9E3779B9u;                                                \
        }                                                                             \
        for (uint32_t it = 0; it < iters; ++it) {                                     \
            _Pragma("unroll") for (int i = 0; i < CH; ++i) { __VA_ARGS__ }                   \
        }                                                                             \
        uint32_t acc = 0;                                                             \
        _Pragma("unroll") for (int i = 0; i < CH; ++i) acc ^= a[i] ^ b[i];            \
        if (acc == 0x1234567u) out[0] = acc;                                          \
    }

// 64-bit product: IMAD.WIDE.U32 (lo in a, hi in b)
KERNEL(k_wide, {
    uint64_t p;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a[i]), "r"(0xD2511F53u));
    a[i] = (uint32_t)p ^ b[i];
    b[i] = (uint32_t)(p >> 32);
})
// hi only: IMAD.HI.U32 (+ xor)
KERNEL(k_hi, {
    uint32_t h;
    asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h) : "r"(a[i]), "r"(0xD2511F53u));
    a[i] = h ^ b[i];
})
// lo only: IMAD (+ xor)
KERNEL(k_lo, {
    uint32_t h;
    asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(h) : "r"(a[i]), "r"(0xD2511F53u));
    a[i] = h ^ b[i];
})
// xor only: LOP3
KERNEL(k_lop, {
    uint32_t h;
    asm volatile("xor.b32 %0, %1, %2;" : "=r"(h) : "r"(a[i]), "r"(b[i]));
    a[i] = h ^ 0x5bd1e995u;
})
// add: IADD3
KERNEL(k_add, {
    uint32_t h;
    asm volatile("add.u32 %0, %1, %2;" : "=r"(h) : "r"(a[i]), "r"(b[i]));
    a[i] = h;
})
// fp32 fma
KERNEL(k_ffma, {
    float f;
    asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(f) : "f"(__uint_as_float(a[i])), "f"(1.0001f), "f"(__uint_as_float(b[i])));
    a[i] = __float_as_uint(f);
})
// prmt
KERNEL(k_prmt, {
    uint32_t h;
    asm volatile("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(h) : "r"(a[i]), "r"(b[i]));
    a[i] = h;
})
// hi + lo as two instructions
KERNEL(k_hilo, {
    uint32_t h, l;
    asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h) : "r"(a[i]), "r"(0xD2511F53u));
    asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(l) : "r"(a[i]), "r"(0xD2511F53u));
    a[i] = h ^ b[i];
    b[i] = l;
})


// heavy-pipe interference: one IMAD.WIDE chain step plus FP work per iteration
KERNEL(k_wide_ffma2, {
    uint64_t p;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a[i]), "r"(0xD2511F53u));
    float2 f = make_float2(__uint_as_float(b[i]), __uint_as_float(a[i]));
    float2 g;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*(uint64_t*)&g) : "l"(*(uint64_t*)&f), "l"(*(uint64_t*)&f), "l"(*(uint64_t*)&f));
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*(uint64_t*)&f) : "l"(*(uint64_t*)&g), "l"(*(uint64_t*)&g), "l"(*(uint64_t*)&g));
    a[i] = (uint32_t)p ^ __float_as_uint(f.x);
    b[i] = (uint32_t)(p >> 32) ^ __float_as_uint(f.y);
})
KERNEL(k_wide_ffma4, {
    uint64_t p;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a[i]), "r"(0xD2511F53u));
    float x = __uint_as_float(b[i]), y = __uint_as_float(a[i]);
    asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x));
    asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(y));
    asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x));
    asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(y));
    a[i] = (uint32_t)p ^ __float_as_uint(x);
    b[i] = (uint32_t)(p >> 32) ^ __float_as_uint(y);
})
KERNEL(k_wide_only, {
    uint64_t p;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a[i]), "r"(0xD2511F53u));
    a[i] = (uint32_t)p ^ b[i];
    b[i] = (uint32_t)(p >> 32) ^ 0x1234u;
})
KERNEL(k_ffma2_only, {
    float2 f = make_float2(__uint_as_float(b[i]), __uint_as_float(a[i]));
    asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(*(uint64_t*)&f));
    a[i] = __float_as_uint(f.x);
    b[i] = __float_as_uint(f.y);
})
KERNEL(k_wide_prmt4, {
    uint64_t p;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a[i]), "r"(0xD2511F53u));
    uint32_t x = b[i], y = a[i];
    asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(x) : "r"(y));
    asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(y) : "r"(x));
    asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(x) : "r"(y));
    asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(y) : "r"(x));
    a[i] = (uint32_t)p ^ x;
    b[i] = (uint32_t)(p >> 32) ^ y;
})

typedef void (*KFn)(uint32_t, uint32_t, uint32_t*);

int main() {
    int sms, clk_khz;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    uint32_t* out;
    cudaMalloc(&out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct { const char* name; KFn f; int ops; } ks[] = {
        {"mul.wide (IMAD.WIDE) +xor", k_wide, 2}, {"mul.hi (IMAD.HI) +xor", k_hi, 2},
        {"mul.lo (IMAD) +xor", k_lo, 2},          {"xor (LOP3) x2", k_lop, 2},
        {"add (IADD3)", k_add, 1},                {"fma.f32 (FFMA)", k_ffma, 1},
        {"prmt", k_prmt, 1},                      {"mul.hi+mul.lo +xor", k_hilo, 3},
        {"wide+xor2 only", k_wide_only, 3},       {"wide + 2 FFMA2", k_wide_ffma2, 5},
        {"wide + 4 FFMA", k_wide_ffma4, 7},       {"FFMA2 only", k_ffma2_only, 1},
        {"wide + 4 PRMT", k_wide_prmt4, 7},
    };
    const uint32_t iters = 4096;
    for (auto& k : ks) {
        for (int wps : {32, 64}) {
            const int threads = 256, blocks = sms * wps / 8;
            k.f<<<blocks, threads>>>(iters, 1, out);
            cudaEventRecord(e0);
            k.f<<<blocks, threads>>>(iters, 2, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double insts = (double)blocks * threads * iters * CH;  // body iterations
            const double per_clk_sm = insts / (ms * 1e-3) / sms / (clk_khz * 1e3);
            printf("%-28s warps/SM=%2d: %.1f body-iters/clk/SM (%d instr each) at %d MHz nominal\n",
                   k.name, wps, per_clk_sm, k.ops, clk_khz / 1000);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
