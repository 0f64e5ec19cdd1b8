// k3_mix.cu -- which instructions share a pipe with the Philox IMAD.WIDEs?
// Per-SMSP cycles per iteration of small instruction mixes (8 independent
// chains per thread, 16-48 warps per SM), and the K3 bf16 b=1 consumer body
// split into Philox alone / codes alone / both, to see whether the two
// instruction streams overlap.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false k3_mix.cu -o k3_mix
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2104_14129_b200/csrc/device.cuh"
using namespace actnn;

constexpr int CH = 8;

#define MIX(NAME, ...)                                                                  \
    __global__ void NAME(uint32_t iters, uint32_t seed, uint32_t* out) {                 \
        uint32_t a[CH], b[CH];                                                           \
        float f[CH], g[CH];                                                              \
        _Pragma("unroll") for (int i = 0; i < CH; ++i) {                                 \
            a[i] = threadIdx.x * 7919u + i * 104729u + seed;                             \
            b[i] = a[i] ^ 0x9E3779B9u;                                                   \
            f[i] = (float)(a[i] & 1023) * 0.37f;                                         \
            g[i] = (float)(b[i] & 511) * 0.11f;                                          \
        }                                                                                \
        for (uint32_t it = 0; it < iters; ++it) {                                        \
            _Pragma("unroll") for (int i = 0; i < CH; ++i) { __VA_ARGS__ }               \
        }                                                                                \
        uint32_t acc = 0;                                                                \
        _Pragma("unroll") for (int i = 0; i < CH; ++i) acc ^= a[i] ^ b[i] ^ __float_as_uint(f[i]) ^ __float_as_uint(g[i]); \
        if (acc == 0x1234567u) out[0] = acc;                                             \
    }

__device__ __forceinline__ void wide(uint32_t& a, uint32_t& b) {
    uint64_t p;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(0xD2511F53u));
    a = (uint32_t)p;
    b ^= (uint32_t)(p >> 32);
}
__device__ __forceinline__ void ffma_imm(float& f, float x) {
    asm volatile("fma.rn.f32 %0, %1, %2, 0f4B400000;" : "=f"(f) : "f"(f), "f"(x));
}
__device__ __forceinline__ void fhadd(float& f, uint32_t w) {
    asm volatile("{\n.reg .b16 lo, hi;\nmov.b32 {lo, hi}, %1;\nsub.rn.f32.bf16 %0, lo, %0;\n}" : "+f"(f) : "r"(w));
}
__device__ __forceinline__ void lop(uint32_t& a, uint32_t b) {
    asm volatile("lop3.b32 %0, %0, %1, 0x3fff3fff, 0x96;" : "+r"(a) : "r"(b));
}
__device__ __forceinline__ void iadd(uint32_t& a, uint32_t b) {
    asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b));
}

__device__ __forceinline__ void ffma2(float& f, float& g, float x) {
    float2 r = __ffma2_rn(make_float2(f, g), make_float2(x, x), make_float2(12582912.0f, 12582912.0f));
    f = r.x;
    g = r.y;
}
__device__ __forceinline__ void imadlo(uint32_t& a, uint32_t b) {
    asm volatile("mad.lo.u32 %0, %0, 0xD2511F53, %1;" : "+r"(a) : "r"(b));
}
__device__ __forceinline__ void imadhi(uint32_t& a, uint32_t b) {
    asm volatile("mul.hi.u32 %0, %0, 0xD2511F53;" : "+r"(a));
    a ^= b;
}
MIX(m_wide, wide(a[i], b[i]);)
MIX(m_ffma2, ffma2(f[i], g[i], 1.0001f);)
MIX(m_wide_ffma2, wide(a[i], b[i]); ffma2(f[i], g[i], 1.0001f);)
MIX(m_imadlo, imadlo(a[i], b[i]);)
MIX(m_imadhi, imadhi(a[i], b[i]);)
MIX(m_wide_lop1, wide(a[i], b[i]); lop(b[i], a[i]);)
__device__ __forceinline__ void hilo(uint32_t& a, uint32_t& b) {  // IMAD.HI + IMAD instead of IMAD.WIDE
    uint32_t h, l;
    asm volatile("mul.hi.u32 %0, %1, 0xD2511F53;" : "=r"(h) : "r"(a));
    asm volatile("mul.lo.u32 %0, %1, 0xD2511F53;" : "=r"(l) : "r"(a));
    a = l;
    b ^= h;
}
__device__ __forceinline__ void hionly(uint32_t& a) {
    asm volatile("mul.hi.u32 %0, %0, 0xD2511F53;" : "+r"(a));
}
MIX(m_hilo, hilo(a[i], b[i]);)
MIX(m_hilo_lop, hilo(a[i], b[i]); lop(b[i], a[i]);)
MIX(m_hionly, hionly(a[i]);)
MIX(m_hionly_lop, hionly(a[i]); lop(b[i], a[i]);)
MIX(m_imadlo_lop, imadlo(a[i], b[i]); lop(b[i], a[i]);)
MIX(m_wide_2ffma_lop, wide(a[i], b[i]); ffma_imm(f[i], g[i]); ffma_imm(g[i], f[i]); lop(b[i], a[i]);)
MIX(m_lop, lop(a[i], b[i]);)
MIX(m_ffma, ffma_imm(f[i], g[i]);)
MIX(m_fhadd, fhadd(f[i], a[i]);)
MIX(m_iadd, iadd(a[i], b[i]);)
MIX(m_wide_lop2, wide(a[i], b[i]); lop(b[i], a[i]); lop(a[i], b[i]);)
MIX(m_wide_ffma, wide(a[i], b[i]); ffma_imm(f[i], g[i]);)
MIX(m_wide_ffma2x, wide(a[i], b[i]); ffma_imm(f[i], g[i]); ffma_imm(g[i], f[i]);)
MIX(m_wide_fhadd, wide(a[i], b[i]); fhadd(f[i], b[i]);)
MIX(m_wide_iadd, wide(a[i], b[i]); iadd(b[i], a[i]);)
MIX(m_lop_ffma, lop(a[i], b[i]); ffma_imm(f[i], g[i]);)
MIX(m_lop_fhadd, lop(a[i], b[i]); fhadd(f[i], b[i]);)

// warp-specialised mix: even warps run an IMAD.WIDE stream, odd warps an ALU + FP
// stream (LOP3 + 2 FFMA) -- do the two overlap when they come from different warps?
__global__ void m_split(uint32_t iters, uint32_t seed, uint32_t* out) {
    uint32_t a[CH], b[CH];
    float f[CH], g[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        a[i] = threadIdx.x * 7919u + i * 104729u + seed;
        b[i] = a[i] ^ 0x9E3779B9u;
        f[i] = (float)(a[i] & 1023) * 0.37f;
        g[i] = (float)(b[i] & 511) * 0.11f;
    }
    if ((threadIdx.x >> 5) & 1) {
        for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < CH; ++i) { lop(a[i], b[i]); ffma_imm(f[i], g[i]); ffma_imm(g[i], f[i]); }
        }
    } else {
        for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < CH; ++i) { wide(a[i], b[i]); }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) acc ^= a[i] ^ b[i] ^ __float_as_uint(f[i]) ^ __float_as_uint(g[i]);
    if (acc == 0x1234567u) out[0] = acc;
}
MIX(m_lop_2ffma, lop(a[i], b[i]); ffma_imm(f[i], g[i]); ffma_imm(g[i], f[i]);)

// ---- the K3 bf16 b = 1 consumer body (one group per lane-iteration)
struct P {
    RoundKeys rk;
};

// Philox4x32-10 with a zero counter high word whose round-0 product M0 * ctr
// is given as (hi, lo) (e.g. a uniform part plus a per-lane constant).
__device__ __forceinline__ Philox4 philox_r0(uint32_t hi0, uint32_t lo0, const RoundKeys& rk) {
    uint32_t hi1, lo1, ahi, alo;
    const uint32_t x2 = hi0 ^ rk.k[1], x3 = lo0;
    mulwide(rk.k[0], 0xD2511F53u, ahi, alo);
    mulwide(x2, 0xCD9E8D57u, hi1, lo1);
    uint32_t a0 = hi1 ^ rk.k[2], a1 = lo1, a2 = ahi ^ x3 ^ rk.k[3], a3 = alo;
#pragma unroll
    for (int r = 2; r < 10; ++r) {
        uint32_t h0, l0;
        mulwide(a0, 0xD2511F53u, h0, l0);
        mulwide(a2, 0xCD9E8D57u, hi1, lo1);
        const uint32_t n0 = hi1 ^ a1 ^ rk.k[2 * r];
        const uint32_t n2 = h0 ^ a3 ^ rk.k[2 * r + 1];
        a0 = n0; a1 = lo1; a2 = n2; a3 = l0;
    }
    return Philox4{a0, a1, a2, a3};
}

// b = 1 codes with the f32x2 FFMA2 for the magic fma (pairs of elements)
__device__ __forceinline__ uint32_t codes_b1_x2(const uint4& raw, float Z, float inv14, const Philox4& o) {
    float d[8];
    deltas8(raw, Z, d);
    const uint32_t w[4] = {o.x, o.y, o.z, o.w};
    const float2 iv = make_float2(inv14, inv14), mg = make_float2(12582912.0f, 12582912.0f);
    uint32_t y = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float2 t = __ffma2_rn(make_float2(d[2 * q], d[2 * q + 1]), iv, mg);
        uint32_t tx, ty;
        asm("mov.b32 %0, %1;" : "=r"(tx) : "f"(t.x));
        asm("mov.b32 %0, %1;" : "=r"(ty) : "f"(t.y));
        uint32_t T = __byte_perm(tx, ty, 0x5410);
        T += w[q] & 0x3FFF3FFFu;
        y |= (T >> (14 - 2 * q)) & (0x40004000u >> (14 - 2 * q));
    }
    return (y | (y >> 15)) & 0xFFu;
}

template <int MODE, int VAR = 0>  // MODE 0 full, 1 Philox only, 2 codes only; VAR bit0 r0-linear, bit1 FFMA2
__global__ void body_b1(const __grid_constant__ P p, uint32_t groups, uint8_t* out) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint4 raw = make_uint4(0x3f803fa0u + lane, 0x40003f00u + lane, 0x3e803ec0u, 0x3fc03f10u);
    const float Z = -1.0f, inv = 2500.0f * 16384.0f;
    uint32_t blk = gw * groups * 32 + lane;
    uint8_t* seg = out + (size_t)gw * 32;
    uint32_t acc = 0;
    for (uint32_t g = 0; g < groups; g += 2) {
        Philox4 o0, o1;
        if (MODE != 2 && (VAR & 1)) {
            // M0 * blk = M0 * (blk - lane) (warp-uniform) + M0 * lane (per-thread constant)
            const uint64_t u = (uint64_t)(blk - lane) * 0xD2511F53u;
            const uint64_t pl = (uint64_t)lane * 0xD2511F53u;
            const uint64_t a = u + pl, c = a + (uint64_t)32 * 0xD2511F53u;
            o0 = philox_r0((uint32_t)(a >> 32), (uint32_t)a, p.rk);
            o1 = philox_r0((uint32_t)(c >> 32), (uint32_t)c, p.rk);
        } else if (MODE != 2) {
            o0 = philox4x32_10_c32(blk, p.rk);
            o1 = philox4x32_10_c32(blk + 32, p.rk);
        } else {
            o0 = Philox4{blk, blk * 3u, blk ^ 0x55u, blk + 7u};
            o1 = Philox4{blk ^ 9u, blk * 5u, blk ^ 0x33u, blk + 9u};
        }
        if (MODE == 1) {
            acc ^= o0.x ^ o0.y ^ o0.z ^ o0.w ^ o1.x ^ o1.y ^ o1.z ^ o1.w;
        } else {
            if (VAR & 2) {
                seg[lane] = (uint8_t)codes_b1_x2(raw, Z, inv, o0);
                seg[lane + 32] = (uint8_t)codes_b1_x2(raw, Z, inv, o1);
            } else {
                seg[lane] = (uint8_t)codes_small<1>(raw, Z, inv, o0);
                seg[lane + 32] = (uint8_t)codes_small<1>(raw, Z, inv, o1);
            }
            raw.x += 0x10001u;
        }
        blk += 64;
    }
    if (acc == 0x9u) out[0] = (uint8_t)acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 1 << 28);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint32_t iters = 4096;
    int clk_khz;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    for (int wps : {16, 32, 48}) {
        const int threads = 256, blocks = sms * wps / 8;
        float ms;
        // cycles per (iteration x chain) per SMSP: warps per SMSP x iters x CH instr groups
        const double its = (double)blocks * (threads / 32) * iters * CH / (sms * 4.0);
#define T(K)                                                                            \
    K<<<blocks, threads>>>(iters, 1, out);                                              \
    cudaEventRecord(e0);                                                                \
    K<<<blocks, threads>>>(iters, 1, out);                                              \
    cudaEventRecord(e1);                                                                \
    cudaEventSynchronize(e1);                                                           \
    cudaEventElapsedTime(&ms, e0, e1);                                                  \
    printf("%-16s warps/SM=%2d: %.2f SMSP-cycles per warp-iteration\n", #K, wps,        \
           ms * 1e-3 * 1.965e9 / its);
        T(m_wide) T(m_lop) T(m_ffma) T(m_fhadd) T(m_iadd) T(m_wide_lop2) T(m_wide_ffma)
        T(m_wide_ffma2x) T(m_wide_fhadd) T(m_wide_iadd) T(m_lop_ffma) T(m_lop_fhadd)
        T(m_ffma2) T(m_wide_ffma2) T(m_imadlo) T(m_imadhi) T(m_wide_lop1)
        T(m_hilo) T(m_hilo_lop) T(m_hionly) T(m_hionly_lop) T(m_imadlo_lop) T(m_wide_2ffma_lop)
        T(m_lop_2ffma) T(m_split)
        P pp;
        pp.rk = make_round_keys(42);
        const uint32_t groups = 512;
        const double gps = (double)blocks * (threads / 32) * groups / (sms * 4.0);
#define B(MODE, NAME, ...)                                                              \
    body_b1<MODE, ##__VA_ARGS__><<<blocks, threads>>>(pp, groups, (uint8_t*)out);        \
    cudaEventRecord(e0);                                                                \
    body_b1<MODE, ##__VA_ARGS__><<<blocks, threads>>>(pp, groups, (uint8_t*)out);        \
    cudaEventRecord(e1);                                                                \
    cudaEventSynchronize(e1);                                                           \
    cudaEventElapsedTime(&ms, e0, e1);                                                  \
    printf("%-16s warps/SM=%2d: %.1f SMSP-cycles per group\n", NAME, wps, ms * 1e-3 * 1.965e9 / gps);
        B(0, "b1 full") B(1, "b1 philox only") B(2, "b1 codes only")
        B(0, "b1 full r0", 1) B(1, "b1 philox r0", 1) B(0, "b1 full ffma2", 2) B(2, "b1 codes ffma2", 2)
        B(0, "b1 full r0+ffma2", 3)
    }
    printf("%s (clock attr %d kHz)\n", cudaGetErrorString(cudaGetLastError()), clk_khz);
    return 0;
}
