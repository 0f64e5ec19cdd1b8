// dequantize.cu -- K4: unpacker + dequantiser ("During
// back-propagation, the activation is dequantized as h_hat = u_hat R/B + Z"),
// ACTNN-Q v1 step O10.  Mirrors K3's layout: a warp's unit is 4 consecutive
// groups of one sample; lane l reads the b bytes holding its 8 codes and
// writes its 8 consecutive outputs with one 256-bit (fp32) or 128-bit (bf16)
// store, so each warp store covers whole 32 B sectors.  The per-group (Z,
// scale) pairs are loaded lane-parallel and broadcast by shuffles.
#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

constexpr int kU = 4;
constexpr int kBlock = 256;
constexpr unsigned kFull = 0xffffffffu;

struct DParams {
    const uint8_t* packed;
    const float* zmin;
    const float* scale;
    const uint8_t* bits;
    const int64_t* off;
    int64_t N, D, ng, nb, units;
    uint64_t nb_magic;
    void* out;
};

__device__ __forceinline__ int64_t div_nb(int64_t u, int64_t nb, uint64_t magic) {
    if (nb == 1) return u;
    if ((uint64_t)u >> 32) return u / nb;
    return (int64_t)__umul64hi((uint64_t)u, magic);
}

// The b bytes of lane `lane` in a group segment, as a little-endian integer.
template <int b>
__device__ __forceinline__ uint64_t load_payload(const uint8_t* seg, int lane) {
    // volatile asm keeps each width's loads inside its own switch arm (ptxas
    // otherwise hoists all arms' loads and doubles the register footprint)
    if constexpr (b == 8) {
        uint32_t lo, hi;
        asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "l"(seg + lane * 8));
        return (uint64_t)lo | ((uint64_t)hi << 32);
    } else if constexpr (b == 4) {
        uint32_t v;
        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(seg + lane * 4));
        return v;
    } else if constexpr (b == 2) {
        uint16_t v;
        asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(seg + lane * 2));
        return v;
    } else if constexpr (b == 1) {
        uint32_t v;
        asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(seg + lane));
        return v;
    } else {
        uint64_t p = 0;
#pragma unroll
        for (int t = 0; t < b; ++t) {
            uint32_t v;
            asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(seg + lane * b + t));
            p |= (uint64_t)v << (8 * t);
        }
        return p;
    }
}

template <typename TO, int b>
__device__ __forceinline__ void dequant_unit(const uint8_t* seg, int gcount, float myZ,
                                             float mySc, TO* dst, int lane) {
    uint64_t pay[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
        if (u < gcount) pay[u] = load_payload<b>(seg + u * 32 * b, lane);
    constexpr uint32_t mask = (1u << b) - 1u;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        if (u < gcount) {
            const float Z = __shfl_sync(kFull, myZ, u);
            const float s = __shfl_sync(kFull, mySc, u);
            float o[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] = dequant1((uint32_t)(pay[u] >> (b * j)) & mask, s, Z);
            store8(dst + u * kG + lane * 8, o);
        }
    }
}

template <typename TO>
__global__ void __launch_bounds__(kBlock, 3) dequantize_fast_kernel(DParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    TO* __restrict__ out = static_cast<TO*>(p.out);
    const int64_t off0 = p.off[0];
    for (int64_t u = warp; u < p.units; u += nwarps) {
        const int64_t n = div_nb(u, p.nb, p.nb_magic);
        const int64_t gi = (u - n * p.nb) * kU;
        const int gcount = (int)min((int64_t)kU, p.ng - gi);
        const int b = p.bits[n];
        const uint8_t* seg = p.packed + (p.off[n] - off0) + gi * 32 * b;
        const int64_t g = n * p.ng + gi;
        TO* dst = out + n * p.D + gi * kG;
        float myZ = 0.0f, mySc = 0.0f;  // lane u holds group u's (Z, scale)
        if (lane < gcount) {
            myZ = __ldg(p.zmin + g + lane);
            mySc = __ldg(p.scale + g + lane);
        }
        // warp-uniform dispatch on the sample's width (an if-chain: a switch
        // becomes an indirect branch that ptxas allocates registers across)
        if (b == 2) dequant_unit<TO, 2>(seg, gcount, myZ, mySc, dst, lane);
        else if (b == 1) dequant_unit<TO, 1>(seg, gcount, myZ, mySc, dst, lane);
        else if (b == 4) dequant_unit<TO, 4>(seg, gcount, myZ, mySc, dst, lane);
        else if (b == 8) dequant_unit<TO, 8>(seg, gcount, myZ, mySc, dst, lane);
        else if (b == 3) dequant_unit<TO, 3>(seg, gcount, myZ, mySc, dst, lane);
        else if (b == 5) dequant_unit<TO, 5>(seg, gcount, myZ, mySc, dst, lane);
        else if (b == 6) dequant_unit<TO, 6>(seg, gcount, myZ, mySc, dst, lane);
        else if (b == 7) dequant_unit<TO, 7>(seg, gcount, myZ, mySc, dst, lane);
    }
}

// Generic path: ragged last group / unaligned output; one group per warp.
template <typename TO>
__global__ void __launch_bounds__(kBlock) dequantize_generic_kernel(DParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    TO* __restrict__ out = static_cast<TO*>(p.out);
    const int64_t off0 = p.off[0];
    const int64_t groups = p.N * p.ng;
    for (int64_t g = warp; g < groups; g += nwarps) {
        const int64_t n = g / p.ng;
        const int64_t i = g - n * p.ng;
        const int len = (int)min((int64_t)kG, p.D - i * kG);
        const int b = p.bits[n];
        if (b < 1 || b > 8) continue;
        const uint8_t* seg = p.packed + (p.off[n] - off0) + i * 32 * b;
        uint64_t pay = 0;
        for (int t = 0; t < b; ++t) pay |= (uint64_t)__ldg(seg + lane * b + t) << (8 * t);
        const float Z = __ldg(p.zmin + g);
        const float s = __ldg(p.scale + g);
        const uint32_t mask = (1u << b) - 1u;
        TO* dst = out + n * p.D + i * kG;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int idx = lane * 8 + j;
            if (idx < len) store1(dst + idx, dequant1((uint32_t)(pay >> (b * j)) & mask, s, Z));
        }
    }
}

template <typename TO>
cudaError_t run(const DequantArgs& a, cudaStream_t s) {
    DParams p;
    p.packed = a.packed;
    p.zmin = a.zmin;
    p.scale = a.scale;
    p.bits = a.bits;
    p.off = a.off;
    p.N = a.N;
    p.D = a.D;
    p.ng = a.ng;
    p.nb = (a.ng + kU - 1) / kU;
    p.units = a.N * p.nb;
    p.nb_magic = p.nb > 1 ? (uint64_t)(~0ull / (uint64_t)p.nb) + 1ull : 0ull;
    p.out = a.out;
    if (a.fast) {
        const int grid = grid_for((const void*)dequantize_fast_kernel<TO>, kBlock, 0,
                                  (p.units + 7) / 8);
        dequantize_fast_kernel<TO><<<grid, kBlock, 0, s>>>(p);
    } else {
        const int grid = grid_for((const void*)dequantize_generic_kernel<TO>, kBlock, 0,
                                  (a.N * a.ng + 7) / 8);
        dequantize_generic_kernel<TO><<<grid, kBlock, 0, s>>>(p);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dequantize(const DequantArgs& a, cudaStream_t s) {
    return a.out_dt == 0 ? run<float>(a, s) : run<uint16_t>(a, s);
}

}  // namespace actnn
