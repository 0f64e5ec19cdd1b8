// quantize.cu -- K3: per-group stochastic-rounding quantiser + bit packer
// (P:491-503 per-group quantisation, "compress them into bit
// streams"), ACTNN-Q v1 steps O1-O9.
//
// Work decomposition (fast path, D % 256 == 0): a warp's unit is U = 4
// consecutive groups of one sample (4 KB of fp32 input).  Each lane owns 8
// consecutive elements of every group: one 256-bit load (fp32) or one 128-bit
// load (bf16) per group, one Philox4x32-10 call per group (8 x 16 random
// bits), and b contiguous bytes of the packed group segment.  The U loads are
// issued before any arithmetic so each warp keeps 4 KB in flight.
//   - group min/max: 8-element local min/max then a 5-step xor shuffle;
//   - per-group constants (two IEEE divisions) are computed lane-parallel, lane
//     u for group u of the unit, then broadcast with one shuffle each;
//   - packing: b = 8 / 4 lanes store their 8 / 4 bytes directly (256 / 128 B
//     per warp); b = 2 / 1 pair / quad lanes with shuffles so every store is a
//     32-bit word and the warp writes whole 32 B sectors (64 / 32 B per group).
// Ragged D or unaligned x take the generic kernel (scalar loads, one group per
// warp iteration); it computes exactly the same bytes.
#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

constexpr int kU = 4;
constexpr int kBlock = 256;
constexpr unsigned kFull = 0xffffffffu;

struct QParams {
    const void* x;
    int64_t N, D, ng, nb, units;
    uint64_t nb_magic;  // ceil(2^64 / nb) (nb >= 2) for the unit -> sample division
    const uint8_t* bits;
    const int64_t* off;
    uint32_t k0, k1;
    int64_t sample_base;
    const float* gmin;
    const float* gmax;
    uint8_t* packed;
    float* zmin;
    float* scale;
};

// floor(u / nb) for u < 2^32, nb < 2^32 (one 64-bit mulhi).
__device__ __forceinline__ int64_t div_nb(int64_t u, int64_t nb, uint64_t magic) {
    if (nb == 1) return u;
    if ((uint64_t)u >> 32) return u / nb;
    return (int64_t)__umul64hi((uint64_t)u, magic);
}

// LSB-first packing of a lane's 8 codes (ACTNN-Q v1 O8): code k of
// the group sits at stream bits [k b, (k+1) b), so lane l's codes fill bytes
// [l b, (l+1) b) of the group's 32 b-byte segment.
template <int b>
__device__ __forceinline__ void pack_store(uint8_t* seg, const uint32_t code[8], int lane) {
    if constexpr (b == 8) {
        const uint32_t lo = code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
        const uint32_t hi = code[4] | (code[5] << 8) | (code[6] << 16) | (code[7] << 24);
        *reinterpret_cast<uint2*>(seg + lane * 8) = make_uint2(lo, hi);
    } else if constexpr (b == 4) {
        uint32_t p = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) p |= code[j] << (4 * j);
        *reinterpret_cast<uint32_t*>(seg + lane * 4) = p;
    } else if constexpr (b == 2) {
        uint32_t p = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) p |= code[j] << (2 * j);
        const uint32_t q = __shfl_down_sync(kFull, p, 1);
        if (!(lane & 1)) *reinterpret_cast<uint32_t*>(seg + lane * 2) = p | (q << 16);
    } else if constexpr (b == 1) {
        uint32_t p = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) p |= code[j] << j;
        const uint32_t q1 = __shfl_down_sync(kFull, p, 1);
        const uint32_t q2 = __shfl_down_sync(kFull, p, 2);
        const uint32_t q3 = __shfl_down_sync(kFull, p, 3);
        if (!(lane & 3))
            *reinterpret_cast<uint32_t*>(seg + lane) = p | (q1 << 8) | (q2 << 16) | (q3 << 24);
    } else {  // b in {3, 5, 6, 7}: b bytes per lane, not word aligned
        uint64_t p = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) p |= (uint64_t)code[j] << (b * j);
#pragma unroll
        for (int t = 0; t < b; ++t) seg[lane * b + t] = (uint8_t)(p >> (8 * t));
    }
}

// One group: Philox draw for the lane's 8-element block, SR codes, pack.
template <int b>
__device__ __forceinline__ void quant_group(const float v[8], float Z, float inv14, uint64_t blk,
                                            uint32_t k0, uint32_t k1, uint8_t* seg, int lane) {
    const Philox4 o = philox4x32_10((uint32_t)blk, (uint32_t)(blk >> 32), k0, k1);
    uint32_t code[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) code[j] = sr_code(v[j], Z, inv14, rnd14(o, j));
    pack_store<b>(seg, code, lane);
}

// Width-dependent tail of a unit: lane-parallel group constants (lane u owns
// group u of the unit), then codes + packing for each group.
template <int b>
__device__ __forceinline__ void quant_unit(const float (&v)[kU][8], int gcount, float myMn,
                                           float myMx, float* zm, float* sc, uint8_t* seg,
                                           uint64_t blk0, uint32_t k0, uint32_t k1, int lane) {
    const GroupConst cc = group_const(myMn, myMx, b);
    if (lane < gcount) {
        zm[lane] = cc.Z;
        sc[lane] = cc.scale;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        if (u < gcount) {
            const float Z = __shfl_sync(kFull, cc.Z, u);
            const float inv = __shfl_sync(kFull, cc.inv14, u);
            quant_group<b>(v[u], Z, inv, blk0 + (uint64_t)(u * 32 + lane), k0, k1,
                           seg + u * 32 * b, lane);
        }
    }
}

template <typename T, bool kStats>
__global__ void __launch_bounds__(kBlock, 3) quantize_fast_kernel(QParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const T* __restrict__ x = static_cast<const T*>(p.x);
    const int64_t off0 = p.off[0];
    for (int64_t u = warp; u < p.units; u += nwarps) {
        const int64_t n = div_nb(u, p.nb, p.nb_magic);
        const int64_t gi = (u - n * p.nb) * kU;  // first group of the unit within sample n
        const int gcount = (int)min((int64_t)kU, p.ng - gi);
        const int b = p.bits[n];
        const T* src = x + n * p.D + gi * kG;
        const int64_t g = n * p.ng + gi;
        uint8_t* seg = p.packed + (p.off[n] - off0) + gi * 32 * b;
        const uint64_t blk0 = ((uint64_t)(p.sample_base + n) * (uint64_t)p.D + (uint64_t)(gi * kG)) >> 3;
        // issue the unit's loads first: 4 groups (4 KB fp32) in flight per warp
        float v[kU][8];
#pragma unroll
        for (int k = 0; k < kU; ++k)
            if (k < gcount) load8(src + k * kG + lane * 8, v[k]);
        float myMn = 0.0f, myMx = 0.0f;
        if constexpr (kStats) {
#pragma unroll
            for (int k = 0; k < kU; ++k) {
                if (k < gcount) {
                    float mn = v[k][0], mx = v[k][0];
#pragma unroll
                    for (int j = 1; j < 8; ++j) {
                        mn = fminf(mn, v[k][j]);
                        mx = fmaxf(mx, v[k][j]);
                    }
                    mn = warp_min(mn);
                    mx = warp_max(mx);
                    if (lane == k) {
                        myMn = mn;
                        myMx = mx;
                    }
                }
            }
        } else {
            if (lane < gcount) {
                myMn = __ldg(p.gmin + g + lane);
                myMx = __ldg(p.gmax + g + lane);
            }
        }
        float* zm = p.zmin + g;
        float* sc = p.scale + g;
        switch (b) {
            case 1: quant_unit<1>(v, gcount, myMn, myMx, zm, sc, seg, blk0, p.k0, p.k1, lane); break;
            case 2: quant_unit<2>(v, gcount, myMn, myMx, zm, sc, seg, blk0, p.k0, p.k1, lane); break;
            case 4: quant_unit<4>(v, gcount, myMn, myMx, zm, sc, seg, blk0, p.k0, p.k1, lane); break;
            case 8: quant_unit<8>(v, gcount, myMn, myMx, zm, sc, seg, blk0, p.k0, p.k1, lane); break;
            case 3: quant_unit<3>(v, gcount, myMn, myMx, zm, sc, seg, blk0, p.k0, p.k1, lane); break;
            case 5: quant_unit<5>(v, gcount, myMn, myMx, zm, sc, seg, blk0, p.k0, p.k1, lane); break;
            case 6: quant_unit<6>(v, gcount, myMn, myMx, zm, sc, seg, blk0, p.k0, p.k1, lane); break;
            case 7: quant_unit<7>(v, gcount, myMn, myMx, zm, sc, seg, blk0, p.k0, p.k1, lane); break;
            default: break;  // invalid width: outside the contract (ACTNN_CHECK=1 reports it)
        }
    }
}

// Generic path: any D (ragged last group), any element alignment.  One group
// per warp iteration; lane l holds elements [8l, 8l+8) of the group, masked
// past the group's real length; the Philox block of element e is e >> 3, so
// a lane needs at most two blocks when D % 8 != 0.
template <typename T, bool kStats>
__global__ void __launch_bounds__(kBlock) quantize_generic_kernel(QParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const T* __restrict__ x = static_cast<const T*>(p.x);
    const int64_t off0 = p.off[0];
    const int64_t groups = p.N * p.ng;
    for (int64_t g = warp; g < groups; g += nwarps) {
        const int64_t n = g / p.ng;
        const int64_t i = g - n * p.ng;
        const int len = (int)min((int64_t)kG, p.D - i * kG);
        const int b = p.bits[n];
        if (b < 1 || b > 8) continue;
        const T* src = x + n * p.D + i * kG;
        float v[8];
        float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int idx = lane * 8 + j;
            v[j] = idx < len ? load1(src + idx) : 0.0f;
            if (idx < len) {
                mn = fminf(mn, v[j]);
                mx = fmaxf(mx, v[j]);
            }
        }
        if (kStats) {
            mn = warp_min(mn);
            mx = warp_max(mx);
        } else {
            mn = __ldg(p.gmin + g);
            mx = __ldg(p.gmax + g);
        }
        const GroupConst cc = group_const(mn, mx, b);
        if (lane == 0) {
            p.zmin[g] = cc.Z;
            p.scale[g] = cc.scale;
        }
        const uint64_t e_first =
            (uint64_t)(p.sample_base + n) * (uint64_t)p.D + (uint64_t)(i * kG + lane * 8);
        const uint64_t blkA = e_first >> 3;
        const Philox4 oA = philox4x32_10((uint32_t)blkA, (uint32_t)(blkA >> 32), p.k0, p.k1);
        const uint64_t blkB = blkA + 1;
        const Philox4 oB = philox4x32_10((uint32_t)blkB, (uint32_t)(blkB >> 32), p.k0, p.k1);
        uint64_t pk = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int idx = lane * 8 + j;
            const uint64_t e = e_first + j;
            const uint32_t r = ((e >> 3) == blkA) ? rnd14(oA, (int)(e & 7)) : rnd14(oB, (int)(e & 7));
            const uint32_t code = idx < len ? sr_code(v[j], cc.Z, cc.inv14, r) : 0u;
            pk |= (uint64_t)code << (b * j);
        }
        uint8_t* seg = p.packed + (p.off[n] - off0) + i * 32 * b;
        for (int t = 0; t < b; ++t) seg[lane * b + t] = (uint8_t)(pk >> (8 * t));
    }
}

template <typename T, bool kStats>
cudaError_t run(const QuantArgs& a, cudaStream_t s) {
    QParams p;
    p.x = a.x;
    p.N = a.N;
    p.D = a.D;
    p.ng = a.ng;
    p.nb = (a.ng + kU - 1) / kU;
    p.units = a.N * p.nb;
    p.nb_magic = p.nb > 1 ? (uint64_t)(~0ull / (uint64_t)p.nb) + 1ull : 0ull;
    p.bits = a.bits;
    p.off = a.off;
    p.k0 = (uint32_t)a.seed;
    p.k1 = (uint32_t)(a.seed >> 32);
    p.sample_base = a.sample_base;
    p.gmin = a.gmin;
    p.gmax = a.gmax;
    p.packed = a.packed;
    p.zmin = a.zmin;
    p.scale = a.scale;
    if (a.fast) {
        const void* k = (const void*)quantize_fast_kernel<T, kStats>;
        const int grid = grid_for(k, kBlock, 0, (p.units + 7) / 8);
        quantize_fast_kernel<T, kStats><<<grid, kBlock, 0, s>>>(p);
    } else {
        const void* k = (const void*)quantize_generic_kernel<T, kStats>;
        const int grid = grid_for(k, kBlock, 0, (a.N * a.ng + 7) / 8);
        quantize_generic_kernel<T, kStats><<<grid, kBlock, 0, s>>>(p);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t s) {
    const bool stats = (a.gmin == nullptr);
    if (a.dt == 0) return stats ? run<float, true>(a, s) : run<float, false>(a, s);
    return stats ? run<uint16_t, true>(a, s) : run<uint16_t, false>(a, s);
}

}  // namespace actnn
