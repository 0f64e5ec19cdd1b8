// stats.cu -- K1 group_stats (with K1b sens_reduce fused): pass 1 of the mixed-precision
// path.  Per group the canonical min Z and max M; per sample the
// range norm S_n = ||R_n||^2 (the ||R_n||^2 factor of w_n in Eq. 7),
// summed in ACTNN-Q v1's canonical order O11 so that the allocator sees the
// same fp64 values as the oracle:
//   K1: a CTA (8 warps) owns one chunk of 32 groups of one sample; warp w
//       reduces groups 4w..4w+3 (one 256-bit load per lane per group, 4 groups
//       in flight), the 32 (Z, M) pairs meet in shared memory, and warp 0
//       writes them coalesced and runs the fp64 xor butterfly over
//       v_l = R_l^2 (lane l = group l; zero past the sample's last group):
//       T_{n,c} = v_0 after v_l <- v_l + v_{l^o}, o = 16, 8, 4, 2, 1.
//   K1b: S_n = ((0 + T_{n,0}) + T_{n,1}) + ... in chunk order, run by the
//       last CTA to finish (an atomicInc ticket in the workspace that wraps
//       back to 0, so no reset launch is needed) -- one launch per tensor.
#include <cstdlib>

#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

// groups per warp per chunk: 4 (fp32: 4 KB in flight per warp) or 8 (bf16:
// also 4 KB); a CTA has 32 / U warps so that a chunk is 32 groups.
#ifndef ACTNN_K1_CTAS_PER_SM
#define ACTNN_K1_CTAS_PER_SM -1  // -1: 4 per SM at fp32, the occupancy limit at bf16
#endif
#ifndef ACTNN_K1_PREFETCH
#define ACTNN_K1_PREFETCH 0  // 1: next tile in flight; measured slower (74 registers, 3 CTAs/SM)
#endif
#ifndef ACTNN_K1_U32
#define ACTNN_K1_U32 4
#endif
#ifndef ACTNN_K1_U16
#define ACTNN_K1_U16 4
#endif
template <typename T>
struct SCfg {
    // groups per warp: 4 (4 KB fp32 / 2 KB bf16 in flight); 8 bf16 groups per
    // warp measured 8% slower on the largest C4 tensor (fewer CTAs per SM)
    static constexpr int U = sizeof(T) == 2 ? ACTNN_K1_U16 : ACTNN_K1_U32;
    static constexpr int Block = (kChunk / U) * 32;
};
constexpr unsigned kFull = 0xffffffffu;

struct SParams {
    const void* x;
    int64_t N, D, ng, nch;
    float* gmin;
    float* gmax;
    double* T;
    double* sens;
    unsigned int* ticket;  // zero before the first call; left zero by every call
};

__device__ __forceinline__ uint4 ldg_nc_u4(const uint16_t* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}


template <typename T, bool kFast>
__global__ void __launch_bounds__(SCfg<T>::Block) group_stats_kernel(SParams p) {
    pdl_trigger();  // the next kernel of the stream may start launching
    pdl_wait();     // the previous grid is complete and visible
    constexpr int kU = SCfg<T>::U;
    constexpr int kBlock = SCfg<T>::Block;
    __shared__ float sZ[kChunk], sM[kChunk];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const T* __restrict__ x = static_cast<const T*>(p.x);
    const int64_t tiles = p.N * p.nch;
    const int gw = w * kU;  // this warp's first group within a chunk
    // fast path: the warp's words of the CTA's next tile are loaded before this
    // tile is reduced (ACTNN_K1_PREFETCH), hiding one load latency per tile
    uint4 cur[kU][2], nxt[kU][2];
    auto load_tile = [&](int64_t t, uint4 (&q)[kU][2]) {
        const int64_t n = t / p.nch;
        const int64_t g0 = (t - n * p.nch) * kChunk;
        const int gcount = (int)min((int64_t)kChunk, p.ng - g0);
        const T* src = x + n * p.D + (g0 + gw) * kG + lane * 8;
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (gw + u < gcount) ldg_raw8(src + u * kG, q[u]);
    };
    if (kFast && ACTNN_K1_PREFETCH && (int64_t)blockIdx.x < tiles) load_tile(blockIdx.x, cur);
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t n = t / p.nch;
        const int64_t c = t - n * p.nch;
        const int64_t g0 = c * kChunk;
        const int gcount = (int)min((int64_t)kChunk, p.ng - g0);
        float myMn = 0.0f, myMx = 0.0f;
        if (kFast && ACTNN_K1_PREFETCH) {
            if (t + gridDim.x < tiles) load_tile(t + gridDim.x, nxt);
        } else if (kFast) {
            load_tile(t, cur);
        }
        if constexpr (kFast && sizeof(T) == 2) {
            // bf16: min and max on packed bf16x2 words (both are exact on bf16
            // values), carried through the butterfly as one (min, -max) pair
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (gw + u < gcount) {
                    float mn, mx;
                    warp_minmax_bf16(cur[u][0], mn, mx);
                    if (lane == u) {
                        myMn = mn;
                        myMx = mx;
                    }
                }
            }
        } else if (kFast) {
            float v[kU][8];
#pragma unroll
            for (int u = 0; u < kU; ++u) raw8_f32<T>(cur[u], v[u]);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (gw + u < gcount) {
                    float mn = v[u][0], mx = v[u][0];
#pragma unroll
                    for (int j = 1; j < 8; ++j) {
                        mn = fminf(mn, v[u][j]);
                        mx = fmaxf(mx, v[u][j]);
                    }
                    mn = warp_min(mn);
                    mx = warp_max(mx);
                    if (lane == u) {
                        myMn = mn;
                        myMx = mx;
                    }
                }
            }
        } else {
            for (int u = 0; u < kU; ++u) {
                if (gw + u < gcount) {
                    const int64_t i = g0 + gw + u;
                    const int len = (int)min((int64_t)kG, p.D - i * kG);
                    const T* src = x + n * p.D + i * kG;
                    float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
                    for (int j = 0; j < 8; ++j) {
                        const int idx = lane * 8 + j;
                        if (idx < len) {
                            const float h = load1(src + idx);
                            mn = fminf(mn, h);
                            mx = fmaxf(mx, h);
                        }
                    }
                    mn = warp_min(mn);
                    mx = warp_max(mx);
                    if (lane == u) {
                        myMn = mn;
                        myMx = mx;
                    }
                }
            }
        }
        if (lane < kU && gw + lane < gcount) {
            sZ[gw + lane] = __fadd_rn(myMn, 0.0f);  // canonical +0 (DESIGN reading 17)
            sM[gw + lane] = __fadd_rn(myMx, 0.0f);
        }
        __syncthreads();
        if (w == 0) {
            double v = 0.0;
            if (lane < gcount) {
                const float Z = sZ[lane], M = sM[lane];
                p.gmin[n * p.ng + g0 + lane] = Z;
                p.gmax[n * p.ng + g0 + lane] = M;
                const float R = __fsub_rn(M, Z);
                v = __dmul_rn((double)R, (double)R);  // exact: 24b x 24b < 53b
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, o));
            if (lane == 0) p.T[c * p.N + n] = v;  // chunk-major: coalesced in K1b
        }
        __syncthreads();
        if (kFast && ACTNN_K1_PREFETCH) {
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                cur[u][0] = nxt[u][0];
                cur[u][1] = nxt[u][1];
            }
        }
    }
    // K1b fused: the last CTA sums every sample's chunk partials in order.
    __shared__ unsigned int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicInc(p.ticket, gridDim.x - 1) == gridDim.x - 1);
    __syncthreads();
    if (s_last) {
        __threadfence();
        for (int64_t n = threadIdx.x; n < p.N; n += kBlock) {
            const double s = sum_chunks_in_order(p.T, p.nch, p.N, n);
            p.sens[n] = s;
        }
    }
}

template <typename T>
cudaError_t run(const StatsArgs& a, cudaStream_t s) {
    SParams p{a.x, a.N, a.D, a.ng, a.nch, a.gmin, a.gmax, a.T, a.sens,
              reinterpret_cast<unsigned int*>(a.T + a.N * a.nch)};
    const int64_t tiles = a.N * a.nch;
    if (a.fast) {
        int grid = grid_for((const void*)group_stats_kernel<T, true>, SCfg<T>::Block, 0, tiles);
        // fp32: a persistent grid of 4 CTAs (32 warps) per SM measured best (the
        // occupancy limit, 8, is 2-4% slower on large tensors); bf16 keeps the
        // occupancy limit (4 per SM is 11% slower there).  -DACTNN_K1_CTAS_PER_SM
        // overrides at build time (0: occupancy limit).
        const int cap_per_sm = ACTNN_K1_CTAS_PER_SM >= 0 ? ACTNN_K1_CTAS_PER_SM
                                                         : (sizeof(T) == 4 ? 4 : 0);
        if (cap_per_sm > 0 && grid > sm_count() * cap_per_sm) grid = sm_count() * cap_per_sm;
        launch_pdl(group_stats_kernel<T, true>, grid, SCfg<T>::Block, 0, s, p);
    } else {
        const int grid = grid_for((const void*)group_stats_kernel<T, false>, SCfg<T>::Block, 0, tiles);
        launch_pdl(group_stats_kernel<T, false>, grid, SCfg<T>::Block, 0, s, p);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_group_stats(const StatsArgs& a, cudaStream_t s) {
    return a.dt == 0 ? run<float>(a, s) : run<uint16_t>(a, s);
}

}  // namespace actnn
