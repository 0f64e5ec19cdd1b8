// quantize_sp8.cu -- K3 single pass (statistics in-kernel: the uniform-width L2
// path; per-group quantisation P:491-503, ACTNN-Q v1 O1-O9) for fp32
// inputs, on units of 8 groups.  Same bytes as quantize.cu.
//
// The single pass is instruction-bound (Philox plus the codes take
// ~64 instructions per group, and on quantize.cu's 4-group units the unit
// hand-off -- ring wait, TMA refill, the (n, j) walk, width and offset lookups
// -- and the lane-parallel divisions add ~45 more).  An 8 KB unit halves those
// per group.  Eight fp32 groups do not fit in registers next to the Philox
// state, so a unit is read from its stage twice:
//   pass 1 (O3-O4): per group the lane's 8 values (two 16-byte shared loads),
//     lane min/max (FMNMX3), one CREDUX each for min and max; lane u keeps
//     group u's pair, then lanes 0-7 compute the constants (two IEEE
//     divisions) and store zmin/scale;
//   pass 2 (O5-O8): per group the Philox draw, the values again, the codes
//     and the store, two groups at a time; after the last shared read the
//     stage goes back to the copy engine with the unit S ahead.
// A warp owns a ring of S stages (cp.async.bulk, mbarrier complete_tx).
#include <cstdlib>

#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

// one CTA of 12 warps per SM, 2 stages (192 KB of rings): C2 K3 161 us against
// 168 for 2 CTAs x 6 warps and for quantize.cu's 4-group kernel; 8 warps x 2
// stages and 4 warps x 3 stages x 2 CTAs measured 195 us
#ifndef ACTNN_SP8_WARPS
#define ACTNN_SP8_WARPS 12
#endif
#ifndef ACTNN_SP8_S
#define ACTNN_SP8_S 2
#endif
#ifndef ACTNN_SP8_MINB
#define ACTNN_SP8_MINB 1
#endif
constexpr int kU = 8;                      // groups per unit
constexpr int kWarps = ACTNN_SP8_WARPS;
constexpr int kBlock = kWarps * 32;
constexpr int kS = ACTNN_SP8_S;
constexpr int kSE = kU * kG;               // elements per stage (8 KB)
constexpr int kNCap = 2048;
constexpr unsigned kFull = 0xffffffffu;

constexpr size_t sp8_smem_bytes() {
    return (size_t)kWarps * kS * kSE * 4 + (size_t)kWarps * kS * 8 + kNCap + 4 * (kNCap + 1);
}

struct SP8Params {
    const float* x;
    uint32_t N, D, ng, nb;    // nb = ceil(ng / 8) units per sample
    uint32_t step_n, step_j;  // unit stride of a warp: nwarps = step_n * nb + step_j
    uint32_t sample_base;
    const uint8_t* bits;
    const int64_t* off;
    uint8_t* packed;
    float* zmin;
    float* scale;
    uint32_t* meta;  // NEXT-1 bf16 metadata words instead of zmin/scale, or null
    RoundKeys rk;
};

// Codes of one group at width b, packed and stored (every lane its own b bytes
// of the group's 32 b-byte segment).
template <int b>
__device__ __forceinline__ void sp8_store(const F8& v, float Z, float inv14, const Philox4& o,
                                          uint8_t* seg, int lane) {
    if constexpr (b == 2) {
        reinterpret_cast<uint16_t*>(seg)[lane] = (uint16_t)codes_small<2>(v, Z, inv14, o);
    } else if constexpr (b == 1) {
        seg[lane] = (uint8_t)codes_small<1>(v, Z, inv14, o);
    } else {
        uint32_t code[8];
        codes_wide(v, Z, inv14, o, code);
        if constexpr (b == 8) {
            const uint32_t lo = code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
            const uint32_t hi = code[4] | (code[5] << 8) | (code[6] << 16) | (code[7] << 24);
            *reinterpret_cast<uint2*>(seg + lane * 8) = make_uint2(lo, hi);
        } else if constexpr (b == 4) {
            uint32_t pl = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) pl |= code[j] << (4 * j);
            *reinterpret_cast<uint32_t*>(seg + lane * 4) = pl;
        } else {  // b in {3, 5, 6, 7}
            uint64_t pl = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) pl |= (uint64_t)code[j] << (b * j);
#pragma unroll
            for (int t = 0; t < b; ++t) seg[lane * b + t] = (uint8_t)(pl >> (8 * t));
        }
    }
}

__device__ __forceinline__ void sp8_store_any(int b, const F8& v, float Z, float inv,
                                              const Philox4& o, uint8_t* seg, int lane) {
    switch (b) {
        case 1: sp8_store<1>(v, Z, inv, o, seg, lane); break;
        case 2: sp8_store<2>(v, Z, inv, o, seg, lane); break;
        case 3: sp8_store<3>(v, Z, inv, o, seg, lane); break;
        case 4: sp8_store<4>(v, Z, inv, o, seg, lane); break;
        case 5: sp8_store<5>(v, Z, inv, o, seg, lane); break;
        case 6: sp8_store<6>(v, Z, inv, o, seg, lane); break;
        case 7: sp8_store<7>(v, Z, inv, o, seg, lane); break;
        case 8: sp8_store<8>(v, Z, inv, o, seg, lane); break;
        default: break;  // invalid width: outside the contract (ACTNN_CHECK=1 reports it)
    }
}

// Pass 2 of a full unit at a width fixed at compile time: two groups at a
// time, their Philox draws issued ahead of the shared loads.
template <int b>
__device__ __forceinline__ void sp8_codes_full(const float* st, float cZ, float cInv, uint64_t blk,
                                               uint8_t* seg, const RoundKeys& rk, int lane) {
#pragma unroll
    for (int h = 0; h < kU; h += 2) {
        const Philox4 o0 = philox4x32_10_c32((uint32_t)(blk + (uint64_t)(h * 32)), rk);
        const Philox4 o1 = philox4x32_10_c32((uint32_t)(blk + (uint64_t)((h + 1) * 32)), rk);
        F8 v0, v1;
        lane_load(st + h * kG + lane * 8, v0);
        lane_load(st + (h + 1) * kG + lane * 8, v1);
        const float Z0 = __shfl_sync(kFull, cZ, h), I0 = __shfl_sync(kFull, cInv, h);
        const float Z1 = __shfl_sync(kFull, cZ, h + 1), I1 = __shfl_sync(kFull, cInv, h + 1);
        sp8_store<b>(v0, Z0, I0, o0, seg + h * 32 * b, lane);
        sp8_store<b>(v1, Z1, I1, o1, seg + (h + 1) * 32 * b, lane);
    }
}

template <bool kCached>
__global__ void __launch_bounds__(kBlock, ACTNN_SP8_MINB)
    quantize_sp8_kernel(const __grid_constant__ SP8Params p) {
    pdl_trigger();  // the next kernel of the stream may start launching
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    float* ring = reinterpret_cast<float*>(smem) + (size_t)w * kS * kSE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * kS * kSE * 4) + w * kS;
    uint8_t* s_bits = smem + (size_t)kWarps * kS * kSE * 4 + (size_t)kWarps * kS * 8;
    uint32_t* s_off = reinterpret_cast<uint32_t*>(s_bits + kNCap);
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kS; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    pdl_wait();  // the previous grid is complete and visible
    const int64_t off0 = p.off[0];
    if (kCached) {
        for (uint32_t i = threadIdx.x; i < p.N; i += kBlock) {
            s_bits[i] = p.bits[i];
            s_off[i] = (uint32_t)((p.off[i] - off0) >> 5);  // offsets are multiples of 32 B
        }
    }
    __syncthreads();

    auto advance = [&](uint32_t& n, uint32_t& j) {
        n += p.step_n;
        j += p.step_j;
        if (j >= p.nb) {
            j -= p.nb;
            ++n;
        }
    };
    auto gcount_of = [&](uint32_t j) { return (int)min((uint32_t)kU, p.ng - j * kU); };
    auto issue = [&](int s, uint32_t n, uint32_t j) {  // lane 0: bulk copy of unit (n, j)
        const uint32_t bytes = (uint32_t)(gcount_of(j) * kG * 4);
        mbar_expect_tx(&bars[s], bytes);
        bulk_g2s(ring + s * kSE, p.x + (uint64_t)n * p.D + (uint64_t)j * kSE, bytes, &bars[s]);
    };

    const uint32_t gw = blockIdx.x * kWarps + w;
    uint32_t n = gw / p.nb, j = gw % p.nb;
    uint32_t pn = n, pj = j;  // lane 0: the next unit to bulk-copy
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kS; ++s) {
            if (pn < p.N) issue(s, pn, pj);
            advance(pn, pj);
        }
    }
    int stage = 0;
    uint32_t phase = 0;
    while (n < p.N) {
        const int gcount = gcount_of(j);
        const int b = kCached ? (int)s_bits[n] : (int)p.bits[n];
        const int64_t sofs = kCached ? ((int64_t)s_off[n] << 5) : (p.off[n] - off0);
        const float* st = ring + stage * kSE;
        mbar_wait(&bars[stage], phase);

        // pass 1: group min / max; lane u keeps group u's (O3)
        float myMn = 0.0f, myMx = 0.0f;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (u < gcount) {
                F8 v;
                lane_load(st + u * kG + lane * 8, v);
                float mn, mx;
                lane_minmax(v, mn, mx);
                mn = warp_min(mn);
                mx = warp_max(mx);
                myMn = lane == u ? mn : myMn;
                myMx = lane == u ? mx : myMx;
            }
        }
        // lanes 0-7: the constants of their group (O4) and its metadata
        const uint32_t g = n * p.ng + j * kU + lane;
        const bool mine = lane < gcount;
        float cZ, cInv;
        if (p.meta) {  // NEXT-1: bf16 words; quantise with the stored values
            const GroupConstB c = group_const_bf16(myMn, myMx, b);
            if (mine) p.meta[g] = c.word;
            cZ = c.Z;
            cInv = c.inv14;
        } else {
            const GroupConst c = group_const(myMn, myMx, b);
            if (mine) {
                p.zmin[g] = c.Z;
                p.scale[g] = c.scale;
            }
            cZ = c.Z;
            cInv = c.inv14;
        }

        // pass 2: codes (O5-O8)
        uint8_t* seg = p.packed + sofs + (uint64_t)j * kU * 32 * b;
        const uint64_t blk = (uint64_t)(p.sample_base + n) * (p.D >> 3) + (uint64_t)j * kU * 32 + lane;
        if (gcount == kU && (b == 1 || b == 2 || b == 4 || b == 8)) {
            if (b == 2) sp8_codes_full<2>(st, cZ, cInv, blk, seg, p.rk, lane);
            else if (b == 1) sp8_codes_full<1>(st, cZ, cInv, blk, seg, p.rk, lane);
            else if (b == 4) sp8_codes_full<4>(st, cZ, cInv, blk, seg, p.rk, lane);
            else sp8_codes_full<8>(st, cZ, cInv, blk, seg, p.rk, lane);
        } else {
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const float Z = __shfl_sync(kFull, cZ, u);
                const float inv = __shfl_sync(kFull, cInv, u);
                if (u < gcount) {
                    F8 v;
                    lane_load(st + u * kG + lane * 8, v);
                    const Philox4 o = philox4x32_10_c32((uint32_t)(blk + (uint64_t)(u * 32)), p.rk);
                    sp8_store_any(b, v, Z, inv, o, seg + u * 32 * b, lane);
                }
            }
        }
        // every shared read of the stage is done: back to the copy engine
        // (cross-proxy WAR: each lane's generic loads are ordered before the
        // async-proxy refill by fence.proxy.async, all lanes before lane 0 by
        // the __syncwarp)
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            if (pn < p.N) issue(stage, pn, pj);
            advance(pn, pj);
        }
        if (++stage == kS) {
            stage = 0;
            phase ^= 1u;
        }
        advance(n, j);
    }
}

template <bool kCached>
void launch_sp8(SP8Params p, int64_t units, cudaStream_t s) {
    const void* k = (const void*)quantize_sp8_kernel<kCached>;
    ensure_smem_attr(k, sp8_smem_bytes());
    const int grid = grid_for(k, kBlock, sp8_smem_bytes(), (units + kWarps - 1) / kWarps);
    const uint32_t nwarps = (uint32_t)grid * kWarps;
    p.step_n = nwarps / p.nb;
    p.step_j = nwarps % p.nb;
    launch_pdl(quantize_sp8_kernel<kCached>, grid, kBlock, sp8_smem_bytes(), s, p);
}

}  // namespace

// fp32 single pass (no gmin/gmax given), fast conditions checked by
// launch_quantize (D % 256 == 0, 32-byte aligned x, 32-bit unit walk, Philox
// counters below 2^32).
cudaError_t launch_quantize_sp8(const QuantArgs& a, cudaStream_t s) {
    SP8Params p;
    p.x = static_cast<const float*>(a.x);
    p.N = (uint32_t)a.N;
    p.D = (uint32_t)a.D;
    p.ng = (uint32_t)a.ng;
    p.nb = (uint32_t)((a.ng + kU - 1) / kU);
    p.step_n = p.step_j = 0;
    p.sample_base = (uint32_t)a.sample_base;
    p.bits = a.bits;
    p.off = a.off;
    p.packed = a.packed;
    p.zmin = a.zmin;
    p.scale = a.scale;
    p.meta = a.meta;
    p.rk = make_round_keys(a.seed);
    const int64_t units = a.N * (int64_t)p.nb;
    if (a.N <= kNCap)
        launch_sp8<true>(p, units, s);
    else
        launch_sp8<false>(p, units, s);
    return cudaGetLastError();
}

}  // namespace actnn
