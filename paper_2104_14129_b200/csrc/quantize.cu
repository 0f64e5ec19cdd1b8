// quantize.cu -- K3: per-group stochastic-rounding quantiser + bit packer
// (P:491-503 per-group quantisation, "compress them into bit
// streams"), ACTNN-Q v1 steps O1-O9.
//
// Fast path (D % 256 == 0, x 32-byte aligned).  A warp's unit is U = 4
// consecutive groups of one sample.  Each warp owns a ring of S shared-memory
// stages fed by cp.async.bulk (TMA, SASS UBLKCP): lane 0 keeps the next units
// in flight, so HBM latency is covered by shared memory, not registers.
// Lane l owns elements [8l, 8l+8) of every group: one Philox4x32-10 call per
// group gives its 8 x 16 random bits, and its codes fill bytes [l b, (l+1) b)
// of the group's 32 b-byte segment.
//   - units are walked without division: (n, j) advances by the constant
//     stride (nwarps / nb, nwarps % nb) with one carry;
//   - group min/max (uniform single pass only): 8-element local min/max, then
//     one redux.sync (CREDUX) each; a full unit at width 1/2/4/8 runs straight
//     line (sp_full_unit: its Philox draws issued first, no per-group
//     branches); in the mixed path (gmin, gmax) come from
//     K1 and are prefetched one unit ahead (the mixed path normally runs the
//     warp-specialised kernel of quantize_ws.cu instead);
//   - per-group constants (two IEEE divisions) are computed lane-parallel, lane
//     u for group u of the unit, and broadcast with one shuffle each;
//   - codes (device.cuh): delta = RN(h - Z) (FADD; bf16 via the mixed-precision
//     FHADD.BF16), q from one scalar FFMA against 1.5*2^23; for b <= 2 two
//     codes share one register (byte permute, one add of both 14-bit draws)
//     and are gathered into the packed byte / half-word by byte permutes and one
//     multiply (device.cuh codes_small_d); b >= 3 one code per element;
//   - Philox round keys live in the parameter constant bank (no key registers);
//   - stores: every lane writes its own b code bytes (b <= 2: 1-2 bytes, b = 4
//     / 8: one 4 / 8-byte word), so one warp store fills the group's 32 b-byte
//     segment (whole sectors).
// Ragged D, unaligned x or huge tensors take the generic kernel (scalar loads,
// one group per warp iteration); it produces exactly the same bytes.
#include <cstdlib>

#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

#ifndef ACTNN_NO_WS
#define ACTNN_NO_WS 0  // build-time diagnostics: 1 sends the mixed path to this file's kernel
#endif
#ifndef ACTNN_SP8
#define ACTNN_SP8 1  // 0: the fp32 single pass runs this file's 4-group kernel
#endif

constexpr int kU = 4;
constexpr int kWarps = 8;
constexpr int kBlock = kWarps * 32;
constexpr int kNCap = 2048;  // samples whose (bits, off) are cached in shared memory
constexpr unsigned kFull = 0xffffffffu;
#ifndef ACTNN_Q_KEYS
#define ACTNN_Q_KEYS 0
#endif

template <typename T>
struct Cfg;
// fp32: 2 CTAs of 8 warps per SM with 3 stages each (round 2, with the
// straight-line full-unit single pass: C2 K3 178 -> 168 us; 3 CTAs x 2 stages
// leaves that path 80 registers and spills)
#ifndef ACTNN_Q_S32
#define ACTNN_Q_S32 3
#endif
#ifndef ACTNN_Q_MINB32
#define ACTNN_Q_MINB32 2
#endif
#ifndef ACTNN_Q_S16
#define ACTNN_Q_S16 4
#endif
#ifndef ACTNN_Q_MINB16
#define ACTNN_Q_MINB16 3
#endif
template <>
struct Cfg<float> {
    static constexpr int S = ACTNN_Q_S32;          // stages per warp (4 KB each)
    static constexpr int MinBlocks = ACTNN_Q_MINB32;  // CTAs per SM
};
template <>
struct Cfg<uint16_t> {
    static constexpr int S = ACTNN_Q_S16;  // 2 KB each
    static constexpr int MinBlocks = ACTNN_Q_MINB16;
};

template <typename T>
__host__ __device__ constexpr int stage_bytes() {
    return kU * kG * (int)sizeof(T);
}
template <typename T>
__host__ __device__ constexpr size_t smem_bytes() {
    return (size_t)kWarps * Cfg<T>::S * stage_bytes<T>() + (size_t)kWarps * Cfg<T>::S * 8 + kNCap +
           4 * (kNCap + 1);
}

struct QParams {
    const void* x;
    uint32_t N, D, ng, nb;      // nb = ceil(ng / U) units per sample
    uint32_t step_n, step_j;    // unit stride of a warp: nwarps = step_n * nb + step_j
    uint32_t sample_base;
    const uint8_t* bits;
    const int64_t* off;
    const float* gmin;
    const float* gmax;
    uint8_t* packed;
    float* zmin;
    float* scale;
    uint32_t* meta;  // bf16 metadata words (NEXT-1) instead of zmin/scale, or null
    RoundKeys rk;
};

struct GParams {  // generic kernel
    const void* x;
    int64_t N, D, ng;
    int64_t sample_base;
    const uint8_t* bits;
    const int64_t* off;
    const float* gmin;
    const float* gmax;
    uint8_t* packed;
    float* zmin;
    float* scale;
    uint32_t* meta;
    RoundKeys rk;
};

// Group constants of either metadata format; stores this group's metadata.
__device__ __forceinline__ void group_const_store(float mn, float mx, int b, uint32_t* meta,
                                                  float* zm, float* sc, bool store, float& Z,
                                                  float& inv14) {
    if (meta) {  // NEXT-1: bf16 words, quantise with the stored values
        const GroupConstB c = group_const_bf16(mn, mx, b);
        if (store) *meta = c.word;
        Z = c.Z;
        inv14 = c.inv14;
    } else {
        const GroupConst c = group_const(mn, mx, b);
        if (store) {
            *zm = c.Z;
            *sc = c.scale;
        }
        Z = c.Z;
        inv14 = c.inv14;
    }
}

// Codes for b in {1, 2}: codes_small (device.cuh).

// Codes for b >= 3: codes_wide (device.cuh).

// One group: Philox draw for the lane's 8-element block, SR codes, pack, store
// (ACTNN-Q v1 O6-O8).  seg = the group's 32 b-byte segment.
template <int b, typename In>
__device__ __forceinline__ void quant_group(const In& v, float Z, float inv14, uint64_t blk,
                                            const RoundKeys& rk, uint8_t* seg, int lane) {
#if ACTNN_Q_KEYS == 1
    const Philox4 o = philox4x32_10((uint32_t)blk, (uint32_t)(blk >> 32), rk.k[0], rk.k[1]);
#else
    const Philox4 o = philox4x32_10_c32((uint32_t)blk, rk);
#endif
    // every lane stores its own b bytes; one warp store fills the group's
    // 32 b-byte segment (measured faster than shuffling into word stores)
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
        } else {  // b in {3, 5, 6, 7}: b bytes per lane, not word aligned
            uint64_t pl = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) pl |= (uint64_t)code[j] << (b * j);
#pragma unroll
            for (int t = 0; t < b; ++t) seg[lane * b + t] = (uint8_t)(pl >> (8 * t));
        }
    }
}

// Width-dependent part of a unit: lane-parallel constants (lane u owns group
// u of the unit), then codes + packing of each group.  kFullUnit: gcount == U.
template <int b, bool kFullUnit, typename In>
__device__ __forceinline__ void quant_unit(const In (&v)[kU], int gcount, float myMn,
                                           float myMx, float* zm, float* sc, uint32_t* mw,
                                           uint8_t* seg, uint64_t blk0, const RoundKeys& rk,
                                           int lane) {
    float cZ, cInv;
    group_const_store(myMn, myMx, b, mw ? mw + lane : nullptr, zm + lane, sc + lane,
                      lane < (kFullUnit ? kU : gcount), cZ, cInv);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        if (kFullUnit || u < gcount) {
            const float Z = __shfl_sync(kFull, cZ, u);
            const float inv = __shfl_sync(kFull, cInv, u);
            quant_group<b>(v[u], Z, inv, blk0 + (uint64_t)(u * 32 + lane), rk, seg + u * 32 * b,
                           lane);
        }
    }
}

template <int b, typename In>
__device__ __forceinline__ void quant_unit_any(const In (&v)[kU], int gcount, float myMn,
                                               float myMx, float* zm, float* sc, uint32_t* mw,
                                               uint8_t* seg, uint64_t blk0, const RoundKeys& rk,
                                               int lane) {
    if (gcount == kU)
        quant_unit<b, true>(v, gcount, myMn, myMx, zm, sc, mw, seg, blk0, rk, lane);
    else
        quant_unit<b, false>(v, gcount, myMn, myMx, zm, sc, mw, seg, blk0, rk, lane);
}

// Full unit (gcount == U) of the single pass (statistics in-kernel), straight
// line with no per-group branches.  The Philox draws depend only on the unit
// index, so they are issued first: their ten-round IMAD.WIDE chains overlap
// the statistics' dependency chain (lane min/max -> CREDUX -> lane-parallel
// divisions -> shuffles) instead of waiting behind it.
#ifndef ACTNN_SP_FULL
#define ACTNN_SP_FULL 1
#endif
#ifndef ACTNN_SP_HOIST
#define ACTNN_SP_HOIST 1  // 0: each group's Philox draw just before its codes
#endif
template <int b, typename In>
__device__ __forceinline__ void sp_full_unit(const In (&v)[kU], float* zm, float* sc,
                                             uint32_t* mw, uint8_t* seg, uint64_t blk0,
                                             const RoundKeys& rk, int lane) {
    Philox4 o[kU];
#if ACTNN_SP_HOIST
#pragma unroll
    for (int u = 0; u < kU; ++u)
        o[u] = philox4x32_10_c32((uint32_t)(blk0 + (uint64_t)(u * 32 + lane)), rk);
#endif
    float gmn[kU], gmx[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        float mn, mx;
        lane_minmax(v[u], mn, mx);
        gmn[u] = warp_min(mn);
        gmx[u] = warp_max(mx);
    }
    // lane u (< U) computes group u's constants
    float myMn = gmn[0], myMx = gmx[0];
#pragma unroll
    for (int u = 1; u < kU; ++u) {
        myMn = lane == u ? gmn[u] : myMn;
        myMx = lane == u ? gmx[u] : myMx;
    }
    float cZ, cInv;
    group_const_store(myMn, myMx, b, mw ? mw + lane : nullptr, zm + lane, sc + lane, lane < kU,
                      cZ, cInv);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        const float Z = __shfl_sync(kFull, cZ, u);
        const float inv = __shfl_sync(kFull, cInv, u);
#if !ACTNN_SP_HOIST
        o[u] = philox4x32_10_c32((uint32_t)(blk0 + (uint64_t)(u * 32 + lane)), rk);
#endif
        uint8_t* sg = seg + u * 32 * b;
        if constexpr (b == 2) {
            reinterpret_cast<uint16_t*>(sg)[lane] = (uint16_t)codes_small<2>(v[u], Z, inv, o[u]);
        } else if constexpr (b == 1) {
            sg[lane] = (uint8_t)codes_small<1>(v[u], Z, inv, o[u]);
        } else {
            uint32_t code[8];
            codes_wide(v[u], Z, inv, o[u], code);
            if constexpr (b == 8) {
                const uint32_t lo = code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
                const uint32_t hi = code[4] | (code[5] << 8) | (code[6] << 16) | (code[7] << 24);
                *reinterpret_cast<uint2*>(sg + lane * 8) = make_uint2(lo, hi);
            } else {
                static_assert(b == 4, "full-unit widths: 1, 2, 4, 8");
                uint32_t pl = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) pl |= code[j] << (4 * j);
                *reinterpret_cast<uint32_t*>(sg + lane * 4) = pl;
            }
        }
    }
}

template <typename T, bool kStats, bool kCached>
__global__ void __launch_bounds__(kBlock, Cfg<T>::MinBlocks)
    quantize_fast_kernel(const __grid_constant__ QParams p) {
    pdl_trigger();  // the next kernel of the stream may start launching
    pdl_wait();     // the previous grid is complete and visible
    constexpr int S = Cfg<T>::S;
    constexpr int SE = stage_bytes<T>() / (int)sizeof(T);  // elements per stage
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    T* ring = reinterpret_cast<T*>(smem) + (size_t)w * S * SE;
    uint64_t* bars =
        reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * S * stage_bytes<T>()) + w * S;
    uint8_t* s_bits = smem + (size_t)kWarps * S * stage_bytes<T>() + (size_t)kWarps * S * 8;
    uint32_t* s_off = reinterpret_cast<uint32_t*>(s_bits + kNCap);

    const int64_t off0 = p.off[0];
    if (kCached) {
        for (uint32_t i = threadIdx.x; i < p.N; i += kBlock) {
            s_bits[i] = p.bits[i];
            s_off[i] = (uint32_t)((p.off[i] - off0) >> 5);  // offsets are multiples of 32 B
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t gw = blockIdx.x * kWarps + w;
    const T* __restrict__ x = static_cast<const T*>(p.x);
    auto advance = [&](uint32_t& n, uint32_t& j) {
        n += p.step_n;
        j += p.step_j;
        if (j >= p.nb) {
            j -= p.nb;
            ++n;
        }
    };
    auto gcount_of = [&](uint32_t j) { return (int)min((uint32_t)kU, p.ng - j * kU); };

    // producer state (lane 0): the next unit to bulk-copy
    uint32_t pn = gw / p.nb, pj = gw % p.nb;
    uint32_t n = pn, j = pj;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (pn < p.N) {
                const uint32_t bytes = (uint32_t)(gcount_of(pj) * kG * (int)sizeof(T));
                mbar_expect_tx(&bars[s], bytes);
                bulk_g2s(ring + s * SE, x + (uint64_t)pn * p.D + (uint64_t)pj * (kU * kG), bytes,
                         &bars[s]);
            }
            advance(pn, pj);
        }
    }
    // mixed path: (gmin, gmax) of the current unit, prefetched one unit ahead
    float nMn = 0.0f, nMx = 0.0f;
    if (!kStats && n < p.N && lane < gcount_of(j)) {
        const uint32_t g = n * p.ng + j * kU + lane;
        nMn = __ldg(p.gmin + g);
        nMx = __ldg(p.gmax + g);
    }
    int stage = 0;
    uint32_t phase = 0;
    while (n < p.N) {
        const int gcount = gcount_of(j);
        const uint32_t gi = j * kU;
        const uint32_t g = n * p.ng + gi;
        float myMn = nMn, myMx = nMx;
        uint32_t nn = n, nj = j;
        advance(nn, nj);
        if (!kStats && nn < p.N && lane < gcount_of(nj)) {
            const uint32_t g2 = nn * p.ng + nj * kU + lane;
            nMn = __ldg(p.gmin + g2);
            nMx = __ldg(p.gmax + g2);
        }
        const int b = kCached ? (int)s_bits[n] : (int)p.bits[n];
        const int64_t sofs = kCached ? ((int64_t)s_off[n] << 5) : (p.off[n] - off0);

        mbar_wait(&bars[stage], phase);
        // a lane's 8 elements per group: widened fp32, or (bf16) the raw words
        typename LaneIn<T>::type v[kU];
        const T* st = ring + stage * SE;
#pragma unroll
        for (int k = 0; k < kU; ++k)
            if (k < gcount) lane_load(st + k * kG + lane * 8, v[k]);
        // Re-arm the stage with the unit S ahead as soon as it has been read, so
        // S units stay in flight while this one is computed.  Cross-proxy WAR
        // (generic-proxy shared loads, then an async-proxy bulk write to the same
        // bytes): every lane orders its loads before the async proxy with
        // fence.proxy.async, the __syncwarp orders all lanes before lane 0, and
        // only then does lane 0 issue the copy into the stage.
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            if (pn < p.N) {
                const uint32_t bytes = (uint32_t)(gcount_of(pj) * kG * (int)sizeof(T));
                mbar_expect_tx(&bars[stage], bytes);
                bulk_g2s(ring + stage * SE, x + (uint64_t)pn * p.D + (uint64_t)pj * (kU * kG),
                         bytes, &bars[stage]);
            }
            advance(pn, pj);
        }
        if constexpr (kStats && ACTNN_SP_FULL) {
            if (gcount == kU && (b == 1 || b == 2 || b == 4 || b == 8)) {
                uint8_t* seg = p.packed + sofs + (uint64_t)gi * 32 * b;
                const uint64_t blk0 = (uint64_t)(p.sample_base + n) * (p.D >> 3) + (uint64_t)gi * 32;
                float* zm = p.zmin + g;
                float* sc = p.scale + g;
                uint32_t* mw = p.meta ? p.meta + g : nullptr;
                if (b == 2) sp_full_unit<2>(v, zm, sc, mw, seg, blk0, p.rk, lane);
                else if (b == 1) sp_full_unit<1>(v, zm, sc, mw, seg, blk0, p.rk, lane);
                else if (b == 4) sp_full_unit<4>(v, zm, sc, mw, seg, blk0, p.rk, lane);
                else sp_full_unit<8>(v, zm, sc, mw, seg, blk0, p.rk, lane);
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1u;
                }
                n = nn;
                j = nj;
                continue;
            }
        }
        if constexpr (kStats) {
#pragma unroll
            for (int k = 0; k < kU; ++k) {
                if (k < gcount) {
                    float mn, mx;
                    lane_minmax(v[k], mn, mx);
                    mn = warp_min(mn);
                    mx = warp_max(mx);
                    if (lane == k) {
                        myMn = mn;
                        myMx = mx;
                    }
                }
            }
        }
        uint8_t* seg = p.packed + sofs + (uint64_t)gi * 32 * b;
        const uint64_t blk0 = (uint64_t)(p.sample_base + n) * (p.D >> 3) + (uint64_t)gi * 32;
        float* zm = p.zmin + g;
        float* sc = p.scale + g;
        uint32_t* mw = p.meta ? p.meta + g : nullptr;
#define ACTNN_QU(B) quant_unit_any<B>(v, gcount, myMn, myMx, zm, sc, mw, seg, blk0, p.rk, lane)
#define ACTNN_QG(B) quant_unit<B, false>(v, gcount, myMn, myMx, zm, sc, mw, seg, blk0, p.rk, lane)
        switch (b) {
            case 1: ACTNN_QU(1); break;
            case 2: ACTNN_QU(2); break;
            case 4: ACTNN_QU(4); break;
            case 8: ACTNN_QU(8); break;
            case 3: ACTNN_QG(3); break;
            case 5: ACTNN_QG(5); break;
            case 6: ACTNN_QG(6); break;
            case 7: ACTNN_QG(7); break;
#undef ACTNN_QU
#undef ACTNN_QG
            default: break;  // invalid width: outside the contract (ACTNN_CHECK=1 reports it)
        }
        if (++stage == S) {
            stage = 0;
            phase ^= 1u;
        }
        n = nn;
        j = nj;
    }
}

// Generic path: any D (ragged last group), any element alignment.  One group
// per warp iteration; lane l holds elements [8l, 8l+8) of the group, masked
// past the group's real length; the Philox block of element e is e >> 3, so a
// lane needs at most two blocks when D % 8 != 0.
template <typename T, bool kStats>
__global__ void __launch_bounds__(kBlock) quantize_generic_kernel(const __grid_constant__ GParams p) {
    pdl_trigger();  // the next kernel of the stream may start launching
    pdl_wait();     // the previous grid is complete and visible
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
        for (int jj = 0; jj < 8; ++jj) {
            const int idx = lane * 8 + jj;
            v[jj] = idx < len ? load1(src + idx) : 0.0f;
            if (idx < len) {
                mn = fminf(mn, v[jj]);
                mx = fmaxf(mx, v[jj]);
            }
        }
        if (kStats) {
            mn = warp_min(mn);
            mx = warp_max(mx);
        } else {
            mn = __ldg(p.gmin + g);
            mx = __ldg(p.gmax + g);
        }
        float cZ, cInv;
        group_const_store(mn, mx, b, p.meta ? p.meta + g : nullptr, p.zmin + g, p.scale + g,
                          lane == 0, cZ, cInv);
        const uint64_t e_first =
            (uint64_t)(p.sample_base + n) * (uint64_t)p.D + (uint64_t)(i * kG + lane * 8);
        const uint64_t blkA = e_first >> 3;
        const Philox4 oA = philox4x32_10((uint32_t)blkA, (uint32_t)(blkA >> 32), p.rk);
        const uint64_t blkB = blkA + 1;
        const Philox4 oB = philox4x32_10((uint32_t)blkB, (uint32_t)(blkB >> 32), p.rk);
        uint64_t pk = 0;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int idx = lane * 8 + jj;
            const uint64_t e = e_first + jj;
            const uint32_t r =
                ((e >> 3) == blkA) ? rnd14(oA, (int)(e & 7)) : rnd14(oB, (int)(e & 7));
            const uint32_t code = idx < len ? sr_code(v[jj], cZ, cInv, r) : 0u;
            pk |= (uint64_t)code << (b * jj);
        }
        uint8_t* seg = p.packed + (p.off[n] - off0) + i * 32 * b;
        for (int t = 0; t < b; ++t) seg[lane * b + t] = (uint8_t)(pk >> (8 * t));
    }
}

template <typename T, bool kStats>
cudaError_t run(const QuantArgs& a, cudaStream_t s) {
    const int64_t nb = (a.ng + kU - 1) / kU;
    // fast path: 32-bit unit walk (N * ng, D, sample_base + N < 2^31)
    // fast kernels: 32-bit unit walks, and Philox counters (global element
    // index >> 3) below 2^32 (philox4x32_10_c32); larger problems take the
    // generic kernel, which carries the full 64-bit counter
    const bool fits = a.N * a.ng < (1ll << 31) && a.D < (1ll << 31) &&
                      a.sample_base + a.N < (1ll << 31) &&
                      (a.sample_base + a.N) * a.D <= (1ll << 35);
    if (a.fast && fits) {
        QParams p;
        p.x = a.x;
        p.N = (uint32_t)a.N;
        p.D = (uint32_t)a.D;
        p.ng = (uint32_t)a.ng;
        p.nb = (uint32_t)nb;
        p.sample_base = (uint32_t)a.sample_base;
        p.bits = a.bits;
        p.off = a.off;
        p.gmin = a.gmin;
        p.gmax = a.gmax;
        p.packed = a.packed;
        p.zmin = a.zmin;
        p.scale = a.scale;
        p.meta = a.meta;
        p.rk = make_round_keys(a.seed);
        const bool cached = a.N <= kNCap;
        const void* k = cached ? (const void*)quantize_fast_kernel<T, kStats, true>
                               : (const void*)quantize_fast_kernel<T, kStats, false>;
        ensure_smem_attr(k, smem_bytes<T>());  // opt-in above 48 KB of dynamic smem
        const int64_t units = a.N * nb;
        const int grid = grid_for(k, kBlock, smem_bytes<T>(), (units + kWarps - 1) / kWarps);
        const uint32_t nwarps = (uint32_t)grid * kWarps;
        p.step_n = nwarps / p.nb;
        p.step_j = nwarps % p.nb;
        if (cached)
            launch_pdl(quantize_fast_kernel<T, kStats, true>, grid, kBlock, smem_bytes<T>(), s, p);
        else
            launch_pdl(quantize_fast_kernel<T, kStats, false>, grid, kBlock, smem_bytes<T>(), s, p);
    } else {
        GParams p;
        p.x = a.x;
        p.N = a.N;
        p.D = a.D;
        p.ng = a.ng;
        p.sample_base = a.sample_base;
        p.bits = a.bits;
        p.off = a.off;
        p.gmin = a.gmin;
        p.gmax = a.gmax;
        p.packed = a.packed;
        p.zmin = a.zmin;
        p.scale = a.scale;
        p.meta = a.meta;
        p.rk = make_round_keys(a.seed);
        const void* k = (const void*)quantize_generic_kernel<T, kStats>;
        const int grid = grid_for(k, kBlock, 0, (a.N * a.ng + kWarps - 1) / kWarps);
        launch_pdl(quantize_generic_kernel<T, kStats>, grid, kBlock, 0, s, p);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t s) {
    const bool stats = (a.gmin == nullptr);
    // fast kernels: 32-bit unit walks, and Philox counters (global element
    // index >> 3) below 2^32 (philox4x32_10_c32); larger problems take the
    // generic kernel, which carries the full 64-bit counter
    const bool fits = a.N * a.ng < (1ll << 31) && a.D < (1ll << 31) &&
                      a.sample_base + a.N < (1ll << 31) &&
                      (a.sample_base + a.N) * a.D <= (1ll << 35);
    // mixed path (group stats given): the warp-specialised kernel (quantize_ws.cu)
    if (!stats && a.fast && fits && !ACTNN_NO_WS) return launch_quantize_ws(a, s);
    // fp32 single pass (uniform widths, statistics in-kernel): 8-group units
    // (quantize_sp8.cu)
    if (stats && a.fast && fits && a.dt == 0 && ACTNN_SP8) return launch_quantize_sp8(a, s);
    if (a.dt == 0) return stats ? run<float, true>(a, s) : run<float, false>(a, s);
    return stats ? run<uint16_t, true>(a, s) : run<uint16_t, false>(a, s);
}

}  // namespace actnn
