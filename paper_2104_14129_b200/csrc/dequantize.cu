// dequantize.cu -- K4: unpacker + dequantiser ("During
// back-propagation, the activation is dequantized as h_hat = u_hat R/B + Z"),
// ACTNN-Q v1 step O10.  Mirrors K3: a warp's unit is 4 consecutive groups of
// one sample.  Everything the unit reads -- its packed bytes (contiguous:
// 4 x 32 b bytes) and, when the tensor's metadata is 16-byte aligned per unit
// (ng % 4 == 0), its 4 zero points and 4 scales -- arrives by cp.async.bulk
// (TMA, SASS UBLKCP) in a per-warp ring of S shared-memory stages; lane 0 keeps
// S units in flight and no global load is left on the warp's critical path.
// Lane l reads the b bytes holding its 8 codes from shared memory (the (Z,
// scale) pairs are broadcast reads) and writes its 8 consecutive outputs with
// one 256-bit (fp32) or 128-bit (bf16) store, so each warp store covers whole
// 32 B sectors -- or, for large fp32 outputs (kTS), into a per-warp staging
// buffer in shared memory that one bulk copy (cp.async.bulk shared -> global)
// writes out per unit.  (float)code uses the exact 2^23 magic; dequantisation is one
// __ffma2_rn per element pair (single rounding, O10).
#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

#ifndef ACTNN_DQ_U
#define ACTNN_DQ_U 4
#endif
constexpr int kU = ACTNN_DQ_U;  // groups per unit
constexpr int kWarps = 8;
constexpr int kBlock = kWarps * 32;
#ifndef ACTNN_DQ_S
#define ACTNN_DQ_S 4
#endif
#ifndef ACTNN_DQ_MINB
#define ACTNN_DQ_MINB 3
#endif
constexpr int kS = ACTNN_DQ_S;            // stages per warp
constexpr int kPay = kU * 32 * 8;         // payload bytes at the widest (b = 8)
constexpr int kStage = kPay + 8 * kU;     // + kU zero points + kU scales
constexpr int kNCap = 2048;
// TMA-store variant (kTS): each warp also owns kO output staging buffers of one
// unit; the outputs go shared -> global by cp.async.bulk (SASS UBLKCP.S.G), so
// the write stream leaves the SM through the TMA engine instead of the LSU.
// ACTNN_DQ_TS: 0 never, 1 always, 2 (default) for fp32 outputs of at least
// ACTNN_DQ_TS_MIN_MB megabytes -- measured per tensor size on the C3 / C4 sets
// (tools/k4_probe.py): the TMA-store kernel (one CTA of 8 warps per SM, 4
// staging buffers per warp) reaches 6.06 TB/s on the 822 MB C3 tensors against
// 5.44 for the LSU-store kernel, is even at 205 MB and slower below (fewer
// warps to cover the launch ramp) and on bf16 outputs.
#ifndef ACTNN_DQ_TS
#define ACTNN_DQ_TS 2
#endif
#ifndef ACTNN_DQ_TS_MIN_MB
#define ACTNN_DQ_TS_MIN_MB 192
#endif
#ifndef ACTNN_DQ_O
#define ACTNN_DQ_O 4
#endif
#ifndef ACTNN_DQ_TSW
#define ACTNN_DQ_TSW 8
#endif
#ifndef ACTNN_DQ_TSMINB
#define ACTNN_DQ_TSMINB 1
#endif
constexpr int kO = ACTNN_DQ_O;
template <bool kTS>
__host__ __device__ constexpr int warps() { return kTS ? ACTNN_DQ_TSW : kWarps; }
template <bool kTS>
__host__ __device__ constexpr size_t smem_base() {
    return (size_t)warps<kTS>() * kS * kStage + (size_t)warps<kTS>() * kS * 8 + kNCap +
           4 * (kNCap + 1);
}
template <bool kTS>
__host__ __device__ constexpr size_t stg_off() { return (smem_base<kTS>() + 127) / 128 * 128; }
template <typename TO, bool kTS>
__host__ __device__ constexpr size_t smem_bytes() {
    return kTS ? stg_off<kTS>() + (size_t)warps<kTS>() * kO * kU * kG * sizeof(TO)
               : smem_base<kTS>();
}

struct DParams {
    const uint8_t* packed;
    const float* zmin;
    const float* scale;
    const uint32_t* meta;  // NEXT-1 bf16 words (kB16)
    const uint8_t* bits;
    const int64_t* off;
    uint32_t N, D, ng, nb;
    uint32_t step_n, step_j;  // unit stride of a warp: nwarps = step_n * nb + step_j
    void* out;
};

struct GDParams {  // generic kernel
    const uint8_t* packed;
    const float* zmin;
    const float* scale;
    const uint32_t* meta;  // NEXT-1 bf16 words, or null
    const uint8_t* bits;
    const int64_t* off;
    int64_t N, D, ng;
    void* out;
};

#ifndef ACTNN_DQ_MASYNC
#define ACTNN_DQ_MASYNC 1
#endif
// 16-byte cp.async global -> shared (L2 only) whose completion performs one
// arrive on `bar` (.noinc: counted against the barrier's expected arrivals)
__device__ __forceinline__ void cp_async16_mbar(void* dst, const void* src, uint64_t* bar) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// The b bytes of a lane in a staged group segment, as a little-endian integer.
template <int b>
__device__ __forceinline__ uint64_t stage_payload(const uint8_t* seg, int lane) {
    if constexpr (b == 8) {
        return reinterpret_cast<const uint64_t*>(seg)[lane];
    } else if constexpr (b == 4) {
        return reinterpret_cast<const uint32_t*>(seg)[lane];
    } else if constexpr (b == 2) {
        return reinterpret_cast<const uint16_t*>(seg)[lane];
    } else if constexpr (b == 1) {
        return seg[lane];
    } else {
        uint64_t p = 0;
#pragma unroll
        for (int t = 0; t < b; ++t) p |= (uint64_t)seg[lane * b + t] << (8 * t);
        return p;
    }
}

// Exact float(code) as the bit pattern 0x4B000000 | code (= 2^23 + code).
template <int b>
__device__ __forceinline__ uint32_t magic_code(uint64_t pay, int j) {
    if constexpr (b == 8) {
        const uint32_t word = j < 4 ? (uint32_t)pay : (uint32_t)(pay >> 32);
        return __byte_perm(word, 0x4B000000u, 0x7540u | (uint32_t)(j & 3));
    } else {
        return (uint32_t)((pay >> (b * j)) & ((1u << b) - 1u)) | 0x4B000000u;
    }
}

// Shared-memory staging stores of a lane's 8 outputs.  fp32: two 16-byte
// halves, the lanes of each quarter warp alternating which half goes first so
// that every st.shared.v4 covers all 32 banks once; bf16: one 16-byte store.
#ifndef ACTNN_DQ_STS_SWZ
#define ACTNN_DQ_STS_SWZ 1
#endif
__device__ __forceinline__ void sts8(float* p, const float v[8]) {
#if !ACTNN_DQ_STS_SWZ  // plain order: 2-way bank conflicts, no selects
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3])
                 : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p) + 16), "f"(v[4]),
                 "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
    return;
#endif
    const int lane = threadIdx.x & 31;
    const int h = (lane >> 2) & 1;
    const uint32_t a = smem_u32(p);
    const uint32_t a0 = a + 16 * h, a1 = a + 16 * (h ^ 1);
    float f0[4], f1[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // selects, not a dynamically indexed (local) array
        f0[i] = h ? v[4 + i] : v[i];
        f1[i] = h ? v[i] : v[4 + i];
    }
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a0), "f"(f0[0]), "f"(f0[1]),
                 "f"(f0[2]), "f"(f0[3])
                 : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a1), "f"(f1[0]), "f"(f1[1]),
                 "f"(f1[2]), "f"(f1[3])
                 : "memory");
}
__device__ __forceinline__ void sts8(uint16_t* p, const float v[8]) {
    const uint32_t a = pack_bf16x2(v[0], v[1]), b = pack_bf16x2(v[2], v[3]);
    const uint32_t c = pack_bf16x2(v[4], v[5]), d = pack_bf16x2(v[6], v[7]);
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
}

// cp.async.bulk shared -> global (bulk async-group of the issuing thread)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// at most N of this thread's bulk groups still reading shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// One group: the lane's 8 codes -> 8 outputs, one vector store (kSh: into the
// shared staging buffer instead of global memory).
// b = 1 (bf16 outputs): every code is 0 or 1, so the group has two possible outputs,
// fmaf(0, scale, Z) and fmaf(1, scale, Z) (the same single-rounding fma as
// O10, computed once per group); each element selects one by its bit (a
// predicate test + select instead of unpack, int->float and fma).
#ifndef ACTNN_DQ_SEL1
#define ACTNN_DQ_SEL1 1
#endif
template <typename TO, int b, bool kSh = false>
__device__ __forceinline__ void dequant_group(uint64_t pay, float Z, float s, TO* dst) {
    if constexpr (b == 1 && ACTNN_DQ_SEL1 && sizeof(TO) == 2) {  // bf16 outputs: -1.5% (C4);
                                                                 // fp32 outputs: no gain
        const float v0 = __fmaf_rn(0.0f, s, Z), v1 = __fmaf_rn(1.0f, s, Z);
        const uint32_t p8 = (uint32_t)pay;
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = (p8 & (1u << j)) ? v1 : v0;
        if constexpr (kSh)
            sts8(dst, o);
        else
            store8(dst, o);
        return;
    }
    const float2 m23 = make_float2(-8388608.0f, -8388608.0f);
    const float2 zz = make_float2(Z, Z), ss = make_float2(s, s);
    float o[8];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        float2 c = make_float2(__uint_as_float(magic_code<b>(pay, 2 * p)),
                               __uint_as_float(magic_code<b>(pay, 2 * p + 1)));
        c = __fadd2_rn(c, m23);     // exact: (float)code
        c = __ffma2_rn(c, ss, zz);  // code * scale + Z, one rounding
        o[2 * p] = c.x;
        o[2 * p + 1] = c.y;
    }
    if constexpr (kSh)
        sts8(dst, o);
    else
        store8(dst, o);
}

// A unit: zq/sq = the unit's 4 zero points / scales.
template <typename TO, int b, bool kFullUnit, bool kSh = false>
__device__ __forceinline__ void dequant_unit(const uint8_t* st, int gcount, const float (&zq)[kU],
                                             const float (&sq)[kU], TO* dst, int lane) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        if (kFullUnit || u < gcount) {
            const uint64_t pay = stage_payload<b>(st + u * 32 * b, lane);
            dequant_group<TO, b, kSh>(pay, zq[u], sq[u], dst + u * kG + lane * 8);
        }
    }
}

template <typename TO, int b, bool kSh = false>
__device__ __forceinline__ void dequant_unit_any(const uint8_t* st, int gcount,
                                                 const float (&zq)[kU], const float (&sq)[kU],
                                                 TO* dst, int lane) {
    if (gcount == kU)
        dequant_unit<TO, b, true, kSh>(st, gcount, zq, sq, dst, lane);
    else
        dequant_unit<TO, b, false, kSh>(st, gcount, zq, sq, dst, lane);
}

// kCached: (bits, off) of all samples in shared memory (N <= kNCap).
// kMeta: the unit's metadata travels in the stage (ng % 4 == 0).
// kB16: NEXT-1 bf16 metadata words (Z', R'): lane u < 4 widens group u's word
// and computes scale = RN(R' / B) once, the unit's lanes get it by shuffle.
template <typename TO, bool kCached, bool kMeta, bool kB16, bool kTS>
__global__ void __launch_bounds__(warps<kTS>() * 32, kTS ? ACTNN_DQ_TSMINB : ACTNN_DQ_MINB)
    dequantize_fast_kernel(const __grid_constant__ DParams p) {
    pdl_trigger();  // the next kernel of the stream may start launching
    pdl_wait();     // the previous grid is complete and visible
    constexpr int kW = warps<kTS>();
    extern __shared__ __align__(128) uint8_t smem[];
    TO* stg = reinterpret_cast<TO*>(smem + stg_off<kTS>()) + (size_t)(threadIdx.x >> 5) * kO * kU * kG;
    uint32_t ounit = 0;  // units this warp has staged (kTS)
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    uint8_t* ring = smem + (size_t)w * kS * kStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kW * kS * kStage) + w * kS;
    uint8_t* s_bits = smem + (size_t)kW * kS * kStage + (size_t)kW * kS * 8;
    uint32_t* s_off = reinterpret_cast<uint32_t*>(s_bits + kNCap);

    const int64_t off0 = p.off[0];
    if (kCached) {
        for (uint32_t i = threadIdx.x; i < p.N; i += kW * 32) {
            s_bits[i] = p.bits[i];
            s_off[i] = (uint32_t)((p.off[i] - off0) >> 5);
        }
    }
    // kMA (TMA-store path): a unit's 4 zero points and 4 scales come by two
    // 16-byte cp.async (lanes 0 and 1) whose completion arrives on the stage's
    // mbarrier (.noinc: 3 arrivals per phase), instead of two more bulk copies
    // from lane 0 -- each bulk copy costs an ELECT / R2UR loop of ~10
    // instructions per unit.  Measured per fp32 output size: 205 MB -4%, 411 MB
    // -2%, 822 MB even; on the LSU-store path (smaller outputs, bf16) +2% / even,
    // so it is used with the TMA stores only.
    constexpr bool kMA = kMeta && !kB16 && kTS && ACTNN_DQ_MASYNC;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kS; ++s) mbar_init(&bars[s], kMA ? 3 : 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t gw = blockIdx.x * kW + w;
    TO* __restrict__ out = static_cast<TO*>(p.out);
    auto advance = [&](uint32_t& n, uint32_t& j) {
        n += p.step_n;
        j += p.step_j;
        if (j >= p.nb) {
            j -= p.nb;
            ++n;
        }
    };
    auto gcount_of = [&](uint32_t j) { return (int)min((uint32_t)kU, p.ng - j * kU); };
    auto width = [&](uint32_t n) { return kCached ? (int)s_bits[n] : (int)p.bits[n]; };
    // lane 0: bulk copies of unit (pn, pj) into stage s
    auto issue = [&](uint32_t pn, uint32_t pj, int s) {
        int b = width(pn);
        if (b < 1 || b > 8) b = 1;  // outside the contract; keeps the ring's phases consistent
        const int64_t sofs = kCached ? ((int64_t)s_off[pn] << 5) : (p.off[pn] - off0);
        const uint32_t bytes = (uint32_t)(gcount_of(pj) * 32 * b);
        uint8_t* dst = ring + s * kStage;
#ifdef ACTNN_DQ_FAKEREAD  // diagnostics: every unit reads unit (0, 0)'s bytes (L2-resident)
        pn = 0;
        pj = 0;
#endif
        if (kMeta && kB16) {
            const uint32_t g = pn * p.ng + pj * kU;
            mbar_expect_tx(&bars[s], bytes + 4 * kU);
            bulk_g2s(dst + kPay, p.meta + g, 4 * kU, &bars[s]);
        } else if (kMeta && !kMA) {
            const uint32_t g = pn * p.ng + pj * kU;
            mbar_expect_tx(&bars[s], bytes + 8 * kU);
            bulk_g2s(dst + kPay, p.zmin + g, 4 * kU, &bars[s]);
            bulk_g2s(dst + kPay + 4 * kU, p.scale + g, 4 * kU, &bars[s]);
        } else {
            mbar_expect_tx(&bars[s], bytes);
        }
        bulk_g2s(dst, p.packed + sofs + (uint64_t)pj * (kU * 32) * b, bytes, &bars[s]);
    };

    // kMA: lanes 0 / 1 copy the unit's zero points / scales (16 bytes each)
    auto issue_meta = [&](uint32_t pn, uint32_t pj, int s) {
        if (lane < 2) {
            const uint32_t g = pn * p.ng + pj * kU;
            const float* src = (lane == 0 ? p.zmin : p.scale) + g;
            cp_async16_mbar(ring + s * kStage + kPay + 16 * lane, src, &bars[s]);
        }
    };

    uint32_t pn = gw / p.nb, pj = gw % p.nb;
    uint32_t n = pn, j = pj;
#ifndef ACTNN_DQ_STOREONLY
#pragma unroll
    for (int s = 0; s < kS; ++s) {
        if (pn < p.N) {
            if (lane == 0) issue(pn, pj, s);
            if constexpr (kMA) issue_meta(pn, pj, s);
        }
        advance(pn, pj);  // every lane tracks the copy cursor
    }
#endif
    int stage = 0;
    uint32_t phase = 0;
    while (n < p.N) {
        const int gcount = gcount_of(j);
        const int b = width(n);
        TO* dst = out + (uint64_t)n * p.D + (uint64_t)j * (kU * kG);
        const uint8_t* st = ring + stage * kStage;
        const uint32_t g = n * p.ng + j * kU;
#ifdef ACTNN_DQ_STOREONLY  // diagnostics: K4's store pattern alone (no reads, no codes)
        if (true) {
            const float o8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int u = 0; u < gcount_of(j); ++u) store8(reinterpret_cast<float*>(dst) + u * kG + lane * 8, o8);
            advance(n, j);
            continue;
        }
#endif
        mbar_wait(&bars[stage], phase);
#ifdef ACTNN_DQ_NOCOMPUTE  // diagnostics: the TMA ring + stores, no unpack/dequantise
        if (true) {
            const float o8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int u = 0; u < gcount; ++u) store8(reinterpret_cast<float*>(dst) + u * kG + lane * 8, o8);
            __syncwarp();
            if (lane == 0) {
                if (pn < p.N) issue(pn, pj, stage);
                advance(pn, pj);
            }
            if (++stage == kS) {
                stage = 0;
                phase ^= 1u;
            }
            advance(n, j);
            continue;
        }
#endif
        float zq[kU], sq[kU];
        if constexpr (kB16) {
            const uint32_t* wq = kMeta ? reinterpret_cast<const uint32_t*>(st + kPay) : p.meta + g;
            const uint32_t wl = lane < gcount ? wq[lane] : 0u;
            const float zl = meta_zero(wl);
            const float sl = meta_scale(wl, (b >= 1 && b <= 8) ? b : 1);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                zq[u] = __shfl_sync(0xffffffffu, zl, u);
                sq[u] = __shfl_sync(0xffffffffu, sl, u);
            }
        } else {
            if (kMeta && kU == 4) {  // the unit's 4 zero points / scales: two 16-byte loads
                const float4 z4 = *reinterpret_cast<const float4*>(st + kPay);
                const float4 s4 = *reinterpret_cast<const float4*>(st + kPay + 16);
                zq[0] = z4.x; zq[1] = z4.y; zq[2] = z4.z; zq[3] = z4.w;
                sq[0] = s4.x; sq[1] = s4.y; sq[2] = s4.z; sq[3] = s4.w;
            } else {
                const float* zp = kMeta ? reinterpret_cast<const float*>(st + kPay) : p.zmin + g;
                const float* sp = kMeta ? reinterpret_cast<const float*>(st + kPay + 4 * kU) : p.scale + g;
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    zq[u] = u < gcount ? zp[u] : 0.0f;
                    sq[u] = u < gcount ? sp[u] : 0.0f;
                }
            }
        }
        TO* ob = dst;
        if constexpr (kTS) {
            // staging buffer ounit % kO: its previous bulk store must have read it
            ob = stg + (size_t)(ounit % kO) * (kU * kG);
            if (lane == 0) bulk_wait_read<kO - 1>();
            __syncwarp();
        }
        if (b == 2) dequant_unit_any<TO, 2, kTS>(st, gcount, zq, sq, ob, lane);
        else if (b == 1) dequant_unit_any<TO, 1, kTS>(st, gcount, zq, sq, ob, lane);
        else if (b == 4) dequant_unit_any<TO, 4, kTS>(st, gcount, zq, sq, ob, lane);
        else if (b == 8) dequant_unit_any<TO, 8, kTS>(st, gcount, zq, sq, ob, lane);
        else if (b == 3) dequant_unit<TO, 3, false, kTS>(st, gcount, zq, sq, ob, lane);
        else if (b == 5) dequant_unit<TO, 5, false, kTS>(st, gcount, zq, sq, ob, lane);
        else if (b == 6) dequant_unit<TO, 6, false, kTS>(st, gcount, zq, sq, ob, lane);
        else if (b == 7) dequant_unit<TO, 7, false, kTS>(st, gcount, zq, sq, ob, lane);
        // the stage's shared loads were consumed by the stores above: re-arm it
        // (cross-proxy WAR: each lane's generic loads are ordered before the
        // async-proxy bulk write by fence.proxy.async, all lanes before lane 0's
        // issue by the __syncwarp).  kTS: the same fence orders the lanes'
        // staging writes before the async-proxy bulk store that reads them.
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            if constexpr (kTS) bulk_s2g(dst, ob, (uint32_t)(gcount * kG * (int)sizeof(TO)));
            if (pn < p.N) issue(pn, pj, stage);
        }
        if constexpr (kMA) {
            if (pn < p.N) issue_meta(pn, pj, stage);
        }
        advance(pn, pj);
        if constexpr (kTS) ++ounit;  // every lane: they all index the staging ring
        if (++stage == kS) {
            stage = 0;
            phase ^= 1u;
        }
        advance(n, j);
    }
    if constexpr (kTS) {
        if (lane == 0) bulk_wait_all();  // shared memory stays valid until the stores read it
    }
}

// Generic path: ragged last group / unaligned output; one group per warp.
template <typename TO>
__global__ void __launch_bounds__(kBlock) dequantize_generic_kernel(const __grid_constant__ GDParams p) {
    pdl_trigger();  // the next kernel of the stream may start launching
    pdl_wait();     // the previous grid is complete and visible
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
        float Z, s;
        if (p.meta) {
            const uint32_t w = __ldg(p.meta + g);
            Z = meta_zero(w);
            s = meta_scale(w, b);
        } else {
            Z = __ldg(p.zmin + g);
            s = __ldg(p.scale + g);
        }
        const uint32_t mask = (1u << b) - 1u;
        TO* dst = out + n * p.D + i * kG;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int idx = lane * 8 + jj;
            if (idx < len) store1(dst + idx, dequant1((uint32_t)(pay >> (b * jj)) & mask, s, Z));
        }
    }
}

template <typename TO, bool kCached, bool kMeta, bool kB16, bool kTS>
void launch_fast_t(const DParams& p0, int64_t units, cudaStream_t s) {
    constexpr size_t kSmem = smem_bytes<TO, kTS>();
    const void* k = (const void*)dequantize_fast_kernel<TO, kCached, kMeta, kB16, kTS>;
    ensure_smem_attr(k, kSmem);  // opt-in above 48 KB of dynamic smem
    DParams p = p0;
    constexpr int kW = warps<kTS>();
    const int grid = grid_for(k, kW * 32, kSmem, (units + kW - 1) / kW);
    const uint32_t nwarps = (uint32_t)grid * kW;
    p.step_n = nwarps / p.nb;
    p.step_j = nwarps % p.nb;
    launch_pdl(dequantize_fast_kernel<TO, kCached, kMeta, kB16, kTS>, grid, kW * 32, kSmem, s, p);
}

template <typename TO, bool kCached, bool kMeta, bool kB16>
void launch_fast(const DParams& p, int64_t units, cudaStream_t s) {
    const bool ts = ACTNN_DQ_TS == 1 ||
                    (ACTNN_DQ_TS == 2 && sizeof(TO) == 4 &&
                     (int64_t)p.N * p.D * (int64_t)sizeof(TO) >= (int64_t)ACTNN_DQ_TS_MIN_MB << 20);
    if (ts)
        launch_fast_t<TO, kCached, kMeta, kB16, true>(p, units, s);
    else
        launch_fast_t<TO, kCached, kMeta, kB16, false>(p, units, s);
}

template <typename TO>
cudaError_t run(const DequantArgs& a, cudaStream_t s) {
    const int64_t nb = (a.ng + kU - 1) / kU;
    const bool fits = a.N * a.ng < (1ll << 31) && a.D < (1ll << 31);
    if (a.fast && fits) {
        DParams p;
        p.packed = a.packed;
        p.zmin = a.zmin;
        p.scale = a.scale;
        p.meta = a.meta;
        p.bits = a.bits;
        p.off = a.off;
        p.N = (uint32_t)a.N;
        p.D = (uint32_t)a.D;
        p.ng = (uint32_t)a.ng;
        p.nb = (uint32_t)nb;
        p.step_n = p.step_j = 0;
        p.out = a.out;
        const bool cached = a.N <= kNCap;
        // metadata by TMA: every unit's 4 floats / words start 16-byte aligned
        const bool b16 = a.meta != nullptr;
        const bool meta = (a.ng % kU == 0) &&
                          (b16 ? (uintptr_t)a.meta % 16 == 0
                               : ((uintptr_t)a.zmin % 16 == 0) && ((uintptr_t)a.scale % 16 == 0));
        const int64_t units = a.N * nb;
        if (b16) {
            if (cached && meta) launch_fast<TO, true, true, true>(p, units, s);
            else if (cached) launch_fast<TO, true, false, true>(p, units, s);
            else if (meta) launch_fast<TO, false, true, true>(p, units, s);
            else launch_fast<TO, false, false, true>(p, units, s);
        } else {
            if (cached && meta) launch_fast<TO, true, true, false>(p, units, s);
            else if (cached) launch_fast<TO, true, false, false>(p, units, s);
            else if (meta) launch_fast<TO, false, true, false>(p, units, s);
            else launch_fast<TO, false, false, false>(p, units, s);
        }
    } else {
        GDParams p{a.packed, a.zmin, a.scale, a.meta, a.bits, a.off, a.N, a.D, a.ng, a.out};
        const int grid = grid_for((const void*)dequantize_generic_kernel<TO>, kBlock, 0,
                                  (a.N * a.ng + kWarps - 1) / kWarps);
        launch_pdl(dequantize_generic_kernel<TO>, grid, kBlock, 0, s, p);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dequantize(const DequantArgs& a, cudaStream_t s) {
    return a.out_dt == 0 ? run<float>(a, s) : run<uint16_t>(a, s);
}

}  // namespace actnn
