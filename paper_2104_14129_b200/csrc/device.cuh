// device.cuh -- sm_100a building blocks shared by the ActNN kernels.
//
// Independent of oracle/ (no shared code).  Floating-point steps use explicit
// round-to-nearest intrinsics and the library is compiled with -fmad=false and
// without -ftz / fast-math so that every rounding is the one ACTNN-Q v1 fixes.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace actnn {

#ifndef ACTNN_REDUX_F32
#define ACTNN_REDUX_F32 1
#endif

constexpr int kG = 256;            // group size ("we set G = 256")

// ------------------------------------------- programmatic dependent launch
// The hot-path kernels are launched with programmatic stream serialization
// (launch.h launch_pdl): each CTA first lets the next kernel of its stream
// start launching (its CTAs take SM slots as this grid's CTAs retire, so the
// launch latency and its prologue overlap this grid's tail), and waits for the
// previous grid to complete -- with all its memory operations visible -- before
// its own first global memory access.  Without the launch attribute both are
// no-ops.
#ifndef ACTNN_PDL
#define ACTNN_PDL 1
#endif
__device__ __forceinline__ void pdl_trigger() {
#if ACTNN_PDL
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if ACTNN_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
constexpr int kWarp = 32;
constexpr int kElemsPerLane = 8;   // kG / kWarp: one Philox call per lane per group
constexpr int kChunk = 32;         // groups per tile = one group per lane for metadata

// -------------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11): multipliers 0xD2511F53 / 0xCD9E8D57,
// Weyl key increments 0x9E3779B9 / 0xBB67AE85, key bumped between rounds.
// The counter words 2,3 are always 0 in ACTNN-Q v1 (ctr = e >> 3 is 64-bit).
// The key depends only on the seed, so ptxas keeps the round keys in uniform
// registers; each round is 2 IMAD.WIDE.U32 + 2 LOP3.
struct Philox4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t k0,
                                                 uint32_t k1) {
    uint32_t c2 = 0u, c3 = 0u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c0;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return Philox4{c0, c1, c2, c3};
}

// Philox with precomputed round keys: rk.k[2r], rk.k[2r+1] are the keys of
// round r.  Passed inside the kernel parameter struct, each key is a
// constant-bank operand of the round's 3-input XOR (LOP3), so a round is
// exactly 2 IMAD.WIDE.U32 + 2 LOP3 and no register holds a key.
struct RoundKeys {
    uint32_t k[20];
};

inline RoundKeys make_round_keys(uint64_t seed) {
    RoundKeys rk;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        rk.k[2 * r] = k0;
        rk.k[2 * r + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return rk;
}

// 32 x 32 -> 64-bit product as one IMAD.WIDE.U32 (4 FMA-heavy cycles; the
// separate IMAD.HI + IMAD form ptxas sometimes picks costs 6).
__device__ __forceinline__ void mulwide(uint32_t a, uint32_t m, uint32_t& hi, uint32_t& lo) {
    uint64_t p;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(m));
    lo = (uint32_t)p;
    hi = (uint32_t)(p >> 32);
}

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, const RoundKeys& rk) {
    // round 0 with c2 = c3 = 0: the second product is 0
    uint32_t hi0, lo0, hi1, lo1;
    mulwide(c0, 0xD2511F53u, hi0, lo0);
    uint32_t n0 = c1 ^ rk.k[0];
    uint32_t n2 = hi0 ^ rk.k[1];
    c0 = n0;
    c1 = 0u;
    uint32_t c2 = n2, c3 = lo0;
#pragma unroll
    for (int r = 1; r < 10; ++r) {
        mulwide(c0, 0xD2511F53u, hi0, lo0);
        mulwide(c2, 0xCD9E8D57u, hi1, lo1);
        n0 = hi1 ^ c1 ^ rk.k[2 * r];
        n2 = hi0 ^ c3 ^ rk.k[2 * r + 1];
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return Philox4{c0, c1, c2, c3};
}

// Philox4x32-10 for a counter whose high word is 0 (every tensor below 2^35
// elements, checked by the launchers): round 0 leaves c0 = k0 for every lane,
// so round 1's first product M0 * k0 is the same for all threads -- ptxas
// computes it once in the uniform datapath -- and each call costs 18 instead of
// 19 per-thread IMAD.WIDE.  Same outputs as philox4x32_10(c0, 0, rk).
__device__ __forceinline__ Philox4 philox4x32_10_c32(uint32_t c0, const RoundKeys& rk) {
    uint32_t hi0, lo0, hi1, lo1;
    mulwide(c0, 0xD2511F53u, hi0, lo0);  // round 0 (c1 = c2 = c3 = 0)
    const uint32_t x2 = hi0 ^ rk.k[1], x3 = lo0;
    uint32_t ahi, alo;
    mulwide(rk.k[0], 0xD2511F53u, ahi, alo);  // round 1, first product: uniform
    mulwide(x2, 0xCD9E8D57u, hi1, lo1);
    uint32_t a0 = hi1 ^ rk.k[2];
    uint32_t a1 = lo1;
    uint32_t a2 = ahi ^ x3 ^ rk.k[3];
    uint32_t a3 = alo;
#pragma unroll
    for (int r = 2; r < 10; ++r) {
        mulwide(a0, 0xD2511F53u, hi0, lo0);
        mulwide(a2, 0xCD9E8D57u, hi1, lo1);
        const uint32_t n0 = hi1 ^ a1 ^ rk.k[2 * r];
        const uint32_t n2 = hi0 ^ a3 ^ rk.k[2 * r + 1];
        a0 = n0;
        a1 = lo1;
        a2 = n2;
        a3 = lo0;
    }
    return Philox4{a0, a1, a2, a3};
}

// 14-bit draw of element j (0..7) of an 8-element Philox block: 16-bit lane j.
__device__ __forceinline__ uint32_t rnd14(const Philox4& o, int j) {
    const uint32_t w = (j >> 1) == 0 ? o.x : (j >> 1) == 1 ? o.y : (j >> 1) == 2 ? o.z : o.w;
    return ((j & 1) ? (w >> 16) : w) & 0x3FFFu;
}

// ------------------------------------------------------------- warp helpers
// per-half min / max of two bf16x2 words
__device__ __forceinline__ uint32_t bmin2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// Group (min, max) of 8 bf16 values per lane (four bf16x2 words) over the
// warp: min and -max travel as one bf16x2 pair through the butterfly (both
// exact on bf16 values); returns them widened to fp32.
__device__ __forceinline__ float warp_min(float v);
__device__ __forceinline__ float warp_max(float v);
__device__ __forceinline__ void warp_minmax_bf16(uint4 w, float& mn, float& mx) {
    const uint32_t mn2 = bmin2(bmin2(w.x, w.y), bmin2(w.z, w.w));
    const uint32_t mx2 = bmax2(bmax2(w.x, w.y), bmax2(w.z, w.w));
#if ACTNN_REDUX_F32
    // the lane's min / max widened (exact), then one warp reduction each
    mn = warp_min(fminf(__uint_as_float(mn2 << 16), __uint_as_float(mn2 & 0xFFFF0000u)));
    mx = warp_max(fmaxf(__uint_as_float(mx2 << 16), __uint_as_float(mx2 & 0xFFFF0000u)));
    return;
#endif
    const uint32_t nmx2 = mx2 ^ 0x80008000u;  // -max, exact
    uint32_t r = bmin2(__byte_perm(mn2, nmx2, 0x5410), __byte_perm(mn2, nmx2, 0x7632));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) r = bmin2(r, __shfl_xor_sync(0xffffffffu, r, o));
    mn = __uint_as_float(r << 16);
    mx = __uint_as_float((r & 0xFFFF0000u) ^ 0x80000000u);
}

// Warp-wide min / max of fp32 values (exact selections; signed zeros are
// canonicalised by the callers).  sm_100a has a one-instruction warp reduction
// for f32 min/max (redux.sync -> CREDUX, result in a uniform register) in place
// of five shuffle + compare steps.
__device__ __forceinline__ float warp_min(float v) {
#if ACTNN_REDUX_F32
    float r;
    asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
#else
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
#endif
}
__device__ __forceinline__ float warp_max(float v) {
#if ACTNN_REDUX_F32
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
#else
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
#endif
}

// ---------------------------------------------------------------- loads
// 8 consecutive elements (32 B fp32 / 16 B bf16) of a lane, widened to fp32.
// fp32 uses the sm_100 256-bit load (LDG.E.256): one instruction moves a
// lane's whole 8-element slice, so every warp load covers 1 KB = 32 full
// sectors.  .nc: read-only path; L1::no_allocate: streamed once per kernel
// (L2 keeps the default policy so the mixed path's second pass can hit L2).
struct F32Tag {};
struct BF16Tag {};

__device__ __forceinline__ void load8(const float* p, float v[8]) {
    asm volatile(
        "ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
          "=f"(v[7])
        : "l"(p));
}

__device__ __forceinline__ void load8(const uint16_t* p, float v[8]) {
    uint32_t a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(p));
    // bf16 -> fp32 is exact: the bf16 bits are the high half of the fp32 bits
    v[0] = __uint_as_float(__byte_perm(a, 0u, 0x1044));
    v[1] = __uint_as_float(a & 0xFFFF0000u);
    v[2] = __uint_as_float(__byte_perm(b, 0u, 0x1044));
    v[3] = __uint_as_float(b & 0xFFFF0000u);
    v[4] = __uint_as_float(__byte_perm(c, 0u, 0x1044));
    v[5] = __uint_as_float(c & 0xFFFF0000u);
    v[6] = __uint_as_float(__byte_perm(d, 0u, 0x1044));
    v[7] = __uint_as_float(d & 0xFFFF0000u);
}

// A lane's 8 elements of a group as raw words (no widening): fp32 one 256-bit
// load into r[0..1], bf16 one 128-bit load into r[0].
__device__ __forceinline__ void ldg_raw8(const float* p, uint4 (&r)[2]) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0].x), "=r"(r[0].y), "=r"(r[0].z), "=r"(r[0].w), "=r"(r[1].x),
                   "=r"(r[1].y), "=r"(r[1].z), "=r"(r[1].w)
                 : "l"(p));
}
__device__ __forceinline__ void ldg_raw8(const uint16_t* p, uint4 (&r)[2]) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0].x), "=r"(r[0].y), "=r"(r[0].z), "=r"(r[0].w)
                 : "l"(p));
}
// ... and widened to fp32 (bf16 -> fp32 is exact)
template <typename T>
__device__ __forceinline__ void raw8_f32(const uint4 (&r)[2], float v[8]) {
    if constexpr (sizeof(T) == 4) {
        v[0] = __uint_as_float(r[0].x); v[1] = __uint_as_float(r[0].y);
        v[2] = __uint_as_float(r[0].z); v[3] = __uint_as_float(r[0].w);
        v[4] = __uint_as_float(r[1].x); v[5] = __uint_as_float(r[1].y);
        v[6] = __uint_as_float(r[1].z); v[7] = __uint_as_float(r[1].w);
    } else {
        v[0] = __uint_as_float(__byte_perm(r[0].x, 0u, 0x1044));
        v[1] = __uint_as_float(r[0].x & 0xFFFF0000u);
        v[2] = __uint_as_float(__byte_perm(r[0].y, 0u, 0x1044));
        v[3] = __uint_as_float(r[0].y & 0xFFFF0000u);
        v[4] = __uint_as_float(__byte_perm(r[0].z, 0u, 0x1044));
        v[5] = __uint_as_float(r[0].z & 0xFFFF0000u);
        v[6] = __uint_as_float(__byte_perm(r[0].w, 0u, 0x1044));
        v[7] = __uint_as_float(r[0].w & 0xFFFF0000u);
    }
}

__device__ __forceinline__ float load1(const float* p) { return __ldg(p); }
__device__ __forceinline__ float load1(const uint16_t* p) {
    return __uint_as_float((uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p)) << 16);
}

// ---------------------------------------------------------------- stores
__device__ __forceinline__ void store8(float* p, const float v[8]) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

// RNE fp32 -> bf16 pair (cvt.rn.bf16x2.f32); low half = first element.
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ void store8(uint16_t* p, const float v[8]) {
    const uint32_t a = pack_bf16x2(v[0], v[1]);
    const uint32_t b = pack_bf16x2(v[2], v[3]);
    const uint32_t c = pack_bf16x2(v[4], v[5]);
    const uint32_t d = pack_bf16x2(v[6], v[7]);
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}

__device__ __forceinline__ void store1(float* p, float v) { *p = v; }
__device__ __forceinline__ void store1(uint16_t* p, float v) {
    *p = (uint16_t)(pack_bf16x2(v, 0.0f) & 0xFFFFu);
}

// ------------------------------------------------------ quantiser constants
// ACTNN-Q v1 O3-O4 for one group from its exact min/max:
// Z, M canonical (+0 for signed zeros), R = RN(M - Z), scale = RN(R / B),
// inv14 = RN(B / R) * 2^14 (0 for the degenerate R < 2^-96).
struct GroupConst {
    float Z, scale, inv14;
};

__device__ __forceinline__ GroupConst group_const(float mn, float mx, int b) {
    GroupConst c;
    const float Z = __fadd_rn(mn, 0.0f);
    const float M = __fadd_rn(mx, 0.0f);
    const float R = __fsub_rn(M, Z);
    const float Bf = (float)((1u << b) - 1u);
    c.Z = Z;
    c.scale = __fdiv_rn(R, Bf);
    c.inv14 = (R < 0x1p-96f) ? 0.0f : __fmul_rn(__fdiv_rn(Bf, R), 16384.0f);
    return c;
}

// NEXT-1, bf16 metadata ("stored and used values identical";
// DESIGN reading 21): Z' = bf16 toward -inf of Z, R' = bf16 toward +inf of
// RU(M - Z'); the word holds Z' (bits 0-15) and R' (bits 16-31), and the
// quantiser runs O4-O8 on (float(Z'), float(R')).  bf16 = the high half of an
// fp32, whose bit pattern is monotone in magnitude for a fixed sign.
struct GroupConstB {
    float Z, inv14;
    uint32_t word;
};

__device__ __forceinline__ GroupConstB group_const_bf16(float mn, float mx, int b) {
    const float Z = __fadd_rn(mn, 0.0f);
    const float M = __fadd_rn(mx, 0.0f);
    const uint32_t zu = __float_as_uint(Z);
    const uint32_t zb = (zu >> 16) + (((zu & 0xFFFFu) != 0u) & (zu >> 31));  // toward -inf
    const float Zp = __uint_as_float(zb << 16);
    const uint32_t tu = __float_as_uint(__fsub_ru(M, Zp));                    // >= +0
    const uint32_t rb = (tu >> 16) + ((tu & 0xFFFFu) != 0u);                  // toward +inf
    const float Rp = __uint_as_float(rb << 16);
    const float Bf = (float)((1u << b) - 1u);
    GroupConstB c;
    c.Z = Zp;
    c.inv14 = (Rp < 0x1p-96f) ? 0.0f : __fmul_rn(__fdiv_rn(Bf, Rp), 16384.0f);
    c.word = (zb & 0xFFFFu) | (rb << 16);
    return c;
}

// The dequantiser's (Z, scale) from a bf16 metadata word: float(Z'),
// RN(float(R') / B) (O10 with the stored values).
__device__ __forceinline__ float meta_zero(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float meta_scale(uint32_t w, int b) {
    return __fdiv_rn(__uint_as_float(w & 0xFFFF0000u), (float)((1u << b) - 1u));
}

// ACTNN-Q v1 O5 + O7: q = RNE((h - Z) * inv14) as an integer in [0, B*2^14],
// obtained exactly from one fma against 1.5*2^23 (the sum stays in
// [2^23, 2^24) where the ulp is 1; the constant is even so ties agree with
// RNE), then code = (q + r) >> 14 (stochastic rounding).
__device__ __forceinline__ uint32_t sr_code(float h, float Z, float inv14, uint32_t r14) {
    const float d = __fsub_rn(h, Z);
    const float t = __fmaf_rn(d, inv14, 12582912.0f);
    return (__float_as_uint(t) - 0x4B400000u + r14) >> 14;
}

// Codes of one lane's 8 elements at b <= 2 (ACTNN-Q v1 O5-O7), two elements
// per 32-bit register: t = RN(d * inv14 + 1.5 2^23) holds q = RNE(d * inv14)
// < 2^16 in its low half (the magic's low 16 bits are zero), so one byte
// permute gives T = q_y << 16 | q_x; adding the two 14-bit draws
// (w & 0x3FFF3FFF) cannot carry across halves (q + r < (B + 1) 2^14 <= 2^16),
// and bits 14.. of each half are the codes.  The codes are moved to their
// packed positions (element j at bits [j b, (j + 1) b)) with shifts and masks
// on the ALU pipe -- no multiply, since the FMA-heavy pipe is the one the
// Philox IMAD.WIDEs saturate.
//
// ACTNN_PACK_MUL=1 (default) gathers the codes with byte permutes and one
// multiply instead of a shift + mask per register pair (4-6 fewer ALU
// instructions per group; on sm_100 the ALU instructions and the Philox
// IMAD.WIDEs add up rather than overlap, tools/cuda_checks/k3_mix.cu):
//   b = 1: the fma uses the magic 1.5 2^23 + 2^14 (still even, so ties are
//   unchanged), so each half holds q + r + 2^14 < 2^16 and its bit 15 (the
//   byte's sign bit) is the code [q + r >= 2^14].  A sign-replicating byte
//   permute turns the four codes of two registers into 0x00 / 0xFF bytes;
//   element j keeps bit j (j < 4 from the first permute, j >= 4 from the
//   second), and one multiply by 0x01010101 ORs the four disjoint bytes into
//   the top byte.
//   b = 2: a byte permute collects bits 14-15 / 30-31 of two registers as
//   bits 6-7 of four bytes (element k at 6 + 8k); times 1 + 2^6 + 2^12 + 2^18
//   moves element k to bits 24 + 2k (every other partial product lands in a
//   disjoint 2-bit field below bit 24 or above bit 31, so nothing carries);
//   a final permute joins the two top bytes.
#ifndef ACTNN_PACK_MUL
#define ACTNN_PACK_MUL 1
#endif
// prmt with sign-replicating selector nibbles (bit 3 of a nibble set: the
// selected byte's sign bit fills the output byte).  __byte_perm ignores that
// bit (CUDA masks each selector nibble to 3 bits), hence the inline PTX.
__device__ __forceinline__ uint32_t prmt_sign(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
template <int b>
__device__ __forceinline__ uint32_t codes_small_d(const float d[8], float inv14, const Philox4& o) {
    // scalar FFMA: measured ~6% faster per group than the f32x2 forms
    // (tools/cuda_checks/k3_compute.cu), which also compete with the Philox
    // IMAD.WIDEs for the FMA-heavy pipe
    const uint32_t w[4] = {o.x, o.y, o.z, o.w};
#if ACTNN_PACK_MUL
    uint32_t T[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float magic = b == 1 ? 12599296.0f : 12582912.0f;  // 1.5 2^23 (+ 2^14)
        const float tx = __fmaf_rn(d[2 * p], inv14, magic);
        const float ty = __fmaf_rn(d[2 * p + 1], inv14, magic);
        T[p] = __byte_perm(__float_as_uint(tx), __float_as_uint(ty), 0x5410) +
               (w[p] & 0x3FFF3FFFu);
    }
    if (b == 1) {
        const uint32_t A = prmt_sign(T[0], T[1], 0xFDB9);  // elements 0-3: 0x00 / 0xFF
        const uint32_t B = prmt_sign(T[2], T[3], 0xFDB9);  // elements 4-7
        const uint32_t X = ((A & 0x0F0F0F0Fu) | (B & 0xF0F0F0F0u)) & 0x88442211u;
        return (X * 0x01010101u) >> 24;
    }
    const uint32_t A = __byte_perm(T[0], T[1], 0x7531) & 0xC0C0C0C0u;
    const uint32_t B = __byte_perm(T[2], T[3], 0x7531) & 0xC0C0C0C0u;
    return __byte_perm(A * 0x00041041u, B * 0x00041041u, 0x0073) & 0xFFFFu;
#else
    uint32_t y = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float tx = __fmaf_rn(d[2 * p], inv14, 12582912.0f);
        const float ty = __fmaf_rn(d[2 * p + 1], inv14, 12582912.0f);
        uint32_t T = __byte_perm(__float_as_uint(tx), __float_as_uint(ty), 0x5410);
        T += w[p] & 0x3FFF3FFFu;
        if (b == 2)  // half 0 code -> bits 4p.., half 1 code -> bits 16 + 4p..
            y |= (T >> (14 - 4 * p)) & (0xC000C000u >> (14 - 4 * p));
        else  // half 0 code -> bit 2p, half 1 code -> bit 16 + 2p
            y |= (T >> (14 - 2 * p)) & (0x40004000u >> (14 - 2 * p));
    }
    if (b == 2) return (y | (y >> 14)) & 0xFFFFu;
    return (y | (y >> 15)) & 0xFFu;
#endif
}

// delta_j = RN(h_j - Z) (ACTNN-Q v1 O5) of a lane's 8 elements.
// fp32: one FADD each.  bf16, from the raw bf16x2 words: the sm_100
// mixed-precision subtract (sub.rn.f32.bf16 -> SASS FHADD.BF16, the bf16
// operand taken from either register half) -- the bf16 value is exact in fp32
// and the difference is rounded once, exactly as RN(float(h) - Z), with no
// instruction spent on widening.
__device__ __forceinline__ void deltas8(const float v[8], float Z, float d[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = __fsub_rn(v[j], Z);
}
__device__ __forceinline__ void sub_bf16x2(uint32_t w, float Z, float& d0, float& d1) {
    asm("{\n.reg .b16 lo, hi;\nmov.b32 {lo, hi}, %2;\nsub.rn.f32.bf16 %0, lo, %3;\n"
        "sub.rn.f32.bf16 %1, hi, %3;\n}\n"
        : "=f"(d0), "=f"(d1)
        : "r"(w), "f"(Z));
}
__device__ __forceinline__ void deltas8(const uint4& raw, float Z, float d[8]) {
    sub_bf16x2(raw.x, Z, d[0], d[1]);
    sub_bf16x2(raw.y, Z, d[2], d[3]);
    sub_bf16x2(raw.z, Z, d[4], d[5]);
    sub_bf16x2(raw.w, Z, d[6], d[7]);
}

// A lane's 8 elements as the consumer holds them: 8 widened fp32 values, or
// (bf16 input) the 4 raw bf16x2 words of its 16-byte slice.
struct F8 {
    float v[8];
};
template <typename T>
struct LaneIn;
template <>
struct LaneIn<float> {
    using type = F8;
};
template <>
struct LaneIn<uint16_t> {
    using type = uint4;
};
__device__ __forceinline__ void deltas8(const F8& x, float Z, float d[8]) { deltas8(x.v, Z, d); }

// A lane's 8 elements of a group from a shared-memory stage.
__device__ __forceinline__ void lds8(const float* p, float v[8]);
__device__ __forceinline__ void lane_load(const float* p, F8& x) { lds8(p, x.v); }
__device__ __forceinline__ void lane_load(const uint16_t* p, uint4& x) {
    x = *reinterpret_cast<const uint4*>(p);
}

// The lane's min / max of its 8 elements (exact selections; fp32 widened,
// bf16 on packed bf16x2 halves, then widened exactly).
__device__ __forceinline__ void lane_minmax(const F8& x, float& mn, float& mx) {
    mn = x.v[0];
    mx = x.v[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) {
        mn = fminf(mn, x.v[j]);
        mx = fmaxf(mx, x.v[j]);
    }
}
__device__ __forceinline__ uint32_t bmin2(uint32_t a, uint32_t b);
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b);
__device__ __forceinline__ void lane_minmax(const uint4& w, float& mn, float& mx) {
    const uint32_t mn2 = bmin2(bmin2(w.x, w.y), bmin2(w.z, w.w));
    const uint32_t mx2 = bmax2(bmax2(w.x, w.y), bmax2(w.z, w.w));
    mn = fminf(__uint_as_float(mn2 << 16), __uint_as_float(mn2 & 0xFFFF0000u));
    mx = fmaxf(__uint_as_float(mx2 << 16), __uint_as_float(mx2 & 0xFFFF0000u));
}

template <int b, typename In>
__device__ __forceinline__ uint32_t codes_small(const In& x, float Z, float inv14,
                                                const Philox4& o) {
    float d[8];
    deltas8(x, Z, d);
    return codes_small_d<b>(d, inv14, o);
}

// Codes of one lane's 8 elements at b >= 3 (q up to 2^22, one code per
// element; ACTNN-Q v1 O5-O7), from the deltas.  ACTNN_WIDE_F32X2=1 forms the
// fma against 1.5*2^23 two elements at a time with the sm_100 f32x2 FFMA2
// (the same IEEE rounding per element as the scalar form).
#ifndef ACTNN_WIDE_F32X2
#define ACTNN_WIDE_F32X2 0
#endif
__device__ __forceinline__ void codes_wide_d(const float d[8], float inv14, const Philox4& o,
                                             uint32_t code[8]) {
    const uint32_t w[4] = {o.x, o.y, o.z, o.w};
#if ACTNN_WIDE_F32X2
    const float2 iv = make_float2(inv14, inv14), mg = make_float2(12582912.0f, 12582912.0f);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float2 t = __ffma2_rn(make_float2(d[2 * p], d[2 * p + 1]), iv, mg);
        // the halves' bit patterns through an opaque move: with a plain
        // __float_as_uint, NVVM (CUDA 12.9) drops the shift that later places the
        // .x half's code into the packed word (tools/cuda_checks/f32x2_miscompile.cu)
        uint32_t tx, ty;
        asm("mov.b32 %0, %1;" : "=r"(tx) : "f"(t.x));
        asm("mov.b32 %0, %1;" : "=r"(ty) : "f"(t.y));
        code[2 * p] = (tx - 0x4B400000u + (w[p] & 0x3FFFu)) >> 14;
        code[2 * p + 1] = (ty - 0x4B400000u + ((w[p] >> 16) & 0x3FFFu)) >> 14;
    }
#else
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t r = ((j & 1) ? (w[j >> 1] >> 16) : w[j >> 1]) & 0x3FFFu;
        const float t = __fmaf_rn(d[j], inv14, 12582912.0f);
        code[j] = (__float_as_uint(t) - 0x4B400000u + r) >> 14;
    }
#endif
}

template <typename In>
__device__ __forceinline__ void codes_wide(const In& x, float Z, float inv14, const Philox4& o,
                                           uint32_t code[8]) {
    float d[8];
    deltas8(x, Z, d);
    codes_wide_d(d, inv14, o, code);
}

// ACTNN-Q v1 O10: h_hat = fmaf((float)code, scale, Z); (float)code is exact
// via the 2^23 magic (code < 2^8).
__device__ __forceinline__ float dequant1(uint32_t code, float scale, float Z) {
    const float c = __fsub_rn(__uint_as_float(0x4B000000u | code), 8388608.0f);
    return __fmaf_rn(c, scale, Z);
}

// --------------------------------------------------- bulk async copies (TMA)
// cp.async.bulk (the non-tensor TMA path, SASS UBLKCP) moves a contiguous
// global range into shared memory and completes on an mbarrier with a byte
// count (complete_tx).  Each warp of K3/K4 owns a ring of such stages: lane 0
// issues the copy S units ahead and the warp waits on the stage's barrier, so
// the data in flight lives in shared memory instead of registers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Wait with a suspend-time hint: the thread sleeps until the phase completes
// (or the hint, in ns, expires) instead of re-polling, so waiting warps do not
// take issue slots from the working ones.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity,
                                                uint32_t hint_ns = 100000u) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(hint_ns)
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// S_n = ((0 + T[0][n]) + T[1][n]) + ... in chunk order (the O11 order), with
// 16 chunk partials in flight per step: the last-CTA tail of K1 / K6 is a
// dependent chain of L2 loads otherwise (98 chunks on the 822 MB tensors).
__device__ __forceinline__ double sum_chunks_in_order(const double* T, int64_t nch, int64_t N,
                                                      int64_t n) {
    double s = 0.0;
    int64_t c = 0;
    for (; c + 16 <= nch; c += 16) {
        double t[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) t[i] = __ldcg(T + (c + i) * N + n);
#pragma unroll
        for (int i = 0; i < 16; ++i) s = __dadd_rn(s, t[i]);
    }
    for (; c < nch; ++c) s = __dadd_rn(s, __ldcg(T + c * N + n));
    return s;
}

// 8 fp32 (two 16-byte shared loads) / 8 bf16 (one) of a lane from a stage.
__device__ __forceinline__ void lds8(const float* p, float v[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0];
    const float4 b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

__device__ __forceinline__ void lds8(const uint16_t* p, float v[8]) {
    const uint4 a = *reinterpret_cast<const uint4*>(p);
    // bits << 16 as a byte permute (ALU pipe, not an IMAD shift)
    v[0] = __uint_as_float(__byte_perm(a.x, 0u, 0x1044));
    v[1] = __uint_as_float(a.x & 0xFFFF0000u);
    v[2] = __uint_as_float(__byte_perm(a.y, 0u, 0x1044));
    v[3] = __uint_as_float(a.y & 0xFFFF0000u);
    v[4] = __uint_as_float(__byte_perm(a.z, 0u, 0x1044));
    v[5] = __uint_as_float(a.z & 0xFFFF0000u);
    v[6] = __uint_as_float(__byte_perm(a.w, 0u, 0x1044));
    v[7] = __uint_as_float(a.w & 0xFFFF0000u);
}

}  // namespace actnn
