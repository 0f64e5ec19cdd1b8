// contexts.cu -- NEXT-4: the lossless contexts of a Conv-BN-ReLU-MaxPool block.
//
// ReLU (App. B.3): "ReLU layers only take a single bit per
// dimension to store, without any approximation."  Pack: bit k of the
// LSB-first mask stream = (x_k > 0), optionally with the forward output
// y = ReLU(x) (+0 for non-positive inputs) from the same read.  Backward:
// grad_x = grad_y where the bit is set, +0 elsewhere.  Both are pure streams:
// a warp step moves 4 KB of activations with four fully coalesced 256-bit
// loads (lane l, load i: bytes [1024 i + 32 l, +32)), so the mask bytes of
// load i are bytes (32 i + l) * V/8 .. of the stream (V elements per load).
//
// Max pooling (App. B.4): "For each output location y_nij, we
// need to store an integer value k_nij = argmax ... We use 8 bits per output
// location."  Forward: thread per output, window max and first argmax tap
// (row-major a * kw + b); for the ResNet stem (3x3, stride 2, pad 1, W a
// multiple of 8 / 16) one thread per run of 4 (fp32) / 8 (bf16) outputs with
// vector loads (maxpool_fwd_k3s2_vec); the backward likewise by runs
// (maxpool_bwd_k3s2_vec), the row-sliding / per-block kernels being the
// fallbacks for other widths.  Backward: thread per input element, a gather over
// the windows that contain it in increasing output order (no atomics, so the
// fp32 sum order is fixed and equals the oracle's / PyTorch CPU's).
#include <algorithm>
#include <cstdlib>

#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

constexpr int kBlock = 256;
#ifndef ACTNN_POOL_K32  // outputs per thread of the vector k3s2 forward (fp32 / bf16);
#define ACTNN_POOL_K32 4  // 8 measured 15% slower for fp32, 4 for bf16 18% slower
#endif
#ifndef ACTNN_POOL_K16
#define ACTNN_POOL_K16 8
#endif

template <typename T>
struct RV;  // elements per 256-bit access
template <>
struct RV<float> {
    static constexpr int V = 8;
};
template <>
struct RV<uint16_t> {
    static constexpr int V = 16;
};

__device__ __forceinline__ float widen1(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float widen1(const uint16_t* p, int64_t i) {
    return __uint_as_float((uint32_t)p[i] << 16);
}

// 256-bit load / store of raw words (no conversion needed: ReLU only tests the
// sign and copies or zeroes)
__device__ __forceinline__ void ldg256(const void* p, uint32_t (&w)[8]) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                   "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}
__device__ __forceinline__ void stg256(void* p, const uint32_t (&w)[8]) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]),
                 "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
}

// positive-test of element j of a 256-bit chunk: fp32 word j, or bf16 half j
template <typename T>
__device__ __forceinline__ bool is_pos(const uint32_t (&w)[8], int j) {
    if constexpr (sizeof(T) == 4) {
        return __uint_as_float(w[j]) > 0.0f;
    } else {
        const uint32_t h = (j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xFFFFu);
        return __uint_as_float(h << 16) > 0.0f;
    }
}

// zero the elements whose bit is clear (bits: V bits, element j at bit j)
template <typename T>
__device__ __forceinline__ void mask_words(uint32_t (&w)[8], uint32_t bits) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (!((bits >> j) & 1u)) w[j] = 0u;
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t keep = (((bits >> (2 * q)) & 1u) ? 0x0000FFFFu : 0u) |
                                  (((bits >> (2 * q + 1)) & 1u) ? 0xFFFF0000u : 0u);
            w[q] &= keep;
        }
    }
}

// ------------------------------------------------------------------ ReLU pack
// Fast path: whole 4 KB warp steps; the tail (E % step elements) is packed by
// relu_tail_kernel.  kY: also write y = ReLU(x).
template <typename T, bool kY>
__global__ void __launch_bounds__(kBlock) relu_pack_kernel(const T* __restrict__ x, int64_t steps,
                                                           uint8_t* __restrict__ mask,
                                                           T* __restrict__ y) {
    constexpr int V = RV<T>::V;          // elements per load
    constexpr int MB = V / 8;            // mask bytes per load
    constexpr int64_t kStep = 4 * 32 * V;  // elements per warp step
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t s = warp; s < steps; s += nwarps) {
        const int64_t e0 = s * kStep;
        uint32_t w[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) ldg256(x + e0 + (int64_t)(i * 32 + lane) * V, w[i]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t bits = 0;
#pragma unroll
            for (int j = 0; j < V; ++j) bits |= (uint32_t)is_pos<T>(w[i], j) << j;
            uint8_t* mb = mask + e0 / 8 + (int64_t)(i * 32 + lane) * MB;
            if constexpr (MB == 1)
                *mb = (uint8_t)bits;
            else
                *reinterpret_cast<uint16_t*>(mb) = (uint16_t)bits;
            if constexpr (kY) {
                mask_words<T>(w[i], bits);
                stg256(y + e0 + (int64_t)(i * 32 + lane) * V, w[i]);
            }
        }
    }
}

// Tail / unaligned path: thread per mask byte (8 elements).
template <typename T>
__global__ void __launch_bounds__(kBlock) relu_pack_generic_kernel(const T* __restrict__ x,
                                                                   int64_t e_begin, int64_t E,
                                                                   uint8_t* __restrict__ mask,
                                                                   T* __restrict__ y) {
    const int64_t nbytes = (E - e_begin + 7) / 8;
    for (int64_t t = (int64_t)blockIdx.x * kBlock + threadIdx.x; t < nbytes;
         t += (int64_t)gridDim.x * kBlock) {
        const int64_t e = e_begin + t * 8;
        uint32_t bits = 0;
        for (int j = 0; j < 8 && e + j < E; ++j) {
            const bool pos = widen1(x, e + j) > 0.0f;
            bits |= (uint32_t)pos << j;
            if (y) y[e + j] = pos ? x[e + j] : (T)0;
        }
        mask[e / 8] = (uint8_t)bits;
    }
}

// ------------------------------------------------------------------ ReLU backward
template <typename T>
__global__ void __launch_bounds__(kBlock) relu_backward_kernel(const uint8_t* __restrict__ mask,
                                                               const T* __restrict__ gy,
                                                               int64_t steps, T* __restrict__ gx) {
    constexpr int V = RV<T>::V;
    constexpr int MB = V / 8;
    constexpr int64_t kStep = 4 * 32 * V;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t s = warp; s < steps; s += nwarps) {
        const int64_t e0 = s * kStep;
        uint32_t w[4][8];
        uint32_t bits[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            ldg256(gy + e0 + (int64_t)(i * 32 + lane) * V, w[i]);
            const uint8_t* mb = mask + e0 / 8 + (int64_t)(i * 32 + lane) * MB;
            bits[i] = MB == 1 ? (uint32_t)__ldg(mb)
                              : (uint32_t)__ldg(reinterpret_cast<const uint16_t*>(mb));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            mask_words<T>(w[i], bits[i]);
            stg256(gx + e0 + (int64_t)(i * 32 + lane) * V, w[i]);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kBlock) relu_backward_generic_kernel(
    const uint8_t* __restrict__ mask, const T* __restrict__ gy, int64_t e_begin, int64_t E,
    T* __restrict__ gx) {
    for (int64_t e = e_begin + (int64_t)blockIdx.x * kBlock + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * kBlock) {
        const bool on = (mask[e >> 3] >> (e & 7)) & 1u;
        gx[e] = on ? gy[e] : (T)0;
    }
}

// ------------------------------------------------------------------ max pool
struct Pool {
    int64_t NC, H, W, OH, OW;
    int kh, kw, sh, sw, ph, pw, dh, dw;
};

// One launch covers planes p = blockIdx.y, blockIdx.y + gridDim.y, ... and, in
// each plane, output positions blockIdx.x * kBlock + threadIdx.x + k * span:
// all index arithmetic is 32-bit (a plane has < 2^31 positions) and the window
// taps are read through L1 (each input is read by ~kh kw / (sh sw) windows).
// kS2: stride 2 in both dimensions (every ResNet max pool) -> shifts.
template <typename T>
__global__ void __launch_bounds__(kBlock) maxpool_fwd_kernel(const T* __restrict__ x, Pool g,
                                                             T* __restrict__ y,
                                                             uint8_t* __restrict__ idx) {
    const int H = (int)g.H, W = (int)g.W, OW = (int)g.OW;
    const int P = (int)(g.OH * g.OW);
    const int span = gridDim.x * kBlock;
    for (int64_t p = blockIdx.y; p < g.NC; p += gridDim.y) {
        const T* __restrict__ plane = x + p * g.H * g.W;
        for (int o = blockIdx.x * kBlock + threadIdx.x; o < P; o += span) {
            const int i = o / OW;
            const int j = o - i * OW;
            float best = 0.0f;
            T bestv = (T)0;
            int arg = -1;
            const int r0 = i * g.sh - g.ph, c0 = j * g.sw - g.pw;
            for (int a = 0; a < g.kh; ++a) {
                const int r = r0 + a * g.dh;
                if (r < 0 || r >= H) continue;
                for (int b = 0; b < g.kw; ++b) {
                    const int c = c0 + b * g.dw;
                    if (c < 0 || c >= W) continue;
                    const T raw = __ldg(plane + r * W + c);
                    const float v = widen1(&raw, 0);
                    if (arg < 0 || v > best) {  // first maximum in row-major tap order
                        best = v;
                        bestv = raw;
                        arg = a * g.kw + b;
                    }
                }
            }
            y[p * P + o] = bestv;
            idx[p * P + o] = (uint8_t)arg;
        }
    }
}

__device__ __forceinline__ void store_acc(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_acc(uint16_t* p, float v) {
    *p = (uint16_t)(pack_bf16x2(v, 0.0f) & 0xFFFFu);
}

// grad_x gather: windows containing (r, c) in increasing (oh, ow) order; tap
// a gives oh = (r + ph - a dh) / sh, so a runs downwards for ascending oh
// (the oracle's accumulation order, bit for bit).
template <typename T, bool kS2>
__global__ void __launch_bounds__(kBlock) maxpool_bwd_kernel(const uint8_t* __restrict__ idx,
                                                             const T* __restrict__ gy, Pool g,
                                                             T* __restrict__ gx) {
    const int W = (int)g.W, OH = (int)g.OH, OW = (int)g.OW;
    const int P = (int)(g.H * g.W), OP = OH * OW;
    const int span = gridDim.x * kBlock;
    for (int64_t p = blockIdx.y; p < g.NC; p += gridDim.y) {
        const uint8_t* __restrict__ ip = idx + p * OP;
        const T* __restrict__ gp = gy + p * OP;
        for (int q = blockIdx.x * kBlock + threadIdx.x; q < P; q += span) {
            const int r = q / W;
            const int c = q - r * W;
            float acc = 0.0f;
            for (int a = g.kh - 1; a >= 0; --a) {
                const int u = r + g.ph - a * g.dh;
                if (u < 0) continue;
                int oh;
                if (kS2) {
                    if (u & 1) continue;
                    oh = u >> 1;
                } else {
                    if (u % g.sh) continue;
                    oh = u / g.sh;
                }
                if (oh >= OH) continue;
                for (int b = g.kw - 1; b >= 0; --b) {
                    const int v = c + g.pw - b * g.dw;
                    if (v < 0) continue;
                    int ow;
                    if (kS2) {
                        if (v & 1) continue;
                        ow = v >> 1;
                    } else {
                        if (v % g.sw) continue;
                        ow = v / g.sw;
                    }
                    if (ow >= OW) continue;
                    const int o = oh * OW + ow;
                    if ((int)__ldg(ip + o) == a * g.kw + b) acc += widen1(gp, o);
                }
            }
            store_acc(gx + p * P + q, acc);
        }
    }
}

// The ResNet max pool (3x3, stride 2, padding 1, dilation 1), specialised.
// Forward: the window's taps unrolled with compile-time offsets.
template <typename T>
__global__ void __launch_bounds__(kBlock) maxpool_fwd_k3s2_kernel(const T* __restrict__ x, Pool g,
                                                                  T* __restrict__ y,
                                                                  uint8_t* __restrict__ idx) {
    const int H = (int)g.H, W = (int)g.W, OW = (int)g.OW;
    const int P = (int)(g.OH * g.OW);
    const int span = gridDim.x * kBlock;
    for (int64_t p = blockIdx.y; p < g.NC; p += gridDim.y) {
        const T* __restrict__ plane = x + p * g.H * g.W;
        for (int o = blockIdx.x * kBlock + threadIdx.x; o < P; o += span) {
            const int i = o / OW;
            const int j = o - i * OW;
            float best = 0.0f;
            T bestv = (T)0;
            int arg = -1;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int r = 2 * i - 1 + a;
                if (r < 0 || r >= H) continue;
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    const int c = 2 * j - 1 + b;
                    if (c < 0 || c >= W) continue;
                    const T raw = __ldg(plane + r * W + c);
                    const float v = widen1(&raw, 0);
                    if (arg < 0 || v > best) {
                        best = v;
                        bestv = raw;
                        arg = a * 3 + b;
                    }
                }
            }
            y[p * P + o] = bestv;
            idx[p * P + o] = (uint8_t)arg;
        }
    }
}

// Forward, W % (2K) == 0 (every ResNet stem): one thread per K adjacent
// outputs (i, Km) .. (i, Km+K-1), whose windows cover columns 2Km-1 .. 2Km+2K-1
// of rows 2i-1 .. 2i+1 -- per row aligned vector loads of columns 2Km ..
// 2Km+2K-1 plus the scalar 2Km-1 (an L1 hit: the neighbouring thread's
// vector), 3 (K/2 + 1) loads for K outputs instead of 9 K.  The taps are
// scanned in the same (a, b) order with the same strict ">" as above, so values
// and first-index ties are unchanged.  K = 4 (bf16: one 16-byte load per row,
// fp32: two).
template <typename T, int K>
__device__ __forceinline__ void ld_cols(const T* p, float (&v)[2 * K]) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int q = 0; q < K / 2; ++q) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(p) + q);
            v[4 * q] = f.x, v[4 * q + 1] = f.y, v[4 * q + 2] = f.z, v[4 * q + 3] = f.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < K / 4; ++q) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(p) + q);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                v[8 * q + 2 * h] = __uint_as_float(w[h] << 16);
                v[8 * q + 2 * h + 1] = __uint_as_float(w[h] & 0xFFFF0000u);
            }
        }
    }
}
template <typename T, int K, bool kRound = false>
__device__ __forceinline__ void st_outs(T* p, const float (&b)[K]) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int q = 0; q < K / 4; ++q)
            reinterpret_cast<float4*>(p)[q] = make_float4(b[4 * q], b[4 * q + 1], b[4 * q + 2], b[4 * q + 3]);
    } else {  // !kRound: exact, the b are bf16 values (forward)
        uint32_t w[K / 2];
#pragma unroll
        for (int h = 0; h < K / 2; ++h)
            w[h] = kRound ? pack_bf16x2(b[2 * h], b[2 * h + 1])  // RNE, as store_acc
                          : (__float_as_uint(b[2 * h]) >> 16) | (__float_as_uint(b[2 * h + 1]) & 0xFFFF0000u);
        if constexpr (K % 8 == 0) {
#pragma unroll
            for (int q = 0; q < K / 8; ++q)
                reinterpret_cast<uint4*>(p)[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        } else if constexpr (K == 4)
            *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
        else
            *reinterpret_cast<uint32_t*>(p) = w[0];
    }
}
template <typename T>
constexpr int kPoolK = sizeof(T) == 2 ? ACTNN_POOL_K16 : ACTNN_POOL_K32;

// flat grid-stride over (plane, row, run): a plane's 56 x 14 runs do not fill
// whole CTAs, so planes share CTAs (32-bit indices; the launcher checks range)
template <typename T>
__global__ void __launch_bounds__(kBlock) maxpool_fwd_k3s2_vec(const T* __restrict__ x, Pool g,
                                                               T* __restrict__ y,
                                                               uint8_t* __restrict__ idx) {
    constexpr int K = kPoolK<T>;
    const int H = (int)g.H, W = (int)g.W, OW = (int)g.OW;
    const uint32_t M = (uint32_t)OW / K;  // output runs per row (OW = W / 2)
    const uint32_t Q = (uint32_t)g.OH * M;
    const uint32_t total = (uint32_t)g.NC * Q;
    for (uint32_t f = blockIdx.x * kBlock + threadIdx.x; f < total; f += gridDim.x * kBlock) {
        {
            const uint32_t p = f / Q;
            const uint32_t q = f - p * Q;
            const int i = (int)(q / M);
            const int m = (int)(q - i * M);
            const T* __restrict__ plane = x + (size_t)p * H * W;
            float best[K];
            int arg[K];
#pragma unroll
            for (int t = 0; t < K; ++t) best[t] = 0.0f, arg[t] = -1;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int r = 2 * i - 1 + a;
                if (r < 0 || r >= H) continue;
                const T* row = plane + r * W + 2 * K * m;
                float v[2 * K];
                ld_cols<T, K>(row, v);
                // column 2Km-1 by a scalar load (an L1 hit); taking it from the
                // previous lane by a shuffle measured 3-5% slower
                const float left = m > 0 ? widen1(row, -1) : 0.0f;
#pragma unroll
                for (int t = 0; t < K; ++t) {
                    // output Km + t: columns 2(Km+t) - 1, 2(Km+t), 2(Km+t) + 1
                    if (t > 0 || m > 0) {
                        const float l = t > 0 ? v[2 * t - 1] : left;
                        if (arg[t] < 0 || l > best[t]) best[t] = l, arg[t] = a * 3;
                    }
                    if (arg[t] < 0 || v[2 * t] > best[t]) best[t] = v[2 * t], arg[t] = a * 3 + 1;
                    if (v[2 * t + 1] > best[t]) best[t] = v[2 * t + 1], arg[t] = a * 3 + 2;
                }
            }
            const size_t o = (size_t)p * (g.OH * g.OW) + i * OW + K * m;
            st_outs<T, K>(y + o, best);
            uint32_t packed[K / 4] = {};
#pragma unroll
            for (int t = 0; t < K; ++t) packed[t / 4] |= (uint32_t)arg[t] << (8 * (t % 4));
            if constexpr (K == 8)
                *reinterpret_cast<uint2*>(idx + o) = make_uint2(packed[0], packed[1]);
            else
                *reinterpret_cast<uint32_t*>(idx + o) = packed[0];
        }
    }
}

// Backward: one thread per 2x2 block of inputs (rows 2i, 2i+1; columns 2j,
// 2j+1), which are covered only by the windows (i, j), (i, j+1), (i+1, j),
// (i+1, j+1): input (2i+s, 2j+t) takes tap a = 1 + s (window row i) or a = 0
// (row i + 1, s = 1), likewise b -- no divergence, four (idx, grad) reads per
// four outputs, contributions added in increasing (oh, ow) order as the oracle.
template <typename T>
__global__ void __launch_bounds__(kBlock) maxpool_bwd_k3s2_kernel(const uint8_t* __restrict__ idx,
                                                                  const T* __restrict__ gy, Pool g,
                                                                  T* __restrict__ gx) {
    const int H = (int)g.H, W = (int)g.W, OH = (int)g.OH, OW = (int)g.OW;
    const int BH = (H + 1) >> 1, BW = (W + 1) >> 1;  // 2x2 blocks per plane
    const int PB = BH * BW, OP = OH * OW;
    const int span = gridDim.x * kBlock;
    for (int64_t p = blockIdx.y; p < g.NC; p += gridDim.y) {
        const uint8_t* __restrict__ ip = idx + p * OP;
        const T* __restrict__ gp = gy + p * OP;
        T* __restrict__ out = gx + p * g.H * g.W;
        for (int q = blockIdx.x * kBlock + threadIdx.x; q < PB; q += span) {
            const int i = q / BW;
            const int j = q - i * BW;
            // the four windows (absent ones never match: tap 255)
            int k00 = 255, k01 = 255, k10 = 255, k11 = 255;
            float g00 = 0.0f, g01 = 0.0f, g10 = 0.0f, g11 = 0.0f;
            if (i < OH && j < OW) { k00 = __ldg(ip + i * OW + j); g00 = widen1(gp, i * OW + j); }
            if (i < OH && j + 1 < OW) { k01 = __ldg(ip + i * OW + j + 1); g01 = widen1(gp, i * OW + j + 1); }
            if (i + 1 < OH && j < OW) { k10 = __ldg(ip + (i + 1) * OW + j); g10 = widen1(gp, (i + 1) * OW + j); }
            if (i + 1 < OH && j + 1 < OW) {
                k11 = __ldg(ip + (i + 1) * OW + j + 1);
                g11 = widen1(gp, (i + 1) * OW + j + 1);
            }
            const int r = 2 * i, c = 2 * j;
            // (2i, 2j): window (i, j) tap (1, 1)
            float a00 = 0.0f;
            if (k00 == 4) a00 += g00;
            // (2i, 2j+1): (i, j) tap (1, 2), then (i, j+1) tap (1, 0)
            float a01 = 0.0f;
            if (k00 == 5) a01 += g00;
            if (k01 == 3) a01 += g01;
            // (2i+1, 2j): (i, j) tap (2, 1), then (i+1, j) tap (0, 1)
            float a10 = 0.0f;
            if (k00 == 7) a10 += g00;
            if (k10 == 1) a10 += g10;
            // (2i+1, 2j+1): (i, j) (2, 2), (i, j+1) (2, 0), (i+1, j) (0, 2), (i+1, j+1) (0, 0)
            float a11 = 0.0f;
            if (k00 == 8) a11 += g00;
            if (k01 == 6) a11 += g01;
            if (k10 == 2) a11 += g10;
            if (k11 == 0) a11 += g11;
            store_acc(out + r * W + c, a00);
            if (c + 1 < W) store_acc(out + r * W + c + 1, a01);
            if (r + 1 < H) {
                store_acc(out + (r + 1) * W + c, a10);
                if (c + 1 < W) store_acc(out + (r + 1) * W + c + 1, a11);
            }
        }
    }
}

// bf16 forward on packed halves (runs of 8 outputs, W a multiple of 16).  Word
// q of a row holds columns (16m + 2q, 16m + 2q + 1), i.e. taps b = 1, 2 of
// output t = q, and its high half is tap b = 0 of output q + 1.  The window
// max is reduced column-wise with max.bf16x2 over the valid rows, then over the
// three columns; the first argmax tap (row-major, as the scalar kernels) is
// found by testing every tap for equality with the max (setp.eq.bf16x2: two
// predicates per word) in reverse tap order, so the earliest match is written
// last.  The stored value is the max's bits -- except for a max of zero, where
// the first equal tap's sign of zero is the oracle's; that rare case takes the
// scalar scan.
__device__ __forceinline__ void eq_row(int& arg, uint32_t w, uint32_t wl, uint32_t mm, int a3) {
    // reverse order: b = 2 (hi of w), b = 1 (lo of w), b = 0 (hi of wl)
    asm("{\n\t.reg .pred l1, h1, l0, h0;\n\t"
        "setp.eq.bf16x2 l1|h1, %1, %3;\n\t"
        "setp.eq.bf16x2 l0|h0, %2, %3;\n\t"
        "@h1 mov.u32 %0, %6;\n\t"
        "@l1 mov.u32 %0, %5;\n\t"
        "@h0 mov.u32 %0, %4;\n\t}"
        : "+r"(arg)
        : "r"(w), "r"(wl), "r"(mm), "r"(a3), "r"(a3 + 1), "r"(a3 + 2));
}
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// 5 CTAs per SM: 48 registers (a bound of 1 lets ptxas take 56, 0.76 -> 0.60)
__global__ void __launch_bounds__(kBlock, 5) maxpool_fwd_k3s2_bf16x2(const uint16_t* __restrict__ x,
                                                                  Pool g, uint16_t* __restrict__ y,
                                                                  uint8_t* __restrict__ idx) {
    constexpr int K = 8;
    constexpr uint32_t kNaN = 0x7FC07FC0u;  // never equal: absent taps
    const int H = (int)g.H, W = (int)g.W, OW = (int)g.OW;
    const uint32_t M = (uint32_t)OW / K;
    const uint32_t Q = (uint32_t)g.OH * M;
    const uint32_t total = (uint32_t)g.NC * Q;
    for (uint32_t f = blockIdx.x * kBlock + threadIdx.x; f < total; f += gridDim.x * kBlock) {
        const uint32_t p = f / Q;
        const uint32_t q = f - p * Q;
        const int i = (int)(q / M);
        const int m = (int)(q - i * M);
        const uint16_t* __restrict__ plane = x + (size_t)p * H * W;
        // rows 2i-1, 2i, 2i+1: row 2i always exists (i < OH)
        const bool v0 = i > 0, v2 = 2 * i + 1 < H;
        uint32_t w[3][K], L[3];  // L: left column 16m - 1 in the high half (NaN if absent)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const bool rv = a == 1 || (a == 0 ? v0 : v2);
            const uint16_t* row = plane + (2 * i - 1 + a) * W + 2 * K * m;
            if (rv) {
                const uint4 u0 = __ldg(reinterpret_cast<const uint4*>(row));
                const uint4 u1 = __ldg(reinterpret_cast<const uint4*>(row) + 1);
                w[a][0] = u0.x, w[a][1] = u0.y, w[a][2] = u0.z, w[a][3] = u0.w;
                w[a][4] = u1.x, w[a][5] = u1.y, w[a][6] = u1.z, w[a][7] = u1.w;
                L[a] = m > 0 ? ((uint32_t)row[-1] << 16) | 0x7FC0u : kNaN;
            } else {
#pragma unroll
                for (int t = 0; t < K; ++t) w[a][t] = kNaN;
                L[a] = kNaN;
            }
        }
        // column maxima over the valid rows (max.bf16x2 drops a NaN operand)
        uint32_t c[K], cl;
#pragma unroll
        for (int t = 0; t < K; ++t) c[t] = bmax2(bmax2(w[0][t], w[1][t]), w[2][t]);
        cl = bmax2(bmax2(L[0], L[1]), L[2]);
        float best[K];
        int arg[K];
#pragma unroll
        for (int t = 0; t < K; ++t) {
            const uint32_t left = t > 0 ? c[t - 1] : cl;  // tap b = 0 in the high half
            float mx = fmaxf(__uint_as_float(c[t] << 16), __uint_as_float(c[t] & 0xFFFF0000u));
            if (t > 0 || m > 0) mx = fmaxf(mx, __uint_as_float(left & 0xFFFF0000u));
            const uint32_t mb = __float_as_uint(mx) >> 16;
            const uint32_t mm = mb | (mb << 16);
            int k = 255;
#pragma unroll
            for (int a = 2; a >= 0; --a) eq_row(k, w[a][t], t > 0 ? w[a][t - 1] : L[a], mm, 3 * a);
            if (mx == 0.0f) {  // sign of zero: the first zero tap's (scalar scan)
                float b = 0.0f;
                uint32_t bits = 0;
                int kk = -1;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const bool rv = a == 1 || (a == 0 ? v0 : v2);
                    if (!rv) continue;
                    const uint32_t tw = t > 0 ? w[a][t - 1] : L[a];
                    const uint32_t h[3] = {tw >> 16, w[a][t] & 0xFFFFu, w[a][t] >> 16};
#pragma unroll
                    for (int bb = 0; bb < 3; ++bb) {
                        if (bb == 0 && t == 0 && m == 0) continue;
                        const float v = __uint_as_float(h[bb] << 16);
                        if (kk < 0 || v > b) b = v, bits = h[bb], kk = 3 * a + bb;
                    }
                }
                mx = __uint_as_float(bits << 16);
            }
            best[t] = mx;
            arg[t] = k;
        }
        const size_t o = (size_t)p * (g.OH * g.OW) + i * OW + K * m;
        st_outs<uint16_t, K>(y + o, best);
        uint32_t packed[2] = {0u, 0u};
#pragma unroll
        for (int t = 0; t < K; ++t) packed[t / 4] |= (uint32_t)arg[t] << (8 * (t % 4));
        *reinterpret_cast<uint2*>(idx + o) = make_uint2(packed[0], packed[1]);
    }
}

// Vector backward of the ResNet max pool (W a multiple of 2K): one thread per
// (plane, block row i, run m of K output columns), i.e. input rows 2i, 2i+1 and
// columns 2Km .. 2Km+2K-1, read from window rows i, i+1 at columns Km .. Km+K
// (column Km+K: a scalar load, L1 hit) with vector idx / grad loads, written
// with vector stores.  Taps and accumulation order as maxpool_bwd_k3s2_kernel.
template <typename T, int K>
__device__ __forceinline__ void ld_idx(const uint8_t* p, int (&k)[K]) {
    uint32_t w[K / 4];
    if constexpr (K == 8) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
        w[0] = u.x, w[1] = u.y;
    } else {
        w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
    }
#pragma unroll
    for (int t = 0; t < K; ++t) k[t] = (int)((w[t / 4] >> (8 * (t % 4))) & 0xFFu);
}
#ifndef ACTNN_POOLB_K32
#define ACTNN_POOLB_K32 4  // fp32 runs of 8 measured 15% slower
#endif
template <typename T>
constexpr int kPoolKB = sizeof(T) == 2 ? ACTNN_POOL_K16 : ACTNN_POOLB_K32;
// CTAs per SM the register budget must allow: bf16 5 (48 registers; 0.78 ->
// 0.81 of HBM over the unbounded 52), fp32 7 (32 registers; 0.76 -> 0.80 over
// the unbounded 36, and a bound of 5 gave 42 registers and 0.74)
template <typename T>
__global__ void __launch_bounds__(kBlock, sizeof(T) == 2 ? 5 : 7) maxpool_bwd_k3s2_vec(const uint8_t* __restrict__ idx,
                                                               const T* __restrict__ gy, Pool g,
                                                               T* __restrict__ gx) {
    constexpr int K = kPoolKB<T>;
    const int H = (int)g.H, W = (int)g.W, OH = (int)g.OH, OW = (int)g.OW;
    const uint32_t BH = (uint32_t)(H + 1) >> 1;
    const uint32_t M = (uint32_t)OW / K;
    const uint32_t Q = BH * M;
    const uint32_t total = (uint32_t)g.NC * Q;
    for (uint32_t f = blockIdx.x * kBlock + threadIdx.x; f < total; f += gridDim.x * kBlock) {
        const uint32_t p = f / Q;
        const uint32_t q = f - p * Q;
        const int i = (int)(q / M);
        const int m = (int)(q - i * M);
        const uint8_t* __restrict__ ipl = idx + (size_t)p * OH * OW;
        const T* __restrict__ gpl = gy + (size_t)p * OH * OW;
        // window rows i (c = 0) and i + 1 (c = 1), columns Km .. Km+K (tap 255: absent)
        int k[2][K + 1];
        float gv[2][K + 1];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int w = i + c;
            if (w < OH) {
                const int o = w * OW + K * m;
                ld_idx<T, K>(ipl + o, *reinterpret_cast<int(*)[K]>(&k[c][0]));
                float tmp[K];
                ld_cols<T, K / 2>(gpl + o, tmp);
#pragma unroll
                for (int t = 0; t < K; ++t) gv[c][t] = tmp[t];
                if (m + 1 < (int)M) {
                    k[c][K] = (int)__ldg(ipl + o + K);
                    gv[c][K] = widen1(gpl, o + K);
                } else {
                    k[c][K] = 255, gv[c][K] = 0.0f;
                }
            } else {
#pragma unroll
                for (int t = 0; t <= K; ++t) k[c][t] = 255, gv[c][t] = 0.0f;
            }
        }
        float top[2 * K], bot[2 * K];
#pragma unroll
        for (int t = 0; t < K; ++t) {
            const int k00 = k[0][t], k01 = k[0][t + 1], k10 = k[1][t], k11 = k[1][t + 1];
            const float g00 = gv[0][t], g01 = gv[0][t + 1], g10 = gv[1][t], g11 = gv[1][t + 1];
            float a00 = 0.0f;
            if (k00 == 4) a00 += g00;
            float a01 = 0.0f;
            if (k00 == 5) a01 += g00;
            if (k01 == 3) a01 += g01;
            float a10 = 0.0f;
            if (k00 == 7) a10 += g00;
            if (k10 == 1) a10 += g10;
            float a11 = 0.0f;
            if (k00 == 8) a11 += g00;
            if (k01 == 6) a11 += g01;
            if (k10 == 2) a11 += g10;
            if (k11 == 0) a11 += g11;
            top[2 * t] = a00, top[2 * t + 1] = a01, bot[2 * t] = a10, bot[2 * t + 1] = a11;
        }
        T* __restrict__ out = gx + (size_t)p * H * W + (size_t)(2 * i) * W + 2 * K * m;
        st_outs<T, 2 * K, true>(out, top);
        if (2 * i + 1 < H) st_outs<T, 2 * K, true>(out + W, bot);
    }
}

// Row-sliding backward of the ResNet max pool (3x3, stride 2, padding 1): a
// warp owns 32 consecutive output columns of one plane and walks its window
// rows; window row i + 1 is loaded once and reused as row i of the next step,
// column j + 1 comes from the neighbouring lane by a shuffle.  No divisions in
// the loop (the per-output forward kernel measured equal to a row-sliding one).
// backward: lane = output column j = input columns 2j, 2j+1; rows of windows i
// (current) and i + 1 (next) give input rows 2i, 2i+1 exactly as in
// maxpool_bwd_k3s2_kernel (same taps, same accumulation order)
template <typename T>
__global__ void __launch_bounds__(kBlock) maxpool_bwd_k3s2_rows(const uint8_t* __restrict__ idx,
                                                                const T* __restrict__ gy, Pool g,
                                                                T* __restrict__ gx) {
    const int H = (int)g.H, W = (int)g.W, OH = (int)g.OH, OW = (int)g.OW;
    const int BH = (H + 1) >> 1, BW = (W + 1) >> 1;
    const int lane = threadIdx.x & 31;
    const int nchunk = (BW + 31) >> 5;
    const int64_t strips = g.NC * nchunk;
    const int64_t nw = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t sw = (((int64_t)blockIdx.x * kBlock) + threadIdx.x) >> 5; sw < strips; sw += nw) {
        const int64_t p = sw / nchunk;
        const int j = (int)(sw - p * nchunk) * 32 + lane;
        const uint8_t* __restrict__ ipl = idx + p * g.OH * g.OW;
        const T* __restrict__ gpl = gy + p * g.OH * g.OW;
        T* __restrict__ out = gx + p * g.H * g.W;
        // window row w: (k, g) at columns j and j + 1 (absent windows: tap 255)
        auto load_wrow = [&](int w, int& k0, float& g0, int& k1, float& g1) {
            const bool wok = w < OH;
            k0 = (wok && j < OW) ? (int)__ldg(ipl + w * OW + j) : 255;
            g0 = (wok && j < OW) ? widen1(gpl, (int64_t)w * OW + j) : 0.0f;
            int kn = __shfl_down_sync(0xffffffffu, k0, 1);
            float gn = __shfl_down_sync(0xffffffffu, g0, 1);
            if (lane == 31) {
                kn = (wok && j + 1 < OW) ? (int)__ldg(ipl + w * OW + j + 1) : 255;
                gn = (wok && j + 1 < OW) ? widen1(gpl, (int64_t)w * OW + j + 1) : 0.0f;
            }
            k1 = (j + 1 < OW) ? kn : 255;
            g1 = gn;
        };
        int k00, k01, k10, k11;
        float g00, g01, g10, g11;
        load_wrow(0, k00, g00, k01, g01);
        for (int i = 0; i < BH; ++i) {
            load_wrow(i + 1, k10, g10, k11, g11);
            if (j < BW) {
                const int r = 2 * i, c = 2 * j;
                float a00 = 0.0f;
                if (k00 == 4) a00 += g00;
                float a01 = 0.0f;
                if (k00 == 5) a01 += g00;
                if (k01 == 3) a01 += g01;
                float a10 = 0.0f;
                if (k00 == 7) a10 += g00;
                if (k10 == 1) a10 += g10;
                float a11 = 0.0f;
                if (k00 == 8) a11 += g00;
                if (k01 == 6) a11 += g01;
                if (k10 == 2) a11 += g10;
                if (k11 == 0) a11 += g11;
                store_acc(out + (int64_t)r * W + c, a00);
                if (c + 1 < W) store_acc(out + (int64_t)r * W + c + 1, a01);
                if (r + 1 < H) {
                    store_acc(out + (int64_t)(r + 1) * W + c, a10);
                    if (c + 1 < W) store_acc(out + (int64_t)(r + 1) * W + c + 1, a11);
                }
            }
            k00 = k10;
            g00 = g10;
            k01 = k11;
            g01 = g11;
        }
    }
}

bool aligned32(const void* p) { return ((uintptr_t)p & 31u) == 0; }

// One warp per 4 KB step (every step's loads in flight at once) instead of a
// persistent grid: 0.90 -> 1.03 of the measured copy bandwidth on the stem
// activation (tools/relu_time.py).  -DACTNN_RELU_FULLGRID=0: the persistent grid.
#ifndef ACTNN_RELU_FULLGRID
#define ACTNN_RELU_FULLGRID 1
#endif
constexpr int relu_full_grid() { return ACTNN_RELU_FULLGRID; }

template <typename T>
cudaError_t relu_pack_t(const ReluArgs& a, cudaStream_t s) {
    constexpr int64_t kStep = 4 * 32 * RV<T>::V;
    const T* x = static_cast<const T*>(a.x);
    T* y = static_cast<T*>(a.y);
    const bool vec = aligned32(a.x) && (!a.y || aligned32(a.y)) &&
                     ((uintptr_t)a.mask % sizeof(T)) == 0;
    const int64_t steps = vec ? a.E / kStep : 0;
    if (steps > 0) {
        const void* k = a.y ? (const void*)relu_pack_kernel<T, true>
                            : (const void*)relu_pack_kernel<T, false>;
        const int64_t wb = (steps + kBlock / 32 - 1) / (kBlock / 32);
        const int grid = relu_full_grid() > 0 ? (int)std::min<int64_t>(wb, 1 << 30) : grid_for(k, kBlock, 0, wb);
        if (a.y)
            relu_pack_kernel<T, true><<<grid, kBlock, 0, s>>>(x, steps, a.mask, y);
        else
            relu_pack_kernel<T, false><<<grid, kBlock, 0, s>>>(x, steps, a.mask, y);
    }
    const int64_t e_begin = steps * kStep;
    if (e_begin < a.E) {
        const int64_t nbytes = (a.E - e_begin + 7) / 8;
        const int grid = grid_for((const void*)relu_pack_generic_kernel<T>, kBlock, 0,
                                  (nbytes + kBlock - 1) / kBlock);
        relu_pack_generic_kernel<T><<<grid, kBlock, 0, s>>>(x, e_begin, a.E, a.mask, y);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t relu_backward_t(const ReluArgs& a, cudaStream_t s) {
    constexpr int64_t kStep = 4 * 32 * RV<T>::V;
    const T* gy = static_cast<const T*>(a.x);
    T* gx = static_cast<T*>(a.y);
    const bool vec = aligned32(a.x) && aligned32(a.y) && ((uintptr_t)a.mask % sizeof(T)) == 0;
    const int64_t steps = vec ? a.E / kStep : 0;
    if (steps > 0) {
        const int64_t wb = (steps + kBlock / 32 - 1) / (kBlock / 32);
        const int grid = relu_full_grid() > 0 ? (int)std::min<int64_t>(wb, 1 << 30)
                                              : grid_for((const void*)relu_backward_kernel<T>, kBlock, 0, wb);
        relu_backward_kernel<T><<<grid, kBlock, 0, s>>>(a.mask, gy, steps, gx);
    }
    const int64_t e_begin = steps * kStep;
    if (e_begin < a.E) {
        const int grid = grid_for((const void*)relu_backward_generic_kernel<T>, kBlock, 0,
                                  (a.E - e_begin + kBlock - 1) / kBlock);
        relu_backward_generic_kernel<T><<<grid, kBlock, 0, s>>>(a.mask, gy, e_begin, a.E, gx);
    }
    return cudaGetLastError();
}

// Build-time variants (measured; the defaults are the fastest):
//   ACTNN_POOL_FULLGRID  1 one thread per run, 0 a persistent grid, -1 per dtype
//   ACTNN_POOL_ROWS      0: the 2x2-block backward instead of the row kernel
//   ACTNN_POOL_VEC       0: the scalar k3s2 forward and backward
//   ACTNN_POOL_PACKED    0: the float-compare bf16 forward
#ifndef ACTNN_POOL_FULLGRID
#define ACTNN_POOL_FULLGRID -1
#endif
#ifndef ACTNN_POOL_ROWS
#define ACTNN_POOL_ROWS 1
#endif
#ifndef ACTNN_POOL_VEC
#define ACTNN_POOL_VEC 1
#endif
#ifndef ACTNN_POOL_PACKED
#define ACTNN_POOL_PACKED 1
#endif
constexpr int pool_full_grid() { return ACTNN_POOL_FULLGRID; }

template <typename T>
cudaError_t maxpool_t(const PoolArgs& a, bool backward, cudaStream_t s) {
    Pool g{a.NC, a.H, a.W, a.OH, a.OW, a.kh, a.kw, a.sh, a.sw, a.ph, a.pw, a.dh, a.dw};
    const int64_t per_plane = backward ? a.H * a.W : a.OH * a.OW;
    const int bx = (int)std::min<int64_t>((per_plane + kBlock - 1) / kBlock, 64);
    const int by = (int)std::min<int64_t>(a.NC, 65535);
    const bool k3s2 = a.kh == 3 && a.kw == 3 && a.sh == 2 && a.sw == 2 && a.ph == 1 &&
                      a.pw == 1 && a.dh == 1 && a.dw == 1;
    constexpr bool rows = ACTNN_POOL_ROWS != 0;
    constexpr bool vec_fwd = ACTNN_POOL_VEC != 0;
    if (k3s2 && backward && a.W % (2 * kPoolKB<T>) == 0 && vec_fwd &&
        a.NC * ((a.H + 1) / 2) * (a.OW / kPoolKB<T>) < (1ll << 32) - kBlock * 65536ll &&
        reinterpret_cast<uintptr_t>(a.in) % (kPoolKB<T> * sizeof(T)) == 0 &&
        reinterpret_cast<uintptr_t>(a.out) % (2 * kPoolKB<T> * sizeof(T)) == 0 &&
        reinterpret_cast<uintptr_t>(a.idx) % kPoolKB<T> == 0) {
        const int64_t runs = a.NC * ((a.H + 1) / 2) * (a.OW / kPoolKB<T>);
        // one thread per run (all runs in flight) for fp32, +16% over a persistent
        // grid; bf16 keeps the persistent grid (6% better there)
        const bool full = pool_full_grid() >= 0 ? pool_full_grid() != 0 : sizeof(T) == 4;
        const int gv = full ? (int)((runs + kBlock - 1) / kBlock)
                            : grid_for((const void*)maxpool_bwd_k3s2_vec<T>, kBlock, 0, (runs + kBlock - 1) / kBlock);
        maxpool_bwd_k3s2_vec<T><<<gv, kBlock, 0, s>>>(a.idx, static_cast<const T*>(a.in), g,
                                                     static_cast<T*>(a.out));
    } else if (k3s2 && rows && backward) {
        const int64_t per = backward ? ((a.W + 1) / 2 + 31) / 32 : (a.OW + 31) / 32;
        const int64_t warps = a.NC * per;
        const int grid = grid_for((const void*)maxpool_bwd_k3s2_rows<T>, kBlock, 0, (warps + 7) / 8);
        maxpool_bwd_k3s2_rows<T><<<grid, kBlock, 0, s>>>(a.idx, static_cast<const T*>(a.in), g,
                                                          static_cast<T*>(a.out));
    } else if (!backward && k3s2 && a.W % (2 * kPoolK<T>) == 0 && vec_fwd &&
               a.NC * a.OH * (a.OW / kPoolK<T>) < (1ll << 32) - kBlock * 65536ll &&
               reinterpret_cast<uintptr_t>(a.in) % (2 * kPoolK<T> * sizeof(T)) == 0 &&
               reinterpret_cast<uintptr_t>(a.out) % (kPoolK<T> * sizeof(T)) == 0 &&
               reinterpret_cast<uintptr_t>(a.idx) % kPoolK<T> == 0) {
        const int64_t runs = a.NC * a.OH * (a.OW / kPoolK<T>);
        // one thread per run for fp32 (+1%), a persistent grid for bf16 (+4%)
        const bool full = pool_full_grid() >= 0 ? pool_full_grid() != 0 : sizeof(T) == 4;
        const int gv = full ? (int)((runs + kBlock - 1) / kBlock)
                            : grid_for((const void*)maxpool_fwd_k3s2_vec<T>, kBlock, 0, (runs + kBlock - 1) / kBlock);
        constexpr bool packed = ACTNN_POOL_PACKED != 0;
        if constexpr (sizeof(T) == 2) {
            if (packed && kPoolK<T> == 8) {
                maxpool_fwd_k3s2_bf16x2<<<gv, kBlock, 0, s>>>(static_cast<const uint16_t*>(a.in), g,
                                                              static_cast<uint16_t*>(a.out), a.idx);
                return cudaGetLastError();
            }
        }
        maxpool_fwd_k3s2_vec<T><<<gv, kBlock, 0, s>>>(static_cast<const T*>(a.in), g,
                                                                static_cast<T*>(a.out), a.idx);
    } else if (!backward && k3s2) {
        maxpool_fwd_k3s2_kernel<T><<<dim3(bx, by), kBlock, 0, s>>>(static_cast<const T*>(a.in), g,
                                                                  static_cast<T*>(a.out), a.idx);
    } else if (!backward) {
        maxpool_fwd_kernel<T><<<dim3(bx, by), kBlock, 0, s>>>(static_cast<const T*>(a.in), g,
                                                             static_cast<T*>(a.out), a.idx);
    } else if (k3s2) {
        const int64_t blocks = ((a.H + 1) / 2) * ((a.W + 1) / 2);
        const int bxb = (int)std::min<int64_t>((blocks + kBlock - 1) / kBlock, 64);
        maxpool_bwd_k3s2_kernel<T><<<dim3(bxb, by), kBlock, 0, s>>>(
            a.idx, static_cast<const T*>(a.in), g, static_cast<T*>(a.out));
    } else if (a.sh == 2 && a.sw == 2) {
        maxpool_bwd_kernel<T, true><<<dim3(bx, by), kBlock, 0, s>>>(
            a.idx, static_cast<const T*>(a.in), g, static_cast<T*>(a.out));
    } else {
        maxpool_bwd_kernel<T, false><<<dim3(bx, by), kBlock, 0, s>>>(
            a.idx, static_cast<const T*>(a.in), g, static_cast<T*>(a.out));
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_relu_pack(const ReluArgs& a, cudaStream_t s) {
    return a.dt == 0 ? relu_pack_t<float>(a, s) : relu_pack_t<uint16_t>(a, s);
}
cudaError_t launch_relu_backward(const ReluArgs& a, cudaStream_t s) {
    return a.dt == 0 ? relu_backward_t<float>(a, s) : relu_backward_t<uint16_t>(a, s);
}
cudaError_t launch_maxpool2d(const PoolArgs& a, bool backward, cudaStream_t s) {
    return a.dt == 0 ? maxpool_t<float>(a, backward, s) : maxpool_t<uint16_t>(a, backward, s);
}

}  // namespace actnn
