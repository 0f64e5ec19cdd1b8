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
// (row-major a * kw + b).  Backward: thread per input element, a gather over
// the windows that contain it in increasing output order (no atomics, so the
// fp32 sum order is fixed and equals the oracle's / PyTorch CPU's).
#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

constexpr int kBlock = 256;
constexpr unsigned kFullMask = 0xffffffffu;

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

template <typename T>
__global__ void __launch_bounds__(kBlock) maxpool_fwd_kernel(const T* __restrict__ x, Pool g,
                                                             T* __restrict__ y,
                                                             uint8_t* __restrict__ idx) {
    const int64_t total = g.NC * g.OH * g.OW;
    for (int64_t o = (int64_t)blockIdx.x * kBlock + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * kBlock) {
        const int64_t j = o % g.OW;
        const int64_t t = o / g.OW;
        const int64_t i = t % g.OH;
        const int64_t p = t / g.OH;
        const T* plane = x + p * g.H * g.W;
        float best = 0.0f;
        T bestv = (T)0;
        int arg = -1;
        for (int a = 0; a < g.kh; ++a) {
            const int64_t r = i * g.sh - g.ph + (int64_t)a * g.dh;
            if (r < 0 || r >= g.H) continue;
            for (int b = 0; b < g.kw; ++b) {
                const int64_t c = j * g.sw - g.pw + (int64_t)b * g.dw;
                if (c < 0 || c >= g.W) continue;
                const float v = widen1(plane, r * g.W + c);
                if (arg < 0 || v > best) {  // first maximum in row-major tap order
                    best = v;
                    bestv = plane[r * g.W + c];
                    arg = a * g.kw + b;
                }
            }
        }
        y[o] = bestv;
        idx[o] = (uint8_t)arg;
    }
}

__device__ __forceinline__ void store_acc(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_acc(uint16_t* p, float v) {
    *p = (uint16_t)(pack_bf16x2(v, 0.0f) & 0xFFFFu);
}

// grad_x gather: windows containing (r, c) in increasing (oh, ow) order; tap
// a gives oh = (r + ph - a dh) / sh, so a runs downwards for ascending oh.
template <typename T>
__global__ void __launch_bounds__(kBlock) maxpool_bwd_kernel(const uint8_t* __restrict__ idx,
                                                             const T* __restrict__ gy, Pool g,
                                                             T* __restrict__ gx) {
    const int64_t total = g.NC * g.H * g.W;
    for (int64_t q = (int64_t)blockIdx.x * kBlock + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * kBlock) {
        const int64_t c = q % g.W;
        const int64_t t = q / g.W;
        const int64_t r = t % g.H;
        const int64_t p = t / g.H;
        const int64_t obase = p * g.OH * g.OW;
        float acc = 0.0f;
        for (int a = g.kh - 1; a >= 0; --a) {
            const int64_t u = r + g.ph - (int64_t)a * g.dh;
            if (u < 0 || u % g.sh) continue;
            const int64_t oh = u / g.sh;
            if (oh >= g.OH) continue;
            for (int b = g.kw - 1; b >= 0; --b) {
                const int64_t v = c + g.pw - (int64_t)b * g.dw;
                if (v < 0 || v % g.sw) continue;
                const int64_t ow = v / g.sw;
                if (ow >= g.OW) continue;
                const int64_t o = obase + oh * g.OW + ow;
                if ((int)__ldg(idx + o) == a * g.kw + b) acc += widen1(gy, o);
            }
        }
        store_acc(gx + q, acc);
    }
}

bool aligned32(const void* p) { return ((uintptr_t)p & 31u) == 0; }

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
        const int grid = grid_for(k, kBlock, 0, (steps + kBlock / 32 - 1) / (kBlock / 32));
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
        const int grid = grid_for((const void*)relu_backward_kernel<T>, kBlock, 0,
                                  (steps + kBlock / 32 - 1) / (kBlock / 32));
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

template <typename T>
cudaError_t maxpool_t(const PoolArgs& a, bool backward, cudaStream_t s) {
    Pool g{a.NC, a.H, a.W, a.OH, a.OW, a.kh, a.kw, a.sh, a.sw, a.ph, a.pw, a.dh, a.dw};
    if (!backward) {
        const int grid = grid_for((const void*)maxpool_fwd_kernel<T>, kBlock, 0,
                                  (a.NC * a.OH * a.OW + kBlock - 1) / kBlock);
        maxpool_fwd_kernel<T><<<grid, kBlock, 0, s>>>(static_cast<const T*>(a.in), g,
                                                      static_cast<T*>(a.out), a.idx);
    } else {
        const int grid = grid_for((const void*)maxpool_bwd_kernel<T>, kBlock, 0,
                                  (a.NC * a.H * a.W + kBlock - 1) / kBlock);
        maxpool_bwd_kernel<T><<<grid, kBlock, 0, s>>>(a.idx, static_cast<const T*>(a.in), g,
                                                      static_cast<T*>(a.out));
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
