// k3_compute.cu -- the K3 consumer's per-group work (Philox + b=1/b=2 codes +
// packing + store) on register data, without TMA, producer or barriers.  If
// this runs much faster per group than quantize_ws_kernel, the pipeline is the
// limiter; if not, the instruction mix is.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2104_14129_b200/csrc/device.cuh"
using namespace actnn;

struct P {
    RoundKeys rk;
};

// scalar-FP variant of codes_small (FADD/FFMA instead of the f32x2 forms)
template <int b>
__device__ __forceinline__ uint32_t codes_small_s(const float v[8], float Z, float inv14,
                                                  const Philox4& o) {
    const uint32_t w[4] = {o.x, o.y, o.z, o.w};
    uint32_t y = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float tx = __fmaf_rn(__fsub_rn(v[2 * p], Z), inv14, 12582912.0f);
        const float ty = __fmaf_rn(__fsub_rn(v[2 * p + 1], Z), inv14, 12582912.0f);
        uint32_t T = __byte_perm(__float_as_uint(tx), __float_as_uint(ty), 0x5410);
        T += w[p] & 0x3FFF3FFFu;
        if (b == 2)
            y |= (T >> (14 - 4 * p)) & (0xC000C000u >> (14 - 4 * p));
        else
            y |= (T >> (14 - 2 * p)) & (0x40004000u >> (14 - 2 * p));
    }
    if (b == 2) return (y | (y >> 14)) & 0xFFFFu;
    return (y | (y >> 15)) & 0xFFu;
}

template <int b, int PH, bool kScalar = false>
__global__ void k3_body(const __grid_constant__ P p, uint32_t groups_per_warp, uint8_t* out) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (float)((lane * 8 + j) % 17) * 0.37f;
    const float Z = -1.0f, inv = 2500.0f;
    uint64_t blk = (uint64_t)gw * groups_per_warp * 32 + lane;
    uint8_t* seg = out + (size_t)gw * 32 * b;
    for (uint32_t g = 0; g < groups_per_warp; g += PH) {
        Philox4 o[PH];
#pragma unroll
        for (int q = 0; q < PH; ++q) {
            const uint64_t c = blk + (uint64_t)(q * 32);
            o[q] = philox4x32_10((uint32_t)c, (uint32_t)(c >> 32), p.rk);
        }
#pragma unroll
        for (int q = 0; q < PH; ++q) {
            const uint32_t pl = kScalar ? codes_small_s<b>(v, Z, inv, o[q]) : codes_small<b>(v, Z, inv, o[q]);
            if (b == 1) {
                const uint32_t q1 = __shfl_down_sync(0xffffffffu, pl, 1);
                const uint32_t q2 = __shfl_down_sync(0xffffffffu, pl, 2);
                const uint32_t q3 = __shfl_down_sync(0xffffffffu, pl, 3);
                if (!(lane & 3))
                    *reinterpret_cast<uint32_t*>(seg + lane) = pl | (q1 << 8) | (q2 << 16) | (q3 << 24);
            } else {
                const uint32_t q1 = __shfl_down_sync(0xffffffffu, pl, 1);
                if (!(lane & 1)) *reinterpret_cast<uint32_t*>(seg + lane * 2) = pl | (q1 << 16);
            }
            v[0] += 1.0f;
        }
        blk += 32 * PH;
    }
}

// Philox alone, one call per group per lane (the floor of the above)
__global__ void philox_only(const __grid_constant__ P p, uint32_t groups_per_warp, uint32_t* out) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t blk = (uint64_t)gw * groups_per_warp * 32 + lane;
    uint32_t acc = 0;
    for (uint32_t g = 0; g < groups_per_warp; g += 2) {
        const Philox4 a = philox4x32_10((uint32_t)blk, (uint32_t)(blk >> 32), p.rk);
        const Philox4 c = philox4x32_10((uint32_t)(blk + 32), (uint32_t)((blk + 32) >> 32), p.rk);
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ c.x ^ c.y ^ c.z ^ c.w;
        blk += 64;
    }
    if (acc == 0x9u) out[0] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* out;
    cudaMalloc(&out, 1 << 28);
    P p;
    p.rk = make_round_keys(42);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint32_t gpw = 512;
    for (int wps : {16, 32, 48}) {
        const int threads = 256, blocks = sms * wps / 8;
        const double groups = (double)blocks * (threads / 32) * gpw;
        float ms;
#define T(KERN, NAME)                                                                     \
    KERN<<<blocks, threads>>>(p, gpw, (decltype(out))out);                               \
    cudaEventRecord(e0);                                                                  \
    KERN<<<blocks, threads>>>(p, gpw, (decltype(out))out);                               \
    cudaEventRecord(e1);                                                                  \
    cudaEventSynchronize(e1);                                                             \
    cudaEventElapsedTime(&ms, e0, e1);                                                    \
    printf("%-14s warps/SM=%2d: %.3f Ggroups/s = %.2f Telem/s (%.1f SMSP-cycles/group at 1965 MHz)\n", \
           NAME, wps, groups / ms / 1e6, groups * 256 / ms / 1e9,                         \
           sms * 4 * 1.965e6 * ms / groups);
        T((k3_body<1, 2>), "b1 PH2");
        T((k3_body<2, 2>), "b2 PH2");
        T((k3_body<1, 4>), "b1 PH4");
        T((k3_body<1, 2, true>), "b1 PH2 scalar");
        T((k3_body<2, 2, true>), "b2 PH2 scalar");
        philox_only<<<blocks, threads>>>(p, gpw, (uint32_t*)out);
        cudaEventRecord(e0);
        philox_only<<<blocks, threads>>>(p, gpw, (uint32_t*)out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-14s warps/SM=%2d: %.3f Ggroups/s (%.1f SMSP-cycles/group)\n", "philox only", wps,
               groups / ms / 1e6, sms * 4 * 1.965e6 * ms / groups);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
