// philox_rate.cu -- Philox4x32-10 throughput on one B200 as a function of the
// number of independent chains per thread (ILP) and of occupancy.  Guides K3:
// one call per 256-element group per lane (8 elements).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2104_14129_b200/csrc/device.cuh"
using namespace actnn;

struct P {
    RoundKeys rk;
};

template <int ILP>
__global__ void philox_kernel(const __grid_constant__ P p, uint32_t iters, uint32_t* out) {
    uint32_t acc = 0;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t i = 0; i < iters; ++i) {
        Philox4 o[ILP];
#pragma unroll
        for (int q = 0; q < ILP; ++q) o[q] = philox4x32_10(t * 977 + i * ILP + q, 0u, p.rk);
#pragma unroll
        for (int q = 0; q < ILP; ++q) acc ^= o[q].x ^ o[q].y ^ o[q].z ^ o[q].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 4);
    P p;
    p.rk = make_round_keys(42);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint32_t iters = 2048;
#define RUN(ILP, WPS)                                                                         \
    {                                                                                         \
        const int threads = 256, blocks = sms * WPS / 8;                                      \
        philox_kernel<ILP><<<blocks, threads>>>(p, iters / ILP, out);                         \
        cudaEventRecord(a);                                                                   \
        philox_kernel<ILP><<<blocks, threads>>>(p, iters / ILP, out);                         \
        cudaEventRecord(b);                                                                   \
        cudaEventSynchronize(b);                                                              \
        float ms;                                                                             \
        cudaEventElapsedTime(&ms, a, b);                                                      \
        const double calls = (double)blocks * threads * iters;                                \
        printf("ILP=%d warps/SM=%2d: %.2f Gcalls/s = %.2f TB/s of fp32 input-equivalent "     \
               "(8 elem/call)\n", ILP, WPS, calls / ms / 1e6, calls * 32 / ms / 1e9);         \
    }
    RUN(1, 16) RUN(2, 16) RUN(4, 16) RUN(1, 32) RUN(2, 32) RUN(4, 32) RUN(1, 64) RUN(2, 64)
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
