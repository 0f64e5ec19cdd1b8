// small_write.cu -- the floor of a serial, event-timed launch that writes an
// output of the K4 tensor sizes (what "K4 at 0.63 on small tensors" should be
// compared with): an empty kernel, and a write-only kernel (STG.128 / STG.256
// per thread on a persistent grid) for 25.7 / 51.4 / 102.8 / 205.5 / 822 MB.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a small_write.cu -o small_write
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void empty_k() {}

// PDL: let the next launch in the stream start (griddepcontrol.launch_dependents),
// then wait for the previous grid's completion before touching memory
__global__ void write_pdl_k(float4* out, size_t n4) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
        out[i] = make_float4(1.f, 2.f, 3.f, (float)i);
}

__global__ void write_k(float4* out, size_t n4) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
        out[i] = make_float4(1.f, 2.f, 3.f, (float)i);
}

// read a small packed buffer (1/16 of the output) and write the output, like K4 at 2 bits
__global__ void k4like_k(const uint2* in, float4* out, size_t n4) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint2 v = __ldg(in + (i >> 3));
        out[i] = make_float4((float)(v.x & 3), (float)(v.y & 3), 3.f, (float)i);
    }
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t maxb = (size_t)900 << 20;
    float4* out;
    uint2* in;
    cudaMalloc(&out, maxb);
    cudaMalloc(&in, maxb / 16 + 64);
    cudaMemset(in, 0, maxb / 16 + 64);
    float* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int r = 0; r < 3; ++r) {
        empty_k<<<sms, 256>>>();
        cudaEventRecord(e0);
        empty_k<<<sms, 256>>>();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("empty kernel: %.2f us\n", ms * 1e3);
    }
    // back-to-back launches in one stream, one event pair around 8 of them
    for (double mb : {0.0, 2.1, 25.7, 102.8}) {
        const size_t n4 = (size_t)(mb * 1e6) / 16;
        for (int pdl = 0; pdl < 2; ++pdl) {
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0);
                for (int k = 0; k < 8; ++k) {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(sms * 8);
                    cfg.blockDim = dim3(256);
                    cfg.stream = 0;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    at[0].val.programmaticStreamSerializationAllowed = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = pdl;
                    cudaLaunchKernelEx(&cfg, write_pdl_k, out, n4);
                }
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("sequence of 8: %6.1f MB writes, PDL %d: %.2f us per launch\n", mb, pdl, best * 1e3 / 8);
        }
    }
    for (double mb : {25.7, 51.4, 102.8, 205.5, 822.1}) {
        const size_t n4 = (size_t)(mb * 1e6) / 16;
        for (int blocksPerSM : {4, 8, 16}) {
            float best = 1e9, best2 = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaMemset(flush, r, 256 << 20);
                cudaEventRecord(e0);
                write_k<<<sms * blocksPerSM, 256>>>(out, n4);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
                cudaMemset(flush, r, 256 << 20);
                cudaEventRecord(e0);
                k4like_k<<<sms * blocksPerSM, 256>>>(in, out, n4);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                best2 = ms < best2 ? ms : best2;
            }
            printf("%7.1f MB  %2d CTA/SM  write-only %7.1f us (%6.0f GB/s)  k4-like %7.1f us (%6.0f GB/s)\n",
                   mb, blocksPerSM, best * 1e3, n4 * 16 / (best * 1e-3) / 1e9, best2 * 1e3,
                   n4 * 16 * 17 / 16 / (best2 * 1e-3) / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
