// bw_probe.cu -- HBM streaming probes on one B200: which load/store shapes reach
// the roofline.  Not part of the library; guides the K1/K3/K4 designs.
//   read_ldg<U>:  warp-strided units of U x 1 KB, one LDG.256 per lane per KB,
//                 min-reduced in registers (U KB in flight per warp)
//   read_tma<S,KB>: per-warp ring of S stages of KB kilobytes fed by
//                 cp.async.bulk, consumer min-reduces from shared memory
//   write_stg:    STG.256 per lane, 1 KB per warp instruction
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2104_14129_b200/csrc/device.cuh"
using namespace actnn;

template <int U>
__global__ void read_ldg(const float* __restrict__ x, size_t n_kb, float* out) {
    const int lane = threadIdx.x & 31;
    size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
    float acc = 1e30f;
    for (size_t u = w * U; u < n_kb; u += nw * U) {
        float v[U][8];
#pragma unroll
        for (int k = 0; k < U; ++k) load8(x + (u + k) * 256 + lane * 8, v[k]);
#pragma unroll
        for (int k = 0; k < U; ++k)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc = fminf(acc, v[k][j]);
    }
    if (acc == -1.0f) out[0] = acc;
}

template <int S, int KB>
__global__ void read_tma(const float* __restrict__ x, size_t n_kb, float* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    float* ring = reinterpret_cast<float*>(smem) + (size_t)wi * S * KB * 256;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nwb * S * KB * 1024) + wi * S;
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const size_t w = blockIdx.x * (size_t)nwb + wi, nw = (size_t)gridDim.x * nwb;
    const size_t units = n_kb / KB;
    size_t pu = w;
    if (lane == 0)
        for (int s = 0; s < S; ++s, pu += nw)
            if (pu < units) {
                mbar_expect_tx(&bars[s], KB * 1024);
                bulk_g2s(ring + s * KB * 256, x + pu * KB * 256, KB * 1024, &bars[s]);
            }
    float acc = 1e30f;
    int stage = 0;
    uint32_t phase = 0;
    for (size_t u = w; u < units; u += nw) {
        mbar_wait(&bars[stage], phase);
        const float* st = ring + stage * KB * 256;
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            float v[8];
            lds8(st + k * 256 + lane * 8, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc = fminf(acc, v[j]);
        }
        __syncwarp();
        if (lane == 0) {
            if (pu < units) {
                mbar_expect_tx(&bars[stage], KB * 1024);
                bulk_g2s(ring + stage * KB * 256, x + pu * KB * 256, KB * 1024, &bars[stage]);
            }
            pu += nw;
        }
        if (++stage == S) { stage = 0; phase ^= 1; }
    }
    if (acc == -1.0f) out[0] = acc;
}

__global__ void write_stg(float* __restrict__ y, size_t n_kb) {
    const int lane = threadIdx.x & 31;
    size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
    float v[8];
    for (int j = 0; j < 8; ++j) v[j] = (float)(lane + j);
    for (size_t u = w; u < n_kb; u += nw) store8(y + u * 256 + lane * 8, v);
}

// STG.256 with the streaming (evict-first) hint
__global__ void write_stg_cs(float* __restrict__ y, size_t n_kb) {
    const int lane = threadIdx.x & 31;
    size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
    float v[8];
    for (int j = 0; j < 8; ++j) v[j] = (float)(lane + j);
    for (size_t u = w; u < n_kb; u += nw)
        asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(y + u * 256 + lane * 8),
                     "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]),
                     "f"(v[7]) : "memory");
}

// TMA bulk store: each warp owns an KB-kilobyte shared buffer (filled once) and
// streams it to consecutive global chunks with cp.async.bulk.global.shared::cta,
// at most D bulk groups in flight.
template <int KB, int D>
__global__ void write_tma(float* __restrict__ y, size_t n_kb) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    float* buf = reinterpret_cast<float*>(smem) + (size_t)wi * KB * 256;
    for (int i = lane; i < KB * 256; i += 32) buf[i] = (float)i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const size_t w = blockIdx.x * (size_t)nwb + wi, nw = (size_t)gridDim.x * nwb;
    const size_t units = n_kb / KB;
    if (lane == 0) {
        for (size_t u = w; u < units; u += nw) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(y + u * KB * 256),
                         "r"(smem_u32(buf)), "r"(KB * 1024) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(D) : "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

template <class F>
float time_ms(F f, int reps = 10) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const size_t bytes = 4ull << 30, n_kb = bytes / 1024;
    float *x, *y, *out;
    cudaMalloc(&x, bytes);
    cudaMalloc(&y, bytes);
    cudaMalloc(&out, 64);
    cudaMemset(x, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto gbs = [&](float ms) { return bytes / (ms * 1e-3) / 1e9; };
    printf("copy (cudaMemcpy D2D, read+write): %.0f GB/s\n",
           2 * gbs(time_ms([&] { cudaMemcpy(y, x, bytes, cudaMemcpyDeviceToDevice); })));
    for (int bps : {2, 4, 8}) {
        printf("read_ldg<2> 256thr x %d/SM: %.0f GB/s\n", bps,
               gbs(time_ms([&] { read_ldg<2><<<sms * bps, 256>>>(x, n_kb, out); })));
        printf("read_ldg<4> 256thr x %d/SM: %.0f GB/s\n", bps,
               gbs(time_ms([&] { read_ldg<4><<<sms * bps, 256>>>(x, n_kb, out); })));
        printf("read_ldg<8> 256thr x %d/SM: %.0f GB/s\n", bps,
               gbs(time_ms([&] { read_ldg<8><<<sms * bps, 256>>>(x, n_kb, out); })));
    }
#define TMA(S, KB, WARPS, BPS)                                                                   \
    {                                                                                            \
        size_t sm = (size_t)WARPS * S * KB * 1024 + WARPS * S * 8;                               \
        cudaFuncSetAttribute(read_tma<S, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                             (int)sm);                                                           \
        printf("read_tma S=%d KB=%d warps=%d x %d/SM (%zu KB smem/CTA): %.0f GB/s\n", S, KB,     \
               WARPS, BPS, sm / 1024,                                                            \
               gbs(time_ms([&] { read_tma<S, KB><<<sms * BPS, WARPS * 32, sm>>>(x, n_kb, out); }))); \
    }
    TMA(2, 4, 8, 2) TMA(3, 4, 8, 2) TMA(4, 4, 4, 3) TMA(2, 8, 4, 3) TMA(4, 2, 8, 3)
    TMA(3, 4, 4, 4) TMA(2, 4, 12, 2) TMA(6, 2, 8, 2) TMA(2, 16, 2, 3) TMA(4, 8, 2, 3)
    for (int bps : {2, 4, 8})
        printf("write_stg 256thr x %d/SM: %.0f GB/s\n", bps,
               gbs(time_ms([&] { write_stg<<<sms * bps, 256>>>(y, n_kb); })));
    for (int bps : {2, 4, 8})
        printf("write_stg_cs 256thr x %d/SM: %.0f GB/s\n", bps,
               gbs(time_ms([&] { write_stg_cs<<<sms * bps, 256>>>(y, n_kb); })));
#define WT(KB, D, WARPS, BPS)                                                                    \
    {                                                                                            \
        size_t sm = (size_t)WARPS * KB * 1024;                                                   \
        cudaFuncSetAttribute(write_tma<KB, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                             (int)sm);                                                           \
        printf("write_tma KB=%d depth=%d warps=%d x %d/SM: %.0f GB/s\n", KB, D, WARPS, BPS,       \
               gbs(time_ms([&] { write_tma<KB, D><<<sms * BPS, WARPS * 32, sm>>>(y, n_kb); }))); \
    }
    WT(4, 2, 8, 2) WT(4, 4, 8, 2) WT(4, 8, 8, 2) WT(8, 4, 4, 2) WT(16, 4, 4, 2) WT(4, 4, 4, 4)
    WT(2, 8, 8, 4) WT(32, 2, 2, 2)
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
