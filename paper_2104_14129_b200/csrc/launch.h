// launch.h -- internal host launchers (C++ linkage, not exported).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace actnn {

struct QuantArgs {
    const void* x;
    int dt;  // 0 f32, 1 bf16
    int64_t N, D, ng;
    const uint8_t* bits;
    const int64_t* off;
    uint64_t seed;
    int64_t sample_base;
    const float* gmin;
    const float* gmax;
    uint8_t* packed;
    float* zmin;
    float* scale;
    uint32_t* meta;  // NEXT-1 bf16 metadata words (then zmin/scale are null), or null
    bool fast;  // D % 256 == 0 and x aligned for vector loads
};

struct DequantArgs {
    const uint8_t* packed;
    const float* zmin;
    const float* scale;
    const uint32_t* meta;  // NEXT-1 bf16 metadata words (then zmin/scale are null), or null
    const uint8_t* bits;
    const int64_t* off;
    int64_t N, D, ng;
    void* out;
    int out_dt;
    bool fast;
};

struct StatsArgs {
    const void* x;
    int dt;
    int64_t N, D, ng, nch;
    float* gmin;
    float* gmax;
    double* sens;
    double* T;  // workspace [N * nch]
    bool fast;
};

struct AllocArgs {
    const double* sens;
    const double* gscale;
    int64_t N;
    int64_t need;  // N * L[0] - budget (bits to free); <= 0 => all at L[0]
    int m;         // number of levels
    int L[8];      // levels, descending
    double slope[8];
    int freed[8];
    int64_t unit;  // bytes per bit of width per sample: ng * G / 8
    uint8_t* bits;
    int64_t* off;
};

// NEXT-4 contexts.  ReLU pack: x -> mask (+ y if non-null); backward: x = grad_y,
// y = grad_x, mask read.
struct ReluArgs {
    const void* x;
    void* y;
    uint8_t* mask;
    int64_t E;
    int dt;
};

// max pool 2d: forward in = x, out = y, idx written; backward in = grad_y,
// out = grad_x, idx read.
struct PoolArgs {
    const void* in;
    void* out;
    uint8_t* idx;
    int dt;
    int64_t NC, H, W, OH, OW;
    int kh, kw, sh, sw, ph, pw, dh, dw;
};

// NEXT-3 run-time adaptation (adapt.cu)
constexpr int kMaxLayers = 1024;

struct GradArgs {
    const void* g;
    int dt;
    int64_t N, D, ng, nch;
    double* out;
    double* T;  // workspace [N * nch] + 8-byte ticket
    bool fast;
};

struct LayerAllocArgs {
    const double* sens;
    const double* gscale;
    const double* lconst;
    const int64_t* D;  // host [L]
    int64_t L, N;
    int m;          // number of levels
    int Lv[8];      // levels, descending
    int dstep[8];   // Lv[c] - Lv[c+1]
    double slope[8];
    int64_t need;   // sum_l D_l N Lv[0] - b_total
    uint8_t* bits;
    int64_t* budgets;
    void* ws;
};

cudaError_t launch_grad_sqnorm(const GradArgs& a, cudaStream_t s);
cudaError_t launch_gradmag_ema(const double* obs, int64_t N, double rho, double* m,
                               cudaStream_t s);
cudaError_t launch_gradmag_gather(const double* table, const int64_t* ids, int64_t N,
                                  double* est, cudaStream_t s);
cudaError_t launch_gradmag_scatter(double* table, const int64_t* ids, const double* obs,
                                   int64_t N, cudaStream_t s);
size_t allocate_layers_ws_bytes(int64_t L, int64_t N, int m_moves);
cudaError_t launch_allocate_layers(const LayerAllocArgs& a, cudaStream_t s);

cudaError_t launch_relu_pack(const ReluArgs& a, cudaStream_t s);
cudaError_t launch_relu_backward(const ReluArgs& a, cudaStream_t s);
cudaError_t launch_maxpool2d(const PoolArgs& a, bool backward, cudaStream_t s);

cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t s);
cudaError_t launch_quantize_ws(const QuantArgs& a, cudaStream_t s);  // mixed-mode fast path
cudaError_t launch_quantize_sp8(const QuantArgs& a, cudaStream_t s);  // fp32 single pass, 8-group units
cudaError_t launch_dequantize(const DequantArgs& a, cudaStream_t s);
cudaError_t launch_group_stats(const StatsArgs& a, cudaStream_t s);
cudaError_t launch_allocate(const AllocArgs& a, cudaStream_t s);
cudaError_t launch_uniform_bits(int64_t N, int b, int64_t unit, uint8_t* bits, int64_t* off,
                                cudaStream_t s);

// SM count of the current device (cached per device)
int sm_count();

// persistent-grid sizing: min(work, SMs * resident blocks per SM)
int grid_for(const void* kernel, int block, size_t smem, int64_t work_blocks);

// Opt `kernel` into `bytes` of dynamic shared memory on the current device, once
// per (kernel, device) (thread-safe; several GPUs in one process are fine).
void ensure_smem_attr(const void* kernel, size_t bytes);

// Launch with programmatic stream serialization (device.cuh pdl_trigger /
// pdl_wait: only for kernels that wait before touching global memory).
#ifndef ACTNN_PDL
#define ACTNN_PDL 1
#endif
template <typename... P, typename... A>
inline void launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       A... args) {
#if ACTNN_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, args...);
#else
    kernel<<<grid, block, smem, s>>>(args...);
#endif
}

}  // namespace actnn
