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

cudaError_t launch_relu_pack(const ReluArgs& a, cudaStream_t s);
cudaError_t launch_relu_backward(const ReluArgs& a, cudaStream_t s);
cudaError_t launch_maxpool2d(const PoolArgs& a, bool backward, cudaStream_t s);

cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t s);
cudaError_t launch_quantize_ws(const QuantArgs& a, cudaStream_t s);  // mixed-mode fast path
cudaError_t launch_dequantize(const DequantArgs& a, cudaStream_t s);
cudaError_t launch_group_stats(const StatsArgs& a, cudaStream_t s);
cudaError_t launch_allocate(const AllocArgs& a, cudaStream_t s);
cudaError_t launch_uniform_bits(int64_t N, int b, int64_t unit, uint8_t* bits, int64_t* off,
                                cudaStream_t s);

// persistent-grid sizing: min(work, SMs * resident blocks per SM)
int grid_for(const void* kernel, int block, size_t smem, int64_t work_blocks);

}  // namespace actnn
