// Minimal repro of the "f32x2 b >= 3 wrong codes" of round 1.
// Root cause: an NVVM (CUDA 12.9, sm_100a) miscompile, not a memory race.
//
// Element j of a lane's 8 codes goes to bits [4j, 4j+4) of a 32-bit word; the
// codes come from t = fma.rn.f32x2(d, inv, 1.5*2^23) as
//     code = (bits(t.h) - 0x4B400000 + r) >> 14.
// With bits() = __float_as_uint of the .x half of a float2 produced by
// __ffma2_rn, NVVM folds ((v >> 14) << 16) for the .x halves of pairs 2 and 3
// into `add v, -0x2D000000` / `and v, 0xFF000000` WITHOUT the shift left (PTX
// of packed_naive below: `add.s32 %r60, %r37, -754974720; and.b32 %r61, %r60,
// -65536` where the scalar build has `shl.b32 ..., 2` first), so codes 4 and 6
// land in the wrong bits.  The .y halves are correct.  Reading the halves'
// bit patterns through an opaque `mov.b32` (packed_fixed, the form used in
// device.cuh codes_wide) restores the shifts.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -ptx f32x2_miscompile.cu
//   (inspect) / -o f32x2_miscompile && ./f32x2_miscompile (on a B200)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t pack4(const uint32_t c[8]) {
    uint32_t pl = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) pl |= c[j] << (4 * j);
    return pl;
}

__global__ void packed_naive(const float* x, const uint4* w, float Z, float inv, uint32_t* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint4 ww = w[i];
    const uint32_t r[4] = {ww.x, ww.y, ww.z, ww.w};
    const float2 nz = make_float2(-Z, -Z), iv = make_float2(inv, inv),
                 mg = make_float2(12582912.0f, 12582912.0f);
    uint32_t c[8];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float2 d = __fadd2_rn(make_float2(x[8 * i + 2 * p], x[8 * i + 2 * p + 1]), nz);
        const float2 t = __ffma2_rn(d, iv, mg);
        c[2 * p] = (__float_as_uint(t.x) - 0x4B400000u + (r[p] & 0x3FFFu)) >> 14;
        c[2 * p + 1] = (__float_as_uint(t.y) - 0x4B400000u + ((r[p] >> 16) & 0x3FFFu)) >> 14;
    }
    out[i] = pack4(c);
}

__global__ void packed_fixed(const float* x, const uint4* w, float Z, float inv, uint32_t* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint4 ww = w[i];
    const uint32_t r[4] = {ww.x, ww.y, ww.z, ww.w};
    const float2 nz = make_float2(-Z, -Z), iv = make_float2(inv, inv),
                 mg = make_float2(12582912.0f, 12582912.0f);
    uint32_t c[8];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float2 d = __fadd2_rn(make_float2(x[8 * i + 2 * p], x[8 * i + 2 * p + 1]), nz);
        const float2 t = __ffma2_rn(d, iv, mg);
        uint32_t tx, ty;
        asm("mov.b32 %0, %1;" : "=r"(tx) : "f"(t.x));
        asm("mov.b32 %0, %1;" : "=r"(ty) : "f"(t.y));
        c[2 * p] = (tx - 0x4B400000u + (r[p] & 0x3FFFu)) >> 14;
        c[2 * p + 1] = (ty - 0x4B400000u + ((r[p] >> 16) & 0x3FFFu)) >> 14;
    }
    out[i] = pack4(c);
}

__global__ void packed_scalar(const float* x, const uint4* w, float Z, float inv, uint32_t* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint4 ww = w[i];
    const uint32_t r[4] = {ww.x, ww.y, ww.z, ww.w};
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float t = __fmaf_rn(__fsub_rn(x[8 * i + j], Z), inv, 12582912.0f);
        const uint32_t rr = ((j & 1) ? (r[j >> 1] >> 16) : r[j >> 1]) & 0x3FFFu;
        c[j] = (__float_as_uint(t) - 0x4B400000u + rr) >> 14;
    }
    out[i] = pack4(c);
}

int main() {
    const int n = 1 << 16;
    float* hx = new float[8 * n];
    uint32_t* hw = new uint32_t[4 * n];
    uint32_t s = 12345;
    auto rnd = [&] { s = s * 1664525u + 1013904223u; return s; };
    for (int i = 0; i < 8 * n; ++i) hx[i] = (float)(rnd() >> 8) / 16777216.0f * 3.0f - 1.0f;
    for (int i = 0; i < 4 * n; ++i) hw[i] = rnd();
    float* dx; uint4* dw; uint32_t *d0, *d1, *d2;
    cudaMalloc(&dx, 32 * n); cudaMalloc(&dw, 16 * n);
    cudaMalloc(&d0, 4 * n); cudaMalloc(&d1, 4 * n); cudaMalloc(&d2, 4 * n);
    cudaMemcpy(dx, hx, 32 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, hw, 16 * n, cudaMemcpyHostToDevice);
    const float Z = -1.0f, inv = 15.0f / 3.0f * 16384.0f;   // b = 4 over [-1, 2]
    packed_scalar<<<n / 128, 128>>>(dx, dw, Z, inv, d0);
    packed_naive<<<n / 128, 128>>>(dx, dw, Z, inv, d1);
    packed_fixed<<<n / 128, 128>>>(dx, dw, Z, inv, d2);
    uint32_t *a = new uint32_t[n], *b = new uint32_t[n], *c = new uint32_t[n];
    cudaMemcpy(a, d0, 4 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(b, d1, 4 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(c, d2, 4 * n, cudaMemcpyDeviceToHost);
    long bad_naive = 0, bad_fixed = 0;
    for (int i = 0; i < n; ++i) {
        bad_naive += a[i] != b[i];
        bad_fixed += a[i] != c[i];
    }
    printf("f32x2 packing vs scalar: naive %ld / %d words differ, opaque-move %ld / %d (%s)\n",
           bad_naive, n, bad_fixed, n, cudaGetErrorString(cudaGetLastError()));
    return bad_fixed != 0;
}
