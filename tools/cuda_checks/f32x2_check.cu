// Standalone check of the sm_100 f32x2 intrinsics in the two patterns K3 uses.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "../../paper_2104_14129_b200/csrc/device.cuh"
using namespace actnn;

__global__ void k(const float* x, const uint32_t* wr, float Z, float inv, uint32_t* outA, uint32_t* outB, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float v[8];
    for (int j = 0; j < 8; ++j) v[j] = x[8 * i + j];
    uint32_t w[4];
    for (int j = 0; j < 4; ++j) w[j] = wr[4 * i + j];
    const float2 nz = make_float2(-Z, -Z), iv = make_float2(inv, inv), mg = make_float2(12582912.0f, 12582912.0f);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float2 d = __fadd2_rn(make_float2(v[2 * p], v[2 * p + 1]), nz);
        const float2 t = __ffma2_rn(d, iv, mg);
        outA[8 * i + 2 * p] = (__float_as_uint(t.x) - 0x4B400000u + (w[p] & 0x3FFFu)) >> 14;
        outA[8 * i + 2 * p + 1] = (__float_as_uint(t.y) - 0x4B400000u + ((w[p] >> 16) & 0x3FFFu)) >> 14;
        for (int h = 0; h < 2; ++h) {
            uint32_t r = (h ? (w[p] >> 16) : w[p]) & 0x3FFFu;
            outB[8 * i + 2 * p + h] = sr_code(v[2 * p + h], Z, inv, r);
        }
    }
}

int main() {
    const int n = 1 << 16;
    float* hx = (float*)malloc(8 * n * 4); uint32_t* hw = (uint32_t*)malloc(16 * n);
    srand(1);
    for (int i = 0; i < 8 * n; ++i) hx[i] = (float)rand() / RAND_MAX * 3.0f - 1.0f;
    for (int i = 0; i < 4 * n; ++i) hw[i] = ((uint32_t)rand() << 16) ^ (uint32_t)rand();
    float* dx; uint32_t *dw, *da, *db;
    cudaMalloc(&dx, 8 * n * 4); cudaMalloc(&dw, 16 * n); cudaMalloc(&da, 32 * n); cudaMalloc(&db, 32 * n);
    cudaMemcpy(dx, hx, 8 * n * 4, cudaMemcpyHostToDevice); cudaMemcpy(dw, hw, 16 * n, cudaMemcpyHostToDevice);
    float Z = -1.0f, inv = 255.0f / 3.0f * 16384.0f;
    k<<<n / 128, 128>>>(dx, dw, Z, inv, da, db, n);
    uint32_t* a = (uint32_t*)malloc(32 * n); uint32_t* b = (uint32_t*)malloc(32 * n);
    cudaMemcpy(a, da, 32 * n, cudaMemcpyDeviceToHost); cudaMemcpy(b, db, 32 * n, cudaMemcpyDeviceToHost);
    long bad = 0; for (int i = 0; i < 8 * n; ++i) if (a[i] != b[i]) { if (bad < 5) printf("mismatch %d: %u %u\n", i, a[i], b[i]); ++bad; }
    printf("f32x2 check: %ld mismatches of %d (%s)\n", bad, 8 * n, cudaGetErrorString(cudaGetLastError()));
    return bad != 0;
}
