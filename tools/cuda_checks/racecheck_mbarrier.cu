// Does compute-sanitizer racecheck model mbarrier arrive/wait ordering?
// One producer warp writes a shared-memory descriptor and arrives on a full
// mbarrier (arrive = release); one consumer warp waits on it (try_wait =
// acquire), reads the descriptor and arrives on an empty mbarrier; the producer
// waits on that before rewriting the descriptor -- the exact hand-off of
// quantize_ws_kernel (Desc).  The program is race-free by the PTX memory model.
// If racecheck reports hazards here, the quantize_ws reports are the same
// false positive.  The __syncthreads variant (mode 1) is the control.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o racecheck_mbarrier racecheck_mbarrier.cu
//   compute-sanitizer --tool racecheck ./racecheck_mbarrier 0   (mbarrier)
//   compute-sanitizer --tool racecheck ./racecheck_mbarrier 1   (__syncthreads)
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n"
                 ::"r"(su(b)), "r"(ph) : "memory");
}

__global__ void handoff(int mode, int rounds, int* out) {
    __shared__ uint64_t full, empty;
    __shared__ int desc[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    int acc = 0;
    for (int r = 0; r < rounds; ++r) {
        if (mode == 0) {
            if (w == 0) {                       // producer
                if (r > 0 && lane == 0) wait(&empty, (r - 1) & 1);
                __syncwarp();
                desc[lane] = r * 32 + lane;
                __syncwarp();
                if (lane == 0) arrive(&full);
            } else {                            // consumer
                wait(&full, r & 1);
                acc += desc[lane];
                __syncwarp();
                if (lane == 0) arrive(&empty);
            }
        } else {
            if (w == 0) desc[lane] = r * 32 + lane;
            __syncthreads();
            if (w == 1) acc += desc[lane];
            __syncthreads();
        }
    }
    if (w == 1) out[lane] = acc;
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    int* d;
    cudaMalloc(&d, 32 * sizeof(int));
    handoff<<<1, 64>>>(mode, 64, d);
    int h[32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long want = 0;
    for (int r = 0; r < 64; ++r) want += r * 32;
    printf("mode %d (%s): lane 0 sum %d (expected %ld) %s\n", mode,
           mode == 0 ? "mbarrier hand-off" : "__syncthreads", h[0], want,
           cudaGetErrorString(cudaGetLastError()));
    return h[0] != want;
}
