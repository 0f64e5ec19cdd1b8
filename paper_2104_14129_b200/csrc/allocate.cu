// allocate.cu -- K2: stage-1 per-sample bit allocation, the
// paper's greedy for Prob. 8 computed in one CTA.
//
// The paper pops moves from a binary heap.  Because each sample's moves have
// non-decreasing keys (the per-bit variance slopes grow as the width shrinks),
// the heap's pop sequence is exactly the ascending (key, n, c) order of ALL
// moves, and the greedy stops at the shortest prefix of that order whose freed
// bits reach need = N * L[0] - budget.  K2 finds that prefix without sorting:
//   1. weighted radix select over the 64-bit key patterns (non-negative
//      doubles order like their bit patterns), 8 passes of 8 bits: a 256-bin
//      histogram of freed bits among the moves matching the prefix so far
//      (warp-aggregated with match.any), then one warp scans it;
//   2. among moves whose key equals the selected key, a block scan in (n, c)
//      order finds the cut move;
//   3. each sample counts its applied moves -> bits[n]; a block scan of
//      bits[n] * ng * G / 8 gives the byte offsets off[N+1].
// Results are identical to the oracle's heap (tests/test_gpu_allocate.py).
#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

constexpr int kThreads = 1024;
constexpr unsigned kFull = 0xffffffffu;

struct AParams {
    const double* sens;
    const double* gscale;
    int64_t N;
    int64_t need;
    int M;  // moves per sample = levels - 1
    int L[8];
    double slope[8];
    int freed[8];
    int64_t unit;
    uint8_t* bits;
    int64_t* off;
};

__device__ __forceinline__ uint64_t key_bits(const AParams& p, int64_t n, int c) {
    double w = __ldg(p.sens + n);
    if (p.gscale) w = __dmul_rn(w, __ldg(p.gscale + n));
    const double k = __dmul_rn(w, p.slope[c]);
    return k == 0.0 ? 0ull : (uint64_t)__double_as_longlong(k);  // -0 orders as +0
}

// Block-wide inclusive scan of a 64-bit value; returns (inclusive, block total).
__device__ __forceinline__ long long block_incl_scan(long long v, long long* s_wsum,
                                                     long long* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        long long ws = s_wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(kFull, ws, o);
            if (lane >= o) ws += t;
        }
        s_wsum[lane] = ws;
    }
    __syncthreads();
    const long long res = incl + (wid > 0 ? s_wsum[wid - 1] : 0);
    *total = s_wsum[31];
    __syncthreads();  // s_wsum may be reused by the next call
    return res;
}

__global__ void __launch_bounds__(kThreads) allocate_kernel(AParams p) {
    __shared__ int hist[256];
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_rem;
    __shared__ long long s_cut;
    __shared__ long long s_wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int M = p.M;
    const bool any = (p.need > 0 && M > 0);
    uint64_t key_star = 0;
    long long cut = -1;

    if (any) {
        if (tid == 0) {
            s_prefix = 0;
            s_rem = p.need;
            s_cut = -1;
        }
        // ---- 1. weighted radix select of the cut key
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
            __syncthreads();
            const uint64_t prefix = s_prefix;
            const uint64_t hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
            for (int c = 0; c < M; ++c) {
                for (int64_t base = 0; base < p.N; base += kThreads) {
                    const int64_t n = base + tid;
                    int digit = 256;
                    if (n < p.N) {
                        const uint64_t k = key_bits(p, n, c);
                        if (((k ^ prefix) & hmask) == 0) digit = (int)((k >> shift) & 255u);
                    }
                    const unsigned peers = __match_any_sync(kFull, digit);
                    if (digit < 256 && lane == __ffs(peers) - 1)
                        atomicAdd(&hist[digit], __popc(peers) * p.freed[c]);
                }
            }
            __syncthreads();
            if (wid == 0) {
                int loc[8];
                int sum = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    loc[j] = hist[lane * 8 + j];
                    sum += loc[j];
                }
                int incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                const long long rem = s_rem;
                const unsigned ball = __ballot_sync(kFull, (long long)incl >= rem);
                if (lane == __ffs(ball) - 1) {
                    long long cum = incl - sum;
                    for (int j = 0; j < 8; ++j) {
                        if (cum + loc[j] >= rem) {
                            s_prefix = prefix | ((uint64_t)(lane * 8 + j) << shift);
                            s_rem = rem - cum;
                            break;
                        }
                        cum += loc[j];
                    }
                }
            }
            __syncthreads();
        }
        key_star = s_prefix;
        long long rem = s_rem;
        // ---- 2. ties on the cut key, in (n, c) order
        const int64_t total_moves = p.N * (int64_t)M;
        for (int64_t base = 0; base < total_moves; base += kThreads) {
            const int64_t mv = base + tid;
            int xv = 0;
            if (mv < total_moves) {
                const int64_t n = mv / M;
                const int c = (int)(mv - n * M);
                if (key_bits(p, n, c) == key_star) xv = p.freed[c];
            }
            if (__syncthreads_or(xv != 0)) {
                long long tot;
                const long long incl = block_incl_scan(xv, s_wsum, &tot);
                if (xv != 0 && incl >= rem && incl - xv < rem) s_cut = mv;
                __syncthreads();
                if (s_cut >= 0) break;
                rem -= tot;
            }
        }
        __syncthreads();
        cut = s_cut;
    }

    // ---- 3. widths and byte offsets
    long long carry = 0;
    if (tid == 0) p.off[0] = 0;
    for (int64_t base = 0; base < p.N; base += kThreads) {
        const int64_t n = base + tid;
        long long bytes = 0;
        if (n < p.N) {
            int cnt = 0;
            if (any) {
                for (int c = 0; c < M; ++c) {
                    const uint64_t k = key_bits(p, n, c);
                    const long long mv = n * (long long)M + c;
                    if (k < key_star || (k == key_star && mv <= cut)) ++cnt;
                }
            }
            const int b = p.L[cnt];
            p.bits[n] = (uint8_t)b;
            bytes = (long long)b * p.unit;
        }
        long long tot;
        const long long incl = block_incl_scan(bytes, s_wsum, &tot);
        if (n < p.N) p.off[n + 1] = carry + incl;
        carry += tot;
    }
}

__global__ void uniform_bits_kernel(int64_t N, int b, int64_t unit, uint8_t* bits, int64_t* off) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n == 0) off[0] = 0;
    if (n < N) {
        bits[n] = (uint8_t)b;
        off[n + 1] = (n + 1) * (int64_t)b * unit;
    }
}

}  // namespace

cudaError_t launch_allocate(const AllocArgs& a, cudaStream_t s) {
    AParams p;
    p.sens = a.sens;
    p.gscale = a.gscale;
    p.N = a.N;
    p.need = a.need;
    p.M = a.m - 1;
    for (int i = 0; i < 8; ++i) {
        p.L[i] = a.L[i];
        p.slope[i] = a.slope[i];
        p.freed[i] = a.freed[i];
    }
    p.unit = a.unit;
    p.bits = a.bits;
    p.off = a.off;
    allocate_kernel<<<1, kThreads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_uniform_bits(int64_t N, int b, int64_t unit, uint8_t* bits, int64_t* off,
                                cudaStream_t s) {
    const int tb = 256;
    const int64_t blocks = (N + tb - 1) / tb;
    uniform_bits_kernel<<<(unsigned)(blocks > 0 ? blocks : 1), tb, 0, s>>>(N, b, unit, bits, off);
    return cudaGetLastError();
}

}  // namespace actnn
