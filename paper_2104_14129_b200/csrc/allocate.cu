// allocate.cu -- K2: stage-1 per-sample bit allocation, the
// paper's greedy for Prob. 8 computed in one CTA.
//
// The paper pops moves from a binary heap.  Because each sample's moves have
// non-decreasing keys (the per-bit variance slopes grow as the width shrinks),
// the heap's pop sequence is exactly the ascending (key, n, c) order of ALL
// moves, and the greedy stops at the shortest prefix of that order whose freed
// bits reach need = N * L[0] - budget.  K2 finds that prefix without sorting:
//   1. min and max key (non-negative doubles order like their bit patterns);
//      the bits above their highest differing bit are common to every move;
//   2. weighted radix select from that bit down, 11-bit digits: a 2048-bin
//      histogram of freed bits (and of move counts) among the moves matching
//      the prefix so far, warp-aggregated with match.any, and a block scan
//      that finds the digit where the cumulative freed bits reach the
//      remainder; stop as soon as the chosen digit holds <= 32 moves;
//   3. those <= 32 candidates are compacted, sorted by (key, move index) with
//      a one-warp bitonic network and scanned -> the cut move (if more than 32
//      moves share one full 64-bit key, a block scan in index order instead);
//   4. each sample counts its applied moves -> bits[n]; a block scan of
//      per-thread contiguous sample ranges gives the byte offsets off[N+1].
// Results are identical to the oracle's heap (tests/test_gpu_parity.py).
#include "device.cuh"
#include "launch.h"

namespace actnn {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kDigit = 11;
constexpr int kBins = 1 << kDigit;
constexpr int kBinsPerThread = kBins / kThreads;
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

struct Shared {
    int whist[kBins];
    int chist[kBins];
    long long wsum[kWarps];
    unsigned long long kmin[kWarps], kmax[kWarps];
    unsigned long long cand_key[32];
    long long cand_mv[32];
    int cand_freed[32];
    int ncand;
    int digit, dcount;
    long long dbefore;
    unsigned long long keystar;
    long long cut;
};

// Block-wide exclusive scan of one 64-bit value per thread; returns the
// exclusive prefix and writes the block total.
__device__ __forceinline__ long long block_excl_scan(long long v, Shared& sh, long long* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) sh.wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        long long ws = lane < kWarps ? sh.wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(kFull, ws, o);
            if (lane >= o) ws += t;
        }
        if (lane < kWarps) sh.wsum[lane] = ws;
    }
    __syncthreads();
    const long long res = incl - v + (wid > 0 ? sh.wsum[wid - 1] : 0);
    *total = sh.wsum[kWarps - 1];
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(kThreads) allocate_kernel(AParams p) {
    pdl_trigger();  // the next kernel of the stream may start launching
    pdl_wait();     // the previous grid is complete and visible
    __shared__ Shared sh;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int M = p.M;
    const int64_t total_moves = p.N * (int64_t)M;
    const bool any = (p.need > 0 && M > 0);
    uint64_t key_star = 0;
    long long cut = -1;

    if (any) {
        // ---- 1. min / max key
        unsigned long long lmin = ~0ull, lmax = 0ull;
        for (int c = 0; c < M; ++c)
            for (int64_t n = tid; n < p.N; n += kThreads) {
                const uint64_t k = key_bits(p, n, c);
                lmin = min(lmin, (unsigned long long)k);
                lmax = max(lmax, (unsigned long long)k);
            }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            lmin = min(lmin, __shfl_xor_sync(kFull, lmin, o));
            lmax = max(lmax, __shfl_xor_sync(kFull, lmax, o));
        }
        if (lane == 0) {
            sh.kmin[wid] = lmin;
            sh.kmax[wid] = lmax;
        }
        __syncthreads();
        unsigned long long kmin = sh.kmin[0], kmax = sh.kmax[0];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) {
            kmin = min(kmin, sh.kmin[w]);
            kmax = max(kmax, sh.kmax[w]);
        }
        // ---- 2. weighted radix select below the common prefix
        uint64_t prefix, pmask;
        long long rem = p.need;
        long long count = total_moves;  // moves matching the prefix
        int hi;                          // highest undecided bit
        if (kmin == kmax) {
            prefix = kmin;
            pmask = ~0ull;
            hi = -1;
        } else {
            hi = 63 - __clzll((long long)(kmin ^ kmax));
            pmask = hi == 63 ? 0ull : (~0ull << (hi + 1));
            prefix = kmin & pmask;
        }
        while (hi >= 0 && count > 32) {
            const int shift = max(0, hi - kDigit + 1);
            const int width = hi - shift + 1;
            const uint64_t dmask = (width == 64) ? ~0ull : ((1ull << width) - 1ull);
            for (int i = tid; i < kBins; i += kThreads) {
                sh.whist[i] = 0;
                sh.chist[i] = 0;
            }
            __syncthreads();
            for (int c = 0; c < M; ++c) {
                for (int64_t base = 0; base < p.N; base += kThreads) {
                    const int64_t n = base + tid;
                    int digit = kBins;  // sentinel: not a candidate
                    if (n < p.N) {
                        const uint64_t k = key_bits(p, n, c);
                        if (((k ^ prefix) & pmask) == 0) digit = (int)((k >> shift) & dmask);
                    }
                    const unsigned peers = __match_any_sync(kFull, digit);
                    if (digit < kBins && lane == __ffs(peers) - 1) {
                        atomicAdd(&sh.whist[digit], __popc(peers) * p.freed[c]);
                        atomicAdd(&sh.chist[digit], __popc(peers));
                    }
                }
            }
            __syncthreads();
            // scan the bins: thread t owns bins [t*K, t*K + K)
            long long loc = 0;
#pragma unroll
            for (int i = 0; i < kBinsPerThread; ++i) loc += sh.whist[tid * kBinsPerThread + i];
            long long tot;
            const long long excl = block_excl_scan(loc, sh, &tot);
            if (excl < rem && rem <= excl + loc) {
                long long cum = excl;
                for (int i = 0; i < kBinsPerThread; ++i) {
                    const int bin = tid * kBinsPerThread + i;
                    if (cum + sh.whist[bin] >= rem) {
                        sh.digit = bin;
                        sh.dbefore = cum;
                        sh.dcount = sh.chist[bin];
                        break;
                    }
                    cum += sh.whist[bin];
                }
            }
            __syncthreads();
            prefix |= (uint64_t)sh.digit << shift;
            pmask |= dmask << shift;
            rem -= sh.dbefore;
            count = sh.dcount;
            hi = shift - 1;
            __syncthreads();  // sh.digit / dbefore / dcount are rewritten next pass
        }
        if (count <= 32) {
            // ---- 3a. <= 32 candidates: compact, sort by (key, index) in one warp, scan
            if (tid == 0) sh.ncand = 0;
            __syncthreads();
            for (int c = 0; c < M; ++c)
                for (int64_t n = tid; n < p.N; n += kThreads) {
                    const uint64_t k = key_bits(p, n, c);
                    if (((k ^ prefix) & pmask) == 0) {
                        const int slot = atomicAdd(&sh.ncand, 1);
                        sh.cand_key[slot] = k;
                        sh.cand_mv[slot] = n * (long long)M + c;
                        sh.cand_freed[slot] = p.freed[c];
                    }
                }
            __syncthreads();
            if (wid == 0) {
                const int nc = sh.ncand;
                unsigned long long k = lane < nc ? sh.cand_key[lane] : ~0ull;
                long long mv = lane < nc ? sh.cand_mv[lane] : 0x7fffffffffffffffll;
                int fr = lane < nc ? sh.cand_freed[lane] : 0;
                // bitonic sort of 32 (key, mv) pairs across the lanes, ascending
#pragma unroll
                for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
                    for (int stride = size >> 1; stride > 0; stride >>= 1) {
                        const unsigned long long ok = __shfl_xor_sync(kFull, k, stride);
                        const long long om = __shfl_xor_sync(kFull, mv, stride);
                        const int of = __shfl_xor_sync(kFull, fr, stride);
                        const bool up = ((lane & size) == 0);
                        const bool lower = ((lane & stride) == 0);
                        const bool other_less = (ok < k) || (ok == k && om < mv);
                        const bool take = (lower == up) ? other_less : !other_less;
                        if (take && !(ok == k && om == mv)) {
                            k = ok;
                            mv = om;
                            fr = of;
                        }
                    }
                }
                int incl = fr;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                const unsigned ball = __ballot_sync(kFull, (long long)incl >= rem);
                const int src = __ffs(ball) - 1;
                const unsigned long long ks = __shfl_sync(kFull, k, src);
                const long long cm = __shfl_sync(kFull, mv, src);
                if (lane == 0) {
                    sh.keystar = ks;
                    sh.cut = cm;
                }
            }
            __syncthreads();
            key_star = sh.keystar;
            cut = sh.cut;
        } else {
            // ---- 3b. > 32 moves share the full key: cut in (n, c) order
            key_star = prefix;
            if (tid == 0) sh.cut = -1;
            __syncthreads();
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
                    const long long excl = block_excl_scan(xv, sh, &tot);
                    if (xv != 0 && excl + xv >= rem && excl < rem) sh.cut = mv;
                    __syncthreads();
                    if (sh.cut >= 0) break;
                    rem -= tot;
                }
            }
            __syncthreads();
            cut = sh.cut;
        }
    }

    // ---- 4. widths and byte offsets (thread t: a contiguous range of samples)
    const int64_t per = (p.N + kThreads - 1) / kThreads;
    const int64_t n0 = min(p.N, (int64_t)tid * per), n1 = min(p.N, n0 + per);
    auto width = [&](int64_t n) {  // bits of sample n: its applied moves
        int cnt = 0;
        if (any) {
            for (int c = 0; c < M; ++c) {
                const uint64_t k = key_bits(p, n, c);
                const long long mv = n * (long long)M + c;
                if (k < key_star || (k == key_star && mv <= cut)) ++cnt;
            }
        }
        return p.L[cnt];
    };
    long long local = 0;
    for (int64_t n = n0; n < n1; ++n) local += (long long)width(n) * p.unit;
    long long tot;
    long long run = block_excl_scan(local, sh, &tot);
    if (tid == 0) p.off[0] = 0;
    for (int64_t n = n0; n < n1; ++n) {  // recomputed: no read-back of global writes
        const int b = width(n);
        p.bits[n] = (uint8_t)b;
        run += (long long)b * p.unit;
        p.off[n + 1] = run;
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
    launch_pdl(allocate_kernel, 1, kThreads, 0, s, p);
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
