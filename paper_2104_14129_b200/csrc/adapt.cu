// adapt.cu -- NEXT-3, the run-time adaptation of P:553-569 on the device:
//   K6 grad_sqnorm_kernel   per-sample ||grad_n||^2 (the gradient factor of
//                           w_n = G/6 ||grad_n||^2 ||R_n||^2)
//   gradmag_ema_kernel      moving average across samples
//   gradmag_gather/scatter  stale per-sample table
//   K5 allocate_layers_kernel  stage 2: Prob. 8 over ALL layers with
//                           the paper's greedy, one cooperative launch
// Arithmetic = the oracle's O14-O17 (DESIGN readings 22-24); no shared code.
#include <cooperative_groups.h>

#include "device.cuh"
#include "launch.h"

namespace cg = cooperative_groups;

namespace actnn {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ K6
// A CTA (8 warps) owns one chunk of 32 groups of one sample; warp w reduces
// groups 4w..4w+3.  Lane l's term of a group is the in-order fp64 sum of the
// squares of its 8 consecutive elements (fma(x, x, a): x^2 is exact in fp64,
// so this is RN(a + x^2)); the 32 lane terms meet in an xor butterfly
// (o = 16..1); the 32 group totals of the chunk meet in a second butterfly
// (lane = group, zero past the sample's end) -> chunk partial T[c][n]; the
// last CTA (ticket) adds the partials in chunk order.  Same structure and
// ticket convention as K1 (stats.cu).
#ifndef ACTNN_K6_U16
#define ACTNN_K6_U16 4
#endif
template <typename T>
struct GCfg {  // groups per warp (8 for bf16 measured 26% slower than 4)
    static constexpr int U = sizeof(T) == 2 ? ACTNN_K6_U16 : 4;
    static constexpr int Block = (kChunk / U) * 32;
};

struct GParams {
    const void* g;
    int64_t N, D, ng, nch;
    double* T;
    double* out;
    unsigned int* ticket;
};

template <typename T, bool kFast>
__global__ void __launch_bounds__(GCfg<T>::Block) grad_sqnorm_kernel(GParams p) {
    constexpr int kGU = GCfg<T>::U;
    constexpr int kGBlock = GCfg<T>::Block;
    __shared__ double sQ[kChunk];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int gw = w * kGU;
    const T* __restrict__ g = static_cast<const T*>(p.g);
    const int64_t tiles = p.N * p.nch;
    // fast path: the next tile's words are in flight while this tile is reduced
    uint4 cur[kGU][2], nxt[kGU][2];
    auto load_tile = [&](int64_t t, uint4 (&q)[kGU][2]) {
        const int64_t n = t / p.nch;
        const int64_t g0 = (t - n * p.nch) * kChunk;
        const int gcount = (int)min((int64_t)kChunk, p.ng - g0);
        const T* src = g + n * p.D + (g0 + gw) * kG + lane * 8;
#pragma unroll
        for (int u = 0; u < kGU; ++u)
            if (gw + u < gcount) ldg_raw8(src + u * kG, q[u]);
    };
    if (kFast && (int64_t)blockIdx.x < tiles) load_tile(blockIdx.x, cur);
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t n = t / p.nch;
        const int64_t c = t - n * p.nch;
        const int64_t g0 = c * kChunk;
        const int gcount = (int)min((int64_t)kChunk, p.ng - g0);
        double myQ = 0.0;
        float v[kGU][8];
        if (kFast) {
            if (t + gridDim.x < tiles) load_tile(t + gridDim.x, nxt);
#pragma unroll
            for (int u = 0; u < kGU; ++u) raw8_f32<T>(cur[u], v[u]);
        } else {
#pragma unroll
            for (int u = 0; u < kGU; ++u) {
                if (gw + u < gcount) {
                    const int64_t i = g0 + gw + u;
                    const int len = (int)min((int64_t)kG, p.D - i * kG);
                    const T* src = g + n * p.D + i * kG;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int idx = lane * 8 + j;
                        v[u][j] = idx < len ? load1(src + idx) : 0.0f;
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kGU; ++u) {
            if (gw + u < gcount) {
                double a = 0.0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const double x = (double)v[u][j];
                    a = __fma_rn(x, x, a);
                }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) a = __dadd_rn(a, __shfl_xor_sync(kFull, a, o));
                if (lane == u) myQ = a;
            }
        }
        if (lane < kGU && gw + lane < gcount) sQ[gw + lane] = myQ;
        __syncthreads();
        if (w == 0) {
            double q = lane < gcount ? sQ[lane] : 0.0;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) q = __dadd_rn(q, __shfl_xor_sync(kFull, q, o));
            if (lane == 0) p.T[c * p.N + n] = q;
        }
        __syncthreads();
        if (kFast) {
#pragma unroll
            for (int u = 0; u < kGU; ++u) {
                cur[u][0] = nxt[u][0];
                cur[u][1] = nxt[u][1];
            }
        }
    }
    __shared__ unsigned int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicInc(p.ticket, gridDim.x - 1) == gridDim.x - 1);
    __syncthreads();
    if (s_last) {
        __threadfence();
        for (int64_t n = threadIdx.x; n < p.N; n += kGBlock) {
            const double s = sum_chunks_in_order(p.T, p.nch, p.N, n);
            p.out[n] = s;
        }
    }
}

template <typename T>
cudaError_t run_sqnorm(const GradArgs& a, cudaStream_t s) {
    GParams p{a.g, a.N, a.D, a.ng, a.nch, a.T, a.out,
              reinterpret_cast<unsigned int*>(a.T + a.N * a.nch)};
    const int64_t tiles = a.N * a.nch;
    if (a.fast) {
        const int grid = grid_for((const void*)grad_sqnorm_kernel<T, true>, GCfg<T>::Block, 0, tiles);
        grad_sqnorm_kernel<T, true><<<grid, GCfg<T>::Block, 0, s>>>(p);
    } else {
        const int grid = grid_for((const void*)grad_sqnorm_kernel<T, false>, GCfg<T>::Block, 0, tiles);
        grad_sqnorm_kernel<T, false><<<grid, GCfg<T>::Block, 0, s>>>(p);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ estimators
// One warp: the canonical sum (32-term chunks, xor butterfly, chunks in
// order), mean = RN(S / N), m <- RN(RN(rho m) + RN(RN(1 - rho) mean)).
__global__ void gradmag_ema_kernel(const double* obs, int64_t N, double rho, double* m) {
    const int lane = threadIdx.x;
    double s = 0.0;
    for (int64_t c = 0; c * 32 < N; ++c) {
        const int64_t i = c * 32 + lane;
        double v = i < N ? obs[i] : 0.0;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, o));
        s = __dadd_rn(s, v);
    }
    if (lane == 0) {
        const double mean = __ddiv_rn(s, (double)N);
        const double a = __dmul_rn(rho, *m);
        const double b = __dmul_rn(__dsub_rn(1.0, rho), mean);
        *m = __dadd_rn(a, b);
    }
}

__global__ void gradmag_gather_kernel(const double* table, const int64_t* ids, int64_t N,
                                      double* est) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n < N) est[n] = table[ids[n]];
}

__global__ void gradmag_scatter_kernel(double* table, const int64_t* ids, const double* obs,
                                       int64_t N) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n < N) table[ids[n]] = obs[n];
}

// ------------------------------------------------------------------ K5
// Stage 2 over K = L*N items (layer-major) with M moves each.  As in
// K2 (allocate.cu), every item's keys are non-decreasing along its moves, so
// the heap's pop sequence is the ascending (key, l, n, c) order of all moves =
// ascending (key, move index) with mv = (l*N + n)*M + c, and the greedy stops
// at the shortest prefix whose freed bits (D_l * (L_c - L_{c+1}) per move)
// reach need = sum_l D_l N L_0 - b_total.  One cooperative launch, one CTA per
// SM, grid-wide barriers between phases:
//   P0  keys RN(RN(w slope_c) / D_l) of all moves into the workspace; the
//       global min/max key (atomicMax of max and of ~min).
//   P1  weighted radix select from the highest differing bit, 11-bit digits:
//       CTA histograms (freed bits and counts, match.any + redux aggregation)
//       flushed to a global histogram (3 rotating buffers, so one barrier per
//       pass); every CTA scans the same global histogram and takes the same
//       digit.  Stops when the chosen bin holds <= 32 moves.
//   P2  the <= 32 candidates are gathered, and every CTA sorts them (one warp,
//       bitonic by (key, index)) and finds the cut; if > 32 moves share one
//       full key, a two-level index-order scan over CTA ranges finds it.
//   P3  each item's width = the level after its applied moves; per-layer
//       budgets b^(l) = sum_n b_ln by warp-aggregated 64-bit atomics.
constexpr int kAThreads = 512;
constexpr int kAWarps = kAThreads / 32;
constexpr int kDigit = 11;
constexpr int kBins = 1 << kDigit;
constexpr int kBinsPerThread = kBins / kAThreads;

struct LWork {  // the device workspace after the key array
    unsigned long long hw[3][kBins];
    unsigned int hc[3][kBins];
    unsigned long long kmax, kmin_inv;
    unsigned long long cand_key[32], cand_mv[32], cand_fr[32];
    unsigned int ncand;
    unsigned int pad;
    long long cut;
    long long partial[1024];
};

struct LParams {
    const double* sens;
    const double* gscale;
    const double* lconst;
    int64_t L, N;
    int M;
    int Lv[8];
    int dstep[8];
    double slope[8];
    int64_t need;
    uint8_t* bits;
    int64_t* budgets;
    uint64_t* keys;
    LWork* wk;
    int64_t D[kMaxLayers];
};

struct LShared {
    unsigned long long whist[kBins];
    unsigned int chist[kBins];
    long long wsum[kAWarps];
    unsigned long long red[kAWarps];
    unsigned long long red2[kAWarps];
    int digit;
    unsigned int dcount;
    long long dbefore;
    unsigned long long keystar;
    long long cut;
};

__device__ __forceinline__ long long block_scan64(long long v, LShared& sh, long long* total) {
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
        long long ws = lane < kAWarps ? sh.wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(kFull, ws, o);
            if (lane >= o) ws += t;
        }
        if (lane < kAWarps) sh.wsum[lane] = ws;
    }
    __syncthreads();
    const long long res = incl - v + (wid > 0 ? sh.wsum[wid - 1] : 0);
    *total = sh.wsum[kAWarps - 1];
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(kAThreads, 1) allocate_layers_kernel(const __grid_constant__ LParams p) {
    __shared__ LShared sh;
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t M = (uint32_t)p.M;
    const uint32_t NM = (uint32_t)(p.N * p.M);
    const uint64_t K = (uint64_t)(p.L * p.N);
    const uint64_t KM = K * M;
    const uint64_t gtid = (uint64_t)blockIdx.x * kAThreads + tid;
    const uint64_t gstride = (uint64_t)gridDim.x * kAThreads;
    LWork& wk = *p.wk;
    const bool any = p.need > 0 && M > 0;
    auto freed_of = [&](uint32_t mv) -> unsigned long long {
        const uint32_t l = mv / NM;
        const uint32_t c = (mv - l * NM) % M;
        return (unsigned long long)p.D[l] * (unsigned long long)p.dstep[c];
    };

    // ---- P0: keys, global min/max, budgets and histogram 0 zeroed
    for (uint64_t i = gtid; i < (uint64_t)p.L; i += gstride) p.budgets[i] = 0;
    for (uint64_t i = gtid; i < (uint64_t)kBins; i += gstride) {
        wk.hw[0][i] = 0ull;
        wk.hc[0][i] = 0u;
    }
    unsigned long long lmax = 0ull, lmin_inv = 0ull;
    if (any) {
        for (uint64_t it = gtid; it < K; it += gstride) {
            const uint32_t l = (uint32_t)(it / (uint64_t)p.N);
            double w = p.sens[it];
            if (p.gscale) w = __dmul_rn(w, p.gscale[it]);
            if (p.lconst) w = __dmul_rn(w, p.lconst[l]);
            const double d = (double)p.D[l];
            for (uint32_t c = 0; c < M; ++c) {
                const double k = __ddiv_rn(__dmul_rn(w, p.slope[c]), d);
                const unsigned long long kb =
                    k == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(k);
                p.keys[it * M + c] = kb;
                lmax = max(lmax, kb);
                lmin_inv = max(lmin_inv, ~kb);
            }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            lmax = max(lmax, __shfl_xor_sync(kFull, lmax, o));
            lmin_inv = max(lmin_inv, __shfl_xor_sync(kFull, lmin_inv, o));
        }
        if (lane == 0) {
            sh.red[wid] = lmax;
            sh.red2[wid] = lmin_inv;
        }
        __syncthreads();
        if (tid == 0) {
            unsigned long long a = 0ull, b = 0ull;
            for (int i = 0; i < kAWarps; ++i) {
                a = max(a, sh.red[i]);
                b = max(b, sh.red2[i]);
            }
            atomicMax(&wk.kmax, a);
            atomicMax(&wk.kmin_inv, b);
        }
    }
    grid.sync();

    unsigned long long key_star = 0ull;
    long long cut = -1;
    if (any) {
        const unsigned long long kmax = *(volatile unsigned long long*)&wk.kmax;
        const unsigned long long kmin = ~*(volatile unsigned long long*)&wk.kmin_inv;
        // ---- P1: weighted radix select
        unsigned long long prefix, pmask;
        long long rem = p.need;
        unsigned long long count = KM;
        int hi;
        if (kmin == kmax) {
            prefix = kmin;
            pmask = ~0ull;
            hi = -1;
        } else {
            hi = 63 - __clzll((long long)(kmin ^ kmax));
            pmask = hi == 63 ? 0ull : (~0ull << (hi + 1));
            prefix = kmin & pmask;
        }
        int pass = 0;
        while (hi >= 0 && count > 32) {
            const int shift = max(0, hi - kDigit + 1);
            const int width = hi - shift + 1;
            const unsigned long long dmask = (width == 64) ? ~0ull : ((1ull << width) - 1ull);
            const int buf = pass % 3;
            for (int i = tid; i < kBins; i += kAThreads) {
                sh.whist[i] = 0ull;
                sh.chist[i] = 0u;
            }
            // the buffer of pass + 1 is free: its last reads (pass - 2's
            // selection) precede the barrier that ended pass - 1
            for (uint64_t i = gtid; i < (uint64_t)kBins; i += gstride) {
                wk.hw[(pass + 1) % 3][i] = 0ull;
                wk.hc[(pass + 1) % 3][i] = 0u;
            }
            __syncthreads();
            for (uint64_t base = (uint64_t)blockIdx.x * kAThreads; base < KM; base += gstride) {
                const uint64_t mv = base + tid;
                int digit = kBins;
                unsigned int fr = 0u;
                if (mv < KM) {
                    const unsigned long long k = p.keys[mv];
                    if (((k ^ prefix) & pmask) == 0) {
                        digit = (int)((k >> shift) & dmask);
                        fr = (unsigned int)freed_of((uint32_t)mv);
                    }
                }
                const unsigned peers = __match_any_sync(kFull, digit);
                const unsigned int fsum = __reduce_add_sync(peers, fr);
                if (digit < kBins && lane == __ffs(peers) - 1) {
                    atomicAdd(&sh.whist[digit], (unsigned long long)fsum);
                    atomicAdd(&sh.chist[digit], (unsigned int)__popc(peers));
                }
            }
            __syncthreads();
            for (int i = tid; i < kBins; i += kAThreads)
                if (sh.chist[i]) {
                    atomicAdd(&wk.hw[buf][i], sh.whist[i]);
                    atomicAdd(&wk.hc[buf][i], sh.chist[i]);
                }
            grid.sync();
            // every CTA scans the same global histogram
            long long loc = 0;
            unsigned long long hv[kBinsPerThread];
#pragma unroll
            for (int i = 0; i < kBinsPerThread; ++i) {
                hv[i] = __ldcg(&wk.hw[buf][tid * kBinsPerThread + i]);
                loc += (long long)hv[i];
            }
            long long tot;
            const long long excl = block_scan64(loc, sh, &tot);
            if (excl < rem && rem <= excl + loc) {
                long long cum = excl;
                for (int i = 0; i < kBinsPerThread; ++i) {
                    const int bin = tid * kBinsPerThread + i;
                    if (cum + (long long)hv[i] >= rem) {
                        sh.digit = bin;
                        sh.dbefore = cum;
                        sh.dcount = __ldcg(&wk.hc[buf][bin]);
                        break;
                    }
                    cum += (long long)hv[i];
                }
            }
            __syncthreads();
            prefix |= (unsigned long long)sh.digit << shift;
            pmask |= dmask << shift;
            rem -= sh.dbefore;
            count = sh.dcount;
            hi = shift - 1;
            ++pass;
            __syncthreads();
        }
        if (count <= 32) {
            // ---- P2a: gather the <= 32 candidates; every CTA sorts them
            for (uint64_t mv = gtid; mv < KM; mv += gstride) {
                const unsigned long long k = p.keys[mv];
                if (((k ^ prefix) & pmask) == 0) {
                    const unsigned int slot = atomicAdd(&wk.ncand, 1u);
                    wk.cand_key[slot] = k;
                    wk.cand_mv[slot] = mv;
                    wk.cand_fr[slot] = freed_of((uint32_t)mv);
                }
            }
            grid.sync();
            if (wid == 0) {
                const int nc = (int)*(volatile unsigned int*)&wk.ncand;
                unsigned long long k = lane < nc ? __ldcg(&wk.cand_key[lane]) : ~0ull;
                unsigned long long mv = lane < nc ? __ldcg(&wk.cand_mv[lane]) : ~0ull;
                long long fr = lane < nc ? (long long)__ldcg(&wk.cand_fr[lane]) : 0;
#pragma unroll
                for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
                    for (int stride = size >> 1; stride > 0; stride >>= 1) {
                        const unsigned long long ok = __shfl_xor_sync(kFull, k, stride);
                        const unsigned long long om = __shfl_xor_sync(kFull, mv, stride);
                        const long long of = __shfl_xor_sync(kFull, fr, stride);
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
                long long incl = fr;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                const unsigned ball = __ballot_sync(kFull, incl >= rem);
                const int src = __ffs(ball) - 1;
                const unsigned long long ks = __shfl_sync(kFull, k, src);
                const unsigned long long cm = __shfl_sync(kFull, mv, src);
                if (lane == 0) {
                    sh.keystar = ks;
                    sh.cut = (long long)cm;
                }
            }
            __syncthreads();
            key_star = sh.keystar;
            cut = sh.cut;
        } else {
            // ---- P2b: > 32 moves share the full key: cut in index order
            key_star = prefix;
            const uint64_t per = (KM + gridDim.x - 1) / gridDim.x;
            const uint64_t lo = min(KM, (uint64_t)blockIdx.x * per), hi2 = min(KM, lo + per);
            long long mine = 0;
            for (uint64_t mv = lo + tid; mv < hi2; mv += kAThreads)
                if (p.keys[mv] == key_star) mine += (long long)freed_of((uint32_t)mv);
            long long tot;
            (void)block_scan64(mine, sh, &tot);
            if (tid == 0) wk.partial[blockIdx.x] = tot;
            grid.sync();
            long long before = 0;
            for (unsigned int b = 0; b < blockIdx.x; ++b) before += __ldcg(&wk.partial[b]);
            long long r = rem - before;
            if (r > 0 && r <= tot) {
                if (tid == 0) sh.cut = -1;
                __syncthreads();
                for (uint64_t base = lo; base < hi2; base += kAThreads) {
                    const uint64_t mv = base + tid;
                    long long xv = 0;
                    if (mv < hi2 && p.keys[mv] == key_star) xv = (long long)freed_of((uint32_t)mv);
                    long long t2;
                    const long long ex = block_scan64(xv, sh, &t2);
                    if (xv != 0 && ex < r && ex + xv >= r) sh.cut = (long long)mv;
                    __syncthreads();
                    if (sh.cut >= 0) break;
                    r -= t2;
                }
                if (tid == 0) wk.cut = sh.cut;
            }
            grid.sync();
            cut = *(volatile long long*)&wk.cut;
        }
    }
    grid.sync();  // every read of the shared words is done: reset them
    if (blockIdx.x == 0 && tid == 0) {
        wk.kmax = 0ull;
        wk.kmin_inv = 0ull;
        wk.ncand = 0u;
        wk.cut = 0;
    }

    // ---- P3: widths and per-layer budgets
    for (uint64_t base = (uint64_t)blockIdx.x * kAThreads; base < K; base += gstride) {
        const uint64_t it = base + tid;
        unsigned int l = 0xffffffffu, b = 0u;
        if (it < K) {
            int cnt = 0;
            if (any)
                for (uint32_t c = 0; c < M; ++c) {
                    const unsigned long long k = p.keys[it * M + c];
                    const long long mv = (long long)(it * M + c);
                    if (k < key_star || (k == key_star && mv <= cut)) ++cnt;
                }
            b = (unsigned int)p.Lv[cnt];
            p.bits[it] = (uint8_t)b;
            l = (unsigned int)(it / (uint64_t)p.N);
        }
        const unsigned peers = __match_any_sync(kFull, l);
        const unsigned int s = __reduce_add_sync(peers, b);
        if (l != 0xffffffffu && lane == __ffs(peers) - 1)
            atomicAdd(reinterpret_cast<unsigned long long*>(&p.budgets[l]),
                      (unsigned long long)s);
    }
}

}  // namespace

cudaError_t launch_grad_sqnorm(const GradArgs& a, cudaStream_t s) {
    return a.dt == 0 ? run_sqnorm<float>(a, s) : run_sqnorm<uint16_t>(a, s);
}

cudaError_t launch_gradmag_ema(const double* obs, int64_t N, double rho, double* m,
                               cudaStream_t s) {
    gradmag_ema_kernel<<<1, 32, 0, s>>>(obs, N, rho, m);
    return cudaGetLastError();
}

cudaError_t launch_gradmag_gather(const double* table, const int64_t* ids, int64_t N,
                                  double* est, cudaStream_t s) {
    gradmag_gather_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(table, ids, N, est);
    return cudaGetLastError();
}

cudaError_t launch_gradmag_scatter(double* table, const int64_t* ids, const double* obs,
                                   int64_t N, cudaStream_t s) {
    gradmag_scatter_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(table, ids, obs, N);
    return cudaGetLastError();
}

size_t allocate_layers_ws_bytes(int64_t L, int64_t N, int M) {
    const size_t keys = (size_t)(L * N * (int64_t)(M > 0 ? M : 0)) * 8;
    return ((keys + 255) / 256) * 256 + sizeof(LWork);
}

cudaError_t launch_allocate_layers(const LayerAllocArgs& a, cudaStream_t s) {
    LParams q;
    q.sens = a.sens;
    q.gscale = a.gscale;
    q.lconst = a.lconst;
    q.L = a.L;
    q.N = a.N;
    q.M = a.m - 1;
    for (int i = 0; i < 8; ++i) {
        q.Lv[i] = a.Lv[i];
        q.dstep[i] = a.dstep[i];
        q.slope[i] = a.slope[i];
    }
    q.need = a.need;
    q.bits = a.bits;
    q.budgets = a.budgets;
    q.keys = reinterpret_cast<uint64_t*>(a.ws);
    const size_t keys = (size_t)(a.L * a.N * (int64_t)(a.m - 1)) * 8;
    q.wk = reinterpret_cast<LWork*>(static_cast<uint8_t*>(a.ws) + ((keys + 255) / 256) * 256);
    for (int64_t l = 0; l < a.L; ++l) q.D[l] = a.D[l];
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, allocate_layers_kernel, kAThreads, 0);
    if (occ < 1) return cudaErrorInvalidConfiguration;
    int grid = sms;  // one CTA per SM (co-resident: cooperative launch checks it)
    const int64_t work = (a.L * a.N * (int64_t)(a.m > 1 ? a.m - 1 : 1) + kAThreads - 1) / kAThreads;
    if (work < grid) grid = (int)(work < 1 ? 1 : work);
    if (grid > 1024) grid = 1024;
    void* args[] = {&q};
    return cudaLaunchCooperativeKernel((const void*)allocate_layers_kernel, dim3(grid),
                                       dim3(kAThreads), args, 0, s);
}

}  // namespace actnn
