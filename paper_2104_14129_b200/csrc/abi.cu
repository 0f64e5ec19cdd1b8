// abi.cu -- the C ABI of libactnn.so (include/actnn.h): host-side argument
// checks, launch-shape selection and error reporting.  No allocation, no
// synchronisation (except the opt-in ACTNN_CHECK=1 debug mode), no copies.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/actnn.h"
#include "launch.h"

namespace actnn {

namespace {
thread_local char g_err[512] = "";

actnn_status_t fail(actnn_status_t st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

actnn_status_t cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return ACTNN_OK;
    return fail(ACTNN_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ACTNN_CHECK is read once, when the library is loaded (the only environment
// variable the library reads).
const bool g_check_mode = [] {
    const char* v = std::getenv("ACTNN_CHECK");
    return v != nullptr && v[0] != '\0' && v[0] != '0';
}();

bool check_mode() { return g_check_mode; }

bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }
int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ACTNN_CHECK=1: synchronise and validate the device-resident widths/offsets.
actnn_status_t debug_validate(const uint8_t* bits, const int64_t* off, int64_t N, int64_t ng,
                              cudaStream_t s) {
    if (!check_mode()) return ACTNN_OK;
    std::vector<uint8_t> hb((size_t)N);
    std::vector<int64_t> ho((size_t)N + 1);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMemcpy(hb.data(), bits, (size_t)N, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess)
        e = cudaMemcpy(ho.data(), off, sizeof(int64_t) * (size_t)(N + 1), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_status(e, "ACTNN_CHECK copy");
    for (int64_t n = 0; n < N; ++n) {
        if (hb[n] < 1 || hb[n] > 8)
            return fail(ACTNN_ERR_CHECK, "ACTNN_CHECK: bits[%lld] = %d outside 1..8", (long long)n,
                        (int)hb[n]);
        if (ho[n + 1] - ho[n] != (int64_t)hb[n] * ng * 32)
            return fail(ACTNN_ERR_CHECK, "ACTNN_CHECK: off[%lld..%lld] inconsistent with bits",
                        (long long)n, (long long)n + 1);
    }
    return ACTNN_OK;
}

actnn_status_t post_launch(cudaError_t e, const char* what, cudaStream_t s) {
    if (e != cudaSuccess) return cuda_status(e, what);
    if (check_mode()) return cuda_status(cudaStreamSynchronize(s), what);
    return ACTNN_OK;
}

struct DeviceInfo {
    int sms = 0;
};
std::mutex g_dev_mu;
std::vector<DeviceInfo> g_dev;
}  // namespace

void ensure_smem_attr(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;  // (kernel, device)
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& e : done)
        if (e.first == kernel && e.second == dev) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    done.emplace_back(kernel, dev);
}

int sm_count() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
    if (g_dev[dev].sms == 0)
        cudaDeviceGetAttribute(&g_dev[dev].sms, cudaDevAttrMultiProcessorCount, dev);
    return g_dev[dev].sms;
}

int grid_for(const void* kernel, int block, size_t smem, int64_t work_blocks) {
    const int sms = sm_count();
    // resident blocks per SM, computed once per (kernel, block, smem)
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int64_t>, int>> occ_cache;
    const int64_t shape = ((int64_t)block << 32) | (int64_t)smem;
    int occ = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const auto& e : occ_cache)
            if (e.first.first == kernel && e.first.second == shape) occ = e.second;
        if (occ == 0) {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, smem) !=
                    cudaSuccess ||
                occ < 1)
                occ = 1;
            occ_cache.push_back({{kernel, shape}, occ});
        }
    }
    const int64_t cap = (int64_t)sms * occ;
    int64_t g = work_blocks < cap ? work_blocks : cap;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace actnn

using namespace actnn;

extern "C" {

const char* actnn_last_error(void) { return g_err; }

int actnn_abi_version(void) { return ACTNN_ABI_VERSION; }

size_t actnn_workspace_bytes(int op, int64_t N, int64_t D, int32_t G) {
    if (N <= 0 || D <= 0 || G <= 0) return 0;
    if (op == ACTNN_OP_GROUP_STATS || op == ACTNN_OP_GRAD_SQNORM)
        return (size_t)(N * ceil_div(ceil_div(D, G), 32)) * 8 + 8;
    return 0;
}

int64_t actnn_packed_bytes(int64_t N, int64_t D, int32_t G, const uint8_t* bits_host) {
    if (N < 0 || D < 0 || G <= 0 || G % 8) return -1;
    const int64_t ng = ceil_div(D, G);
    if (!bits_host) return N * ng * G;  // 8-bit bound
    int64_t s = 0;
    for (int64_t n = 0; n < N; ++n) {
        if (bits_host[n] < 1 || bits_host[n] > 8) return -1;
        s += (int64_t)bits_host[n] * ng * G / 8;
    }
    return s;
}

static actnn_status_t common_checks(int64_t N, int64_t D, int32_t G) {
    if (N < 0 || D < 0) return fail(ACTNN_ERR_INVALID, "negative size N=%lld D=%lld",
                                    (long long)N, (long long)D);
    if (G != 256) return fail(ACTNN_ERR_UNSUPPORTED, "G=%d unsupported (ABI v1: G=256)", G);
    return ACTNN_OK;
}

static bool dtype_ok(int dt) { return dt == ACTNN_F32 || dt == ACTNN_BF16; }

actnn_status_t actnn_group_stats(const void* x, actnn_dtype_t dt, int64_t N, int64_t D, int32_t G,
                                 float* gmin, float* gmax, double* sens, void* ws,
                                 size_t ws_bytes, void* stream) {
    actnn_status_t st = common_checks(N, D, G);
    if (st) return st;
    if (!dtype_ok(dt)) return fail(ACTNN_ERR_INVALID, "bad dtype %d", (int)dt);
    if (N == 0 || D == 0) return ACTNN_OK;
    if (!x || !gmin || !gmax || !sens || !ws)
        return fail(ACTNN_ERR_INVALID, "actnn_group_stats: null pointer");
    const size_t es = dt == ACTNN_F32 ? 4 : 2;
    if (!aligned(x, es) || !aligned(gmin, 4) || !aligned(gmax, 4) || !aligned(sens, 8) ||
        !aligned(ws, 8))
        return fail(ACTNN_ERR_INVALID, "actnn_group_stats: misaligned pointer");
    if (ws_bytes < actnn_workspace_bytes(ACTNN_OP_GROUP_STATS, N, D, G))
        return fail(ACTNN_ERR_INVALID, "actnn_group_stats: workspace %zu < %zu bytes", ws_bytes,
                    actnn_workspace_bytes(ACTNN_OP_GROUP_STATS, N, D, G));
    StatsArgs a;
    a.x = x;
    a.dt = (int)dt;
    a.N = N;
    a.D = D;
    a.ng = ceil_div(D, G);
    a.nch = ceil_div(a.ng, 32);
    a.gmin = gmin;
    a.gmax = gmax;
    a.sens = sens;
    a.T = static_cast<double*>(ws);
    a.fast = (D % G == 0) && aligned(x, dt == ACTNN_F32 ? 32 : 16);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_group_stats(a, s), "actnn_group_stats", s);
}

static actnn_status_t levels_from_mask(uint32_t mask, int* L, int* m) {
    if (mask == 0 || (mask & ~0x1FEu))
        return fail(ACTNN_ERR_INVALID, "level_mask 0x%x must be a non-empty subset of bits 1..8",
                    mask);
    *m = 0;
    for (int b = 8; b >= 1; --b)
        if (mask & (1u << b)) L[(*m)++] = b;
    return ACTNN_OK;
}

actnn_status_t actnn_allocate_bits(const double* sens, const double* gscale, int64_t N,
                                   int64_t budget, uint32_t level_mask, int64_t D, int32_t G,
                                   uint8_t* bits, int64_t* off, void* ws, size_t ws_bytes,
                                   void* stream) {
    (void)ws;
    (void)ws_bytes;
    actnn_status_t st = common_checks(N, D, G);
    if (st) return st;
    AllocArgs a;
    std::memset(&a, 0, sizeof(a));
    st = levels_from_mask(level_mask, a.L, &a.m);
    if (st) return st;
    if (budget < N * (int64_t)a.L[a.m - 1])
        return fail(ACTNN_ERR_BUDGET, "budget %lld < N * %d = %lld (infeasible)",
                    (long long)budget, a.L[a.m - 1], (long long)(N * a.L[a.m - 1]));
    if (N == 0) {
        if (!off) return fail(ACTNN_ERR_INVALID, "actnn_allocate_bits: null off");
        return cuda_status(cudaMemsetAsync(off, 0, sizeof(int64_t), (cudaStream_t)stream),
                           "actnn_allocate_bits");
    }
    if (!sens || !bits || !off) return fail(ACTNN_ERR_INVALID, "actnn_allocate_bits: null pointer");
    if (!aligned(sens, 8) || !aligned(off, 8) || (gscale && !aligned(gscale, 8)))
        return fail(ACTNN_ERR_INVALID, "actnn_allocate_bits: misaligned pointer");
    // per-bit variance slope of each move (Eq. 8 with B = 2^b - 1): the move
    // from L[c] to L[c+1] raises w/B^2 by w (1/B_{c+1}^2 - 1/B_c^2) and frees
    // L[c] - L[c+1] bits (DESIGN reading 9).
    for (int c = 0; c + 1 < a.m; ++c) {
        const double Bh = (double)((1 << a.L[c]) - 1), Bl = (double)((1 << a.L[c + 1]) - 1);
        const double fh = 1.0 / (Bh * Bh), fl = 1.0 / (Bl * Bl);
        a.freed[c] = a.L[c] - a.L[c + 1];
        a.slope[c] = (fl - fh) / (double)a.freed[c];
    }
    a.sens = sens;
    a.gscale = gscale;
    a.N = N;
    a.need = N * (int64_t)a.L[0] - budget;
    a.unit = ceil_div(D, G) * G / 8;
    a.bits = bits;
    a.off = off;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_allocate(a, s), "actnn_allocate_bits", s);
}

actnn_status_t actnn_uniform_bits(int64_t N, int64_t D, int32_t G, int32_t b, uint8_t* bits,
                                  int64_t* off, void* stream) {
    actnn_status_t st = common_checks(N, D, G);
    if (st) return st;
    if (b < 1 || b > 8) return fail(ACTNN_ERR_INVALID, "width %d outside 1..8", b);
    if (!off || (N > 0 && !bits)) return fail(ACTNN_ERR_INVALID, "actnn_uniform_bits: null pointer");
    if (!aligned(off, 8)) return fail(ACTNN_ERR_INVALID, "actnn_uniform_bits: misaligned off");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_uniform_bits(N, b, ceil_div(D, G) * G / 8, bits, off, s),
                       "actnn_uniform_bits", s);
}

// Shared body of actnn_quantize / actnn_quantize_bf16meta: exactly one of
// (zmin, scale) and meta is in use.
static actnn_status_t quantize_impl(const char* fn, const void* x, actnn_dtype_t dt, int64_t N,
                                    int64_t D, int32_t G, const uint8_t* bits, const int64_t* off,
                                    uint64_t seed, int64_t sample_base, const float* gmin,
                                    const float* gmax, uint8_t* packed, float* zmin, float* scale,
                                    uint32_t* meta, void* stream) {
    actnn_status_t st = common_checks(N, D, G);
    if (st) return st;
    if (!dtype_ok(dt)) return fail(ACTNN_ERR_INVALID, "bad dtype %d", (int)dt);
    if (sample_base < 0) return fail(ACTNN_ERR_INVALID, "negative sample_base");
    if (N == 0 || D == 0) return ACTNN_OK;
    if (!x || !bits || !off || !packed || (meta ? false : (!zmin || !scale)))
        return fail(ACTNN_ERR_INVALID, "%s: null pointer", fn);
    if ((gmin == nullptr) != (gmax == nullptr))
        return fail(ACTNN_ERR_INVALID, "%s: gmin and gmax must both be set or NULL", fn);
    const size_t es = dt == ACTNN_F32 ? 4 : 2;
    if (!aligned(x, es) || !aligned(off, 8) || (zmin && !aligned(zmin, 4)) ||
        (scale && !aligned(scale, 4)) || (meta && !aligned(meta, 4)) ||
        (gmin && (!aligned(gmin, 4) || !aligned(gmax, 4))))
        return fail(ACTNN_ERR_INVALID, "%s: misaligned pointer", fn);
    if (!aligned(packed, 16))
        return fail(ACTNN_ERR_UNSUPPORTED, "%s: packed must be 16-byte aligned", fn);
    const int64_t ng = ceil_div(D, G);
    st = debug_validate(bits, off, N, ng, (cudaStream_t)stream);
    if (st) return st;
    QuantArgs a;
    a.x = x;
    a.dt = (int)dt;
    a.N = N;
    a.D = D;
    a.ng = ng;
    a.bits = bits;
    a.off = off;
    a.seed = seed;
    a.sample_base = sample_base;
    a.gmin = gmin;
    a.gmax = gmax;
    a.packed = packed;
    a.zmin = meta ? nullptr : zmin;
    a.scale = meta ? nullptr : scale;
    a.meta = meta;
    a.fast = (D % G == 0) && aligned(x, dt == ACTNN_F32 ? 32 : 16);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_quantize(a, s), fn, s);
}

actnn_status_t actnn_quantize(const void* x, actnn_dtype_t dt, int64_t N, int64_t D, int32_t G,
                              const uint8_t* bits, const int64_t* off, uint64_t seed,
                              int64_t sample_base, const float* gmin, const float* gmax,
                              uint8_t* packed, float* zmin, float* scale, void* stream) {
    return quantize_impl("actnn_quantize", x, dt, N, D, G, bits, off, seed, sample_base, gmin,
                         gmax, packed, zmin, scale, nullptr, stream);
}

actnn_status_t actnn_quantize_bf16meta(const void* x, actnn_dtype_t dt, int64_t N, int64_t D,
                                       int32_t G, const uint8_t* bits, const int64_t* off,
                                       uint64_t seed, int64_t sample_base, const float* gmin,
                                       const float* gmax, uint8_t* packed, uint32_t* meta,
                                       void* stream) {
    if (N > 0 && D > 0 && !meta)
        return fail(ACTNN_ERR_INVALID, "actnn_quantize_bf16meta: null pointer");
    return quantize_impl("actnn_quantize_bf16meta", x, dt, N, D, G, bits, off, seed, sample_base,
                         gmin, gmax, packed, nullptr, nullptr, meta, stream);
}

static actnn_status_t dequantize_impl(const char* fn, const uint8_t* packed, const float* zmin,
                                      const float* scale, const uint32_t* meta,
                                      const uint8_t* bits, const int64_t* off, int64_t N,
                                      int64_t D, int32_t G, void* out, actnn_dtype_t out_dt,
                                      void* stream) {
    actnn_status_t st = common_checks(N, D, G);
    if (st) return st;
    if (!dtype_ok(out_dt)) return fail(ACTNN_ERR_INVALID, "bad dtype %d", (int)out_dt);
    if (N == 0 || D == 0) return ACTNN_OK;
    if (!packed || (meta ? false : (!zmin || !scale)) || !bits || !off || !out)
        return fail(ACTNN_ERR_INVALID, "%s: null pointer", fn);
    const size_t es = out_dt == ACTNN_F32 ? 4 : 2;
    if (!aligned(out, es) || !aligned(off, 8) || (zmin && !aligned(zmin, 4)) ||
        (scale && !aligned(scale, 4)) || (meta && !aligned(meta, 4)))
        return fail(ACTNN_ERR_INVALID, "%s: misaligned pointer", fn);
    if (!aligned(packed, 16))
        return fail(ACTNN_ERR_UNSUPPORTED, "%s: packed must be 16-byte aligned", fn);
    const int64_t ng = ceil_div(D, G);
    st = debug_validate(bits, off, N, ng, (cudaStream_t)stream);
    if (st) return st;
    DequantArgs a;
    a.packed = packed;
    a.zmin = meta ? nullptr : zmin;
    a.scale = meta ? nullptr : scale;
    a.meta = meta;
    a.bits = bits;
    a.off = off;
    a.N = N;
    a.D = D;
    a.ng = ng;
    a.out = out;
    a.out_dt = (int)out_dt;
    a.fast = (D % G == 0) && aligned(out, out_dt == ACTNN_F32 ? 32 : 16);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_dequantize(a, s), fn, s);
}

actnn_status_t actnn_dequantize(const uint8_t* packed, const float* zmin, const float* scale,
                                const uint8_t* bits, const int64_t* off, int64_t N, int64_t D,
                                int32_t G, void* out, actnn_dtype_t out_dt, void* stream) {
    return dequantize_impl("actnn_dequantize", packed, zmin, scale, nullptr, bits, off, N, D, G,
                           out, out_dt, stream);
}

actnn_status_t actnn_dequantize_bf16meta(const uint8_t* packed, const uint32_t* meta,
                                         const uint8_t* bits, const int64_t* off, int64_t N,
                                         int64_t D, int32_t G, void* out, actnn_dtype_t out_dt,
                                         void* stream) {
    if (N > 0 && D > 0 && !meta)
        return fail(ACTNN_ERR_INVALID, "actnn_dequantize_bf16meta: null pointer");
    return dequantize_impl("actnn_dequantize_bf16meta", packed, nullptr, nullptr, meta, bits, off,
                           N, D, G, out, out_dt, stream);
}

// ------------------------------------------------------------ NEXT-3 adaptation
actnn_status_t actnn_grad_sqnorm(const void* g, actnn_dtype_t dt, int64_t N, int64_t D,
                                 int32_t G, double* out, void* ws, size_t ws_bytes,
                                 void* stream) {
    actnn_status_t st = common_checks(N, D, G);
    if (st) return st;
    if (!dtype_ok(dt)) return fail(ACTNN_ERR_INVALID, "bad dtype %d", (int)dt);
    if (N == 0) return ACTNN_OK;
    if (D == 0) {  // empty rows: ||grad_n||^2 = 0
        if (!out) return fail(ACTNN_ERR_INVALID, "actnn_grad_sqnorm: null pointer");
        return cuda_status(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)N,
                                           (cudaStream_t)stream), "actnn_grad_sqnorm");
    }
    if (!g || !out || !ws) return fail(ACTNN_ERR_INVALID, "actnn_grad_sqnorm: null pointer");
    const size_t es = dt == ACTNN_F32 ? 4 : 2;
    if (!aligned(g, es) || !aligned(out, 8) || !aligned(ws, 8))
        return fail(ACTNN_ERR_INVALID, "actnn_grad_sqnorm: misaligned pointer");
    const size_t need = actnn_workspace_bytes(ACTNN_OP_GRAD_SQNORM, N, D, G);
    if (ws_bytes < need)
        return fail(ACTNN_ERR_INVALID, "actnn_grad_sqnorm: workspace %zu < %zu bytes", ws_bytes,
                    need);
    GradArgs a;
    a.g = g;
    a.dt = (int)dt;
    a.N = N;
    a.D = D;
    a.ng = ceil_div(D, G);
    a.nch = ceil_div(a.ng, 32);
    a.out = out;
    a.T = static_cast<double*>(ws);
    a.fast = (D % G == 0) && aligned(g, dt == ACTNN_F32 ? 32 : 16);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_grad_sqnorm(a, s), "actnn_grad_sqnorm", s);
}

actnn_status_t actnn_gradmag_ema(const double* obs, int64_t N, double rho, double* m,
                                 void* stream) {
    if (N < 0) return fail(ACTNN_ERR_INVALID, "actnn_gradmag_ema: negative N");
    if (!(rho >= 0.0 && rho <= 1.0))
        return fail(ACTNN_ERR_INVALID, "actnn_gradmag_ema: rho outside [0, 1]");
    if (N == 0) return ACTNN_OK;
    if (!obs || !m) return fail(ACTNN_ERR_INVALID, "actnn_gradmag_ema: null pointer");
    if (!aligned(obs, 8) || !aligned(m, 8))
        return fail(ACTNN_ERR_INVALID, "actnn_gradmag_ema: misaligned pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_gradmag_ema(obs, N, rho, m, s), "actnn_gradmag_ema", s);
}

actnn_status_t actnn_gradmag_gather(const double* table, int64_t T, const int64_t* ids,
                                    int64_t N, double* est, void* stream) {
    if (N < 0 || T < 0) return fail(ACTNN_ERR_INVALID, "actnn_gradmag_gather: negative size");
    if (N == 0) return ACTNN_OK;
    if (T == 0) return fail(ACTNN_ERR_INVALID, "actnn_gradmag_gather: empty table");
    if (!table || !ids || !est) return fail(ACTNN_ERR_INVALID, "actnn_gradmag_gather: null pointer");
    if (!aligned(table, 8) || !aligned(ids, 8) || !aligned(est, 8))
        return fail(ACTNN_ERR_INVALID, "actnn_gradmag_gather: misaligned pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_gradmag_gather(table, ids, N, est, s), "actnn_gradmag_gather", s);
}

actnn_status_t actnn_gradmag_scatter(double* table, int64_t T, const int64_t* ids,
                                     const double* obs, int64_t N, void* stream) {
    if (N < 0 || T < 0) return fail(ACTNN_ERR_INVALID, "actnn_gradmag_scatter: negative size");
    if (N == 0) return ACTNN_OK;
    if (T == 0) return fail(ACTNN_ERR_INVALID, "actnn_gradmag_scatter: empty table");
    if (!table || !ids || !obs) return fail(ACTNN_ERR_INVALID, "actnn_gradmag_scatter: null pointer");
    if (!aligned(table, 8) || !aligned(ids, 8) || !aligned(obs, 8))
        return fail(ACTNN_ERR_INVALID, "actnn_gradmag_scatter: misaligned pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_gradmag_scatter(table, ids, obs, N, s), "actnn_gradmag_scatter", s);
}

size_t actnn_allocate_layers_ws_bytes(int64_t L, int64_t N, uint32_t level_mask) {
    if (L < 0 || N < 0 || level_mask == 0 || (level_mask & ~0x1FEu)) return 0;
    const int m = __builtin_popcount(level_mask);  // number of allowed widths
    return allocate_layers_ws_bytes(L, N, m - 1);
}

actnn_status_t actnn_allocate_layers(const double* sens, const double* gscale,
                                     const double* lconst, const int64_t* D_host, int64_t L,
                                     int64_t N, int64_t b_total, uint32_t level_mask,
                                     uint8_t* bits, int64_t* budgets, void* ws, size_t ws_bytes,
                                     void* stream) {
    if (L < 0 || N < 0) return fail(ACTNN_ERR_INVALID, "actnn_allocate_layers: negative size");
    if (L > ACTNN_MAX_LAYERS)
        return fail(ACTNN_ERR_UNSUPPORTED, "actnn_allocate_layers: L=%lld > %d", (long long)L,
                    ACTNN_MAX_LAYERS);
    LayerAllocArgs a;
    std::memset(&a, 0, sizeof(a));
    actnn_status_t st = levels_from_mask(level_mask, a.Lv, &a.m);
    if (st) return st;
    if (L > 0 && !D_host) return fail(ACTNN_ERR_INVALID, "actnn_allocate_layers: null D_host");
    int64_t start = 0, floor_bits = 0;
    for (int64_t l = 0; l < L; ++l) {
        if (D_host[l] < 1 || D_host[l] > (1ll << 24))
            return fail(ACTNN_ERR_UNSUPPORTED, "actnn_allocate_layers: D[%lld]=%lld outside 1..2^24",
                        (long long)l, (long long)D_host[l]);
        start += D_host[l] * N * a.Lv[0];
        floor_bits += D_host[l] * N * a.Lv[a.m - 1];
    }
    if (b_total < floor_bits)
        return fail(ACTNN_ERR_BUDGET, "b_total %lld < sum_l D_l N %d = %lld (infeasible)",
                    (long long)b_total, a.Lv[a.m - 1], (long long)floor_bits);
    if (L * N * (int64_t)(a.m - 1) > (1ll << 31))
        return fail(ACTNN_ERR_UNSUPPORTED, "actnn_allocate_layers: %lld moves > 2^31",
                    (long long)(L * N * (a.m - 1)));
    if (L == 0) return ACTNN_OK;
    if (!budgets) return fail(ACTNN_ERR_INVALID, "actnn_allocate_layers: null budgets");
    if (N == 0)
        return cuda_status(cudaMemsetAsync(budgets, 0, sizeof(int64_t) * (size_t)L,
                                           (cudaStream_t)stream), "actnn_allocate_layers");
    if (!sens || !bits || !ws) return fail(ACTNN_ERR_INVALID, "actnn_allocate_layers: null pointer");
    if (!aligned(sens, 8) || !aligned(budgets, 8) || (gscale && !aligned(gscale, 8)) ||
        (lconst && !aligned(lconst, 8)) || !aligned(ws, 256))
        return fail(ACTNN_ERR_INVALID, "actnn_allocate_layers: misaligned pointer");
    if (ws_bytes < allocate_layers_ws_bytes(L, N, a.m - 1))
        return fail(ACTNN_ERR_INVALID, "actnn_allocate_layers: workspace %zu < %zu bytes",
                    ws_bytes, allocate_layers_ws_bytes(L, N, a.m - 1));
    for (int c = 0; c + 1 < a.m; ++c) {
        const double Bh = (double)((1 << a.Lv[c]) - 1), Bl = (double)((1 << a.Lv[c + 1]) - 1);
        const double fh = 1.0 / (Bh * Bh), fl = 1.0 / (Bl * Bl);
        a.dstep[c] = a.Lv[c] - a.Lv[c + 1];
        a.slope[c] = (fl - fh) / (double)a.dstep[c];
    }
    a.sens = sens;
    a.gscale = gscale;
    a.lconst = lconst;
    a.D = D_host;
    a.L = L;
    a.N = N;
    a.need = start - b_total;
    a.bits = bits;
    a.budgets = budgets;
    a.ws = ws;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_allocate_layers(a, s), "actnn_allocate_layers", s);
}

// ------------------------------------------------------------ NEXT-4 contexts
actnn_status_t actnn_relu_pack(const void* x, actnn_dtype_t dt, int64_t E, uint8_t* mask,
                               void* y, void* stream) {
    if (!dtype_ok(dt)) return fail(ACTNN_ERR_INVALID, "bad dtype %d", (int)dt);
    if (E < 0) return fail(ACTNN_ERR_INVALID, "actnn_relu_pack: negative E");
    if (E == 0) return ACTNN_OK;
    if (!x || !mask) return fail(ACTNN_ERR_INVALID, "actnn_relu_pack: null pointer");
    const size_t es = dt == ACTNN_F32 ? 4 : 2;
    if (!aligned(x, es) || (y && !aligned(y, es)))
        return fail(ACTNN_ERR_INVALID, "actnn_relu_pack: misaligned pointer");
    ReluArgs a{x, y, mask, E, (int)dt};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_relu_pack(a, s), "actnn_relu_pack", s);
}

actnn_status_t actnn_relu_backward(const uint8_t* mask, const void* grad_y, actnn_dtype_t dt,
                                   int64_t E, void* grad_x, void* stream) {
    if (!dtype_ok(dt)) return fail(ACTNN_ERR_INVALID, "bad dtype %d", (int)dt);
    if (E < 0) return fail(ACTNN_ERR_INVALID, "actnn_relu_backward: negative E");
    if (E == 0) return ACTNN_OK;
    if (!mask || !grad_y || !grad_x)
        return fail(ACTNN_ERR_INVALID, "actnn_relu_backward: null pointer");
    const size_t es = dt == ACTNN_F32 ? 4 : 2;
    if (!aligned(grad_y, es) || !aligned(grad_x, es))
        return fail(ACTNN_ERR_INVALID, "actnn_relu_backward: misaligned pointer");
    ReluArgs a{grad_y, grad_x, const_cast<uint8_t*>(mask), E, (int)dt};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_relu_backward(a, s), "actnn_relu_backward", s);
}

static int64_t pool_extent(int64_t H, int k, int s, int p, int d) {
    return (H + 2 * (int64_t)p - (int64_t)d * (k - 1) - 1) / s + 1;
}

// Every output window along one axis holds at least one in-bounds tap
// (o s - p + t d in [0, H) for some tap t).  With dilation > 1 a padded window
// can miss the input entirely (e.g. k = 2, d = 2, p = 1, H = 1); such
// geometries are rejected -- PyTorch would return -inf there and no 8-bit tap
// index could name the winner.
static bool windows_hit_input(int64_t H, int64_t OH, int k, int s, int p, int d) {
    for (int64_t o = 0; o < OH; ++o) {
        bool hit = false;
        for (int t = 0; t < k && !hit; ++t) {
            const int64_t i = o * s - p + (int64_t)t * d;
            hit = i >= 0 && i < H;
        }
        if (!hit) return false;
    }
    return true;
}

static actnn_status_t pool_args(const char* fn, actnn_dtype_t dt, int64_t NC, int64_t H,
                                int64_t W, int32_t kh, int32_t kw, int32_t sh, int32_t sw,
                                int32_t ph, int32_t pw, int32_t dh, int32_t dw, PoolArgs* a) {
    if (!dtype_ok(dt)) return fail(ACTNN_ERR_INVALID, "bad dtype %d", (int)dt);
    if (NC < 0 || H < 1 || W < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1 || dh < 1 || dw < 1 ||
        ph < 0 || pw < 0 || 2 * ph > kh || 2 * pw > kw)
        return fail(ACTNN_ERR_INVALID, "%s: invalid pooling geometry", fn);
    if (kh * kw > 256)
        return fail(ACTNN_ERR_UNSUPPORTED, "%s: %d taps do not fit the 8-bit index", fn,
                    kh * kw);
    if (H * W >= (1ll << 31) || (int64_t)kh * dh + H + ph >= (1ll << 30) ||
        (int64_t)kw * dw + W + pw >= (1ll << 30))
        return fail(ACTNN_ERR_UNSUPPORTED, "%s: planes of 2^31 or more positions", fn);
    a->dt = (int)dt;
    a->NC = NC;
    a->H = H;
    a->W = W;
    a->OH = pool_extent(H, kh, sh, ph, dh);
    a->OW = pool_extent(W, kw, sw, pw, dw);
    if (a->OH < 1 || a->OW < 1) return fail(ACTNN_ERR_INVALID, "%s: empty output", fn);
    if (!windows_hit_input(H, a->OH, kh, sh, ph, dh) || !windows_hit_input(W, a->OW, kw, sw, pw, dw))
        return fail(ACTNN_ERR_UNSUPPORTED, "%s: a pooling window lies entirely in the padding", fn);
    a->kh = kh;
    a->kw = kw;
    a->sh = sh;
    a->sw = sw;
    a->ph = ph;
    a->pw = pw;
    a->dh = dh;
    a->dw = dw;
    return ACTNN_OK;
}

actnn_status_t actnn_maxpool2d_forward(const void* x, actnn_dtype_t dt, int64_t NC, int64_t H,
                                       int64_t W, int32_t kh, int32_t kw, int32_t sh,
                                       int32_t sw, int32_t ph, int32_t pw, int32_t dh,
                                       int32_t dw, void* y, uint8_t* idx, void* stream) {
    PoolArgs a;
    actnn_status_t st =
        pool_args("actnn_maxpool2d_forward", dt, NC, H, W, kh, kw, sh, sw, ph, pw, dh, dw, &a);
    if (st) return st;
    if (NC == 0) return ACTNN_OK;
    if (!x || !y || !idx) return fail(ACTNN_ERR_INVALID, "actnn_maxpool2d_forward: null pointer");
    const size_t es = dt == ACTNN_F32 ? 4 : 2;
    if (!aligned(x, es) || !aligned(y, es))
        return fail(ACTNN_ERR_INVALID, "actnn_maxpool2d_forward: misaligned pointer");
    a.in = x;
    a.out = y;
    a.idx = idx;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_maxpool2d(a, false, s), "actnn_maxpool2d_forward", s);
}

actnn_status_t actnn_maxpool2d_backward(const uint8_t* idx, const void* grad_y,
                                        actnn_dtype_t dt, int64_t NC, int64_t H, int64_t W,
                                        int32_t kh, int32_t kw, int32_t sh, int32_t sw,
                                        int32_t ph, int32_t pw, int32_t dh, int32_t dw,
                                        void* grad_x, void* stream) {
    PoolArgs a;
    actnn_status_t st =
        pool_args("actnn_maxpool2d_backward", dt, NC, H, W, kh, kw, sh, sw, ph, pw, dh, dw, &a);
    if (st) return st;
    if (NC == 0) return ACTNN_OK;
    if (!idx || !grad_y || !grad_x)
        return fail(ACTNN_ERR_INVALID, "actnn_maxpool2d_backward: null pointer");
    const size_t es = dt == ACTNN_F32 ? 4 : 2;
    if (!aligned(grad_y, es) || !aligned(grad_x, es))
        return fail(ACTNN_ERR_INVALID, "actnn_maxpool2d_backward: misaligned pointer");
    a.in = grad_y;
    a.out = grad_x;
    a.idx = const_cast<uint8_t*>(idx);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return post_launch(launch_maxpool2d(a, true, s), "actnn_maxpool2d_backward", s);
}

}  // extern "C"
