/*
 * actnn.h -- C ABI of libactnn.so, the B200 (sm_100a) hot path of ActNN
 * (Chen et al., "ActNN: Reducing Training Memory Footprint via 2-Bit
 * Activation Compressed Training", ICML 2021, arXiv 2104.14129).
 *
 * Citations: P:<line> = PAPER.md line, S:<line> = SPEC.md line; "ACTNN-Q v1"
 * is the arithmetic contract in DESIGN.md that
 * makes the GPU codes bit-identical to the CPU oracle's.
 *
 * Conventions (every entry point):
 *  - All array pointers are DEVICE pointers unless the name ends in _host.
 *  - Calls are asynchronous on `stream` (a cudaStream_t passed as void*; NULL
 *    = legacy default stream).  The library never allocates, frees,
 *    synchronises or copies; the caller owns every buffer.  Reentrant.
 *  - Arguments that can be checked on the host are checked before anything is
 *    launched; a non-OK status launches nothing and actnn_last_error() returns
 *    a thread-local message.  Launch failures return ACTNN_ERR_CUDA.
 *  - N == 0 or D == 0 is a valid empty problem: OK, nothing launched.
 *  - Device-resident data (bits[], off[], inputs) is not validated on the fast
 *    path.  Inputs must be finite with |x| < 2^125 (SPEC "values finite",
 *    S:125); bits[n] must lie in 1..8.  Setting ACTNN_CHECK=1 in the
 *    environment makes every call synchronise and validate bits/off.
 *  - Layouts: an activation is [N, D] row-major (sample n's flattened NCHW
 *    tensor is row n).  Groups are G = 256 contiguous elements of one sample
 *    ("partition its dimensions into groups h_ni"); ng = ceil(D/G); the
 *    last group of a sample may be ragged.  Per-group arrays
 *    (gmin, gmax, zmin, scale) are [N * ng], sample-major.
 *  - Only G == 256 is supported in ABI v1 ("we set G = 256");
 *    other G return ACTNN_ERR_UNSUPPORTED.
 */
#ifndef ACTNN_H
#define ACTNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACTNN_ABI_VERSION 1

typedef enum {
    ACTNN_OK = 0,
    ACTNN_ERR_INVALID = -1,      /* null pointer, negative size, bad enum, misalignment */
    ACTNN_ERR_UNSUPPORTED = -2,  /* valid but outside ABI v1 (G != 256, packed not 16B-aligned) */
    ACTNN_ERR_BUDGET = -3,       /* budget < N * (smallest allowed width) */
    ACTNN_ERR_CUDA = -4,         /* kernel launch / CUDA runtime failure */
    ACTNN_ERR_CHECK = -5         /* ACTNN_CHECK=1 found invalid device data */
} actnn_status_t;

typedef enum { ACTNN_F32 = 0, ACTNN_BF16 = 1 } actnn_dtype_t;

/* level_mask: bit b set <=> width b allowed, b in 1..8. */
#define ACTNN_LEVELS_POW2 ((1u << 1) | (1u << 2) | (1u << 4) | (1u << 8)) /* {1,2,4,8}: hot path */
#define ACTNN_LEVELS_UNIT 0x1FEu /* 1..8: the paper's unit-step greedy */

/* op ids for actnn_workspace_bytes */
#define ACTNN_OP_GROUP_STATS 0
#define ACTNN_OP_ALLOCATE_BITS 1
#define ACTNN_OP_GRAD_SQNORM 2

/* Largest layer count of actnn_allocate_layers. */
#define ACTNN_MAX_LAYERS 1024

/* Thread-local message describing the last non-OK status of this thread. */
const char* actnn_last_error(void);

/* ACTNN_ABI_VERSION of the loaded library. */
int actnn_abi_version(void);

/* Device workspace (bytes) `op` needs for an [N, D] problem; 0 = none. */
size_t actnn_workspace_bytes(int op, int64_t N, int64_t D, int32_t G);

/* Size in bytes of the packed code buffer: sum_n bits_host[n] * ng * G / 8
 * (S:115).  bits_host == NULL gives the 8-bit upper bound 8*N*ng*G/8.
 * Returns -1 on invalid arguments. */
int64_t actnn_packed_bytes(int64_t N, int64_t D, int32_t G, const uint8_t* bits_host);

/* Pass 1 of the mixed-precision path: for every
 * group the canonical min Z and max M (signed zeros mapped to +0), and for
 * every sample the range norm S_n = ||R_n||^2 = sum_i (M_ni - Z_ni)^2 in fp64,
 * summed in the canonical order of ACTNN-Q v1 step O11 (32-group chunks, xor
 * butterfly inside a chunk, chunks in order).  S_n is the sample's sensitivity
 * w_n up to the per-sample gradient factor of Eq. 7.
 *   x        [N, D] activations of dtype dt
 *   gmin/gmax [N*ng] fp32 outputs;  sens [N] fp64 output
 *   ws       >= actnn_workspace_bytes(ACTNN_OP_GROUP_STATS, N, D, G) bytes, 8B-aligned,
 *            ZERO-FILLED before its first use (its last 8 bytes hold a completion
 *            ticket that every call leaves at zero again); one workspace per
 *            stream: concurrent calls must not share it.  One kernel launch. */
actnn_status_t actnn_group_stats(const void* x, actnn_dtype_t dt, int64_t N, int64_t D, int32_t G,
                                 float* gmin, float* gmax, double* sens, void* ws,
                                 size_t ws_bytes, void* stream);

/* Stage 1 of the run-time adaptation (Prob. 8 at P:541-547 for one
 * layer): the paper's greedy, computed on the device in one CTA.
 * w_n = sens[n] * (gscale ? gscale[n] : 1).  Every sample starts at the widest
 * allowed width; moves (one allowed width down) are applied in ascending
 * (w_n * slope_c, n, c) order, slope_c = (1/B_{c+1}^2 - 1/B_c^2) / freed bits,
 * until sum_n bits[n] <= budget.  Bit-identical to the oracle's binary heap.
 *   sens, gscale [N] fp64, finite and >= 0;  budget: max sum_n bits[n]
 *   level_mask: allowed widths (ACTNN_LEVELS_POW2 on the hot path)
 *   D, G: used for the offsets only
 *   bits [N] u8 output;  off [N+1] i64 output: off[0] = 0,
 *   off[n+1] = off[n] + bits[n] * ng * G / 8 (byte offsets into `packed`)
 *   ws: unused in v1 (pass NULL, 0). */
actnn_status_t actnn_allocate_bits(const double* sens, const double* gscale, int64_t N,
                                   int64_t budget, uint32_t level_mask, int64_t D, int32_t G,
                                   uint8_t* bits, int64_t* off, void* ws, size_t ws_bytes,
                                   void* stream);

/* Uniform widths (optimization level L2): bits[n] = b for all n and
 * the matching off[N+1].  b in 1..8. */
actnn_status_t actnn_uniform_bits(int64_t N, int64_t D, int32_t G, int32_t b, uint8_t* bits,
                                  int64_t* off, void* stream);

/* Compressor: per group Z = min, R = max - min,
 * scale = RN(R/B), u_bar = B (h - Z)/R in 14-bit fixed point, unbiased
 * stochastic rounding with Philox4x32-10(ctr = e >> 3, key = seed) where
 * e = (sample_base + n) * D + d is the element's global index, and LSB-first
 * packing of the b_n-bit codes.
 *   x [N, D] dtype dt;  bits [N], off [N+1] as produced by actnn_allocate_bits
 *   (sample n's bytes start at packed + off[n] - off[0], so a rank may pass a
 *   slice of a global off[] array);  sample_base: global index of this shard's
 *   first sample (ranks of a batch-sharded job pass r * N_local);
 *   gmin/gmax: NULL => one pass computing min/max in-kernel, else the
 *   actnn_group_stats outputs (results are identical either way);
 *   packed: off[N] - off[0] bytes, 16-byte aligned;  zmin/scale [N*ng] fp32. */
actnn_status_t actnn_quantize(const void* x, actnn_dtype_t dt, int64_t N, int64_t D, int32_t G,
                              const uint8_t* bits, const int64_t* off, uint64_t seed,
                              int64_t sample_base, const float* gmin, const float* gmax,
                              uint8_t* packed, float* zmin, float* scale, void* stream);

/* Decompressor: h_hat = code * scale + Z with a single rounding
 * (fmaf); bf16 output is RNE(h_hat).  Buffers as for actnn_quantize;
 * out [N, D] of dtype out_dt. */
actnn_status_t actnn_dequantize(const uint8_t* packed, const float* zmin, const float* scale,
                                const uint8_t* bits, const int64_t* off, int64_t N, int64_t D,
                                int32_t G, void* out, actnn_dtype_t out_dt, void* stream);

/* NEXT-1, bf16 metadata: the paper's storage format, "store the per-group range
 * and zero points in bfloat16, so each group costs extra 32 bits, which is
 * 0.125 bits on average" (the values are rounded
 * BEFORE scaling, so the quantiser and the dequantiser use the same stored
 * values).  meta [N*ng] u32, one word per group (4-byte aligned; 16-byte
 * alignment with ng % 4 == 0 lets the dequantiser fetch it by TMA):
 *   bits 0-15  Z' = bf16 of Z rounded toward -inf,
 *   bits 16-31 R' = bf16 of RU(M - Z') rounded toward +inf,
 * so [Z', Z' + R'] contains every element of the group (outward rounding,
 * DESIGN reading 21).  Codes are those of actnn_quantize run with
 * (Z, R) := (float(Z'), float(R')); all other arguments, layouts, ownership
 * and errors as for actnn_quantize (zmin/scale are replaced by meta). */
actnn_status_t actnn_quantize_bf16meta(const void* x, actnn_dtype_t dt, int64_t N, int64_t D,
                                       int32_t G, const uint8_t* bits, const int64_t* off,
                                       uint64_t seed, int64_t sample_base, const float* gmin,
                                       const float* gmax, uint8_t* packed, uint32_t* meta,
                                       void* stream);

/* Decompressor for bf16 metadata: h_hat = fmaf(code, RN(float(R') / B),
 * float(Z')), bf16 output RNE(h_hat).  Arguments as for actnn_dequantize with
 * meta (as written by actnn_quantize_bf16meta) in place of zmin/scale. */
actnn_status_t actnn_dequantize_bf16meta(const uint8_t* packed, const uint32_t* meta,
                                         const uint8_t* bits, const int64_t* off, int64_t N,
                                         int64_t D, int32_t G, void* out, actnn_dtype_t out_dt,
                                         void* stream);

/* ---------------------------------------------------------------- NEXT-3 */
/* Run-time adaptation: the gradient-magnitude factor of the
 * sensitivity, its two estimators, and stage 2 of the allocation.  For a
 * linear layer w_n = G/6 ||grad_n||^2 ||R_n||^2 (Eq. 7); other
 * layer types differ by a per-layer constant (App. B: G K / (6 I A) for
 * convolutions; a constant for normalisation). */

/* Per-sample squared L2 norm of a gradient tensor, ||grad_n||^2, fp64,
 * in the canonical order of DESIGN reading 22 (lane terms = in-order sums of
 * the squares of G/32 consecutive elements, xor butterfly over the 32 lanes of
 * a group, group totals in the O11 order), so results are bit-identical to the
 * oracle.  g [N, D] of dtype dt (any D; vector path when D % 256 == 0 and g is
 * 32-byte (fp32) / 16-byte (bf16) aligned); out [N] fp64.  ws: >=
 * actnn_workspace_bytes(ACTNN_OP_GRAD_SQNORM, N, D, G) bytes, 8-byte aligned,
 * zero-filled before its first use and left zero by every call (a completion
 * ticket, as for actnn_group_stats); one workspace per stream.  One launch. */
actnn_status_t actnn_grad_sqnorm(const void* g, actnn_dtype_t dt, int64_t N, int64_t D,
                                 int32_t G, double* out, void* ws, size_t ws_bytes,
                                 void* stream);

/* Moving-average estimator ("the moving average of gradient magnitude
 * across samples"): *m <- RN(rho * m) + RN(RN(1 - rho) * mean), mean =
 * RN(S / N) with S the canonical (O11-order) sum of obs[0..N).  obs [N] fp64
 * (e.g. the actnn_grad_sqnorm output of this step), m: one fp64 in device
 * memory (the caller's state, initialised e.g. to 1.0).  rho in [0, 1]
 * (else ACTNN_ERR_INVALID).  N == 0: no launch, m unchanged.  One launch. */
actnn_status_t actnn_gradmag_ema(const double* obs, int64_t N, double rho, double* m,
                                 void* stream);

/* Stale estimator ("the stale gradient magnitude in the last epoch";
 * S:369): a table [T] fp64 indexed by dataset sample id, owned and initialised
 * by the caller (1.0 = cold start).  gather: est[n] = table[ids[n]];
 * scatter: table[ids[n]] = obs[n].  ids [N] i64 must lie in [0, T) and be
 * distinct within one scatter (device data, not validated).  One launch each. */
actnn_status_t actnn_gradmag_gather(const double* table, int64_t T, const int64_t* ids,
                                    int64_t N, double* est, void* stream);
actnn_status_t actnn_gradmag_scatter(double* table, int64_t T, const int64_t* ids,
                                     const double* obs, int64_t N, void* stream);

/* Workspace bytes of actnn_allocate_layers for L layers of N samples. */
size_t actnn_allocate_layers_ws_bytes(int64_t L, int64_t N, uint32_t level_mask);

/* Stage 2 of the run-time adaptation ("After finishing the back
 * propagation, ActNN solves Prob. (8) again for all the layers together, and
 * sets b^(l) <- sum_n b_n^(l)"), with the paper's greedy over every
 * (layer l, sample n): all start at the widest allowed width; the move of
 * (l, n) from L_c to L_{c+1} frees D_l (L_c - L_{c+1}) bits and has key
 * RN(RN(w_ln slope_c) / D_l) (variance increase per freed bit, DESIGN reading
 * 24), w_ln = RN(RN(sens * gscale) * lconst) (absent factors skipped, reading
 * 23); moves apply in ascending (key, l, n, c) order until
 * sum_l D_l sum_n b_ln <= b_total.  Bit-identical to the oracle's heap.
 *   sens [L*N] fp64 (layer-major; actnn_group_stats outputs of every layer),
 *   gscale [L*N] fp64 or NULL (gradient estimates), lconst [L] fp64 or NULL
 *   (per-layer constants), all finite and >= 0;
 *   D_host [L] HOST array of per-sample feature dimensions D_l (1 <= D_l <= 2^24),
 *   read at call time (it travels in the launch parameters; the caller may
 *   reuse it as soon as the call returns);
 *   L in 0..ACTNN_MAX_LAYERS (else ACTNN_ERR_UNSUPPORTED), L*N*(levels-1) <= 2^31;
 *   b_total: total bits; ACTNN_ERR_BUDGET when below sum_l D_l N min-width;
 *   bits [L*N] u8 output; budgets [L] i64 output: b^(l) = sum_n b_ln, the
 *   stage-1 budget of layer l for the next iteration (actnn_allocate_bits);
 *   ws: >= actnn_allocate_layers_ws_bytes(L, N, level_mask) bytes, 256-byte
 *   aligned, zero-filled before its first use and left in that state by every
 *   call; one workspace per stream.
 * One cooperative launch (one CTA per SM, grid-wide barriers). */
actnn_status_t actnn_allocate_layers(const double* sens, const double* gscale,
                                     const double* lconst, const int64_t* D_host, int64_t L,
                                     int64_t N, int64_t b_total, uint32_t level_mask,
                                     uint8_t* bits, int64_t* budgets, void* ws, size_t ws_bytes,
                                     void* stream);

/* ---------------------------------------------------------------- NEXT-4 */
/* Lossless contexts of a Conv-BN-ReLU-MaxPool block (the rest of the paper's
 * per-block memory arithmetic: "2.125 bits (Conv) + 2.125 bits (BN)
 * + 1 bit (ReLU)").  Exact: no quantisation, zero variance. */

/* ReLU context (App. B.3: "ReLU layers only take a single bit per
 * dimension to store, without any approximation").  x: E elements of dtype dt
 * (any shape, contiguous).  mask: ceil(E/8) bytes; bit k of the LSB-first
 * stream = (x_k > 0).  y: NULL, or E elements receiving ReLU(x) (+0 for
 * non-positive inputs) from the same read.  Vector path when x and y are
 * 32-byte aligned (mask 2-byte aligned for bf16); any alignment is valid. */
actnn_status_t actnn_relu_pack(const void* x, actnn_dtype_t dt, int64_t E, uint8_t* mask,
                               void* y, void* stream);

/* ReLU backward from the mask: grad_x[k] = grad_y[k] where bit k is set, +0
 * elsewhere (equal, bit for bit, to the full-precision ReLU gradient). */
actnn_status_t actnn_relu_backward(const uint8_t* mask, const void* grad_y, actnn_dtype_t dt,
                                   int64_t E, void* grad_x, void* stream);

/* Max-pool context (App. B.4: "We use 8 bits per output
 * location").  x [NC, H, W] (NCHW with NC = N*C planes), PyTorch geometry:
 * kernel kh x kw (kh*kw <= 256, else ACTNN_ERR_UNSUPPORTED), stride sh, sw >= 1,
 * padding ph <= kh/2, pw <= kw/2 (padded taps never win), dilation dh, dw >= 1,
 * floor mode: OH = (H + 2 ph - dh (kh - 1) - 1) / sh + 1, OW likewise.  Every
 * window must hold at least one in-bounds tap; a geometry with a window lying
 * entirely in the padding (possible with dilation > 1) returns
 * ACTNN_ERR_UNSUPPORTED and launches nothing.
 * y [NC, OH, OW] = window maximum; idx [NC, OH, OW] u8 = first argmax tap
 * a*kw + b in row-major window order (PyTorch's tie rule).  x finite: a NaN
 * tap gives an unspecified (but memory-safe) result. */
actnn_status_t actnn_maxpool2d_forward(const void* x, actnn_dtype_t dt, int64_t NC, int64_t H,
                                       int64_t W, int32_t kh, int32_t kw, int32_t sh,
                                       int32_t sw, int32_t ph, int32_t pw, int32_t dh,
                                       int32_t dw, void* y, uint8_t* idx, void* stream);

/* Max-pool backward from the 8-bit context: grad_x[p, r, c] = sum of grad_y
 * over the windows whose stored argmax is (r, c), accumulated in fp32 in
 * increasing output order (bf16 output: RNE of the sum).  grad_x [NC, H, W] is
 * fully written (zeros where no window selected the input). */
actnn_status_t actnn_maxpool2d_backward(const uint8_t* idx, const void* grad_y,
                                        actnn_dtype_t dt, int64_t NC, int64_t H, int64_t W,
                                        int32_t kh, int32_t kw, int32_t sh, int32_t sw,
                                        int32_t ph, int32_t pw, int32_t dh, int32_t dw,
                                        void* grad_x, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ACTNN_H */
