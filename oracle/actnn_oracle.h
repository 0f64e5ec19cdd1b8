/*
 * actnn_oracle.h -- CPU oracle for the ActNN hot path ("ACTNN-Q v1" contract).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path may include, link or
 * call this code: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header,
 * table or constant generator with paper_2104_14129_b200/csrc (the CUDA path).
 *
 * Citations: P:<line> = /root/reference/PAPER.md line (ActNN, ICML 2021),
 *            S:<line> = /root/reference/SPEC.md line, SURVEY = SURVEY.md §8(c)
 *            step ids O1..O13, DESIGN = DESIGN.md "Readings".
 *
 * Plain scalar C++17, built with -O2 -ffp-contract=off (no FMA contraction,
 * no fast-math), IEEE binary32/binary64 with round-to-nearest-even.
 */
#ifndef ACTNN_ORACLE_H
#define ACTNN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_F32 = 0, ORACLE_BF16 = 1 };
enum { ORACLE_OK = 0, ORACLE_ERR_INVALID = -1, ORACLE_ERR_BUDGET = -3,
       ORACLE_ERR_INVARIANT = -5 };

/* Philox4x32-10 (Salmon et al., SC'11 / Random123), the counter-based RNG the
 * contract uses for the stochastic rounding of P:499-503 (DESIGN reading 7). */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* O6: the 14-bit uniform draw r in [0, 2^14) for global element index e. */
uint32_t oracle_random14(uint64_t seed, uint64_t e);

/* O1-O3: per-group canonical minimum Z and maximum M of the real
 * elements of every group; x is [N, D] row-major, dtype ORACLE_F32/BF16.
 * gmin/gmax have N*ceil(D/G) entries (sample-major). */
int oracle_group_minmax(const void* x, int dtype, int64_t N, int64_t D, int32_t G,
                        float* gmin, float* gmax);

/* O11: S_n = ||R_n||^2 = sum_i R_ni^2 in the canonical
 * order (32-group chunks, xor butterfly within a chunk, chunks in order). */
void oracle_sensitivity(const float* gmin, const float* gmax, int64_t N, int64_t ng,
                        double* S);

/* O12: greedy per-sample bit allocation with a binary
 * heap.  Start every sample at the highest allowed level, repeatedly apply the
 * move with the smallest variance increase per freed bit (ties: sample index,
 * then move index) until sum_n b_n <= budget.  level_mask: bit b set <=> width
 * b allowed (b in 1..8).  0x116 = {1,2,4,8} (hot path), 0x1FE = 1..8 (the
 * paper's unit-step greedy).  Returns ORACLE_ERR_BUDGET when budget < N*min. */
int oracle_allocate_bits(const double* w, int64_t N, int64_t budget, uint32_t level_mask,
                         uint8_t* bits);

/* Eq. 8 objective for one layer: sum_n w_n / (2^b_n - 1)^2. */
double oracle_objective(const double* w, const uint8_t* bits, int64_t N);

/* Exact minimisers of Eq. 8 for one layer ("solved exactly by DP"),
 * test pins only: brute force (|levels|^N, N <= 10) and knapsack DP.
 * Both return the optimal objective and write one optimal assignment. */
double oracle_allocate_bruteforce(const double* w, int64_t N, int64_t budget,
                                  uint32_t level_mask, uint8_t* bits);
double oracle_allocate_dp(const double* w, int64_t N, int64_t budget, uint32_t level_mask,
                          uint8_t* bits);

/* O8: packed byte offsets, off[0]=0, off[n+1] = off[n] + b_n*ceil(D/G)*G/8. */
void oracle_offsets(const uint8_t* bits, int64_t N, int64_t D, int32_t G, int64_t* off);

/* O3-O9 for ONE group: len real elements h[0..len) (len <= G) of
 * a group whose first element has global index e0 = (sample_base+n)*D + i*G.
 * Writes the group's G*b/8-byte segment (padding codes 0), Z and scale.
 * Returns ORACLE_ERR_INVARIANT if the q <= B*2^14 invariant fails. */
int oracle_quantize_group(const float* h, int32_t len, int32_t G, int32_t b, uint64_t seed,
                          uint64_t e0, uint8_t* seg, float* zmin, float* scale);

/* O1-O9 over a whole [N, D] tensor: bits[N] per sample, packed has off[N]
 * bytes, zmin/scale have N*ceil(D/G) entries.  threads >= 1 splits samples
 * over std::threads (results are independent of the thread count). */
int oracle_quantize(const void* x, int dtype, int64_t N, int64_t D, int32_t G,
                    const uint8_t* bits, uint64_t seed, int64_t sample_base,
                    uint8_t* packed, float* zmin, float* scale, int threads);

/* O10: h_hat = code*scale + Z with one rounding (fmaf); bf16
 * output is RNE(h_hat).  out is [N, D] row-major in out_dtype. */
int oracle_dequantize(const uint8_t* packed, const float* zmin, const float* scale,
                      const uint8_t* bits, int64_t N, int64_t D, int32_t G,
                      void* out, int out_dtype, int threads);

/* NEXT-1, bf16 metadata ("store the per-group range and zero points in
 * bfloat16, so each group costs extra 32 bits"; DESIGN
 * reading 21).  One 32-bit word per group: bits 0-15 = Z' = bf16 of Z rounded
 * toward -inf, bits 16-31 = R' = bf16 of RU32(M - Z') rounded toward +inf, so
 * [Z', Z' + R'] contains every element of the group.  Quantisation and
 * dequantisation use the stored values: O4-O10 with Z := float(Z'),
 * R := float(R'), scale = RN(R / B). */
uint32_t oracle_meta_bf16(float Z, float M);
int oracle_quantize_group_bf16meta(const float* h, int32_t len, int32_t G, int32_t b,
                                   uint64_t seed, uint64_t e0, uint8_t* seg, uint32_t* meta);
int oracle_quantize_bf16meta(const void* x, int dtype, int64_t N, int64_t D, int32_t G,
                             const uint8_t* bits, uint64_t seed, int64_t sample_base,
                             uint8_t* packed, uint32_t* meta, int threads);
int oracle_dequantize_bf16meta(const uint8_t* packed, const uint32_t* meta,
                               const uint8_t* bits, int64_t N, int64_t D, int32_t G,
                               void* out, int out_dtype, int threads);

/* NEXT-4, lossless contexts.  ReLU (App. B.3): one bit per
 * element, bit k of the LSB-first stream = (x_k > 0); y (optional) = ReLU(x)
 * with +0 for non-positive inputs; backward: grad_x = grad_y where the bit is
 * set, +0 elsewhere.  E elements, mask has ceil(E/8) bytes. */
int oracle_relu_pack(const void* x, int dtype, int64_t E, uint8_t* mask, void* y);
int oracle_relu_backward(const uint8_t* mask, const void* gy, int dtype, int64_t E, void* gx);

/* Max pooling (App. B.4) on NC planes of H x W (PyTorch
 * geometry: kernel kh x kw <= 256 taps, stride, padding <= kernel/2,
 * dilation, floor mode; OH/OW as PyTorch computes them).  Forward: y = window
 * max, idx = first argmax tap (a*kw + b) in 8 bits per output location.
 * Backward: grad_x = sum of grad_y over the windows whose argmax is that input,
 * accumulated in fp32 in increasing output order, then stored in dtype. */
int oracle_maxpool2d_forward(const void* x, int dtype, int64_t NC, int64_t H, int64_t W, int kh,
                             int kw, int sh, int sw, int ph, int pw, int dh, int dw, int64_t OH,
                             int64_t OW, void* y, uint8_t* idx);
int oracle_maxpool2d_backward(const uint8_t* idx, const void* gy, int dtype, int64_t NC,
                              int64_t H, int64_t W, int kh, int kw, int sh, int sw, int ph,
                              int pw, int dh, int dw, int64_t OH, int64_t OW, void* gx);

/* NEXT-3, run-time adaptation.  O14: per-sample ||grad_n||^2 of a
 * gradient tensor [N, D] in fp64 (lane terms of G/32 consecutive squares in
 * order, xor butterfly over the 32 lanes per group, group totals in the O11
 * order).  O15: moving average m <- rho m + (1 - rho) mean(obs).  O16: stale
 * per-sample table gather / scatter.  O17: stage-2 joint greedy over all
 * layers (key RN(RN(w slope_c) / D_l), ties (l, n, c)), budgets[l] = sum_n b.
 * w_ln = RN(RN(sens * gscale) * lconst), absent factors skipped. */
int oracle_grad_sqnorm(const void* g, int dtype, int64_t N, int64_t D, int32_t G, double* out);
int oracle_gradmag_ema(const double* obs, int64_t N, double rho, double* m);
int oracle_gradmag_gather(const double* table, int64_t T, const int64_t* ids, int64_t N,
                          double* est);
int oracle_gradmag_scatter(double* table, int64_t T, const int64_t* ids, const double* obs,
                           int64_t N);
int oracle_allocate_layers(const double* sens, const double* gscale, const double* lconst,
                           const int64_t* D, int64_t L, int64_t N, int64_t b_total,
                           uint32_t level_mask, uint8_t* bits, int64_t* budgets);
double oracle_objective_layers(const double* sens, const double* gscale, const double* lconst,
                               int64_t L, int64_t N, const uint8_t* bits);
double oracle_allocate_layers_dp(const double* sens, const double* gscale, const double* lconst,
                                 const int64_t* D, int64_t L, int64_t N, int64_t b_total,
                                 uint32_t level_mask, uint8_t* bits);

/* O10 for one group: codes from a segment and dequantised fp32 values. */
void oracle_dequantize_group(const uint8_t* seg, int32_t len, int32_t b, float zmin,
                             float scale, uint32_t* codes, float* out);

#ifdef __cplusplus
}
#endif
#endif
