/*
 * actnn_oracle.cpp -- the CPU oracle ("ACTNN-Q v1"), plain and slow on purpose.
 *
 * TEST INFRASTRUCTURE ONLY (see actnn_oracle.h).  Every function follows the
 * passage it cites step by step; there is no blocking, vectorisation or fusion.
 * The CUDA path (paper_2104_14129_b200/csrc) is an independent implementation.
 *
 * Build: g++ -std=c++17 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared
 */
#include "actnn_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <queue>
#include <thread>
#include <tuple>
#include <vector>

/* ------------------------------------------------------------------------- */
/* Philox4x32-10.  Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as    */
/* easy as 1, 2, 3" (SC'11): round multipliers 0xD2511F53 / 0xCD9E8D57, Weyl   */
/* key bumps 0x9E3779B9 / 0xBB67AE85, 10 rounds, the key bumped between rounds.*/
/* DESIGN reading 7: the paper needs "stochastic rounding" but     */
/* names no generator; SPEC asks for a counter-based one.               */
/* ------------------------------------------------------------------------- */
extern "C" void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                                     uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* O6: element e draws 16-bit lane (e & 7) of Philox(ctr = e >> 3, key = seed)
 * and keeps its low 14 bits.  (DESIGN reading 6: 14-bit fixed-point SR.) */
extern "C" uint32_t oracle_random14(uint64_t seed, uint64_t e) {
    uint64_t block = e >> 3;
    uint32_t ctr[4] = {(uint32_t)block, (uint32_t)(block >> 32), 0u, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    oracle_philox4x32_10(ctr, key, o);
    uint32_t j = (uint32_t)(e & 7u);
    uint32_t word = o[j >> 1];
    uint32_t half = (j & 1u) ? (word >> 16) : (word & 0xFFFFu);
    return half & 0x3FFFu;
}

/* O1: widen one element to fp32 (bf16 -> fp32 is exact: bits << 16). */
static float widen(const void* x, int dtype, int64_t idx) {
    if (dtype == ORACLE_F32) return ((const float*)x)[idx];
    uint16_t h = ((const uint16_t*)x)[idx];
    uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

/* RNE of an fp32 value to bf16 (DESIGN reading 15), finite inputs. */
static uint16_t to_bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return 0x7FC0u; /* NaN */
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    return (uint16_t)(u >> 16);
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* O3 for one group: exact min and max, each canonicalised (x + 0.0f maps -0
 * to +0; DESIGN reading 17).  P:493-498: Z = min h, R = max h - min h. */
static void group_min_max(const float* h, int32_t len, float* Z, float* M) {
    float z = h[0], m = h[0];
    for (int32_t k = 1; k < len; ++k) {
        if (h[k] < z) z = h[k];
        if (h[k] > m) m = h[k];
    }
    *Z = z + 0.0f;
    *M = m + 0.0f;
}

extern "C" int oracle_group_minmax(const void* x, int dtype, int64_t N, int64_t D, int32_t G,
                                   float* gmin, float* gmax) {
    if (N < 0 || D < 0 || G < 1) return ORACLE_ERR_INVALID;
    int64_t ng = ceil_div(D, G);
    std::vector<float> h(G);
    for (int64_t n = 0; n < N; ++n) {
        for (int64_t i = 0; i < ng; ++i) {
            int32_t len = (int32_t)std::min<int64_t>(G, D - i * G);
            for (int32_t k = 0; k < len; ++k) h[k] = widen(x, dtype, n * D + i * G + k);
            group_min_max(h.data(), len, &gmin[n * ng + i], &gmax[n * ng + i]);
        }
    }
    return ORACLE_OK;
}

/* O11: S_n = sum_i R_ni^2 (the ||R_n||^2 factor of w_n, P:547 / Eq. 7).
 * Canonical order (DESIGN reading 11): chunks of 32 consecutive groups
 * (zero padded), v[l] = R_l^2 exactly in fp64, then for o = 16,8,4,2,1 every
 * v[l] <- v[l] + v[l^o] simultaneously; T_c = v[0]; S_n = ((0+T_0)+T_1)+... */
extern "C" void oracle_sensitivity(const float* gmin, const float* gmax, int64_t N,
                                   int64_t ng, double* S) {
    int64_t nch = ceil_div(ng, 32);
    for (int64_t n = 0; n < N; ++n) {
        double s = 0.0;
        for (int64_t c = 0; c < nch; ++c) {
            double v[32], t[32];
            for (int l = 0; l < 32; ++l) {
                int64_t i = c * 32 + l;
                if (i < ng) {
                    float R = gmax[n * ng + i] - gmin[n * ng + i];
                    v[l] = (double)R * (double)R;
                } else {
                    v[l] = 0.0;
                }
            }
            for (int o = 16; o >= 1; o >>= 1) {
                for (int l = 0; l < 32; ++l) t[l] = v[l] + v[l ^ o];
                for (int l = 0; l < 32; ++l) v[l] = t[l];
            }
            s = s + v[0];
        }
        S[n] = s;
    }
}

/* Levels of the mask in descending order (the greedy starts at the top). */
static int mask_levels(uint32_t level_mask, int* L) {
    if (level_mask == 0 || (level_mask & ~0x1FEu)) return -1;
    int m = 0;
    for (int b = 8; b >= 1; --b)
        if (level_mask & (1u << b)) L[m++] = b;
    return m;
}

/* 1 / B^2 with B = 2^b - 1 (Eq. 8). */
static double inv_B2(int b) {
    double B = (double)((1 << b) - 1);
    return 1.0 / (B * B);
}

/* O12: the paper's greedy: "starts with high numerical precision ...
 * progressively reduces the precision until it fits in the total bits budget.
 * In each move, it chooses a b to reduce ..., such that the increment of
 * variance is minimal.  With a binary heap for picking up the optimal move".
 * Move (n, c) takes sample n from level L[c] to L[c+1]; its priority is the
 * variance increase per freed bit, w_n (1/B_{c+1}^2 - 1/B_c^2) / (L[c]-L[c+1])
 * (DESIGN reading 9); ties break by sample index, then move index. */
extern "C" int oracle_allocate_bits(const double* w, int64_t N, int64_t budget,
                                    uint32_t level_mask, uint8_t* bits) {
    int L[8];
    int m = mask_levels(level_mask, L);
    if (m < 1 || N < 0) return ORACLE_ERR_INVALID;
    if (budget < N * (int64_t)L[m - 1]) return ORACLE_ERR_BUDGET;
    double slope[8];
    for (int c = 0; c + 1 < m; ++c)
        slope[c] = (inv_B2(L[c + 1]) - inv_B2(L[c])) / (double)(L[c] - L[c + 1]);

    std::vector<int> lvl((size_t)N, 0);
    int64_t total = N * (int64_t)L[0];
    typedef std::tuple<double, int64_t, int> Move; /* (key, n, c) */
    std::priority_queue<Move, std::vector<Move>, std::greater<Move>> heap;
    if (m > 1)
        for (int64_t n = 0; n < N; ++n) heap.push(Move(w[n] * slope[0], n, 0));
    while (total > budget) {
        Move mv = heap.top();
        heap.pop();
        int64_t n = std::get<1>(mv);
        int c = std::get<2>(mv);
        lvl[n] = c + 1;
        total -= (int64_t)(L[c] - L[c + 1]);
        if (c + 2 < m) heap.push(Move(w[n] * slope[c + 1], n, c + 1));
    }
    for (int64_t n = 0; n < N; ++n) bits[n] = (uint8_t)L[lvl[n]];
    return ORACLE_OK;
}

extern "C" double oracle_objective(const double* w, const uint8_t* bits, int64_t N) {
    double s = 0.0;
    for (int64_t n = 0; n < N; ++n) {
        double B = (double)((1 << bits[n]) - 1);
        s += w[n] / (B * B);
    }
    return s;
}

/* Exhaustive search over all level assignments (tiny N only). */
static void brute_rec(const double* w, int64_t N, int64_t budget, const int* L, int m,
                      int64_t n, int64_t used, std::vector<uint8_t>& cur,
                      std::vector<uint8_t>& best, double& best_obj) {
    if (n == N) {
        double obj = oracle_objective(w, cur.data(), N);
        if (obj < best_obj) {
            best_obj = obj;
            best = cur;
        }
        return;
    }
    for (int c = 0; c < m; ++c) {
        if (used + L[c] + (N - n - 1) * (int64_t)L[m - 1] > budget) continue;
        cur[n] = (uint8_t)L[c];
        brute_rec(w, N, budget, L, m, n + 1, used + L[c], cur, best, best_obj);
    }
}

extern "C" double oracle_allocate_bruteforce(const double* w, int64_t N, int64_t budget,
                                             uint32_t level_mask, uint8_t* bits) {
    int L[8];
    int m = mask_levels(level_mask, L);
    if (m < 1 || N < 0 || N > 12 || budget < N * (int64_t)L[m - 1]) return -1.0;
    std::vector<uint8_t> cur((size_t)N), best((size_t)N);
    double best_obj = HUGE_VAL;
    brute_rec(w, N, budget, L, m, 0, 0, cur, best, best_obj);
    for (int64_t n = 0; n < N; ++n) bits[n] = best[n];
    return oracle_objective(w, bits, N);
}

/* Knapsack DP over (sample, bits used): "can be solved exactly by DP". */
extern "C" double oracle_allocate_dp(const double* w, int64_t N, int64_t budget,
                                     uint32_t level_mask, uint8_t* bits) {
    int L[8];
    int m = mask_levels(level_mask, L);
    if (m < 1 || N < 0 || budget < N * (int64_t)L[m - 1]) return -1.0;
    int64_t cap = std::min<int64_t>(budget, N * (int64_t)L[0]);
    const double INF = HUGE_VAL;
    /* dp[n][u]: min objective of samples < n using exactly u bits */
    std::vector<std::vector<double>> dp((size_t)N + 1, std::vector<double>((size_t)cap + 1, INF));
    std::vector<std::vector<int8_t>> choice((size_t)N + 1,
                                            std::vector<int8_t>((size_t)cap + 1, -1));
    dp[0][0] = 0.0;
    for (int64_t n = 0; n < N; ++n)
        for (int64_t u = 0; u <= cap; ++u) {
            if (dp[n][u] == INF) continue;
            for (int c = 0; c < m; ++c) {
                int64_t v = u + L[c];
                if (v > cap) continue;
                double B = (double)((1 << L[c]) - 1);
                double o = dp[n][u] + w[n] / (B * B);
                if (o < dp[n + 1][v]) {
                    dp[n + 1][v] = o;
                    choice[n + 1][v] = (int8_t)c;
                }
            }
        }
    int64_t bu = -1;
    for (int64_t u = 0; u <= cap; ++u)
        if (dp[N][u] < INF && (bu < 0 || dp[N][u] < dp[N][bu])) bu = u;
    if (bu < 0) return -1.0;
    int64_t u = bu;
    for (int64_t n = N; n >= 1; --n) {
        int c = choice[n][u];
        bits[n - 1] = (uint8_t)L[c];
        u -= L[c];
    }
    return oracle_objective(w, bits, N);
}

/* O8: sample n's segment holds b_n * ceil(D/G) * G / 8 bytes. */
extern "C" void oracle_offsets(const uint8_t* bits, int64_t N, int64_t D, int32_t G,
                               int64_t* off) {
    int64_t ng = ceil_div(D, G);
    off[0] = 0;
    for (int64_t n = 0; n < N; ++n) off[n + 1] = off[n] + (int64_t)bits[n] * ng * G / 8;
}

/* O4-O8 for one group whose zero point Z and range R are given:
 *   scale = RN(R / B); u_bar = B (h - Z) / R as the 14-bit fixed point
 *       q = RNE(RN(h - Z) * RN(B / R) * 2^14)                      (O4-O5)
 *   u_hat = ceil(u_bar) w.p. frac(u_bar) else floor   (O6-O7)
 *       code = (q + r) >> 14 with r uniform in [0, 2^14)
 *   codes LSB-first into a bit stream                (O8)
 * Returns the scale, or NaN if the q <= B*2^14 invariant fails. */
static float sr_pack_group(const float* h, int32_t len, int32_t G, int32_t b, uint64_t seed,
                           uint64_t e0, float Z, float R, uint8_t* seg) {
    uint32_t B = (1u << b) - 1u;
    float Bf = (float)B;
    float scale = R / Bf;
    /* degenerate group (DESIGN reading 16): every code 0, dequantises to Z */
    float inv14 = (R < 0x1p-96f) ? 0.0f : (Bf / R) * 16384.0f;
    std::memset(seg, 0, (size_t)G * (size_t)b / 8);
    for (int32_t k = 0; k < len; ++k) {
        float delta = h[k] - Z;
        /* 24b x 24b product is exact in binary64; nearbyint is RNE */
        double qd = std::nearbyint((double)delta * (double)inv14);
        uint64_t q = (uint64_t)qd;
        if (q > ((uint64_t)B << 14)) return NAN;
        uint64_t r = oracle_random14(seed, e0 + (uint64_t)k);
        uint32_t code = (uint32_t)((q + r) >> 14);
        for (int32_t t = 0; t < b; ++t) {
            int64_t bit = (int64_t)k * b + t;
            if ((code >> t) & 1u) seg[bit >> 3] |= (uint8_t)(1u << (bit & 7));
        }
    }
    return scale;
}

/* O3-O9 for one group, in the paper's order: Z = min,
 * R = RN(max - min) (O3), then O4-O8 above. */
extern "C" int oracle_quantize_group(const float* h, int32_t len, int32_t G, int32_t b,
                                     uint64_t seed, uint64_t e0, uint8_t* seg, float* zmin,
                                     float* scale) {
    float Z, M;
    group_min_max(h, len, &Z, &M);
    float R = M - Z;
    *zmin = Z;
    float s = sr_pack_group(h, len, G, b, seed, e0, Z, R, seg);
    if (std::isnan(s)) return ORACLE_ERR_INVARIANT;
    *scale = s;
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------- */
/* NEXT-1: bf16 metadata ("store the per-group range and zero points in  */
/* bfloat16, so each group costs extra 32 bits"; "R and Z ... */
/* rounded to bfloat16 BEFORE scaling (stored and used values identical)").    */
/* DESIGN reading 21: outward rounding, so [Z', Z' + R'] contains the group:   */
/*   Z' = bf16 rounded toward -inf of Z                                         */
/*   R' = bf16 rounded toward +inf of RU32(M - Z')  (>= the exact M - Z')       */
/* then O4-O10 run with (Z, R) := (float(Z'), float(R')).                       */
/* ------------------------------------------------------------------------- */
static uint32_t f2u(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}
static float u2f(uint32_t u) {
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

/* bf16 toward -inf / toward +inf of a finite fp32 value (bf16 = high 16 bits;
 * the bit pattern of same-signed floats is monotone in magnitude). */
static uint16_t bf16_down(float f) {
    uint32_t u = f2u(f);
    uint32_t hi = u >> 16;
    if ((u & 0xFFFFu) && (u >> 31)) hi += 1; /* negative: away from zero */
    return (uint16_t)hi;
}
static uint16_t bf16_up(float f) {
    uint32_t u = f2u(f);
    uint32_t hi = u >> 16;
    if ((u & 0xFFFFu) && !(u >> 31)) hi += 1; /* positive: away from zero */
    return (uint16_t)hi;
}

/* RU(a - b) in fp32: RN difference plus Knuth's exact TwoSum error term. */
static float sub_round_up(float a, float b) {
    float nb = -b;
    float s = a + nb;
    float bv = s - a;
    float av = s - bv;
    float err = (a - av) + (nb - bv);
    if (err > 0.0f) s = std::nextafterf(s, INFINITY);
    return s;
}

extern "C" uint32_t oracle_meta_bf16(float Z, float M) {
    uint16_t zb = bf16_down(Z);
    float Zp = u2f((uint32_t)zb << 16);
    uint16_t rb = bf16_up(sub_round_up(M, Zp));
    return (uint32_t)zb | ((uint32_t)rb << 16);
}

extern "C" int oracle_quantize_group_bf16meta(const float* h, int32_t len, int32_t G, int32_t b,
                                              uint64_t seed, uint64_t e0, uint8_t* seg,
                                              uint32_t* meta) {
    float Z, M;
    group_min_max(h, len, &Z, &M);
    uint32_t w = oracle_meta_bf16(Z, M);
    *meta = w;
    float Zs = u2f(w << 16), Rs = u2f(w & 0xFFFF0000u);
    float s = sr_pack_group(h, len, G, b, seed, e0, Zs, Rs, seg);
    return std::isnan(s) ? ORACLE_ERR_INVARIANT : ORACLE_OK;
}

/* Samples [n0, n1) of a tensor; shared by the thread fan-out below. */
static int quantize_range(const void* x, int dtype, int64_t n0, int64_t n1, int64_t D,
                          int32_t G, const uint8_t* bits, const int64_t* off, uint64_t seed,
                          int64_t sample_base, uint8_t* packed, float* zmin, float* scale,
                          uint32_t* meta) {
    int64_t ng = ceil_div(D, G);
    std::vector<float> h(G);
    for (int64_t n = n0; n < n1; ++n) {
        int32_t b = bits[n];
        for (int64_t i = 0; i < ng; ++i) {
            int32_t len = (int32_t)std::min<int64_t>(G, D - i * G);
            for (int32_t k = 0; k < len; ++k) h[k] = widen(x, dtype, n * D + i * G + k);
            uint64_t e0 = (uint64_t)(sample_base + n) * (uint64_t)D + (uint64_t)(i * G);
            uint8_t* seg = packed + off[n] + i * (int64_t)G * b / 8;
            int st = meta ? oracle_quantize_group_bf16meta(h.data(), len, G, b, seed, e0, seg,
                                                           &meta[n * ng + i])
                          : oracle_quantize_group(h.data(), len, G, b, seed, e0, seg,
                                                  &zmin[n * ng + i], &scale[n * ng + i]);
            if (st != ORACLE_OK) return st;
        }
    }
    return ORACLE_OK;
}

static bool bits_ok(const uint8_t* bits, int64_t N) {
    for (int64_t n = 0; n < N; ++n)
        if (bits[n] < 1 || bits[n] > 8) return false;
    return true;
}

template <class F>
static int fan_out(int64_t N, int threads, F fn) {
    if (threads < 1) threads = 1;
    if (threads > N) threads = (int)(N > 0 ? N : 1);
    std::vector<int> st((size_t)threads, ORACLE_OK);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        int64_t n0 = N * t / threads, n1 = N * (t + 1) / threads;
        pool.emplace_back([&, t, n0, n1]() { st[t] = fn(n0, n1); });
    }
    for (auto& th : pool) th.join();
    for (int s : st)
        if (s != ORACLE_OK) return s;
    return ORACLE_OK;
}

extern "C" int oracle_quantize(const void* x, int dtype, int64_t N, int64_t D, int32_t G,
                               const uint8_t* bits, uint64_t seed, int64_t sample_base,
                               uint8_t* packed, float* zmin, float* scale, int threads) {
    if (N < 0 || D < 0 || G < 8 || G % 8 || sample_base < 0) return ORACLE_ERR_INVALID;
    if (!bits_ok(bits, N)) return ORACLE_ERR_INVALID;
    std::vector<int64_t> off((size_t)N + 1);
    oracle_offsets(bits, N, D, G, off.data());
    return fan_out(N, threads, [&](int64_t n0, int64_t n1) {
        return quantize_range(x, dtype, n0, n1, D, G, bits, off.data(), seed, sample_base,
                              packed, zmin, scale, nullptr);
    });
}

extern "C" int oracle_quantize_bf16meta(const void* x, int dtype, int64_t N, int64_t D,
                                        int32_t G, const uint8_t* bits, uint64_t seed,
                                        int64_t sample_base, uint8_t* packed, uint32_t* meta,
                                        int threads) {
    if (N < 0 || D < 0 || G < 8 || G % 8 || sample_base < 0) return ORACLE_ERR_INVALID;
    if (!bits_ok(bits, N)) return ORACLE_ERR_INVALID;
    std::vector<int64_t> off((size_t)N + 1);
    oracle_offsets(bits, N, D, G, off.data());
    return fan_out(N, threads, [&](int64_t n0, int64_t n1) {
        return quantize_range(x, dtype, n0, n1, D, G, bits, off.data(), seed, sample_base,
                              packed, nullptr, nullptr, meta);
    });
}

/* O10: h_hat = u_hat R / B + Z, evaluated as fmaf(code, scale, Z)
 * with scale = RN(R/B) (one rounding; DESIGN reading 5). */
extern "C" void oracle_dequantize_group(const uint8_t* seg, int32_t len, int32_t b,
                                        float zmin, float scale, uint32_t* codes, float* out) {
    for (int32_t k = 0; k < len; ++k) {
        uint32_t code = 0;
        for (int32_t t = 0; t < b; ++t) {
            int64_t bit = (int64_t)k * b + t;
            code |= (uint32_t)((seg[bit >> 3] >> (bit & 7)) & 1u) << t;
        }
        if (codes) codes[k] = code;
        if (out) out[k] = std::fmaf((float)code, scale, zmin);
    }
}

/* [N, D] tensor: per group (Z, scale) from fp32 arrays (v1) or from the bf16
 * word (NEXT-1: Z = float(Z'), scale = RN(float(R') / B)). */
static int dequantize_all(const uint8_t* packed, const float* zmin, const float* scale,
                          const uint32_t* meta, const uint8_t* bits, int64_t N, int64_t D,
                          int32_t G, void* out, int out_dtype, int threads) {
    if (N < 0 || D < 0 || G < 8 || G % 8) return ORACLE_ERR_INVALID;
    if (!bits_ok(bits, N)) return ORACLE_ERR_INVALID;
    int64_t ng = ceil_div(D, G);
    std::vector<int64_t> off((size_t)N + 1);
    oracle_offsets(bits, N, D, G, off.data());
    return fan_out(N, threads, [&](int64_t n0, int64_t n1) {
        std::vector<float> v(G);
        for (int64_t n = n0; n < n1; ++n) {
            int32_t b = bits[n];
            for (int64_t i = 0; i < ng; ++i) {
                int32_t len = (int32_t)std::min<int64_t>(G, D - i * G);
                const uint8_t* seg = packed + off[n] + i * (int64_t)G * b / 8;
                float Z, s;
                if (meta) {
                    uint32_t w = meta[n * ng + i];
                    Z = u2f(w << 16);
                    s = u2f(w & 0xFFFF0000u) / (float)((1u << b) - 1u);
                } else {
                    Z = zmin[n * ng + i];
                    s = scale[n * ng + i];
                }
                oracle_dequantize_group(seg, len, b, Z, s, nullptr, v.data());
                for (int32_t k = 0; k < len; ++k) {
                    int64_t idx = n * D + i * G + k;
                    if (out_dtype == ORACLE_F32)
                        ((float*)out)[idx] = v[k];
                    else
                        ((uint16_t*)out)[idx] = to_bf16_rne(v[k]);
                }
            }
        }
        return ORACLE_OK;
    });
}

extern "C" int oracle_dequantize(const uint8_t* packed, const float* zmin, const float* scale,
                                 const uint8_t* bits, int64_t N, int64_t D, int32_t G,
                                 void* out, int out_dtype, int threads) {
    return dequantize_all(packed, zmin, scale, nullptr, bits, N, D, G, out, out_dtype, threads);
}

extern "C" int oracle_dequantize_bf16meta(const uint8_t* packed, const uint32_t* meta,
                                          const uint8_t* bits, int64_t N, int64_t D, int32_t G,
                                          void* out, int out_dtype, int threads) {
    return dequantize_all(packed, nullptr, nullptr, meta, bits, N, D, G, out, out_dtype,
                          threads);
}

/* ------------------------------------------------------------------------- */
/* NEXT-4: lossless contexts of a Conv-BN-ReLU-MaxPool block.                  */
/* ------------------------------------------------------------------------- */

static void store_val(void* p, int dtype, int64_t idx, float v) {
    if (dtype == ORACLE_F32)
        ((float*)p)[idx] = v;
    else
        ((uint16_t*)p)[idx] = to_bf16_rne(v);
}

/* ReLU (App. B.3): "ReLU layers are particularly simple, which
 * have f'(x_i) = I(x_i > 0).  Therefore, ReLU layers only take a single bit per
 * dimension to store, without any approximation."  Bit k of the LSB-first
 * stream = (x_k > 0); y_k = x_k if x_k > 0 else +0 (when y is given). */
extern "C" int oracle_relu_pack(const void* x, int dtype, int64_t E, uint8_t* mask, void* y) {
    if (E < 0) return ORACLE_ERR_INVALID;
    std::memset(mask, 0, (size_t)((E + 7) / 8));
    for (int64_t k = 0; k < E; ++k) {
        float v = widen(x, dtype, k);
        bool pos = v > 0.0f;
        if (pos) mask[k >> 3] |= (uint8_t)(1u << (k & 7));
        if (y) store_val(y, dtype, k, pos ? v : 0.0f);
    }
    return ORACLE_OK;
}

/* grad_x = f'(x) * grad_y with the stored bit: grad_y where the bit is set,
 * +0 elsewhere (exact, zero variance). */
extern "C" int oracle_relu_backward(const uint8_t* mask, const void* gy, int dtype, int64_t E,
                                    void* gx) {
    if (E < 0) return ORACLE_ERR_INVALID;
    for (int64_t k = 0; k < E; ++k) {
        bool on = (mask[k >> 3] >> (k & 7)) & 1u;
        store_val(gx, dtype, k, on ? widen(gy, dtype, k) : 0.0f);
    }
    return ORACLE_OK;
}

/* Max pooling (App. B.4) over NCHW planes, PyTorch geometry
 * (kernel kh x kw, stride, zero-free padding, dilation, floor mode):
 *   y[n,c,i,j] = max over the window's in-bounds taps,
 *   k[n,c,i,j] = argmax_{Delta} (first maximum in row-major tap order), stored
 *   as 8 bits per output location ("We use 8 bits per output location").
 * OH/OW must equal floor((H + 2p - d(k-1) - 1)/s) + 1. */
static int64_t pool_out(int64_t H, int k, int s, int p, int d) {
    return (H + 2 * (int64_t)p - (int64_t)d * (k - 1) - 1) / s + 1;
}

static bool pool_ok(int64_t NC, int64_t H, int64_t W, int kh, int kw, int sh, int sw, int ph,
                    int pw, int dh, int dw, int64_t OH, int64_t OW) {
    if (NC < 0 || H < 1 || W < 1 || kh < 1 || kw < 1 || kh * kw > 256) return false;
    if (sh < 1 || sw < 1 || dh < 1 || dw < 1 || ph < 0 || pw < 0) return false;
    if (2 * ph > kh || 2 * pw > kw) return false; /* PyTorch: pad <= kernel / 2 */
    return OH == pool_out(H, kh, sh, ph, dh) && OW == pool_out(W, kw, sw, pw, dw) && OH > 0 &&
           OW > 0;
}

extern "C" int oracle_maxpool2d_forward(const void* x, int dtype, int64_t NC, int64_t H,
                                        int64_t W, int kh, int kw, int sh, int sw, int ph, int pw,
                                        int dh, int dw, int64_t OH, int64_t OW, void* y,
                                        uint8_t* idx) {
    if (!pool_ok(NC, H, W, kh, kw, sh, sw, ph, pw, dh, dw, OH, OW)) return ORACLE_ERR_INVALID;
    for (int64_t p = 0; p < NC; ++p)
        for (int64_t i = 0; i < OH; ++i)
            for (int64_t j = 0; j < OW; ++j) {
                bool have = false;
                float best = 0.0f;
                int arg = 0;
                for (int a = 0; a < kh; ++a)
                    for (int b = 0; b < kw; ++b) {
                        int64_t r = i * sh - ph + (int64_t)a * dh;
                        int64_t c = j * sw - pw + (int64_t)b * dw;
                        if (r < 0 || r >= H || c < 0 || c >= W) continue;
                        float v = widen(x, dtype, (p * H + r) * W + c);
                        if (!have || v > best) {
                            best = v;
                            arg = a * kw + b;
                            have = true;
                        }
                    }
                int64_t o = (p * OH + i) * OW + j;
                store_val(y, dtype, o, best);
                idx[o] = (uint8_t)arg;
            }
    return ORACLE_OK;
}

/* grad_x[n,c,r,c'] = sum over output windows containing (r, c') whose stored
 * argmax is that tap, of grad_y, accumulated in fp32 in
 * increasing output (i, j) order from +0, then stored (bf16: RNE). */
extern "C" int oracle_maxpool2d_backward(const uint8_t* idx, const void* gy, int dtype,
                                         int64_t NC, int64_t H, int64_t W, int kh, int kw,
                                         int sh, int sw, int ph, int pw, int dh, int dw,
                                         int64_t OH, int64_t OW, void* gx) {
    if (!pool_ok(NC, H, W, kh, kw, sh, sw, ph, pw, dh, dw, OH, OW)) return ORACLE_ERR_INVALID;
    std::vector<float> acc((size_t)(H * W));
    for (int64_t p = 0; p < NC; ++p) {
        std::fill(acc.begin(), acc.end(), 0.0f);
        for (int64_t i = 0; i < OH; ++i)
            for (int64_t j = 0; j < OW; ++j) {
                int64_t o = (p * OH + i) * OW + j;
                int k = idx[o];
                int a = k / kw, b = k % kw;
                int64_t r = i * sh - ph + (int64_t)a * dh;
                int64_t c = j * sw - pw + (int64_t)b * dw;
                if (r < 0 || r >= H || c < 0 || c >= W) return ORACLE_ERR_INVARIANT;
                acc[(size_t)(r * W + c)] += widen(gy, dtype, o);
            }
        for (int64_t q = 0; q < H * W; ++q) store_val(gx, dtype, p * H * W + q, acc[(size_t)q]);
    }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------ NEXT-3 */
/* Run-time adaptation beyond stage 1: the gradient-magnitude
 * factor of the sensitivity, its two estimators, and the stage-2 per-layer
 * allocation.  DESIGN readings 22-26. */

/* Canonical sum of K fp64 terms (the O11 order, DESIGN reading 11): chunks of
 * 32 consecutive terms (zero padded), xor butterfly o = 16..1 inside a chunk,
 * chunk totals added in order starting from +0. */
static double canonical_sum(const double* t, int64_t K) {
    double s = 0.0;
    for (int64_t c = 0; c * 32 < K; ++c) {
        double v[32], u[32];
        for (int l = 0; l < 32; ++l) v[l] = (c * 32 + l < K) ? t[c * 32 + l] : 0.0;
        for (int o = 16; o >= 1; o >>= 1) {
            for (int l = 0; l < 32; ++l) u[l] = v[l] + v[l ^ o];
            for (int l = 0; l < 32; ++l) v[l] = u[l];
        }
        s = s + v[0];
    }
    return s;
}

/* O14 (the ||grad_n||^2 factor of w_n): per-sample squared
 * L2 norm of a gradient tensor g [N, D] (fp32 or bf16), fp64.  Reading 22: the
 * group of G elements is split into 32 lanes of G/32 consecutive elements;
 * lane l's term is the in-order fp64 sum of its squares (each square exact);
 * the 32 lane terms are combined by the xor butterfly o = 16..1 (elements past
 * D count as 0); the group totals are then summed in the canonical O11 order. */
extern "C" int oracle_grad_sqnorm(const void* g, int dtype, int64_t N, int64_t D, int32_t G,
                                  double* out) {
    if (N < 0 || D < 0 || G < 32 || G % 32) return ORACLE_ERR_INVALID;
    const int64_t ng = ceil_div(D, G);
    const int per = G / 32;
    std::vector<double> q((size_t)ng);
    for (int64_t n = 0; n < N; ++n) {
        for (int64_t i = 0; i < ng; ++i) {
            double v[32], u[32];
            for (int l = 0; l < 32; ++l) {
                double a = 0.0;
                for (int k = 0; k < per; ++k) {
                    int64_t d = i * G + (int64_t)l * per + k;
                    double x = d < D ? (double)widen(g, dtype, n * D + d) : 0.0;
                    a = a + x * x;
                }
                v[l] = a;
            }
            for (int o = 16; o >= 1; o >>= 1) {
                for (int l = 0; l < 32; ++l) u[l] = v[l] + v[l ^ o];
                for (int l = 0; l < 32; ++l) v[l] = u[l];
            }
            q[(size_t)i] = v[0];
        }
        out[n] = canonical_sum(q.data(), ng);
    }
    return ORACLE_OK;
}

/* O15 ("the moving average of gradient magnitude across samples"; S:369,
 * S:372-373): m <- RN(rho * m) + RN(RN(1 - rho) * mean), mean = RN(S / N) with
 * S the canonical sum of the N observations.  N == 0 leaves m unchanged. */
extern "C" int oracle_gradmag_ema(const double* obs, int64_t N, double rho, double* m) {
    if (N < 0 || !(rho >= 0.0 && rho <= 1.0)) return ORACLE_ERR_INVALID;
    if (N == 0) return ORACLE_OK;
    const double mean = canonical_sum(obs, N) / (double)N;
    const double a = rho * *m;
    const double b = (1.0 - rho) * mean;
    *m = a + b;
    return ORACLE_OK;
}

/* O16 ("the stale gradient magnitude in the last epoch"): a table
 * indexed by dataset sample id.  gather: est[n] = table[ids[n]] (cold start =
 * the caller's initial fill, 1.0 in SPEC S:371); scatter: table[ids[n]] =
 * obs[n] (ids within one batch are distinct). */
extern "C" int oracle_gradmag_gather(const double* table, int64_t T, const int64_t* ids,
                                     int64_t N, double* est) {
    for (int64_t n = 0; n < N; ++n) {
        if (ids[n] < 0 || ids[n] >= T) return ORACLE_ERR_INVALID;
        est[n] = table[ids[n]];
    }
    return ORACLE_OK;
}

extern "C" int oracle_gradmag_scatter(double* table, int64_t T, const int64_t* ids,
                                      const double* obs, int64_t N) {
    for (int64_t n = 0; n < N; ++n) {
        if (ids[n] < 0 || ids[n] >= T) return ORACLE_ERR_INVALID;
        table[ids[n]] = obs[n];
    }
    return ORACLE_OK;
}

/* Sensitivity of one (layer, sample) (P:547 w_n = G/6 ||grad_n||^2 ||R_n||^2;
 * App. B per-layer constants): reading 23,
 * w = RN(RN(sens * gscale) * lconst), absent factors = 1 (not multiplied). */
static double sens_weight(const double* sens, const double* gscale, const double* lconst,
                          int64_t l, int64_t N, int64_t n) {
    double w = sens[l * N + n];
    if (gscale) w = w * gscale[l * N + n];
    if (lconst) w = w * lconst[l];
    return w;
}

/* O17 (P:560 stage 2, Prob. 8 over all layers; P:566 greedy;
 * S:332-335): joint greedy over every (layer l, sample n).  All
 * start at the widest allowed width; the move of (l, n) from level c to c+1
 * frees D_l * (L_c - L_{c+1}) bits and has key RN(RN(w_ln * slope_c) / D_l)
 * (variance increase per freed bit, reading 24); moves are applied in
 * ascending (key, l, n, c) order from a binary heap until
 * sum_l D_l sum_n b_ln <= b_total.  budgets[l] = sum_n b_ln (P:560
 * "b^(l) <- sum_n b_n^(l)").  bits [L*N] layer-major. */
extern "C" int oracle_allocate_layers(const double* sens, const double* gscale,
                                      const double* lconst, const int64_t* D, int64_t L,
                                      int64_t N, int64_t b_total, uint32_t level_mask,
                                      uint8_t* bits, int64_t* budgets) {
    int Lv[8];
    int m = mask_levels(level_mask, Lv);
    if (m < 1 || L < 0 || N < 0) return ORACLE_ERR_INVALID;
    int64_t total = 0, floor_bits = 0;
    for (int64_t l = 0; l < L; ++l) {
        if (D[l] < 1) return ORACLE_ERR_INVALID;
        total += D[l] * N * (int64_t)Lv[0];
        floor_bits += D[l] * N * (int64_t)Lv[m - 1];
    }
    if (b_total < floor_bits) return ORACLE_ERR_BUDGET;
    double slope[8];
    for (int c = 0; c + 1 < m; ++c)
        slope[c] = (inv_B2(Lv[c + 1]) - inv_B2(Lv[c])) / (double)(Lv[c] - Lv[c + 1]);
    std::vector<int> lvl((size_t)(L * N), 0);
    typedef std::tuple<double, int64_t, int64_t, int> Move; /* (key, l, n, c) */
    std::priority_queue<Move, std::vector<Move>, std::greater<Move>> heap;
    auto key = [&](int64_t l, int64_t n, int c) {
        const double w = sens_weight(sens, gscale, lconst, l, N, n);
        return (w * slope[c]) / (double)D[l];
    };
    if (m > 1)
        for (int64_t l = 0; l < L; ++l)
            for (int64_t n = 0; n < N; ++n) heap.push(Move(key(l, n, 0), l, n, 0));
    while (total > b_total) {
        Move mv = heap.top();
        heap.pop();
        const int64_t l = std::get<1>(mv), n = std::get<2>(mv);
        const int c = std::get<3>(mv);
        lvl[(size_t)(l * N + n)] = c + 1;
        total -= D[l] * (int64_t)(Lv[c] - Lv[c + 1]);
        if (c + 2 < m) heap.push(Move(key(l, n, c + 1), l, n, c + 1));
    }
    for (int64_t l = 0; l < L; ++l) {
        int64_t s = 0;
        for (int64_t n = 0; n < N; ++n) {
            const int b = Lv[lvl[(size_t)(l * N + n)]];
            bits[l * N + n] = (uint8_t)b;
            s += b;
        }
        budgets[l] = s;
    }
    return ORACLE_OK;
}

/* Eq. 8 objective over all layers: sum_l sum_n w_ln / (2^b_ln - 1)^2. */
extern "C" double oracle_objective_layers(const double* sens, const double* gscale,
                                          const double* lconst, int64_t L, int64_t N,
                                          const uint8_t* bits) {
    double s = 0.0;
    for (int64_t l = 0; l < L; ++l)
        for (int64_t n = 0; n < N; ++n) {
            const double B = (double)((1 << bits[l * N + n]) - 1);
            s += sens_weight(sens, gscale, lconst, l, N, n) / (B * B);
        }
    return s;
}

/* Exact minimiser of Eq. 8 over all layers under sum_l D_l sum_n b_ln <=
 * b_total ("solved exactly by dynamic programming"), a knapsack DP over
 * (item, bits used); test pin only, tiny instances (L*N*b_total <= 2e6). */
extern "C" double oracle_allocate_layers_dp(const double* sens, const double* gscale,
                                            const double* lconst, const int64_t* D, int64_t L,
                                            int64_t N, int64_t b_total, uint32_t level_mask,
                                            uint8_t* bits) {
    int Lv[8];
    int m = mask_levels(level_mask, Lv);
    const int64_t K = L * N;
    if (m < 1 || K < 0 || b_total < 0 || K * (b_total + 1) > 2000000) return -1.0;
    const double INF = HUGE_VAL;
    std::vector<std::vector<double>> dp((size_t)K + 1, std::vector<double>((size_t)b_total + 1, INF));
    std::vector<std::vector<int8_t>> ch((size_t)K + 1, std::vector<int8_t>((size_t)b_total + 1, -1));
    dp[0][0] = 0.0;
    for (int64_t k = 0; k < K; ++k) {
        const int64_t l = k / N, n = k % N;
        const double w = sens_weight(sens, gscale, lconst, l, N, n);
        for (int64_t u = 0; u <= b_total; ++u) {
            if (dp[(size_t)k][(size_t)u] == INF) continue;
            for (int c = 0; c < m; ++c) {
                const int64_t v = u + D[l] * Lv[c];
                if (v > b_total) continue;
                const double B = (double)((1 << Lv[c]) - 1);
                const double o = dp[(size_t)k][(size_t)u] + w / (B * B);
                if (o < dp[(size_t)k + 1][(size_t)v]) {
                    dp[(size_t)k + 1][(size_t)v] = o;
                    ch[(size_t)k + 1][(size_t)v] = (int8_t)c;
                }
            }
        }
    }
    int64_t best_u = -1;
    double best = INF;
    for (int64_t u = 0; u <= b_total; ++u)
        if (dp[(size_t)K][(size_t)u] < best) {
            best = dp[(size_t)K][(size_t)u];
            best_u = u;
        }
    if (best_u < 0) return -1.0;
    for (int64_t k = K, u = best_u; k > 0; --k) {
        const int c = ch[(size_t)k][(size_t)u];
        const int64_t l = (k - 1) / N;
        bits[k - 1] = (uint8_t)Lv[c];
        u -= D[l] * Lv[c];
    }
    return best;
}
