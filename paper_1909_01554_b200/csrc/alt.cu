// alt.cu -- K4/K5/K7: the <2,2,2;7> recursion (Strassen-Winograd and the two
// Karstadt-Schwartz alternative-basis schemes) for GF(2), recursing down to
// the batched block-product kernel.
//
// Reference path: multiply (engine.cpp:351-382) -> basis_change (146-172) ->
// multiply_alt (293-349) with alt_recurse / parallel_leaf / fused_block_stage
// (202-289) -> yates::mode_step (yates.cpp:112-141) -> kernel64.
//
// B200 layout.  The reference stores operands Morton-interleaved down to 64x64
// blocks because its leaf is kernel64.  Here the leaf is a whole L x L product
// on the block-product kernel (L = 2^leaf_log2, thousands of bits), so only
// the top e = log2(n/L) recursion levels exist as passes and every matrix in
// flight stays row-major (the right operand as Bt, row j = column j of B):
//   * level quadrants are strided views, no interleave kernel is needed;
//   * basis change (phi/psi over the top e levels, chi on the way out) is an
//     in-place pass per level over the strided quadrants (K4);
//   * expand (alpha on A, beta on Bt) writes 7 half-size row-major children
//     per parent per level (K5), compress (gamma) folds 7 children back into
//     the 4 quadrants of the parent (K7);
//   * the 7^e leaves run as one batched launch of the block-product kernel.
// The e-level recursion with exact block products is a valid bilinear
// algorithm over the (non-commutative) ring of L x L GF(2) matrices, so C is
// bit-identical to the cubic product and to the reference's 64-level-deep run.
// All passes are HBM-streaming XOR kernels: bytes moved, not XORs, bound them.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/bmmgpu.h"
#include "common.cuh"
#include "schemes.h"

namespace bmmgpu {

int launch_transpose(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                     uint64_t kw, cudaStream_t stream);
int launch_cubic_fold(const uint64_t* dApar, uint64_t ld_a, uint64_t s_a, const uint64_t* dBtpar, uint64_t ld_b,
                      uint64_t s_b, uint64_t parents, uint64_t L, uint32_t ma, uint32_t mb, uint64_t* dQ, uint64_t ldq,
                      uint64_t s_q, cudaStream_t stream);
int launch_transpose_ld(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                        uint64_t kw, uint64_t ldbt, cudaStream_t stream);
int launch_cubic(int kernel, const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                 uint64_t ldc, uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate,
                 cudaStream_t stream, uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch);
int granularity(int kernel, uint64_t* gm, uint64_t* gn, uint64_t* gk);
int resolve_kernel(int kernel);
void set_umma_pair_reserve(int pairs);

namespace {

struct Masks7 {
    uint8_t m[7];
};
struct Masks4 {
    uint8_t m[4];
};
struct Steps {
    uint8_t t[4], s[4];
    int n;
};

// ---------------------------------------------------------------- kernels

// ---- fused passes.  The basis changes are folded into the coefficient masks (an
// e-level recursion over exact leaf products computes chi^(x)e gamma^(x)e [leaves of
// (alpha phi)^(x)e A and (beta psi)^(x)e B], and Kronecker powers compose factor-wise), so
// no separate phi / psi / chi pass exists; and one pass covers up to two recursion
// levels (16 sub-blocks in, 49 grandchildren out, or the reverse), so the level-(l+1)
// arrays are never written or read back.  HBM bytes per operand at n = 65536, e = 4:
// 16.5 x (n^2/8) instead of 30.7 x (plus 2 x 4 x (n^2/8) of in-place basis change).

template <int V>
struct Words;
template <>
struct Words<1> {
    using T = uint64_t;
    __device__ static T zero() { return 0; }
    __device__ static T x(T a, T b) { return a ^ b; }
};
template <>
struct Words<2> {
    using T = ulonglong2;
    __device__ static T zero() { return make_ulonglong2(0, 0); }
    __device__ static T x(T a, T b) { return make_ulonglong2(a.x ^ b.x, a.y ^ b.y); }
};

// Position decode shared by the fused passes: sub-blocks of ls rows x (wv * V) words,
// all extents powers of two (shifts only).
struct PassGeom {
    uint32_t sh_wv, sh_ls;  // log2(words / V per sub-block row), log2(sub-block rows)
    uint64_t ls, ws;        // sub-block rows, sub-block words
};

// Expand D levels at once: P parents (L x L, row stride ld_in words, batch stride
// bs_in) -> 7^D P descendants of size L / 2^D.  Descendant (h_1 .. h_D) of parent p
// is index p 7^D + h_1 7^(D-1) + .. + h_D, and equals sum over quadrant digits
// q_1 .. q_D of prod_i M[h_i][q_i] times the sub-block (q_1 .. q_D) of the parent
// (reference yates::mode_step with the alpha / beta programs, yates.cpp:112-141,
// engine.cpp:284-285, applied D times).
#ifndef BMMGPU_EXPAND_MINB
#define BMMGPU_EXPAND_MINB 2  // resident CTAs per SM the expand pass is compiled for (1 at 140 registers)
#endif
template <int D, int V>
__global__ void __launch_bounds__(256, BMMGPU_EXPAND_MINB) expand_pass_kernel(const uint64_t* __restrict__ in, uint64_t ld_in,
                                                          uint64_t bs_in, uint64_t total, PassGeom g,
                                                          uint64_t* __restrict__ out, uint64_t ld_out,
                                                          uint64_t bs_out, Masks7 m) {
    using W = Words<V>;
    using T = typename W::T;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = (idx & ((1ull << g.sh_wv) - 1)) * V;
        const uint64_t r = (idx >> g.sh_wv) & (g.ls - 1);
        const uint64_t p = idx >> (g.sh_wv + g.sh_ls);
        const uint64_t* base = in + p * bs_in + r * ld_in + w;
        if (D == 1) {
            T x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                x[q] = *reinterpret_cast<const T*>(base + (q >> 1) * g.ls * ld_in + (q & 1) * g.ws);
            uint64_t* dst = out + (p * 7) * bs_out + r * ld_out + w;
#pragma unroll
            for (int h = 0; h < 7; ++h) {
                T v = W::zero();
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (m.m[h] & (1u << q)) v = W::x(v, x[q]);
                *reinterpret_cast<T*>(dst + h * bs_out) = v;
            }
        } else {
            // x[4 q + q']: quadrant q of the parent, sub-quadrant q' of it
            T x[16];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2)
                    x[4 * q + q2] = *reinterpret_cast<const T*>(
                        base + ((q >> 1) * 2 + (q2 >> 1)) * g.ls * ld_in + ((q & 1) * 2 + (q2 & 1)) * g.ws);
            uint64_t* dst = out + (p * 49) * bs_out + r * ld_out + w;
#pragma unroll
            for (int h = 0; h < 7; ++h) {
                T y[4];  // sub-quadrants of child h
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2) {
                    T v = W::zero();
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (m.m[h] & (1u << q)) v = W::x(v, x[4 * q + q2]);
                    y[q2] = v;
                }
#pragma unroll
                for (int h2 = 0; h2 < 7; ++h2) {
                    T v = W::zero();
#pragma unroll
                    for (int q2 = 0; q2 < 4; ++q2)
                        if (m.m[h2] & (1u << q2)) v = W::x(v, y[q2]);
                    *reinterpret_cast<T*>(dst + (h * 7 + h2) * bs_out) = v;
                }
            }
        }
    }
}

// Compress D levels at once: 7^D P descendants (size L / 2^D, ld_in, bs_in) -> P
// parents (L x L, ld_out, bs_out); sub-block (q_1 .. q_D) of parent p = sum over
// (h_1 .. h_D) of prod_i G[q_i][h_i] times descendant (h_1 .. h_D) (gamma folded
// with chi; reference engine.cpp:288 and the chi basis change 379-380).
#ifndef BMMGPU_COMPRESS_MINB
#define BMMGPU_COMPRESS_MINB 2  // resident CTAs per SM the compress pass is compiled for
#endif
template <int D, int V>
__global__ void __launch_bounds__(256, BMMGPU_COMPRESS_MINB) compress_pass_kernel(const uint64_t* __restrict__ in, uint64_t ld_in,
                                                            uint64_t bs_in, uint64_t total, PassGeom g,
                                                            uint64_t* __restrict__ out, uint64_t ld_out,
                                                            uint64_t bs_out, Masks4 m) {
    using W = Words<V>;
    using T = typename W::T;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = (idx & ((1ull << g.sh_wv) - 1)) * V;
        const uint64_t r = (idx >> g.sh_wv) & (g.ls - 1);
        const uint64_t p = idx >> (g.sh_wv + g.sh_ls);
        uint64_t* base = out + p * bs_out + r * ld_out + w;
        if (D == 1) {
            const uint64_t* src = in + (p * 7) * bs_in + r * ld_in + w;
            T y[7];
#pragma unroll
            for (int h = 0; h < 7; ++h) y[h] = *reinterpret_cast<const T*>(src + h * bs_in);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                T v = W::zero();
#pragma unroll
                for (int h = 0; h < 7; ++h)
                    if (m.m[q] & (1u << h)) v = W::x(v, y[h]);
                *reinterpret_cast<T*>(base + (q >> 1) * g.ls * ld_out + (q & 1) * g.ws) = v;
            }
        } else {
            const uint64_t* src = in + (p * 49) * bs_in + r * ld_in + w;
            T acc[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] = W::zero();
#pragma unroll 1
            for (int h = 0; h < 7; ++h) {  // rolled: 7 loads in flight per step, acc stays in registers
                T y[7];
#pragma unroll
                for (int h2 = 0; h2 < 7; ++h2) y[h2] = *reinterpret_cast<const T*>(src + (h * 7 + h2) * bs_in);
                T c[4];  // sub-quadrants of compressed child h
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2) {
                    T v = W::zero();
#pragma unroll
                    for (int h2 = 0; h2 < 7; ++h2)
                        if (m.m[q2] & (1u << h2)) v = W::x(v, y[h2]);
                    c[q2] = v;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (m.m[q] & (1u << h))
#pragma unroll
                        for (int q2 = 0; q2 < 4; ++q2) acc[4 * q + q2] = W::x(acc[4 * q + q2], c[q2]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2)
                    *reinterpret_cast<T*>(base + ((q >> 1) * 2 + (q2 >> 1)) * g.ls * ld_out +
                                          ((q & 1) * 2 + (q2 & 1)) * g.ws) = acc[4 * q + q2];
        }
    }
}

#ifndef BMMGPU_ALT_OVERLAP
#define BMMGPU_ALT_OVERLAP 1  // CTA pairs the overlapped leaf groups leave to their passes (0: off)
#endif
#ifndef BMMGPU_ALT_OVERLAP_ORDER
#define BMMGPU_ALT_OVERLAP_ORDER 0  // pass stream order per group (alt_breadth)
#endif
#ifndef BMMGPU_ALT_OVERLAP_MIN
#define BMMGPU_ALT_OVERLAP_MIN 343  // fewest leaves per group (smaller groups: end to end lost ~1 %, profiles/r02/experiment_overlap_groups.txt)
#endif

unsigned grid_for(uint64_t total) {
    const uint64_t blocks = ceil_div(total, 256);
    return unsigned(std::min<uint64_t>(blocks, 148ull * 64));
}

// sigma: quadrant index of B (2j + k) <-> quadrant index of Bt (2k + j).
inline int sigma(int q) { return ((q & 1) << 1) | (q >> 1); }

// Linear map of an in-place program (x[t] ^= x[s] in order): bit q2 of row q says
// that the new x[q] contains the old x[q2].
void program_map(const InPlaceStep* st, int n, uint32_t (&f)[4]) {
    for (int q = 0; q < 4; ++q) f[q] = 1u << q;
    for (int i = 0; i < n; ++i) f[st[i].target] ^= f[st[i].source];
}

// alpha . phi (or beta . psi): the expand coefficients with the operand's basis change
// folded in; B's quadrant indices are mapped to Bt's through sigma when `transposed`.
Masks7 fused_expand(const char* const rows[7], const InPlaceStep* st, int n_st, bool transposed) {
    uint32_t f[4];
    program_map(st, n_st, f);
    Masks7 m{};
    for (int h = 0; h < 7; ++h) {
        const uint32_t r = row_mask(rows[h]);
        uint32_t comb = 0;
        for (int q = 0; q < 4; ++q)
            if (r & (1u << q)) comb ^= f[q];
        uint32_t out = 0;
        for (int t = 0; t < 4; ++t)
            if (comb & (1u << (transposed ? sigma(t) : t))) out |= 1u << t;
        m.m[h] = uint8_t(out);
    }
    return m;
}

// chi . gamma: the compress coefficients with the output basis change folded in.
Masks4 fused_compress(const Scheme* sc) {
    uint32_t x[4];
    program_map(sc->chi, sc->n_chi, x);
    Masks4 m{};
    for (int q = 0; q < 4; ++q) {
        uint32_t g = 0;
        for (int q2 = 0; q2 < 4; ++q2)
            if (x[q] & (1u << q2)) g ^= row_mask(sc->gamma[q2]);
        m.m[q] = uint8_t(g);
    }
    return m;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

PassGeom pass_geom(uint64_t L, int D, int V) {
    const uint64_t ls = L >> D, ws = ls / 64;
    return PassGeom{uint32_t(__builtin_ctzll(ws / V)), uint32_t(__builtin_ctzll(ls)), ls, ws};
}

int launch_expand(int D, const uint64_t* in, uint64_t ld_in, uint64_t bs_in, uint64_t P, uint64_t L, uint64_t* out,
                  uint64_t ld_out, uint64_t bs_out, const Masks7& m, cudaStream_t s) {
    const uint64_t ws = (L >> D) / 64;
    const int V = (ws % 2 == 0 && ld_in % 2 == 0 && ld_out % 2 == 0 && bs_in % 2 == 0 && bs_out % 2 == 0 &&
                   aligned16(in) && aligned16(out))
                      ? 2
                      : 1;
    const PassGeom g = pass_geom(L, D, V);
    const uint64_t total = P * g.ls * (ws / V);
    const unsigned grid = grid_for(total);
    if (D == 1 && V == 1) expand_pass_kernel<1, 1><<<grid, 256, 0, s>>>(in, ld_in, bs_in, total, g, out, ld_out, bs_out, m);
    if (D == 1 && V == 2) expand_pass_kernel<1, 2><<<grid, 256, 0, s>>>(in, ld_in, bs_in, total, g, out, ld_out, bs_out, m);
    if (D == 2 && V == 1) expand_pass_kernel<2, 1><<<grid, 256, 0, s>>>(in, ld_in, bs_in, total, g, out, ld_out, bs_out, m);
    if (D == 2 && V == 2) expand_pass_kernel<2, 2><<<grid, 256, 0, s>>>(in, ld_in, bs_in, total, g, out, ld_out, bs_out, m);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

#ifndef BMMGPU_COMPRESS_V
#define BMMGPU_COMPRESS_V 2
#endif
int launch_compress(int D, const uint64_t* in, uint64_t ld_in, uint64_t bs_in, uint64_t P, uint64_t L, uint64_t* out,
                    uint64_t ld_out, uint64_t bs_out, const Masks4& m, cudaStream_t s) {
    const uint64_t ws = (L >> D) / 64;
    const int V = (BMMGPU_COMPRESS_V == 2 && ws % 2 == 0 && ld_in % 2 == 0 && ld_out % 2 == 0 && bs_in % 2 == 0 && bs_out % 2 == 0 &&
                   aligned16(in) && aligned16(out))
                      ? 2
                      : 1;
    const PassGeom g = pass_geom(L, D, V);
    const uint64_t total = P * g.ls * (ws / V);
    const unsigned grid = grid_for(total);
    if (D == 1 && V == 1) compress_pass_kernel<1, 1><<<grid, 256, 0, s>>>(in, ld_in, bs_in, total, g, out, ld_out, bs_out, m);
    if (D == 1 && V == 2) compress_pass_kernel<1, 2><<<grid, 256, 0, s>>>(in, ld_in, bs_in, total, g, out, ld_out, bs_out, m);
    if (D == 2 && V == 1) compress_pass_kernel<2, 1><<<grid, 256, 0, s>>>(in, ld_in, bs_in, total, g, out, ld_out, bs_out, m);
    if (D == 2 && V == 2) compress_pass_kernel<2, 2><<<grid, 256, 0, s>>>(in, ld_in, bs_in, total, g, out, ld_out, bs_out, m);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

// Levels at which the breadth-first part materialises arrays: 0, then (e odd) 1, then
// every second level up to e.  The one single-level step sits at the top, where the
// arrays are smallest.
std::vector<int> pass_levels(int e) {
    std::vector<int> lv{0};
    int l = 0;
    if (e % 2) lv.push_back(l = 1);
    while (l < e) lv.push_back(l += 2);
    return lv;
}

using DevMem = DeviceBuffer;  // stream-ordered, pool-cached (common.cuh)

}  // namespace

// Breadth-first ("parallel") levels of the recursion in the scheme's basis:
// e whole-array expand passes, one batched launch of the 7^e leaf products,
// e compress passes into dC (reference parallel_leaf, engine.cpp:232-272).
int alt_breadth(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                uint64_t n, const Scheme* sc, int e, int kernel, cudaStream_t s) {
    int st;
    if (e == 0)
        return launch_cubic(kernel, dA, lda, dBt, ldbt, dC, ldc, n, n, n / 64, true, false, s, 1, 0, 0, 0);
    const Masks7 ma = fused_expand(sc->alpha, sc->phi, sc->n_phi, false);
    const Masks7 mb = fused_expand(sc->beta, sc->psi, sc->n_psi, true);
    const Masks4 mg = fused_compress(sc);

    uint64_t gm, gn, gk;
    if ((st = granularity(kernel, &gm, &gn, &gk))) return st;
    const uint64_t L = n >> e;
    // Level shifting (reference fused_block_stage, engine.cpp:202-228): with the tensor-core
    // kernel and tile-aligned leaves the last expand level runs inside the leaf launch (K2
    // fold mode forms each leaf operand from its parent's quadrants), so level e is never
    // materialised.  BMMGPU_ALT_FOLD=1 turns it on (read per call: tests switch it).
    const char* fold_env = getenv("BMMGPU_ALT_FOLD");
    const bool fold = fold_env && *fold_env == '1' && resolve_kernel(kernel) == BMMGPU_KERNEL_UMMA_F4 && L % 256 == 0;
    // Leaf panels padded to the kernel's tiles (pads stay zero).
    const uint64_t t_rows = round_up(L, gm), s_rows = round_up(L, gn);
    const uint64_t kwl = round_up(L / 64, gk / 64);
    const uint64_t cwl = s_rows / 64;
    uint64_t batch = 1;
    for (int l = 0; l < e; ++l) batch *= 7;
    auto pow7 = [](int l) {
        uint64_t p = 1;
        while (l-- > 0) p *= 7;
        return p;
    };

    // Level arrays: level 0 is the operand itself, intermediate levels are plain
    // row-major (stride L_l/64), level e uses the padded leaf panels.
    std::vector<DevMem> T(e + 1), S(e + 1);
    std::vector<uint64_t> t_ld(e + 1), s_ld(e + 1), t_bs(e + 1), s_bs(e + 1);
    for (int l = 1; l <= e; ++l) {
        const uint64_t Ll = n >> l;
        if (l < e) {
            t_ld[l] = s_ld[l] = Ll / 64;
            t_bs[l] = s_bs[l] = Ll * (Ll / 64);
        } else {
            t_ld[l] = s_ld[l] = kwl;
            t_bs[l] = t_rows * kwl;
            s_bs[l] = s_rows * kwl;
        }
    }
    t_ld[0] = lda;
    s_ld[0] = ldbt;
    t_bs[0] = s_bs[0] = 0;
    const std::vector<int> lv = pass_levels(e);
    const std::vector<int> lv_expand = fold ? pass_levels(e - 1) : lv;

    // Overlapped leaf groups (default when a group holds >= 343 leaves, i.e. e >= 4): the
    // last expand pass (level lg -> e) and the first compress pass (e -> lg) run per group of
    // 1/7 of the level-lg parents on a second stream, next to the leaf launches of the
    // neighbouring groups (in practice the compresses: profiles/r02/experiment_overlap_*), which leave
    // BMMGPU_ALT_OVERLAP CTA pairs (2 SMs each) idle for them; the leaf launches go on a
    // high-priority stream so their CTAs take SMs ahead of pending pass blocks.  Level e
    // is never whole in HBM: two group slots of T / S / Q (2/7 of the arrays).
    const int lg = lv[lv.size() - 2];  // last materialised level above the leaves
    const char* ov_env = getenv("BMMGPU_ALT_OVERLAP");
    const int ov_pairs = ov_env ? atoi(ov_env) : BMMGPU_ALT_OVERLAP;
    const char* ov_min_env = getenv("BMMGPU_ALT_OVERLAP_MIN");  // dev: fewest leaves per group
    const uint64_t ov_min = ov_min_env ? strtoull(ov_min_env, nullptr, 10) : BMMGPU_ALT_OVERLAP_MIN;
    const bool grouped = !fold && lg >= 1 && ov_pairs > 0 && pow7(e - 1) >= ov_min;
    const size_t n_pre = grouped ? lv.size() - 2 : lv_expand.size() - 1;  // whole-array expand passes

    // Expand, one or two levels per pass, freeing each parent level once consumed.
    const uint64_t* tin = dA;
    const uint64_t* sin = dBt;
    for (size_t i = 0; i < n_pre; ++i) {
        const std::vector<int>& lv = lv_expand;
        const int l0 = lv[i], l1 = lv[i + 1];
        const uint64_t Pn = pow7(l1);
        const size_t tb = size_t(Pn * t_bs[l1] * 8), sb = size_t(Pn * s_bs[l1] * 8);
        if ((st = T[l1].alloc(tb, s)) || (st = S[l1].alloc(sb, s))) return st;
        if (l1 == e && (t_rows != L || s_rows != L || kwl != L / 64)) {
            BMMGPU_CUDA_TRY(cudaMemsetAsync(T[l1].p, 0, tb, s));
            BMMGPU_CUDA_TRY(cudaMemsetAsync(S[l1].p, 0, sb, s));
            count_launch(2);
        }
        const uint64_t Ll = n >> l0, P = pow7(l0);
        if ((st = launch_expand(l1 - l0, tin, t_ld[l0], t_bs[l0], P, Ll, T[l1].u(), t_ld[l1], t_bs[l1], ma, s)) ||
            (st = launch_expand(l1 - l0, sin, s_ld[l0], s_bs[l0], P, Ll, S[l1].u(), s_ld[l1], s_bs[l1], mb, s)))
            return st;
        if (l0 > 0) {
            // parents no longer needed (stream-ordered free: no host sync)
            T[l0].release();
            S[l0].release();
        }
        tin = T[l1].u();
        sin = S[l1].u();
    }

    if (grouped) {
        const int D = e - lg;
        const uint64_t Pg = pow7(lg) / 7, per = Pg * pow7(D);  // parents / leaves per group
        const uint64_t Lg = n >> lg, q_bs = t_rows * cwl;
        const uint64_t out_ld = Lg / 64, out_bs = Lg * (Lg / 64);
        // order 0: the pass stream compresses group g, then expands g + 2 (Q in two slots);
        // order 1: expands g + 2 first, then compresses g (Q in three slots)
        const char* ord_env = getenv("BMMGPU_ALT_OVERLAP_ORDER");
        const int order = ord_env ? atoi(ord_env) : BMMGPU_ALT_OVERLAP_ORDER;
        const int q_slots = order == 1 ? 3 : 2;
        DevMem N, Tg[2], Sg[2], Qg[3];  // level-lg products; group slots
        if ((st = N.alloc(size_t(pow7(lg) * out_bs * 8), s))) return st;
        for (int k = 0; k < q_slots; ++k)
            if ((st = Qg[k].alloc(size_t(per * q_bs * 8), s))) return st;
        for (int k = 0; k < 2; ++k) {
            if ((st = Tg[k].alloc(size_t(per * t_bs[e] * 8), s)) || (st = Sg[k].alloc(size_t(per * s_bs[e] * 8), s)))
                return st;
            if (t_rows != L || s_rows != L || kwl != L / 64) {  // pads stay zero: the passes write interiors
                BMMGPU_CUDA_TRY(cudaMemsetAsync(Tg[k].p, 0, size_t(per * t_bs[e] * 8), s));
                BMMGPU_CUDA_TRY(cudaMemsetAsync(Sg[k].p, 0, size_t(per * s_bs[e] * 8), s));
                count_launch(2);
            }
        }
        StreamSet hi, lo;
        const char* prio_env = getenv("BMMGPU_ALT_OVERLAP_PRIO");  // dev: 0 = leaves at default priority
        if ((st = hi.acquire(1, prio_env && *prio_env == '0' ? 0 : 1)) || (st = lo.acquire(1, 0))) return st;
        const cudaStream_t ks = hi[0], ps = lo[0];
        struct Events {
            cudaEvent_t e[23] = {};
            ~Events() {
                for (auto v : e)
                    if (v) cudaEventDestroy(v);
            }
        } ev;
        for (auto& v : ev.e) BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&v, cudaEventDisableTiming));
        cudaEvent_t* expanded = ev.e;     // [g] on ps: group g's T / S written
        cudaEvent_t* leaves = ev.e + 7;   // [g] on ks: group g's Q written (T / S slot free)
        cudaEvent_t start = ev.e[14], done = ev.e[15];
        cudaEvent_t* compressed = ev.e + 16;  // [g] on ps: group g's Q slot read
        // error returns: both streams idle before the buffers' frees (a normal return stays
        // asynchronous: s waits for `done`, and the frees are ordered on s)
        struct DrainOnError {
            cudaStream_t a, b;
            bool ok = false;
            ~DrainOnError() {
                if (!ok) {
                    cudaStreamSynchronize(a);
                    cudaStreamSynchronize(b);
                }
            }
        } drain{ks, ps};
        struct Reserve {
            explicit Reserve(int p) { set_umma_pair_reserve(p); }
            ~Reserve() { set_umma_pair_reserve(0); }
        };
        BMMGPU_CUDA_TRY(cudaEventRecord(start, s));
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(ks, start, 0));
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(ps, start, 0));
        auto expand_group = [&](int g) -> int {
            const int k = g & 1;
            int r = launch_expand(D, tin + g * Pg * t_bs[lg], t_ld[lg], t_bs[lg], Pg, Lg, Tg[k].u(), t_ld[e], t_bs[e],
                                  ma, ps);
            if (!r)
                r = launch_expand(D, sin + g * Pg * s_bs[lg], s_ld[lg], s_bs[lg], Pg, Lg, Sg[k].u(), s_ld[e], s_bs[e],
                                  mb, ps);
            if (!r && cudaEventRecord(expanded[g], ps) != cudaSuccess) r = kEcuda;
            return r;
        };
        // dev trace (BMMGPU_GROUP_TRACE): per group, when its expand / leaves / compress end
        const bool gtrace = getenv("BMMGPU_GROUP_TRACE") != nullptr;
        struct TraceEv {
            std::vector<cudaEvent_t> v;
            ~TraceEv() {
                for (auto x : v) cudaEventDestroy(x);
            }
        } tev;
        auto mark = [&](cudaStream_t on) {
            if (!gtrace) return;
            cudaEvent_t x;
            if (cudaEventCreate(&x) == cudaSuccess) {
                cudaEventRecord(x, on);
                tev.v.push_back(x);
            }
        };
        std::vector<char> tag;
        auto tmark = [&](char c, cudaStream_t on) {
            if (gtrace) tag.push_back(c);
            mark(on);
        };
        tmark('s', ps);
        if ((st = expand_group(0))) return st;
        tmark('x', ps);
        if ((st = expand_group(1))) return st;
        tmark('x', ps);
        {
            Reserve reserve(ov_pairs);
            for (int g = 0; g < 7; ++g) {
                const int k = g & 1, kq = g % q_slots;
                BMMGPU_CUDA_TRY(cudaStreamWaitEvent(ks, expanded[g], 0));
                if (g >= q_slots) BMMGPU_CUDA_TRY(cudaStreamWaitEvent(ks, compressed[g - q_slots], 0));
                tmark('k', ks);
                for (uint64_t b0 = 0; b0 < per; b0 += 65535) {
                    const uint64_t nb = std::min<uint64_t>(65535, per - b0);
                    if ((st = launch_cubic(kernel, Tg[k].u() + b0 * t_bs[e], kwl, Sg[k].u() + b0 * s_bs[e], kwl,
                                           Qg[kq].u() + b0 * q_bs, cwl, t_rows, s_rows, kwl, true, false, ks, nb,
                                           t_bs[e], s_bs[e], q_bs)))
                        return st;
                }
                tmark('K', ks);
                BMMGPU_CUDA_TRY(cudaEventRecord(leaves[g], ks));
                BMMGPU_CUDA_TRY(cudaStreamWaitEvent(ps, leaves[g], 0));
                // T / S slot k is free once leaves g are done (ps waited for it)
                if (order == 1 && g + 2 < 7) {
                    if ((st = expand_group(g + 2))) return st;
                    tmark('x', ps);
                }
                tmark('c', ps);
                if ((st = launch_compress(D, Qg[kq].u(), cwl, q_bs, Pg, Lg, N.u() + g * Pg * out_bs, out_ld, out_bs,
                                          mg, ps)))
                    return st;
                BMMGPU_CUDA_TRY(cudaEventRecord(compressed[g], ps));
                tmark('C', ps);
                if (order != 1 && g + 2 < 7) {
                    if ((st = expand_group(g + 2))) return st;
                    tmark('x', ps);
                }
            }
        }
        BMMGPU_CUDA_TRY(cudaEventRecord(done, ps));
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(s, done, 0));
        drain.ok = true;
        if (gtrace && !tev.v.empty()) {
            // s = start, x = an expand ended, k / K = leaves began / ended, c / C = compress began / ended (ms)
            cudaEventSynchronize(tev.v.back());
            fprintf(stderr, "groups n=%llu e=%d lg=%d:", (unsigned long long)n, e, lg);
            for (size_t i = 0; i < tev.v.size(); ++i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, tev.v[0], tev.v[i]);
                fprintf(stderr, " %c%.2f", tag[i], ms);
            }
            fprintf(stderr, "\n");
        }
        T[lg].release();
        S[lg].release();
        // the remaining compress passes, level lg up to dC, on s
        DevMem cur = std::move(N), nxt;
        uint64_t cur_ld = out_ld, cur_bs = out_bs;
        for (size_t i = lv.size() - 2; i > 0; --i) {
            const int l1 = lv[i], l0 = lv[i - 1];
            const uint64_t Ll = n >> l0, Pp = pow7(l0);
            uint64_t* out;
            uint64_t o_ld, o_bs;
            if (l0 == 0) {
                out = dC;
                o_ld = ldc;
                o_bs = 0;
            } else {
                o_ld = Ll / 64;
                o_bs = Ll * (Ll / 64);
                if ((st = nxt.alloc(size_t(Pp * o_bs * 8), s))) return st;
                out = nxt.u();
            }
            if ((st = launch_compress(l1 - l0, cur.u(), cur_ld, cur_bs, Pp, Ll, out, o_ld, o_bs, mg, s))) return st;
            cur = std::move(nxt);
            cur_ld = o_ld;
            cur_bs = o_bs;
        }
        return kOk;
    }

    // Leaves: 7^e batched block products, Q row-major (t_rows x cwl words each).
    DevMem Q;
    const uint64_t q_bs = t_rows * cwl;
    if ((st = Q.alloc(size_t(batch * q_bs * 8), s))) return st;
    if (fold) {
        // leaf 7 p + h from parent p of level e - 1 (the operands themselves when e = 1)
        uint32_t pma = 0, pmb = 0;
        for (int h = 0; h < 7; ++h) {
            pma |= uint32_t(ma.m[h]) << (4 * h);
            pmb |= uint32_t(mb.m[h]) << (4 * h);
        }
        const int lp = e - 1;
        if ((st = launch_cubic_fold(tin, t_ld[lp], t_bs[lp], sin, s_ld[lp], s_bs[lp], pow7(lp), L, pma, pmb, Q.u(), cwl,
                                    q_bs, s)))
            return st;
        if (lp > 0) {
            T[lp].release();
            S[lp].release();
        }
    }
    for (uint64_t b0 = 0; b0 < (fold ? 0 : batch); b0 += 65535) {
        const uint64_t nb = std::min<uint64_t>(65535, batch - b0);
        if ((st = launch_cubic(kernel, T[e].u() + b0 * t_bs[e], kwl, S[e].u() + b0 * s_bs[e], kwl,
                               Q.u() + b0 * q_bs, cwl, t_rows, s_rows, kwl, true, false, s, nb, t_bs[e], s_bs[e],
                               q_bs)))
            return st;
    }
    if (!fold) {
        T[e].release();
        S[e].release();
    }

    // Compress back up the same levels into dC.
    DevMem cur = std::move(Q), nxt;
    uint64_t cur_ld = cwl, cur_bs = q_bs;
    for (size_t i = lv.size() - 1; i > 0; --i) {
        const int l1 = lv[i], l0 = lv[i - 1];
        const uint64_t Ll = n >> l0, Pp = pow7(l0);
        uint64_t* out;
        uint64_t out_ld, out_bs;
        if (l0 == 0) {
            out = dC;
            out_ld = ldc;
            out_bs = 0;
        } else {
            out_ld = Ll / 64;
            out_bs = Ll * (Ll / 64);
            if ((st = nxt.alloc(size_t(Pp * out_bs * 8), s))) return st;
            out = nxt.u();
        }
        if ((st = launch_compress(l1 - l0, cur.u(), cur_ld, cur_bs, Pp, Ll, out, out_ld, out_bs, mg, s))) return st;
        cur = std::move(nxt);
        cur_ld = out_ld;
        cur_bs = out_bs;
    }
    return kOk;
}

namespace {

// child = XOR of the quadrants of an L x L matrix selected by a 4-bit mask
// (one alpha / beta row of a depth-first level, reference engine.cpp:284-285).
template <int V>
__global__ void __launch_bounds__(256) select_kernel(const uint64_t* __restrict__ in, uint64_t ld_in, uint64_t total,
                                                     PassGeom g, uint64_t* __restrict__ out, uint64_t ld_out,
                                                     uint32_t mask) {
    using W = Words<V>;
    using T = typename W::T;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = (idx & ((1ull << g.sh_wv) - 1)) * V;
        const uint64_t r = idx >> g.sh_wv;
        const uint64_t* base = in + r * ld_in + w;
        T v = W::zero();
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (mask & (1u << q))
                v = W::x(v, *reinterpret_cast<const T*>(base + (q >> 1) * g.ls * ld_in + (q & 1) * g.ws));
        *reinterpret_cast<T*>(out + r * ld_out + w) = v;
    }
}

// quadrant q of C ^= child for every q in mask (one gamma column, folded as
// each child product finishes; reference engine.cpp:288).
template <int V>
__global__ void __launch_bounds__(256) scatter_xor_kernel(const uint64_t* __restrict__ q_in, uint64_t ld_q,
                                                          uint64_t total, PassGeom g, uint64_t* C, uint64_t ldc,
                                                          uint32_t mask) {
    using W = Words<V>;
    using T = typename W::T;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = (idx & ((1ull << g.sh_wv) - 1)) * V;
        const uint64_t r = idx >> g.sh_wv;
        const T v = *reinterpret_cast<const T*>(q_in + r * ld_q + w);
        uint64_t* base = C + r * ldc + w;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (mask & (1u << q)) {
                T* p = reinterpret_cast<T*>(base + (q >> 1) * g.ls * ldc + (q & 1) * g.ws);
                *p = W::x(*p, v);
            }
    }
}

// Quadrant geometry of a select / scatter: L/2 x L/2 blocks whose four sources (or
// targets) start sp rows / sp/64 words apart (sp = L/2: the quadrants of an L x L
// matrix; sp > L/2: the same-position sub-blocks of four larger quadrants).
PassGeom quad_geom(uint64_t L, uint64_t sp, int V) {
    PassGeom g = pass_geom(L, 1, V);
    if (sp) {
        g.ls = sp;
        g.ws = sp / 64;
    }
    return g;
}

int launch_select(const uint64_t* in, uint64_t ld_in, uint64_t L, uint64_t* out, uint64_t ld_out, uint32_t mask,
                  cudaStream_t s, uint64_t sp = 0) {
    const uint64_t ws = L / 128;
    const int V = (ws % 2 == 0 && ld_in % 2 == 0 && ld_out % 2 == 0 && (sp / 64) % 2 == 0 && aligned16(in) &&
                   aligned16(out))
                      ? 2
                      : 1;
    const PassGeom g = quad_geom(L, sp, V);
    const uint64_t total = (L / 2) * (ws / V);
    if (V == 2)
        select_kernel<2><<<grid_for(total), 256, 0, s>>>(in, ld_in, total, g, out, ld_out, mask);
    else
        select_kernel<1><<<grid_for(total), 256, 0, s>>>(in, ld_in, total, g, out, ld_out, mask);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

int launch_scatter(const uint64_t* q_in, uint64_t ld_q, uint64_t L, uint64_t* C, uint64_t ldc, uint32_t mask,
                   cudaStream_t s, uint64_t sp = 0) {
    if (!mask) return kOk;
    const uint64_t ws = L / 128;
    const int V = (ws % 2 == 0 && ld_q % 2 == 0 && ldc % 2 == 0 && (sp / 64) % 2 == 0 && aligned16(q_in) &&
                   aligned16(C))
                      ? 2
                      : 1;
    const PassGeom g = quad_geom(L, sp, V);
    const uint64_t total = (L / 2) * (ws / V);
    if (V == 2)
        scatter_xor_kernel<2><<<grid_for(total), 256, 0, s>>>(q_in, ld_q, total, g, C, ldc, mask);
    else
        scatter_xor_kernel<1><<<grid_for(total), 256, 0, s>>>(q_in, ld_q, total, g, C, ldc, mask);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

}  // namespace

// Depth-first ("serial") levels on top of the breadth-first ones: the 7
// children of a level are formed, multiplied and folded into C one at a
// time, so the working set per level is three quarter-size matrices
// (reference alt_recurse with its per-level T/S/Q scratch, engine.cpp:274-289).
// This is what lets products whose fully expanded levels would not fit in HBM
// (n = 262144: (7/4)^e growth) run the fast algorithm.
int alt_serial(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
               uint64_t n, const Scheme* sc, int e_serial, int e_par, int kernel, cudaStream_t s) {
    if (e_serial == 0) return alt_breadth(dA, lda, dBt, ldbt, dC, ldc, n, sc, e_par, kernel, s);
    const uint64_t half = n / 2, hw = half / 64;
    const Masks7 ma = fused_expand(sc->alpha, sc->phi, sc->n_phi, false);
    const Masks7 mb = fused_expand(sc->beta, sc->psi, sc->n_psi, true);
    const Masks4 mg = fused_compress(sc);
    int st;
    BMMGPU_CUDA_TRY(cudaMemset2DAsync(dC, ldc * 8, 0, (n / 64) * 8, n, s));
    count_launch();
    DevMem T, S, Q;
    if ((st = T.alloc(half * hw * 8, s)) || (st = S.alloc(half * hw * 8, s)) || (st = Q.alloc(half * hw * 8, s)))
        return st;
    for (int h = 0; h < 7; ++h) {
        if ((st = launch_select(dA, lda, n, T.u(), hw, ma.m[h], s)) ||
            (st = launch_select(dBt, ldbt, n, S.u(), hw, mb.m[h], s)))
            return st;
        if ((st = alt_serial(T.u(), hw, S.u(), hw, Q.u(), hw, half, sc, e_serial - 1, e_par, kernel, s))) return st;
        uint32_t cmask = 0;
        for (int q = 0; q < 4; ++q)
            if (mg.m[q] & (1u << h)) cmask |= 1u << q;
        if ((st = launch_scatter(Q.u(), hw, n, dC, ldc, cmask, s))) return st;
    }
    return kOk;
}

// Device-resident fast product: dA (n x n/64, stride lda), dBt (Bt of B, n x
// n/64, stride ldbt), dC (n x n/64, stride ldc).  e recursion levels (leaves of
// size n >> e), the top e_serial of them depth-first.  The reference's basis changes
// (phi / psi on the operands, chi on the result, engine.cpp:371-380) are folded into
// the expand / compress coefficients, so dA and dBt are only read.
int alt_multiply_device(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                        uint64_t ldc, uint64_t n, int algo, int e, int e_serial, int kernel, cudaStream_t s) {
    const Scheme* sc = scheme_for(algo);
    if (!sc) {
        set_error("no bilinear scheme for this algorithm");
        return kEinval;
    }
    if (e < 1 || (n >> e) < 64 || e_serial < 0 || e_serial > e) {
        set_error("alt_multiply_device: need 1 <= e, 0 <= e_serial <= e and leaves of at least 64 bits");
        return kEinval;
    }
    return alt_serial(dA, lda, dBt, ldbt, dC, ldc, n, sc, e_serial, e - e_serial, kernel, s);
}

// Depth-first levels needed so the breadth-first part fits in `budget` bytes:
// its peak is about four level-e arrays, 4 (7/4)^e_par (n >> e_serial)^2 / 8 bytes.
// At least one level stays breadth-first (it pads the leaves to the kernel's tiles).
int alt_serial_levels(uint64_t n, int e, uint64_t budget) {
    for (int es = 0; es < e - 1; ++es) {
        const uint64_t L = n >> es;
        double bytes = 4.0 * double(L) * double(L) / 8.0;
        for (int l = 0; l < e - es; ++l) bytes *= 1.75;
        if (bytes <= double(budget)) return es;
    }
    return e > 0 ? e - 1 : 0;
}

uint64_t free_budget(bool refresh = false) { return uint64_t(double(device_free_bytes(refresh)) * 0.8); }

// Depth-first level count for this device (BMMGPU_ALT_SERIAL forces it; tests use it).  The
// free-memory estimate is non-blocking (device_free_bytes); a plan whose breadth-first part
// would take more than half of it is re-checked against a fresh query.
int choose_serial_levels(uint64_t n, int e) {
    if (const char* env = getenv("BMMGPU_ALT_SERIAL")) return std::max(0, std::min(atoi(env), e - 1));
    const uint64_t budget = free_budget();
    const int es = alt_serial_levels(n, e, budget);
    if (alt_serial_levels(n, e, budget / 2) != es) return alt_serial_levels(n, e, free_budget(true));
    return es;
}

// Recursion levels run as passes: the leaf dimension is 2^leaf_log2
// (default 2^12: the block-product kernels reach full speed at K >= 4096).
int alt_levels(uint64_t n, int leaf_log2) {
    int depth = 0;
    while ((64ull << depth) < n) ++depth;
    int leaf = leaf_log2 > 0 ? leaf_log2 : 12;
    if (leaf < 6) leaf = 6;
    int e = depth + 6 - leaf;
    if (e < 0) e = 0;
    if (e > depth) e = depth;
    return e;
}

namespace {

bool host_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

struct EventSet {
    cudaEvent_t ev[12] = {};
    ~EventSet() {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }
};

}  // namespace

// Streamed host path of the fast product (e >= 2).  The top recursion level runs
// depth-first: its 7 children are ordered so that the first ones read the fewest
// operand quadrants, each child starts as soon as the quadrants it reads have been
// uploaded (a copy stream uploads A and B quadrant by quadrant, Bt quadrants are
// transposed as their B quadrant lands), and each quadrant of C goes back to the host
// (second copy stream) as soon as the last child contributing to it has been folded
// in.  The H2D of most of the operands and the D2H of most of C overlap the leaf
// products.  With pageable host memory the copies are host-synchronous, so the
// uploads are interleaved with the children and the downloads run at the end.
int alt_multiply_host_streamed2(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, const Scheme* sc,
                                int e, int kernel, const int* child, uint32_t split, double* timing_ms);

int alt_multiply_host_streamed(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, const Scheme* sc,
                               int e, int kernel, double* timing_ms) {
    const uint64_t w = n / 64, half = n / 2, hw = w / 2;
    const Masks7 ma = fused_expand(sc->alpha, sc->phi, sc->n_phi, false);
    const Masks7 mb = fused_expand(sc->beta, sc->psi, sc->n_psi, true);  // Bt quadrant indices
    const Masks4 mg = fused_compress(sc);
    // Child order: an exhaustive search over the 7! orders with a pipeline model --
    // one upload engine (a quadrant takes tq), children compute back to back once their
    // quadrants are in (tc each), one download engine takes each C quadrant as soon as
    // its last contributing child is done.  Minimises the modelled makespan, i.e. the
    // exposed head (first child's quadrants) plus the exposed tail (quadrants that only
    // complete with the last children).
    int order[7];
    static std::mutex order_mu;
    static std::map<std::pair<const Scheme*, uint64_t>, std::array<int, 7>> order_cache;
    std::unique_lock<std::mutex> order_lock(order_mu);
    if (auto it = order_cache.find({sc, n}); it != order_cache.end()) {
        std::copy(it->second.begin(), it->second.end(), order);
    } else {
        const double quad_bytes = double(n) * double(n) / 32.0;  // one quadrant of one operand
        const double tq = quad_bytes / 50e9;                     // PCIe 5 x16, measured ~55 GB/s
        const double tc = (2.0 * double(n) * n * n / 7.0) / 10e15; // a child at ~10 effective Pbop/s
        int perm[7] = {0, 1, 2, 3, 4, 5, 6};
        double best = 1e300;
        do {
            uint32_t upA = 0, upB = 0;
            double t_copy = 0, t_comp = 0, done[7];
            for (int i = 0; i < 7; ++i) {
                const int h = perm[i];
                t_copy += tq * (__builtin_popcount(ma.m[h] & ~upA) + __builtin_popcount(mb.m[h] & ~upB));
                upA |= ma.m[h];
                upB |= mb.m[h];
                t_comp = std::max(t_comp, t_copy) + tc;
                done[i] = t_comp;
            }
            double t_d = 0;
            for (int i = 0; i < 7; ++i)
                for (int q = 0; q < 4; ++q) {
                    bool last = (mg.m[q] >> perm[i]) & 1;
                    for (int j = i + 1; last && j < 7; ++j) last = !((mg.m[q] >> perm[j]) & 1);
                    if (last) t_d = std::max(t_d, done[i]) + tq;
                }
            const double t = std::max(t_d, done[6]);
            if (t < best - 1e-12) {
                best = t;
                std::copy(perm, perm + 7, order);
            }
        } while (std::next_permutation(perm, perm + 7));
        std::array<int, 7> o;
        std::copy(order, order + 7, o.begin());
        order_cache.emplace(std::make_pair(sc, n), o);
    }
    order_lock.unlock();
    // Page-locked operands and result: the same top level, streamed in sub-blocks.  At
    // n >= 2^17 every child runs as its 7 grandchildren (n = 262144: -45 ms span, +3.2 %
    // end to end); below that only the first and the last child do -- the exposed head
    // and tail -- since 49 grandchildren are too small to run at full rate (n = 65536:
    // +1.6 ms in the block products; microbench/stream2_diag.py).
    // BMMGPU_ALT_STREAM_LEVELS forces: 1 quadrants, 2 all children split, 3 first / last.
    const char* lv_env = getenv("BMMGPU_ALT_STREAM_LEVELS");
    const int stream_mode = lv_env ? atoi(lv_env) : (n >= (1u << 17) ? 2 : 3);
    // BMMGPU_ALT_SPLIT_MASK (dev): which child positions run as grandchildren (bit i = position i)
    const char* sm_env = getenv("BMMGPU_ALT_SPLIT_MASK");
    const uint32_t split_mask = sm_env ? uint32_t(strtoul(sm_env, nullptr, 0)) & 0x7Fu : stream_mode == 2 ? 0x7Fu : 0x41u;
    if (stream_mode >= 2 && e >= 3 && n >= 1024 && host_pinned(A) && host_pinned(B) && host_pinned(C))
        return alt_multiply_host_streamed2(A, B, C, n, sc, e, kernel, order, split_mask, timing_ms);
    int last_pos[4] = {-1, -1, -1, -1};  // position in `order` after which quadrant q of C is final
    for (int i = 0; i < 7; ++i)
        for (int q = 0; q < 4; ++q)
            if (mg.m[q] & (1u << order[i])) last_pos[q] = i;

    StreamSet ss;  // compute, uploads, downloads
    if (int r = ss.acquire(3)) return r;
    struct {
        cudaStream_t c, h, d;
    } st3{ss[0], ss[1], ss[2]};
    const cudaStream_t s = st3.c;
    EventSet evs;  // 0-3 A quadrants, 4-7 B quadrants, 8-11 C quadrants
    for (auto& ev : evs.ev) BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaEvent_t t0, t1;
    BMMGPU_CUDA_TRY(cudaEventCreate(&t0));
    BMMGPU_CUDA_TRY(cudaEventCreate(&t1));
    struct TE {
        cudaEvent_t a, b;
        ~TE() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } te{t0, t1};

    int rc;
    DevMem dA, dB, dBt, dC, T, S, Q;
    StreamDrain drain{{st3.c, st3.h, st3.d, nullptr}};
    if ((rc = dA.alloc(n * w * 8, s)) || (rc = dB.alloc(n * w * 8, s)) || (rc = dBt.alloc(n * w * 8, s)) ||
        (rc = dC.alloc(n * w * 8, s)) || (rc = T.alloc(half * hw * 8, s)) || (rc = S.alloc(half * hw * 8, s)) ||
        (rc = Q.alloc(half * hw * 8, s)))
        return rc;
    // the allocations exist once s reaches this point: the copy streams start after it, and
    // the depth-first split of the children below sees the memory they take
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
    BMMGPU_CUDA_TRY(cudaMemsetAsync(dC.p, 0, n * w * 8, s));
    count_launch();
    BMMGPU_CUDA_TRY(cudaEventRecord(t0, s));
    const bool pinned_c = host_pinned(C);
    auto quad = [&](uint64_t* base, int q) { return base + (q >> 1) * half * w + (q & 1) * hw; };
    auto cquad = [&](const uint64_t* base, int q) { return base + (q >> 1) * half * w + (q & 1) * hw; };
    uint32_t upA = 0, upB = 0, waitA = 0, doneBt = 0;
    const int e_sub = e - 1;
    const int es_sub = choose_serial_levels(half, e_sub);
    for (int i = 0; i < 7; ++i) {
        const int h = order[i];
        // uploads this child needs (B quadrant p = sigma(t) for Bt quadrant t)
        for (int q = 0; q < 4; ++q)
            if ((ma.m[h] & (1u << q)) && !(upA & (1u << q))) {
                BMMGPU_CUDA_TRY(memcpy2d_counted(quad(dA.u(), q), w * 8, cquad(A, q), w * 8, hw * 8, half,
                                                  cudaMemcpyHostToDevice, st3.h));
                BMMGPU_CUDA_TRY(cudaEventRecord(evs.ev[q], st3.h));
                upA |= 1u << q;
            }
        for (int t = 0; t < 4; ++t) {
            const int p = sigma(t);
            if ((mb.m[h] & (1u << t)) && !(upB & (1u << p))) {
                BMMGPU_CUDA_TRY(memcpy2d_counted(quad(dB.u(), p), w * 8, cquad(B, p), w * 8, hw * 8, half,
                                                  cudaMemcpyHostToDevice, st3.h));
                BMMGPU_CUDA_TRY(cudaEventRecord(evs.ev[4 + p], st3.h));
                upB |= 1u << p;
            }
        }
        for (int q = 0; q < 4; ++q)
            if ((ma.m[h] & (1u << q)) && !(waitA & (1u << q))) {
                BMMGPU_CUDA_TRY(cudaStreamWaitEvent(s, evs.ev[q]));
                waitA |= 1u << q;
            }
        for (int t = 0; t < 4; ++t)
            if ((mb.m[h] & (1u << t)) && !(doneBt & (1u << t))) {
                const int p = sigma(t);
                BMMGPU_CUDA_TRY(cudaStreamWaitEvent(s, evs.ev[4 + p]));
                if ((rc = launch_transpose_ld(quad(dB.u(), p), w, half, half, quad(dBt.u(), t), half, hw, w, s)))
                    return rc;
                doneBt |= 1u << t;
            }
        if ((rc = launch_select(dA.u(), w, n, T.u(), hw, ma.m[h], s)) ||
            (rc = launch_select(dBt.u(), w, n, S.u(), hw, mb.m[h], s)))
            return rc;
        if ((rc = alt_serial(T.u(), hw, S.u(), hw, Q.u(), hw, half, sc, es_sub, e_sub - es_sub, kernel, s)))
            return rc;
        uint32_t cmask = 0;
        for (int q = 0; q < 4; ++q)
            if (mg.m[q] & (1u << h)) cmask |= 1u << q;
        if ((rc = launch_scatter(Q.u(), hw, n, dC.u(), w, cmask, s))) return rc;
        if (pinned_c)
            for (int q = 0; q < 4; ++q)
                if (last_pos[q] == i) {
                    BMMGPU_CUDA_TRY(cudaEventRecord(evs.ev[8 + q], s));
                    BMMGPU_CUDA_TRY(cudaStreamWaitEvent(st3.d, evs.ev[8 + q]));
                    BMMGPU_CUDA_TRY(memcpy2d_counted(quad(C, q), w * 8, quad(dC.u(), q), w * 8, hw * 8, half,
                                                      cudaMemcpyDeviceToHost, st3.d));
                }
    }
    BMMGPU_CUDA_TRY(cudaEventRecord(t1, s));
    if (!pinned_c)
        BMMGPU_CUDA_TRY(memcpy2d_counted(C, w * 8, dC.p, w * 8, w * 8, n, cudaMemcpyDeviceToHost, s));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(st3.d));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    if (timing_ms) *timing_ms = ms;
    return kOk;
}

// Two-level streamed host path (e >= 3, page-locked A, B and C).  The top two levels
// run depth-first as 49 grandchildren (child-major), and the copies move n/4 x n/4
// sub-blocks instead of quadrants: a child's operand T_h (S_h) is formed sub-block
// by sub-block as the A (Bt) sub-blocks it sums arrive, a grandchild starts once the
// sub-blocks of T_h / S_h it selects exist, and each sub-block of C goes home as soon
// as its last contribution is folded in.  The exposed head shrinks from the first
// child's quadrants to the first grandchild's sub-blocks (4x smaller), the exposed
// tail from the last child's C quadrants to the sub-blocks its last grandchild
// finishes.  Orders: children by the quadrant model above, then each child's
// grandchildren by an exhaustive 7! search over a sub-block pipeline model (one
// upload engine, compute in order, one download engine), cached per (scheme, n).
namespace {

struct Orders2 {
    int child[7];
    int gc[7][7];
};

struct Model2 {
    Masks7 ma, mb;
    Masks4 mg;
    double ts, tg;  // one sub-block copy, one grandchild product

    // state after a prefix of the schedule
    struct State {
        uint32_t upA = 0, upB = 0;  // uploaded A sub-blocks (4q + u), B sub-blocks (4p + v), B indexing
        double t_up = 0, t_comp = 0, t_d = 0;
        double availA[16] = {}, availB[16] = {};
    };

    // last child (position) folding into C quadrant q
    int last_child_pos(const int* child, int q) const {
        int last = -1;
        for (int i = 0; i < 7; ++i)
            if (mg.m[q] & (1u << child[i])) last = i;
        return last;
    }

    // run child `pos` (= child[pos]) from state `st`: split, its grandchildren in order
    // `gco`; whole, one product over all four sub-blocks of its operands
    void run_child(State& st, const int* child, int pos, const int* gco, bool split) const {
        const int h = child[pos];
        int lastg[4];  // step after which Q_h sub-block j is final
        for (int j = 0; j < 4; ++j) {
            lastg[j] = split ? -1 : 0;
            for (int i = 0; split && i < 7; ++i)
                if (mg.m[j] & (1u << gco[i])) lastg[j] = i;
        }
        for (int i = 0; i < (split ? 7 : 1); ++i) {
            const uint32_t am = split ? ma.m[gco[i]] : 0xF, bm = split ? mb.m[gco[i]] : 0xF;
            double ready = 0;
            for (int q = 0; q < 4; ++q)
                for (int u = 0; u < 4; ++u) {
                    if ((ma.m[h] >> q & 1) && (am >> u & 1)) {
                        const int b = 4 * q + u;
                        if (!(st.upA >> b & 1)) {
                            st.t_up += ts;
                            st.availA[b] = st.t_up;
                            st.upA |= 1u << b;
                        }
                        ready = std::max(ready, st.availA[b]);
                    }
                    if ((mb.m[h] >> q & 1) && (bm >> u & 1)) {
                        const int b = 4 * sigma(q) + sigma(u);
                        if (!(st.upB >> b & 1)) {
                            st.t_up += ts;
                            st.availB[b] = st.t_up;
                            st.upB |= 1u << b;
                        }
                        ready = std::max(ready, st.availB[b]);
                    }
                }
            st.t_comp = std::max(st.t_comp, ready) + (split ? tg : 7 * tg);
            for (int j = 0; j < 4; ++j)
                if (lastg[j] == i)
                    for (int q = 0; q < 4; ++q)
                        if ((mg.m[q] >> h & 1) && last_child_pos(child, q) == pos) st.t_d = std::max(st.t_d, st.t_comp) + ts;
        }
    }
};

const Orders2& orders2(const Scheme* sc, const Masks7& ma, const Masks7& mb, const Masks4& mg, const int* child,
                       uint64_t n, uint32_t split) {
    static std::mutex mu;
    static std::map<std::tuple<const Scheme*, uint64_t, uint32_t>, Orders2> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({sc, n, split});
    if (it != cache.end()) return it->second;
    Model2 m{ma, mb, mg, 0, 0};
    const double q4 = double(n) / 4;
    m.ts = q4 * q4 / 8 / 50e9;
    m.tg = 2.0 * q4 * q4 * q4 / 10e15;
    Orders2 o{};
    std::copy(child, child + 7, o.child);
    Model2::State st;
    for (int pos = 0; pos < 7; ++pos) {
        int perm[7] = {0, 1, 2, 3, 4, 5, 6}, best_perm[7] = {0, 1, 2, 3, 4, 5, 6};
        double best = 1e300;
        const bool sp = split >> pos & 1;
        if (sp) do {
            Model2::State t = st;
            m.run_child(t, o.child, pos, perm, true);
            const double cost = std::max(t.t_comp, t.t_d) + 1e-3 * t.t_comp;  // finish, then compute first
            if (cost < best - 1e-12) {
                best = cost;
                std::copy(perm, perm + 7, best_perm);
            }
        } while (std::next_permutation(perm, perm + 7));
        std::copy(best_perm, best_perm + 7, o.gc[pos]);
        m.run_child(st, o.child, pos, o.gc[pos], sp);
    }
    return cache.emplace(std::make_tuple(sc, n, split), o).first->second;
}

}  // namespace

int alt_multiply_host_streamed2(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, const Scheme* sc,
                                int e, int kernel, const int* child, uint32_t split, double* timing_ms) {
    const uint64_t w = n / 64, half = n / 2, hw = w / 2, quarter = n / 4, qw = w / 4;
    const Masks7 ma = fused_expand(sc->alpha, sc->phi, sc->n_phi, false);
    const Masks7 mb = fused_expand(sc->beta, sc->psi, sc->n_psi, true);
    const Masks4 mg = fused_compress(sc);
    const Orders2& ord = orders2(sc, ma, mb, mg, child, n, split);

    StreamSet ss;  // compute, uploads, downloads
    if (int r = ss.acquire(3)) return r;
    struct Streams {
        cudaStream_t c = nullptr, h = nullptr, d = nullptr;
        cudaEvent_t ev[73] = {};  // 0-15 A blocks, 16-31 B blocks, 32-47 C blocks, 48/49 timing,
                                  // trace: 50-56 child ends, 57-72 C downloads done
        ~Streams() {
            for (auto e : ev)
                if (e) cudaEventDestroy(e);
        }
    } st3;
    st3.c = ss[0];
    st3.h = ss[1];
    st3.d = ss[2];
    const bool trace = getenv("BMMGPU_ALT_TRACE") != nullptr;  // dev: per-block timeline on stderr
    for (int i = 0; i < (trace ? 73 : 50); ++i)
        BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&st3.ev[i], trace || i >= 48 ? 0 : cudaEventDisableTiming));
    const cudaStream_t s = st3.c;
    int rc;
    DevMem dA, dB, dBt, dC, T1, S1, Q1, T2, S2, Q2;
    StreamDrain drain{{st3.c, st3.h, st3.d, nullptr}};
    if ((rc = dA.alloc(n * w * 8, s)) || (rc = dB.alloc(n * w * 8, s)) || (rc = dBt.alloc(n * w * 8, s)) ||
        (rc = dC.alloc(n * w * 8, s)) || (rc = T1.alloc(half * hw * 8, s)) || (rc = S1.alloc(half * hw * 8, s)) ||
        (rc = Q1.alloc(half * hw * 8, s)) || (rc = T2.alloc(quarter * qw * 8, s)) ||
        (rc = S2.alloc(quarter * qw * 8, s)) || (rc = Q2.alloc(quarter * qw * 8, s)))
        return rc;
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
    BMMGPU_CUDA_TRY(cudaMemsetAsync(dC.p, 0, n * w * 8, s));
    count_launch();
    BMMGPU_CUDA_TRY(cudaEventRecord(st3.ev[48], s));
    // sub-block (q, u) of an n x n matrix (ld w): quadrant q, its quadrant u
    auto blk = [&](auto* base, int q, int u) {
        return base + ((q >> 1) * half + (u >> 1) * quarter) * w + (q & 1) * hw + (u & 1) * qw;
    };
    auto sub = [&](uint64_t* base, int u) { return base + (u >> 1) * quarter * hw + (u & 1) * qw; };  // of a half
    const int e2 = e - 2, es2 = choose_serial_levels(quarter, e2);
    const int e1 = e - 1, es1 = choose_serial_levels(half, e1);
    uint32_t upA = 0, upB = 0, waitA = 0, doneBt = 0;
    // position of the last child folding into each C quadrant
    int last_pos[4] = {-1, -1, -1, -1};
    for (int i = 0; i < 7; ++i)
        for (int q = 0; q < 4; ++q)
            if (mg.m[q] & (1u << ord.child[i])) last_pos[q] = i;
    for (int pos = 0; pos < 7; ++pos) {
        const int h = ord.child[pos];
        // split: the child's 7 grandchildren one by one; whole: one product of the
        // child's full operands (its sub-blocks still formed as they arrive)
        const bool split_h = split >> pos & 1;
        uint32_t formT = 0, formS = 0;
        int lastg[4];
        for (int j = 0; j < 4; ++j) {
            lastg[j] = split_h ? -1 : 0;
            for (int i = 0; split_h && i < 7; ++i)
                if (mg.m[j] & (1u << ord.gc[pos][i])) lastg[j] = i;
        }
        if (split_h) {
            BMMGPU_CUDA_TRY(cudaMemsetAsync(Q1.p, 0, half * hw * 8, s));
            count_launch();
        }
        for (int i = 0; i < (split_h ? 7 : 1); ++i) {
            const int g = ord.gc[pos][i];
            const uint32_t am = split_h ? ma.m[g] : 0xF, bm = split_h ? mb.m[g] : 0xF;
            // T_h sub-block u = XOR of A sub-blocks (q, u), q in ma[h]; needed for u in am
            for (int u = 0; u < 4; ++u) {
                if (!(am >> u & 1) || (formT >> u & 1)) continue;
                for (int q = 0; q < 4; ++q) {
                    if (!(ma.m[h] >> q & 1)) continue;
                    const int b = 4 * q + u;
                    if (!(upA >> b & 1)) {
                        BMMGPU_CUDA_TRY(memcpy2d_counted(blk(dA.u(), q, u), w * 8, blk(A, q, u), w * 8, qw * 8,
                                                          quarter, cudaMemcpyHostToDevice, st3.h));
                        BMMGPU_CUDA_TRY(cudaEventRecord(st3.ev[b], st3.h));
                        upA |= 1u << b;
                    }
                    if (!(waitA >> b & 1)) {
                        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(s, st3.ev[b]));
                        waitA |= 1u << b;
                    }
                }
                if ((rc = launch_select(blk(dA.u(), 0, u), w, half, sub(T1.u(), u), hw, ma.m[h], s, half))) return rc;
                formT |= 1u << u;
            }
            // S_h sub-block v = XOR of Bt sub-blocks (t, v), t in mb[h]; Bt (t, v) is the
            // transpose of B (sigma t, sigma v)
            for (int v = 0; v < 4; ++v) {
                if (!(bm >> v & 1) || (formS >> v & 1)) continue;
                for (int t = 0; t < 4; ++t) {
                    if (!(mb.m[h] >> t & 1)) continue;
                    const int bt = 4 * t + v, b = 4 * sigma(t) + sigma(v);
                    if (!(upB >> b & 1)) {
                        BMMGPU_CUDA_TRY(memcpy2d_counted(blk(dB.u(), sigma(t), sigma(v)), w * 8,
                                                          blk(B, sigma(t), sigma(v)), w * 8, qw * 8, quarter,
                                                          cudaMemcpyHostToDevice, st3.h));
                        BMMGPU_CUDA_TRY(cudaEventRecord(st3.ev[16 + b], st3.h));
                        upB |= 1u << b;
                    }
                    if (!(doneBt >> bt & 1)) {
                        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(s, st3.ev[16 + b]));
                        if ((rc = launch_transpose_ld(blk(dB.u(), sigma(t), sigma(v)), w, quarter, quarter,
                                                      blk(dBt.u(), t, v), quarter, qw, w, s)))
                            return rc;
                        doneBt |= 1u << bt;
                    }
                }
                if ((rc = launch_select(blk(dBt.u(), 0, v), w, half, sub(S1.u(), v), hw, mb.m[h], s, half)))
                    return rc;
                formS |= 1u << v;
            }
            if (split_h) {
                if ((rc = launch_select(T1.u(), hw, half, T2.u(), qw, ma.m[g], s)) ||
                    (rc = launch_select(S1.u(), hw, half, S2.u(), qw, mb.m[g], s)))
                    return rc;
                if ((rc = alt_serial(T2.u(), qw, S2.u(), qw, Q2.u(), qw, quarter, sc, es2, e2 - es2, kernel, s)))
                    return rc;
                uint32_t jmask = 0;  // Q_h sub-blocks this grandchild folds into
                for (int j = 0; j < 4; ++j)
                    if (mg.m[j] & (1u << g)) jmask |= 1u << j;
                if ((rc = launch_scatter(Q2.u(), qw, half, Q1.u(), hw, jmask, s))) return rc;
            } else if ((rc = alt_serial(T1.u(), hw, S1.u(), hw, Q1.u(), hw, half, sc, es1, e1 - es1, kernel, s))) {
                return rc;
            }
            // Q_h sub-blocks that are now final go into C's quadrants (chi . gamma column h)
            uint32_t cmask = 0;
            for (int q = 0; q < 4; ++q)
                if (mg.m[q] & (1u << h)) cmask |= 1u << q;
            for (int j = 0; j < 4; ++j) {
                if (lastg[j] != i) continue;
                if ((rc = launch_scatter(sub(Q1.u(), j), hw, half, blk(dC.u(), 0, j), w, cmask, s, half))) return rc;
                for (int q = 0; q < 4; ++q)
                    if ((cmask >> q & 1) && last_pos[q] == pos) {
                        BMMGPU_CUDA_TRY(cudaEventRecord(st3.ev[32 + 4 * q + j], s));
                        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(st3.d, st3.ev[32 + 4 * q + j]));
                        BMMGPU_CUDA_TRY(memcpy2d_counted(blk(C, q, j), w * 8, blk(dC.u(), q, j), w * 8, qw * 8,
                                                          quarter, cudaMemcpyDeviceToHost, st3.d));
                        if (trace) BMMGPU_CUDA_TRY(cudaEventRecord(st3.ev[57 + 4 * q + j], st3.d));
                    }
            }
        }
        if (trace) BMMGPU_CUDA_TRY(cudaEventRecord(st3.ev[50 + pos], s));
    }
    BMMGPU_CUDA_TRY(cudaEventRecord(st3.ev[49], s));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(st3.d));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, st3.ev[48], st3.ev[49]);
    if (timing_ms) *timing_ms = ms;
    if (trace) {
        auto at = [&](int i) {
            float t = -1.f;
            if (cudaEventElapsedTime(&t, st3.ev[48], st3.ev[i]) != cudaSuccess) {
                cudaGetLastError();
                return -1.f;
            }
            return t;
        };
        fprintf(stderr, "alt streamed2 n=%llu split=0x%x span %.2f ms\n", (unsigned long long)n, split, ms);
        for (int pos = 0; pos < 7; ++pos)
            fprintf(stderr, "  child %d (h=%d): ends %.2f\n", pos, ord.child[pos], at(50 + pos));
        for (int b = 0; b < 16; ++b) fprintf(stderr, "  A(%d,%d) up %.2f   B(%d,%d) up %.2f   C(%d,%d) down %.2f\n",
                                             b / 4, b % 4, at(b), b / 4, b % 4, at(16 + b), b / 4, b % 4, at(57 + b));
    }
    return kOk;
}

// Host entry: reference-layout host buffers in, C out.
int alt_multiply_host(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int algo, const bmmgpu_plan* plan,
                      int kernel, int leaf_log2, double* timing_ms) {
    (void)plan;  // the plan's host/serial/parallel split is a CPU schedule; the GPU picks e from leaf_log2
    const int e = alt_levels(n, leaf_log2);
    kernel = resolve_kernel(kernel);
    if (e >= 2 && n >= 512 && !getenv("BMMGPU_ALT_NO_STREAM")) {
        const Scheme* sc = scheme_for(algo);
        if (!sc) {
            set_error("no bilinear scheme for this algorithm");
            return kEinval;
        }
        return alt_multiply_host_streamed(A, B, C, n, sc, e, kernel, timing_ms);
    }
    const uint64_t w = n / 64;
    StreamSet ss;
    if (int r = ss.acquire(1)) return r;
    const cudaStream_t s = ss[0];
    int st;
    DevMem dA, dB, dBt, dC;
    uint64_t gm, gn, gk;
    if ((st = granularity(kernel, &gm, &gn, &gk))) return st;
    // e == 0 needs padded panels; e > 0 works on exact n x n (leaves are padded internally)
    const uint64_t rows_a = e == 0 ? round_up(n, gm) : n;
    const uint64_t rows_b = e == 0 ? round_up(n, gn) : n;
    const uint64_t kw = e == 0 ? round_up(w, gk / 64) : w;
    const uint64_t cw = e == 0 ? rows_b / 64 : w;
    if ((st = dA.alloc(rows_a * kw * 8, s)) || (st = dB.alloc(n * w * 8, s)) ||
        (st = dBt.alloc(round_up(rows_b, 256) * kw * 8, s)) || (st = dC.alloc(rows_a * cw * 8, s)))
        return st;
    if (e == 0) {
        BMMGPU_CUDA_TRY(cudaMemsetAsync(dA.p, 0, rows_a * kw * 8, s));
        count_launch();
    }
    BMMGPU_CUDA_TRY(memcpy2d_counted(dA.p, kw * 8, A, w * 8, w * 8, n, cudaMemcpyHostToDevice, s));
    BMMGPU_CUDA_TRY(memcpy_counted(dB.p, B, n * w * 8, cudaMemcpyHostToDevice, s));
    cudaEvent_t e0, e1;
    BMMGPU_CUDA_TRY(cudaEventCreate(&e0));
    BMMGPU_CUDA_TRY(cudaEventCreate(&e1));
    BMMGPU_CUDA_TRY(cudaEventRecord(e0, s));
    if ((st = launch_transpose(dB.u(), w, n, n, dBt.u(), round_up(rows_b, 256), kw, s))) return st;
    if (e == 0)
        st = launch_cubic(kernel, dA.u(), kw, dBt.u(), kw, dC.u(), cw, rows_a, rows_b, kw, true, false, s, 1, 0, 0,
                          0);
    else
        st = alt_multiply_device(dA.u(), w, dBt.u(), w, dC.u(), w, n, algo, e, choose_serial_levels(n, e), kernel, s);
    if (st) return st;
    BMMGPU_CUDA_TRY(cudaEventRecord(e1, s));
    BMMGPU_CUDA_TRY(memcpy2d_counted(C, w * 8, dC.p, cw * 8, w * 8, n, cudaMemcpyDeviceToHost, s));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (timing_ms) *timing_ms = ms;
    return kOk;
}

int dev_multiply_partial(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                         uint64_t ldc, uint64_t n, int algo, int dh, uint32_t first, uint32_t stride, int leaf_log2,
                         int kernel, cudaStream_t s);
int host_levels_for(uint64_t n, uint32_t parts, int e);

namespace {
// Host threads of one multi-device call meet here between phases; a failed thread still
// arrives, so the others never wait forever.
struct PhaseBarrier {
    std::mutex mu;
    std::condition_variable cv;
    size_t parties, waiting = 0, gen = 0;
    explicit PhaseBarrier(size_t n) : parties(n) {}
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        const size_t g = gen;
        if (++waiting == parties) {
            waiting = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
}  // namespace

// Fast GF(2) product on several devices (one host thread each): every device holds A and
// Bt and computes the partial product of its share of the 7^dh host-layer sub-instances
// (dev_multiply_partial, dealt round robin); then device g owns output-row slab g
// (bmmgpu_slab_rows) and XOR-folds the other devices' partials of that slab, pulled by
// peer copies over NVLink, before copying it home.  The only exchange is that fold:
// (G - 1) / G of n^2 / 8 bytes in and out per device.
int alt_multiply_multi(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int algo, int dh,
                       const std::vector<int>& phys, int kernel, int leaf_log2, double* timing_ms) {
    const uint32_t G = uint32_t(phys.size());
    const uint64_t w = n / 64, rows_bt = round_up(n, 256);
    std::vector<uint64_t*> partial(G, nullptr);
    std::vector<int> status(G, kOk);
    std::vector<std::string> errors(G);
    std::vector<float> ms(G, 0.f);
    std::atomic<bool> failed{false};
    PhaseBarrier bar(G);
    void* stats = call_stats();
    auto work = [&](uint32_t g) {
        adopt_call_stats(stats);
        int st = kOk;
        StreamSet ss;
        DevMem dA, dB, dBt, dC, tmp;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        uint64_t r0 = 0, r1 = 0;
        auto fail = [&](int code) {
            status[g] = code;
            errors[g] = bmmgpu_last_error();
            failed = true;
        };
        auto phase1 = [&]() -> int {
            BMMGPU_CUDA_TRY(cudaSetDevice(phys[g]));
            int r;
            if ((r = ss.acquire(1))) return r;
            const cudaStream_t s = ss[0];
            if ((r = dA.alloc(n * w * 8, s)) || (r = dB.alloc(n * w * 8, s)) || (r = dBt.alloc(rows_bt * w * 8, s)) ||
                (r = dC.alloc(n * w * 8, s)))
                return r;
            BMMGPU_CUDA_TRY(memcpy_counted(dA.p, A, n * w * 8, cudaMemcpyHostToDevice, s));
            BMMGPU_CUDA_TRY(memcpy_counted(dB.p, B, n * w * 8, cudaMemcpyHostToDevice, s));
            BMMGPU_CUDA_TRY(cudaEventCreate(&e0));
            BMMGPU_CUDA_TRY(cudaEventCreate(&e1));
            BMMGPU_CUDA_TRY(cudaEventRecord(e0, s));
            if ((r = launch_transpose(dB.u(), w, n, n, dBt.u(), rows_bt, w, s))) return r;
            dB.release();
            if ((r = dev_multiply_partial(dA.u(), w, dBt.u(), w, dC.u(), w, n, algo, dh, g, G, leaf_log2, kernel, s)))
                return r;
            BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
            partial[g] = dC.u();
            return kOk;
        };
        auto phase2 = [&]() -> int {
            const cudaStream_t s = ss[0];
            bmmgpu_slab_rows(n, G, g, 64, &r0, &r1);
            if (r1 > r0) {
                int r;
                if ((r = tmp.alloc((r1 - r0) * w * 8, s))) return r;
                for (uint32_t d = 0; d < G; ++d) {
                    if (d == g) continue;
                    BMMGPU_CUDA_TRY(cudaMemcpyPeerAsync(tmp.p, phys[g], partial[d] + r0 * w, phys[d],
                                                        (r1 - r0) * w * 8, s));
                    if ((r = bmmgpu_dev_fold(dC.u() + r0 * w, w, tmp.u(), w, r1 - r0, w, BMMGPU_GF2_XOR_AND, s)))
                        return r;
                }
            }
            BMMGPU_CUDA_TRY(cudaEventRecord(e1, s));
            if (r1 > r0)
                BMMGPU_CUDA_TRY(memcpy2d_counted(C + r0 * w, w * 8, dC.u() + r0 * w, w * 8, w * 8, r1 - r0,
                                                 cudaMemcpyDeviceToHost, s));
            BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
            cudaEventElapsedTime(&ms[g], e0, e1);
            return kOk;
        };
        if ((st = phase1())) fail(st);
        bar.wait();  // every partial is complete (or someone failed)
        if (!failed && (st = phase2())) fail(st);
        bar.wait();  // nobody reads this device's partial any more
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (ss.n) cudaStreamSynchronize(ss[0]);
        adopt_call_stats(nullptr);
    };
    std::vector<std::thread> threads;
    for (uint32_t g = 0; g < G; ++g) threads.emplace_back(work, g);
    for (auto& t : threads) t.join();
    float worst = 0.f;
    for (uint32_t g = 0; g < G; ++g) {
        if (status[g]) {
            set_error("device " + std::to_string(phys[g]) + " (part " + std::to_string(g) + "): " + errors[g]);
            return status[g];
        }
        worst = std::max(worst, ms[g]);
    }
    if (timing_ms) *timing_ms = worst;
    return kOk;
}

int dev_multiply(uint64_t* dA, uint64_t lda, uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc, uint64_t n,
                 int algo, int leaf_log2, int kernel, cudaStream_t s) {
    if (n < 64 || (n & (n - 1))) {
        set_error("fast algorithms need n = 64 * 2^k");
        return kEshape;
    }
    if (!scheme_for(algo)) {
        set_error("no bilinear scheme for this algorithm");
        return kEinval;
    }
    kernel = resolve_kernel(kernel);
    const int e = alt_levels(n, leaf_log2);
    if (e == 0) return launch_cubic(kernel, dA, lda, dBt, ldbt, dC, ldc, n, n, n / 64, true, false, s, 1, 0, 0, 0);
    return alt_multiply_device(dA, lda, dBt, ldbt, dC, ldc, n, algo, e, choose_serial_levels(n, e), kernel, s);
}

// ------------------------------------------------ host layer on devices
// The top `dh` recursion levels as 7^dh independent sub-instances (reference pipeline
// coordinate / generate_into / aggregate, pipeline.cpp:108-179, 198-369, and the paper's
// Alg. 3): sub-instance h = (h_1 .. h_dh) multiplies
//     T_h = sum_q prod_l M_A[h_l][q_l] A_q      S_h = sum_q prod_l M_B[h_l][q_l] Bt_q
// (A_q: the sub-block of A at quadrant digits q = (q_1 .. q_dh), level 1 outermost), and
// its product Q_h goes into every C sub-block q with prod_l G[q_l][h_l] = 1.  With the
// basis changes folded into M_A = alpha.phi, M_B = beta.psi (Bt quadrant order) and
// G = chi.gamma, as in alt_serial, this is alt_serial's top dh levels flattened, so any
// subset of sub-instances gives an exact partial product and the XOR of the partials of
// a partition of the 7^dh sub-instances is A.B.  Sub-instances dealt to devices or ranks
// need no exchange until that final XOR.
namespace {

constexpr int kMaxHostLevels = 4;  // 4^4 source sub-blocks per generated operand
struct BlockList {
    uint64_t off[1 << (2 * kMaxHostLevels)];  // word offsets of the selected sub-blocks
    uint32_t count;
};

// out = XOR of the listed sub-blocks of `in` (ls rows x ws words each, row stride ld_in).
template <int V>
__global__ void __launch_bounds__(256) gather_xor_kernel(const uint64_t* __restrict__ in, uint64_t ld_in,
                                                         uint64_t total, uint32_t sh_wv, BlockList blocks,
                                                         uint64_t* __restrict__ out, uint64_t ld_out) {
    using W = Words<V>;
    using T = typename W::T;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = (idx & ((1ull << sh_wv) - 1)) * V, r = idx >> sh_wv;
        const uint64_t* base = in + r * ld_in + w;
        T v = W::zero();
        for (uint32_t i = 0; i < blocks.count; ++i) v = W::x(v, *reinterpret_cast<const T*>(base + blocks.off[i]));
        *reinterpret_cast<T*>(out + r * ld_out + w) = v;
    }
}

// every listed sub-block of C ^= q_in (distinct targets: no two threads touch one word).
template <int V>
__global__ void __launch_bounds__(256) scatter_list_kernel(const uint64_t* __restrict__ q_in, uint64_t ld_q,
                                                           uint64_t total, uint32_t sh_wv, BlockList blocks,
                                                           uint64_t* C, uint64_t ldc) {
    using W = Words<V>;
    using T = typename W::T;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = (idx & ((1ull << sh_wv) - 1)) * V, r = idx >> sh_wv;
        const T v = *reinterpret_cast<const T*>(q_in + r * ld_q + w);
        uint64_t* base = C + r * ldc + w;
        for (uint32_t i = 0; i < blocks.count; ++i) {
            T* p = reinterpret_cast<T*>(base + blocks.off[i]);
            *p = W::x(*p, v);
        }
    }
}

// Offsets of the sub-blocks q = (q_1 .. q_dh) with prod_l bit(coef(l, q_l)) = 1, for a
// matrix of n rows and row stride ld: sub-block rows = n >> dh.
template <class Coef>
BlockList block_list(int dh, uint64_t n, uint64_t ld, Coef coef) {
    BlockList b{};
    const uint64_t ls = n >> dh;
    for (uint32_t q = 0; q < (1u << (2 * dh)); ++q) {
        bool on = true;
        uint64_t br = 0, bc = 0;
        for (int l = 0; l < dh && on; ++l) {
            const uint32_t ql = (q >> (2 * (dh - 1 - l))) & 3;  // level l + 1, outermost first
            on = coef(l, ql);
            br = 2 * br + (ql >> 1);
            bc = 2 * bc + (ql & 1);
        }
        if (on) b.off[b.count++] = br * ls * ld + bc * (ls / 64);
    }
    return b;
}

int launch_block_list(bool scatter, const uint64_t* src, uint64_t ld_src, uint64_t* dst, uint64_t ld_dst,
                      uint64_t ls, const BlockList& b, cudaStream_t s) {
    const uint64_t ws = ls / 64;
    bool v2 = ws % 2 == 0 && ld_src % 2 == 0 && ld_dst % 2 == 0 && aligned16(src) && aligned16(dst);
    for (uint32_t i = 0; i < b.count; ++i) v2 = v2 && b.off[i] % 2 == 0;
    const int V = v2 ? 2 : 1;
    const uint64_t total = ls * (ws / V);
    const uint32_t sh = uint32_t(__builtin_ctzll(ws / V));
    if (scatter) {
        if (!b.count) return kOk;
        if (V == 2)
            scatter_list_kernel<2><<<grid_for(total), 256, 0, s>>>(src, ld_src, total, sh, b, dst, ld_dst);
        else
            scatter_list_kernel<1><<<grid_for(total), 256, 0, s>>>(src, ld_src, total, sh, b, dst, ld_dst);
    } else if (V == 2) {
        gather_xor_kernel<2><<<grid_for(total), 256, 0, s>>>(src, ld_src, total, sh, b, dst, ld_dst);
    } else {
        gather_xor_kernel<1><<<grid_for(total), 256, 0, s>>>(src, ld_src, total, sh, b, dst, ld_dst);
    }
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

}  // namespace

// Recursion levels of the host layer for n on `parts` devices / ranks when the caller
// does not fix them: the smallest dh whose deal is within 3 % of even (ceil(7^dh / parts)
// sub-instances on the busiest part against 7^dh / parts), keeping sub-instances of at
// least 2^13 (the fast product's own leaves stay at 4096) and at least one level below.
int host_levels_for(uint64_t n, uint32_t parts, int e) {
    if (parts <= 1) return 0;
    int best = 1;
    for (int dh = 1; dh <= kMaxHostLevels && dh < e && (n >> dh) >= 8192; ++dh) {
        uint64_t subs = 1;
        for (int l = 0; l < dh; ++l) subs *= 7;
        best = dh;
        if (double((subs + parts - 1) / parts) <= 1.03 * double(subs) / parts) break;
    }
    return best;
}

// dC = the XOR of sub-instances first, first + stride, ... of the top dh levels
// (see above).  dA / dBt are only read; dC (n x n/64, stride ldc) is overwritten.
int dev_multiply_partial(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                         uint64_t ldc, uint64_t n, int algo, int dh, uint32_t first, uint32_t stride, int leaf_log2,
                         int kernel, cudaStream_t s) {
    const Scheme* sc = scheme_for(algo);
    if (!sc) {
        set_error("no bilinear scheme for this algorithm");
        return kEinval;
    }
    if (n < 64 || (n & (n - 1))) {
        set_error("fast algorithms need n = 64 * 2^k");
        return kEshape;
    }
    if (stride == 0 || first >= stride) {
        set_error("partial product: need 0 <= first < stride");
        return kEinval;
    }
    kernel = resolve_kernel(kernel);
    const int e = alt_levels(n, leaf_log2);
    if (dh < 0 || dh > kMaxHostLevels || (dh > 0 && dh > e - 1)) {
        set_error("partial product: host levels must leave at least one recursion level below them (and <= 4)");
        return kEinval;
    }
    BMMGPU_CUDA_TRY(cudaMemset2DAsync(dC, ldc * 8, 0, (n / 64) * 8, n, s));
    count_launch();
    if (dh == 0) {
        if (first != 0) return kOk;  // one sub-instance: the whole product
        if (e == 0) return launch_cubic(kernel, dA, lda, dBt, ldbt, dC, ldc, n, n, n / 64, true, false, s, 1, 0, 0, 0);
        return alt_multiply_device(dA, lda, dBt, ldbt, dC, ldc, n, algo, e, choose_serial_levels(n, e), kernel, s);
    }
    const Masks7 ma = fused_expand(sc->alpha, sc->phi, sc->n_phi, false);
    const Masks7 mb = fused_expand(sc->beta, sc->psi, sc->n_psi, true);
    const Masks4 mg = fused_compress(sc);
    uint64_t subs = 1;
    for (int l = 0; l < dh; ++l) subs *= 7;
    const uint64_t ls = n >> dh, lw = ls / 64;
    const int e_sub = e - dh;
    int st;
    DevMem T, S, Q;
    if ((st = T.alloc(ls * lw * 8, s)) || (st = S.alloc(ls * lw * 8, s)) || (st = Q.alloc(ls * lw * 8, s))) return st;
    const int e_serial = choose_serial_levels(ls, e_sub);
    for (uint64_t i = first; i < subs; i += stride) {
        int h[kMaxHostLevels];
        uint64_t r = i;
        for (int l = dh - 1; l >= 0; --l, r /= 7) h[l] = int(r % 7);
        const BlockList la = block_list(dh, n, lda, [&](int l, uint32_t q) { return (ma.m[h[l]] >> q) & 1; });
        const BlockList lb = block_list(dh, n, ldbt, [&](int l, uint32_t q) { return (mb.m[h[l]] >> q) & 1; });
        const BlockList lc = block_list(dh, n, ldc, [&](int l, uint32_t q) { return (mg.m[q] >> h[l]) & 1; });
        if ((st = launch_block_list(false, dA, lda, T.u(), lw, ls, la, s)) ||
            (st = launch_block_list(false, dBt, ldbt, S.u(), lw, ls, lb, s)) ||
            (st = alt_multiply_device(T.u(), lw, S.u(), lw, Q.u(), lw, ls, algo, e_sub, e_serial, kernel, s)) ||
            (st = launch_block_list(true, Q.u(), lw, dC, ldc, ls, lc, s)))
            return st;
    }
    return kOk;
}

// ------------------------------------------------ out of core through the host levels
// The paper's route for products beyond accelerator memory (reference
// pipeline::coordinate, pipeline.cpp:198-369) with the generation moved onto the device:
// the top dh levels are 7^dh sub-instances of n >> dh; for sub-instance h the source
// sub-blocks its fused alpha.phi / beta.psi rows select are streamed from host memory one by
// one and XOR-accumulated on the device into T_h / S_h (B's sub-blocks transposed on the
// way), the product Q_h runs as the device-resident recursion of the remaining levels, and
// Q_h goes home where host threads XOR it into every C sub-block its chi.gamma column
// selects.  Against output tiles of full block products (alt_tiles.cu) this does the
// recursion's own 7^dh products instead of 8^dh (49 against 64 at dh = 2), at the price of
// more uploads (each source sub-block once per sub-instance that selects it) and a host
// fold.  Per device buffers: T, S, Q twice (the next sub-instance is generated while the
// current one multiplies), two upload slots per operand and one transpose buffer.
namespace {

struct BlockCoords {
    uint32_t br[1 << (2 * kMaxHostLevels)], bc[1 << (2 * kMaxHostLevels)];
    uint32_t count;
};
template <class Coef>
BlockCoords block_coords(int dh, Coef coef) {
    BlockCoords b{};
    for (uint32_t q = 0; q < (1u << (2 * dh)); ++q) {
        bool on = true;
        uint32_t br = 0, bc = 0;
        for (int l = 0; l < dh && on; ++l) {
            const uint32_t ql = (q >> (2 * (dh - 1 - l))) & 3;
            on = coef(l, ql);
            br = 2 * br + (ql >> 1);
            bc = 2 * bc + (ql & 1);
        }
        if (on) {
            b.br[b.count] = br;
            b.bc[b.count++] = bc;
        }
    }
    return b;
}

// page-locked host buffers for the Q_h downloads, kept across calls (pinning GiBs costs ~0.1 s/GiB)
constexpr int kQSlots = 4;  // downloaded Q's the host fold may lag behind by
struct PinnedCache {
    std::mutex call_mu;  // one out-of-core sub-instance call per device at a time (they share these)
    std::mutex mu;
    void* p[kQSlots] = {};
    size_t bytes = 0;
    bool get(size_t need, void* (&out)[kQSlots]) {
        std::lock_guard<std::mutex> lk(mu);
        if (bytes < need) {
            for (auto& x : p)
                if (x) cudaFreeHost(x), x = nullptr;
            bytes = 0;
            for (auto& x : p)
                if (cudaHostAlloc(&x, need, cudaHostAllocPortable) != cudaSuccess) return false;
            bytes = need;
        }
        for (int k = 0; k < kQSlots; ++k) out[k] = p[k];
        return true;
    }
};
PinnedCache g_q_pinned[32];

}  // namespace

// Host levels for the out-of-core sub-instance driver: the fewest (>= 1) whose per-device
// working set -- the two generated top-level children (2 (n/2)^2/8) and ~11 sub-instance
// arrays -- fits `budget`, with sub-instances of at least 2^13 and one level below them.
int subinst_levels(uint64_t n, int e, uint64_t budget) {
    for (int dh = 1; dh <= kMaxHostLevels && dh < e && (n >> dh) >= 8192; ++dh) {
        const double ls = double(n >> dh), h = double(n / 2);
        if (2.0 * h * h / 8.0 + 11.0 * ls * ls / 8.0 <= double(budget)) return dh;
    }
    return std::min(std::max(1, e - 1), kMaxHostLevels);
}

int alt_multiply_subinst(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int algo, int dh,
                         int kernel, int leaf_log2, uint64_t budget, double* timing_ms) {
    const Scheme* sc = scheme_for(algo);
    if (!sc) {
        set_error("no bilinear scheme for this algorithm");
        return kEinval;
    }
    kernel = resolve_kernel(kernel);
    const int e = alt_levels(n, leaf_log2);
    if (e < 2 || n < 512) {
        set_error("out-of-core sub-instances need n >= 512 and at least two recursion levels");
        return kEinval;
    }
    if (dh <= 0) dh = subinst_levels(n, e, budget);
    dh = std::min({dh, kMaxHostLevels, e - 1});
    while (dh > 1 && (n >> dh) < 256) --dh;  // sub-instances stay multiples of the kernel tile
    const Masks7 ma = fused_expand(sc->alpha, sc->phi, sc->n_phi, false);
    const Masks7 mb = fused_expand(sc->beta, sc->psi, sc->n_psi, true);
    const Masks4 mg = fused_compress(sc);
    const uint64_t w = n / 64, half = n / 2, hw = half / 64, ls = n >> dh, lw = ls / 64, blk = ls * lw * 8;
    const uint64_t P = uint64_t(1) << (dh - 1);  // pieces per quadrant side (ls x ls each)
    uint64_t subs = 1, per_top = 1;
    for (int l = 0; l < dh; ++l) subs *= 7;
    per_top = subs / 7;
    const int e_sub = e - dh;
    int dev = 0;
    BMMGPU_CUDA_TRY(cudaGetDevice(&dev));
    void* qh[kQSlots];
    if (dev >= 32) {
        set_error("out-of-core sub-instances: device index");
        return kEinval;
    }
    std::lock_guard<std::mutex> one_call(g_q_pinned[dev].call_mu);
    if (!g_q_pinned[dev].get(blk, qh)) {
        set_error("out-of-core sub-instances: page-locked host buffers for Q");
        return kEcuda;
    }
    StreamSet ss;  // 0 compute, 1 uploads, 2 generation, 3 downloads
    if (int r = ss.acquire(4)) return r;
    const cudaStream_t s = ss[0], h = ss[1], x = ss[2], d = ss[3];
    struct Events {
        cudaEvent_t e[16] = {};
        ~Events() {
            for (auto v : e)
                if (v) cudaEventDestroy(v);
        }
    } ev;
    for (int i = 0; i < 14; ++i) BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev.e[i], cudaEventDisableTiming));
    BMMGPU_CUDA_TRY(cudaEventCreate(&ev.e[14]));
    BMMGPU_CUDA_TRY(cudaEventCreate(&ev.e[15]));
    cudaEvent_t* formed = ev.e + 0;    // [slot] on x: T / S of the slot's sub-instance ready
    cudaEvent_t* consumed = ev.e + 2;  // [slot] on s: its product done (T, S read; Q written)
    cudaEvent_t* hdown = ev.e + 4;     // [host slot] on d: Q copied home (kQSlots of them)
    cudaEvent_t up = ev.e[8];          // on h: the upload slot filled
    cudaEvent_t up_free = ev.e[9];     // on x: the upload slot read
    cudaEvent_t top_free = ev.e[10];   // on x: the generated children TA / SB read for the last time
    static_assert(kQSlots == 4, "event layout");
    int rc;
    // TA / SB: the top-level child h1 of A / Bt (n/2 x n/2), generated from uploaded pieces;
    // the sub-instances of h1 gather their operands from it on the device
    DevMem TA, SB, T[2], S[2], Q[2], st, bt;
    StreamDrain drain{{s, h, x, d}};
    if ((rc = TA.alloc(half * hw * 8, s)) || (rc = SB.alloc(half * hw * 8, s)) || (rc = st.alloc(blk, s)) ||
        (rc = bt.alloc(blk, s)))
        return rc;
    for (int k = 0; k < 2; ++k)
        if ((rc = T[k].alloc(blk, s)) || (rc = S[k].alloc(blk, s)) || (rc = Q[k].alloc(blk, s))) return rc;
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));  // the pool allocations, before the other streams use them
    const uint64_t driver_bytes = 2 * half * hw * 8 + 8 * blk;
    const int e_serial = budget > driver_bytes ? alt_serial_levels(ls, e_sub, uint64_t(0.8 * double(budget - driver_bytes)))
                                               : std::max(0, e_sub - 1);
    // host fold: one thread consumes the downloaded Q's in order
    std::mutex mu;
    std::condition_variable cv;
    uint64_t queued = 0, folded = 0;
    int fold_status = kOk;
    std::vector<uint8_t> touched(size_t(1) << (2 * dh), 0);
    std::vector<BlockCoords> lcs(static_cast<size_t>(subs));
    const bool trace = getenv("BMMGPU_SUBINST_TRACE") != nullptr;  // dev: host-side waits on stderr
    // dev trace: compute start / end of every sub-instance on s (timing events)
    std::vector<cudaEvent_t> tr_ev;
    struct TrEv {
        std::vector<cudaEvent_t>& v;
        ~TrEv() {
            for (auto e2 : v) cudaEventDestroy(e2);
        }
    } tr_guard{tr_ev};
    if (trace) {
        tr_ev.resize(size_t(2 * subs));
        for (auto& e2 : tr_ev) BMMGPU_CUDA_TRY(cudaEventCreate(&e2));
    }
    double fold_busy_s = 0, main_wait_s = 0;
    const auto wall0 = std::chrono::steady_clock::now();
    std::thread folder([&] {
        for (uint64_t i = 0; i < subs; ++i) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return queued > i || fold_status != kOk; });
                if (fold_status != kOk) return;
            }
            const int hslot = int(i % kQSlots);
            if (cudaEventSynchronize(hdown[hslot]) != cudaSuccess) {
                std::lock_guard<std::mutex> lk(mu);
                fold_status = kEcuda;
                cv.notify_all();
                return;
            }
            const auto f0 = std::chrono::steady_clock::now();
            const uint64_t* q = static_cast<const uint64_t*>(qh[hslot]);
            const BlockCoords& lc = lcs[size_t(i)];
            for (uint32_t t = 0; t < lc.count; ++t) {
                const uint32_t id = (lc.br[t] << dh) | lc.bc[t];
                const bool first = !touched[id];
                touched[id] = 1;
                uint64_t* c0 = C + uint64_t(lc.br[t]) * ls * w + uint64_t(lc.bc[t]) * lw;
                const unsigned parts = std::max(1u, host_parallel_width());
                const uint64_t step = (ls + parts - 1) / parts;
                host_parallel(parts, [&](unsigned pi) {
                    const uint64_t r0 = std::min<uint64_t>(ls, pi * step), r1 = std::min<uint64_t>(ls, r0 + step);
                    for (uint64_t r = r0; r < r1; ++r) {
                        uint64_t* dst = c0 + r * w;
                        const uint64_t* src = q + r * lw;
                        if (first)
                            std::memcpy(dst, src, lw * 8);
                        else
                            for (uint64_t j = 0; j < lw; ++j) dst[j] ^= src[j];
                    }
                });
            }
            std::lock_guard<std::mutex> lk(mu);
            fold_busy_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - f0).count();
            ++folded;
            cv.notify_all();
        }
    });
    auto stop_folder = [&](int status) {
        {
            std::lock_guard<std::mutex> lk(mu);
            if (status != kOk && fold_status == kOk) fold_status = status;
        }
        cv.notify_all();
        if (folder.joinable()) folder.join();
    };
    // every early return below (BMMGPU_CUDA_TRY) must still stop and join the fold thread
    struct FolderGuard {
        std::function<void()> f;
        ~FolderGuard() { f(); }
    } folder_guard{[&] { stop_folder(kEcuda); }};
    // Order of the top-level children: consecutive children update TA / SB in place by the
    // quadrants in which their alpha.phi (beta.psi) rows differ (XOR is its own inverse), so
    // the order with the fewest such quadrants (the first child's full rows plus the
    // symmetric differences) is searched over the 7! orders
    int h1_order[7] = {0, 1, 2, 3, 4, 5, 6};
    {
        int perm[7] = {0, 1, 2, 3, 4, 5, 6}, best = 1 << 30;
        do {
            int cost = __builtin_popcount(ma.m[perm[0]]) + __builtin_popcount(mb.m[perm[0]]);
            for (int k = 1; k < 7; ++k)
                cost += __builtin_popcount(ma.m[perm[k]] ^ ma.m[perm[k - 1]]) +
                        __builtin_popcount(mb.m[perm[k]] ^ mb.m[perm[k - 1]]);
            if (cost < best) {
                best = cost;
                std::copy(perm, perm + 7, h1_order);
            }
        } while (std::next_permutation(perm, perm + 7));
    }
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[14], s));
    uint64_t uploads = 0;
    // one ls x ls piece from host memory into the upload slot (or straight into `direct`)
    auto upload_piece = [&](const uint64_t* src, uint64_t* direct, uint64_t ld_direct) -> cudaError_t {
        if (uploads++ > 0) {
            cudaError_t e2 = cudaStreamWaitEvent(h, up_free, 0);
            if (e2 != cudaSuccess) return e2;
        }
        cudaError_t e2 = memcpy2d_counted(direct ? static_cast<void*>(direct) : st.p, (direct ? ld_direct : lw) * 8,
                                          src, w * 8, lw * 8, ls, cudaMemcpyHostToDevice, h);
        if (e2 == cudaSuccess) e2 = cudaEventRecord(up, h);
        if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(x, up, 0);
        return e2;
    };
    rc = kOk;
    for (uint64_t i = 0; i < subs && rc == kOk; ++i) {
        const int slot = int(i & 1);
        int hd[kMaxHostLevels];
        uint64_t r = i;
        for (int l = dh - 1; l >= 0; --l, r /= 7) hd[l] = int(r % 7);
        hd[0] = h1_order[hd[0]];
        const int prev_h1 = i >= per_top ? h1_order[(i / per_top) - 1] : -1;
        lcs[size_t(i)] = block_coords(dh, [&](int l, uint32_t q) { return (mg.m[q] >> hd[l]) & 1; });
        if (i % per_top == 0) {
            // new top-level child h1: TA = XOR of the A quadrants alpha.phi row h1 selects, SB the
            // same for Bt (beta.psi), generated piece by piece as the pieces land -- the first
            // child from scratch, the next ones by XORing in the quadrants where their rows differ
            if (i > 0) BMMGPU_CUDA_TRY(cudaStreamWaitEvent(h, top_free, 0));
            for (int op = 0; op < 2 && rc == kOk; ++op) {
                uint64_t* dst = op ? SB.u() : TA.u();
                const Masks7& mm = op ? mb : ma;
                const uint32_t mask = prev_h1 < 0 ? mm.m[hd[0]] : (mm.m[hd[0]] ^ mm.m[prev_h1]);
                bool first = prev_h1 < 0;
                for (uint32_t q = 0; q < 4 && rc == kOk; ++q) {
                    if (!(mask >> q & 1)) continue;
                    for (uint64_t pr = 0; pr < P && rc == kOk; ++pr)
                        for (uint64_t pc = 0; pc < P && rc == kOk; ++pc) {
                            uint64_t* piece = dst + pr * ls * hw + pc * lw;  // piece of the child
                            const uint64_t gr = (q >> 1) * P + pr, gc = (q & 1) * P + pc;  // piece of A / Bt
                            if (op == 0) {
                                const uint64_t* src = A + gr * ls * w + gc * lw;
                                BMMGPU_CUDA_TRY(upload_piece(src, first ? piece : nullptr, hw));
                                if (!first) rc = bmmgpu_dev_fold(piece, hw, st.u(), lw, ls, lw, BMMGPU_GF2_XOR_AND, x);
                            } else {
                                // Bt piece (gr, gc) is B piece (gc, gr) transposed
                                const uint64_t* src = B + gc * ls * w + gr * lw;
                                BMMGPU_CUDA_TRY(upload_piece(src, nullptr, 0));
                                if (first)
                                    rc = launch_transpose_ld(st.u(), lw, ls, ls, piece, ls, lw, hw, x);
                                else if (!(rc = launch_transpose_ld(st.u(), lw, ls, ls, bt.u(), ls, lw, lw, x)))
                                    rc = bmmgpu_dev_fold(piece, hw, bt.u(), lw, ls, lw, BMMGPU_GF2_XOR_AND, x);
                            }
                            BMMGPU_CUDA_TRY(cudaEventRecord(up_free, x));
                        }
                    first = false;
                }
            }
            if (rc) break;
        }
        // the sub-instance's operands from the children: levels 2 .. dh as device gathers
        if (i >= 2) BMMGPU_CUDA_TRY(cudaStreamWaitEvent(x, consumed[slot], 0));
        const BlockList la = block_list(dh - 1, half, hw, [&](int l, uint32_t q) { return (ma.m[hd[l + 1]] >> q) & 1; });
        const BlockList lb = block_list(dh - 1, half, hw, [&](int l, uint32_t q) { return (mb.m[hd[l + 1]] >> q) & 1; });
        if ((rc = launch_block_list(false, TA.u(), hw, T[slot].u(), lw, ls, la, x)) ||
            (rc = launch_block_list(false, SB.u(), hw, S[slot].u(), lw, ls, lb, x)))
            break;
        BMMGPU_CUDA_TRY(cudaEventRecord(formed[slot], x));
        if (i % per_top == per_top - 1) BMMGPU_CUDA_TRY(cudaEventRecord(top_free, x));
        // Q_h on the compute stream (its Q slot free once the download two back is done)
        if (i >= 2) BMMGPU_CUDA_TRY(cudaStreamWaitEvent(s, hdown[(i - 2) % kQSlots], 0));
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(s, formed[slot], 0));
        if (trace) BMMGPU_CUDA_TRY(cudaEventRecord(tr_ev[2 * i], s));
        if ((rc = alt_multiply_device(T[slot].u(), lw, S[slot].u(), lw, Q[slot].u(), lw, ls, algo, e_sub, e_serial,
                                      kernel, s)))
            break;
        if (trace) BMMGPU_CUDA_TRY(cudaEventRecord(tr_ev[2 * i + 1], s));
        BMMGPU_CUDA_TRY(cudaEventRecord(consumed[slot], s));
        // download into the slot's page-locked buffer once the host fold two back released it
        {
            const auto w0 = std::chrono::steady_clock::now();
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return folded + kQSlots > i || fold_status != kOk; });
            main_wait_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
            if (fold_status != kOk) {
                rc = fold_status;
                break;
            }
        }
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(d, consumed[slot], 0));
        BMMGPU_CUDA_TRY(memcpy_counted(qh[i % kQSlots], Q[slot].p, blk, cudaMemcpyDeviceToHost, d));
        BMMGPU_CUDA_TRY(cudaEventRecord(hdown[i % kQSlots], d));
        {
            std::lock_guard<std::mutex> lk(mu);
            queued = i + 1;
        }
        cv.notify_all();
    }
    stop_folder(rc);
    if (rc) return rc;
    if (fold_status != kOk) {
        set_error("out-of-core sub-instances: a download failed");
        return fold_status;
    }
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[15], s));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
    // every C sub-block receives a contribution from some sub-instance; zero any that did not
    for (size_t id = 0; id < touched.size(); ++id)
        if (!touched[id]) {
            const uint64_t br = id >> dh, bc = id & ((uint64_t(1) << dh) - 1);
            for (uint64_t r = 0; r < ls; ++r) std::memset(C + (br * ls + r) * w + bc * lw, 0, lw * 8);
        }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev.e[14], ev.e[15]);
    if (trace) {
        double busy = 0, gap_top = 0, gap_other = 0;
        float prev_end = 0.f;
        for (uint64_t i = 0; i < subs; ++i) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, ev.e[14], tr_ev[2 * i]);
            cudaEventElapsedTime(&b, ev.e[14], tr_ev[2 * i + 1]);
            busy += (b - a) / 1e3;
            (i % per_top == 0 ? gap_top : gap_other) += (a - prev_end) / 1e3;
            prev_end = b;
        }
        fprintf(stderr, "subinst compute %.3f s, waits before top-level children %.3f s, other waits %.3f s, tail %.3f s\n",
                busy, gap_top, gap_other, ms / 1e3 - prev_end / 1e3);
    }
    if (trace)
        fprintf(stderr, "subinst n=%llu dh=%d e_sub=%d e_serial=%d: wall %.3f s, device %.3f s, fold busy %.3f s, "
                        "enqueue waited on the fold %.3f s\n",
                (unsigned long long)n, dh, e_sub, e_serial,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count(), ms / 1e3,
                fold_busy_s, main_wait_s);
    if (timing_ms) *timing_ms = ms;
    return kOk;
}

// ------------------------------------------------ interleaved basis change (K4)

namespace {

// [outer][4][inner] in place, one thread per (o, t) (reference yates.cpp:143-172).
__global__ void mode_step_in_place_kernel(uint64_t* __restrict__ v, uint64_t outer, uint64_t inner, Steps steps) {
    const uint64_t total = outer * inner;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t o = idx / inner, t = idx % inner;
        uint64_t* g = v + o * 4 * inner + t;
        uint64_t x[4] = {g[0], g[inner], g[2 * inner], g[3 * inner]};
        for (int i = 0; i < steps.n; ++i) x[steps.t[i]] ^= x[steps.s[i]];
#pragma unroll
        for (int q = 0; q < 4; ++q) g[q * inner] = x[q];
    }
}

}  // namespace

Steps basis_steps(const Scheme* sc, int factor, int inverse) {
    const InPlaceStep* st = factor == 0 ? sc->phi : factor == 1 ? sc->psi : sc->chi;
    const int n = factor == 0 ? sc->n_phi : factor == 1 ? sc->n_psi : sc->n_chi;
    Steps s{};
    s.n = n;
    for (int i = 0; i < n; ++i) {
        // the inverse of a sequence of x[t] ^= x[s] is the reversed sequence
        const InPlaceStep& p = inverse ? st[n - 1 - i] : st[i];
        s.t[i] = p.target;
        s.s[i] = p.source;
    }
    return s;
}

// One level of a basis change on [outer][4][inner] words on the device.
int interleaved_basis_change_level_dev(uint64_t* d, uint64_t outer, uint64_t inner, int algo, int factor, int inverse,
                                       cudaStream_t stream) {
    const Scheme* sc = scheme_for(algo);
    if (!sc || factor < 0 || factor > 2) {
        set_error("basis change: unknown scheme or factor");
        return kEinval;
    }
    const Steps s = basis_steps(sc, factor, inverse);
    if (s.n == 0 || outer * inner == 0) return kOk;
    mode_step_in_place_kernel<<<grid_for(outer * inner), 256, 0, stream>>>(d, outer, inner, s);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

// In-place basis change of an interleaved vector already on the device: factor 0 phi,
// 1 psi, 2 chi of the scheme; one pass per level (reference yates.cpp:143-172).
int interleaved_basis_change_dev(uint64_t* d, uint64_t total_words, int levels, int algo, int factor, int inverse,
                                 cudaStream_t stream) {
    const Scheme* sc = scheme_for(algo);
    if (!sc || factor < 0 || factor > 2 || levels < 0) {
        set_error("basis change: unknown scheme or factor");
        return kEinval;
    }
    const InPlaceStep* st = factor == 0 ? sc->phi : factor == 1 ? sc->psi : sc->chi;
    const int n = factor == 0 ? sc->n_phi : factor == 1 ? sc->n_psi : sc->n_chi;
    if (n == 0 || levels == 0 || total_words == 0) return kOk;
    Steps s{};
    s.n = n;
    for (int i = 0; i < n; ++i) {
        // the inverse of a sequence of x[t] ^= x[s] is the reversed sequence
        const InPlaceStep& p = inverse ? st[n - 1 - i] : st[i];
        s.t[i] = p.target;
        s.s[i] = p.source;
    }
    uint64_t outer = 1;
    for (int l = 0; l < levels; ++l) {
        const uint64_t inner = total_words / (outer * 4);
        mode_step_in_place_kernel<<<grid_for(outer * inner), 256, 0, stream>>>(d, outer, inner, s);
        count_launch();
        BMMGPU_CUDA_TRY(cudaGetLastError());
        outer *= 4;
    }
    return kOk;
}

// Host-vector basis change (bmm::basis_change, reference engine.cpp:146-172; the
// standalone `transform` of bmm_cli.cpp:210-234).  Vectors that fit the device budget
// go up once, get every level, come back.  Larger ones (a 2^20 operand is 128 GiB)
// stream: level l pairs words 4 inner_l apart (inner_l = total / 4^(l+1)), so the
// levels whose 4-way groups span at most a device block are applied together to
// contiguous blocks in one pass, and each level with wider groups takes its own pass
// that gathers the four strided pieces of a chunk of positions (one upload and one
// download of the vector per pass).
int interleaved_basis_change(uint64_t* words, uint64_t total_words, int levels, int algo, int factor, int inverse) {
    int rc;
    if (levels == 0 || total_words == 0) return kOk;
    uint64_t budget = free_budget();
    if (const char* b = getenv("BMMGPU_BASIS_BUDGET")) budget = strtoull(b, nullptr, 10);
    if (total_words * 8 <= budget) {
        DevMem d;
        if ((rc = d.alloc(total_words * 8, nullptr))) return rc;
        BMMGPU_CUDA_TRY(memcpy_counted(d.p, words, total_words * 8, cudaMemcpyHostToDevice, nullptr));
        if ((rc = interleaved_basis_change_dev(d.u(), total_words, levels, algo, factor, inverse, nullptr))) return rc;
        BMMGPU_CUDA_TRY(memcpy_counted(words, d.p, total_words * 8, cudaMemcpyDeviceToHost, nullptr));
        BMMGPU_CUDA_TRY(cudaStreamSynchronize(nullptr));
        return kOk;
    }
    if (total_words % (uint64_t(1) << (2 * levels))) {
        set_error("basis change: the vector has fewer than 4^levels words");
        return kEinval;
    }
    // device block: a power of two of words within the budget
    uint64_t bw = 1;
    while (bw * 2 * 8 <= budget && bw * 2 <= total_words) bw *= 2;
    if (bw < 4) {
        set_error("basis change: device budget below one 4-way group");
        return kEinval;
    }
    auto inner_of = [&](int l) { return total_words >> (2 * (l + 1)); };
    int l0 = 0;  // first level whose groups (4 inner_l words) fit a block
    while (l0 < levels && 4 * inner_of(l0) > bw) ++l0;
    DevMem d;
    if ((rc = d.alloc(bw * 8, nullptr))) return rc;
    // strided levels, one pass each: chunks of c positions, pieces q at q * inner
    for (int l = 0; l < l0; ++l) {
        const uint64_t inner = inner_of(l), outer = total_words / (4 * inner), c = bw / 4;
        for (uint64_t o = 0; o < outer; ++o)
            for (uint64_t t0 = 0; t0 < inner; t0 += c) {
                const uint64_t cl = std::min(c, inner - t0);
                uint64_t* base = words + o * 4 * inner + t0;
                BMMGPU_CUDA_TRY(memcpy2d_counted(d.p, cl * 8, base, inner * 8, cl * 8, 4, cudaMemcpyHostToDevice,
                                                 nullptr));
                if ((rc = interleaved_basis_change_dev(d.u(), 4 * cl, 1, algo, factor, inverse, nullptr))) return rc;
                BMMGPU_CUDA_TRY(memcpy2d_counted(base, inner * 8, d.p, cl * 8, cl * 8, 4, cudaMemcpyDeviceToHost,
                                                 nullptr));
            }
    }
    // the remaining levels together, block by block: within a block of bw words the
    // level-l groups are [bw / (4 inner_l)][4][inner_l], i.e. levels l0.. of a vector
    // of bw words whose outermost mode starts at l0
    // Blocks are whole level-l0 groups (4 inner_l0 words; every deeper level's group divides
    // it), so vectors whose inner mode is not a power of two ([4]*levels [7 * 64], say) split
    // cleanly and the last block may be shorter.
    if (l0 < levels) {
        const uint64_t g0 = 4 * inner_of(l0), blk = (bw / g0) * g0;
        for (uint64_t b0 = 0; b0 < total_words; b0 += blk) {
            const uint64_t len = std::min(blk, total_words - b0);
            BMMGPU_CUDA_TRY(memcpy_counted(d.p, words + b0, len * 8, cudaMemcpyHostToDevice, nullptr));
            for (int l = l0; l < levels; ++l) {
                const uint64_t inner = inner_of(l), outer_b = len / (4 * inner);
                if ((rc = interleaved_basis_change_level_dev(d.u(), outer_b, inner, algo, factor, inverse, nullptr)))
                    return rc;
            }
            BMMGPU_CUDA_TRY(memcpy_counted(words + b0, d.p, len * 8, cudaMemcpyDeviceToHost, nullptr));
        }
    }
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(nullptr));
    return kOk;
}

namespace {

// Interleave bit spread: bit i of x -> bit 2i.
__device__ __forceinline__ uint64_t spread_bits(uint64_t x) {
    x &= 0xFFFFFFFFull;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}

// Block permutation between the interleaved vector (64-word blocks in Morton order:
// level-l row digit at bit 2l+1, column digit at bit 2l, reference bitmatrix.cpp
// interleaved_bit_index / to_interleaved / from_interleaved 112-173) and a row-major
// matrix of nb x nb blocks (row stride ld words).  One thread per (block row, row,
// block column) word, block column fastest: the row-major side is coalesced.
//   swap = 0: row-major block (bi, bj) <-> vector block morton(bi, bj)  (left operand, result)
//   swap = 1: row-major block (bi, bj) <-> vector block morton(bj, bi)  (right operand
//             straight into Bt: Bt block (p, q) = B block (q, p) transposed = the stored
//             block, since the vector holds right-operand blocks transposed)
__global__ void block_permute_kernel(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, uint64_t nb,
                                     uint64_t ld, int to_rowmajor, int swap) {
    const uint64_t total = nb * 64 * nb;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t bj = idx % nb;
        const uint64_t R = idx / nb;  // row of the row-major matrix
        const uint64_t bi = R >> 6, r = R & 63;
        const uint64_t mb = swap ? (spread_bits(bj) << 1) | spread_bits(bi) : (spread_bits(bi) << 1) | spread_bits(bj);
        const uint64_t vi = mb * 64 + r, mi = R * ld + bj;
        if (to_rowmajor)
            dst[mi] = src[vi];
        else
            dst[vi] = src[mi];
    }
}

int launch_block_permute(const uint64_t* src, uint64_t* dst, uint64_t nb, uint64_t ld, bool to_rowmajor, bool swap,
                         cudaStream_t s) {
    const uint64_t total = nb * 64 * nb;
    block_permute_kernel<<<grid_for(total), 256, 0, s>>>(src, dst, nb, ld, to_rowmajor ? 1 : 0, swap ? 1 : 0);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

}  // namespace

// bmm::multiply_alt on interleaved host vectors, entirely on one device
// (reference engine.cpp:293-349): c_hat = chi^-1( phi^-1 a_hat . psi^-1 b_hat ).
// Upload, inverse basis changes (K4), Morton -> row-major / Bt block permutes, the
// fast product (folded coefficients), permute back, inverse chi, download.
int multiply_alt_interleaved(const uint64_t* a_hat, const uint64_t* b_hat, uint64_t* c_hat, int depth, int algo,
                             int kernel, int leaf_log2, int device, double* timing_ms) {
    BMMGPU_CUDA_TRY(cudaSetDevice(device));
    const uint64_t n = 64ull << depth, w = n / 64, nb = n / 64, total = n * w;
    kernel = resolve_kernel(kernel);
    uint64_t gm, gn, gk;
    int st;
    if ((st = granularity(kernel, &gm, &gn, &gk))) return st;
    const int e = alt_levels(n, leaf_log2);
    const uint64_t rows_pad = round_up(n, std::max(gm, gn)), kw = round_up(w, gk / 64), cw = rows_pad / 64;
    StreamSet ss;
    if (int r = ss.acquire(1)) return r;
    const cudaStream_t s = ss[0];
    DevMem dV, dA, dBt, dC;
    if ((st = dV.alloc(total * 8, s)) || (st = dA.alloc(rows_pad * kw * 8, s)) ||
        (st = dBt.alloc(round_up(rows_pad, 256) * kw * 8, s)) || (st = dC.alloc(rows_pad * cw * 8, s)))
        return st;
    BMMGPU_CUDA_TRY(cudaMemsetAsync(dA.p, 0, rows_pad * kw * 8, s));
    BMMGPU_CUDA_TRY(cudaMemsetAsync(dBt.p, 0, round_up(rows_pad, 256) * kw * 8, s));
    count_launch(2);
    cudaEvent_t e0, e1;
    BMMGPU_CUDA_TRY(cudaEventCreate(&e0));
    BMMGPU_CUDA_TRY(cudaEventCreate(&e1));
    struct TE {
        cudaEvent_t a, b;
        ~TE() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } te{e0, e1};
    BMMGPU_CUDA_TRY(cudaEventRecord(e0, s));
    BMMGPU_CUDA_TRY(memcpy_counted(dV.p, a_hat, total * 8, cudaMemcpyHostToDevice, s));
    if ((st = interleaved_basis_change_dev(dV.u(), total, depth, algo, 0, 1, s)) ||
        (st = launch_block_permute(dV.u(), dA.u(), nb, kw, true, false, s)))
        return st;
    BMMGPU_CUDA_TRY(memcpy_counted(dV.p, b_hat, total * 8, cudaMemcpyHostToDevice, s));
    float ms_a = 0.f;
    if ((st = interleaved_basis_change_dev(dV.u(), total, depth, algo, 1, 1, s)) ||
        (st = launch_block_permute(dV.u(), dBt.u(), nb, kw, true, true, s)))
        return st;
    if (e == 0)
        st = launch_cubic(kernel, dA.u(), kw, dBt.u(), kw, dC.u(), cw, rows_pad, rows_pad, kw, true, false, s, 1, 0, 0,
                          0);
    else
        st = alt_multiply_device(dA.u(), kw, dBt.u(), kw, dC.u(), cw, n, algo, e, choose_serial_levels(n, e), kernel,
                                 s);
    if (st) return st;
    if ((st = launch_block_permute(dC.u(), dV.u(), nb, cw, false, false, s)) ||
        (st = interleaved_basis_change_dev(dV.u(), total, depth, algo, 2, 1, s)))
        return st;
    BMMGPU_CUDA_TRY(memcpy_counted(c_hat, dV.p, total * 8, cudaMemcpyDeviceToHost, s));
    BMMGPU_CUDA_TRY(cudaEventRecord(e1, s));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
    cudaEventElapsedTime(&ms_a, e0, e1);
    if (timing_ms) *timing_ms = ms_a;
    return kOk;
}

}  // namespace bmmgpu

extern "C" int bmmgpu_dev_multiply(uint64_t* dA, uint64_t lda, uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                                   uint64_t ldc, uint64_t n, int32_t algo, int32_t leaf_log2, int32_t kernel,
                                   void* stream) {
    return bmmgpu::dev_multiply(dA, lda, dBt, ldbt, dC, ldc, n, algo, leaf_log2, kernel,
                                static_cast<cudaStream_t>(stream));
}

extern "C" int bmmgpu_dev_multiply_partial(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt,
                                           uint64_t* dC, uint64_t ldc, uint64_t n, int32_t algo, int32_t host_levels,
                                           uint32_t first, uint32_t stride, int32_t leaf_log2, int32_t kernel,
                                           void* stream) {
    return bmmgpu::dev_multiply_partial(dA, lda, dBt, ldbt, dC, ldc, n, algo, host_levels, first, stride, leaf_log2,
                                        kernel, static_cast<cudaStream_t>(stream));
}

extern "C" int bmmgpu_host_levels(uint64_t n, uint32_t parts, int32_t leaf_log2) {
    const int e = bmmgpu::alt_levels(n, leaf_log2);
    return std::max(0, std::min({bmmgpu::host_levels_for(n, parts, e), 4, e - 1}));
}

extern "C" int bmmgpu_multiply_alt(const uint64_t* a_hat, const uint64_t* b_hat, uint64_t* c_hat, int32_t depth,
                                   int32_t algo, const bmmgpu_opts* opts) {
    bmmgpu::reset_call_stats();
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        bmmgpu::set_error("no CUDA device available; the bit-matrix engine has no CPU fallback");
        return bmmgpu::kEnodev;
    }
    if (!bmmgpu::scheme_for(algo)) {
        bmmgpu::set_error("no bilinear scheme for this algorithm");
        return bmmgpu::kEinval;
    }
    if (depth < 0 || depth > 16) {
        bmmgpu::set_error("multiply_alt: depth out of range");
        return bmmgpu::kEinval;
    }
    int device = 0;
    const uint32_t mask = opts ? opts->device_mask : 0u;
    if (mask) device = __builtin_ctz(mask);
    if (device >= count) {
        bmmgpu::set_error("device_mask names a missing device");
        return bmmgpu::kEinval;
    }
    return bmmgpu::multiply_alt_interleaved(a_hat, b_hat, c_hat, depth, algo, opts ? opts->kernel : 0,
                                            opts ? opts->leaf_log2 : 0, device, opts ? opts->timing_ms : nullptr);
}

extern "C" int bmmgpu_basis_change(uint64_t* words, uint64_t total_words, int32_t levels, int32_t algo,
                                   int32_t factor, int32_t inverse) {
    bmmgpu::reset_call_stats();
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        bmmgpu::set_error("no CUDA device available; the bit-matrix engine has no CPU fallback");
        return bmmgpu::kEnodev;
    }
    return bmmgpu::interleaved_basis_change(words, total_words, levels, algo, factor, inverse);
}
