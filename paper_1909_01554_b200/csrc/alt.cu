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
#include <cstring>
#include <vector>

#include "../../include/bmmgpu.h"
#include "common.cuh"
#include "schemes.h"

namespace bmmgpu {

int launch_transpose(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                     uint64_t kw, cudaStream_t stream);
int launch_cubic(int kernel, const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                 uint64_t ldc, uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate,
                 cudaStream_t stream, uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch);
int granularity(int kernel, uint64_t* gm, uint64_t* gn, uint64_t* gk);
int resolve_kernel(int kernel);

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

// In-place basis change on every (sub_rows x sub_cols) submatrix of size L:
// quadrant q = 2*qi + qj at row offset qi*L/2, word offset qj*L/128; the
// program is a list of x[t] ^= x[s] (reference yates.cpp:143-172).
__global__ void basis_change_kernel(uint64_t* __restrict__ M, uint64_t ld, uint64_t sub, uint64_t L, Steps steps) {
    const uint64_t half = L / 2, hw = L / 128;
    const uint64_t per_sub = half * hw;
    const uint64_t total = sub * sub * per_sub;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = idx % hw;
        const uint64_t r = (idx / hw) % half;
        const uint64_t s = idx / per_sub;
        const uint64_t sr = s / sub, sc = s % sub;
        uint64_t* base = M + (sr * L + r) * ld + sc * (L / 64) + w;
        uint64_t* p[4] = {base, base + hw, base + half * ld, base + half * ld + hw};
        uint64_t x[4] = {*p[0], *p[1], *p[2], *p[3]};
        uint32_t dirty = 0;
        for (int i = 0; i < steps.n; ++i) {
            x[steps.t[i]] ^= x[steps.s[i]];
            dirty |= 1u << steps.t[i];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (dirty & (1u << q)) *p[q] = x[q];
    }
}

// Expand: P parents of size L (row stride ld_in, batch stride bs_in) -> 7P
// children of size L/2 (ld_out, bs_out), child h = XOR of the parent
// quadrants in mask m[h] (reference yates.cpp:112-141 with the alpha / beta
// programs; engine.cpp:284-285).
__global__ void expand_kernel(const uint64_t* __restrict__ in, uint64_t ld_in, uint64_t bs_in, uint64_t P, uint64_t L,
                              uint64_t* __restrict__ out, uint64_t ld_out, uint64_t bs_out, Masks7 masks) {
    const uint64_t half = L / 2, hw = L / 128;
    const uint64_t per_p = half * hw;
    const uint64_t total = P * per_p;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = idx % hw;
        const uint64_t r = (idx / hw) % half;
        const uint64_t p = idx / per_p;
        const uint64_t* base = in + p * bs_in + r * ld_in + w;
        const uint64_t x0 = base[0], x1 = base[hw], x2 = base[half * ld_in], x3 = base[half * ld_in + hw];
        uint64_t* dst = out + (p * 7) * bs_out + r * ld_out + w;
#pragma unroll
        for (int h = 0; h < 7; ++h) {
            const uint32_t m = masks.m[h];
            uint64_t v = 0;
            if (m & 1) v ^= x0;
            if (m & 2) v ^= x1;
            if (m & 4) v ^= x2;
            if (m & 8) v ^= x3;
            dst[h * bs_out] = v;
        }
    }
}

// Compress: 7P children of size L/2 -> P parents of size L, parent quadrant q
// = XOR of the children in mask m[q] (gamma; reference engine.cpp:288).
__global__ void compress_kernel(const uint64_t* __restrict__ in, uint64_t ld_in, uint64_t bs_in, uint64_t P,
                                uint64_t L, uint64_t* __restrict__ out, uint64_t ld_out, uint64_t bs_out,
                                Masks4 masks) {
    const uint64_t half = L / 2, hw = L / 128;
    const uint64_t per_p = half * hw;
    const uint64_t total = P * per_p;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = idx % hw;
        const uint64_t r = (idx / hw) % half;
        const uint64_t p = idx / per_p;
        const uint64_t* src = in + (p * 7) * bs_in + r * ld_in + w;
        uint64_t y[7];
#pragma unroll
        for (int h = 0; h < 7; ++h) y[h] = src[h * bs_in];
        uint64_t* dst = out + p * bs_out + r * ld_out + w;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t m = masks.m[q];
            uint64_t v = 0;
#pragma unroll
            for (int h = 0; h < 7; ++h)
                if (m & (1u << h)) v ^= y[h];
            dst[(q >> 1) * half * ld_out + (q & 1) * hw] = v;
        }
    }
}

unsigned grid_for(uint64_t total) {
    const uint64_t blocks = ceil_div(total, 256);
    return unsigned(std::min<uint64_t>(blocks, 148ull * 64));
}

// sigma: quadrant index of B (2j + k) <-> quadrant index of Bt (2k + j).
inline int sigma(int q) { return ((q & 1) << 1) | (q >> 1); }

Steps make_steps(const InPlaceStep* st, int n, bool transposed) {
    Steps s{};
    s.n = n;
    for (int i = 0; i < n; ++i) {
        s.t[i] = uint8_t(transposed ? sigma(st[i].target) : st[i].target);
        s.s[i] = uint8_t(transposed ? sigma(st[i].source) : st[i].source);
    }
    return s;
}

Masks7 make_expand(const char* const rows[7], bool transposed) {
    Masks7 m{};
    for (int h = 0; h < 7; ++h) {
        const uint32_t r = row_mask(rows[h]);
        uint32_t out = 0;
        for (int t = 0; t < 4; ++t)
            if (r & (1u << (transposed ? sigma(t) : t))) out |= 1u << t;
        m.m[h] = uint8_t(out);
    }
    return m;
}

int launch_basis_change(uint64_t* M, uint64_t ld, uint64_t n, int levels, const Steps& steps, cudaStream_t s) {
    if (steps.n == 0) return kOk;
    for (int l = 0; l < levels; ++l) {
        const uint64_t sub = 1ull << l, L = n >> l;
        const uint64_t total = sub * sub * (L / 2) * (L / 128);
        basis_change_kernel<<<grid_for(total), 256, 0, s>>>(M, ld, sub, L, steps);
        count_launch();
        BMMGPU_CUDA_TRY(cudaGetLastError());
    }
    return kOk;
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
    const Masks7 ma = make_expand(sc->alpha, false), mb = make_expand(sc->beta, true);
    Masks4 mg{};
    for (int q = 0; q < 4; ++q) mg.m[q] = uint8_t(row_mask(sc->gamma[q]));

    uint64_t gm, gn, gk;
    if ((st = granularity(kernel, &gm, &gn, &gk))) return st;
    const uint64_t L = n >> e;
    // Leaf panels padded to the kernel's tiles (pads stay zero).
    const uint64_t t_rows = round_up(L, gm), s_rows = round_up(L, gn);
    const uint64_t kwl = round_up(L / 64, gk / 64);
    const uint64_t cwl = s_rows / 64;
    uint64_t batch = 1;
    for (int l = 0; l < e; ++l) batch *= 7;

    // Level buffers: intermediate levels 1..e-1 are plain row-major (stride
    // L_l/64), level e uses the padded leaf panels.
    std::vector<DevMem> T(e + 1), S(e + 1);
    std::vector<uint64_t> t_ld(e + 1), s_ld(e + 1), t_bs(e + 1), s_bs(e + 1);
    uint64_t P = 1;
    for (int l = 1; l <= e; ++l) {
        P *= 7;
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

    // Expand level by level, freeing each parent level once consumed.
    const uint64_t* tin = dA;
    const uint64_t* sin = dBt;
    P = 1;
    for (int l = 0; l < e; ++l) {
        const uint64_t Ll = n >> l;
        const uint64_t Pn = P * 7;
        const size_t tb = size_t(Pn * t_bs[l + 1] * 8), sb = size_t(Pn * s_bs[l + 1] * 8);
        if ((st = T[l + 1].alloc(tb, s)) || (st = S[l + 1].alloc(sb, s))) return st;
        if (l + 1 == e && (t_rows != L || s_rows != L || kwl != L / 64)) {
            BMMGPU_CUDA_TRY(cudaMemsetAsync(T[l + 1].p, 0, tb, s));
            BMMGPU_CUDA_TRY(cudaMemsetAsync(S[l + 1].p, 0, sb, s));
            count_launch(2);
        }
        const uint64_t total = P * (Ll / 2) * (Ll / 128);
        expand_kernel<<<grid_for(total), 256, 0, s>>>(tin, t_ld[l], t_bs[l], P, Ll, T[l + 1].u(), t_ld[l + 1],
                                                      t_bs[l + 1], ma);
        expand_kernel<<<grid_for(total), 256, 0, s>>>(sin, s_ld[l], s_bs[l], P, Ll, S[l + 1].u(), s_ld[l + 1],
                                                      s_bs[l + 1], mb);
        count_launch(2);
        BMMGPU_CUDA_TRY(cudaGetLastError());
        if (l > 0) {
            // parents no longer needed (stream-ordered free: no host sync)
            T[l].release();
            S[l].release();
        }
        tin = T[l + 1].u();
        sin = S[l + 1].u();
        P = Pn;
    }

    // Leaves: 7^e batched block products, Q row-major (t_rows x cwl words each).
    DevMem Q;
    const uint64_t q_bs = t_rows * cwl;
    if ((st = Q.alloc(size_t(batch * q_bs * 8), s))) return st;
    for (uint64_t b0 = 0; b0 < batch; b0 += 65535) {
        const uint64_t nb = std::min<uint64_t>(65535, batch - b0);
        if ((st = launch_cubic(kernel, T[e].u() + b0 * t_bs[e], kwl, S[e].u() + b0 * s_bs[e], kwl,
                               Q.u() + b0 * q_bs, cwl, t_rows, s_rows, kwl, true, false, s, nb, t_bs[e], s_bs[e],
                               q_bs)))
            return st;
    }
    T[e].release();
    S[e].release();

    // Compress level by level back into dC.
    DevMem cur = std::move(Q), nxt;
    uint64_t cur_ld = cwl, cur_bs = q_bs;
    P = batch;
    for (int l = e - 1; l >= 0; --l) {
        const uint64_t Ll = n >> l;
        const uint64_t Pp = P / 7;
        uint64_t* out;
        uint64_t out_ld, out_bs;
        if (l == 0) {
            out = dC;
            out_ld = ldc;
            out_bs = 0;
        } else {
            out_ld = Ll / 64;
            out_bs = Ll * (Ll / 64);
            if ((st = nxt.alloc(size_t(Pp * out_bs * 8), s))) return st;
            out = nxt.u();
        }
        const uint64_t total = Pp * (Ll / 2) * (Ll / 128);
        compress_kernel<<<grid_for(total), 256, 0, s>>>(cur.u(), cur_ld, cur_bs, Pp, Ll, out, out_ld, out_bs, mg);
        count_launch();
        BMMGPU_CUDA_TRY(cudaGetLastError());
        cur = std::move(nxt);
        cur_ld = out_ld;
        cur_bs = out_bs;
        P = Pp;
    }
    return kOk;
}

namespace {

// child = XOR of the quadrants of an L x L matrix selected by a 4-bit mask
// (one alpha / beta row of a depth-first level, reference engine.cpp:284-285).
__global__ void select_kernel(const uint64_t* __restrict__ in, uint64_t ld_in, uint64_t L, uint64_t* __restrict__ out,
                              uint64_t ld_out, uint32_t mask) {
    const uint64_t half = L / 2, hw = L / 128, total = half * hw;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = idx % hw, r = idx / hw;
        const uint64_t* base = in + r * ld_in + w;
        uint64_t v = 0;
        if (mask & 1) v ^= base[0];
        if (mask & 2) v ^= base[hw];
        if (mask & 4) v ^= base[half * ld_in];
        if (mask & 8) v ^= base[half * ld_in + hw];
        out[r * ld_out + w] = v;
    }
}

// quadrant q of C ^= child for every q in mask (one gamma column, folded as
// each child product finishes; reference engine.cpp:288).
__global__ void scatter_xor_kernel(const uint64_t* __restrict__ q_in, uint64_t ld_q, uint64_t L, uint64_t* C,
                                   uint64_t ldc, uint32_t mask) {
    const uint64_t half = L / 2, hw = L / 128, total = half * hw;
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t w = idx % hw, r = idx / hw;
        const uint64_t v = q_in[r * ld_q + w];
        uint64_t* base = C + r * ldc + w;
        if (mask & 1) base[0] ^= v;
        if (mask & 2) base[hw] ^= v;
        if (mask & 4) base[half * ldc] ^= v;
        if (mask & 8) base[half * ldc + hw] ^= v;
    }
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
    const Masks7 ma = make_expand(sc->alpha, false), mb = make_expand(sc->beta, true);
    int st;
    BMMGPU_CUDA_TRY(cudaMemset2DAsync(dC, ldc * 8, 0, (n / 64) * 8, n, s));
    count_launch();
    DevMem T, S, Q;
    if ((st = T.alloc(half * hw * 8, s)) || (st = S.alloc(half * hw * 8, s)) || (st = Q.alloc(half * hw * 8, s)))
        return st;
    const uint64_t total = half * hw;
    for (int h = 0; h < 7; ++h) {
        select_kernel<<<grid_for(total), 256, 0, s>>>(dA, lda, n, T.u(), hw, ma.m[h]);
        select_kernel<<<grid_for(total), 256, 0, s>>>(dBt, ldbt, n, S.u(), hw, mb.m[h]);
        count_launch(2);
        BMMGPU_CUDA_TRY(cudaGetLastError());
        if ((st = alt_serial(T.u(), hw, S.u(), hw, Q.u(), hw, half, sc, e_serial - 1, e_par, kernel, s))) return st;
        uint32_t cmask = 0;
        for (int q = 0; q < 4; ++q)
            if (row_mask(sc->gamma[q]) & (1u << h)) cmask |= 1u << q;
        scatter_xor_kernel<<<grid_for(total), 256, 0, s>>>(Q.u(), hw, n, dC, ldc, cmask);
        count_launch();
        BMMGPU_CUDA_TRY(cudaGetLastError());
    }
    return kOk;
}

// Device-resident fast product: dA (n x n/64, stride lda), dBt (Bt of B, n x
// n/64, stride ldbt), dC (n x n/64, stride ldc).  dA and dBt are CLOBBERED
// (basis-changed in place).  e recursion levels (leaves of size n >> e), the
// top e_serial of them depth-first.
int alt_multiply_device(uint64_t* dA, uint64_t lda, uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                        uint64_t n, int algo, int e, int e_serial, int kernel, cudaStream_t s) {
    const Scheme* sc = scheme_for(algo);
    if (!sc) {
        set_error("no bilinear scheme for this algorithm");
        return kEinval;
    }
    int st;
    if (e < 1 || (n >> e) < 64 || e_serial < 0 || e_serial > e) {
        set_error("alt_multiply_device: need 1 <= e, 0 <= e_serial <= e and leaves of at least 64 bits");
        return kEinval;
    }
    // phi on A, psi on B (seen through Bt) over the top e levels (reference engine.cpp:371-374).
    if ((st = launch_basis_change(dA, lda, n, e, make_steps(sc->phi, sc->n_phi, false), s))) return st;
    if ((st = launch_basis_change(dBt, ldbt, n, e, make_steps(sc->psi, sc->n_psi, true), s))) return st;
    if ((st = alt_serial(dA, lda, dBt, ldbt, dC, ldc, n, sc, e_serial, e - e_serial, kernel, s))) return st;
    // chi on C over the top e levels (reference engine.cpp:379-380).
    return launch_basis_change(dC, ldc, n, e, make_steps(sc->chi, sc->n_chi, false), s);
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

uint64_t free_budget() {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return 0;
    return uint64_t(double(free_b) * 0.8);
}

// Depth-first level count for this device (BMMGPU_ALT_SERIAL forces it; tests use it).
int choose_serial_levels(uint64_t n, int e) {
    if (const char* env = getenv("BMMGPU_ALT_SERIAL")) return std::max(0, std::min(atoi(env), e - 1));
    return alt_serial_levels(n, e, free_budget());
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

// Host entry: reference-layout host buffers in, C out.
int alt_multiply_host(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int algo, const bmmgpu_plan* plan,
                      int kernel, int leaf_log2, double* timing_ms) {
    (void)plan;  // the plan's host/serial/parallel split is a CPU schedule; the GPU picks e from leaf_log2
    const int e = alt_levels(n, leaf_log2);
    kernel = resolve_kernel(kernel);
    const uint64_t w = n / 64;
    cudaStream_t s;
    BMMGPU_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct G {
        cudaStream_t s;
        ~G() { cudaStreamDestroy(s); }
    } guard{s};
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
    BMMGPU_CUDA_TRY(cudaMemcpy2DAsync(dA.p, kw * 8, A, w * 8, w * 8, n, cudaMemcpyHostToDevice, s));
    BMMGPU_CUDA_TRY(cudaMemcpyAsync(dB.p, B, n * w * 8, cudaMemcpyHostToDevice, s));
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
    BMMGPU_CUDA_TRY(cudaMemcpy2DAsync(C, w * 8, dC.p, cw * 8, w * 8, n, cudaMemcpyDeviceToHost, s));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (timing_ms) *timing_ms = ms;
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

int interleaved_basis_change(uint64_t* words, uint64_t total_words, int levels, int algo, int factor, int inverse) {
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
    DevMem d;
    int rc;
    if ((rc = d.alloc(total_words * 8, nullptr))) return rc;
    BMMGPU_CUDA_TRY(cudaMemcpy(d.p, words, total_words * 8, cudaMemcpyHostToDevice));
    uint64_t outer = 1;
    for (int l = 0; l < levels; ++l) {
        const uint64_t inner = total_words / (outer * 4);
        mode_step_in_place_kernel<<<grid_for(outer * inner), 256>>>(d.u(), outer, inner, s);
        count_launch();
        BMMGPU_CUDA_TRY(cudaGetLastError());
        outer *= 4;
    }
    BMMGPU_CUDA_TRY(cudaMemcpy(words, d.p, total_words * 8, cudaMemcpyDeviceToHost));
    return kOk;
}

}  // namespace bmmgpu

extern "C" int bmmgpu_dev_multiply(uint64_t* dA, uint64_t lda, uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                                   uint64_t ldc, uint64_t n, int32_t algo, int32_t leaf_log2, int32_t kernel,
                                   void* stream) {
    return bmmgpu::dev_multiply(dA, lda, dBt, ldbt, dC, ldc, n, algo, leaf_log2, kernel,
                                static_cast<cudaStream_t>(stream));
}

extern "C" int bmmgpu_basis_change(uint64_t* words, uint64_t total_words, int32_t levels, int32_t algo,
                                   int32_t factor, int32_t inverse) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        bmmgpu::set_error("no CUDA device available; the bit-matrix engine has no CPU fallback");
        return bmmgpu::kEnodev;
    }
    return bmmgpu::interleaved_basis_change(words, total_words, levels, algo, factor, inverse);
}
