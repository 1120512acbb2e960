// HISTORY ONLY -- superseded by csrc/cubic_umma2.cu (persistent CTA pairs); not built or linked.
// Kept for the round-1 A/B measurements in profiles/r01/history/.
// cubic_umma.cu -- K2 (single-CTA form, kernel id BMMGPU_KERNEL_UMMA_F4_1SM): the
// cubic bit-matrix product on the 5th-generation tensor cores (tcgen05.mma
// kind::mxf4, f32 accumulators in TMEM).  The CTA-pair form in
// cubic_umma2.cu is the default; this one stays as the simpler reference.
//
// Same contract as cubic_lop3.cu (reference kernel64 + cubic_blocked,
// engine.cpp:34-100): C bit (i,j) = parity (GF(2)) or any (Boolean) of the
// K-long AND of A row i and Bt row j.  Every bit is mapped to one fp4 (e2m1)
// element in {0, 1.0} or {0, 0.5}; the tensor core sums exact 0/1 products
// into an fp32 accumulator (exact: K <= 2^20 < 2^24), and the epilogue reads
// the integer count's parity or non-zeroness.
//
// Bit -> element expansion (per 32-bit word x of a row, y = x >> 2):
//     x & 0x22222222   bits = 1 mod 4, value 1.0   "even" class
//     y & 0x22222222   bits = 3 mod 4, value 1.0   "even" class
//     x & 0x11111111   bits = 0 mod 4, value 0.5   "odd"  class
//     y & 0x11111111   bits = 2 mod 4, value 0.5   "odd"  class
// Each nibble holds exactly one bit.  Both operands use the same map, so the
// K permutation cancels in the dot product.  Each 64-element MMA reads one
// class only, so its block scales are uniform: UE8M0 1.0 for even MMAs and
// 2.0 for odd ones (0.5*2 x 0.5*2 = 1); the scale factors are two constant
// TMEM regions written once.  5 ALU ops expand 32 bits.
//
// CTA: 128 x 256 output tile, one fp32 accumulator (256 TMEM columns).
// 8 producer warps stream packed bits from L2 (LDG.128, one row x 128 K-bits
// per item), expand them and store the nibbles into a 4-stage ring in the
// UMMA K-major no-swizzle layout (core matrix = 8 rows x 16 B; K-chunk
// stride padded by 16 B so the producers' STS.128 are bank-conflict free);
// one thread issues 4 MMAs (M128 N256 K64) per 256-bit stage and commits
// each stage back to the producers; producer warps 0-3 run the epilogue.
#include "umma.cuh"

namespace bmmgpu {

namespace {

constexpr int U_BM = 128;
constexpr int U_BN = 256;
constexpr int U_KBITS = 256;                     // K bits per stage (4 MMAs of K=64)
constexpr int U_STAGES = 4;
constexpr int U_CHUNKS = 8;                      // 16-byte K chunks per row per stage
constexpr int U_CSA = U_BM * 16 + 16;            // chunk stride, A (bytes)
constexpr int U_CSB = U_BN * 16 + 16;            // chunk stride, B (bytes)
constexpr int U_STAGE_A = U_CHUNKS * U_CSA;
constexpr int U_STAGE_B = U_CHUNKS * U_CSB;
constexpr int U_STAGE = U_STAGE_A + U_STAGE_B;
constexpr int U_PRODUCERS = 256;
constexpr int U_THREADS = U_PRODUCERS + 32;
constexpr size_t U_SMEM = size_t(U_STAGES) * U_STAGE;
constexpr uint32_t U_TMEM_COLS = 512;
constexpr uint32_t U_SF_EVEN = 256;  // TMEM column of the 1.0 scale region
constexpr uint32_t U_SF_ODD = 384;   // TMEM column of the 2.0 scale region

static_assert(U_SMEM <= 232448 - 1024, "stage ring exceeds shared memory");

__device__ __forceinline__ void expand_store(uint8_t* stage_base, int cs, int row, int g, const uint4& x) {
    constexpr uint32_t M2 = 0x22222222u, M1 = 0x11111111u;
    const uint4 y = make_uint4(x.x >> 2, x.y >> 2, x.z >> 2, x.w >> 2);
    uint8_t* p = stage_base + row * 16 + (4 * g) * cs;
    *reinterpret_cast<uint4*>(p) = make_uint4(x.x & M2, x.y & M2, x.z & M2, x.w & M2);
    *reinterpret_cast<uint4*>(p + cs) = make_uint4(y.x & M2, y.y & M2, y.z & M2, y.w & M2);
    *reinterpret_cast<uint4*>(p + 2 * cs) = make_uint4(x.x & M1, x.y & M1, x.z & M1, x.w & M1);
    *reinterpret_cast<uint4*>(p + 3 * cs) = make_uint4(y.x & M1, y.y & M1, y.z & M1, y.w & M1);
}

template <bool kGf2>
__global__ void __launch_bounds__(U_THREADS, 1)
    cubic_umma_kernel(const uint64_t* __restrict__ A, uint64_t lda, const uint64_t* __restrict__ Bt, uint64_t ldbt,
                      uint64_t* __restrict__ C, uint64_t ldc, uint64_t kw, int accumulate, uint32_t n_tiles,
                      uint32_t m_tiles, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full_bar[U_STAGES];
    __shared__ __align__(8) uint64_t empty_bar[U_STAGES];
    __shared__ __align__(8) uint64_t accum_bar;
    __shared__ uint32_t tmem_base_sh;

    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    A += blockIdx.y * sA_batch;
    Bt += blockIdx.y * sB_batch;
    C += blockIdx.y * sC_batch;

    // grouped rasterisation (8 row panels per sweep), as in the LOP3 kernel
    const uint32_t group = 8, bid = blockIdx.x;
    const uint32_t per_group = group * n_tiles;
    const uint32_t first_m = (bid / per_group) * group;
    const uint32_t gsize = min(group, m_tiles - first_m);
    const uint32_t in_g = bid % per_group;
    const uint64_t row0 = uint64_t(first_m + in_g % gsize) * U_BM;
    const uint64_t col0 = uint64_t(in_g / gsize) * U_BN;
    const uint64_t n_stages = kw / (U_KBITS / 64);

    if (warp == 8) umma::tmem_alloc(&tmem_base_sh, U_TMEM_COLS);
    if (tid == 0) {
        for (int s = 0; s < U_STAGES; ++s) {
            umma::mbar_init(&full_bar[s], U_PRODUCERS / 32);
            umma::mbar_init(&empty_bar[s], 1);
        }
        umma::mbar_init(&accum_bar, 1);
        umma::mbar_fence_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tmem_base_sh;

    if (warp < 4) {
        // constant block-scale regions: 1.0 (0x7F) for even MMAs, 2.0 (0x80) for odd ones
        const uint32_t lane_base = (warp * 32) << 16;
#pragma unroll
        for (int c = 0; c < 4; ++c) umma::tmem_st32_fill(tmem + lane_base + U_SF_EVEN + 32 * c, 0x7F7F7F7Fu);
#pragma unroll
        for (int c = 0; c < 4; ++c) umma::tmem_st32_fill(tmem + lane_base + U_SF_ODD + 32 * c, 0x80808080u);
        umma::tmem_st_wait();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();

    if (warp < 8) {
        // ------------------------------------------------ producers
        // item t: A row t/2, 128-bit group t%2; items t and t+256 of B likewise
        const int r_a = tid >> 1, g = tid & 1;
        const int r_b0 = tid >> 1, r_b1 = 128 + (tid >> 1);
        const uint4* pa = reinterpret_cast<const uint4*>(A + (row0 + r_a) * lda) + g;
        const uint4* pb0 = reinterpret_cast<const uint4*>(Bt + (col0 + r_b0) * ldbt) + g;
        const uint4* pb1 = reinterpret_cast<const uint4*>(Bt + (col0 + r_b1) * ldbt) + g;
        // each stage advances 256 bits = two uint4 per row
        uint4 xa = make_uint4(0, 0, 0, 0), xb0 = xa, xb1 = xa;
        if (n_stages > 0) {
            xa = __ldg(pa);
            xb0 = __ldg(pb0);
            xb1 = __ldg(pb1);
        }
        for (uint64_t it = 0; it < n_stages; ++it) {
            uint4 na = xa, nb0 = xb0, nb1 = xb1;
            if (it + 1 < n_stages) {
                na = __ldg(pa + 2 * (it + 1));
                nb0 = __ldg(pb0 + 2 * (it + 1));
                nb1 = __ldg(pb1 + 2 * (it + 1));
            }
            const int s = int(it % U_STAGES);
            if (it >= U_STAGES) umma::mbar_wait(&empty_bar[s], uint32_t(((it / U_STAGES) + 1) & 1));
            uint8_t* sa = smem + size_t(s) * U_STAGE;
            uint8_t* sb = sa + U_STAGE_A;
            expand_store(sa, U_CSA, r_a, g, xa);
            expand_store(sb, U_CSB, r_b0, g, xb0);
            expand_store(sb, U_CSB, r_b1, g, xb1);
            umma::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(&full_bar[s]);
            xa = na;
            xb0 = nb0;
            xb1 = nb1;
        }
    } else if (lane == 0) {
        // ------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = umma::idesc_mxf4(U_BM, U_BN);
        const uint32_t smem_base = smem_u32(smem);
        for (uint64_t it = 0; it < n_stages; ++it) {
            const int s = int(it % U_STAGES);
            umma::mbar_wait(&full_bar[s], uint32_t((it / U_STAGES) & 1));
            umma::fence_after_sync();
            const uint32_t a0 = smem_base + uint32_t(s) * U_STAGE;
            const uint32_t b0 = a0 + U_STAGE_A;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t da = umma::smem_desc(a0 + 2 * j * U_CSA, U_CSA, 128);
                const uint64_t db = umma::smem_desc(b0 + 2 * j * U_CSB, U_CSB, 128);
                const uint32_t sf = tmem + ((j & 1) ? U_SF_ODD : U_SF_EVEN);
                umma::mma_mxf4(tmem, da, db, idesc, sf, sf, (it | j) ? 1u : 0u);
            }
            umma::mma_commit(&empty_bar[s]);
        }
        umma::mma_commit(&accum_bar);
    }

    // ------------------------------------------------ epilogue (warps 0-3)
    if (warp < 4) {
        uint32_t words[8];
        if (n_stages > 0) {
            umma::mbar_wait(&accum_bar, 0);
            umma::fence_after_sync();
#pragma unroll 1
            for (int c = 0; c < 8; ++c) {
                uint32_t v[32];
                umma::tmem_ld32(tmem + ((warp * 32) << 16) + 32 * c, v);
                umma::tmem_ld_wait();
                uint32_t w = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    uint32_t bit;
                    if (kGf2)
                        bit = __float_as_uint(__uint_as_float(v[j]) + 8388608.0f) & 1u;
                    else
                        bit = v[j] != 0u;
                    w |= bit << j;
                }
                words[c] = w;
            }
        } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) words[c] = 0;
        }
        uint4* dst = reinterpret_cast<uint4*>(C + (row0 + warp * 32 + lane) * ldc + col0 / 64);
        uint4 w0 = make_uint4(words[0], words[1], words[2], words[3]);
        uint4 w1 = make_uint4(words[4], words[5], words[6], words[7]);
        if (accumulate) {
            const uint4 o0 = dst[0], o1 = dst[1];
            if (kGf2) {
                w0 = make_uint4(w0.x ^ o0.x, w0.y ^ o0.y, w0.z ^ o0.z, w0.w ^ o0.w);
                w1 = make_uint4(w1.x ^ o1.x, w1.y ^ o1.y, w1.z ^ o1.z, w1.w ^ o1.w);
            } else {
                w0 = make_uint4(w0.x | o0.x, w0.y | o0.y, w0.z | o0.z, w0.w | o0.w);
                w1 = make_uint4(w1.x | o1.x, w1.y | o1.y, w1.z | o1.z, w1.w | o1.w);
            }
        }
        dst[0] = w0;
        dst[1] = w1;
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 8) {
        umma::fence_after_sync();
        umma::tmem_dealloc(tmem, U_TMEM_COLS);
    }
}

}  // namespace

void umma1_granularity(uint64_t* gm, uint64_t* gn, uint64_t* gk_bits) {
    *gm = U_BM;
    *gn = U_BN;
    *gk_bits = U_KBITS;
}

int launch_cubic_umma1(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                      uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate, cudaStream_t stream,
                      uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch) {
    if (m_pad % U_BM || n_pad % U_BN || (kw * 64) % U_KBITS || lda % 2 || ldbt % 2 || ldc % 4) {
        set_error("umma kernel: m_pad % 128, n_pad % 256, K % 256 bits must be 0 and strides 16-byte aligned");
        return kEinval;
    }
    if (m_pad == 0 || n_pad == 0 || batch == 0) return kOk;
    if (kw * 64 > (1ull << 24)) {
        set_error("umma kernel: K above 2^24 bits would exceed exact fp32 accumulation");
        return kEinval;
    }
    auto kern = gf2 ? cubic_umma_kernel<true> : cubic_umma_kernel<false>;
    BMMGPU_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(U_SMEM)));
    const uint64_t m_tiles = m_pad / U_BM, n_tiles = n_pad / U_BN;
    const uint64_t blocks = m_tiles * n_tiles;
    if (blocks > 0x7fffffffull || batch > 65535) {
        set_error("umma kernel: grid too large");
        return kEinval;
    }
    const dim3 grid{unsigned(blocks), unsigned(batch), 1u};
    kern<<<grid, U_THREADS, U_SMEM, stream>>>(dA, lda, dBt, ldbt, dC, ldc, kw, accumulate ? 1 : 0, uint32_t(n_tiles),
                                              uint32_t(m_tiles), sA_batch, sB_batch, sC_batch);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

}  // namespace bmmgpu
