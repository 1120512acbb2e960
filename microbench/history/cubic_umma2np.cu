// HISTORY ONLY -- superseded by csrc/cubic_umma2.cu (persistent CTA pairs); not built or linked.
// Kept for the round-1 A/B measurements in profiles/r01/history/.
// cubic_umma2np.cu -- K2, CTA-pair form without the persistent tile loop
// (kernel id BMMGPU_KERNEL_UMMA_F4_PAIR_NP), kept for A/B measurement against
// the persistent default in cubic_umma2.cu.  The cubic bit-matrix product
// on CTA pairs of 5th-generation tensor cores (tcgen05.mma.cta_group::2
// kind::mxf4, M256 x N256 x K64 per instruction, f32 accumulators in TMEM).
//
// Contract and bit -> fp4 expansion exactly as cubic_umma.cu (reference
// kernel64 + cubic_blocked, engine.cpp:34-100): each bit becomes one e2m1
// element (x & 0x22222222 / (x>>2) & 0x22222222 -> 1.0, x & 0x11111111 /
// (x>>2) & 0x11111111 -> 0.5, uniform UE8M0 block scales 1.0 / 2.0 per MMA),
// exact 0/1 dot products accumulate in fp32, the epilogue takes the count's
// parity (GF(2)) or non-zeroness (Boolean).
//
// Why the pair: the 1-CTA form (cubic_umma.cu) is shared-memory bound --
// producers write the expanded operands with STS while the tensor core reads
// them back.  With cta_group::2 each SM holds 128 rows of A and 128 rows of
// Bt per 256 x 256 pair tile, so per MMA-cycle it stores and reads a third
// less than the 1-CTA M128 x N256 tile.  Operands are stored in the K-major
// 128-byte-swizzle layout (8-row x 128-byte atoms, chunk j of row r at
// j ^ (r & 7)): tensor-core reads stay 128-B aligned and the producers'
// STS.128 are conflict free.  Producers prefetch packed bits three stages
// ahead in registers to cover L2 latency.
//
// Roles per CTA (288 threads): warps 0-7 produce (LDG.128 -> expand ->
// STS.128, fence.proxy.async, arrive on the leader's full barrier, remotely
// from the peer CTA); warp 8 allocates TMEM for the pair and, in the leader
// CTA, one lane issues 4 MMAs per 256-bit stage and commits each stage to
// both CTAs' empty barriers (multicast); warps 0-3 of each CTA drain its
// 128 accumulator rows.
#include "umma.cuh"

namespace bmmgpu {

namespace {

constexpr int P_BM = 256;                 // pair tile rows (128 per CTA)
constexpr int P_BN = 256;                 // pair tile columns (Bt rows, 128 per CTA)
constexpr int P_KBITS = 256;              // K bits per stage (4 MMAs of K = 64)
constexpr int P_STAGES = 6;
constexpr int P_ROWS = 128;               // rows of A and of Bt held per CTA
constexpr int P_REGION = P_ROWS * 128;    // bytes of one operand per stage (16 KB)
constexpr int P_STAGE = 2 * P_REGION;
constexpr int P_PRODUCERS = 256;
constexpr int P_THREADS = P_PRODUCERS + 32;
constexpr size_t P_SMEM = size_t(P_STAGES) * P_STAGE + 1024;  // + alignment slack
constexpr uint32_t P_TMEM_COLS = 512;
constexpr uint32_t P_SF_EVEN = 256;
constexpr uint32_t P_SF_ODD = 384;
constexpr int P_PREFETCH = 3;

static_assert(P_SMEM <= 232448 - 1024, "stage ring exceeds shared memory");

// Row r of an operand region: 16-B chunk j lives at atom(r>>3)*1024 + (r&7)*128 + ((j ^ (r&7)) << 4).
__device__ __forceinline__ void expand_store_sw128(uint8_t* region, int r, int g, const uint4& x) {
    constexpr uint32_t M2 = 0x22222222u, M1 = 0x11111111u;
    const uint4 y = make_uint4(x.x >> 2, x.y >> 2, x.z >> 2, x.w >> 2);
    const int rr = r & 7;
    uint8_t* row = region + (r >> 3) * 1024 + rr * 128;
    const int j0 = 4 * g;
    *reinterpret_cast<uint4*>(row + (((j0 + 0) ^ rr) << 4)) = make_uint4(x.x & M2, x.y & M2, x.z & M2, x.w & M2);
    *reinterpret_cast<uint4*>(row + (((j0 + 1) ^ rr) << 4)) = make_uint4(y.x & M2, y.y & M2, y.z & M2, y.w & M2);
    *reinterpret_cast<uint4*>(row + (((j0 + 2) ^ rr) << 4)) = make_uint4(x.x & M1, x.y & M1, x.z & M1, x.w & M1);
    *reinterpret_cast<uint4*>(row + (((j0 + 3) ^ rr) << 4)) = make_uint4(y.x & M1, y.y & M1, y.z & M1, y.w & M1);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P_THREADS, 1)
    cubic_umma2np_kernel(const uint64_t* __restrict__ A, uint64_t lda, const uint64_t* __restrict__ Bt, uint64_t ldbt,
                       uint64_t* __restrict__ C, uint64_t ldc, uint64_t kw, int accumulate, uint32_t n_tiles,
                       uint32_t m_tiles, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch) {
    extern __shared__ uint8_t smem_raw[];
    // semiring as a runtime flag (bit 1 of `accumulate`): one compiled main loop for both
    const bool kGf2 = (accumulate & 2) != 0;
    __shared__ __align__(8) uint64_t full_bar[P_STAGES];
    __shared__ __align__(8) uint64_t empty_bar[P_STAGES];
    __shared__ __align__(8) uint64_t accum_bar;
    __shared__ uint32_t tmem_base_sh;

    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = umma::cluster_ctarank();
    A += blockIdx.y * sA_batch;
    Bt += blockIdx.y * sB_batch;
    C += blockIdx.y * sC_batch;

    // pair tile, grouped rasterisation over 8 row panels
    const uint32_t group = 8, pid = blockIdx.x >> 1;
    const uint32_t per_group = group * n_tiles;
    const uint32_t first_m = (pid / per_group) * group;
    const uint32_t gsize = min(group, m_tiles - first_m);
    const uint32_t in_g = pid % per_group;
    const uint64_t row0 = uint64_t(first_m + in_g % gsize) * P_BM + rank * P_ROWS;
    const uint64_t colp = uint64_t(in_g / gsize) * P_BN;  // first column of the pair tile
    const uint64_t bt0 = colp + rank * P_ROWS;            // this CTA's Bt rows
    const uint64_t n_stages = kw / (P_KBITS / 64);

    if (warp == 8) umma::tmem_alloc2(&tmem_base_sh, P_TMEM_COLS);
    if (tid == 0) {
        for (int s = 0; s < P_STAGES; ++s) {
            umma::mbar_init(&full_bar[s], 2 * (P_PRODUCERS / 32));
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
        const uint32_t lane_base = (warp * 32) << 16;
#pragma unroll
        for (int c = 0; c < 4; ++c) umma::tmem_st32_fill(tmem + lane_base + P_SF_EVEN + 32 * c, 0x7F7F7F7Fu);
#pragma unroll
        for (int c = 0; c < 4; ++c) umma::tmem_st32_fill(tmem + lane_base + P_SF_ODD + 32 * c, 0x80808080u);
        umma::tmem_st_wait();
    }
    umma::fence_before_sync();
    umma::cluster_sync();  // barriers of both CTAs initialised, TMEM of both allocated and scaled
    umma::fence_after_sync();

    if (warp < 8) {
        // ------------------------------------------------ producers
        const int r = tid >> 1, g = tid & 1;
        const uint4* pa = reinterpret_cast<const uint4*>(A + (row0 + r) * lda) + g;
        const uint4* pb = reinterpret_cast<const uint4*>(Bt + (bt0 + r) * ldbt) + g;
        const uint32_t full_leader0 = umma::mapa_shared(smem_u32(&full_bar[0]), 0);
        uint4 a0 = make_uint4(0, 0, 0, 0), b0 = a0, a1 = a0, b1 = a0, a2 = a0, b2 = a0;
        if (n_stages > 0) { a0 = __ldg(pa); b0 = __ldg(pb); }
        if (n_stages > 1) { a1 = __ldg(pa + 2); b1 = __ldg(pb + 2); }
        if (n_stages > 2) { a2 = __ldg(pa + 4); b2 = __ldg(pb + 4); }
        for (uint64_t it = 0; it < n_stages; ++it) {
            const int s = int(it % P_STAGES);
            if (it >= P_STAGES) umma::mbar_wait_cluster(&empty_bar[s], uint32_t(((it / P_STAGES) + 1) & 1));
            uint8_t* sa = smem + size_t(s) * P_STAGE;
            expand_store_sw128(sa, r, g, a0);
            expand_store_sw128(sa + P_REGION, r, g, b0);
            umma::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) umma::mbar_arrive_cluster(full_leader0 + s * 8);
            a0 = a1; b0 = b1;
            a1 = a2; b1 = b2;
            if (it + P_PREFETCH < n_stages) {
                a2 = __ldg(pa + 2 * (it + P_PREFETCH));
                b2 = __ldg(pb + 2 * (it + P_PREFETCH));
            }
        }
    } else if (rank == 0 && lane == 0) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        constexpr uint32_t idesc = umma::idesc_mxf4(P_BM, P_BN);
        const uint32_t base = smem_u32(smem);
        for (uint64_t it = 0; it < n_stages; ++it) {
            const int s = int(it % P_STAGES);
            umma::mbar_wait_cluster(&full_bar[s], uint32_t((it / P_STAGES) & 1));
            umma::fence_after_sync();
            const uint32_t a0 = base + uint32_t(s) * P_STAGE;
            const uint32_t b0 = a0 + P_REGION;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t da = umma::smem_desc_sw128(a0 + 32 * k, 1024);
                const uint64_t db = umma::smem_desc_sw128(b0 + 32 * k, 1024);
                const uint32_t sf = tmem + ((k & 1) ? P_SF_ODD : P_SF_EVEN);
                umma::mma_mxf4_pair(tmem, da, db, idesc, sf, sf, (it | k) ? 1u : 0u);
            }
            umma::mma_commit_pair(&empty_bar[s], 0x3);
        }
        umma::mma_commit_pair(&accum_bar, 0x3);
    }

    // ------------------------------------------------ epilogue (warps 0-3 of each CTA)
    if (warp < 4) {
        uint32_t words[8];
        if (n_stages > 0) {
            umma::mbar_wait_cluster(&accum_bar, 0);
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
        uint4* dst = reinterpret_cast<uint4*>(C + (row0 + warp * 32 + lane) * ldc + colp / 64);
        uint4 w0 = make_uint4(words[0], words[1], words[2], words[3]);
        uint4 w1 = make_uint4(words[4], words[5], words[6], words[7]);
        if (accumulate & 1) {
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
    umma::cluster_sync();  // all MMAs retired and all TMEM reads done in both CTAs
    if (warp == 8) {
        umma::fence_after_sync();
        umma::tmem_dealloc2(tmem, P_TMEM_COLS);
    }
}

}  // namespace

void umma2np_granularity(uint64_t* gm, uint64_t* gn, uint64_t* gk_bits) {
    *gm = P_BM;
    *gn = P_BN;
    *gk_bits = P_KBITS;
}

int launch_cubic_umma2np(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                      uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate, cudaStream_t stream,
                      uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch) {
    if (m_pad % P_BM || n_pad % P_BN || (kw * 64) % P_KBITS || lda % 2 || ldbt % 2 || ldc % 4) {
        set_error("umma2np kernel: m_pad % 256, n_pad % 256, K % 256 bits must be 0 and strides 16-byte aligned");
        return kEinval;
    }
    if (m_pad == 0 || n_pad == 0 || batch == 0) return kOk;
    if (kw * 64 > (1ull << 24)) {
        set_error("umma2np kernel: K above 2^24 bits would exceed exact fp32 accumulation");
        return kEinval;
    }
    auto kern = cubic_umma2np_kernel;
    BMMGPU_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P_SMEM)));
    const uint64_t m_tiles = m_pad / P_BM, n_tiles = n_pad / P_BN;
    const uint64_t blocks = 2 * m_tiles * n_tiles;
    if (blocks > 0x7fffffffull || batch > 65535) {
        set_error("umma2np kernel: grid too large");
        return kEinval;
    }
    const dim3 grid{unsigned(blocks), unsigned(batch), 1u};
    kern<<<grid, P_THREADS, P_SMEM, stream>>>(dA, lda, dBt, ldbt, dC, ldc, kw, (accumulate ? 1 : 0) | (gf2 ? 2 : 0), uint32_t(n_tiles),
                                              uint32_t(m_tiles), sA_batch, sB_batch, sC_batch);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

}  // namespace bmmgpu
