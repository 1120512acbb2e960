// cubic_lop3.cu -- K1: cubic bit-matrix product on the integer ALU.
//
// Replaces the reference's kernel64 + cubic_blocked (engine.cpp:34-100).  The
// reference computes each 64x64 output block as the XOR/OR fold over K-blocks
// of kernel64, where output bit (i,k) = parity/any of popcount(a[i] & bt[k]).
// Over the whole K range that is one reduction per output bit, so this kernel
// keeps the reduction in a 32-bit register per output bit and folds 32 bit
// products per instruction:
//     GF(2):   acc = (a & b) ^ acc      one LOP3 (immLut 0x6A), parity at the end
//     Boolean: acc = (a & b) | acc      one LOP3 (immLut 0xEA), nonzero at the end
// Roofline: the alu pipe issues 64 lanes/clk/SM, each LOP3 lane is 32 ANDs +
// 32 XOR/ORs, i.e. 4096 bop/clk/SM (measured 1.85e13 LOP3 lanes/s on B200 ->
// 1.19 Pbop/s).  Bits along K of A rows and Bt rows are operands; the 8x8
// register tile (8 rows x 8 columns per thread) gives 64 LOP3 per 16 operand
// words, so the SMEM crossbar runs at ~30% while the alu pipe is saturated.
//
// CTA tile 64 rows x 256 columns, K chunk 1024 bits, 3-stage cp.async ring.
// Warp w owns rows 8w..8w+7 (A reads are warp broadcasts); lane l owns
// columns l + 32q, q = 0..7 (B reads: 8 lanes x 16 B per wavefront, rows
// padded to 36 words so the 8 lanes hit distinct bank quads).
#include "common.cuh"

namespace bmmgpu {

namespace {

constexpr int L_BM = 64;
constexpr int L_BN = 256;
constexpr int L_KC = 32;             // 32-bit words per K chunk (1024 bits)
constexpr int L_STRIDE = L_KC + 4;   // padded smem row (words)
constexpr int L_STAGES = 3;
constexpr int L_THREADS = 256;
constexpr int L_STAGE_WORDS = (L_BM + L_BN) * L_STRIDE;
constexpr size_t L_SMEM = size_t(L_STAGES) * L_STAGE_WORDS * 4;

template <bool kGf2>
__device__ __forceinline__ uint32_t lop_fold(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    if (kGf2)
        asm("lop3.b32 %0, %1, %2, %3, 0x6A;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    else
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// A: m_pad x kw u64 words (stride lda u64); Bt: n_pad x kw (stride ldbt); C: m_pad x n_pad/64 (ldc).
template <bool kGf2>
__global__ void __launch_bounds__(L_THREADS, 1)
    cubic_lop3_kernel(const uint64_t* __restrict__ A, uint64_t lda, const uint64_t* __restrict__ Bt, uint64_t ldbt,
                      uint64_t* __restrict__ C, uint64_t ldc, uint64_t kw, int accumulate, uint32_t n_tiles,
                      uint32_t m_tiles, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch) {
    extern __shared__ __align__(16) uint32_t smem[];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // Grouped rasterisation: 8 row panels share a sweep over the column tiles
    // so the A panels stay L2-resident while B panels stream.
    const uint32_t group = 8;
    const uint32_t bid = blockIdx.x;
    // blockIdx.y selects one product of a batch (alt-basis leaves)
    A += blockIdx.y * sA_batch;
    Bt += blockIdx.y * sB_batch;
    C += blockIdx.y * sC_batch;
    const uint32_t per_group = group * n_tiles;
    const uint32_t g = bid / per_group;
    const uint32_t first_m = g * group;
    const uint32_t gsize = min(group, m_tiles - first_m);
    const uint32_t in_g = bid % per_group;
    const uint32_t tm = first_m + in_g % gsize;
    const uint32_t tn = in_g / gsize;

    const uint64_t row0 = uint64_t(tm) * L_BM;
    const uint64_t col0 = uint64_t(tn) * L_BN;
    const char* gA = reinterpret_cast<const char*>(A + row0 * lda);
    const char* gB = reinterpret_cast<const char*>(Bt + col0 * ldbt);
    const uint64_t lda_b = lda * 8, ldb_b = ldbt * 8;
    const uint64_t n_chunks = kw / (L_KC / 2);  // 16 u64 words per chunk

    auto load_stage = [&](uint64_t chunk, int stage) {
        uint32_t* sA = smem + stage * L_STAGE_WORDS;
        uint32_t* sB = sA + L_BM * L_STRIDE;
        const uint64_t koff = chunk * (L_KC * 4);  // bytes
        // 8 x 16 B per row; A: 64 rows -> 512 pieces, B: 256 rows -> 2048 pieces
#pragma unroll
        for (int it = 0; it < (L_BM * 8) / L_THREADS; ++it) {
            const unsigned p = tid + it * L_THREADS;
            const unsigned r = p >> 3, c = p & 7;
            cp_async16(sA + r * L_STRIDE + c * 4, gA + r * lda_b + koff + c * 16);
        }
#pragma unroll
        for (int it = 0; it < (L_BN * 8) / L_THREADS; ++it) {
            const unsigned p = tid + it * L_THREADS;
            const unsigned r = p >> 3, c = p & 7;
            cp_async16(sB + r * L_STRIDE + c * 4, gB + r * ldb_b + koff + c * 16);
        }
    };

    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0u;

#pragma unroll
    for (int s = 0; s < L_STAGES - 1; ++s) {
        if (s < n_chunks) load_stage(s, s);
        cp_async_commit();
    }

    for (uint64_t chunk = 0; chunk < n_chunks; ++chunk) {
        cp_async_wait<L_STAGES - 2>();
        __syncthreads();
        // prefetch chunk + STAGES - 1 into the slot freed last iteration
        {
            const uint64_t nxt = chunk + L_STAGES - 1;
            if (nxt < n_chunks) load_stage(nxt, int(nxt % L_STAGES));
            cp_async_commit();
        }
        const int stage = int(chunk % L_STAGES);
        const uint32_t* sA = smem + stage * L_STAGE_WORDS + (warp * 8) * L_STRIDE;
        const uint32_t* sB = smem + stage * L_STAGE_WORDS + L_BM * L_STRIDE + lane * L_STRIDE;
#pragma unroll 2
        for (int k4 = 0; k4 < L_KC / 4; ++k4) {
            uint4 a[8], b[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) a[r] = *reinterpret_cast<const uint4*>(sA + r * L_STRIDE + k4 * 4);
#pragma unroll
            for (int q = 0; q < 8; ++q) b[q] = *reinterpret_cast<const uint4*>(sB + q * 32 * L_STRIDE + k4 * 4);
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    acc[r][q] = lop_fold<kGf2>(a[r].x, b[q].x, acc[r][q]);
                    acc[r][q] = lop_fold<kGf2>(a[r].y, b[q].y, acc[r][q]);
                    acc[r][q] = lop_fold<kGf2>(a[r].z, b[q].z, acc[r][q]);
                    acc[r][q] = lop_fold<kGf2>(a[r].w, b[q].w, acc[r][q]);
                }
        }
    }
    cp_async_wait<0>();

    // Epilogue: output bit (row, col) -> ballot across lanes builds the 32-bit
    // word of columns col0 + 32q .. +31 for each of the warp's 8 rows.
    uint32_t keep0 = 0, keep1 = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const bool bit = kGf2 ? (__popc(acc[r][q]) & 1) : (acc[r][q] != 0u);
            const uint32_t word = __ballot_sync(0xffffffffu, bit);
            const int idx = r * 8 + q;
            if ((idx & 31) == int(lane)) {
                if (idx < 32)
                    keep0 = word;
                else
                    keep1 = word;
            }
        }
    uint32_t* C32 = reinterpret_cast<uint32_t*>(C);
    const uint64_t ldc32 = ldc * 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int idx = int(lane) + 32 * h;
        const int r = idx >> 3, q = idx & 7;
        const uint64_t row = row0 + warp * 8 + r;
        uint32_t* dst = C32 + row * ldc32 + col0 / 32 + q;
        uint32_t v = h ? keep1 : keep0;
        if (accumulate) v = kGf2 ? (v ^ *dst) : (v | *dst);
        *dst = v;
    }
}

}  // namespace

void lop3_granularity(uint64_t* gm, uint64_t* gn, uint64_t* gk_bits) {
    *gm = L_BM;
    *gn = L_BN;
    *gk_bits = L_KC * 32;
}

int launch_cubic_lop3(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                      uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate, cudaStream_t stream,
                      uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch) {
    if (m_pad % L_BM || n_pad % L_BN || (kw * 64) % (L_KC * 32)) {
        set_error("lop3 kernel: m_pad % 64, n_pad % 256 and K % 1024 bits must be 0");
        return kEinval;
    }
    if (m_pad == 0 || n_pad == 0) return kOk;
    if (kw == 0) {
        if (!accumulate) {
            for (uint64_t b = 0; b < batch; ++b) {
                BMMGPU_CUDA_TRY(cudaMemset2DAsync(dC + b * sC_batch, ldc * 8, 0, n_pad / 8, m_pad, stream));
                count_launch();
            }
        }
        return kOk;
    }
    auto kern = gf2 ? cubic_lop3_kernel<true> : cubic_lop3_kernel<false>;
    BMMGPU_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L_SMEM)));
    const uint64_t m_tiles = m_pad / L_BM, n_tiles = n_pad / L_BN;
    const uint64_t blocks = m_tiles * n_tiles;
    if (blocks > 0x7fffffffull || m_tiles > 0xffffffffull || batch > 65535) {
        set_error("lop3 kernel: grid too large");
        return kEinval;
    }
    if (batch == 0) return kOk;
    const dim3 grid{unsigned(blocks), unsigned(batch), 1u};
    kern<<<grid, L_THREADS, L_SMEM, stream>>>(dA, lda, dBt, ldbt, dC, ldc, kw, accumulate ? 1 : 0, uint32_t(n_tiles),
                                              uint32_t(m_tiles), sA_batch, sB_batch, sC_batch);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

}  // namespace bmmgpu
