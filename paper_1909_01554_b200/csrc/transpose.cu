// transpose.cu -- K3 layout kernel: row-major B (k x n bits) -> Bt (n_pad x kw
// words), i.e. column j of B becomes bit-row j of Bt, so the block-product
// kernels read both operands as rows along K.  This is the reference's
// "copy B and transpose_blocks64" step (engine.cpp:65-66, bitmatrix.cpp:97-110)
// fused with the block-position transpose the dot-product form needs.
//
// HBM-bound: 16 B read + 16 B written per 128 bits... per 64x64 block 512 B in,
// 512 B out.  A CTA stages a 256-row x 4-word tile through shared memory so
// both the loads and the stores move whole 32-byte sectors.
#include "common.cuh"

namespace bmmgpu {

namespace {

constexpr int TB_K = 4;  // 64-row blocks of B (K direction) per CTA
constexpr int TB_N = 4;  // 64-bit words of a B row (N direction) per CTA

__global__ void __launch_bounds__(128) transpose_kernel(const uint64_t* __restrict__ B, uint64_t ldb, uint64_t k,
                                                        uint64_t n, uint64_t* __restrict__ Bt, uint64_t kw) {
    __shared__ uint64_t tile[TB_N][TB_K][64];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t nb_words = (n + 63) / 64;
    const uint64_t bk = blockIdx.y * TB_K + warp;  // K block this warp loads
    const uint64_t bj0 = blockIdx.x * TB_N;        // first N word of the tile
    // Load rows bk*64 + lane (+32), words bj0..bj0+3, and transpose each block.
    uint64_t x0[TB_N], x1[TB_N];
#pragma unroll
    for (int b = 0; b < TB_N; ++b) {
        const uint64_t bj = bj0 + b;
        const uint64_t r0 = bk * 64 + lane, r1 = r0 + 32;
        uint64_t mask = ~0ull;
        if (bj == nb_words - 1 && (n & 63)) mask = (1ull << (n & 63)) - 1;
        x0[b] = (bj < nb_words && r0 < k) ? (B[r0 * ldb + bj] & mask) : 0ull;
        x1[b] = (bj < nb_words && r1 < k) ? (B[r1 * ldb + bj] & mask) : 0ull;
    }
#pragma unroll
    for (int b = 0; b < TB_N; ++b) {
        warp_transpose64(x0[b], x1[b], lane);
        tile[b][warp][lane] = x0[b];
        tile[b][warp][lane + 32] = x1[b];
    }
    __syncthreads();
    // Warp w now writes N block bj0 + w: rows (bj0+w)*64 + lane (+32), K words
    // blockIdx.y*4 .. +3 (32 contiguous bytes per row).
    const uint64_t row0 = (bj0 + warp) * 64 + lane;
    const uint64_t kw0 = blockIdx.y * TB_K;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint64_t row = row0 + 32 * h;
        uint64_t* dst = Bt + row * kw + kw0;
#pragma unroll
        for (int kb = 0; kb < TB_K; ++kb)
            if (kw0 + kb < kw) dst[kb] = tile[warp][kb][lane + 32 * h];
    }
}

}  // namespace

// n_pad must be a multiple of 256 (TB_N * 64).  Rows j >= n and K words past
// ceil(k/64) come out zero.
int launch_transpose(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                     uint64_t kw, cudaStream_t stream) {
    if (n_pad % (TB_N * 64) != 0 || n_pad < n || kw * 64 < k) {
        set_error("bmmgpu_dev_transpose: n_pad must be a multiple of 256 covering n, kw*64 must cover k");
        return kEinval;
    }
    if (n_pad == 0 || kw == 0) return kOk;
    dim3 grid(static_cast<unsigned>(n_pad / (TB_N * 64)), static_cast<unsigned>(ceil_div(kw, TB_K)));
    transpose_kernel<<<grid, 128, 0, stream>>>(dB, ldb, k, n, dBt, kw);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

}  // namespace bmmgpu
