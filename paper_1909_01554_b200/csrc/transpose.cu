// transpose.cu -- K3 layout kernel: row-major B (k x n bits) -> Bt (n_pad x kw
// words), i.e. column j of B becomes bit-row j of Bt, so the block-product
// kernels read both operands as rows along K.  This is the reference's
// "copy B and transpose_blocks64" step (engine.cpp:65-66, bitmatrix.cpp:97-110)
// fused with the block-position transpose the dot-product form needs.
//
// HBM-bound: per 64x64 block 512 B in, 512 B out.  A CTA of 8 warps stages an
// 8 x 8 grid of blocks (512 K rows x 8 words of B) through shared memory: warp w
// loads K block w of the tile (64 B per row, 16-byte loads) and transposes each of
// its 8 blocks with shuffles, then writes N block w of the tile as 64 contiguous
// bytes per Bt row (16-byte stores).
#include <cstdlib>

#include "common.cuh"

namespace bmmgpu {

namespace {

constexpr int TB = 8;  // blocks per tile side: 8 K blocks (512 rows) x 8 words (512 columns)

__global__ void __launch_bounds__(256) transpose_kernel(const uint64_t* __restrict__ B, uint64_t ldb, uint64_t k,
                                                        uint64_t n, uint64_t* __restrict__ Bt, uint64_t n_pad,
                                                        uint64_t kw, uint64_t ldbt) {
    __shared__ uint64_t tile[TB][TB][64];  // [N block][K block][row of the transposed block]
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t nb_words = (n + 63) / 64;
    const uint64_t bk = blockIdx.y * uint64_t(TB) + warp;  // K block this warp loads
    const uint64_t bj0 = blockIdx.x * uint64_t(TB);        // first N word of the tile
    const uint64_t r0 = bk * 64 + lane, r1 = r0 + 32;
    uint64_t x0[TB], x1[TB];
    const bool fast = (ldb % 2 == 0) && bj0 + TB <= nb_words && r1 < k && (n & 63) == 0;
    if (fast) {
        const ulonglong2* p0 = reinterpret_cast<const ulonglong2*>(B + r0 * ldb + bj0);
        const ulonglong2* p1 = reinterpret_cast<const ulonglong2*>(B + r1 * ldb + bj0);
#pragma unroll
        for (int b = 0; b < TB / 2; ++b) {
            const ulonglong2 u = p0[b], v = p1[b];
            x0[2 * b] = u.x;
            x0[2 * b + 1] = u.y;
            x1[2 * b] = v.x;
            x1[2 * b + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int b = 0; b < TB; ++b) {
            const uint64_t bj = bj0 + b;
            uint64_t mask = ~0ull;
            if (bj == nb_words - 1 && (n & 63)) mask = (1ull << (n & 63)) - 1;
            x0[b] = (bj < nb_words && r0 < k) ? (B[r0 * ldb + bj] & mask) : 0ull;
            x1[b] = (bj < nb_words && r1 < k) ? (B[r1 * ldb + bj] & mask) : 0ull;
        }
    }
#pragma unroll
    for (int b = 0; b < TB; ++b) {
        warp_transpose64(x0[b], x1[b], lane);
        tile[b][warp][lane] = x0[b];
        tile[b][warp][lane + 32] = x1[b];
    }
    __syncthreads();
    // Warp w writes N block bj0 + w: rows (bj0+w)*64 + lane (+32), K words
    // blockIdx.y*8 .. +7 (64 contiguous bytes per row).
    const uint64_t kw0 = blockIdx.y * uint64_t(TB);
    const bool vec = (ldbt % 2 == 0) && (reinterpret_cast<uintptr_t>(Bt) & 15) == 0 && kw0 + TB <= kw;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint64_t row = (bj0 + warp) * 64 + lane + 32 * h;
        if (row >= n_pad) continue;
        uint64_t* dst = Bt + row * ldbt + kw0;
        if (vec) {
#pragma unroll
            for (int kb = 0; kb < TB; kb += 2)
                *reinterpret_cast<ulonglong2*>(dst + kb) =
                    make_ulonglong2(tile[warp][kb][lane + 32 * h], tile[warp][kb + 1][lane + 32 * h]);
        } else {
#pragma unroll
            for (int kb = 0; kb < TB; ++kb)
                if (kw0 + kb < kw) dst[kb] = tile[warp][kb][lane + 32 * h];
        }
    }
}

// Staged form for 16-byte aligned operands.  The direct kernel above reads and writes
// one 16-byte piece of 32 different rows per warp instruction, so its L1 wavefronts,
// not DRAM, bound it (ncu: L1/TEX 77 %, DRAM 28 %).  Here the global side is
// row-contiguous -- four lanes cover a row's 64 bytes, a warp instruction touches 8
// rows -- and the 64 x 64 bit transposes work from shared memory.  The tile is staged in,
// transposed in registers, written back into the same buffer, and streamed out.
// Shared layout: 8 words per row, word c of row r at c ^ ((r >> 1) & 7).  Both access
// patterns are conflict-free per half-warp (16 lanes x 8 bytes): the row-contiguous ones
// (4 lanes per row, rows r .. r + 3) see 4 distinct word groups per row pair, the column
// ones (one word of rows r .. r + 15) 16 distinct (r & 1, word) pairs.  (Round 1 padded
// rows to 9 words: conflict-free columns but 23 % of the row-side wavefronts conflicted,
// profiles/r01/full_transpose_staged_c2.txt.)
constexpr int TS_ROWS = TB * 64;  // 512 rows of B per tile
__device__ __forceinline__ int ts_at(int r, int c) { return r * TB + (c ^ ((r >> 1) & 7)); }

__global__ void __launch_bounds__(256) transpose_staged_kernel(const uint64_t* __restrict__ B, uint64_t ldb,
                                                               uint64_t k, uint64_t n, uint64_t* __restrict__ Bt,
                                                               uint64_t n_pad, uint64_t kw, uint64_t ldbt) {
    __shared__ uint64_t tile[TS_ROWS * TB];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t nb_words = (n + 63) / 64;
    const uint64_t bj0 = blockIdx.x * uint64_t(TB);        // first word column (N direction)
    const uint64_t r0 = blockIdx.y * uint64_t(TS_ROWS);    // first row of B (K direction)
    const uint64_t tail_mask = (n & 63) ? (1ull << (n & 63)) - 1 : ~0ull;
    // 1. rows r0 .. r0 + 511, words bj0 .. bj0 + 7: thread t moves words 2 (t % 4) .. +1
    //    of rows t / 4 + 64 i
    {
        const unsigned q = threadIdx.x & 3, rr = threadIdx.x >> 2;
#pragma unroll
        for (int i = 0; i < TS_ROWS / 64; ++i) {
            const uint64_t row = r0 + rr + 64 * i;
            const uint64_t c = bj0 + 2 * q;
            uint64_t v0 = 0, v1 = 0;
            if (row < k) {
                if (c + 1 < nb_words) {
                    const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(B + row * ldb + c);
                    v0 = u.x;
                    v1 = u.y;
                } else if (c < nb_words) {
                    v0 = B[row * ldb + c];
                }
                if (c == nb_words - 1) v0 &= tail_mask;
                if (c + 1 == nb_words - 1) v1 &= tail_mask;
            }
            const int r = rr + 64 * i;
            tile[ts_at(r, 2 * q)] = v0;
            tile[ts_at(r, 2 * q + 1)] = v1;
        }
    }
    __syncthreads();
    // 2. warp w transposes K block w against each of the 8 word columns
    uint64_t x0[TB], x1[TB];
#pragma unroll
    for (int b = 0; b < TB; ++b) {
        x0[b] = tile[ts_at(warp * 64 + lane, b)];
        x1[b] = tile[ts_at(warp * 64 + 32 + lane, b)];
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < TB; ++b) {
        warp_transpose64(x0[b], x1[b], lane);
        // Bt row (bj0 + b) * 64 + j, K word blockIdx.y * 8 + warp -> tile[ts_at(b * 64 + j, warp)]
        tile[ts_at(b * 64 + lane, warp)] = x0[b];
        tile[ts_at(b * 64 + 32 + lane, warp)] = x1[b];
    }
    __syncthreads();
    // 3. Bt rows (bj0 * 64) .. +511, K words blockIdx.y * 8 .. +7: four lanes per row
    {
        const unsigned q = threadIdx.x & 3, rr = threadIdx.x >> 2;
        const uint64_t kw0 = blockIdx.y * uint64_t(TB) + 2 * q;
#pragma unroll
        for (int i = 0; i < TS_ROWS / 64; ++i) {
            const uint64_t trow = bj0 * 64 + rr + 64 * i;
            if (trow >= n_pad) continue;
            const int r = rr + 64 * i;
            const uint64_t w0 = tile[ts_at(r, 2 * q)], w1 = tile[ts_at(r, 2 * q + 1)];
            uint64_t* dst = Bt + trow * ldbt + kw0;
            if (kw0 + 1 < kw)
                *reinterpret_cast<ulonglong2*>(dst) = make_ulonglong2(w0, w1);
            else if (kw0 < kw)
                dst[0] = w0;
        }
    }
}

}  // namespace

// n_pad must be a multiple of 256.  Rows j >= n and K words past ceil(k/64) come
// out zero.  Bt rows are ldbt words apart (kw for a dense panel; larger when Bt is
// a quadrant of a bigger matrix, as in the streamed fast path).
int launch_transpose_ld(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                        uint64_t kw, uint64_t ldbt, cudaStream_t stream) {
    if (n_pad % 256 != 0 || n_pad < n || kw * 64 < k || ldbt < kw) {
        set_error("bmmgpu_dev_transpose: n_pad must be a multiple of 256 covering n, kw*64 must cover k");
        return kEinval;
    }
    if (n_pad == 0 || kw == 0) return kOk;
    dim3 grid(static_cast<unsigned>(ceil_div(n_pad, TB * 64)), static_cast<unsigned>(ceil_div(kw, TB)));
    const bool aligned = ldb % 2 == 0 && ldbt % 2 == 0 && (reinterpret_cast<uintptr_t>(dB) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(dBt) & 15) == 0;
    if (aligned && !getenv("BMMGPU_TRANSPOSE_DIRECT"))
        transpose_staged_kernel<<<grid, 256, 0, stream>>>(dB, ldb, k, n, dBt, n_pad, kw, ldbt);
    else
        transpose_kernel<<<grid, 256, 0, stream>>>(dB, ldb, k, n, dBt, n_pad, kw, ldbt);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

int launch_transpose(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                     uint64_t kw, cudaStream_t stream) {
    return launch_transpose_ld(dB, ldb, k, n, dBt, n_pad, kw, kw, stream);
}

}  // namespace bmmgpu
