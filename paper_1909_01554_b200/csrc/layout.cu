// layout.cu -- K8: the layout conversions of the bmm:: API on the device, and their
// host-streamed drivers for matrices larger than HBM (the
// reference CLI's `transform`, tools/bmm_cli.cpp:210-234, on 2^20-sized operands).
//
//   transpose_blocks64 (reference bitmatrix.cpp:97-110): every 64 x 64 block transposed
//     in place, blocks stay where they are;
//   to_interleaved / from_interleaved (bitmatrix.cpp:112-173): 64-word blocks in Morton
//     order (level-l row digit at bit 2l+1, column digit at bit 2l, outermost level
//     first), a right operand's blocks stored transposed.
//
// HBM-bound byte permutation: per 64 x 64 block 512 B in, 512 B out.  A CTA of 8 warps
// takes an 8 x 8 square of blocks; warp w owns block row w: lane l loads rows l and
// l + 32 of its 8 blocks (64 contiguous bytes per row, 16-byte loads), transposes each
// block across the warp with shuffles when the conversion asks for it, and stores each
// block as 512 contiguous bytes (lane l: words l and l + 32).  An aligned 2^k x 2^k
// square of blocks is a contiguous Morton range, so the 64 blocks of a CTA land in
// 32 KB of contiguous output.  No shared memory.
//
// Host driver: the matrix is cut into Morton-aligned square super-tiles (S x S bits,
// S = min(n, 16384): 32 MiB) or, for the block transpose, row panels; each goes up
// (2-D copy of S rows for a super-tile of a row-major matrix), is converted, and comes
// back (one contiguous copy into its Morton range), three slots on three streams so
// the upload of one, the kernel of another and the download of a third overlap.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <string>
#include <vector>

#include "bmmgpu.h"
#include "common.cuh"

namespace bmmgpu {

namespace {

// bit i of x -> bit 2i (x < 2^32)
__device__ __forceinline__ uint64_t spread2(uint64_t x) {
    x &= 0xFFFFFFFFull;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}
// Morton index of block (bi, bj): row digit at the odd bit (reference morton2,
// bitmatrix.cpp:35-42)
__device__ __forceinline__ uint64_t morton_block(uint64_t bi, uint64_t bj) { return (spread2(bi) << 1) | spread2(bj); }

enum Mode : int {
    kTranspose = 0,    // row-major -> row-major, blocks transposed (in place allowed)
    kToMorton = 1,     // row-major -> Morton
    kFromMorton = 2,   // Morton -> row-major
};

// A square of nb x nb blocks (row-major side: row pitch ld words) or, for kTranspose, a
// rows x cols-word rectangle of blocks.  `tr`: transpose every block.
__global__ void __launch_bounds__(256) layout_kernel(const uint64_t* src, uint64_t* dst,
                                                     uint64_t nbr, uint64_t nbc, uint64_t ld, int mode, int tr) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t bi = blockIdx.y * 8ull + warp;   // block row
    const uint64_t bj0 = blockIdx.x * 8ull;         // first block column of the CTA
    if (bi >= nbr) return;
    const int nblk = nbc - bj0 < 8 ? int(nbc - bj0) : 8;
    uint64_t x0[8], x1[8];
    const bool vec = nblk == 8 && (ld % 2) == 0;
    if (mode == kFromMorton) {
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (b < nblk) {
                const uint64_t* s = src + morton_block(bi, bj0 + b) * 64;
                x0[b] = s[lane];
                x1[b] = s[lane + 32];
            }
    } else {
        const uint64_t* r0 = src + (bi * 64 + lane) * ld + bj0;
        const uint64_t* r1 = r0 + 32 * ld;
        if (vec) {
#pragma unroll
            for (int b = 0; b < 8; b += 2) {
                const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(r0 + b);
                const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(r1 + b);
                x0[b] = u.x;
                x0[b + 1] = u.y;
                x1[b] = v.x;
                x1[b + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int b = 0; b < 8; ++b)
                if (b < nblk) {
                    x0[b] = r0[b];
                    x1[b] = r1[b];
                }
        }
    }
    if (tr) {
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (b < nblk) warp_transpose64(x0[b], x1[b], lane);
    }
    if (mode == kToMorton) {
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (b < nblk) {
                uint64_t* d = dst + morton_block(bi, bj0 + b) * 64;
                d[lane] = x0[b];
                d[lane + 32] = x1[b];
            }
    } else {
        uint64_t* r0 = dst + (bi * 64 + lane) * ld + bj0;
        uint64_t* r1 = r0 + 32 * ld;
        if (vec) {
#pragma unroll
            for (int b = 0; b < 8; b += 2) {
                *reinterpret_cast<ulonglong2*>(r0 + b) = make_ulonglong2(x0[b], x0[b + 1]);
                *reinterpret_cast<ulonglong2*>(r1 + b) = make_ulonglong2(x1[b], x1[b + 1]);
            }
        } else {
#pragma unroll
            for (int b = 0; b < 8; ++b)
                if (b < nblk) {
                    r0[b] = x0[b];
                    r1[b] = x1[b];
                }
        }
    }
}

int launch_layout(const uint64_t* src, uint64_t* dst, uint64_t nbr, uint64_t nbc, uint64_t ld, int mode, bool tr,
                  cudaStream_t s) {
    if (nbr == 0 || nbc == 0) return kOk;
    const dim3 grid(unsigned(ceil_div(nbc, 8)), unsigned(ceil_div(nbr, 8)));
    layout_kernel<<<grid, 256, 0, s>>>(src, dst, nbr, nbc, ld, mode, tr ? 1 : 0);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

// op -> (interleave direction, transpose blocks)
bool decode_op(int op, int* mode, bool* tr) {
    switch (op) {
        case BMMGPU_LAYOUT_TRANSPOSE_BLOCKS64: *mode = kTranspose; *tr = true; return true;
        case BMMGPU_LAYOUT_TO_INTERLEAVED: *mode = kToMorton; *tr = false; return true;
        case BMMGPU_LAYOUT_TO_INTERLEAVED_RIGHT: *mode = kToMorton; *tr = true; return true;
        case BMMGPU_LAYOUT_FROM_INTERLEAVED: *mode = kFromMorton; *tr = false; return true;
        case BMMGPU_LAYOUT_FROM_INTERLEAVED_RIGHT: *mode = kFromMorton; *tr = true; return true;
        default: return false;
    }
}

int check_shape(uint64_t rows, uint64_t cols, int mode) {
    if (mode == kTranspose) {
        if (rows % 64 || cols % 64) {
            set_error("block transpose needs dimensions divisible by 64");
            return kEshape;
        }
        return kOk;
    }
    if (rows != cols || rows < 64 || (rows & (rows - 1))) {
        set_error("matrix does not match plan dimension");  // interleave: n = 64 * 2^depth
        return kEshape;
    }
    return kOk;
}

}  // namespace

int layout_dev(const uint64_t* src, uint64_t* dst, uint64_t rows, uint64_t cols, int op, cudaStream_t s) {
    int mode;
    bool tr;
    if (!decode_op(op, &mode, &tr)) {
        set_error("unknown layout op " + std::to_string(op));
        return kEinval;
    }
    if (int rc = check_shape(rows, cols, mode)) return rc;
    if (mode != kTranspose && src == dst) {
        set_error("interleave conversions are out of place");
        return kEinval;
    }
    return launch_layout(src, dst, rows / 64, cols / 64, cols / 64, mode, tr, s);
}

// Host buffers (page-locked or pageable), streamed through the device in pieces.
int layout_host(const uint64_t* src, uint64_t* dst, uint64_t rows, uint64_t cols, int op, uint64_t piece_bits) {
    int mode;
    bool tr;
    if (!decode_op(op, &mode, &tr)) {
        set_error("unknown layout op " + std::to_string(op));
        return kEinval;
    }
    if (int rc = check_shape(rows, cols, mode)) return rc;
    if (mode != kTranspose && src == dst) {
        set_error("interleave conversions are out of place");
        return kEinval;
    }
    if (rows == 0 || cols == 0) return kOk;
    const uint64_t wpr = cols / 64;
    // pieces: row panels of the block transpose (contiguous), square super-tiles otherwise
    uint64_t S = piece_bits ? piece_bits : 16384;
    S = std::max<uint64_t>(64, S & ~63ull);
    std::vector<std::array<uint64_t, 2>> pieces;  // (row or tile-row, column tile) in units of S
    uint64_t piece_words;
    if (mode == kTranspose) {
        const uint64_t panel = std::max<uint64_t>(64, ((uint64_t(4) << 20) / wpr) & ~63ull);  // ~32 MiB
        for (uint64_t r = 0; r < rows; r += panel) pieces.push_back({r, std::min(panel, rows - r)});
        piece_words = std::min(panel, rows) * wpr;
    } else {
        uint64_t side = 64;
        while (side * 2 <= std::min(S, rows)) side *= 2;  // power of two: Morton-aligned tiles
        S = side;
        for (uint64_t I = 0; I < rows / S; ++I)
            for (uint64_t J = 0; J < rows / S; ++J) pieces.push_back({I, J});
        piece_words = S * S / 64;
    }
    constexpr int kSlots = 3;
    StreamSet ss;
    if (int r = ss.acquire(kSlots)) return r;
    DeviceBuffer bin[kSlots], bout[kSlots];
    StreamDrain drain{{ss[0], ss[1], ss[2], nullptr}};
    const int nslots = int(std::min<size_t>(kSlots, pieces.size()));
    for (int i = 0; i < nslots; ++i) {
        if (int r = bin[i].alloc(piece_words * 8, ss[i])) return r;
        if (mode != kTranspose)
            if (int r = bout[i].alloc(piece_words * 8, ss[i])) return r;
    }
    // Pageable buffers: the staged copies are host-synchronous, so the slots only
    // overlap the kernels with the copies; page-locked ones overlap everything.
    const uint64_t n = rows;
    for (size_t p = 0; p < pieces.size(); ++p) {
        const int k = int(p % kSlots);
        const cudaStream_t s = ss[k];
        if (mode == kTranspose) {
            const uint64_t r0 = pieces[p][0], nr = pieces[p][1];
            BMMGPU_CUDA_TRY(memcpy_counted(bin[k].p, src + r0 * wpr, nr * wpr * 8, cudaMemcpyHostToDevice, s));
            if (int rc = launch_layout(bin[k].u(), bin[k].u(), nr / 64, wpr, wpr, kTranspose, true, s)) return rc;
            BMMGPU_CUDA_TRY(memcpy_counted(dst + r0 * wpr, bin[k].p, nr * wpr * 8, cudaMemcpyDeviceToHost, s));
            continue;
        }
        const uint64_t I = pieces[p][0], J = pieces[p][1], sw = S / 64;
        // Morton range of the super-tile: morton(I * sw, J * sw) .. + sw^2 blocks
        uint64_t mb = 0;
        for (int bit = 0; bit < 32; ++bit) {
            const uint64_t bi = I * sw, bj = J * sw;
            mb |= ((bi >> bit) & 1) << (2 * bit + 1);
            mb |= ((bj >> bit) & 1) << (2 * bit);
        }
        const uint64_t moff = mb * 64;  // words
        if (mode == kToMorton) {
            BMMGPU_CUDA_TRY(memcpy2d_counted(bin[k].p, sw * 8, src + I * S * (n / 64) + J * sw, (n / 64) * 8, sw * 8,
                                             S, cudaMemcpyHostToDevice, s));
            if (int rc = launch_layout(bin[k].u(), bout[k].u(), sw, sw, sw, kToMorton, tr, s)) return rc;
            BMMGPU_CUDA_TRY(memcpy_counted(dst + moff, bout[k].p, piece_words * 8, cudaMemcpyDeviceToHost, s));
        } else {
            BMMGPU_CUDA_TRY(memcpy_counted(bin[k].p, src + moff, piece_words * 8, cudaMemcpyHostToDevice, s));
            if (int rc = launch_layout(bin[k].u(), bout[k].u(), sw, sw, sw, kFromMorton, tr, s)) return rc;
            BMMGPU_CUDA_TRY(memcpy2d_counted(dst + I * S * (n / 64) + J * sw, (n / 64) * 8, bout[k].p, sw * 8, sw * 8,
                                             S, cudaMemcpyDeviceToHost, s));
        }
    }
    for (int i = 0; i < nslots; ++i) BMMGPU_CUDA_TRY(cudaStreamSynchronize(ss[i]));
    return kOk;
}

}  // namespace bmmgpu

extern "C" int bmmgpu_layout(const uint64_t* src, uint64_t* dst, uint64_t rows, uint64_t cols, int32_t op,
                             const bmmgpu_opts* opts) {
    bmmgpu::reset_call_stats();
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        bmmgpu::set_error("no CUDA device available; the bit-matrix engine has no CPU fallback");
        return bmmgpu::kEnodev;
    }
    const uint32_t mask = opts ? opts->device_mask : 0u;
    const int device = mask ? __builtin_ctz(mask) : 0;
    if (device >= count) {
        bmmgpu::set_error("device_mask names a missing device");
        return bmmgpu::kEinval;
    }
    BMMGPU_CUDA_TRY(cudaSetDevice(device));
    // BMMGPU_LAYOUT_PIECE: super-tile side in bits (tests force small pieces)
    const char* pe = getenv("BMMGPU_LAYOUT_PIECE");
    return bmmgpu::layout_host(src, dst, rows, cols, op, pe ? strtoull(pe, nullptr, 10) : 0);
}

extern "C" int bmmgpu_dev_layout(const uint64_t* d_src, uint64_t* d_dst, uint64_t rows, uint64_t cols, int32_t op,
                                 void* stream) {
    return bmmgpu::layout_dev(d_src, d_dst, rows, cols, op, static_cast<cudaStream_t>(stream));
}
