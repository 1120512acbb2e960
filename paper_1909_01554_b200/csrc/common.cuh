// common.cuh -- shared helpers for the sm_100a bit-product kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <functional>
#include <string>

namespace bmmgpu {

// Status codes mirror include/bmmgpu.h.
constexpr int kOk = 0, kEinval = 1, kEshape = 3, kEcuda = 5, kEnodev = 6;

void set_error(const std::string& msg);
void count_launch(uint64_t n = 1);
// Host<->device bytes moved by the host-API drivers (bmmgpu_last_copy_bytes).
void count_copy(cudaMemcpyKind kind, uint64_t bytes);
// Per-call diagnostics (launch count, copied bytes) belong to the calling thread: a
// host-API call resets its thread's tallies, and the worker threads it spawns (one per
// device) add into the caller's with call_stats() / adopt_call_stats(), so concurrent
// calls on different threads never see each other's counts.
void* call_stats();
void adopt_call_stats(void* stats);  // nullptr: back to this thread's own tallies
void reset_call_stats();
// Host<->device copies of the host-API drivers.  Page-locked host buffers go straight
// to the DMA engines (asynchronous on `s`); large pageable ones (the reference API's
// std::vector storage) are staged through pinned double buffers, with host threads
// filling / draining one slot while the DMA engine moves the other -- host-synchronous
// for the pageable side, like the runtime's own pageable copies, but at a multiple of
// their bandwidth.
cudaError_t memcpy2d_counted(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                             cudaMemcpyKind kind, cudaStream_t s);
inline cudaError_t memcpy_counted(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    return memcpy2d_counted(dst, bytes, src, bytes, bytes, 1, kind, s);
}
#define BMMGPU_CUDA_TRY(expr)                                                                     \
    do {                                                                                          \
        cudaError_t _e = (expr);                                                                  \
        if (_e != cudaSuccess) {                                                                  \
            ::bmmgpu::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));              \
            return ::bmmgpu::kEcuda;                                                              \
        }                                                                                         \
    } while (0)

// Stream-ordered device buffer from the device's default memory pool.  The
// pool keeps freed memory (release threshold = max), so the multi-GB level
// buffers of repeated calls are recycled instead of re-mapped, and freeing a
// level's buffer needs no stream synchronisation.
void enable_pool_caching();
// Free bytes on the current device for planning (capi.cu): a cached cudaMemGetInfo snapshot
// corrected by the memory pool's reservations; refresh = a fresh (possibly blocking) query.
uint64_t device_free_bytes(bool refresh);
// f(0) .. f(parts - 1) over the library's host helper threads (capi.cu), and their number.
void host_parallel(unsigned parts, const std::function<void(unsigned)>& f);
unsigned host_parallel_width();

// Non-blocking streams leased from a per-device pool: creating and destroying a
// stream costs ~100 us of host time (measured, microbench/api_cost.py), three per call
// were most of a small product's end-to-end time.  Concurrent calls lease distinct
// streams; a lease goes back to the pool when the set is destroyed -- declare it
// before the driver's buffers and StreamDrain, so the streams are idle by then.
struct StreamSet {
    int device = -1, n = 0, prio = 0;
    cudaStream_t s[4] = {nullptr, nullptr, nullptr, nullptr};
    StreamSet() = default;
    StreamSet(const StreamSet&) = delete;
    StreamSet& operator=(const StreamSet&) = delete;
    // on the current device; 0 or a CUDA status.  priority: 0 default, 1 the device's
    // greatest (its pending blocks are scheduled first), -1 its least
    int acquire(int count, int priority = 0);
    ~StreamSet();
    cudaStream_t operator[](int i) const { return s[i]; }
};

// Declared after a driver's buffers, so it is destroyed first: waits for every stream
// the driver used before the buffers' stream-ordered frees run (on error returns the
// copy streams may still be reading or writing them).
struct StreamDrain {
    cudaStream_t s[4] = {nullptr, nullptr, nullptr, nullptr};
    ~StreamDrain() {
        for (cudaStream_t x : s)
            if (x) cudaStreamSynchronize(x);
    }
};

struct DeviceBuffer {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    DeviceBuffer() = default;
    explicit DeviceBuffer(cudaStream_t stream) : s(stream) {}
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p(o.p), s(o.s) { o.p = nullptr; }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            s = o.s;
            o.p = nullptr;
        }
        return *this;
    }
    ~DeviceBuffer() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
    }
    int alloc(size_t bytes, cudaStream_t stream) {
        release();
        s = stream;
        enable_pool_caching();
        cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, s);
        if (e != cudaSuccess) {
            set_error("cudaMallocAsync(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
            p = nullptr;
            return kEcuda;
        }
        return kOk;
    }
    uint64_t* u() const { return static_cast<uint64_t*>(p); }
};

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline uint64_t round_up(uint64_t a, uint64_t b) { return ceil_div(a, b) * b; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// One stage of the warp-wide 64x64 bit transpose (reference bitmatrix.cpp:16-31
// restated across lanes): lane l holds rows l and l+32.  For w >= 1 and < 32 the
// partner rows live in lane l^w; w = 32 is the in-lane swap.
__device__ __forceinline__ uint64_t tr_stage(uint64_t x, unsigned lane, unsigned w, uint64_t m) {
    const uint64_t p = __shfl_xor_sync(0xffffffffu, x, w);
    if (lane & w) {
        const uint64_t t = ((p >> w) ^ x) & m;
        return x ^ t;
    } else {
        const uint64_t t = ((x >> w) ^ p) & m;
        return x ^ (t << w);
    }
}

// Full 64x64 transpose of the block held as (x0 = row lane, x1 = row lane+32).
__device__ __forceinline__ void warp_transpose64(uint64_t& x0, uint64_t& x1, unsigned lane) {
    {
        const uint64_t t = ((x0 >> 32) ^ x1) & 0x00000000FFFFFFFFull;
        x0 ^= t << 32;
        x1 ^= t;
    }
    x0 = tr_stage(x0, lane, 16, 0x0000FFFF0000FFFFull);
    x1 = tr_stage(x1, lane, 16, 0x0000FFFF0000FFFFull);
    x0 = tr_stage(x0, lane, 8, 0x00FF00FF00FF00FFull);
    x1 = tr_stage(x1, lane, 8, 0x00FF00FF00FF00FFull);
    x0 = tr_stage(x0, lane, 4, 0x0F0F0F0F0F0F0F0Full);
    x1 = tr_stage(x1, lane, 4, 0x0F0F0F0F0F0F0F0Full);
    x0 = tr_stage(x0, lane, 2, 0x3333333333333333ull);
    x1 = tr_stage(x1, lane, 2, 0x3333333333333333ull);
    x0 = tr_stage(x0, lane, 1, 0x5555555555555555ull);
    x1 = tr_stage(x1, lane, 1, 0x5555555555555555ull);
}

}  // namespace bmmgpu
