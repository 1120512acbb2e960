// kernel64.cu -- K9: one 64 x 64 block product in the reference's own operand form
// (reference engine.cpp:34-56 kernel64: out[i] bit k = parity(popcount(a[i] & bt[k])) for
// GF(2), (a[i] & bt[k]) != 0 for Boolean; bt is B column-major, word k = column k).
//
// The reference calls it ~4.6 us of one core per block; a caller that loops over
// bmm::kernel64 must not pay a full host-API product per block (stream lease, three
// copies, a transpose and a persistent launch: ~50-100 us).  So this entry point is one
// launch and one synchronisation: the caller's 128 input words are staged in this
// thread's page-locked, device-mapped buffer, one warp-pair reads them straight over the
// link (zero-copy), forms the 64 output words with AND + POPC, and writes them back into
// the mapped buffer.  Latency-bound by construction (launch + PCIe round trip), not a
// throughput path: the block products of real matrices run in K1/K2.
#include <cstring>
#include <string>

#include "bmmgpu.h"
#include "common.cuh"

namespace bmmgpu {

void set_error(const std::string& msg);
void count_launch(uint64_t n);

namespace {

// 64 threads: thread i owns output row i; the 64 B columns sit in shared memory.
__global__ void __launch_bounds__(64) kernel64_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                      int gf2) {
    __shared__ uint64_t bt[64];
    const unsigned i = threadIdx.x;
    const uint64_t a = in[i];
    bt[i] = in[64 + i];
    __syncthreads();
    uint64_t w = 0;
#pragma unroll 8
    for (int k = 0; k < 64; ++k) {
        const uint64_t x = a & bt[k];
        const uint64_t bit = gf2 ? uint64_t(__popcll(x) & 1) : uint64_t(x != 0);
        w |= bit << k;
    }
    out[i] = w;
}

struct K64State {
    int device = -1;
    uint64_t* host = nullptr;  // 192 words: a, bt, out (page-locked, mapped)
    uint64_t* dev = nullptr;   // device alias of host
    cudaStream_t stream = nullptr;
    ~K64State() {
        // thread exit; at process exit the runtime may already be unloading (then the OS
        // reclaims the 1.5 KB and the stream)
        int prev = 0;
        if (!host || cudaGetDevice(&prev) != cudaSuccess) return;
        if (prev != device) cudaSetDevice(device);
        if (stream) cudaStreamDestroy(stream);
        cudaFreeHost(host);
        if (prev != device) cudaSetDevice(prev);
    }
};
thread_local K64State t_k64;

int k64_state(K64State& s) {
    int dev = 0;
    BMMGPU_CUDA_TRY(cudaGetDevice(&dev));
    if (s.host && s.device == dev) return kOk;
    if (s.host) {  // the thread moved to another device
        if (s.stream) cudaStreamDestroy(s.stream);
        cudaFreeHost(s.host);
        s = K64State{};
    }
    BMMGPU_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&s.host), 192 * sizeof(uint64_t), cudaHostAllocMapped));
    BMMGPU_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&s.dev), s.host, 0));
    BMMGPU_CUDA_TRY(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    s.device = dev;
    return kOk;
}

}  // namespace
}  // namespace bmmgpu

using namespace bmmgpu;

extern "C" int bmmgpu_kernel64(const uint64_t* a, const uint64_t* bt, uint64_t* out, int32_t semiring) {
    if (!a || !bt || !out) {
        set_error("bmmgpu_kernel64: null operand");
        return kEinval;
    }
    if (semiring != 0 && semiring != 1) {
        set_error("unknown semiring");
        return kEinval;
    }
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        set_error("no CUDA device available; the bit-matrix engine has no CPU fallback");
        return kEnodev;
    }
    K64State& s = t_k64;
    if (const int st = k64_state(s)) return st;
    std::memcpy(s.host, a, 64 * sizeof(uint64_t));
    std::memcpy(s.host + 64, bt, 64 * sizeof(uint64_t));
    kernel64_kernel<<<1, 64, 0, s.stream>>>(s.dev, s.dev + 128, semiring == BMMGPU_GF2_XOR_AND ? 1 : 0);
    BMMGPU_CUDA_TRY(cudaGetLastError());
    count_launch(1);
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(s.stream));
    std::memcpy(out, s.host + 128, 64 * sizeof(uint64_t));
    return kOk;
}
