// Shared-memory write bandwidth per SM on B200: STS.128 from registers versus
// bulk async copies (cp.async.bulk global->shared, L2-resident source).
// Decides whether the expanded-operand producer of the tcgen05 bit product is
// bound by the STS path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void sts_kernel(uint32_t* out, int iters) {
    extern __shared__ __align__(16) uint4 sm[];
    uint4 v = make_uint4(threadIdx.x, threadIdx.x * 3, threadIdx.x * 5, threadIdx.x * 7);
    const int n = 96 * 1024 / 16;  // 96 KB ring
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            sm[i] = v;
            v.x += 1;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sm[5].x;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const uint8_t* src, uint32_t* out, int iters, size_t src_bytes) {
    extern __shared__ __align__(128) uint8_t sm8[];
    __shared__ __align__(8) uint64_t bar;
    const int chunk = 16 * 1024, nchunks = 6;  // 96 KB per round
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                         "r"(chunk * nchunks));
            for (int c = 0; c < nchunks; ++c) {
                const uint8_t* g = src + ((size_t(blockIdx.x) * 7 + it * 13 + c) * chunk) % (src_bytes - chunk);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(sm8 + c * chunk)),
                    "l"(g), "r"(chunk), "r"(smem_u32(&bar))
                    : "memory");
            }
        }
        uint32_t done = 0;
        while (!done)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(done)
                         : "r"(smem_u32(&bar)), "r"(phase));
        phase ^= 1;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = sm8[100];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 4096 * 4);
    const size_t src_bytes = 64ull << 20;  // 64 MB, L2 resident
    uint8_t* src;
    cudaMalloc(&src, src_bytes);
    cudaMemset(src, 1, src_bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaFuncSetAttribute(sts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int threads : {256, 512, 1024}) {
        const int iters = 2000;
        sts_kernel<<<sms, threads, 96 * 1024>>>(out, 10);
        cudaEventRecord(e0);
        sts_kernel<<<sms, threads, 96 * 1024>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = double(sms) * iters * 96 * 1024;
        printf("{\"bench\": \"sts128\", \"threads\": %d, \"TBps\": %.3f, \"B_per_clk_per_sm_at_max\": %.1f, \"err\": \"%s\"}\n",
               threads, bytes / ms / 1e9, bytes / (ms * 1e-3) / sms / (clk * 1e3), cudaGetErrorString(cudaGetLastError()));
    }
    {
        const int iters = 4000;
        bulk_kernel<<<sms, 32, 96 * 1024>>>(src, out, 10, src_bytes);
        cudaEventRecord(e0);
        bulk_kernel<<<sms, 32, 96 * 1024>>>(src, out, iters, src_bytes);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = double(sms) * iters * 96 * 1024;
        printf("{\"bench\": \"bulk_g2s_L2\", \"TBps\": %.3f, \"B_per_clk_per_sm_at_max\": %.1f, \"err\": \"%s\"}\n",
               bytes / ms / 1e9, bytes / (ms * 1e-3) / sms / (clk * 1e3), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
