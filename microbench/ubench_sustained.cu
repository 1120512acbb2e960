// Sustained issue rate of the K2 tensor-core instruction (tcgen05.mma cta_group::2
// kind::mxf4 block_scale, M256 N256 K64, both operands in shared memory with the 128-byte
// swizzle) on operand values like K2's (random bits expanded to e2m1: each nibble 1.0 or 0
// in the x & 0x22222222 chunks, 0.5 or 0 in the x & 0x11111111 chunks), over a 4-stage
// ring, as a burst (~0.3 ms) and back to back for several seconds under the board power
// cap.  The pure MMA loop has no producers, so it draws less power than K2 itself: the
// sustained figure is an upper bound on what K2 can reach inside a long step.
//   ubench_sustained [seconds]
#include <cstdio>
#include <cstdlib>
#include "../paper_1909_01554_b200/csrc/umma.cuh"

using namespace bmmgpu;

constexpr int STAGES = 4, STAGE = 32768;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_sus(unsigned long long* out, long long iters) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base_sh;
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const unsigned tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = umma::cluster_ctarank();
    // 16-byte chunk c of a row: chunks 0,1 of every 4 hold 1.0-class nibbles, 2,3 0.5-class
    for (int i = tid; i < STAGES * STAGE / 4; i += blockDim.x) {
        const uint32_t chunk = (uint32_t(i) >> 2) & 7;  // physical chunk; logical class is a permutation of it
        const uint32_t r = hash32(uint32_t(i) * 2654435761u + blockIdx.x * 977u);
        reinterpret_cast<uint32_t*>(smem)[i] = (chunk & 2) ? (r & 0x11111111u) : (r & 0x22222222u);
    }
    if (warp == 0) umma::tmem_alloc2(&tmem_base_sh, 512);
    if (tid == 0) {
        umma::mbar_init(&bar, 1);
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tmem_base_sh;
    const uint32_t lb = (warp * 32) << 16;
    umma::tmem_st8_fill(tmem + lb + 480, 0x7F7F7F7Fu);
    umma::tmem_st8_fill(tmem + lb + 488, 0x80808080u);
    umma::tmem_st_wait();
    umma::fence_before_sync();
    umma::cluster_sync();
    umma::fence_after_sync();
    if (rank == 0 && tid == 0) {
        constexpr uint32_t idesc = umma::idesc_mxf4(256, 256);
        const uint32_t base = smem_u32(smem);
        unsigned long long g0, g1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        const long long c0 = clock64();
        for (long long it = 0; it < iters; ++it) {
            const uint32_t s = uint32_t(it & (STAGES - 1));
            const uint32_t a0 = base + s * STAGE, b0 = a0 + STAGE / 2;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t sf = tmem + ((j & 1) ? 488 : 480);
                umma::mma_mxf4_pair(tmem, umma::smem_desc_sw128(a0 + 32 * j, 1024),
                                    umma::smem_desc_sw128(b0 + 32 * j, 1024), idesc, sf, sf, (it | j) ? 1u : 0u);
            }
        }
        umma::mma_commit_pair(&bar, 0x3);
        umma::mbar_wait(&bar, 0);
        const long long c1 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        out[blockIdx.x * 2] = c1 - c0;
        out[blockIdx.x * 2 + 1] = g1 - g0;
    } else if (tid == 0) {
        umma::mbar_wait(&bar, 0);
    }
    __syncthreads();
    umma::fence_before_sync();
    umma::cluster_sync();
    if (warp == 0) {
        umma::fence_after_sync();
        umma::tmem_dealloc2(tmem, 512);
    }
}

int main(int argc, char** argv) {
    const double seconds = argc > 1 ? atof(argv[1]) : 4.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* out;
    cudaMalloc(&out, 16 * 256);
    const int smem = STAGES * STAGE + 1024;
    cudaFuncSetAttribute(k_sus, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    static unsigned long long h[2 * 256];
    const double macs_per_it = 4 * (128.0 * 256 * 64);  // per SM
    // calibrate: ~560 clk per iteration at ~1.9 GHz -> ~3.4 M iterations per second
    for (int pass = 0; pass < 3; ++pass) {
        const long long iters = pass == 0 ? 1000 : pass == 1 ? 1000 : (long long)(seconds * 3.3e6);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_sus<<<sms, 128, smem>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h, out, sizeof(unsigned long long) * 2 * sms, cudaMemcpyDeviceToHost);
        double clk = 0, ns = 0;
        int n = 0;
        for (int b = 0; b < sms; b += 2, ++n) clk += h[2 * b], ns += h[2 * b + 1];
        clk /= n, ns /= n;
        if (pass == 0) continue;  // warm-up
        const double mac_s = macs_per_it * iters * sms / (ns * 1e-9);
        printf("{\"bench\": \"mxf4_pair_%s\", \"iters\": %lld, \"ms\": %.3f, \"mac_per_s\": %.4e, \"bop_per_s\": %.4e, "
               "\"mac_per_clk_per_sm\": %.0f, \"mhz\": %.0f, \"err\": \"%s\"}\n",
               pass == 1 ? "burst" : "sustained", iters, ms, mac_s, 2 * mac_s, macs_per_it * iters / clk,
               clk / ns * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
