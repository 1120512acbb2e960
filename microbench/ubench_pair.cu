// Issue rate of the CTA-pair MMA used by cubic_umma2.cu (tcgen05.mma
// cta_group::2 kind::mxf4, M256 N256 K64, 128-byte-swizzled K-major operands)
// without the producer pipeline, adding the MMA lane's per-stage overheads one
// at a time: stage ring addresses, tcgen05.fence, mbarrier waits, per-stage
// multicast commits.
#include <cstdio>
#include "../paper_1909_01554_b200/csrc/umma.cuh"

using namespace bmmgpu;

constexpr int STAGES = 6, STAGE = 32768;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_pair(uint32_t* out, int iters, int variant) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar[STAGES + 1];
    __shared__ uint32_t tmem_base_sh;
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const unsigned tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = umma::cluster_ctarank();
    for (int i = tid; i < STAGES * STAGE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22222222u;
    if (warp == 0) umma::tmem_alloc2(&tmem_base_sh, 512);
    if (tid == 0) {
        for (int s = 0; s <= STAGES; ++s) umma::mbar_init(&bar[s], 1);
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tmem_base_sh;
    umma::tmem_st32_fill(tmem + ((warp * 32) << 16) + 256, 0x7F7F7F7Fu);
    umma::tmem_st32_fill(tmem + ((warp * 32) << 16) + 384, 0x80808080u);
    umma::tmem_st_wait();
    umma::fence_before_sync();
    umma::cluster_sync();
    umma::fence_after_sync();
    // variant bits: 1 rotate over the 6-stage ring, 2 fence::after_thread_sync per stage,
    // 4 commit each stage to its own barrier (multicast), 8 wait on the commit of stage it-6
    if (rank == 0 && tid == 0) {
        constexpr uint32_t idesc = umma::idesc_mxf4(256, 256);
        const uint32_t base = smem_u32(smem);
        for (int it = 0; it < iters; ++it) {
            const int s = (variant & 1) ? it % STAGES : 0;
            if ((variant & 8) && it >= STAGES) umma::mbar_wait(&bar[s], ((it / STAGES) + 1) & 1);
            if (variant & 2) umma::fence_after_sync();
            const uint32_t a0 = base + s * STAGE, b0 = a0 + STAGE / 2;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t sf = tmem + ((j & 1) ? 384 : 256);
                umma::mma_mxf4_pair(tmem, umma::smem_desc_sw128(a0 + 32 * j, 1024),
                                    umma::smem_desc_sw128(b0 + 32 * j, 1024), idesc, sf, sf, (it | j) ? 1u : 0u);
            }
            if (variant & 4) umma::mma_commit_pair(&bar[s], 0x1);
        }
        umma::mma_commit_pair(&bar[STAGES], 0x3);
    }
    if (tid == 0) umma::mbar_wait(&bar[STAGES], 0);
    __syncthreads();
    umma::fence_before_sync();
    umma::cluster_sync();
    if (warp == 0) {
        umma::fence_after_sync();
        umma::tmem_dealloc2(tmem, 512);
    }
    if (tid == 0) out[blockIdx.x] = rank;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 4096);
    const int smem = STAGES * STAGE + 1024;
    cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int variant : {0, 1, 3, 7, 15}) {
        const int iters = 12000;
        k_pair<<<sms, 128, smem>>>(out, 60, variant);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        k_pair<<<sms, 128, smem>>>(out, iters, variant);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double macs = double(sms / 2) * iters * 4 * (256.0 * 256 * 64);
        printf("{\"bench\": \"pair_mxf4_sw128\", \"variant\": %d, \"ms\": %.3f, \"bop_per_s\": %.4e, \"err\": \"%s\"}\n",
               variant, ms, 2 * macs / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
