// Peak issue rate of the CTA-pair MMA used by cubic_umma2.cu (tcgen05.mma
// cta_group::2 kind::mxf4, M256 N256 K64, 128-byte-swizzled K-major operands),
// with no producer pipeline: one resident stage, back-to-back MMAs.
#include <cstdio>
#include "../paper_1909_01554_b200/csrc/umma.cuh"

using namespace bmmgpu;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_pair(uint32_t* out, int iters, int per_commit, int alt_sf) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base_sh;
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const unsigned tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = umma::cluster_ctarank();
    for (int i = tid; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22222222u;
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
    umma::tmem_st32_fill(tmem + ((warp * 32) << 16) + 256, 0x7F7F7F7Fu);
    umma::tmem_st32_fill(tmem + ((warp * 32) << 16) + 384, 0x80808080u);
    umma::tmem_st_wait();
    umma::fence_before_sync();
    umma::cluster_sync();
    umma::fence_after_sync();
    if (rank == 0 && tid == 0) {
        constexpr uint32_t idesc = umma::idesc_mxf4(256, 256);
        const uint32_t a0 = smem_u32(smem), b0 = a0 + 16384;
        uint32_t n = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                umma::mma_mxf4_pair(tmem, umma::smem_desc_sw128(a0 + 32 * j, 1024),
                                    umma::smem_desc_sw128(b0 + 32 * j, 1024), idesc, tmem + ((alt_sf && (j & 1)) ? 384 : 256), tmem + ((alt_sf && (j & 1)) ? 384 : 256),
                                    (it | j) ? 1u : 0u);
            }
            if (per_commit && (++n % per_commit) == 0) umma::mma_commit_pair(&bar, 0x1);  // mimic per-stage commits
        }
        umma::mma_commit_pair(&bar, 0x3);
    }
    // both CTAs wait for the final commit (phase count depends on per_commit; wait on the last phase)
    if (tid == 0) {
        const uint32_t phases = (rank == 0 && per_commit) ? uint32_t(iters / per_commit) : 0u;
        umma::mbar_wait(&bar, phases & 1);
    }
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
    cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int alt_sf : {0, 1}) for (int per_commit : {0, 1}) {
        const int iters = 20000;
        k_pair<<<sms, 128, 40 * 1024>>>(out, 100, per_commit, alt_sf);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        k_pair<<<sms, 128, 40 * 1024>>>(out, iters, per_commit, alt_sf);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double macs = double(sms / 2) * iters * 4 * (256.0 * 256 * 64);
        printf("{\"bench\": \"pair_mxf4_m256n256k64_sw128\", \"alt_sf\": %d, \"commit_every_4\": %d, \"ms\": %.3f, \"MAC_per_s\": %.4e, "
               "\"bop_per_s\": %.4e, \"err\": \"%s\"}\n",
               alt_sf, per_commit, ms, macs / (ms * 1e-3), 2 * macs / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
