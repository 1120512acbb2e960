// Does the CTA-pair mxf4 MMA stream (tensor-core shared-memory reads) slow down
// when 8 warps store expanded operands with STS.128 at the same time, and vice
// versa?  Decides whether the persistent kernel's producer/MMA ring is bound by
// shared-memory bandwidth (writes + tensor reads share the SM's data path) or by
// synchronisation latency.
// mode 1: MMA only; 2: STS only; 3: both concurrently (no synchronisation between them)
#include <cstdio>
#include "../paper_1909_01554_b200/csrc/umma.cuh"

using namespace bmmgpu;

constexpr int STAGES = 6, STAGE = 32768;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    k_contend(uint32_t* out, int mma_iters, int sts_iters, int mode, unsigned long long* cycles, int fill) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tmem_base_sh;
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const unsigned tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = umma::cluster_ctarank();
    // operand data: fill 0 = all 1.0 (0x22222222), 1 = random bits expanded like the
    // product kernel (x & 0x22222222 / x & 0x11111111 chunks), 2 = zeros
    for (int i = tid; i < STAGES * STAGE / 4; i += blockDim.x) {
        uint32_t x = (i + 1) * 2654435761u + blockIdx.x * 40503u;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        reinterpret_cast<uint32_t*>(smem)[i] = fill == 0 ? 0x22222222u : fill == 2 ? 0u : (x & (((i >> 2) & 2) ? 0x11111111u : 0x22222222u));
    }
    if (warp == 0) umma::tmem_alloc2(&tmem_base_sh, 512);
    if (tid == 0) {
        umma::mbar_init(&bar[0], 1);
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tmem_base_sh;
    if (warp < 4) {
        umma::tmem_st32_fill(tmem + ((warp * 32) << 16) + 256, 0x7F7F7F7Fu);
        umma::tmem_st32_fill(tmem + ((warp * 32) << 16) + 384, 0x80808080u);
        umma::tmem_st_wait();
    }
    umma::fence_before_sync();
    umma::cluster_sync();
    umma::fence_after_sync();
    const long long t0 = clock64();
    if ((mode & 1) && rank == 0 && tid == 0) {
        constexpr uint32_t idesc = umma::idesc_mxf4(256, 256);
        const uint64_t d0 = umma::smem_desc_sw128(smem_u32(smem), 1024);
        int s = 0;
        for (int it = 0; it < mma_iters; ++it) {
            const uint64_t da = d0 + uint64_t((uint32_t(s) * STAGE) >> 4), db = da + (STAGE / 2 >> 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t sf = tmem + ((j & 1) ? 384 : 256);
                umma::mma_mxf4_pair(tmem, da + 2 * j, db + 2 * j, idesc, sf, sf, (it | j) ? 1u : 0u);
            }
            s = (s + 1 == STAGES) ? 0 : s + 1;
        }
        umma::mma_commit_pair(&bar[0], 0x3);
    }
    if ((mode & 2) && warp >= 4) {
        // 256 threads, two per row of a 128-row region, four swizzled 16-B chunks per operand
        const int r = (tid - 128) >> 1, g = tid & 1, rr = r & 7;
        uint4 v = make_uint4(tid, tid * 3, tid * 5, tid * 7);
        int s = 0;
        for (int it = 0; it < sts_iters; ++it) {
            uint8_t* row = smem + s * STAGE + (r >> 3) * 1024 + rr * 128;
#pragma unroll
            for (int op = 0; op < 2; ++op)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<uint4*>(row + op * (STAGE / 2) + (((4 * g + c) ^ rr) << 4)) = v;
            v.x += 1;
            s = (s + 1 == STAGES) ? 0 : s + 1;
        }
    }
    if ((mode & 2) && tid == 128) cycles[blockIdx.x * 2 + 1] = clock64() - t0;
    if ((mode & 1) && tid == 0) {
        umma::mbar_wait(&bar[0], 0);
        cycles[blockIdx.x * 2] = clock64() - t0;
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
    unsigned long long* cyc;
    cudaMalloc(&out, 4096);
    cudaMallocManaged(&cyc, 2 * 4096 * sizeof(unsigned long long));
    const int smem = STAGES * STAGE + 1024;
    cudaFuncSetAttribute(k_contend, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int mma_iters = 60000, sts_iters = 60000;  // ~18 ms: long enough for power limits to act
    for (int fill : {0, 1, 2})
    for (int mode : {1, 3}) {
        k_contend<<<sms, 384, smem>>>(out, 60, 60, mode, cyc, fill);
        cudaDeviceSynchronize();
        for (int i = 0; i < 2 * sms; ++i) cyc[i] = 0;
        cudaEventRecord(e0);
        k_contend<<<sms, 384, smem>>>(out, mma_iters, sts_iters, mode, cyc, fill);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double mma_c = 0, sts_c = 0;
        for (int i = 0; i < sms; i += 2) mma_c += cyc[2 * i];
        for (int i = 0; i < sms; ++i) sts_c += cyc[2 * i + 1];
        mma_c /= (sms / 2);
        sts_c /= sms;
        // per stage: MMA cycles (4 pair MMAs, M256 N256 K256) and STS bytes per cycle per SM (32 KB / stage)
        printf("{\"fill\": %d, \"mode\": %d, \"ms\": %.3f, \"Pbops\": %.3f, \"mma_cycles_per_stage\": %.1f, \"sts_bytes_per_cycle\": %.1f, \"err\": \"%s\"}\n",
               fill, mode, ms, double(sms / 2) * mma_iters * 2.0 * 256 * 256 * 256 / (ms * 1e-3) / 1e15, mma_c / mma_iters, sts_c > 0 ? 32768.0 * sts_iters / sts_c : 0.0,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
