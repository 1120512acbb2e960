// Issue rate of the CTA-pair kind::mxf4 MMA with operand A in shared memory (SS, the
// form cubic_umma2.cu uses) or in tensor memory (TS), at N = 256 and N = 128, no
// producers: MACs per SM clock, from clock64 around the issue loop of the leader CTA.
// Also a layout check of the TS form: A row r of TMEM holds one e2m1 1.0 at K element
// (r * 7) % 64, B row n (smem, 128-byte swizzle) one 1.0 at K element n % 64, so
// D[r][n] = 1 iff (r * 7) % 64 == n % 64 under the column/nibble order assumed for A.
#include <cstdio>
#include "../paper_1909_01554_b200/csrc/umma.cuh"

using namespace bmmgpu;

constexpr int STAGE = 32768;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_ts(unsigned long long* out, int iters, int N, int ts, int check, uint32_t* dout) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base_sh;
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = umma::cluster_ctarank();
    if (check) {
        // B region (second half): row n (0..127) one-hot at K element n % 64 (+ 64 * (n / 64) ignored)
        for (int i = tid; i < STAGE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
        __syncthreads();
        if (tid < 128) {
            const int n = tid, k = n % 64, byte = k / 2, nib = k % 2;
            const int chunk = byte / 16, off = byte % 16;
            uint8_t* row = smem + STAGE / 2 + (n >> 3) * 1024 + (n & 7) * 128;
            row[((chunk ^ (n & 7)) << 4) + off] = uint8_t(0x2 << (4 * nib));
        }
    } else {
        for (int i = tid; i < STAGE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22222222u;
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
    // A in TMEM at columns [256, 288): 32 columns = 256 e2m1 elements per row
    if (check) {
        const int r = warp * 32 + lane, k = (r * 7) % 64;
        for (int c = 0; c < 32; ++c) {
            uint32_t v = 0;
            if (c == k / 8) v = 0x2u << (4 * (k % 8));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lb + 256 + c), "r"(v));
        }
    } else {
        umma::tmem_st32_fill(tmem + lb + 256, 0x22222222u);
    }
    umma::tmem_st_wait();
    umma::fence_before_sync();
    umma::cluster_sync();
    umma::fence_after_sync();
    long long c0 = 0, c1 = 0;
    unsigned long long g0 = 0, g1 = 0;
    if (rank == 0 && tid == 0) {
        const uint32_t idesc = umma::idesc_mxf4(256, N);
        const uint32_t base = smem_u32(smem);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        c0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t sf = tmem + ((j & 1) ? 488 : 480);
                const uint64_t bd = umma::smem_desc_sw128(base + STAGE / 2 + 32 * j, 1024);
                const uint32_t acc = (it | j) ? 1u : 0u;
                if (ts) {
                    asm volatile(
                        "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale [%0], [%1], %2, %3, [%5], [%6], p;}" ::"r"(tmem),
                        "r"(tmem + 256 + 8 * j), "l"(bd), "r"(idesc), "r"(acc), "r"(sf), "r"(sf));
                } else {
                    umma::mma_mxf4_pair(tmem, umma::smem_desc_sw128(base + 32 * j, 1024), bd, idesc, sf, sf, acc);
                }
                if (check) break;  // one K = 64 MMA
            }
            if (check) break;
        }
        umma::mma_commit_pair(&bar, 0x3);
        umma::mbar_wait(&bar, 0);
        c1 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        out[blockIdx.x * 2] = c1 - c0;
        out[blockIdx.x * 2 + 1] = g1 - g0;
    } else if (tid == 0) {
        umma::mbar_wait(&bar, 0);
    }
    __syncthreads();
    umma::fence_after_sync();
    if (check && blockIdx.x < 2) {
        // D rows of this CTA: lanes = rows 0..127, columns 0..N-1
        for (int c = 0; c < N; c += 16) {
            uint32_t v[16];
            umma::tmem_ld16(tmem + lb + c, v);
            umma::tmem_ld_wait();
            for (int i = 0; i < 16; ++i)
                dout[(blockIdx.x * 128 + warp * 32 + lane) * 256 + c + i] = __float_as_uint(__uint_as_float(v[i]));
        }
    }
    umma::fence_before_sync();
    umma::cluster_sync();
    if (warp == 0) {
        umma::fence_after_sync();
        umma::tmem_dealloc2(tmem, 512);
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* out;
    cudaMalloc(&out, 8 * 2 * 256);
    uint32_t* dout;
    cudaMalloc(&dout, 256 * 256 * 4);
    const int smem = STAGE + 1024;
    cudaFuncSetAttribute(k_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long h[2 * 256];
    for (int ts : {0, 1})
        for (int N : {256, 128}) {
            const int iters = 20000;
            k_ts<<<sms, 128, smem>>>(out, 100, N, ts, 0, dout);
            k_ts<<<sms, 128, smem>>>(out, iters, N, ts, 0, dout);
            cudaDeviceSynchronize();
            cudaMemcpy(h, out, sizeof(unsigned long long) * 2 * sms, cudaMemcpyDeviceToHost);
            double clk = 0, ns = 0;
            int n = 0;
            for (int b = 0; b < sms; b += 2, ++n) clk += h[2 * b], ns += h[2 * b + 1];
            clk /= n, ns /= n;
            const double macs_per_sm = double(iters) * 4 * (128.0 * N * 64);
            printf("{\"bench\": \"pair_mxf4\", \"A\": \"%s\", \"N\": %d, \"mac_per_clk_per_sm\": %.0f, \"mhz\": %.0f, "
                   "\"mac_per_s\": %.4e, \"err\": \"%s\"}\n",
                   ts ? "tmem" : "smem", N, macs_per_sm / clk, clk / ns * 1e3, macs_per_sm * sms / (ns * 1e-9),
                   cudaGetErrorString(cudaGetLastError()));
        }
    // TS layout check at N = 256
    for (int N : {256, 128}) {
        k_ts<<<2, 128, smem>>>(out, 1, N, 1, 1, dout);
        cudaDeviceSynchronize();
        static uint32_t d[256 * 256];
        cudaMemcpy(d, dout, sizeof(d), cudaMemcpyDeviceToHost);
        int bad = 0, ones = 0;
        for (int r = 0; r < 256; ++r)
            for (int c = 0; c < N; ++c) {
                const float v = *reinterpret_cast<float*>(&d[r * 256 + c]);
                // B row of output column c: CTA c / (N/2), row c % (N/2) of that CTA's region
                const int brow = c % (N / 2);
                const int want = ((r % 128) * 7) % 64 == brow % 64 ? 1 : 0;
                ones += v != 0.f;
                if (v != float(want)) {
                    if (bad < 5) printf("  N=%d D[%d][%d] = %g want %d\n", N, r, c, v, want);
                    ++bad;
                }
            }
        printf("{\"check\": \"ts_layout\", \"N\": %d, \"bad\": %d, \"nonzero\": %d, \"err\": \"%s\"}\n", N, bad, ones,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
