// Per-SM bandwidth of a two-level expand-shaped pass confined to a few SMs (dev helper):
// each thread reads 16 x 16 B (the 16 sub-blocks of a parent at one position) and writes
// 49 x 16 B (its 49 grandchildren), like alt.cu's expand_pass_kernel<2,2>; grid = k SMs x
// 2 resident blocks.  Prints GB/s (read + write) per grid size, alone on an idle GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench/side_bw microbench/side_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) expand_like(const uint4* __restrict__ in, uint4* __restrict__ out,
                                                   uint64_t positions, uint64_t sub_stride_in, uint64_t sub_stride_out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < positions;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint4 x[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) x[q] = in[q * sub_stride_in + i];
#pragma unroll
        for (int h = 0; h < 49; ++h) {
            uint4 v = x[h % 16];
            v.x ^= x[(h + 3) % 16].x;
            v.y ^= x[(h + 5) % 16].y;
            out[h * sub_stride_out + i] = v;
        }
    }
}

int main() {
    const uint64_t positions = uint64_t(1) << 21;  // 32 MiB per sub-block of 16-byte vectors
    uint4 *in, *out;
    cudaMalloc(&in, 16 * positions * sizeof(uint4));
    cudaMalloc(&out, 49 * positions * sizeof(uint4));
    cudaMemset(in, 1, 16 * positions * sizeof(uint4));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int ks[] = {1, 2, 4, 8, 16, 148};
    for (int k : ks) {
        const int grid = k * 2;
        const uint64_t pos = k >= 148 ? positions : positions / 8;  // keep small runs short
        expand_like<<<grid, 256>>>(in, out, pos, positions, positions);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) expand_like<<<grid, 256>>>(in, out, pos, positions, positions);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = 3.0 * double(pos) * 65 * 16;
        printf("{\"sms\": %d, \"grid\": %d, \"GBps\": %.1f, \"GBps_per_sm\": %.1f}\n", k, grid, bytes / (ms * 1e6),
               bytes / (ms * 1e6) / k);
    }
    return 0;
}
