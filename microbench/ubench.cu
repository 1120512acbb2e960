// Throughput microbenchmarks for the bit-product building blocks on sm_100a.
// Each kernel runs a fixed instruction mix from registers (or a resident SMEM
// tile for tcgen05) so the measured rate is the pipe's issue rate, not memory.
//   lop3   : acc ^= a & b        (32-bit LOP3, alu pipe)
//   popc   : acc += popc(a)      (POPC)
//   bmma   : mma.sync m16n8k256 b1 and.popc  (legacy tensor path)
//   imma   : mma.sync m16n8k32 s8            (legacy tensor path)
//   umma_i8: tcgen05.mma kind::i8 M=128 N=256 K=32 (5th-gen tensor core)
//   umma_f4: tcgen05.mma kind::f8f6f4 e2m1 M=128 N=256 K=32
//   umma_mxf4: tcgen05.mma kind::mxf4 block_scale M=128 N=256 K=64
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void k_lop3(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[8], b[8], acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i); b[i] = seed ^ (i * 77 + threadIdx.x); }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("lop3.b32 %0, %1, %2, %0, 0x6A;" : "+r"(acc[i][j]) : "r"(a[i]), "r"(b[j]));
    // 0x6A = (a & b) ^ c
  }
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) r ^= acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_popc(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[16], acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { a[i] = seed * (threadIdx.x + i); acc[i] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint32_t p;
      asm volatile("popc.b32 %0, %1;" : "=r"(p) : "r"(a[i] ^ acc[i]));
      acc[i] += p;
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_bmma(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[4], b[2];
  int32_t c[8][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + i);
  b[0] = seed ^ threadIdx.x; b[1] = seed + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
          "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  int32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) r ^= c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_imma(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[4], b[2];
  int32_t c[8][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + i);
  b[0] = seed ^ threadIdx.x; b[1] = seed + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 "
          "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  int32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) r ^= c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no-swizzle canonical layout: core matrix = 8 rows x 16 B.
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) k_umma(uint32_t* out, int iters) {
  // A: 128 rows x 128 B, B: 256 rows x 128 B  (K-major, no swizzle)
  __shared__ __align__(1024) uint8_t sA[128 * 64];
  __shared__ __align__(1024) uint8_t sB[256 * 64];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) uint8_t sSF[1024];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) sA[i] = (KIND == 0) ? (i & 1) : ((i & 1) ? 0x22 : 0x02);
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) sB[i] = (KIND == 0) ? ((i >> 1) & 1) : 0x22;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sSF[i] = 127;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    // LBO: next 16B K-chunk = 128 B (8 rows x 16 B core matrix); SBO: next 8 rows = 8*16*8 = 1024 B
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    uint32_t idesc = 0;
    if (KIND == 0) {
      // kind::i8: c_format S32 (2) bits[4,6), a/b format unsigned (0), K-major
      idesc = (2u << 4) | (0u << 7) | (0u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    } else if (KIND == 1) {
      // kind::f8f6f4 e2m1 (5), c F32 (1)
      idesc = (1u << 4) | (5u << 7) | (5u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    } else {
      // kind::mxf4 block scaled: a/b format E2M1=1, scale_format UE8M0 (bit 23 = 1)
      idesc = (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        // each instruction consumes 32 B of K (i8/f8f6f4 containers) -> 2 core-matrix columns
        const uint64_t da = make_desc(a0 + k * 256, 128, 512);
        const uint64_t db = make_desc(b0 + k * 256, 128, 512);
        const uint32_t acc = (it | k) ? 1u : 0u;
        if (KIND == 0) {
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
              ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        } else if (KIND == 1) {
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;}"
              ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        } else {
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::mxf4.block_scale [%0], %1, %2, %3, [%5], [%6], p;}"
              ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(tmem + 256), "r"(tmem + 384));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  __syncwarp();
  // wait for MMA completion
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
          : "=r"(done) : "r"(smem_u32(&bar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v0;
  // warp w reads lanes 32w..32w+31, column 0
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v0) : "r"(tmem + ((warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  out[blockIdx.x * blockDim.x + threadIdx.x] = v0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d}\n", prop.name, sms, clk_khz);
  uint32_t* out;
  CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto run = [&](const char* name, auto launch, double ops_per_launch, const char* unit) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    const double rate = ops_per_launch * 5 / (ms * 1e-3);
    printf("{\"bench\": \"%s\", \"ms\": %.3f, \"rate\": %.4e, \"unit\": \"%s\", \"err\": \"%s\"}\n", name, ms / 5, rate, unit,
           cudaGetErrorString(err));
    fflush(stdout);
  };
  const int threads = 512, blocks = sms * 4;
  {
    const int iters = 20000;
    run("lop3", [&] { k_lop3<<<blocks, threads>>>(out, 12345u, iters); },
        double(blocks) * threads * iters * 64, "lop3_lanes/s");
  }
  {
    const int iters = 20000;
    run("popc", [&] { k_popc<<<blocks, threads>>>(out, 12345u, iters); },
        double(blocks) * threads * iters * 16, "popc_lanes/s");
  }
  {
    const int iters = 4000;
    // bit-MACs per mma: 16*8*256 = 32768 per warp-instruction
    run("bmma_m16n8k256", [&] { k_bmma<<<blocks, threads>>>(out, 12345u, iters); },
        double(blocks) * (threads / 32) * iters * 8 * 32768.0, "bitMAC/s");
  }
  {
    const int iters = 4000;
    run("imma_m16n8k32", [&] { k_imma<<<blocks, threads>>>(out, 12345u, iters); },
        double(blocks) * (threads / 32) * iters * 8 * (16 * 8 * 32.0), "MAC/s");
  }
  {
    const int iters = 2000;
    run("umma_i8_m128n256k32", [&] { k_umma<0><<<sms, 128>>>(out, iters); },
        double(sms) * iters * 2 * (128.0 * 256 * 32), "MAC/s");
    run("umma_f8f6f4_e2m1_m128n256k32", [&] { k_umma<1><<<sms, 128>>>(out, iters); },
        double(sms) * iters * 2 * (128.0 * 256 * 32), "MAC/s");
    run("umma_mxf4_m128n256k64", [&] { k_umma<2><<<sms, 128>>>(out, iters); },
        double(sms) * iters * 2 * (128.0 * 256 * 64), "MAC/s");
  }
  return 0;
}
