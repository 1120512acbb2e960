// alt_tiles.cu -- the out-of-core fast GF(2) product (BASELINE configs[4]:
// operands far larger than HBM, streamed from host memory): C is cut into b x b output
// tiles, b a power of two (131072 by default), and
//
//     C[I, J] = XOR_K  A[I, K] . B[K, J]
//
// where every block product is the device-resident alternative-basis recursion
// (alt_multiply_device, the reference's multiply with the basis changes folded into the
// expand / compress coefficients) and the XOR is the reference's fold of partial products
// (engine.cpp:81-84).  This is the paper's host layer for products beyond accelerator
// memory (output segments owned by one host thread each, no locks)
// with the fast algorithm inside each block product.
//
// Per device (row panels I dealt round robin over the devices): the C row panel I (b x n
// bits) stays in HBM; for each K the A tile goes up once, for each J the B tile goes up
// on a copy stream while the previous block product runs (double buffers), is transposed
// to Bt, multiplied, and XOR-folded into its slot of the panel; the finished panel goes
// home in one contiguous copy.  Traffic per block product: 2 b^2/8 bytes up (A amortised
// over the J sweep), against ~2 b^3 / 14e15 s of tensor work -- compute-bound for b >= 2^16.
#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "bmmgpu.h"
#include "common.cuh"

namespace bmmgpu {

int launch_transpose(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                     uint64_t kw, cudaStream_t s);
int alt_multiply_device(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                        uint64_t ldc, uint64_t n, int algo, int e, int e_serial, int kernel, cudaStream_t s);
int choose_serial_levels(uint64_t n, int e);
int alt_levels(uint64_t n, int leaf_log2);
int resolve_kernel(int kernel);

// Tile side for an n x n out-of-core fast product (BMMGPU_ALT_TILE = log2 forces it).
uint64_t alt_tile_side(uint64_t n) {
    if (const char* env = getenv("BMMGPU_ALT_TILE")) {
        const int l = atoi(env);
        if (l >= 8 && l < 40) return std::min<uint64_t>(n, uint64_t(1) << l);
    }
    return std::min<uint64_t>(n / 2, uint64_t(1) << 17);
}

// Output row panels [p0, p1) of b x b tiles (b = 0: alt_tile_side), dealt round robin over
// `devs`.  Only the rows of A and C inside those panels are touched.
int alt_multiply_tiles(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int algo,
                       const std::vector<int>& devs, int kernel, int leaf_log2, double* timing_ms, uint64_t b,
                       uint64_t p0, uint64_t p1) {
    if (b == 0) b = alt_tile_side(n);
    if (b < 256 || (b & (b - 1)) || n % b) {
        set_error("alt tiles: the tile side must be a power of two >= 256 dividing n");
        return kEinval;
    }
    const uint64_t w = n / 64, bw = b / 64, T = n / b;
    if (p1 == 0 || p1 > T) p1 = T;
    if (p0 >= p1) return kOk;
    kernel = resolve_kernel(kernel);
    const int e = alt_levels(b, leaf_log2);
    const uint32_t G = uint32_t(std::min<uint64_t>(devs.size(), p1 - p0));
    std::vector<int> status(G, kOk);
    std::vector<std::string> errors(G);
    std::vector<float> ms(G, 0.f);
    void* stats = call_stats();
    auto work = [&](uint32_t g) -> int {
        BMMGPU_CUDA_TRY(cudaSetDevice(devs[g]));
        StreamSet ss;  // 0 compute, 1 uploads
        if (int r = ss.acquire(2)) return r;
        const cudaStream_t s = ss[0], h = ss[1];
        DeviceBuffer dC, dA[2], dB[2], dBt, dP;
        struct Events {
            cudaEvent_t up_a[2] = {}, up_b[2] = {}, done[4] = {}, t0 = nullptr, t1 = nullptr;
            ~Events() {
                for (auto x : up_a) if (x) cudaEventDestroy(x);
                for (auto x : up_b) if (x) cudaEventDestroy(x);
                for (auto x : done) if (x) cudaEventDestroy(x);
                if (t0) cudaEventDestroy(t0);
                if (t1) cudaEventDestroy(t1);
            }
        } ev;
        StreamDrain drain{{s, h, nullptr, nullptr}};
        for (int i = 0; i < 2; ++i) {
            BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev.up_a[i], cudaEventDisableTiming));
            BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev.up_b[i], cudaEventDisableTiming));
        }
        for (auto& x : ev.done) BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        BMMGPU_CUDA_TRY(cudaEventCreate(&ev.t0));
        BMMGPU_CUDA_TRY(cudaEventCreate(&ev.t1));
        int r;
        const uint64_t tile_bytes = b * bw * 8;
        if ((r = dC.alloc(b * w * 8, s)) || (r = dA[0].alloc(tile_bytes, s)) || (r = dA[1].alloc(tile_bytes, s)) ||
            (r = dB[0].alloc(tile_bytes, s)) || (r = dB[1].alloc(tile_bytes, s)) ||
            (r = dBt.alloc(round_up(b, 256) * bw * 8, s)) || (r = dP.alloc(tile_bytes, s)))
            return r;
        // the block products' depth-first level count, with this driver's buffers in place
        BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
        const int e_serial = e > 0 ? choose_serial_levels(b, e) : 0;
        BMMGPU_CUDA_TRY(cudaEventRecord(ev.t0, s));
        uint64_t q = 0;  // block products issued on this device
        for (uint64_t I = p0 + g; I < p1; I += G) {
            BMMGPU_CUDA_TRY(cudaMemsetAsync(dC.p, 0, b * w * 8, s));
            count_launch();
            for (uint64_t K = 0; K < T; ++K) {
                const int ka = int(K & 1);
                for (uint64_t J = 0; J < T; ++J, ++q) {
                    const int kb = int(q & 1);
                    // the upload stream may overwrite a buffer once the product that read it
                    // two steps ago is done
                    if (q >= 2) BMMGPU_CUDA_TRY(cudaStreamWaitEvent(h, ev.done[(q - 2) & 3], 0));
                    if (J == 0) {
                        BMMGPU_CUDA_TRY(memcpy2d_counted(dA[ka].p, bw * 8, A + I * b * w + K * bw, w * 8, bw * 8, b,
                                                         cudaMemcpyHostToDevice, h));
                        BMMGPU_CUDA_TRY(cudaEventRecord(ev.up_a[ka], h));
                    }
                    BMMGPU_CUDA_TRY(memcpy2d_counted(dB[kb].p, bw * 8, B + K * b * w + J * bw, w * 8, bw * 8, b,
                                                     cudaMemcpyHostToDevice, h));
                    BMMGPU_CUDA_TRY(cudaEventRecord(ev.up_b[kb], h));
                    if (J == 0) BMMGPU_CUDA_TRY(cudaStreamWaitEvent(s, ev.up_a[ka], 0));
                    BMMGPU_CUDA_TRY(cudaStreamWaitEvent(s, ev.up_b[kb], 0));
                    if ((r = launch_transpose(dB[kb].u(), bw, b, b, dBt.u(), round_up(b, 256), bw, s))) return r;
                    if (e == 0)
                        r = bmmgpu_dev_cubic(dA[ka].u(), bw, dBt.u(), bw, dC.u() + J * bw, w, b, b, bw, BMMGPU_GF2_XOR_AND,
                                             kernel, 1, s);
                    else if (!(r = alt_multiply_device(dA[ka].u(), bw, dBt.u(), bw, dP.u(), bw, b, algo, e, e_serial,
                                                       kernel, s)))
                        r = bmmgpu_dev_fold(dC.u() + J * bw, w, dP.u(), bw, b, bw, BMMGPU_GF2_XOR_AND, s);
                    if (r) return r;
                    BMMGPU_CUDA_TRY(cudaEventRecord(ev.done[q & 3], s));
                }
            }
            BMMGPU_CUDA_TRY(memcpy_counted(C + I * b * w, dC.p, b * w * 8, cudaMemcpyDeviceToHost, s));
        }
        BMMGPU_CUDA_TRY(cudaEventRecord(ev.t1, s));
        BMMGPU_CUDA_TRY(cudaStreamSynchronize(s));
        cudaEventElapsedTime(&ms[g], ev.t0, ev.t1);
        return kOk;
    };
    std::vector<std::thread> threads;
    for (uint32_t g = 0; g < G; ++g)
        threads.emplace_back([&, g] {
            adopt_call_stats(stats);
            if ((status[g] = work(g))) errors[g] = bmmgpu_last_error();
            adopt_call_stats(nullptr);
        });
    for (auto& t : threads) t.join();
    float worst = 0.f;
    for (uint32_t g = 0; g < G; ++g) {
        if (status[g]) {
            set_error("device " + std::to_string(devs[g]) + ": " + errors[g]);
            return status[g];
        }
        worst = std::max(worst, ms[g]);
    }
    if (timing_ms) *timing_ms = worst;
    return kOk;
}

}  // namespace bmmgpu

extern "C" int bmmgpu_multiply_panels(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int32_t algo,
                                      int32_t tile_log2, uint64_t panel_begin, uint64_t panel_end,
                                      const bmmgpu_opts* opts) {
    bmmgpu::reset_call_stats();
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        bmmgpu::set_error("no CUDA device available; the bit-matrix engine has no CPU fallback");
        return bmmgpu::kEnodev;
    }
    if (algo < BMMGPU_ALGO_STRASSEN_WINOGRAD || algo > BMMGPU_ALGO_ALT_CHAINING) {
        bmmgpu::set_error("multiply_panels: a fast algorithm is required");
        return bmmgpu::kEinval;
    }
    if (n < 64 || (n & (n - 1))) {
        bmmgpu::set_error("fast algorithms need n = 64 * 2^k");
        return bmmgpu::kEshape;
    }
    const uint32_t mask = opts && opts->device_mask ? opts->device_mask : 1u;
    std::vector<int> devs;
    for (int g = 0; g < 32; ++g)
        if (mask >> g & 1) {
            if (g >= count) {
                bmmgpu::set_error("device_mask names a missing device");
                return bmmgpu::kEinval;
            }
            devs.push_back(g);
        }
    const uint64_t b = tile_log2 > 0 ? uint64_t(1) << tile_log2 : 0;
    return bmmgpu::alt_multiply_tiles(A, B, C, n, algo, devs, opts ? opts->kernel : 0, opts ? opts->leaf_log2 : 0,
                                      opts ? opts->timing_ms : nullptr, b, panel_begin, panel_end);
}
