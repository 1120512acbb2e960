// stream.cu -- the out-of-core driver: one device's output-row slab of
// C = A.B when A, B and C do not fit in HBM together (BASELINE configs[4],
// n = 2^20: 128 GiB per operand).
//
// Reference counterpart: the paper's host layer for the cubic product
// (disjoint output blocks per GPU, one host thread per
// output segment, no locks) and the K-split fold of cubic_blocked
// (engine.cpp:81-84), here the accumulate flag of the block-product kernel
// (K8).  Per device:
//   for each row tile I of the slab (TM rows):
//       upload A[I, :] once (resident panel, zero padded)
//       for each column tile J (TN columns):
//           for each K chunk (KC bits), double buffered on a copy stream:
//               H2D B[kc, J] (2-D copy from the host row-major B)
//               transpose to Bt chunk, multiply-accumulate into the C tile
//           D2H the C tile into its disjoint region of the host C
// The copy stream runs one chunk ahead of the compute stream (events gate
// buffer reuse), so PCIe transfers overlap the tensor-core work.  Tile sizes
// are chosen from the byte budget so the working set stays inside it.
#include <algorithm>
#include <string>

#include "common.cuh"

namespace bmmgpu {

int launch_transpose(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                     uint64_t kw, cudaStream_t stream);
int launch_cubic(int kernel, const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                 uint64_t ldc, uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate,
                 cudaStream_t stream, uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch);
int granularity(int kernel, uint64_t* gm, uint64_t* gn, uint64_t* gk);

namespace {

struct Plan {
    uint64_t TM, TN, KCw;  // rows, columns (multiples of the kernel tiles), K chunk in words
    uint64_t bytes;
};

Plan plan_tiles(uint64_t m, uint64_t n, uint64_t kw, uint64_t gm, uint64_t gn, uint64_t gkw, uint64_t budget) {
    Plan p{};
    // tall A panels: B is re-streamed once per row tile, so fewer, taller panels cut H2D
    p.TM = std::min<uint64_t>(round_up(m, gm), 131072);
    p.TN = std::min<uint64_t>(round_up(std::max<uint64_t>(n, 1), gn), 32768);
    p.KCw = std::min<uint64_t>(kw, round_up(2048, gkw));  // 128 Ki bits of K per chunk
    auto need = [&](const Plan& q) {
        const uint64_t a_panel = q.TM * kw * 8;
        const uint64_t b_chunk = q.KCw * 64 * (q.TN / 64) * 8;  // row-major B chunk
        const uint64_t bt_chunk = q.TN * q.KCw * 8;
        const uint64_t c_tile = q.TM * (q.TN / 64) * 8;
        return a_panel + 2 * (b_chunk + bt_chunk) + c_tile;
    };
    p.bytes = need(p);
    while (p.bytes > budget) {
        if (p.TN > gn && p.TN >= p.TM / 2)
            p.TN = std::max(gn, round_up(p.TN / 2, gn));
        else if (p.KCw > gkw && p.KCw * 64 > p.TN)
            p.KCw = std::max(gkw, round_up(p.KCw / 2, gkw));
        else if (p.TM > gm)
            p.TM = std::max(gm, round_up(p.TM / 2, gm));
        else if (p.TN > gn)
            p.TN = std::max(gn, round_up(p.TN / 2, gn));
        else if (p.KCw > gkw)
            p.KCw = std::max(gkw, round_up(p.KCw / 2, gkw));
        else
            break;
        p.bytes = need(p);
    }
    return p;
}

struct Events {
    cudaEvent_t e[8] = {};
    ~Events() {
        for (auto& x : e)
            if (x) cudaEventDestroy(x);
    }
};

}  // namespace

// Rows [row_begin, row_end) of C; host buffers in the reference layout.
int stream_cubic_slab(int device, uint64_t row_begin, uint64_t row_end, const uint64_t* A, const uint64_t* B,
                      uint64_t* C, uint64_t k, uint64_t n, bool gf2, int kernel, bool accumulate, uint64_t budget,
                      float* ms_out) {
    BMMGPU_CUDA_TRY(cudaSetDevice(device));
    const uint64_t m = row_end - row_begin;
    if (m == 0 || n == 0) return kOk;
    uint64_t gm, gn, gk;
    int st = granularity(kernel, &gm, &gn, &gk);
    if (st) return st;
    const uint64_t gkw = gk / 64;
    const uint64_t ka = ceil_div(k, 64), nb = ceil_div(n, 64);
    const uint64_t kw = round_up(std::max<uint64_t>(ka, 1), gkw);
    if (budget == 0) {
        size_t free_b = 0, total_b = 0;
        BMMGPU_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
        budget = uint64_t(double(free_b) * 0.9);
    }
    const Plan P = plan_tiles(m, n, kw, gm, gn, gkw, budget);
    if (P.bytes > budget) {
        set_error("out-of-core driver: even the smallest tiles (" + std::to_string(P.bytes) +
                  " B) exceed the device budget of " + std::to_string(budget) + " B");
        return kEinval;
    }
    // K chunks must tile kw exactly: round kw up to the chunk (extra words are zero).
    const uint64_t kwc = round_up(kw, P.KCw);
    const uint64_t TNw = P.TN / 64;
    const uint64_t KC = P.KCw * 64;

    cudaStream_t cs, xs;  // compute, copy
    BMMGPU_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    BMMGPU_CUDA_TRY(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
    struct Guard {
        cudaStream_t a, b;
        ~Guard() {
            cudaStreamDestroy(a);
            cudaStreamDestroy(b);
        }
    } guard{cs, xs};
    Events ev;  // 0,1 b_ready[buf]; 2,3 buf_free[buf]; 4 a_ready; 5 start; 6 stop; 7 a_free
    for (int i = 0; i < 8; ++i) BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev.e[i], i == 5 || i == 6 ? 0 : cudaEventDisableTiming));
    DeviceBuffer dA, dB[2], dBt[2], dC;
    if ((st = dA.alloc(P.TM * kwc * 8, cs)) || (st = dB[0].alloc(KC * TNw * 8, cs)) ||
        (st = dB[1].alloc(KC * TNw * 8, cs)) || (st = dBt[0].alloc(P.TN * P.KCw * 8, cs)) ||
        (st = dBt[1].alloc(P.TN * P.KCw * 8, cs)) || (st = dC.alloc(P.TM * TNw * 8, cs)))
        return st;
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(cs));  // buffers exist before the copy stream touches them
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[5], cs));
    // both buffers start free
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[2], cs));
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[3], cs));
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[7], cs));
    uint64_t chunk_no = 0;
    for (uint64_t r0 = 0; r0 < m; r0 += P.TM) {
        const uint64_t rows = std::min(P.TM, m - r0);
        // resident A panel: rows r0.., all of K (zero padded), on the copy stream
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(xs, ev.e[7], 0));
        BMMGPU_CUDA_TRY(cudaMemsetAsync(dA.p, 0, P.TM * kwc * 8, xs));
        count_launch();
        if (ka > 0)
            BMMGPU_CUDA_TRY(memcpy2d_counted(dA.p, kwc * 8, A + (row_begin + r0) * ka, ka * 8, ka * 8, rows,
                                              cudaMemcpyHostToDevice, xs));
        BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[4], xs));
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[4], 0));
        for (uint64_t c0 = 0; c0 < n; c0 += P.TN) {
            const uint64_t cols = std::min(P.TN, n - c0);
            const uint64_t cw0 = c0 / 64, cwn = ceil_div(cols, 64);
            if (accumulate) {
                BMMGPU_CUDA_TRY(cudaMemsetAsync(dC.p, 0, P.TM * TNw * 8, cs));
                BMMGPU_CUDA_TRY(memcpy2d_counted(dC.p, TNw * 8, C + (row_begin + r0) * nb + cw0, nb * 8, cwn * 8,
                                                  rows, cudaMemcpyHostToDevice, cs));
                count_launch();
            }
            const uint64_t n_chunks = kwc / P.KCw;
            for (uint64_t q = 0; q < n_chunks; ++q, ++chunk_no) {
                const int buf = int(chunk_no & 1);
                const uint64_t k0 = q * KC;
                const uint64_t krows = k0 < k ? std::min<uint64_t>(KC, k - k0) : 0;
                // copy stream: wait until compute released this buffer, then fetch B[k0.., c0..]
                BMMGPU_CUDA_TRY(cudaStreamWaitEvent(xs, ev.e[2 + buf], 0));
                if (krows > 0)
                    BMMGPU_CUDA_TRY(memcpy2d_counted(dB[buf].p, TNw * 8, B + k0 * nb + cw0, nb * 8, cwn * 8, krows,
                                                      cudaMemcpyHostToDevice, xs));
                BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[buf], xs));
                // compute stream: transpose the chunk and fold its product into the C tile
                BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[buf], 0));
                if ((st = launch_transpose(dB[buf].u(), TNw, krows, cols, dBt[buf].u(), P.TN, P.KCw, cs))) return st;
                if ((st = launch_cubic(kernel, dA.u() + q * P.KCw, kwc, dBt[buf].u(), P.KCw, dC.u(), TNw,
                                       round_up(rows, gm), P.TN, P.KCw, gf2, accumulate || q > 0, cs, 1, 0, 0, 0)))
                    return st;
                BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[2 + buf], cs));
            }
            BMMGPU_CUDA_TRY(memcpy2d_counted(C + (row_begin + r0) * nb + cw0, nb * 8, dC.p, TNw * 8, cwn * 8, rows,
                                              cudaMemcpyDeviceToHost, cs));
        }
        BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[7], cs));  // the A panel may be replaced
    }
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[6], cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(xs));
    if (ms_out) cudaEventElapsedTime(ms_out, ev.e[5], ev.e[6]);
    return kOk;
}

// K-outer pipelined form for slabs whose C fits in HBM (the common in-core case
// of the host API): K is cut into chunks; while the tensor cores fold chunk q
// into the resident C, the copy stream uploads A[:, q+1] and B[q+1, :].  The
// transfer of the inputs therefore hides behind the product instead of
// preceding it; only the first chunk and the final D2H of C are exposed.
int stream_kouter_slab(int device, uint64_t row_begin, uint64_t row_end, const uint64_t* A, const uint64_t* B,
                       uint64_t* C, uint64_t k, uint64_t n, bool gf2, int kernel, bool accumulate, uint64_t budget,
                       float* ms_out, int chunks) {
    BMMGPU_CUDA_TRY(cudaSetDevice(device));
    const uint64_t m = row_end - row_begin;
    if (m == 0 || n == 0) return kOk;
    uint64_t gm, gn, gk;
    int st = granularity(kernel, &gm, &gn, &gk);
    if (st) return st;
    const uint64_t gkw = gk / 64;
    const uint64_t ka = ceil_div(k, 64), nb = ceil_div(n, 64);
    const uint64_t m_pad = round_up(m, gm), n_pad = round_up(n, gn), cw = n_pad / 64;
    const uint64_t kw = round_up(std::max<uint64_t>(ka, 1), gkw);
    uint64_t KCw = round_up(ceil_div(kw, uint64_t(std::max(chunks, 1))), gkw);
    auto need = [&](uint64_t kc) { return (m_pad * cw + 2 * (m_pad * kc + kc * 64 * nb + n_pad * kc)) * 8; };
    while (need(KCw) > budget && KCw > gkw) KCw = round_up(KCw / 2, gkw);
    if (need(KCw) > budget) {
        set_error("K-outer driver: the resident C slab does not fit the device budget");
        return kEinval;
    }
    const uint64_t KC = KCw * 64, n_chunks = ceil_div(kw, KCw);

    cudaStream_t cs, xs;
    BMMGPU_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    BMMGPU_CUDA_TRY(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
    struct Guard {
        cudaStream_t a, b;
        ~Guard() {
            cudaStreamDestroy(a);
            cudaStreamDestroy(b);
        }
    } guard{cs, xs};
    Events ev;  // 0,1 ready[buf]; 2,3 free[buf]; 5 start; 6 stop
    for (int i = 0; i < 8; ++i)
        BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev.e[i], i == 5 || i == 6 ? 0 : cudaEventDisableTiming));
    DeviceBuffer dC, dA[2], dB[2], dBt[2];
    if ((st = dC.alloc(m_pad * cw * 8, cs))) return st;
    for (int b = 0; b < 2; ++b)
        if ((st = dA[b].alloc(m_pad * KCw * 8, cs)) || (st = dB[b].alloc(KC * nb * 8, cs)) ||
            (st = dBt[b].alloc(n_pad * KCw * 8, cs)))
            return st;
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(cs));
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[5], cs));
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[2], cs));
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[3], cs));
    if (accumulate) {
        BMMGPU_CUDA_TRY(cudaMemsetAsync(dC.p, 0, m_pad * cw * 8, cs));
        BMMGPU_CUDA_TRY(memcpy2d_counted(dC.p, cw * 8, C + row_begin * nb, nb * 8, nb * 8, m,
                                          cudaMemcpyHostToDevice, cs));
        count_launch();
    }
    for (uint64_t q = 0; q < n_chunks; ++q) {
        const int buf = int(q & 1);
        const uint64_t w0 = q * KCw;
        const uint64_t aw = w0 < ka ? std::min<uint64_t>(KCw, ka - w0) : 0;  // A words of this chunk
        const uint64_t k0 = q * KC;
        const uint64_t krows = k0 < k ? std::min<uint64_t>(KC, k - k0) : 0;
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(xs, ev.e[2 + buf], 0));
        BMMGPU_CUDA_TRY(cudaMemsetAsync(dA[buf].p, 0, m_pad * KCw * 8, xs));
        count_launch();
        if (aw > 0)
            BMMGPU_CUDA_TRY(memcpy2d_counted(dA[buf].p, KCw * 8, A + row_begin * ka + w0, ka * 8, aw * 8, m,
                                              cudaMemcpyHostToDevice, xs));
        if (krows > 0)
            BMMGPU_CUDA_TRY(memcpy_counted(dB[buf].p, B + k0 * nb, krows * nb * 8, cudaMemcpyHostToDevice, xs));
        BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[buf], xs));
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[buf], 0));
        if ((st = launch_transpose(dB[buf].u(), nb, krows, n, dBt[buf].u(), n_pad, KCw, cs))) return st;
        if ((st = launch_cubic(kernel, dA[buf].u(), KCw, dBt[buf].u(), KCw, dC.u(), cw, m_pad, n_pad, KCw, gf2,
                               accumulate || q > 0, cs, 1, 0, 0, 0)))
            return st;
        BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[2 + buf], cs));
    }
    BMMGPU_CUDA_TRY(memcpy2d_counted(C + row_begin * nb, nb * 8, dC.p, cw * 8, nb * 8, m, cudaMemcpyDeviceToHost,
                                      cs));
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[6], cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(xs));
    if (ms_out) cudaEventElapsedTime(ms_out, ev.e[5], ev.e[6]);
    return kOk;
}

}  // namespace bmmgpu
