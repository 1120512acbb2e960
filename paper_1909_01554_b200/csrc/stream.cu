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
//       upload A[I, :] once (resident panel, zero padded; the next row tile's
//       panel is prefetched into a second buffer on its own stream)
//       for each column tile J (TN columns):
//           for each K chunk (KC bits), double buffered on a copy stream:
//               H2D B[kc, J] (2-D copy from the host row-major B)
//               transpose to Bt chunk, multiply-accumulate into the C tile
//           D2H the C tile into its disjoint region of the host C (double-
//           buffered C tiles on a third stream, behind the next tile's work)
// The copy streams run ahead of the compute stream (events gate buffer reuse),
// so PCIe transfers in both directions overlap the tensor-core work.  Tile
// sizes are chosen from the byte budget so the working set stays inside it.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

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
    // a second A panel (prefetch) only when there is a next row tile; two C tiles
    auto need = [&](const Plan& q) {
        const uint64_t a_panel = q.TM * kw * 8;
        const uint64_t b_chunk = q.KCw * 64 * (q.TN / 64) * 8;  // row-major B chunk
        const uint64_t bt_chunk = q.TN * q.KCw * 8;
        const uint64_t c_tile = q.TM * (q.TN / 64) * 8;
        return (m > q.TM ? 2 : 1) * a_panel + 2 * (b_chunk + bt_chunk) + 2 * c_tile;
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
    cudaEvent_t e[14] = {};
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
    // out-of-core calls run for seconds: a fresh (possibly blocking) query costs nothing here
    if (budget == 0) budget = uint64_t(double(device_free_bytes(true)) * 0.9);
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

    StreamSet ss;  // compute, B copies, A prefetch, C downloads
    if ((st = ss.acquire(4))) return st;
    const cudaStream_t cs = ss[0], xs = ss[1], as = ss[2], ds = ss[3];
    // 0,1 b_ready[buf]  2,3 b_free[buf]  4,5 a_ready[abuf]  6,7 a_free[abuf]
    // 8,9 c_done[cbuf]  10,11 c_free[cbuf]  12 start  13 stop
    Events ev;
    for (int i = 0; i < 14; ++i)
        BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev.e[i], i >= 12 ? 0 : cudaEventDisableTiming));
    const int n_abuf = m > P.TM ? 2 : 1;
    DeviceBuffer dA[2], dB[2], dBt[2], dC[2];
    StreamDrain drain{{cs, xs, as, ds}};
    for (int i = 0; i < n_abuf; ++i)
        if ((st = dA[i].alloc(P.TM * kwc * 8, cs))) return st;
    for (int i = 0; i < 2; ++i)
        if ((st = dB[i].alloc(KC * TNw * 8, cs)) || (st = dBt[i].alloc(P.TN * P.KCw * 8, cs)) ||
            (st = dC[i].alloc(P.TM * TNw * 8, cs)))
            return st;
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(cs));  // buffers exist before the copy streams touch them
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[12], cs));
    // every buffer starts free
    for (int i : {2, 3, 6, 7, 10, 11}) BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[i], cs));
    auto upload_a = [&](uint64_t r0, int abuf) -> int {
        const uint64_t rows = std::min(P.TM, m - r0);
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(as, ev.e[6 + abuf], 0));
        BMMGPU_CUDA_TRY(cudaMemsetAsync(dA[abuf].p, 0, P.TM * kwc * 8, as));
        count_launch();
        if (ka > 0)
            BMMGPU_CUDA_TRY(memcpy2d_counted(dA[abuf].p, kwc * 8, A + (row_begin + r0) * ka, ka * 8, ka * 8, rows,
                                             cudaMemcpyHostToDevice, as));
        BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[4 + abuf], as));
        return kOk;
    };
    uint64_t chunk_no = 0, tile_no = 0;
    if ((st = upload_a(0, 0))) return st;
    for (uint64_t r0 = 0, rt = 0; r0 < m; r0 += P.TM, ++rt) {
        const uint64_t rows = std::min(P.TM, m - r0);
        const int abuf = int(rt % n_abuf);
        // prefetch the next row tile's panel into the other buffer (a stream of its own)
        if (n_abuf == 2 && r0 + P.TM < m && (st = upload_a(r0 + P.TM, abuf ^ 1))) return st;
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[4 + abuf], 0));
        for (uint64_t c0 = 0; c0 < n; c0 += P.TN, ++tile_no) {
            const uint64_t cols = std::min(P.TN, n - c0);
            const uint64_t cw0 = c0 / 64, cwn = ceil_div(cols, 64);
            const int cbuf = int(tile_no & 1);
            BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[10 + cbuf], 0));  // its last download is done
            if (accumulate) {
                BMMGPU_CUDA_TRY(cudaMemsetAsync(dC[cbuf].p, 0, P.TM * TNw * 8, cs));
                BMMGPU_CUDA_TRY(memcpy2d_counted(dC[cbuf].p, TNw * 8, C + (row_begin + r0) * nb + cw0, nb * 8,
                                                 cwn * 8, rows, cudaMemcpyHostToDevice, cs));
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
                if ((st = launch_cubic(kernel, dA[abuf].u() + q * P.KCw, kwc, dBt[buf].u(), P.KCw, dC[cbuf].u(),
                                       TNw, round_up(rows, gm), P.TN, P.KCw, gf2, accumulate || q > 0, cs, 1, 0, 0,
                                       0)))
                    return st;
                BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[2 + buf], cs));
            }
            // the finished tile goes home on the download stream while the next tile computes
            BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[8 + cbuf], cs));
            BMMGPU_CUDA_TRY(cudaStreamWaitEvent(ds, ev.e[8 + cbuf], 0));
            BMMGPU_CUDA_TRY(memcpy2d_counted(C + (row_begin + r0) * nb + cw0, nb * 8, dC[cbuf].p, TNw * 8, cwn * 8,
                                             rows, cudaMemcpyDeviceToHost, ds));
            BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[10 + cbuf], ds));
        }
        BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[6 + abuf], cs));  // this A panel may be replaced
    }
    BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[10], 0));
    BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[11], 0));
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[13], cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(xs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(as));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(ds));
    if (ms_out) cudaEventElapsedTime(ms_out, ev.e[12], ev.e[13]);
    return kOk;
}

// K-outer pipelined form for slabs whose C fits in HBM (the common in-core case
// of the host API): K is cut into chunks; while the tensor cores fold chunk q
// into the resident C, the copy stream uploads A[:, q+1] and B[q+1, :].  The
// chunks grow geometrically (first 1/32 of K, then x5 ...): the exposed
// upload of the first chunk is small, and each later upload (bytes ~ (m + n) s)
// still hides behind the previous chunk's product (work ~ m n s).  The last
// chunk's product runs in row slices (shrinking geometrically) whose C rows go home
// on a download stream while the next slice computes, so only the last, small
// slice's D2H is exposed.
namespace {
std::vector<uint64_t> kouter_chunks(uint64_t kw, uint64_t gkw, uint64_t max_w, int chunks) {
    std::vector<uint64_t> c;
    if (chunks > 0) {  // fixed count (tests)
        const uint64_t w = std::min(max_w, round_up(ceil_div(kw, uint64_t(chunks)), gkw));
        for (uint64_t o = 0; o < kw; o += w) c.push_back(std::min(w, kw - o));
        return c;
    }
    uint64_t s = std::min(max_w, std::max(gkw, round_up(ceil_div(kw, 32), std::max<uint64_t>(gkw, 16))));
    // each upload (bytes ~ (m + n) s) must hide behind the previous chunk's product
    // (work ~ m n s): at n = 131072, 55 GB/s and ~8 Pbop/s that allows ~7x growth per
    // chunk; 5x keeps margin for slower links.  Fewer chunks = fewer accumulator drains.
    const uint64_t growth[] = {5, 5, 5};
    int g = 0;
    for (uint64_t o = 0; o < kw;) {
        uint64_t w = std::min(s, kw - o);
        if (kw - o - w < s / 2) w = kw - o;  // no sliver at the end
        w = std::min(w, max_w);
        c.push_back(w);
        o += w;
        s = std::min(max_w, round_up(s * growth[std::min(g++, 2)], gkw));
    }
    return c;
}

// Row slices of the last chunk, in launch order.  Slice i's rows go home while slice
// i + 1 computes, so the exposed tail is the last slice's download.  Compute per row
// over download per row is r = (2 n K_last / R) / (n / 8 / BW) = 16 K_last BW / R
// (~12 at n = 131072, 55 GB/s, 8 Pbop/s): when it is large the slices shrink
// geometrically (each <= shrink x the next, shrink = min(4, r / 2)) down to a last
// slice of ~1/128 of the rows; otherwise six equal slices.
std::vector<uint64_t> last_chunk_slices(uint64_t m_pad, uint64_t gm, uint64_t k_last) {
    std::vector<uint64_t> sl;
    const double r = 16.0 * double(k_last) * 55e9 / 8e15;
    double max_shrink = 4.0, last_div = 128.0;
    const char* mode = getenv("BMMGPU_KOUTER_SLICES");  // dev: "equal" = six equal slices, "S,D" = shrink, 1/last
    if (mode && strcmp(mode, "equal")) sscanf(mode, "%lf,%lf", &max_shrink, &last_div);
    const double shrink = std::min(max_shrink, r / 2);
    if (shrink < 1.5 || (mode && !strcmp(mode, "equal"))) {
        const uint64_t n_slices = std::max<uint64_t>(1, std::min<uint64_t>(6, m_pad / gm));
        const uint64_t slice = round_up(ceil_div(m_pad, n_slices), gm);
        for (uint64_t r0 = 0; r0 < m_pad; r0 += slice) sl.push_back(std::min(slice, m_pad - r0));
        return sl;
    }
    uint64_t total = 0, s = round_up(std::max<uint64_t>(gm, uint64_t(double(m_pad) / last_div)), gm);
    for (;;) {
        if (m_pad - total <= s) {
            sl.push_back(m_pad - total);
            break;
        }
        sl.push_back(s);
        total += s;
        s = round_up(uint64_t(double(s) * shrink), gm);
    }
    std::reverse(sl.begin(), sl.end());
    return sl;
}
}  // namespace

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
    // largest chunk the budget allows (double-buffered A, B and Bt chunks + resident C)
    uint64_t KCw = kw;  // the last, largest chunk may take most of K
    auto need = [&](uint64_t kc) { return (m_pad * cw + 2 * (m_pad * kc + kc * 64 * nb + n_pad * kc)) * 8; };
    while (need(KCw) > budget && KCw > gkw) KCw = round_up(KCw / 2, gkw);
    if (need(KCw) > budget) {
        set_error("K-outer driver: the resident C slab does not fit the device budget");
        return kEinval;
    }
    const std::vector<uint64_t> sched = kouter_chunks(kw, gkw, KCw, chunks);
    const uint64_t n_chunks = sched.size();

    StreamSet ss;  // compute, uploads, downloads
    if ((st = ss.acquire(3))) return st;
    const cudaStream_t cs = ss[0], xs = ss[1], ds = ss[2];
    Events ev;  // 0,1 ready[buf]; 2,3 free[buf]; 5 start; 6 stop; 8.. slice done
    for (int i = 0; i < 14; ++i)
        BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev.e[i], i == 5 || i == 6 ? 0 : cudaEventDisableTiming));
    DeviceBuffer dC, dA[2], dB[2], dBt[2];
    StreamDrain drain{{cs, xs, ds, nullptr}};
    if ((st = dC.alloc(m_pad * cw * 8, cs))) return st;
    for (int b = 0; b < 2; ++b)
        if ((st = dA[b].alloc(m_pad * KCw * 8, cs)) || (st = dB[b].alloc(KCw * 64 * nb * 8, cs)) ||
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
    // row slices of the last chunk (multiples of the kernel's row tile)
    const std::vector<uint64_t> slices = last_chunk_slices(m_pad, gm, sched.back() * 64);
    const uint64_t n_slices = slices.size();
    const char* xp_env = getenv("BMMGPU_KOUTER_XPOSE");
    const bool xpose_on_cs = xp_env && !strcmp(xp_env, "cs");
    uint64_t w0 = 0;
    for (uint64_t q = 0; q < n_chunks; ++q) {
        const int buf = int(q & 1);
        const uint64_t cwq = sched[q];  // words of this chunk
        const uint64_t aw = w0 < ka ? std::min<uint64_t>(cwq, ka - w0) : 0;  // A words of this chunk
        const uint64_t k0 = w0 * 64;
        const uint64_t krows = k0 < k ? std::min<uint64_t>(cwq * 64, k - k0) : 0;
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(xs, ev.e[2 + buf], 0));
        if (aw < cwq || m_pad > m) {  // zero pad rows / words (none when the chunk is dense)
            BMMGPU_CUDA_TRY(cudaMemsetAsync(dA[buf].p, 0, m_pad * cwq * 8, xs));
            count_launch();
        }
        if (aw > 0)
            BMMGPU_CUDA_TRY(memcpy2d_counted(dA[buf].p, cwq * 8, A + row_begin * ka + w0, ka * 8, aw * 8, m,
                                              cudaMemcpyHostToDevice, xs));
        if (krows > 0)
            BMMGPU_CUDA_TRY(memcpy_counted(dB[buf].p, B + k0 * nb, krows * nb * 8, cudaMemcpyHostToDevice, xs));
        // Later chunks' B transposes run on the copy stream, queued behind the running
        // product instead of between two products on the compute stream
        // (BMMGPU_KOUTER_XPOSE=cs: on the compute stream, dev A/B).
        if (q > 0 && !xpose_on_cs) {
            if ((st = launch_transpose(dB[buf].u(), nb, krows, n, dBt[buf].u(), n_pad, cwq, xs))) return st;
            BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[buf], xs));
            BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[buf], 0));
        } else {
            BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[buf], xs));
            BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[buf], 0));
            if ((st = launch_transpose(dB[buf].u(), nb, krows, n, dBt[buf].u(), n_pad, cwq, cs))) return st;
        }
        const bool acc = accumulate || q > 0;
        if (q + 1 < n_chunks || n_slices < 2) {
            if ((st = launch_cubic(kernel, dA[buf].u(), cwq, dBt[buf].u(), cwq, dC.u(), cw, m_pad, n_pad, cwq, gf2,
                                   acc, cs, 1, 0, 0, 0)))
                return st;
        } else {
            int e_slot = 0;
            uint64_t r0 = 0;
            for (const uint64_t rs : slices) {
                if ((st = launch_cubic(kernel, dA[buf].u() + r0 * cwq, cwq, dBt[buf].u(), cwq, dC.u() + r0 * cw, cw,
                                       rs, n_pad, cwq, gf2, acc, cs, 1, 0, 0, 0)))
                    return st;
                if (r0 < m) {
                    const uint64_t rows = std::min(rs, m - r0);
                    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[8 + e_slot], cs));
                    BMMGPU_CUDA_TRY(cudaStreamWaitEvent(ds, ev.e[8 + e_slot], 0));
                    BMMGPU_CUDA_TRY(memcpy2d_counted(C + (row_begin + r0) * nb, nb * 8, dC.u() + r0 * cw, cw * 8,
                                                      nb * 8, rows, cudaMemcpyDeviceToHost, ds));
                }
                r0 += rs;
                e_slot ^= 1;
            }
        }
        BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[2 + buf], cs));
        w0 += cwq;
    }
    if (n_slices < 2)
        BMMGPU_CUDA_TRY(memcpy2d_counted(C + row_begin * nb, nb * 8, dC.p, cw * 8, nb * 8, m, cudaMemcpyDeviceToHost,
                                          cs));
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[10], ds));
    BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, ev.e[10], 0));
    BMMGPU_CUDA_TRY(cudaEventRecord(ev.e[6], cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(xs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(ds));
    if (ms_out) cudaEventElapsedTime(ms_out, ev.e[5], ev.e[6]);
    return kOk;
}

}  // namespace bmmgpu
