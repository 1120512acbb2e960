// capi.cu -- the extern "C" boundary (include/bmmgpu.h) and the host-side
// multi-GPU driver.
//
// Host API calls take reference-layout host buffers (BitMatrix::words), move
// them to HBM, run the device pipeline and copy the result back.  With more
// than one device in opts.device_mask the output rows are partitioned into
// contiguous slabs, one host thread per device, each device holding its A
// slab and all of Bt: output tiles are independent, so there is no exchange
// step (the paper's "one host thread per output
// segment").
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bmmgpu.h"
#include "common.cuh"

namespace bmmgpu {

int launch_transpose(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                     uint64_t kw, cudaStream_t stream);
int launch_cubic_lop3(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                      uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate, cudaStream_t stream,
                      uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch);
void lop3_granularity(uint64_t* gm, uint64_t* gn, uint64_t* gk_bits);
int launch_cubic_umma(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                      uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate, cudaStream_t stream,
                      uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch);
void umma_granularity(uint64_t* gm, uint64_t* gn, uint64_t* gk_bits);
int alt_multiply_host(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int algo, const bmmgpu_plan* plan,
                      int kernel, int leaf_log2, double* timing_ms);
int stream_kouter_slab(int device, uint64_t row_begin, uint64_t row_end, const uint64_t* A, const uint64_t* B,
                       uint64_t* C, uint64_t k, uint64_t n, bool gf2, int kernel, bool accumulate, uint64_t budget,
                       float* ms_out, int chunks);
int alt_multiply_multi(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int algo, int dh,
                       const std::vector<int>& phys, int kernel, int leaf_log2, double* timing_ms);
int host_levels_for(uint64_t n, uint32_t parts, int e);
int alt_levels(uint64_t n, int leaf_log2);
int alt_multiply_subinst(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int algo, int dh,
                         int kernel, int leaf_log2, uint64_t budget, double* timing_ms);
int alt_multiply_tiles(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int algo,
                       const std::vector<int>& devs, int kernel, int leaf_log2, double* timing_ms, uint64_t b,
                       uint64_t p0, uint64_t p1);
int stream_cubic_slab(int device, uint64_t row_begin, uint64_t row_end, const uint64_t* A, const uint64_t* B,
                      uint64_t* C, uint64_t k, uint64_t n, bool gf2, int kernel, bool accumulate, uint64_t budget,
                      float* ms_out);

namespace {
thread_local std::string g_error;
struct CallStats {
    std::atomic<uint64_t> launches{0}, h2d{0}, d2h{0};
};
thread_local CallStats t_stats;               // this thread's last host-API call
thread_local CallStats* t_parent = nullptr;   // worker thread of a call on another thread
CallStats& cur_stats() { return t_parent ? *t_parent : t_stats; }
}  // namespace

void* call_stats() { return &cur_stats(); }
void adopt_call_stats(void* stats) { t_parent = static_cast<CallStats*>(stats); }
void reset_call_stats() {
    CallStats& c = cur_stats();
    c.launches.store(0);
    c.h2d.store(0);
    c.d2h.store(0);
}

void set_error(const std::string& msg) { g_error = msg; }

void enable_pool_caching() {
    static std::mutex mu;
    static uint32_t done_mask = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 32) return;
    std::lock_guard<std::mutex> lock(mu);
    if (done_mask & (1u << dev)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t threshold = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    done_mask |= 1u << dev;
}
// Free device memory without cudaMemGetInfo on every call: measured on the box, that call
// blocked host threads for 9-68 ms now and then while the device was busy (microbench/
// c2_steps.py, profiles/r02/c2_step_enqueue.txt), which stalled the enqueue of a whole
// fast-product step.  One real query per device is kept as a snapshot together with the
// stream-ordered pool's reserved bytes at that time; later estimates = snapshot free - what
// the pool reserved since + the pool's idle (reserved, unused) bytes, which the library's
// own stream-ordered allocations reuse.  Allocations by others after the snapshot are not
// seen: callers that size a plan close to the estimate ask for a fresh query
// (device_free_bytes(true)).
uint64_t device_free_bytes(bool refresh) {
    static std::mutex mu;
    static bool have[32] = {};
    static uint64_t free0[32] = {}, reserved0[32] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) return 0;
    enable_pool_caching();
    uint64_t reserved = 0, used = 0;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    }
    std::lock_guard<std::mutex> lock(mu);
    if (refresh || !have[dev]) {
        size_t f = 0, t = 0;
        if (cudaMemGetInfo(&f, &t) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        have[dev] = true;
        free0[dev] = f;
        reserved0[dev] = reserved;
    }
    const int64_t est = int64_t(free0[dev]) - (int64_t(reserved) - int64_t(reserved0[dev])) +
                        (int64_t(reserved) - int64_t(used));
    return est > 0 ? uint64_t(est) : 0;
}

namespace {
std::mutex g_stream_mu;
std::vector<cudaStream_t> g_stream_pool[32][3];  // idle leased-and-returned streams per device and priority
}  // namespace

int StreamSet::acquire(int count, int priority) {
    if (cudaGetDevice(&device) != cudaSuccess || device < 0 || device >= 32) return kEcuda;
    n = 0;
    prio = priority > 0 ? 1 : priority < 0 ? 2 : 0;
    {
        std::lock_guard<std::mutex> lock(g_stream_mu);
        auto& pool = g_stream_pool[device][prio];
        while (n < count && !pool.empty()) {
            s[n++] = pool.back();
            pool.pop_back();
        }
    }
    int least = 0, greatest = 0;
    if (n < count && prio) cudaDeviceGetStreamPriorityRange(&least, &greatest);
    for (; n < count; ++n) {
        const cudaError_t e = cudaStreamCreateWithPriority(&s[n], cudaStreamNonBlocking,
                                                           prio == 1 ? greatest : prio == 2 ? least : 0);
        if (e != cudaSuccess) {
            s[n] = nullptr;
            set_error(std::string("cudaStreamCreateWithPriority: ") + cudaGetErrorString(e));
            return kEcuda;
        }
    }
    return kOk;
}

StreamSet::~StreamSet() {
    if (n == 0) return;
    std::lock_guard<std::mutex> lock(g_stream_mu);
    for (int i = 0; i < n; ++i)
        if (s[i]) g_stream_pool[device][prio].push_back(s[i]);
}

void count_launch(uint64_t n) { cur_stats().launches.fetch_add(n, std::memory_order_relaxed); }
void count_copy(cudaMemcpyKind kind, uint64_t bytes) {
    if (kind == cudaMemcpyHostToDevice) cur_stats().h2d.fetch_add(bytes, std::memory_order_relaxed);
    if (kind == cudaMemcpyDeviceToHost) cur_stats().d2h.fetch_add(bytes, std::memory_order_relaxed);
}

namespace {

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Two 64 MiB page-locked slots per device and direction, allocated on first use and kept:
// uploads and downloads stage concurrently (the streamed fast path downloads finished C
// quadrants while later operand quadrants go up).
struct Stager {
    static constexpr size_t kSlot = size_t(64) << 20;
    std::mutex mu;
    void* slot[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    bool ready = false;
    bool init() {
        if (ready) return true;
        for (int i = 0; i < 2; ++i) {
            if (cudaHostAlloc(&slot[i], kSlot, cudaHostAllocPortable) != cudaSuccess) return false;
            if (cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess) return false;
        }
        ready = true;
        return true;
    }
};
Stager g_stagers[16][2];  // [device][0: host -> device, 1: device -> host]

// Persistent memcpy helpers for the staged copies: spawning threads per 64 MiB chunk cost
// a large share of the chunk's time (staged uploads measured 10.8 GB/s against 63 GB/s for
// an 8-thread memcpy on the box, microbench/staging.py, memcpy_bw.cu).  run(n, f) calls
// f(0) .. f(n - 1), f(0) on the caller, the rest on the pool.
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool* pool = new CopyPool();  // never destroyed: workers may outlive main
        return *pool;
    }
    unsigned width() const { return unsigned(workers_.size()) + 1; }
    void run(unsigned n, const std::function<void(unsigned)>& f) {
        std::lock_guard<std::mutex> one(call_mu_);  // one staged copy at a time per pool
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &f;
            parts_ = n;
            next_ = 1;
            pending_ = n - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    CopyPool() {
        const unsigned hc = std::thread::hardware_concurrency();
        const unsigned n = std::max(1u, std::min(12u, hc ? hc * 3 / 4 : 4u));
        for (unsigned i = 0; i + 1 < n; ++i) workers_.emplace_back([this] { loop(); });
        for (auto& t : workers_) t.detach();
    }
    void loop() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [&] { return gen_ != seen && job_ && next_ < parts_; });
            seen = gen_;
            while (job_ && next_ < parts_) {
                const unsigned i = next_++;
                const std::function<void(unsigned)>* f = job_;
                lk.unlock();
                (*f)(i);
                lk.lock();
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }
    std::vector<std::thread> workers_;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(unsigned)>* job_ = nullptr;
    unsigned parts_ = 0, next_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
};

}  // namespace

// f(0) .. f(parts - 1) over the library's host helper threads (the staging copy pool).
void host_parallel(unsigned parts, const std::function<void(unsigned)>& f) {
    if (parts <= 1) {
        if (parts == 1) f(0);
        return;
    }
    CopyPool::get().run(parts, f);
}
unsigned host_parallel_width() { return CopyPool::get().width(); }

namespace {

// `rows` rows of `width` bytes from src (pitch spitch) to dst (pitch dpitch), split
// across the copy pool (8 MiB per part, at most the pool's width: one memcpy thread
// moves ~8-10 GB/s, the link takes ~55 GB/s)
void copy_rows(char* dst, size_t dpitch, const char* src, size_t spitch, size_t width, size_t rows) {
    const size_t bytes = rows * width;
    CopyPool& pool = CopyPool::get();
    const unsigned n = unsigned(std::min<size_t>(pool.width(), std::max<size_t>(1, bytes >> 23)));
    const size_t step = (rows + n - 1) / n;
    auto part = [&](unsigned i) {
        const size_t a = std::min(rows, i * step), b = std::min(rows, (i + 1) * step);
        if (width == spitch && width == dpitch)
            std::memcpy(dst + a * dpitch, src + a * spitch, (b - a) * width);
        else
            for (size_t r = a; r < b; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, width);
    };
    if (n == 1)
        part(0);
    else
        pool.run(n, part);
}

}  // namespace

namespace {
// The staged copy proper (no byte counting): pageable host buffers go through the page-locked
// slots, everything else straight to cudaMemcpy2DAsync.
cudaError_t memcpy2d_staged(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                            cudaMemcpyKind kind, cudaStream_t s) {
    const bool h2d = kind == cudaMemcpyHostToDevice, d2h = kind == cudaMemcpyDeviceToHost;
    const void* host = h2d ? src : d2h ? static_cast<const void*>(dst) : nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    static const bool disabled = getenv("BMMGPU_NO_STAGING") != nullptr;
    if (disabled || !host || width * height < (size_t(16) << 20) || width > Stager::kSlot || dev < 0 || dev >= 16 ||
        is_pinned(host))
        return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, s);
    Stager& st = g_stagers[dev][h2d ? 0 : 1];
    std::lock_guard<std::mutex> lk(st.mu);
    if (!st.init()) return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, s);
    const size_t rows_per = std::max<size_t>(1, Stager::kSlot / width);
    cudaError_t e = cudaSuccess;
    int k = 0;
    if (h2d) {
        for (size_t r0 = 0; r0 < height; r0 += rows_per, k ^= 1) {
            const size_t r1 = std::min(height, r0 + rows_per);
            if ((e = cudaEventSynchronize(st.done[k])) != cudaSuccess) return e;  // slot's last DMA finished
            copy_rows(static_cast<char*>(st.slot[k]), width, static_cast<const char*>(src) + r0 * spitch, spitch, width,
                      r1 - r0);
            if ((e = cudaMemcpy2DAsync(static_cast<char*>(dst) + r0 * dpitch, dpitch, st.slot[k], width, width,
                                       r1 - r0, kind, s)) != cudaSuccess ||
                (e = cudaEventRecord(st.done[k], s)) != cudaSuccess)
                return e;
        }
        return cudaSuccess;
    }
    // D2H: DMA chunk i + 1 into one slot while host threads drain chunk i from the other
    size_t pending_r0 = 0, pending_r1 = 0;
    int pending = -1;
    for (size_t r0 = 0; r0 < height; r0 += rows_per, k ^= 1) {
        const size_t r1 = std::min(height, r0 + rows_per);
        if ((e = cudaMemcpy2DAsync(st.slot[k], width, static_cast<const char*>(src) + r0 * spitch, spitch, width,
                                   r1 - r0, kind, s)) != cudaSuccess ||
            (e = cudaEventRecord(st.done[k], s)) != cudaSuccess)
            return e;
        if (pending >= 0) {
            if ((e = cudaEventSynchronize(st.done[pending])) != cudaSuccess) return e;
            copy_rows(static_cast<char*>(dst) + pending_r0 * dpitch, dpitch,
                      static_cast<const char*>(st.slot[pending]), width, width, pending_r1 - pending_r0);
        }
        pending = k;
        pending_r0 = r0;
        pending_r1 = r1;
    }
    if (pending >= 0) {
        if ((e = cudaEventSynchronize(st.done[pending])) != cudaSuccess) return e;
        copy_rows(static_cast<char*>(dst) + pending_r0 * dpitch, dpitch, static_cast<const char*>(st.slot[pending]),
                  width, width, pending_r1 - pending_r0);
    }
    return cudaSuccess;
}
}  // namespace

cudaError_t memcpy2d_counted(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                             cudaMemcpyKind kind, cudaStream_t s) {
    count_copy(kind, uint64_t(width) * height);
    // A contiguous region wider than a staging slot (memcpy_counted of a whole operand is one
    // "row" of hundreds of MiB) is staged as rows of 1 MiB: it used to fall through to the
    // runtime's own pageable copy, ~10 GB/s against ~50 staged (microbench/staging.py)
    constexpr size_t kPiece = size_t(1) << 20;
    if (width > (size_t(64) << 20) && (height == 1 || (spitch == width && dpitch == width))) {
        const size_t total = width * height, main = total / kPiece * kPiece;
        if (main) {
            const cudaError_t e = memcpy2d_staged(dst, kPiece, src, kPiece, kPiece, main / kPiece, kind, s);
            if (e != cudaSuccess || total == main) return e;
        }
        return cudaMemcpyAsync(static_cast<char*>(dst) + main, static_cast<const char*>(src) + main, total - main,
                               kind, s);
    }
    return memcpy2d_staged(dst, dpitch, src, spitch, width, height, kind, s);
}

int resolve_kernel(int kernel) {
    // The tcgen05 kind::mxf4 kernel beats the LOP3 kernel 3.4-3.8x in bop/s on
    // B200 (profiles/r01), so it is the default block product.
    if (kernel == BMMGPU_KERNEL_AUTO) return BMMGPU_KERNEL_UMMA_F4;
    return kernel;
}

int granularity(int kernel, uint64_t* gm, uint64_t* gn, uint64_t* gk) {
    switch (resolve_kernel(kernel)) {
        case BMMGPU_KERNEL_LOP3: lop3_granularity(gm, gn, gk); return kOk;
        case BMMGPU_KERNEL_UMMA_F4: umma_granularity(gm, gn, gk); return kOk;
        default: set_error("unknown kernel id " + std::to_string(kernel)); return kEinval;
    }
}

// Block-product timer: while enabled, every block-product launch is bracketed by a
// pair of CUDA events on its stream, so a caller (bench.py) can report the dominant
// kernel's device time even when it runs inside a longer pipeline (the leaves of the
// fast recursion).  Off by default: no events are recorded.
namespace {
struct BlockTimer {
    std::mutex mu;
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spans;
};
BlockTimer g_timer;
}  // namespace

int launch_cubic_dispatch(int kernel, const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt,
                          uint64_t* dC, uint64_t ldc, uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2,
                          bool accumulate, cudaStream_t stream, uint64_t batch, uint64_t sA_batch, uint64_t sB_batch,
                          uint64_t sC_batch);

int launch_cubic(int kernel, const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                 uint64_t ldc, uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate,
                 cudaStream_t stream, uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch) {
    bool timed;
    {
        std::lock_guard<std::mutex> lk(g_timer.mu);
        timed = g_timer.on;
    }
    if (!timed)
        return launch_cubic_dispatch(kernel, dA, lda, dBt, ldbt, dC, ldc, m_pad, n_pad, kw, gf2, accumulate, stream,
                                     batch, sA_batch, sB_batch, sC_batch);
    cudaEvent_t e0, e1;
    BMMGPU_CUDA_TRY(cudaEventCreate(&e0));
    BMMGPU_CUDA_TRY(cudaEventCreate(&e1));
    BMMGPU_CUDA_TRY(cudaEventRecord(e0, stream));
    const int st = launch_cubic_dispatch(kernel, dA, lda, dBt, ldbt, dC, ldc, m_pad, n_pad, kw, gf2, accumulate,
                                         stream, batch, sA_batch, sB_batch, sC_batch);
    BMMGPU_CUDA_TRY(cudaEventRecord(e1, stream));
    std::lock_guard<std::mutex> lk(g_timer.mu);
    g_timer.spans.emplace_back(e0, e1);
    return st;
}

int launch_cubic_kernel(int kernel, const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt,
                        uint64_t* dC, uint64_t ldc, uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2,
                        bool accumulate, cudaStream_t stream, uint64_t batch, uint64_t sA_batch, uint64_t sB_batch,
                        uint64_t sC_batch);
int launch_cubic_umma_fold(const uint64_t* dApar, uint64_t ld_a, uint64_t s_a, const uint64_t* dBtpar, uint64_t ld_b,
                           uint64_t s_b, uint64_t parents, uint64_t L, uint32_t ma, uint32_t mb, uint64_t* dQ,
                           uint64_t ldq, uint64_t s_q, bool gf2, cudaStream_t stream);

// Level-shifted leaf layer (K2 fold mode), bracketed by the block timer like launch_cubic.
int launch_cubic_fold(const uint64_t* dApar, uint64_t ld_a, uint64_t s_a, const uint64_t* dBtpar, uint64_t ld_b,
                      uint64_t s_b, uint64_t parents, uint64_t L, uint32_t ma, uint32_t mb, uint64_t* dQ, uint64_t ldq,
                      uint64_t s_q, cudaStream_t stream) {
    bool timed;
    {
        std::lock_guard<std::mutex> lk(g_timer.mu);
        timed = g_timer.on;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
        BMMGPU_CUDA_TRY(cudaEventCreate(&e0));
        BMMGPU_CUDA_TRY(cudaEventCreate(&e1));
        BMMGPU_CUDA_TRY(cudaEventRecord(e0, stream));
    }
    const int st = launch_cubic_umma_fold(dApar, ld_a, s_a, dBtpar, ld_b, s_b, parents, L, ma, mb, dQ, ldq, s_q, true,
                                          stream);
    if (timed) {
        BMMGPU_CUDA_TRY(cudaEventRecord(e1, stream));
        std::lock_guard<std::mutex> lk(g_timer.mu);
        g_timer.spans.emplace_back(e0, e1);
    }
    return st;
}

// The tensor-core kernels count in fp32 (exact below 2^23 terms): longer inner
// dimensions run as K-chunks folded into C with the accumulate flag -- the
// reference's XOR / OR fold of partial block products (engine.cpp:81-84).
constexpr uint64_t kMaxTensorKWords = (uint64_t(1) << 22) / 64;  // 2^22 bits per launch

int launch_cubic_dispatch(int kernel, const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt,
                          uint64_t* dC, uint64_t ldc, uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2,
                          bool accumulate, cudaStream_t stream, uint64_t batch, uint64_t sA_batch, uint64_t sB_batch,
                          uint64_t sC_batch) {
    if (resolve_kernel(kernel) != BMMGPU_KERNEL_LOP3 && kw > kMaxTensorKWords) {
        for (uint64_t w0 = 0; w0 < kw; w0 += kMaxTensorKWords) {
            const int st = launch_cubic_kernel(kernel, dA + w0, lda, dBt + w0, ldbt, dC, ldc, m_pad, n_pad,
                                               std::min(kMaxTensorKWords, kw - w0), gf2, accumulate || w0 > 0,
                                               stream, batch, sA_batch, sB_batch, sC_batch);
            if (st) return st;
        }
        return kOk;
    }
    return launch_cubic_kernel(kernel, dA, lda, dBt, ldbt, dC, ldc, m_pad, n_pad, kw, gf2, accumulate, stream, batch,
                               sA_batch, sB_batch, sC_batch);
}

int launch_cubic_kernel(int kernel, const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt,
                        uint64_t* dC, uint64_t ldc, uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2,
                        bool accumulate, cudaStream_t stream, uint64_t batch, uint64_t sA_batch, uint64_t sB_batch,
                        uint64_t sC_batch) {
    switch (resolve_kernel(kernel)) {
        case BMMGPU_KERNEL_LOP3:
            return launch_cubic_lop3(dA, lda, dBt, ldbt, dC, ldc, m_pad, n_pad, kw, gf2, accumulate, stream, batch,
                                     sA_batch, sB_batch, sC_batch);
        case BMMGPU_KERNEL_UMMA_F4:
            return launch_cubic_umma(dA, lda, dBt, ldbt, dC, ldc, m_pad, n_pad, kw, gf2, accumulate, stream, batch,
                                     sA_batch, sB_batch, sC_batch);
        default: set_error("unknown kernel id " + std::to_string(kernel)); return kEinval;
    }
}

namespace {

struct SlabJob {
    int device;
    uint64_t row_begin, row_end;  // output rows of this device
    int status = kOk;
    std::string error;
    float ms = 0.f;
};

// One device's share of C = A.B: rows [row_begin, row_end) of A and C.  In
// core when A slab, B, Bt and C fit the budget, else the streamed driver.
int run_cubic_slab(SlabJob& job, const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t k, uint64_t n,
                   bool gf2, int kernel, bool accumulate, uint64_t budget, int force_streaming) {
    BMMGPU_CUDA_TRY(cudaSetDevice(job.device));
    const uint64_t m = job.row_end - job.row_begin;
    if (m == 0) return kOk;
    uint64_t gm, gn, gk;
    int st = granularity(kernel, &gm, &gn, &gk);
    if (st) return st;
    const uint64_t ka = ceil_div(k, 64), nb = ceil_div(n, 64);
    const uint64_t m_pad = round_up(m, gm), n_pad = round_up(std::max<uint64_t>(n, 1), gn);
    const uint64_t kw = round_up(std::max<uint64_t>(ka, 1), gk / 64);
    const uint64_t cw = n_pad / 64;
    {
        const uint64_t in_core = (m_pad * kw + k * nb + n_pad * kw + m_pad * cw) * 8;
        const uint64_t c_slab = m_pad * cw * 8;
        uint64_t limit = budget;
        if (limit == 0) {
            // cudaMemGetInfo costs ~65 us of host time: small products (under 1/32 of the
            // device) skip it and take the in-core path
            static std::mutex mu;
            static uint64_t total_mem[32] = {};
            uint64_t total = 0;
            {
                std::lock_guard<std::mutex> lock(mu);
                total = job.device < 32 ? total_mem[job.device] : 0;
            }
            if (total && in_core * 32 <= total && k < 32768) {
                limit = in_core;
            } else {
                uint64_t free_b = device_free_bytes(false);
                if (in_core * 2 > free_b) free_b = device_free_bytes(true);  // close call: a fresh query
                limit = uint64_t(double(free_b) * 0.9);
                if (!total) {
                    size_t f = 0, t = 0;
                    BMMGPU_CUDA_TRY(cudaMemGetInfo(&f, &t));
                    std::lock_guard<std::mutex> lock(mu);
                    if (job.device < 32) total_mem[job.device] = t;
                }
            }
        }
        // force_streaming 1: the out-of-core tile driver; 2: the K-outer pipeline.
        // Otherwise: long K with C resident -> K-outer pipeline (H2D hidden behind
        // the product); everything fits -> in core; else the tile driver.
        if (force_streaming == 1 || (force_streaming == 0 && in_core > limit && 3 * c_slab > limit))
            return stream_cubic_slab(job.device, job.row_begin, job.row_end, A, B, C, k, n, gf2, kernel,
                                     accumulate, limit, &job.ms);
        if (force_streaming == 2 || (force_streaming == 0 && k >= 32768 && 3 * c_slab <= limit) ||
            in_core > limit)
            return stream_kouter_slab(job.device, job.row_begin, job.row_end, A, B, C, k, n, gf2, kernel,
                                      accumulate, limit, &job.ms, getenv("BMMGPU_KOUTER_CHUNKS")
                                                                       ? atoi(getenv("BMMGPU_KOUTER_CHUNKS"))
                                                                       : 0);
    }
    // In core, pipelined over row slices of A / C: B goes up first (every slice needs
    // all of it) and is transposed while the A slices follow on the copy stream; slice
    // i's product starts when its rows of A have landed and its rows of C go home on a
    // download stream while slice i + 1 computes.  Exposed: B's upload, one A slice,
    // the last slice's product and download (n = 8192: the in-order H2D / product /
    // D2H sequence was ~0.62 ms of copies and kernels).  Slices keep >= 8 row tiles.
    const char* sl_env = getenv("BMMGPU_INCORE_SLICES");  // dev: 1 = one slice (in order)
    const uint64_t row_tiles = m_pad / gm;
    const uint64_t n_slices =
        std::max<uint64_t>(1, std::min<uint64_t>(sl_env ? std::max(1, atoi(sl_env)) : 4, row_tiles / 8));
    const uint64_t slice = round_up(ceil_div(m_pad, n_slices), gm);
    StreamSet ss;
    if ((st = ss.acquire(3))) return st;
    struct Events {
        std::vector<cudaEvent_t> ev;
        ~Events() {
            for (auto e : ev)
                if (e) cudaEventDestroy(e);
        }
    } pp;
    // events: 0 allocated, 1 B ready, 2 / 3 timing, then per slice: A ready, C ready
    pp.ev.assign(4 + 2 * size_t(ceil_div(m_pad, slice)), nullptr);
    for (size_t i = 0; i < pp.ev.size(); ++i)
        BMMGPU_CUDA_TRY(cudaEventCreateWithFlags(&pp.ev[i], i == 2 || i == 3 ? 0 : cudaEventDisableTiming));
    const cudaStream_t cs = ss[0], xs = ss[1], ds = ss[2];
    DeviceBuffer dA, dB, dBt, dC;
    StreamDrain drain{{cs, xs, ds, nullptr}};
    if ((st = dA.alloc(m_pad * kw * 8, cs)) || (st = dBt.alloc(n_pad * kw * 8, cs)) ||
        (st = dC.alloc(m_pad * cw * 8, cs)) || (k > 0 && (st = dB.alloc(k * nb * 8, cs))))
        return st;
    BMMGPU_CUDA_TRY(cudaEventRecord(pp.ev[0], cs));
    BMMGPU_CUDA_TRY(cudaStreamWaitEvent(xs, pp.ev[0], 0));
    BMMGPU_CUDA_TRY(cudaStreamWaitEvent(ds, pp.ev[0], 0));
    // B, then Bt on device
    if (k > 0) BMMGPU_CUDA_TRY(memcpy_counted(dB.p, B, k * nb * 8, cudaMemcpyHostToDevice, xs));
    BMMGPU_CUDA_TRY(cudaEventRecord(pp.ev[1], xs));
    // A slab into the zero-padded panel (pad columns / rows stay zero)
    if (m_pad != m || kw != ka) {
        BMMGPU_CUDA_TRY(cudaMemsetAsync(dA.p, 0, m_pad * kw * 8, xs));
        count_launch();
    }
    if (accumulate) {
        BMMGPU_CUDA_TRY(cudaMemsetAsync(dC.p, 0, m_pad * cw * 8, xs));
        count_launch();
    }
    BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, pp.ev[1], 0));
    if (k > 0) {
        if ((st = launch_transpose(dB.u(), nb, k, n, dBt.u(), n_pad, kw, cs))) return st;
    } else {
        BMMGPU_CUDA_TRY(cudaMemsetAsync(dBt.p, 0, n_pad * kw * 8, cs));
        count_launch();
    }
    BMMGPU_CUDA_TRY(cudaEventRecord(pp.ev[2], cs));
    size_t si = 0;
    for (uint64_t r0 = 0; r0 < m_pad; r0 += slice, ++si) {
        const uint64_t rs = std::min(slice, m_pad - r0);
        const uint64_t rows = r0 < m ? std::min(rs, m - r0) : 0;  // real rows of this slice
        cudaEvent_t a_ready = pp.ev[4 + 2 * si], c_ready = pp.ev[5 + 2 * si];
        if (rows > 0 && ka > 0)
            BMMGPU_CUDA_TRY(memcpy2d_counted(dA.u() + r0 * kw, kw * 8, A + (job.row_begin + r0) * ka, ka * 8,
                                              ka * 8, rows, cudaMemcpyHostToDevice, xs));
        if (rows > 0 && accumulate)
            BMMGPU_CUDA_TRY(memcpy2d_counted(dC.u() + r0 * cw, cw * 8, C + (job.row_begin + r0) * nb, nb * 8,
                                              nb * 8, rows, cudaMemcpyHostToDevice, xs));
        BMMGPU_CUDA_TRY(cudaEventRecord(a_ready, xs));
        BMMGPU_CUDA_TRY(cudaStreamWaitEvent(cs, a_ready, 0));
        if ((st = launch_cubic(kernel, dA.u() + r0 * kw, kw, dBt.u(), kw, dC.u() + r0 * cw, cw, rs, n_pad, kw, gf2,
                               accumulate, cs, 1, 0, 0, 0)))
            return st;
        BMMGPU_CUDA_TRY(cudaEventRecord(c_ready, cs));
        if (rows > 0) {
            BMMGPU_CUDA_TRY(cudaStreamWaitEvent(ds, c_ready, 0));
            BMMGPU_CUDA_TRY(memcpy2d_counted(C + (job.row_begin + r0) * nb, nb * 8, dC.u() + r0 * cw, cw * 8, nb * 8,
                                              rows, cudaMemcpyDeviceToHost, ds));
        }
    }
    BMMGPU_CUDA_TRY(cudaEventRecord(pp.ev[3], cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(ds));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(cs));
    BMMGPU_CUDA_TRY(cudaStreamSynchronize(xs));
    cudaEventElapsedTime(&job.ms, pp.ev[2], pp.ev[3]);
    return kOk;
}

// Devices named by a device_mask.  Test hook: BMMGPU_LOGICAL_DEVICES=k makes k logical
// devices, bit g running on physical device g % count, so the multi-device drivers
// (one host thread and one set of buffers per logical device, peer copies between
// them) run on a one-GPU box.
std::vector<int> devices_of(uint32_t mask, int* status) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    std::vector<int> devs;
    if (e != cudaSuccess || count == 0) {
        set_error(std::string("no CUDA device available (") + cudaGetErrorString(e) +
                  "); the bit-matrix engine has no CPU fallback");
        *status = kEnodev;
        return devs;
    }
    const int physical = count;
    if (const char* lg = getenv("BMMGPU_LOGICAL_DEVICES")) count = std::max(1, std::min(32, atoi(lg)));
    if (mask == 0) mask = 1;
    for (int g = 0; g < 32 && g < count; ++g)
        if (mask & (1u << g)) devs.push_back(g % physical);
    if (devs.empty() || (count < 32 && (mask >> count) > 0)) {
        set_error("device_mask selects devices that do not exist");
        *status = kEinval;
        devs.clear();
        return devs;
    }
    *status = kOk;
    return devs;
}

}  // namespace

}  // namespace bmmgpu

using namespace bmmgpu;

extern "C" {

const char* bmmgpu_last_error(void) { return g_error.c_str(); }

int bmmgpu_slab_rows(uint64_t m, uint32_t parts, uint32_t index, uint64_t gran, uint64_t* begin, uint64_t* end) {
    if (parts == 0 || index >= parts || gran == 0 || !begin || !end) {
        set_error("bmmgpu_slab_rows: need 0 <= index < parts and gran > 0");
        return kEinval;
    }
    const uint64_t blocks = ceil_div(m, gran);
    *begin = std::min(m, (blocks * index / parts) * gran);
    *end = std::min(m, (blocks * (index + 1) / parts) * gran);
    return kOk;
}
const char* bmmgpu_version(void) { return "bmm-b200 0.1 (sm_100a)"; }
uint64_t bmmgpu_last_launch_count(void) { return t_stats.launches.load(); }

int bmmgpu_host_alloc(uint64_t bytes, void** ptr) {
    if (!ptr) {
        set_error("bmmgpu_host_alloc: null output pointer");
        return kEinval;
    }
    *ptr = nullptr;
    const cudaError_t e = cudaHostAlloc(ptr, bytes ? bytes : 8, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        set_error(std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
        *ptr = nullptr;
        return kEcuda;
    }
    return kOk;
}

int bmmgpu_host_free(void* ptr) {
    if (ptr && cudaFreeHost(ptr) != cudaSuccess) {
        set_error("cudaFreeHost failed");
        return kEcuda;
    }
    return kOk;
}

int bmmgpu_last_copy_bytes(uint64_t* h2d, uint64_t* d2h) {
    if (h2d) *h2d = t_stats.h2d.load();
    if (d2h) *d2h = t_stats.d2h.load();
    return kOk;
}

int bmmgpu_block_timer(int32_t enable) {
    std::lock_guard<std::mutex> lk(g_timer.mu);
    for (auto& p : g_timer.spans) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    g_timer.spans.clear();
    g_timer.on = enable != 0;
    return kOk;
}

int bmmgpu_block_timer_read(double* ms, uint64_t* launches) {
    std::lock_guard<std::mutex> lk(g_timer.mu);
    double total = 0.0;
    for (auto& p : g_timer.spans) {
        BMMGPU_CUDA_TRY(cudaEventSynchronize(p.second));
        float t = 0.f;
        BMMGPU_CUDA_TRY(cudaEventElapsedTime(&t, p.first, p.second));
        total += t;
    }
    if (ms) *ms = total;
    if (launches) *launches = g_timer.spans.size();
    return kOk;
}

int bmmgpu_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

int bmmgpu_mem_info(int32_t device, uint64_t* free_bytes, uint64_t* total_bytes) {
    int prev = 0;
    cudaGetDevice(&prev);
    BMMGPU_CUDA_TRY(cudaSetDevice(device));
    size_t f = 0, t = 0;
    const cudaError_t e = cudaMemGetInfo(&f, &t);
    cudaSetDevice(prev);
    BMMGPU_CUDA_TRY(e);
    if (free_bytes) *free_bytes = f;
    if (total_bytes) *total_bytes = t;
    return kOk;
}

int bmmgpu_dev_granularity(int32_t kernel, uint64_t* m_gran, uint64_t* n_gran, uint64_t* k_gran_bits) {
    return granularity(kernel, m_gran, n_gran, k_gran_bits);
}

int bmmgpu_dev_transpose(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                         uint64_t kw, void* stream) {
    return launch_transpose(dB, ldb, k, n, dBt, n_pad, kw, static_cast<cudaStream_t>(stream));
}

int bmmgpu_dev_cubic(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                     uint64_t m_pad, uint64_t n_pad, uint64_t kw, int32_t semiring, int32_t kernel,
                     int32_t accumulate, void* stream) {
    if (semiring != BMMGPU_BOOLEAN_OR_AND && semiring != BMMGPU_GF2_XOR_AND) {
        set_error("unknown semiring");
        return kEinval;
    }
    return launch_cubic(kernel, dA, lda, dBt, ldbt, dC, ldc, m_pad, n_pad, kw, semiring == BMMGPU_GF2_XOR_AND,
                        accumulate != 0, static_cast<cudaStream_t>(stream), 1, 0, 0, 0);
}

}  // extern "C"

namespace bmmgpu {
namespace {
// dst (+)= src over a rows x words region: XOR for GF(2), OR for Boolean -- the
// integration of partial products (reference cubic_blocked fold, engine.cpp:81-84).
__global__ void fold_kernel(uint64_t* __restrict__ dst, uint64_t ldd, const uint64_t* __restrict__ src, uint64_t lds,
                            uint64_t rows, uint64_t words, int gf2) {
    const uint64_t total = rows * words;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = i / words, w = i - r * words;
        const uint64_t v = src[r * lds + w];
        uint64_t& d = dst[r * ldd + w];
        d = gf2 ? (d ^ v) : (d | v);
    }
}
}  // namespace
}  // namespace bmmgpu

extern "C" {

int bmmgpu_dev_fold(uint64_t* dst, uint64_t ldd, const uint64_t* src, uint64_t lds, uint64_t rows, uint64_t words,
                    int32_t semiring, void* stream) {
    if (semiring != BMMGPU_BOOLEAN_OR_AND && semiring != BMMGPU_GF2_XOR_AND) {
        set_error("unknown semiring");
        return kEinval;
    }
    if (rows == 0 || words == 0) return kOk;
    const uint64_t total = rows * words;
    const unsigned grid = unsigned(std::min<uint64_t>((total + 255) / 256, 148ull * 32));
    fold_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, ldd, src, lds, rows, words,
                                                                      semiring == BMMGPU_GF2_XOR_AND);
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

int bmmgpu_dev_cubic_batched(const uint64_t* dA, uint64_t lda, uint64_t sA, const uint64_t* dBt, uint64_t ldbt,
                             uint64_t sB, uint64_t* dC, uint64_t ldc, uint64_t sC, uint64_t batch, uint64_t m_pad,
                             uint64_t n_pad, uint64_t kw, int32_t semiring, int32_t kernel, int32_t accumulate,
                             void* stream) {
    if (semiring != BMMGPU_BOOLEAN_OR_AND && semiring != BMMGPU_GF2_XOR_AND) {
        set_error("unknown semiring");
        return kEinval;
    }
    // sA / sB may be 0 (one panel broadcast to every product); outputs must not overlap
    if (batch > 1 && ((sA && sA < m_pad * lda) || (sB && sB < n_pad * ldbt) || sC < m_pad * ldc)) {
        set_error("batched product: batch strides smaller than one panel");
        return kEinval;
    }
    // the kernels take at most 65535 products per launch (grid.y / tile-id range)
    for (uint64_t b0 = 0; b0 < batch; b0 += 65535) {
        const uint64_t nb = std::min<uint64_t>(65535, batch - b0);
        const int st = launch_cubic(kernel, dA + b0 * sA, lda, dBt + b0 * sB, ldbt, dC + b0 * sC, ldc, m_pad, n_pad,
                                    kw, semiring == BMMGPU_GF2_XOR_AND, accumulate != 0,
                                    static_cast<cudaStream_t>(stream), nb, sA, sB, sC);
        if (st) return st;
    }
    return kOk;
}

int bmmgpu_cubic(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t m, uint64_t k, uint64_t n,
                 int32_t semiring, const bmmgpu_opts* opts) {
    reset_call_stats();
    if (semiring != BMMGPU_BOOLEAN_OR_AND && semiring != BMMGPU_GF2_XOR_AND) {
        set_error("unknown semiring");
        return kEinval;
    }
    const bmmgpu_opts defaults{};
    const bmmgpu_opts& o = opts ? *opts : defaults;
    int st = kOk;
    std::vector<int> devs = devices_of(o.device_mask, &st);
    if (st) return st;
    if (m == 0 || n == 0) {
        if (o.timing_ms) *o.timing_ms = 0.0;
        return kOk;
    }
    // Contiguous row slabs, aligned to 64 rows so device tiles never straddle.
    const uint64_t G = devs.size();
    std::vector<SlabJob> jobs;
    for (uint64_t g = 0; g < G; ++g) {
        SlabJob j;
        j.device = devs[g];
        bmmgpu_slab_rows(m, uint32_t(G), uint32_t(g), 64, &j.row_begin, &j.row_end);
        jobs.push_back(j);
    }
    const bool gf2 = semiring == BMMGPU_GF2_XOR_AND;
    auto work = [&](SlabJob& j) {
        j.status = run_cubic_slab(j, A, B, C, k, n, gf2, o.kernel, o.accumulate != 0, o.device_budget,
                                  o.force_streaming);
        if (j.status) j.error = g_error;
    };
    if (G == 1) {
        work(jobs[0]);
    } else {
        std::vector<std::thread> threads;
        void* stats = call_stats();
        for (auto& j : jobs)
            threads.emplace_back([&work, stats](SlabJob& jj) {
                adopt_call_stats(stats);
                work(jj);
            }, std::ref(j));
        for (auto& t : threads) t.join();
    }
    float worst = 0.f;
    for (auto& j : jobs) {
        if (j.status) {
            set_error("device " + std::to_string(j.device) + ": " + j.error);
            return j.status;
        }
        worst = std::max(worst, j.ms);
    }
    if (o.timing_ms) *o.timing_ms = worst;
    return kOk;
}

int bmmgpu_multiply(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int32_t algo,
                    const bmmgpu_plan* plan, int32_t semiring, const bmmgpu_opts* opts) {
    reset_call_stats();
    const bmmgpu_opts defaults{};
    const bmmgpu_opts& o = opts ? *opts : defaults;
    if (algo == BMMGPU_ALGO_CUBIC) return bmmgpu_cubic(A, B, C, n, n, n, semiring, opts);
    if (algo < 0 || algo > BMMGPU_ALGO_ALT_CHAINING) {
        set_error("unknown algorithm");
        return kEinval;
    }
    if (semiring == BMMGPU_BOOLEAN_OR_AND) {
        set_error(
            "the Boolean semiring has no subtraction, so cancellation-based fast algorithms are unsound over it; "
            "use the cubic algorithm");
        return kEinval;
    }
    if (n < 64 || (n & (n - 1))) {
        set_error("fast algorithms need n = 64 * 2^k");
        return kEshape;
    }
    if (!plan) {
        set_error("plan is required");
        return kEinval;
    }
    int depth = 0;
    while ((64ull << depth) < n) ++depth;
    if (plan->d_host < 0 || plan->d_serial < 0 || plan->d_parallel < 0 || plan->d_inner != 1 || plan->workers < 1 ||
        plan->d_host + plan->d_serial + plan->d_parallel != depth) {
        set_error("layer plan does not match the operands");
        return kEinval;
    }
    int st = kOk;
    std::vector<int> devs = devices_of(o.device_mask, &st);
    if (st) return st;
    BMMGPU_CUDA_TRY(cudaSetDevice(devs[0]));
    {
        // Operands beyond HBM (configs[4]): output tiles of alt-basis block products
        // streamed from host memory (alt_tiles.cu).  In core the recursion needs about six
        // n^2/8 arrays (A, B, Bt, C and the level buffers of the breadth-first part).
        const double need = 6.0 * double(n) * double(n) / 8.0;
        uint64_t free_b = o.device_budget ? 0 : device_free_bytes(false);
        if (!o.device_budget && need * 2 > double(free_b)) free_b = device_free_bytes(true);
        const uint64_t budget = o.device_budget ? o.device_budget : free_b;
        if (o.force_streaming == 1 || need > double(budget)) {
            // one device: the recursion's own top-level sub-instances, generated on the device
            // from streamed source sub-blocks (alt.cu); several devices or BMMGPU_ALT_OOC=tiles:
            // output tiles of block products dealt over the devices (alt_tiles.cu)
            const char* ooc = getenv("BMMGPU_ALT_OOC");
            const bool tiles = devs.size() > 1 || (ooc && !strcmp(ooc, "tiles"));
            if (!tiles && alt_levels(n, o.leaf_log2) >= 2)
                return alt_multiply_subinst(A, B, C, n, algo, plan->d_host, o.kernel, o.leaf_log2, budget,
                                            o.timing_ms);
            return alt_multiply_tiles(A, B, C, n, algo, devs, o.kernel, o.leaf_log2, o.timing_ms, 0, 0, 0);
        }
    }
    if (devs.size() > 1) {
        // several devices: the top host levels of the recursion are dealt across them
        // (plan.d_host when the caller sets it, else the most even deal), and the partial
        // products are XOR-folded slab by slab (alt_multiply_multi)
        const int e = alt_levels(n, o.leaf_log2);
        const int dh = plan->d_host > 0 ? std::max(0, std::min({int(plan->d_host), 4, e - 1}))
                                        : bmmgpu_host_levels(n, uint32_t(devs.size()), o.leaf_log2);
        return alt_multiply_multi(A, B, C, n, algo, dh, devs, o.kernel, o.leaf_log2, o.timing_ms);
    }
    return alt_multiply_host(A, B, C, n, algo, plan, o.kernel, o.leaf_log2, o.timing_ms);
}

}  // extern "C"
