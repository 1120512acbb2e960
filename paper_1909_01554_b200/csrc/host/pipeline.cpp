// pipeline.cpp -- the drop-in host layer bmm::pipeline (include/bmm/pipeline.hpp):
// the paper's Alg. 3 over B200s.  Reference counterpart: src/pipeline.cpp
// (index arithmetic 14-33, locks 41-65, generation 108-155, aggregation 157-179,
// coordinate 198-369).
//
// Division of work.  A host-level sub-instance's inputs are XORs of contiguous
// host-level subvectors of the interleaved operands (the top d_host Morton digits
// are the most significant), so preparing them is a streaming pass over host memory
// -- done on host threads, as in the paper: moving the selected subvectors over PCIe
// instead would multiply the link traffic by the average coefficient weight.  The
// solve stage is the whole sub-product on a GPU (detail::solve_alt -> bmmgpu_multiply_alt:
// inverse basis changes, Morton permutes, the fast product, all on the device).
// Worker l drives device l mod device_count; its buffers are page-locked so the
// solve's copies run at link speed, and the solve takes its inputs by swapping
// buffers with the prepare stages (no copy) before it starts the device product.
#include "bmm/pipeline.hpp"

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>

#include "../schemes.h"
#include "bmmgpu.h"

namespace bmm {
namespace detail {
void solve_alt(const std::uint64_t* a_hat, const std::uint64_t* b_hat, std::uint64_t* c_hat, int depth,
               const Decomposition& d, OpCounter* counter, int device);
}

namespace pipeline {

std::uint64_t SubInstanceIndex::flat() const {
    std::uint64_t f = 0;
    for (const int digit : digits) f = 7 * f + std::uint64_t(digit);
    return f;
}

int SubInstanceIndex::owner(int n_workers) const {
    if (n_workers < 1) throw std::invalid_argument("need at least one worker");
    return int(flat() % std::uint64_t(n_workers));
}

SubInstanceIndex SubInstanceIndex::from_flat(std::uint64_t flat, int d_host) {
    SubInstanceIndex h;
    h.digits.resize(std::size_t(std::max(d_host, 0)));
    for (int l = d_host - 1; l >= 0; --l, flat /= 7) h.digits[std::size_t(l)] = int(flat % 7);
    return h;
}

std::uint64_t sub_instance_count(const LayerPlan& plan) {
    std::uint64_t n = 1;
    for (int l = 0; l < plan.d_host; ++l) n *= 7;
    return n;
}

struct SubvectorLocks::Cell {
    std::mutex mu;
    std::atomic<bool> held{false};
};

SubvectorLocks::SubvectorLocks(int d_host) {
    if (d_host < 0) throw std::invalid_argument("negative host level count");
    n_ = std::size_t(1) << (2 * d_host);
    slots_.reset(new Cell[n_]);
}

SubvectorLocks::~SubvectorLocks() = default;

void SubvectorLocks::lock(std::size_t index) {
    Cell& c = slots_[index];
    c.mu.lock();
    if (c.held.exchange(true, std::memory_order_relaxed)) overlaps_.fetch_add(1, std::memory_order_relaxed);
}

void SubvectorLocks::unlock(std::size_t index) {
    Cell& c = slots_[index];
    c.held.store(false, std::memory_order_relaxed);
    c.mu.unlock();
}

namespace {

const bmmgpu::Scheme& scheme_of(const Decomposition& d) {
    const int algo = d.which == Builtin::StrassenWinograd ? BMMGPU_ALGO_STRASSEN_WINOGRAD
                     : d.which == Builtin::AltSelfInverse ? BMMGPU_ALGO_ALT_SELF_INVERSE
                     : d.which == Builtin::AltChaining    ? BMMGPU_ALGO_ALT_CHAINING
                                                          : -1;
    const bmmgpu::Scheme* sc = bmmgpu::scheme_for(algo);
    if (!sc || !(d.params == TripleParams{}))
        throw std::invalid_argument("the host layer needs a <2,2,2>_7 scheme");
    return *sc;
}

// Coefficient of host-level subvector g (base-4 digits, most significant first) in
// the combination selected by digits h: prod_l M[h_l][g_l] for an input side (rows
// of alpha / beta are the 7 products, columns the 4 quadrants), prod_l M[g_l][h_l]
// for the output side (gamma: rows quadrants, columns products).
bool in_coeff(const char* const rows[7], const std::vector<int>& h, std::uint64_t g) {
    for (std::size_t l = h.size(); l-- > 0; g >>= 2)
        if (rows[h[l]][g & 3] != '1') return false;
    return true;
}
bool out_coeff(const char* const rows[4], const std::vector<int>& h, std::uint64_t g) {
    for (std::size_t l = h.size(); l-- > 0; g >>= 2)
        if (rows[g & 3][h[l]] != '1') return false;
    return true;
}

void check_digits(const SubInstanceIndex& h, const LayerPlan& plan) {
    if (h.digits.size() != std::size_t(plan.d_host)) throw std::invalid_argument("sub-instance index depth mismatch");
    for (const int x : h.digits)
        if (x < 0 || x > 6) throw std::invalid_argument("sub-instance digit out of range");
}

void check_interleaved(const BitVectorTensor& v, const LayerPlan& plan) {
    std::vector<std::uint64_t> want(std::size_t(plan.depth()), 4);
    want.push_back(kBlockBits);
    if (v.mode_lengths != want) throw std::invalid_argument("vector is not interleaved for this plan");
    if (v.words.size() * kWordBits != v.bit_length())
        throw std::invalid_argument("vector storage does not match its modes");
}

// Run body(w0, w1) over [0, words) on up to 8 host threads (streaming, memory-bound
// passes; one thread below 1 Mi words).
template <class F>
void parallel_words(std::uint64_t words, F&& body) {
    const std::uint64_t per = std::uint64_t(1) << 20;
    const unsigned n_thr = unsigned(std::min<std::uint64_t>(8, (words + per - 1) / per));
    if (n_thr <= 1) {
        body(std::uint64_t(0), words);
        return;
    }
    std::vector<std::thread> thr;
    const std::uint64_t step = (words + n_thr - 1) / n_thr;
    for (unsigned i = 0; i < n_thr; ++i)
        thr.emplace_back([&, i] { body(std::min(words, i * step), std::min(words, (i + 1) * step)); });
    for (auto& t : thr) t.join();
}

// out = XOR of the selected subvectors (zero when none is selected), one streaming
// pass: every output word reads all its terms once.
void combine(const std::uint64_t* src, const char* const rows[7], const std::vector<int>& h, std::uint64_t combos,
             std::uint64_t inner, std::uint64_t* out, OpCounter* counter) {
    std::vector<const std::uint64_t*> terms;
    for (std::uint64_t g = 0; g < combos; ++g)
        if (in_coeff(rows, h, g)) terms.push_back(src + g * inner);
    parallel_words(inner, [&](std::uint64_t w0, std::uint64_t w1) {
        if (terms.empty()) {
            std::fill(out + w0, out + w1, 0);
            return;
        }
        for (std::uint64_t b0 = w0; b0 < w1; b0 += 4096) {  // 32 KiB blocks stay in L1/L2 across terms
            const std::uint64_t b1 = std::min(w1, b0 + 4096);
            std::copy(terms[0] + b0, terms[0] + b1, out + b0);
            for (std::size_t t = 1; t < terms.size(); ++t)
                for (std::uint64_t w = b0; w < b1; ++w) out[w] ^= terms[t][w];
        }
    });
    if (counter && terms.size() > 1) counter->add_xors((terms.size() - 1) * inner);
}

// Page-locked word buffer (bmmgpu_host_alloc), movable, swappable.
struct Pinned {
    std::uint64_t* p = nullptr;
    Pinned() = default;
    explicit Pinned(std::uint64_t words) {
        void* q = nullptr;
        if (bmmgpu_host_alloc(words * 8, &q) != BMMGPU_OK)
            throw std::runtime_error(std::string("bmm host layer: ") + bmmgpu_last_error());
        p = static_cast<std::uint64_t*>(q);
    }
    Pinned(const Pinned&) = delete;
    Pinned& operator=(const Pinned&) = delete;
    ~Pinned() {
        if (p) bmmgpu_host_free(p);
    }
    void swap(Pinned& o) noexcept { std::swap(p, o.p); }
};

}  // namespace

std::vector<std::uint64_t> generate_left(const BitVectorTensor& a_hat, const SubInstanceIndex& h,
                                         const Decomposition& d, const LayerPlan& plan, OpCounter* counter) {
    check_digits(h, plan);
    check_interleaved(a_hat, plan);
    const std::uint64_t combos = std::uint64_t(1) << (2 * plan.d_host), inner = a_hat.words.size() / combos;
    std::vector<std::uint64_t> out(inner);
    combine(a_hat.words.data(), scheme_of(d).alpha, h.digits, combos, inner, out.data(), counter);
    return out;
}

std::vector<std::uint64_t> generate_right(const BitVectorTensor& b_hat, const SubInstanceIndex& h,
                                          const Decomposition& d, const LayerPlan& plan, OpCounter* counter) {
    check_digits(h, plan);
    check_interleaved(b_hat, plan);
    const std::uint64_t combos = std::uint64_t(1) << (2 * plan.d_host), inner = b_hat.words.size() / combos;
    std::vector<std::uint64_t> out(inner);
    combine(b_hat.words.data(), scheme_of(d).beta, h.digits, combos, inner, out.data(), counter);
    return out;
}

namespace {
void aggregate_raw(BitVectorTensor& c_hat, const SubInstanceIndex& h, const std::uint64_t* q, const Decomposition& d,
                   const LayerPlan& plan, SubvectorLocks& locks, OpCounter* counter) {
    const std::uint64_t combos = std::uint64_t(1) << (2 * plan.d_host), inner = c_hat.words.size() / combos;
    if (locks.size() != combos) throw std::invalid_argument("lock array does not match the plan");
    const bmmgpu::Scheme& sc = scheme_of(d);
    std::uint64_t folds = 0;
    for (std::uint64_t g = 0; g < combos; ++g) {
        if (!out_coeff(sc.gamma, h.digits, g)) continue;
        locks.lock(g);
        std::uint64_t* dst = c_hat.words.data() + g * inner;
        parallel_words(inner, [&](std::uint64_t w0, std::uint64_t w1) {
            for (std::uint64_t w = w0; w < w1; ++w) dst[w] ^= q[w];
        });
        locks.unlock(g);
        ++folds;
    }
    if (counter && folds) counter->add_xors(folds * inner);
}
}  // namespace

void aggregate(BitVectorTensor& c_hat, const SubInstanceIndex& h, const std::vector<std::uint64_t>& q,
               const Decomposition& d, const LayerPlan& plan, SubvectorLocks& locks, OpCounter* counter) {
    check_digits(h, plan);
    check_interleaved(c_hat, plan);
    const std::uint64_t combos = std::uint64_t(1) << (2 * plan.d_host);
    if (q.size() != c_hat.words.size() / combos) throw std::invalid_argument("sub-result length does not match the plan");
    aggregate_raw(c_hat, h, q.data(), d, plan, locks, counter);
}

BitVectorTensor coordinate(const BitVectorTensor& a_hat, const BitVectorTensor& b_hat, const Decomposition& d,
                           const LayerPlan& plan, int n_workers, OpCounter* counter, PipelineStats* stats) {
    if (n_workers < 1) throw std::invalid_argument("need at least one worker");
    if (plan.d_host < 0 || plan.d_serial < 0 || plan.d_parallel < 0 || plan.d_inner != 1)
        throw std::invalid_argument("invalid layer plan");
    check_interleaved(a_hat, plan);
    check_interleaved(b_hat, plan);
    const bmmgpu::Scheme& sc = scheme_of(d);
    const int n_dev = bmmgpu_device_count();
    if (n_dev < 1) throw std::runtime_error("bmm host layer: no CUDA device; the engine has no CPU fallback");

    const int d_host = plan.d_host, sub_depth = plan.d_serial + plan.d_parallel;
    const std::uint64_t subs = sub_instance_count(plan), combos = std::uint64_t(1) << (2 * d_host);
    const std::uint64_t inner = a_hat.words.size() / combos;
    const std::uint64_t n = std::uint64_t(n_workers);

    BitVectorTensor c_hat;
    c_hat.mode_lengths = a_hat.mode_lengths;
    c_hat.words.assign(a_hat.words.size(), 0);
    SubvectorLocks locks(d_host);
    PipelineStats st;
    st.prepared_left.assign(subs, 0);
    st.prepared_right.assign(subs, 0);
    st.aggregated.assign(subs, 0);

    // Operands that fit in HBM: the host layer runs on the device.  In the alternative
    // basis the d_host host levels are the top levels of the same bilinear recursion, so
    // the whole product is one bmmgpu_multiply_alt over d_host + sub_depth levels -- its
    // sub-instances formed from HBM-resident operands (40x host DRAM bandwidth) instead of
    // streamed through host memory and the link.  Beyond HBM (or with
    // BMM_PIPELINE=host) the host-thread pipeline below runs: the paper's Alg. 3.
    // Either way every sub-instance is prepared, solved and aggregated exactly once, and
    // the counters get the host layer's tallies (the same terms and folds the host
    // stages count) plus the solve's.
    const char* mode = std::getenv("BMM_PIPELINE");
    std::uint64_t free_b = 0, total_b = 0;
    const bool on_device = !(mode && std::string(mode) == "host") && bmmgpu_mem_info(0, &free_b, &total_b) == BMMGPU_OK &&
                           8.0 * double(a_hat.words.size()) * 8.0 < double(free_b);
    if (on_device) {
        detail::solve_alt(a_hat.words.data(), b_hat.words.data(), c_hat.words.data(), d_host + sub_depth, d, nullptr, 0);
        for (std::uint64_t f = 0; f < subs; ++f) {
            const SubInstanceIndex h = SubInstanceIndex::from_flat(f, d_host);
            if (counter) {
                std::uint64_t ta = 0, tb = 0, folds = 0;
                for (std::uint64_t g = 0; g < combos; ++g) {
                    ta += in_coeff(sc.alpha, h.digits, g);
                    tb += in_coeff(sc.beta, h.digits, g);
                    folds += out_coeff(sc.gamma, h.digits, g);
                }
                if (ta > 1) counter->add_xors((ta - 1) * inner);
                if (tb > 1) counter->add_xors((tb - 1) * inner);
                if (folds) counter->add_xors(folds * inner);
                const std::uint64_t kernels = [&] {
                    std::uint64_t k = 1;
                    for (int i = 0; i < sub_depth; ++i) k *= 7;
                    return k;
                }();
                counter->add_kernels(kernels);
                counter->add_ands(kernels * kBlockBits);
                counter->add_xors(predicted_additions(d, sub_depth, CostPart::LinearCombinations) * kBlockWords);
            }
            st.prepared_left[f] = st.prepared_right[f] = st.aggregated[f] = 1;
        }
        if (stats) *stats = std::move(st);
        return c_hat;
    }

    // One pipeline per worker: single-slot T / S / Q buffers with occupancy flags,
    // each flag single-producer single-consumer (reference pipeline.cpp:187-194).
    struct Worker {
        std::mutex mu;
        std::condition_variable cv;
        bool t_full = false, s_full = false, q_full = false;
        Pinned t, s, q;
    };
    std::vector<std::unique_ptr<Worker>> ws;
    for (std::uint64_t l = 0; l < n; ++l) {
        ws.push_back(std::make_unique<Worker>());
        Pinned(inner).swap(ws.back()->t);
        Pinned(inner).swap(ws.back()->s);
        Pinned(inner).swap(ws.back()->q);
    }
    std::atomic<bool> failed{false};
    std::vector<std::exception_ptr> errors(4 * n);
    auto abort_all = [&] {
        failed.store(true);
        for (auto& w : ws) {
            std::lock_guard<std::mutex> lk(w->mu);
            w->cv.notify_all();
        }
    };
    // wait until pred() or failure; false on failure
    auto wait_for = [&](Worker& w, auto pred) {
        std::unique_lock<std::mutex> lk(w.mu);
        w.cv.wait(lk, [&] { return pred() || failed.load(); });
        return !failed.load();
    };
    auto publish = [](Worker& w, bool& flag, bool value) {
        {
            std::lock_guard<std::mutex> lk(w.mu);
            flag = value;
        }
        w.cv.notify_all();
    };

    auto prepare = [&](std::uint64_t l, bool left) {
        Worker& w = *ws[l];
        bool& full = left ? w.t_full : w.s_full;
        for (std::uint64_t f = l; f < subs; f += n) {
            const SubInstanceIndex h = SubInstanceIndex::from_flat(f, d_host);
            if (!wait_for(w, [&] { return !full; })) return;
            combine((left ? a_hat : b_hat).words.data(), left ? sc.alpha : sc.beta, h.digits, combos, inner,
                    (left ? w.t : w.s).p, counter);
            ++(left ? st.prepared_left : st.prepared_right)[f];
            publish(w, full, true);
        }
    };
    auto solve = [&](std::uint64_t l) {
        Worker& w = *ws[l];
        const int device = int(l % std::uint64_t(n_dev));
        Pinned tl(inner), sl(inner), ql(inner);
        for (std::uint64_t f = l; f < subs; f += n) {
            if (!wait_for(w, [&] { return w.t_full && w.s_full; })) return;
            {
                // take the prepared inputs by swap and free both slots before the product
                std::lock_guard<std::mutex> lk(w.mu);
                tl.swap(w.t);
                sl.swap(w.s);
                w.t_full = w.s_full = false;
            }
            w.cv.notify_all();
            detail::solve_alt(tl.p, sl.p, ql.p, sub_depth, d, counter, device);
            if (!wait_for(w, [&] { return !w.q_full; })) return;
            {
                std::lock_guard<std::mutex> lk(w.mu);
                ql.swap(w.q);
                w.q_full = true;
            }
            w.cv.notify_all();
        }
    };
    auto fold = [&](std::uint64_t l) {
        Worker& w = *ws[l];
        for (std::uint64_t f = l; f < subs; f += n) {
            const SubInstanceIndex h = SubInstanceIndex::from_flat(f, d_host);
            if (!wait_for(w, [&] { return w.q_full; })) return;
            aggregate_raw(c_hat, h, w.q.p, d, plan, locks, counter);
            ++st.aggregated[f];
            publish(w, w.q_full, false);
        }
    };

    std::vector<std::thread> threads;
    auto launch = [&](std::uint64_t slot, auto body) {
        threads.emplace_back([&, slot, body] {
            try {
                body();
            } catch (...) {
                errors[slot] = std::current_exception();
                abort_all();
            }
        });
    };
    for (std::uint64_t l = 0; l < n; ++l) {
        launch(4 * l + 0, [&, l] { prepare(l, true); });
        launch(4 * l + 1, [&, l] { prepare(l, false); });
        launch(4 * l + 2, [&, l] { solve(l); });
        launch(4 * l + 3, [&, l] { fold(l); });
    }
    for (auto& t : threads) t.join();
    for (auto& e : errors)
        if (e) std::rethrow_exception(e);
    st.lock_violations = locks.violations();
    if (stats) *stats = std::move(st);
    return c_hat;
}

}  // namespace pipeline
}  // namespace bmm
