// engine.cpp -- the drop-in bmm:: engine entry points (include/bmm/engine.hpp)
// over the C ABI (include/bmmgpu.h).  Validation and exception types follow
// the reference (src/engine.cpp); every product runs on the GPU, and the
// OpCounter tallies are filled with the reference algorithm's exact counts.
#include "bmm/engine.hpp"

#include <algorithm>
#include <bit>
#include <stdexcept>
#include <string>

#include "bmmgpu.h"
#include "../schemes.h"

namespace bmm {

namespace {

[[noreturn]] void raise(int status) {
    const std::string msg = bmmgpu_last_error();
    switch (status) {
        case BMMGPU_ESHAPE: throw ShapeError(msg);
        case BMMGPU_EINVAL: throw std::invalid_argument(msg);
        default: throw std::runtime_error("bmm GPU engine: " + msg);
    }
}

void check(int status) {
    if (status != BMMGPU_OK) raise(status);
}

std::uint64_t ipow(std::uint64_t b, int e) {
    std::uint64_t v = 1;
    while (e-- > 0) v *= b;
    return v;
}

int algo_id(Builtin b) {
    switch (b) {
        case Builtin::StrassenWinograd: return BMMGPU_ALGO_STRASSEN_WINOGRAD;
        case Builtin::AltSelfInverse: return BMMGPU_ALGO_ALT_SELF_INVERSE;
        case Builtin::AltChaining: return BMMGPU_ALGO_ALT_CHAINING;
        case Builtin::Elementary: break;
    }
    throw std::invalid_argument("engine layers require <2,2,2>_7 schemes");
}

bool factor_identity(const Decomposition& d, BasisFactor f) {
    return (f == BasisFactor::Phi ? d.adds_phi : f == BasisFactor::Psi ? d.adds_psi : d.adds_chi) == 0;
}

int factor_id(BasisFactor f) { return f == BasisFactor::Phi ? 0 : f == BasisFactor::Psi ? 1 : 2; }

// Reference SLP addition counts (decomposition.cpp:57-216).
const Decomposition kSw{Builtin::StrassenWinograd, {2, 2, 2, 7}, {true, true}, 4, 4, 7, 0, 0, 0};
const Decomposition kAsi{Builtin::AltSelfInverse, {2, 2, 2, 7}, {true, false}, 3, 3, 6, 2, 2, 2};
const Decomposition kAch{Builtin::AltChaining, {2, 2, 2, 7}, {false, true}, 3, 3, 6, 2, 2, 2};
const Decomposition kEl{Builtin::Elementary, {2, 2, 2, 8}, {true, true}, 0, 0, 4, 0, 0, 0};

std::vector<std::uint64_t> modes_for(int depth) {
    std::vector<std::uint64_t> m(depth, 4);
    m.push_back(kBlockBits);
    return m;
}

}  // namespace

LayerPlan LayerPlan::auto_plan(std::uint64_t n, int workers) {
    if (n < kBlockDim || !std::has_single_bit(n)) throw ShapeError("matrix dimension must be 64 * 2^k");
    const int k = std::countr_zero(n) - 6;
    LayerPlan p;
    p.d_parallel = k < 3 ? k : 3;
    p.d_serial = k - p.d_parallel;
    p.workers = workers < 1 ? 1 : workers;
    return p;
}

const Decomposition& builtin(Builtin which) {
    switch (which) {
        case Builtin::StrassenWinograd: return kSw;
        case Builtin::AltSelfInverse: return kAsi;
        case Builtin::AltChaining: return kAch;
        case Builtin::Elementary: return kEl;
    }
    throw std::invalid_argument("unknown builtin decomposition");
}

std::uint64_t predicted_additions(const Decomposition& d, int depth, CostPart part) {
    const TripleParams& p = d.params;
    if (p.s != p.t || p.t != p.u) throw std::invalid_argument("addition prediction needs s = t = u");
    const std::uint64_t s2 = std::uint64_t(p.s) * p.s;
    if (std::uint64_t(p.r) <= s2) throw std::invalid_argument("addition prediction needs r > s^2");
    if (depth < 0) throw std::invalid_argument("negative depth");
    if (depth == 0) return 0;
    if (part == CostPart::BasisChanges)
        return std::uint64_t(d.adds_phi + d.adds_psi + d.adds_chi) * ipow(s2, depth - 1) * depth;
    std::uint64_t geo = 0;
    for (int l = 0; l < depth; ++l) geo += ipow(s2, l) * ipow(p.r, depth - 1 - l);
    return std::uint64_t(d.adds_alpha + d.adds_beta + d.adds_gamma) * geo;
}

const Decomposition& decomposition_for(Algo algo) {
    switch (algo) {
        case Algo::StrassenWinograd: return kSw;
        case Algo::AltSelfInverse: return kAsi;
        case Algo::AltChaining: return kAch;
        case Algo::Cubic: break;
    }
    throw std::invalid_argument("the cubic algorithm has no bilinear scheme");
}

void kernel64(const std::uint64_t* a, const std::uint64_t* b_transposed, std::uint64_t* out, Semiring ring) {
    // one launch on page-locked mapped staging (K9, csrc/kernel64.cu); b_transposed is B
    // column-major, exactly the reference's operand form
    check(bmmgpu_kernel64(a, b_transposed, out, ring == Semiring::Gf2XorAnd ? BMMGPU_GF2_XOR_AND : BMMGPU_BOOLEAN_OR_AND));
}

BitMatrix multiply_cubic(const BitMatrix& a, const BitMatrix& b, Semiring ring, int workers, OpCounter* counter) {
    if (a.cols != b.rows) throw ShapeError("inner dimensions differ");
    (void)workers;
    BitMatrix c = BitMatrix::zeros(a.rows, b.cols);
    const bool gf2 = ring == Semiring::Gf2XorAnd;
    check(bmmgpu_cubic(a.words.data(), b.words.data(), c.words.data(), a.rows, a.cols, b.cols,
                       gf2 ? BMMGPU_GF2_XOR_AND : BMMGPU_BOOLEAN_OR_AND, nullptr));
    if (counter) {
        const bool blocked = a.rows % kBlockDim == 0 && a.cols % kBlockDim == 0 && b.cols % kBlockDim == 0;
        if (blocked) {
            // cubic_blocked tallies (reference engine.cpp:89-98)
            const std::uint64_t pairs = (a.rows / kBlockDim) * (b.cols / kBlockDim), bj = a.cols / kBlockDim;
            counter->add_kernels(pairs * bj);
            counter->add_ands(pairs * bj * kBlockBits);
            const std::uint64_t folds = bj ? pairs * (bj - 1) * kBlockWords : 0;
            gf2 ? counter->add_xors(folds) : counter->add_ors(folds);
        } else {
            // cubic_rowwise tallies: one row fold per set bit of A (engine.cpp:108-126)
            std::uint64_t ones = 0;
            for (std::uint64_t w : a.words) ones += std::popcount(w);
            const std::uint64_t n = ones * c.words_per_row();
            gf2 ? counter->add_xors(n) : counter->add_ors(n);
        }
    }
    return c;
}

void basis_change(BitVectorTensor& v, const Decomposition& d, BasisFactor which, int levels, int workers,
                  OpCounter* counter) {
    (void)workers;
    if (levels < 0 || v.mode_lengths.size() < static_cast<std::size_t>(levels) + 1)
        throw std::invalid_argument("vector has fewer modes than basis levels");
    for (int l = 0; l < levels; ++l)
        if (v.mode_lengths[l] != 4) throw std::invalid_argument("mode length does not match the basis");
    if (v.words.size() * kWordBits != v.bit_length())
        throw std::invalid_argument("vector storage does not match its modes");
    if (factor_identity(d, which) || levels == 0) return;
    check(bmmgpu_basis_change(v.words.data(), v.words.size(), levels, algo_id(d.which), factor_id(which), 0));
    if (counter) {
        const int adds = which == BasisFactor::Phi ? d.adds_phi : which == BasisFactor::Psi ? d.adds_psi : d.adds_chi;
        counter->add_xors(std::uint64_t(levels) * (v.words.size() / 4) * adds);
    }
}

namespace detail {

// The device solve of multiply_alt on raw interleaved buffers of depth `depth` (4^depth
// blocks of 64 words), on CUDA device `device`, with the reference's tallies: the
// whole sub-product runs on the GPU (inverse basis changes, Morton block permutes, the
// fast product, permute back, inverse chi).  Shared by multiply_alt and the pipeline's
// solve stage (reference pipeline.cpp:310).
void solve_alt(const std::uint64_t* a_hat, const std::uint64_t* b_hat, std::uint64_t* c_hat, int depth,
               const Decomposition& d, OpCounter* counter, int device) {
    bmmgpu_opts o{};
    o.device_mask = 1u << device;
    check(bmmgpu_multiply_alt(a_hat, b_hat, c_hat, depth, algo_id(d.which), &o));
    if (counter) {
        const std::uint64_t kernels = ipow(7, depth);
        counter->add_kernels(kernels);
        counter->add_ands(kernels * kBlockBits);
        counter->add_xors(predicted_additions(d, depth, CostPart::LinearCombinations) * kBlockWords);
    }
}

}  // namespace detail

// multiply_alt is the bilinear map (a_hat, b_hat) -> chi^-1( phi^-1 a_hat . psi^-1 b_hat )
// in interleaved form (reference engine.cpp:293-349).
BitVectorTensor multiply_alt(const BitVectorTensor& a_hat, const BitVectorTensor& b_hat, const Decomposition& d,
                             const LayerPlan& plan, OpCounter* counter) {
    if (plan.d_serial < 0 || plan.d_parallel < 0 || plan.d_inner != 1 || plan.workers < 1)
        throw std::invalid_argument("invalid layer plan");
    if (!(d.params == TripleParams{})) throw std::invalid_argument("engine layers require <2,2,2>_7 schemes");
    const int depth = plan.d_serial + plan.d_parallel;
    const std::vector<std::uint64_t> want = modes_for(depth);
    if (a_hat.mode_lengths != want || b_hat.mode_lengths != want)
        throw std::invalid_argument("operands are not interleaved for this plan");
    if (a_hat.words.size() * kWordBits != a_hat.bit_length() || b_hat.words.size() * kWordBits != b_hat.bit_length())
        throw std::invalid_argument("operand storage does not match its modes");
    BitVectorTensor c;
    c.mode_lengths = a_hat.mode_lengths;
    c.words.assign(a_hat.words.size(), 0);
    detail::solve_alt(a_hat.words.data(), b_hat.words.data(), c.words.data(), depth, d, counter, 0);
    return c;
}

BitMatrix multiply(const BitMatrix& a, const BitMatrix& b, Algo algo, const LayerPlan& plan, Semiring ring,
                   OpCounter* counter) {
    if (algo == Algo::Cubic) return multiply_cubic(a, b, ring, plan.workers, counter);
    if (ring == Semiring::BooleanOrAnd)
        throw std::invalid_argument(
            "the Boolean semiring has no subtraction, so cancellation-based fast algorithms are unsound over it; "
            "use the cubic algorithm");
    if (a.rows != a.cols || b.rows != b.cols || a.rows != b.rows)
        throw ShapeError("fast algorithms need equal square operands");
    if (a.rows < kBlockDim || !std::has_single_bit(a.rows)) throw ShapeError("fast algorithms need n = 64 * 2^k");
    if (plan.matrix_dim() != a.rows || plan.d_host < 0 || plan.d_serial < 0 || plan.d_parallel < 0 ||
        plan.d_inner != 1 || plan.workers < 1)
        throw std::invalid_argument("layer plan does not match the operands");
    const Decomposition& d = decomposition_for(algo);
    BitMatrix c = BitMatrix::zeros(a.rows, a.rows);
    bmmgpu_plan gp{plan.d_host, plan.d_serial, plan.d_parallel, plan.d_inner, plan.workers};
    // With host levels the reference runs pipeline::coordinate with plan.workers emulated
    // accelerators (engine.cpp:375-378); here the workers are GPUs: the host-layer
    // sub-instances are dealt over min(workers, devices) of them (bmmgpu_multiply).
    bmmgpu_opts opts{};
    if (plan.d_host > 0) {
        const int g = std::max(1, std::min(plan.workers, bmmgpu_device_count()));
        opts.device_mask = g >= 32 ? 0xffffffffu : (1u << g) - 1;
    }
    check(bmmgpu_multiply(a.words.data(), b.words.data(), c.words.data(), a.rows, algo_id(d.which), &gp,
                          BMMGPU_GF2_XOR_AND, &opts));
    if (counter) {
        const int depth = plan.depth();
        const std::uint64_t kernels = ipow(7, depth);
        counter->add_kernels(kernels);
        counter->add_ands(kernels * kBlockBits);
        std::uint64_t xors = predicted_additions(d, depth, CostPart::BasisChanges) * kBlockWords;
        if (plan.d_host == 0) {
            xors += predicted_additions(d, depth, CostPart::LinearCombinations) * kBlockWords;
        } else {
            // The reference runs the top d_host levels through pipeline::coordinate
            // (engine.cpp:375-378), which tallies folds, not SLP additions: per sub-instance
            // h, (nnz(alpha^(x)d_host row h) - 1) + (nnz(beta row h) - 1) generation folds and
            // nnz(gamma column h) aggregation folds of inner_words each (pipeline.cpp:108-179),
            // plus each sub-instance's multiply_alt at depth - d_host.  Summed over h the
            // Kronecker row weights factor: sum_h prod_l nnz(h_l) = (sum_h nnz(h))^d_host.
            const bmmgpu::Scheme* sc = bmmgpu::scheme_for(algo_id(d.which));
            std::uint64_t wa = 0, wb = 0, wg = 0;
            for (int h = 0; h < 7; ++h) {
                wa += std::popcount(bmmgpu::row_mask(sc->alpha[h]));
                wb += std::popcount(bmmgpu::row_mask(sc->beta[h]));
            }
            for (int q = 0; q < 4; ++q) wg += std::popcount(bmmgpu::row_mask(sc->gamma[q]));
            const std::uint64_t subs = ipow(7, plan.d_host);
            const std::uint64_t inner_words = (a.rows * a.rows / kWordBits) >> (2 * plan.d_host);
            xors += (ipow(wa, plan.d_host) - subs + ipow(wb, plan.d_host) - subs + ipow(wg, plan.d_host)) * inner_words;
            xors += subs * predicted_additions(d, depth - plan.d_host, CostPart::LinearCombinations) * kBlockWords;
        }
        counter->add_xors(xors);
    }
    return c;
}

BitMatrix multiply_strassen_winograd(const BitMatrix& a, const BitMatrix& b, const LayerPlan& plan, Semiring ring,
                                     OpCounter* counter) {
    return multiply(a, b, Algo::StrassenWinograd, plan, ring, counter);
}

BitVectorTensor chain_multiply(const std::vector<BitVectorTensor>& matrices_hat, const Decomposition& d,
                               const LayerPlan& plan, OpCounter* counter) {
    if (!d.traits.supports_chaining)
        throw std::invalid_argument("this scheme cannot chain: its output basis is not its input basis");
    if (matrices_hat.size() < 2) throw std::invalid_argument("a chain needs at least two operands");
    BitVectorTensor acc = multiply_alt(matrices_hat[0], matrices_hat[1], d, plan, counter);
    for (std::size_t i = 2; i < matrices_hat.size(); ++i) acc = multiply_alt(acc, matrices_hat[i], d, plan, counter);
    return acc;
}

}  // namespace bmm
