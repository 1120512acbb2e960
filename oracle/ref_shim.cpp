// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library (bmm_core, compiled by oracle/Makefile straight from
// /root/reference/proj/src into oracle/_ref/libbmmref.so).
//
// TEST / BASELINE INFRASTRUCTURE ONLY: loaded by tests/ (to pin the oracle and
// generate golden vectors) and by bench.py's cpu_baseline and --impl reference
// legs.  Never part of the product path.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "bmm/bitmatrix.hpp"
#include "bmm/counter.hpp"
#include "bmm/decomposition.hpp"
#include "bmm/engine.hpp"
#include "bmm/pipeline.hpp"
#include "bmm/plan.hpp"

using namespace bmm;

namespace {
thread_local std::string g_err;

BitMatrix wrap(const std::uint64_t* w, std::uint64_t rows, std::uint64_t cols) {
    BitMatrix m = BitMatrix::zeros(rows, cols);
    std::memcpy(m.words.data(), w, m.words.size() * 8);
    return m;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 3;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}
}  // namespace

extern "C" {

const char* bmmref_last_error() { return g_err.c_str(); }

// BitMatrix::random (bitmatrix.cpp:64-77)
void bmmref_random(std::uint64_t rows, std::uint64_t cols, std::uint64_t seed, std::uint64_t* out) {
    BitMatrix m = BitMatrix::random(rows, cols, seed);
    std::memcpy(out, m.words.data(), m.words.size() * 8);
}

// multiply_cubic (engine.cpp:132-144). counts: optional [ands, xors, ors, kernels]
int bmmref_multiply_cubic(const std::uint64_t* a, const std::uint64_t* b, std::uint64_t* c, std::uint64_t m,
                          std::uint64_t k, std::uint64_t n, int ring, int workers, std::uint64_t* counts) {
    return guard([&] {
        OpCounter ctr;
        BitMatrix am = wrap(a, m, k), bm = wrap(b, k, n);
        BitMatrix cm = multiply_cubic(am, bm, ring == 1 ? Semiring::Gf2XorAnd : Semiring::BooleanOrAnd,
                                      workers, counts ? &ctr : nullptr);
        std::memcpy(c, cm.words.data(), cm.words.size() * 8);
        if (counts) {
            counts[0] = ctr.word_ands;
            counts[1] = ctr.word_xors;
            counts[2] = ctr.word_ors;
            counts[3] = ctr.kernel_invocations;
        }
    });
}

// multiply (engine.cpp:351-382). algo: 0 cubic, 1 sw, 2 alt-si, 3 alt-chain
int bmmref_multiply(const std::uint64_t* a, const std::uint64_t* b, std::uint64_t* c, std::uint64_t n, int algo,
                    int d_host, int d_serial, int d_parallel, int workers, int ring, std::uint64_t* counts) {
    return guard([&] {
        LayerPlan plan;
        plan.d_host = d_host;
        plan.d_serial = d_serial;
        plan.d_parallel = d_parallel;
        plan.workers = workers;
        OpCounter ctr;
        BitMatrix am = wrap(a, n, n), bm = wrap(b, n, n);
        BitMatrix cm = multiply(am, bm, static_cast<Algo>(algo), plan,
                                ring == 1 ? Semiring::Gf2XorAnd : Semiring::BooleanOrAnd, counts ? &ctr : nullptr);
        std::memcpy(c, cm.words.data(), cm.words.size() * 8);
        if (counts) {
            counts[0] = ctr.word_ands;
            counts[1] = ctr.word_xors;
            counts[2] = ctr.word_ors;
            counts[3] = ctr.kernel_invocations;
        }
    });
}

// auto_plan (engine.cpp:13-22): out = {d_host, d_serial, d_parallel}
int bmmref_auto_plan(std::uint64_t n, int workers, int* out) {
    return guard([&] {
        LayerPlan p = LayerPlan::auto_plan(n, workers);
        out[0] = p.d_host;
        out[1] = p.d_serial;
        out[2] = p.d_parallel;
    });
}

// transpose_blocks64 (bitmatrix.cpp:97-110), in place
int bmmref_transpose_blocks64(std::uint64_t rows, std::uint64_t cols, std::uint64_t* w) {
    return guard([&] {
        BitMatrix m = wrap(w, rows, cols);
        transpose_blocks64(m);
        std::memcpy(w, m.words.data(), m.words.size() * 8);
    });
}

// to_interleaved / from_interleaved (bitmatrix.cpp:124-173) with plan.d_serial = depth
int bmmref_to_interleaved(int depth, int which, const std::uint64_t* m, std::uint64_t* t) {
    return guard([&] {
        LayerPlan plan;
        plan.d_serial = depth;
        const std::uint64_t n = plan.matrix_dim();
        BitVectorTensor v = to_interleaved(wrap(m, n, n), plan, static_cast<Operand>(which));
        std::memcpy(t, v.words.data(), v.words.size() * 8);
    });
}

int bmmref_from_interleaved(int depth, int which, const std::uint64_t* t, std::uint64_t* m) {
    return guard([&] {
        LayerPlan plan;
        plan.d_serial = depth;
        const std::uint64_t n = plan.matrix_dim();
        BitVectorTensor v;
        v.mode_lengths.assign(depth, 4);
        v.mode_lengths.push_back(kBlockBits);
        v.words.assign(t, t + n * n / 64);
        BitMatrix r = from_interleaved(v, plan, static_cast<Operand>(which));
        std::memcpy(m, r.words.data(), r.words.size() * 8);
    });
}

// basis_change (engine.cpp:146-172) of the alt-si scheme; which 0 Phi 1 Psi 2 Chi
int bmmref_basis_change(std::uint64_t* v, int depth, int which, int scheme) {
    return guard([&] {
        const Decomposition& d = builtin(static_cast<Builtin>(scheme));
        BitVectorTensor t;
        t.mode_lengths.assign(depth, 4);
        t.mode_lengths.push_back(kBlockBits);
        const std::uint64_t words = (std::uint64_t{64} << depth) * (std::uint64_t{64} << depth) / 64;
        t.words.assign(v, v + words);
        basis_change(t, d, static_cast<BasisFactor>(which), depth);
        std::memcpy(v, t.words.data(), words * 8);
    });
}

// multiply_alt (engine.cpp:293-349)
int bmmref_multiply_alt(const std::uint64_t* a_hat, const std::uint64_t* b_hat, std::uint64_t* c_hat, int d_serial,
                        int d_parallel, int workers, int scheme) {
    return guard([&] {
        const Decomposition& d = builtin(static_cast<Builtin>(scheme));
        LayerPlan plan;
        plan.d_serial = d_serial;
        plan.d_parallel = d_parallel;
        plan.workers = workers;
        const int depth = d_serial + d_parallel;
        const std::uint64_t words = (std::uint64_t{64} << depth) * (std::uint64_t{64} << depth) / 64;
        BitVectorTensor a, b;
        a.mode_lengths.assign(depth, 4);
        a.mode_lengths.push_back(kBlockBits);
        b.mode_lengths = a.mode_lengths;
        a.words.assign(a_hat, a_hat + words);
        b.words.assign(b_hat, b_hat + words);
        BitVectorTensor c = multiply_alt(a, b, d, plan);
        std::memcpy(c_hat, c.words.data(), words * 8);
    });
}

// pipeline::coordinate (pipeline.cpp:198-369) on hat vectors of depth d_host + d_serial +
// d_parallel; counts: optional [ands, xors, ors, kernels]
int bmmref_coordinate(const std::uint64_t* a_hat, const std::uint64_t* b_hat, std::uint64_t* c_hat, int d_host,
                      int d_serial, int d_parallel, int workers, int scheme, std::uint64_t* counts) {
    return guard([&] {
        const Decomposition& d = builtin(static_cast<Builtin>(scheme));
        LayerPlan plan;
        plan.d_host = d_host;
        plan.d_serial = d_serial;
        plan.d_parallel = d_parallel;
        plan.workers = 1;
        const int depth = d_host + d_serial + d_parallel;
        const std::uint64_t words = (std::uint64_t{64} << depth) * (std::uint64_t{64} << depth) / 64;
        BitVectorTensor a, b;
        a.mode_lengths.assign(depth, 4);
        a.mode_lengths.push_back(kBlockBits);
        b.mode_lengths = a.mode_lengths;
        a.words.assign(a_hat, a_hat + words);
        b.words.assign(b_hat, b_hat + words);
        OpCounter ctr;
        BitVectorTensor c = pipeline::coordinate(a, b, d, plan, workers, counts ? &ctr : nullptr);
        std::memcpy(c_hat, c.words.data(), words * 8);
        if (counts) {
            counts[0] = ctr.word_ands;
            counts[1] = ctr.word_xors;
            counts[2] = ctr.word_ors;
            counts[3] = ctr.kernel_invocations;
        }
    });
}

// kernel64 (engine.cpp:34-56)
void bmmref_kernel64(const std::uint64_t* a, const std::uint64_t* bt, std::uint64_t* out, int ring) {
    kernel64(a, bt, out, ring == 1 ? Semiring::Gf2XorAnd : Semiring::BooleanOrAnd);
}

// read_bmm1 / write_bmm1 (bitmatrix.cpp:187-233). read: dims first (words==nullptr), then data.
int bmmref_read_bmm1(const char* path, std::uint64_t* rows, std::uint64_t* cols, std::uint64_t* words) {
    return guard([&] {
        BitMatrix m = read_bmm1(path);
        *rows = m.rows;
        *cols = m.cols;
        if (words) std::memcpy(words, m.words.data(), m.words.size() * 8);
    });
}

int bmmref_write_bmm1(const char* path, std::uint64_t rows, std::uint64_t cols, const std::uint64_t* words) {
    return guard([&] { write_bmm1(wrap(words, rows, cols), path); });
}

// predicted_additions (decomposition.cpp:509-531); part 0 BasisChanges 1 LinearCombinations
std::uint64_t bmmref_predicted_additions(int scheme, int depth, int part) {
    return predicted_additions(builtin(static_cast<Builtin>(scheme)), depth, static_cast<CostPart>(part));
}

}  // extern "C"
