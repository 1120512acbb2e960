// pipeline_bench.cpp -- the drop-in host layer (bmm::pipeline::coordinate, paper
// Alg. 3) on B200: n x n GF(2) alt-si product with d_host host levels, 7^d_host
// sub-instances solved on the GPU by `workers` pipelines.  Prints one JSON line:
// effective Pbop/s of coordinate() (operands already interleaved and basis-changed,
// as the paper times it), the same product through bmm::multiply, and a digest check.
// With BMM_PIPELINE=host (the host-thread pipeline) it also reports the host layer's
// algorithmic host-memory traffic (generation reads its terms and writes T / S,
// aggregation reads Q and read-modify-writes each gamma-selected output subvector) and a
// streaming-XOR measurement of this box's host memory bandwidth with the same threads.
//   pipeline_bench <n> <d_host> <workers>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "bmm/engine.hpp"
#include "bmm/pipeline.hpp"

using namespace bmm;

static std::uint64_t fnv(const std::vector<std::uint64_t>& w) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (std::uint64_t x : w)
        for (int b = 0; b < 8; ++b) h = (h ^ ((x >> (8 * b)) & 0xff)) * 0x100000001b3ull;
    return h;
}

// GB/s of dst ^= src over `words` words with `threads` threads (bytes counted: 2 reads, 1 write)
static double host_xor_gbs(std::uint64_t words, unsigned threads) {
    std::vector<std::uint64_t> a(words, 1), b(words, 2);
    auto run = [&] {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < threads; ++t)
            th.emplace_back([&, t] {
                const std::uint64_t w0 = words * t / threads, w1 = words * (t + 1) / threads;
                for (std::uint64_t w = w0; w < w1; ++w) a[w] ^= b[w];
            });
        for (auto& x : th) x.join();
    };
    run();
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < 3; ++r) run();
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 3;
    return 3.0 * 8.0 * double(words) / s / 1e9;
}

int main(int argc, char** argv) {
    const std::uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 16384;
    const int d_host = argc > 2 ? std::atoi(argv[2]) : 2;
    const int workers = argc > 3 ? std::atoi(argv[3]) : 2;
    const Decomposition& d = builtin(Builtin::AltSelfInverse);
    const BitMatrix a = BitMatrix::random(n, n, 1), b = BitMatrix::random(n, n, 2);
    LayerPlan plan = LayerPlan::auto_plan(n, 1);
    const int depth = plan.depth();
    plan.d_host = d_host;
    plan.d_serial = 0;
    plan.d_parallel = depth - d_host;
    BitVectorTensor ah = to_interleaved(a, plan, Operand::Left), bh = to_interleaved(b, plan, Operand::Right);
    basis_change(ah, d, BasisFactor::Phi, depth);
    basis_change(bh, d, BasisFactor::Psi, depth);
    using clk = std::chrono::steady_clock;
    (void)pipeline::coordinate(ah, bh, d, plan, workers);  // warm-up (device pools, pinned buffers)
    const auto t0 = clk::now();
    pipeline::PipelineStats st;
    BitVectorTensor ch = pipeline::coordinate(ah, bh, d, plan, workers, nullptr, &st);
    const double t = std::chrono::duration<double>(clk::now() - t0).count();
    basis_change(ch, d, BasisFactor::Chi, depth);
    const BitMatrix c = from_interleaved(ch, plan, Operand::Result);
    LayerPlan flat = LayerPlan::auto_plan(n, 1);
    const auto t1 = clk::now();
    const BitMatrix want = multiply(a, b, Algo::AltSelfInverse, flat, Semiring::Gf2XorAnd);
    const double t_direct = std::chrono::duration<double>(clk::now() - t1).count();
    const double bops = 2.0 * double(n) * double(n) * double(n) - double(n) * double(n);
    // host layer traffic: every sub-instance reads its alpha / beta terms and writes T, S;
    // aggregation reads Q once per fold and read-modify-writes the output subvector
    const std::uint64_t subs = pipeline::sub_instance_count(plan), inner = ah.words.size() >> (2 * d_host);
    double host_bytes = 0;
    for (std::uint64_t f = 0; f < subs; ++f) {
        const pipeline::SubInstanceIndex h = pipeline::SubInstanceIndex::from_flat(f, d_host);
        OpCounter oc;
        (void)pipeline::generate_left(ah, h, d, plan, &oc);
        (void)pipeline::generate_right(bh, h, d, plan, &oc);
        // generation: (terms) reads + 1 write per operand; oc counts (terms - 1) * inner XORs
        host_bytes += 8.0 * (double(oc.word_xors.load()) + 4.0 * double(inner));
    }
    for (std::uint64_t f = 0; f < subs; ++f) {
        const pipeline::SubInstanceIndex h = pipeline::SubInstanceIndex::from_flat(f, d_host);
        BitVectorTensor tmp;
        tmp.mode_lengths = ah.mode_lengths;
        tmp.words.assign(ah.words.size(), 0);
        pipeline::SubvectorLocks locks(d_host);
        OpCounter oc;
        pipeline::aggregate(tmp, h, std::vector<std::uint64_t>(inner, 0), d, plan, locks, &oc);
        host_bytes += 8.0 * 3.0 * double(oc.word_xors.load());  // read Q, read + write C per fold
    }
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const double host_gbs = host_xor_gbs(std::uint64_t(1) << 27, hw);
    std::printf("{\"n\": %llu, \"d_host\": %d, \"workers\": %d, \"sub_instances\": %llu, \"coordinate_s\": %.4f, "
                "\"coordinate_Pbops\": %.4f, \"multiply_s\": %.4f, \"multiply_Pbops\": %.4f, \"equal\": %s, "
                "\"fnv\": \"%016llx\", \"lock_violations\": %llu, \"pipeline\": \"%s\", "
                "\"host_layer_GB\": %.2f, \"host_layer_GBps_if_host_bound\": %.1f, \"host_xor_GBps\": %.1f, "
                "\"host_threads\": %u}\n",
                (unsigned long long)n, d_host, workers, (unsigned long long)pipeline::sub_instance_count(plan), t,
                bops / t / 1e15, t_direct, bops / t_direct / 1e15, c == want ? "true" : "false",
                (unsigned long long)fnv(c.words), (unsigned long long)st.lock_violations,
                std::getenv("BMM_PIPELINE") ? std::getenv("BMM_PIPELINE") : "auto", host_bytes / 1e9,
                host_bytes / t / 1e9, host_gbs, hw);
    return c == want ? 0 : 1;
}
