// pipeline_bench.cpp -- the drop-in host layer (bmm::pipeline::coordinate, paper
// Alg. 3) on B200: n x n GF(2) alt-si product with d_host host levels, 7^d_host
// sub-instances solved on the GPU by `workers` pipelines.  Prints one JSON line:
// effective Pbop/s of coordinate() (operands already interleaved and basis-changed,
// as the paper times it), the same product through bmm::multiply, and a digest check.
//   pipeline_bench <n> <d_host> <workers>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "bmm/engine.hpp"
#include "bmm/pipeline.hpp"

using namespace bmm;

static std::uint64_t fnv(const std::vector<std::uint64_t>& w) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (std::uint64_t x : w)
        for (int b = 0; b < 8; ++b) h = (h ^ ((x >> (8 * b)) & 0xff)) * 0x100000001b3ull;
    return h;
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
    std::printf("{\"n\": %llu, \"d_host\": %d, \"workers\": %d, \"sub_instances\": %llu, \"coordinate_s\": %.4f, "
                "\"coordinate_Pbops\": %.4f, \"multiply_s\": %.4f, \"multiply_Pbops\": %.4f, \"equal\": %s, "
                "\"fnv\": \"%016llx\", \"lock_violations\": %llu}\n",
                (unsigned long long)n, d_host, workers, (unsigned long long)pipeline::sub_instance_count(plan), t,
                bops / t / 1e15, t_direct, bops / t_direct / 1e15, c == want ? "true" : "false",
                (unsigned long long)fnv(c.words), (unsigned long long)st.lock_violations);
    return c == want ? 0 : 1;
}
