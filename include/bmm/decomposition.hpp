#pragma once
// Drop-in subset of the reference's include/bmm/decomposition.hpp: the scheme
// handles the engine entry points take (builtin(), Decomposition, traits) and
// predicted_additions() (reference decomposition.cpp:509-531), which the
// operation counters use.  The coefficient-algebra toolkit (Gf2Matrix, SLP
// evaluation, Kronecker/triple-product verification) is host-side algebra
// outside the product hot path and is not part of this engine.

#include <cstdint>

namespace bmm {

enum class Builtin { StrassenWinograd, AltSelfInverse, AltChaining, Elementary };

struct DecompositionTraits {
    bool self_inverse_bases = false;
    bool supports_chaining = false;
};

struct TripleParams {
    int s = 2;
    int t = 2;
    int u = 2;
    int r = 7;
    bool operator==(const TripleParams&) const = default;
};

// A <2,2,2;r> scheme.  The coefficient matrices live in the GPU engine
// (paper_1909_01554_b200/csrc/schemes.h); this handle carries the identity,
// shape, traits and the addition counts of its straight-line programs.
struct Decomposition {
    Builtin which;
    TripleParams params;
    DecompositionTraits traits;
    int adds_alpha, adds_beta, adds_gamma;  // SLP Xor steps per level
    int adds_phi, adds_psi, adds_chi;
};

const Decomposition& builtin(Builtin which);

enum class CostPart { BasisChanges, LinearCombinations };

std::uint64_t predicted_additions(const Decomposition& d, int depth, CostPart part);

}  // namespace bmm
