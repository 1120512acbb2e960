// schemes.h -- the <2,2,2;7> bilinear schemes of the reference, as constants
// the GPU passes bake into their coefficient masks.
//
// Matrices are copied as the reference writes them (one '0'/'1' string per
// row, leftmost character = column 0, quadrant order 00,01,10,11) from
// reference src/decomposition.cpp; in-place basis-change programs are the
// reference's SLP step lists (target ^= source, applied in order).
#pragma once
#include <cstdint>

namespace bmmgpu {

struct InPlaceStep {
    uint8_t target, source;
};

struct Scheme {
    const char* alpha[7];  // 7 x 4
    const char* beta[7];   // 7 x 4
    const char* gamma[4];  // 4 x 7
    InPlaceStep phi[2];
    int n_phi;
    InPlaceStep psi[2];
    int n_psi;
    InPlaceStep chi[2];
    int n_chi;
};

// Strassen-Winograd, standard basis (decomposition.cpp:57-102): no basis change.
constexpr Scheme kStrassenWinograd = {
    {"0011", "0100", "0101", "0111", "1111", "0010", "1000"},
    {"0011", "0010", "0101", "0111", "0100", "1111", "1000"},
    {"0100001", "1101100", "0111010", "1111000"},
    {},
    0,
    {},
    0,
    {},
    0,
};

// Alternative basis, self-inverse (decomposition.cpp:104-142).
// phi = psi: x11 ^= x01, x11 ^= x10 (136-137); chi: x01 ^= x11, x10 ^= x11 (139).
constexpr Scheme kAltSelfInverse = {
    {"1000", "0100", "0010", "0001", "1001", "0101", "0011"},
    {"1000", "0010", "1001", "0001", "0100", "0101", "0011"},
    {"1100000", "0000101", "0010010", "0101011"},
    {{3, 1}, {3, 2}},
    2,
    {{3, 1}, {3, 2}},
    2,
    {{1, 3}, {2, 3}},
    2,
};

// Alternative basis, chaining (decomposition.cpp:144-183).
// phi = psi: x11 ^= x01 then x10 ^= x11 (177-178); chi: x10 ^= x11 then x11 ^= x01 (180).
constexpr Scheme kAltChaining = {
    {"1000", "0100", "0010", "0001", "1010", "0110", "0011"},
    {"1000", "0011", "0010", "0001", "0100", "0110", "1010"},
    {"1100000", "0110110", "0110101", "0001100"},
    {{3, 1}, {2, 3}},
    2,
    {{3, 1}, {2, 3}},
    2,
    {{2, 3}, {3, 1}},
    2,
};

// algo ids follow bmm::Algo (reference engine.hpp:16): 1 sw, 2 alt-si, 3 alt-chain
inline const Scheme* scheme_for(int algo) {
    switch (algo) {
        case 1: return &kStrassenWinograd;
        case 2: return &kAltSelfInverse;
        case 3: return &kAltChaining;
        default: return nullptr;
    }
}

inline uint32_t row_mask(const char* row) {
    uint32_t m = 0;
    for (int c = 0; row[c]; ++c)
        if (row[c] == '1') m |= 1u << c;
    return m;
}

}  // namespace bmmgpu
