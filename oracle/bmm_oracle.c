/*
 * bmm_oracle.c -- CPU restatement of the reference bit-matrix product path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path in paper_1909_01554_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product never links or calls it; the CUDA path fails loudly when its
 * extension is missing instead of falling back here.
 *
 * Parity pinning: every function is cross-checked in tests/ against the
 * reference itself (oracle/_ref, built from /root/reference/proj/src by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/
 * that tests/golden/make_golden.py generated from oracle/_ref.
 *
 * All citations are /root/reference/proj/<file>:<line>.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ mt19937_64
 * BitMatrix::random draws one std::mt19937_64 word per packed word, row-major,
 * and masks the tail of each row (src/bitmatrix.cpp:64-77).  std::mt19937_64 is
 * fully specified by [rand.predef]; this is the standard algorithm. */
typedef struct { uint64_t mt[312]; int idx; } mt64_t;

EXPORT void bmmo_mt64_seed(mt64_t* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

EXPORT uint64_t bmmo_mt64_next(mt64_t* s) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    static const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= MATRIX_A;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

EXPORT uint64_t bmmo_mt64_state_size(void) { return sizeof(mt64_t); }

/* BitMatrix::random(rows, cols, seed) into caller storage of rows*wpr words
 * (src/bitmatrix.cpp:64-77). */
EXPORT void bmmo_random(uint64_t rows, uint64_t cols, uint64_t seed, uint64_t* words) {
    mt64_t s;
    bmmo_mt64_seed(&s, seed);
    const uint64_t wpr = (cols + 63) / 64;
    const unsigned tail = (unsigned)(cols % 64);
    const uint64_t tail_mask = tail ? ((1ULL << tail) - 1) : ~0ULL;
    for (uint64_t i = 0; i < rows; ++i) {
        uint64_t* r = words + i * wpr;
        for (uint64_t w = 0; w < wpr; ++w) r[w] = bmmo_mt64_next(&s);
        r[wpr - 1] &= tail_mask;
    }
}

/* ------------------------------------------------------------------ layout */

/* In-place 64x64 bit transpose, recursive block swap with six mask stages
 * (src/bitmatrix.cpp:16-31). */
EXPORT void bmmo_transpose64(uint64_t* x) {
    static const uint64_t masks[6] = {
        0x00000000FFFFFFFFULL, 0x0000FFFF0000FFFFULL, 0x00FF00FF00FF00FFULL,
        0x0F0F0F0F0F0F0F0FULL, 0x3333333333333333ULL, 0x5555555555555555ULL,
    };
    unsigned w = 32;
    for (int s = 0; s < 6; ++s) {
        const uint64_t m = masks[s];
        for (unsigned k = 0; k < 64; ++k) {
            if (k & w) continue;
            uint64_t t = ((x[k] >> w) ^ x[k | w]) & m;
            x[k] ^= t << w;
            x[k | w] ^= t;
        }
        w >>= 1;
    }
}

/* transpose_blocks64: every aligned 64x64 block transposed in place
 * (src/bitmatrix.cpp:97-110).  Returns 3 (shape) when dims are not /64. */
EXPORT int bmmo_transpose_blocks64(uint64_t rows, uint64_t cols, uint64_t* words) {
    if (rows % 64 || cols % 64) return 3;
    const uint64_t wpr = cols / 64;
    uint64_t blk[64];
    for (uint64_t bi = 0; bi < rows / 64; ++bi)
        for (uint64_t bj = 0; bj < wpr; ++bj) {
            uint64_t* base = words + bi * 64 * wpr + bj;
            for (unsigned r = 0; r < 64; ++r) blk[r] = base[r * wpr];
            bmmo_transpose64(blk);
            for (unsigned r = 0; r < 64; ++r) base[r * wpr] = blk[r];
        }
    return 0;
}

/* Row digit of level l to bit 2l+1, column digit to bit 2l
 * (src/bitmatrix.cpp:35-42). */
EXPORT uint64_t bmmo_morton2(uint64_t row_blk, uint64_t col_blk, int levels) {
    uint64_t out = 0;
    for (int l = 0; l < levels; ++l) {
        out |= ((row_blk >> l) & 1ULL) << (2 * l + 1);
        out |= ((col_blk >> l) & 1ULL) << (2 * l);
    }
    return out;
}

/* Operand: 0 Left, 1 Right, 2 Result (include/bmm/bitmatrix.hpp:25). */
EXPORT uint64_t bmmo_interleaved_bit_index(int depth, int which, uint64_t i, uint64_t j) {
    const uint64_t block = bmmo_morton2(i / 64, j / 64, depth);
    const uint64_t r = i % 64, c = j % 64;
    const uint64_t inner = which == 1 ? c * 64 + r : r * 64 + c;
    return block * 4096 + inner; /* src/bitmatrix.cpp:112-122 */
}

/* to_interleaved (src/bitmatrix.cpp:124-146): n = 64 << depth. */
EXPORT void bmmo_to_interleaved(int depth, int which, const uint64_t* m, uint64_t* t) {
    const uint64_t n = 64ULL << depth, wpr = n / 64;
    uint64_t blk[64];
    for (uint64_t bi = 0; bi < n / 64; ++bi)
        for (uint64_t bj = 0; bj < n / 64; ++bj) {
            const uint64_t* src = m + bi * 64 * wpr + bj;
            for (unsigned r = 0; r < 64; ++r) blk[r] = src[r * wpr];
            if (which == 1) bmmo_transpose64(blk);
            memcpy(t + bmmo_morton2(bi, bj, depth) * 64, blk, sizeof(blk));
        }
}

/* from_interleaved (src/bitmatrix.cpp:148-173). */
EXPORT void bmmo_from_interleaved(int depth, int which, const uint64_t* t, uint64_t* m) {
    const uint64_t n = 64ULL << depth, wpr = n / 64;
    uint64_t blk[64];
    for (uint64_t bi = 0; bi < n / 64; ++bi)
        for (uint64_t bj = 0; bj < n / 64; ++bj) {
            memcpy(blk, t + bmmo_morton2(bi, bj, depth) * 64, sizeof(blk));
            if (which == 1) bmmo_transpose64(blk);
            uint64_t* dst = m + bi * 64 * wpr + bj;
            for (unsigned r = 0; r < 64; ++r) dst[r * wpr] = blk[r];
        }
}

/* ------------------------------------------------------------------ cubic */

/* Semiring: 0 BooleanOrAnd, 1 Gf2XorAnd (include/bmm/engine.hpp:14). */
/* kernel64: bit k of out[i] = parity(popcount(a[i] & bt[k])) over GF(2), or
 * (a[i] & bt[k]) != 0 over the Boolean semiring (src/engine.cpp:34-56). */
EXPORT void bmmo_kernel64(const uint64_t* a, const uint64_t* bt, uint64_t* out, int ring) {
    for (unsigned i = 0; i < 64; ++i) {
        const uint64_t row = a[i];
        uint64_t bits = 0;
        for (unsigned k = 0; k < 64; ++k) {
            const uint64_t v = row & bt[k];
            const uint64_t bit = ring == 1 ? (uint64_t)(__builtin_popcountll(v) & 1) : (uint64_t)(v != 0);
            bits |= bit << k;
        }
        out[i] = bits;
    }
}

/* multiply_cubic (src/engine.cpp:132-144): blocked path when all dims are
 * multiples of 64 (cubic_blocked, 60-100: B copied and block-transposed, each
 * output block folds kernel64 over bj with XOR/OR), else the row-combination
 * fallback (cubic_rowwise, 102-128).  c must hold m * ceil(n/64) words and
 * is fully overwritten.  Returns 3 on a.cols != b.rows. */
EXPORT int bmmo_multiply_cubic(const uint64_t* a, const uint64_t* b, uint64_t* c,
                               uint64_t m, uint64_t k, uint64_t n, int ring) {
    const uint64_t a_wpr = (k + 63) / 64, b_wpr = (n + 63) / 64, c_wpr = b_wpr;
    memset(c, 0, m * c_wpr * sizeof(uint64_t));
    if (m % 64 == 0 && k % 64 == 0 && n % 64 == 0) {
        uint64_t* bt = (uint64_t*)malloc(k * b_wpr * sizeof(uint64_t) + 8);
        memcpy(bt, b, k * b_wpr * sizeof(uint64_t));
        bmmo_transpose_blocks64(k, n, bt);
        const uint64_t bi_n = m / 64, bj_n = k / 64, bk_n = n / 64;
        uint64_t a_blk[64], bt_blk[64], acc[64], q[64];
        for (uint64_t bi = 0; bi < bi_n; ++bi)
            for (uint64_t bk = 0; bk < bk_n; ++bk) {
                for (uint64_t bj = 0; bj < bj_n; ++bj) {
                    for (unsigned u = 0; u < 64; ++u) {
                        a_blk[u] = a[(bi * 64 + u) * a_wpr + bj];
                        bt_blk[u] = bt[(bj * 64 + u) * b_wpr + bk];
                    }
                    bmmo_kernel64(a_blk, bt_blk, bj == 0 ? acc : q, ring);
                    if (bj == 0) continue;
                    for (unsigned u = 0; u < 64; ++u) acc[u] = ring == 1 ? (acc[u] ^ q[u]) : (acc[u] | q[u]);
                }
                for (unsigned u = 0; u < 64; ++u) c[(bi * 64 + u) * c_wpr + bk] = acc[u];
            }
        free(bt);
    } else {
        for (uint64_t i = 0; i < m; ++i) {
            const uint64_t* arow = a + i * a_wpr;
            uint64_t* crow = c + i * c_wpr;
            for (uint64_t j = 0; j < k; ++j) {
                if (!((arow[j >> 6] >> (j & 63)) & 1)) continue;
                const uint64_t* brow = b + j * b_wpr;
                for (uint64_t w = 0; w < c_wpr; ++w) crow[w] = ring == 1 ? (crow[w] ^ brow[w]) : (crow[w] | brow[w]);
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ alt-basis
 * Alternative-basis self-inverse scheme constants (src/decomposition.cpp:104-142):
 *   alpha rows 1000,0100,0010,0001,1001,0101,0011 (quadrant order 00,01,10,11)
 *   beta       1000,0010,1001,0001,0100,0101,0011
 *   gamma      1100000,0000101,0010010,0101011
 *   phi = psi  x11 ^= x01 ^ x10            chi  x01 ^= x11, x10 ^= x11
 * Restated as the direct matrix application (same results as the SLPs, which
 * tests/test_oracle.py checks against the reference). */
static const uint8_t ALPHA[7][4] = {{1,0,0,0},{0,1,0,0},{0,0,1,0},{0,0,0,1},{1,0,0,1},{0,1,0,1},{0,0,1,1}};
static const uint8_t BETA[7][4]  = {{1,0,0,0},{0,0,1,0},{1,0,0,1},{0,0,0,1},{0,1,0,0},{0,1,0,1},{0,0,1,1}};
static const uint8_t GAMMA[4][7] = {{1,1,0,0,0,0,0},{0,0,0,0,1,0,1},{0,0,1,0,0,1,0},{0,1,0,1,0,1,1}};

/* mode_step (src/yates.cpp:112-141): out[o][h][t] = XOR_q M[h][q] in[o][q][t].
 * rows x cols coefficient matrix given row-major as bytes. */
static void mode_apply(const uint8_t* M, int rows, int cols, const uint64_t* in, uint64_t* out,
                       uint64_t outer, uint64_t inner) {
    for (uint64_t o = 0; o < outer; ++o)
        for (int h = 0; h < rows; ++h) {
            uint64_t* dst = out + (o * rows + h) * inner;
            memset(dst, 0, inner * sizeof(uint64_t));
            for (int q = 0; q < cols; ++q) {
                if (!M[h * cols + q]) continue;
                const uint64_t* src = in + (o * cols + q) * inner;
                for (uint64_t t = 0; t < inner; ++t) dst[t] ^= src[t];
            }
        }
}

/* basis_change (src/engine.cpp:146-172 -> yates.cpp:143-172): for the outer
 * `levels` modes, outermost first, the in-place 4-arity SLP.
 * which: 0 Phi, 1 Psi (both x11 ^= x01 ^ x10), 2 Chi (x01 ^= x11, x10 ^= x11). */
EXPORT void bmmo_basis_change(uint64_t* v, uint64_t total_words, int levels, int which) {
    uint64_t outer = 1;
    for (int l = 0; l < levels; ++l) {
        const uint64_t inner = total_words / (outer * 4);
        for (uint64_t o = 0; o < outer; ++o) {
            uint64_t* g = v + o * 4 * inner;
            for (uint64_t t = 0; t < inner; ++t) {
                if (which == 2) {
                    g[1 * inner + t] ^= g[3 * inner + t];
                    g[2 * inner + t] ^= g[3 * inner + t];
                } else {
                    g[3 * inner + t] ^= g[1 * inner + t];
                    g[3 * inner + t] ^= g[2 * inner + t];
                }
            }
        }
        outer *= 4;
    }
}

/* Depth-first alt-basis recursion: alpha/beta expand 4 -> 7, seven child
 * products, gamma compress 7 -> 4; kernel64 over GF(2) at the leaf block
 * (src/engine.cpp:274-289 with parallel_leaf 232-272; the parallel layers
 * compute the same linear map breadth-first, so one recursion restates all
 * d_serial / d_parallel splits). */
static void alt_rec(const uint64_t* a, const uint64_t* b, uint64_t* c, uint64_t words) {
    if (words == 64) {
        bmmo_kernel64(a, b, c, 1);
        return;
    }
    const uint64_t sub = words / 4;
    uint64_t* t = (uint64_t*)malloc(7 * sub * sizeof(uint64_t));
    uint64_t* s = (uint64_t*)malloc(7 * sub * sizeof(uint64_t));
    uint64_t* q = (uint64_t*)malloc(7 * sub * sizeof(uint64_t));
    mode_apply(&ALPHA[0][0], 7, 4, a, t, 1, sub);
    mode_apply(&BETA[0][0], 7, 4, b, s, 1, sub);
    for (int h = 0; h < 7; ++h) alt_rec(t + h * sub, s + h * sub, q + h * sub, sub);
    mode_apply(&GAMMA[0][0], 4, 7, q, c, 1, sub);
    free(t); free(s); free(q);
}

/* multiply_alt (src/engine.cpp:293-349) on interleaved, basis-changed operands. */
EXPORT void bmmo_multiply_alt(const uint64_t* a_hat, const uint64_t* b_hat, uint64_t* c_hat, int depth) {
    const uint64_t words = (64ULL << depth) * (64ULL << depth) / 64;
    alt_rec(a_hat, b_hat, c_hat, words);
}

/* multiply(a, b, AltSelfInverse, plan, Gf2XorAnd) (src/engine.cpp:351-382):
 * interleave, phi/psi, multiply_alt, chi, de-interleave.  n = 64 << depth. */
EXPORT void bmmo_multiply_alt_si(const uint64_t* a, const uint64_t* b, uint64_t* c, int depth) {
    const uint64_t n = 64ULL << depth, words = n * n / 64;
    uint64_t* ah = (uint64_t*)malloc(words * 8);
    uint64_t* bh = (uint64_t*)malloc(words * 8);
    uint64_t* ch = (uint64_t*)malloc(words * 8);
    bmmo_to_interleaved(depth, 0, a, ah);
    bmmo_to_interleaved(depth, 1, b, bh);
    bmmo_basis_change(ah, words, depth, 0);
    bmmo_basis_change(bh, words, depth, 1);
    bmmo_multiply_alt(ah, bh, ch, depth);
    bmmo_basis_change(ch, words, depth, 2);
    bmmo_from_interleaved(depth, 2, ch, c);
    free(ah); free(bh); free(ch);
}

/* ------------------------------------------------------------------ digests */

/* FNV-1a 64 over the little-endian bytes of the word array (the digest the
 * golden vectors in SURVEY.md section 8c and tests/golden use). */
EXPORT uint64_t bmmo_fnv1a64(const uint64_t* w, uint64_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t i = 0; i < n; ++i)
        for (int b = 0; b < 8; ++b) {
            h ^= (w[i] >> (8 * b)) & 0xFF;
            h *= 0x100000001b3ULL;
        }
    return h;
}

EXPORT uint64_t bmmo_popcount(const uint64_t* w, uint64_t n) {
    uint64_t c = 0;
    for (uint64_t i = 0; i < n; ++i) c += (uint64_t)__builtin_popcountll(w[i]);
    return c;
}
