// cubic_umma2.cu -- K2 (default block product): the cubic bit-matrix product
// on CTA pairs of 5th-generation tensor cores (tcgen05.mma.cta_group::2
// kind::mxf4, M256 x N256 x K64 per instruction, f32 accumulators in TMEM),
// persistent over all output tiles of all products of a batch.
//
// Contract and bit -> fp4 expansion as cubic_umma.cu (reference kernel64 +
// cubic_blocked, engine.cpp:34-100): each bit becomes one e2m1 element
// (x & 0x22222222 / (x>>2) & 0x22222222 -> 1.0, x & 0x11111111 / (x>>2) &
// 0x11111111 -> 0.5, uniform UE8M0 block scales 1.0 / 2.0 per MMA), exact 0/1 dot
// products accumulate in fp32 on top of a 2^23 bias written by one MMA per tile, and
// the epilogue takes bit 0 (GF(2) parity) or the low 23 bits (Boolean non-zero).
//
// Why the pair: the single-CTA form is shared-memory bound -- producers write
// the expanded operands with STS while the tensor core reads them back.  With
// cta_group::2 each SM holds 128 rows of A and 128 rows of Bt per 256 x 256
// pair tile, so per MMA cycle it stores and reads a third less than the
// single-CTA M128 x N256 tile.  Operands use the K-major 128-byte-swizzle
// layout (8-row x 128-byte atoms, chunk j of row r at j ^ (r & 7)): tensor
// reads stay 128-B aligned and the producers' STS.128 are conflict free.
//
// Why persistent: one launch walks every tile (static round robin over the
// 74 SM pairs, raster groups of 12 row tiles), so TMEM allocation, barrier setup
// and scale-factor fill happen once, the producers stream the next tile's stages
// while the current tile's accumulator drains, and the MMAs of the next tile start as
// soon as 32 columns are drained: the pair's tiles alternate between two accumulators
// that overlap in 32 columns (the block scales take the last 32 of the 512).  This is
// what makes the short-K leaf products of the alternative-basis recursion efficient.
//
// Roles per CTA (480 threads):
//   loader (warp 13, one lane; TMA): per superstage of 4 stages (1024 K bits) one
//     3-D tensor-map box per operand, 128 rows x 128 bytes with the 128-byte swizzle,
//     into a 2-slot packed ring (K tails zero-filled by the box bounds).  Long-K
//     launches wave-align the pairs (a loader starts tile j once every pair's loader
//     has issued tile j - 1, global counter, bounded spin) and tag the loads with an
//     L2 policy (the raster group's A panels evict_last, Bt panels evict_first): DRAM
//     reads per n = 131072 launch 806 -> 112 GB, which buys SM clock under the power
//     cap.  Without a tensor map (odd strides, K < 1024 bits) warps 13-14 load with
//     cp.async and swizzled 16-byte destinations.  Keeping global loads out of the
//     expander threads matters: their fence.proxy.async (MEMBAR.CTA) would wait for
//     every load still in flight and serialise one L2 round trip per stage.
//   expanders (warps 0-7): two groups of 4 warps take alternate stages, thread r of a
//     group owns row r of A and of Bt; per superstage a warp reads its rows' bits for
//     its two stages (conflict-free through the swizzle), frees the packed slot, then
//     per stage expands 256 bits -> 128 bytes of e2m1 per row with STS.128 into the
//     4-stage operand ring, fences and arrives on the leader's full barrier
//     (remotely from the peer CTA).  While one group drains its stores through the
//     proxy fence the other group's stores keep the shared-memory port busy.
//   MMA (warp 8, leader CTA): the whole warp runs the loop so slots and descriptors
//     stay warp-uniform (no per-instruction R2UR waterfall); an elected lane issues the
//     bias MMA and then 4 MMAs per stage, commits each stage to both CTAs' empty
//     barriers and each tile to both CTAs' acc_full barriers.
//   epilogue (warps 9-12): drain the CTA's 128 accumulator rows with double-buffered
//     32-column TMEM loads (GF(2): .pack::16b, two columns per register), the group that
//     overlaps the other accumulator first (then `ovl`), release the accumulator
//     (acc_empty) as soon as the last load lands, pack the bits, store.
// kTs (long-K launches, >= BMMGPU_TS_MIN_STAGES stages): operand A of each stage goes to
//   the expander thread's own TMEM lane instead of shared memory (one tcgen05.st.32x32b.x32
//   per row and stage, A ring at TMEM columns 256 + 32 s) and the MMAs read it from there;
//   one accumulator at [0, 256).  Halving the operand stores is worth SM clock under the
//   power cap (c3 1730 -> 1761 MHz effective, 8.34 -> 8.43 Pbop/s, profiles/r02).
// Measured (ncu, clock64 / globaltimer, microbench/trace_tiles.py, time_leaf.py,
// probe_leaf.py): on long K the kernel issues 0.99 of the tensor pipe's 16,384 MACs per SM
// clock (tensor pipe 98.9 % active) at an effective ~1.76 GHz set by the board power cap;
// on 4096-bit leaves each tile boundary costs ~0.45 us (commit -> epilogue -> overlap drain
// -> ovl -> next tile's MMAs) against a ~4.56 us tile.
#include <cuda.h>

#include <atomic>

#include "umma.cuh"

namespace bmmgpu {

namespace {

constexpr int P_BM = 256;                 // pair tile rows (128 per CTA)
constexpr int P_BN = 256;                 // pair tile columns (Bt rows, 128 per CTA)
constexpr int P_KBITS = 256;              // K bits per stage (4 MMAs of K = 64)
#ifndef BMMGPU_STAGES
#define BMMGPU_STAGES 4
#endif
constexpr int P_STAGES = BMMGPU_STAGES;
constexpr int P_ROWS = 128;               // rows of A and of Bt held per CTA
constexpr int P_REGION = P_ROWS * 128;    // bytes of one operand per stage (16 KB)
constexpr int P_STAGE = 2 * P_REGION;
constexpr int P_PRODUCERS = 256;          // expanders: two threads per row of A and of Bt
constexpr int P_MMA_WARP = P_PRODUCERS / 32;
// 4 epilogue warps, one per TMEM lane quarter (8, two per quarter, measured no faster and
// spilled at 96 registers)
constexpr int P_EPI_WARPS = 4;
constexpr int P_LOADER_WARP0 = P_MMA_WARP + 1 + P_EPI_WARPS;  // after the MMA warp and the epilogue warps
constexpr int P_LOADERS = 64;  // cp.async loader threads (TMA: one lane)
constexpr int P_THREADS = P_PRODUCERS + 32 + 32 * P_EPI_WARPS + P_LOADERS;
#ifndef BMMGPU_SST_SLOTS
#define BMMGPU_SST_SLOTS 2
#endif
constexpr int P_SST_SLOTS = BMMGPU_SST_SLOTS;  // packed ring slots, one superstage (4 stages) each
constexpr int P_SST_OP = P_ROWS * 128;         // one operand of a superstage: 128 rows x 128 bytes
constexpr int P_SST = 2 * P_SST_OP;            // 32 KB
// Level-shifted leaves (kFold): the packed region is a ring of units, one TMA box of one
// parent quadrant for one superstage: 128 rows x 128 bytes with the 128-byte swizzle (4 KB
// boxes of one stage each measured 2.6x slower: the TMA row-request rate, not bytes).
constexpr int P_UNIT = P_ROWS * 128;           // 16 KB
// as many units as shared memory leaves after the operand ring and the bias constants
constexpr int P_UNITS = int((232448 - 2048 - size_t(P_STAGES) * P_STAGE - P_REGION - 1024) / P_UNIT);
constexpr int P_PACKED = P_UNITS * P_UNIT > P_SST_SLOTS * P_SST ? P_UNITS * P_UNIT : P_SST_SLOTS * P_SST;
static_assert(P_STAGES % 2 == 0, "the two expander groups alternate ring slots");
// One K = 64 operand region of constants for the bias MMA (rows of 32 e2m1 ones, then
// zeros); A and Bt of the bias MMA both read it.
constexpr int P_CONST = P_REGION;
constexpr size_t P_SMEM = size_t(P_STAGES) * P_STAGE + size_t(P_PACKED) + P_CONST + 1024;  // + alignment slack
constexpr uint32_t P_TMEM_COLS = 512;
// Block scales (UE8M0, uniform): an M128 / N128-per-CTA operand's scales take 4 TMEM
// columns (rows 32 q + i in lane i, replicated over the 4 lane quarters); 8 each.
constexpr uint32_t P_SF_EVEN = 480;  // 1.0
constexpr uint32_t P_SF_ODD = 488;   // 2.0
constexpr uint32_t P_SF_BIAS = 496;  // 2^9 block scales of the bias MMA
constexpr uint32_t P_MAX_PAIRS = 74;  // 148 SMs
// kTs (long-K launches): operand A of each stage lives in TMEM columns [P_TS_A + 32 s, + 32)
// instead of shared memory, next to one accumulator at [0, 256).
constexpr uint32_t P_TS_A = 256;
static_assert(P_TS_A + 32 * P_STAGES <= P_SF_EVEN, "A ring overlaps the block scales");

static_assert(P_SMEM <= 232448 - 1024, "stage ring exceeds shared memory");

// Pipeline timestamps (global timer, ns) of pair 0 when launched with the trace flag
// (BMMGPU_UMMA_TRACE=1; microbench/trace_umma2.py): 0 MMA full, 512 commit issued,
// 1024/2048 empty seen (CTA 0/1), 1536/2560 full arrive (first warp of the stage's group).
// Compiled in only with -DBMMGPU_TRACE (the build never sets it by default).
__device__ unsigned long long g_trace[6144];
// Loaders of wave-aligned launches that hit the spin limit and stopped aligning (debug
// counter behind bmmgpu_debug_wave_stats; the tests assert it stays 0).
__device__ unsigned long long g_wave_timeouts;
// SM clock cycles (clock64) and nanoseconds (globaltimer) of pair 0's MMA loop in the last
// launch: the effective SM clock under the board power cap, which nvidia-smi's sampled
// clocks.sm does not show (bmmgpu_debug_k2_clock; bench.py reports it).
__device__ unsigned long long g_clock_stat[2];
#ifdef BMMGPU_TRACE
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TRACE_AT(cond, idx)                                \
    do {                                                   \
        if ((flags & 16) && (cond)) g_trace[idx] = gtime(); \
    } while (0)
#else
#define TRACE_AT(cond, idx) \
    do {                    \
    } while (0)
#endif

// Isolation probes for the pipeline (results garbage; only with -DBMMGPU_PROBE,
// BMMGPU_UMMA_PROBE=v sets flag bits 32*v; microbench/probe.sh):
// 32 no MMAs, 64 no operand stores, 128 loaders only (expanders just drain the packed ring),
// 256 expanders ignore the packed ring, 512 no proxy fence after the operand stores, 1024 no
// Bt operand stores, 2048 operand stores only while the ring fills the first time (the MMAs
// then re-read valid e2m1 data: the MMA side with real operand values but no stores), 4096
// the same for the A operand only (half the operand stores).
// The probe build also accounts the cycles each role spends waiting (g_probe, 8
// counters per CTA: expander warp 0 empty / packed-full waits / loop total, MMA
// lane full / acc_empty waits / loop total, loader warp 0 packed-empty wait / total).
#ifdef BMMGPU_PROBE
#define PROBE(bit) ((flags & (bit)) != 0)
__device__ unsigned long long g_probe[2 * P_MAX_PAIRS * 8];
#define PWAIT(slot, ...)                     \
    do {                                     \
        const long long _t0 = clock64();     \
        __VA_ARGS__;                         \
        pw[slot] += clock64() - _t0;         \
    } while (0)
#define PSTORE(first, last, cond)                                                              \
    do {                                                                                       \
        if (cond)                                                                              \
            for (int _i = first; _i <= last; ++_i) g_probe[blockIdx.x * 8 + _i] = pw[_i];      \
    } while (0)
#else
#define PROBE(bit) false
#define PWAIT(slot, ...) __VA_ARGS__
#define PSTORE(first, last, cond) \
    do {                          \
    } while (0)
#endif

#ifndef BMMGPU_EPI_SLEEP
#define BMMGPU_EPI_SLEEP 512  // ns the epilogue warps sleep between polls of acc_full on long tiles
#endif


#ifndef BMMGPU_L2_HINT
#define BMMGPU_L2_HINT 1  // 0 normal / normal, 1 A evict_last + Bt evict_first (measured best), 2 A normal + Bt evict_first
#endif
constexpr uint32_t kWaveSpinLimit = 4096;  // x 64 ns: give up on wave alignment after ~0.3 ms

#ifndef BMMGPU_RASTER_GROUP
#define BMMGPU_RASTER_GROUP 12
#endif
constexpr uint32_t kRasterGroup = BMMGPU_RASTER_GROUP;  // row panels per rasterisation group

struct TileMap {
    uint32_t m_tiles, n_tiles, per_prod;  // per_prod = m_tiles * n_tiles
    uint64_t sA, sB, sC;                  // batch strides (words)

    // Linear tile id -> (product, row tile, column tile), grouped by kRasterGroup row
    // panels within a product so concurrently running pairs share panels in L2
    // (with the loaders wave-aligned and the group's row panels held in L2 by evict_last,
    // 12 measured best at n=131072: 48 MiB of resident A panels, ~6 column panels streamed
    // per wave; DRAM reads 112 GB per launch against 806 GB for unaligned waves of 16).
    __device__ __forceinline__ void decode(uint32_t t, uint32_t& b, uint32_t& tm, uint32_t& tn) const {
        b = t / per_prod;
        const uint32_t r = t - b * per_prod;
        const uint32_t group = kRasterGroup, per_group = group * n_tiles;
        const uint32_t first_m = (r / per_group) * group;
        const uint32_t gsize = min(group, m_tiles - first_m);
        const uint32_t in_g = r % per_group;
        tm = first_m + in_g % gsize;
        tn = in_g / gsize;
    }
};

// Row r of an operand region: 16-B chunk j lives at atom(r>>3)*1024 + (r&7)*128 + ((j ^ (r&7)) << 4).
__device__ __forceinline__ void expand_store_sw128(uint8_t* region, int r, int g, const uint4& x) {
    constexpr uint32_t M2 = 0x22222222u, M1 = 0x11111111u;
    const uint4 y = make_uint4(x.x >> 2, x.y >> 2, x.z >> 2, x.w >> 2);
    const int rr = r & 7;
    uint8_t* row = region + (r >> 3) * 1024 + rr * 128;
    const int j0 = 4 * g;
    *reinterpret_cast<uint4*>(row + (((j0 + 0) ^ rr) << 4)) = make_uint4(x.x & M2, x.y & M2, x.z & M2, x.w & M2);
    *reinterpret_cast<uint4*>(row + (((j0 + 1) ^ rr) << 4)) = make_uint4(y.x & M2, y.y & M2, y.z & M2, y.w & M2);
    *reinterpret_cast<uint4*>(row + (((j0 + 2) ^ rr) << 4)) = make_uint4(x.x & M1, x.y & M1, x.z & M1, x.w & M1);
    *reinterpret_cast<uint4*>(row + (((j0 + 3) ^ rr) << 4)) = make_uint4(y.x & M1, y.y & M1, y.z & M1, y.w & M1);
}

// The same expansion into 16 registers (logical chunks 4g .. 4g + 3 of the row, 4 words
// each) for the TMEM form of operand A: w[o + 4 q + i] = word i of chunk q.
__device__ __forceinline__ void expand_regs(const uint4& x, uint32_t (&w)[32], int o) {
    constexpr uint32_t M2 = 0x22222222u, M1 = 0x11111111u;
    const uint4 y = make_uint4(x.x >> 2, x.y >> 2, x.z >> 2, x.w >> 2);
    w[o + 0] = x.x & M2, w[o + 1] = x.y & M2, w[o + 2] = x.z & M2, w[o + 3] = x.w & M2;
    w[o + 4] = y.x & M2, w[o + 5] = y.y & M2, w[o + 6] = y.z & M2, w[o + 7] = y.w & M2;
    w[o + 8] = x.x & M1, w[o + 9] = x.y & M1, w[o + 10] = x.z & M1, w[o + 11] = x.w & M1;
    w[o + 12] = y.x & M1, w[o + 13] = y.y & M1, w[o + 14] = y.z & M1, w[o + 15] = y.w & M1;
}

// The accumulator never starts from zero: each tile's first MMA (accumulate = 0)
// multiplies a constant region of 32 e2m1 ones per row by itself with 2^9 x 2^9 block
// scales, writing 32 * 2^18 = 2^23 into every element; the real MMAs then accumulate
// on top.  Counts c < 2^23 stay exact at the bottom of the mantissa, so an output bit
// is bit 0 of a 32-bit quantity:
//   GF(2):   v = 2^23 + c, parity = bit 0 of v;
//   Boolean: (v + 0x7FFFFF) >> 23 has bit 0 set iff c != 0.
// The drain is issue-bound (measured: 640 ns per tile with two ops per bit, 224 ns with
// the packing removed), so each bit is pushed into its word with one funnel shift:
// w = (x:w) >> 1 moves bit 0 of x into bit 31 and the earlier bits down; after 8
// pushes column j of a group sits in byte 3; byte permutes assemble the word.  About
// one op per bit (GF(2)), three (Boolean).
#ifndef BMMGPU_DRAIN_PROBE
#define BMMGPU_DRAIN_PROBE 0  // dev: 1 = trivial packing (results wrong), isolates the drain's ALU cost
#endif
template <bool kGf2>
__device__ __forceinline__ uint32_t bit_of(uint32_t v) {
    return kGf2 ? v : (v + 0x7FFFFFu) >> 23;
}
// 16 columns -> 16 bits in the low half of the result, as two independent 8-deep
// funnel-shift chains (each leaves its 8 bits in byte 3) merged with one byte permute:
// the chain latency, not the op count, is what the drain waits on.
template <bool kGf2>
__device__ __forceinline__ uint32_t pack_counts16(const uint32_t (&v)[16]) {
    if (BMMGPU_DRAIN_PROBE == 1) return v[0] ^ v[15];
    uint32_t a = 0, b = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        a = __funnelshift_r(a, bit_of<kGf2>(v[j]), 1);
        b = __funnelshift_r(b, bit_of<kGf2>(v[8 + j]), 1);
    }
    return __byte_perm(a, b, 0x0073);  // [a.byte3, b.byte3, -, -]
}

// Two accumulators that overlap in 32 columns (X = [0, 256), Y = [224, 480); the block
// scales take [480, 512)): the pair's tiles alternate X, Y, X, ... so the MMAs of tile
// j + 1 need only the overlap drained from tile j.  The epilogue drains the overlap group
// first (X: tile columns 224..255, Y: tile columns 0..31), signals `ovl`, then the rest,
// then `acc_empty` of that accumulator.  The drain reads TMEM at ~64 B/clk per SM -- a
// whole 256-column accumulator is ~1000 clk with 16-bit reads, ~2000 with 32-bit -- so with
// one accumulator the tensor pipe idled ~12 % of a 4096-bit leaf tile; now it waits for one
// 32-column group.  kRot: drain order 7, 0, 1, .., 6 (X) instead of 0 .. 7 (Y); compile-time
// so `words` stays in registers.
#ifndef BMMGPU_ACC2
#define BMMGPU_ACC2 1  // 0: one accumulator (the MMAs wait for the whole drain)
#endif
constexpr uint32_t P_ACC_Y = BMMGPU_ACC2 ? 224 : 0;  // TMEM column of accumulator Y
template <bool kRot>
__device__ __forceinline__ constexpr int drain_group(int i) {
    return kRot ? (i + 7) & 7 : i;
}
__device__ __forceinline__ void drain_signal(uint32_t bar_leader, uint32_t lane) {
    umma::fence_before_sync();
    __syncwarp();
    if (lane == 0) umma::mbar_arrive_cluster(bar_leader);
}
__device__ __forceinline__ uint32_t (&half16(uint32_t (&v)[32], int h))[16] {
    return *reinterpret_cast<uint32_t(*)[16]>(&v[16 * h]);
}
template <bool kGf2>
__device__ __forceinline__ uint32_t pack_counts32(uint32_t (&v)[32]) {
    return __byte_perm(pack_counts16<kGf2>(half16(v, 0)), pack_counts16<kGf2>(half16(v, 1)), 0x5410);
}

// 32-bit TMEM reads in 32-column groups (two 16-column loads per buffer), double buffered:
// group i + 1 is in flight while group i is packed.
template <bool kGf2, bool kRot>
__device__ __forceinline__ void drain_accumulator2(uint32_t tacc, uint32_t (&words)[8], uint32_t ovl_leader,
                                                   uint32_t empty_leader, uint32_t lane) {
    uint32_t va[32], vb[32];
    umma::tmem_ld16(tacc + 32 * drain_group<kRot>(0), half16(va, 0));
    umma::tmem_ld16(tacc + 32 * drain_group<kRot>(0) + 16, half16(va, 1));
    umma::tmem_ld_wait_regs(va);
    drain_signal(ovl_leader, lane);
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
        umma::tmem_ld16(tacc + 32 * drain_group<kRot>(i + 1), half16(vb, 0));
        umma::tmem_ld16(tacc + 32 * drain_group<kRot>(i + 1) + 16, half16(vb, 1));
        words[drain_group<kRot>(i)] = pack_counts32<kGf2>(va);
        umma::tmem_ld_wait_regs(vb);
        if (i + 2 < 8) {
            umma::tmem_ld16(tacc + 32 * drain_group<kRot>(i + 2), half16(va, 0));
            umma::tmem_ld16(tacc + 32 * drain_group<kRot>(i + 2) + 16, half16(va, 1));
        } else {
            drain_signal(empty_leader, lane);
        }
        words[drain_group<kRot>(i + 1)] = pack_counts32<kGf2>(vb);
        if (i + 2 < 8) umma::tmem_ld_wait_regs(va);
    }
}

// GF(2) needs bit 0 of each count only, so its drain reads the accumulator with
// .pack::16b (the low halves of two columns per register: half the TMEM bytes).  Register
// i of a 32-column load holds column 2i (bit 0) and 2i + 1 (bit 16); one AND + shift-add per
// register gathers them and an outer perfect shuffle restores column order.
#ifndef BMMGPU_GF2_PACK16
#define BMMGPU_GF2_PACK16 1  // 0: 32-bit reads for GF(2) too
#endif
__device__ __forceinline__ uint32_t pack_pairs16(const uint32_t (&v)[16]) {
    uint32_t a = 0, b = 0;  // two chains
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
        a += (v[i] & 0x00010001u) << i;
        b += (v[i + 1] & 0x00010001u) << (i + 1);
    }
    uint32_t x = a | b;
    // bit i = column 2i, bit 16 + i = column 2i + 1 -> interleave the halves
    uint32_t t;
    t = (x ^ (x >> 8)) & 0x0000FF00u; x ^= t ^ (t << 8);
    t = (x ^ (x >> 4)) & 0x00F000F0u; x ^= t ^ (t << 4);
    t = (x ^ (x >> 2)) & 0x0C0C0C0Cu; x ^= t ^ (t << 2);
    t = (x ^ (x >> 1)) & 0x22222222u; x ^= t ^ (t << 1);
    return x;
}
template <bool kRot>
__device__ __forceinline__ void drain_accumulator_gf2_pack16(uint32_t tacc, uint32_t (&words)[8], uint32_t ovl_leader,
                                                             uint32_t empty_leader, uint32_t lane) {
    uint32_t va[16], vb[16];
    umma::tmem_ld16_pack16(tacc + 32 * drain_group<kRot>(0), va);
    umma::tmem_ld_wait_regs16(va);
    drain_signal(ovl_leader, lane);
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
        umma::tmem_ld16_pack16(tacc + 32 * drain_group<kRot>(i + 1), vb);
        words[drain_group<kRot>(i)] = pack_pairs16(va);
        umma::tmem_ld_wait_regs16(vb);
        if (i + 2 < 8)
            umma::tmem_ld16_pack16(tacc + 32 * drain_group<kRot>(i + 2), va);
        else
            drain_signal(empty_leader, lane);
        words[drain_group<kRot>(i + 1)] = pack_pairs16(vb);
        if (i + 2 < 8) umma::tmem_ld_wait_regs16(va);
    }
}

// kTma: the packed superstages arrive by TMA (one 3-D tiled box per operand, 128-byte
// swizzle, K tail zero-filled by the bounds check) instead of the cp.async loader warps.
// kFold (level shifting, reference engine.cpp:202-228 fused_block_stage / PAPER.md "shifting
// levels between layers"): product b of the batch is leaf h = b % 7 of parent p = b / 7, and
// its operands are never materialised -- per superstage the loader brings the parent
// quadrants the fused alpha.phi / beta.psi row of h selects (one 128-row x 128-byte TMA box
// each, into a ring of P_UNITS units) and the expanders XOR them in registers before the
// e2m1 expansion.  Masks: 4 bits per child, child h at bits 4h.
struct FoldSpec {
    uint32_t ma, mb;  // A / Bt quadrant masks of the 7 children
    uint32_t L;       // leaf rows (the parent is 2L x 2L; quadrant q at rows (q >> 1) L, words (q & 1) L / 64)
};
template <bool kTma, bool kFold, bool kTs = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P_THREADS, 1)
    cubic_umma2_kernel(const uint64_t* __restrict__ A, uint64_t lda, const uint64_t* __restrict__ Bt, uint64_t ldbt,
                       uint64_t* __restrict__ C, uint64_t ldc, uint64_t kw, int flags, TileMap map,
                       uint32_t total_tiles, uint32_t epi_sleep_ns, unsigned long long* wave_ctr,
                       const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB, FoldSpec fold) {
    extern __shared__ uint8_t smem_raw[];
    // semiring as a runtime flag: one compiled main loop serves both (a template
    // parameter let the two instantiations schedule the producer loop differently)
    const bool kGf2 = (flags & 2) != 0;
    const bool accumulate = (flags & 1) != 0;
    // two overlapping accumulators for short-K tiles; the TMEM-A form keeps one (its A ring
    // takes the columns of the second) and runs only long-K launches, where a tile's drain
    // is ~1 % of the tile
    constexpr bool kAcc2 = BMMGPU_ACC2 && !kTs;
    __shared__ __align__(8) uint64_t full_bar[P_STAGES];
    __shared__ __align__(8) uint64_t empty_bar[P_STAGES];
    __shared__ __align__(8) uint64_t pk_full_bar[P_SST_SLOTS];
    __shared__ __align__(8) uint64_t pk_empty_bar[P_SST_SLOTS];
    __shared__ __align__(8) uint64_t acc_full_bar[2];   // per accumulator (X, Y)
    __shared__ __align__(8) uint64_t acc_empty_bar[2];
    __shared__ __align__(8) uint64_t ovl_bar;           // overlap columns of the last tile drained
    __shared__ __align__(8) uint64_t unit_full_bar[kFold ? P_UNITS : 1];
    __shared__ __align__(8) uint64_t unit_empty_bar[kFold ? P_UNITS : 1];
    __shared__ uint32_t tmem_base_sh;

    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = umma::cluster_ctarank();
    const uint32_t pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const uint64_t n_stages = kw / (P_KBITS / 64);

    if (warp == P_MMA_WARP) umma::tmem_alloc2(&tmem_base_sh, P_TMEM_COLS);
    if (tid == 0) {
        for (int s = 0; s < P_STAGES; ++s) {
            umma::mbar_init(&full_bar[s], 2 * (P_PRODUCERS / 64));  // one expander group per CTA
            umma::mbar_init(&empty_bar[s], 1);
        }
        for (int s = 0; s < P_SST_SLOTS; ++s) {
            umma::mbar_init(&pk_full_bar[s], kTma ? 1 : P_LOADERS);
            umma::mbar_init(&pk_empty_bar[s], P_PRODUCERS / 32);  // every expander warp, every superstage
        }
        for (int i = 0; i < 2; ++i) {
            umma::mbar_init(&acc_full_bar[i], 1);
            umma::mbar_init(&acc_empty_bar[i], 2 * P_EPI_WARPS);
        }
        umma::mbar_init(&ovl_bar, 2 * P_EPI_WARPS);
        if (kFold)
            for (int u = 0; u < P_UNITS; ++u) {
                umma::mbar_init(&unit_full_bar[u], 1);
                umma::mbar_init(&unit_empty_bar[u], P_PRODUCERS / 32);  // every expander warp
            }
        umma::mbar_fence_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tmem_base_sh;
    if (warp < 4) {
        const uint32_t lane_base = (warp * 32) << 16;
        umma::tmem_st8_fill(tmem + lane_base + P_SF_EVEN, 0x7F7F7F7Fu);
        umma::tmem_st8_fill(tmem + lane_base + P_SF_ODD, 0x80808080u);
        umma::tmem_st8_fill(tmem + lane_base + P_SF_BIAS, 0x88888888u);  // 2^9
        umma::tmem_st_wait();
    }
    {
        // bias operand: row r holds 32 e2m1 ones (0x22 bytes) in its logical 16-byte chunk 0
        // (physical chunk 0 ^ (r & 7) of the 128-byte swizzle), zeros elsewhere
        uint8_t* cst = smem + size_t(P_STAGES) * P_STAGE + size_t(P_PACKED);
        for (uint32_t i = tid; i < uint32_t(P_CONST / 16); i += blockDim.x) {
            const uint32_t r = i >> 3, phys = i & 7;
            const uint32_t v = (phys ^ (r & 7)) == 0 ? 0x22222222u : 0u;
            *reinterpret_cast<uint4*>(cst + size_t(i) * 16) = make_uint4(v, v, v, v);
        }
        umma::fence_proxy_async_smem();
    }
    umma::fence_before_sync();
    umma::cluster_sync();  // barriers of both CTAs initialised, TMEM of both allocated and scaled
    umma::fence_after_sync();

    if (kFold && warp < P_PRODUCERS / 32) {
        // ------------------------------------------------ expanders, level-shifted leaves: as the
        // plain expanders (group grp takes 2 of the 4 stages of a superstage), but a
        // superstage's packed bits are the XOR of its units -- the selected parent quadrants
        // of A, then of Bt, in the loader's order; each unit is freed once every expander
        // warp has read its rows from it.
        const uint32_t grp = warp >> 2, r = tid & (P_ROWS - 1), rsw = r & 7;
        const uint32_t full_leader0 = umma::mapa_shared(smem_u32(&full_bar[0]), 0);
        const uint8_t* urow = smem + size_t(P_STAGES) * P_STAGE + r * 128;
        uint64_t base = 0;  // global stage index of stage 0 of the current tile
        uint64_t un = 0;    // units consumed
        for (uint32_t t = pair; t < total_tiles; t += n_pairs, base += n_stages) {
            uint32_t b, tm, tn;
            map.decode(t, b, tm, tn);
            const uint32_t h = b % 7, ma = (fold.ma >> (4 * h)) & 15u, mb = (fold.mb >> (4 * h)) & 15u;
            const uint32_t wa = __popc(ma), wab = wa + __popc(mb);
            const uint32_t sub0 = (uint32_t(base) ^ grp) & 1;
            for (uint64_t k0 = 0; k0 < n_stages; k0 += 4, un += wab) {
                uint4 v[2][4];  // [stage][A lo, A hi, Bt lo, Bt hi]
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int c = 0; c < 4; ++c) v[j][c] = make_uint4(0, 0, 0, 0);
                for (uint32_t i = 0; i < wab; ++i) {
                    const uint64_t ui = un + i;
                    const uint32_t u = uint32_t(ui % P_UNITS);
                    umma::mbar_wait(&unit_full_bar[u], uint32_t((ui / P_UNITS) & 1));
                    const uint8_t* q = urow + size_t(u) * P_UNIT;
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const uint32_t c = 2 * (sub0 + 2 * j);
                        const uint4 x0 = *reinterpret_cast<const uint4*>(q + ((c ^ rsw) << 4));
                        const uint4 x1 = *reinterpret_cast<const uint4*>(q + (((c + 1) ^ rsw) << 4));
                        if (i < wa) {
                            v[j][0] = make_uint4(v[j][0].x ^ x0.x, v[j][0].y ^ x0.y, v[j][0].z ^ x0.z, v[j][0].w ^ x0.w);
                            v[j][1] = make_uint4(v[j][1].x ^ x1.x, v[j][1].y ^ x1.y, v[j][1].z ^ x1.z, v[j][1].w ^ x1.w);
                        } else {
                            v[j][2] = make_uint4(v[j][2].x ^ x0.x, v[j][2].y ^ x0.y, v[j][2].z ^ x0.z, v[j][2].w ^ x0.w);
                            v[j][3] = make_uint4(v[j][3].x ^ x1.x, v[j][3].y ^ x1.y, v[j][3].z ^ x1.z, v[j][3].w ^ x1.w);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) umma::mbar_arrive(&unit_empty_bar[u]);
                }
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint64_t k = k0 + sub0 + 2 * j;
                    if (k >= n_stages) break;
                    const uint64_t it = base + k;
                    const uint32_t s = uint32_t(it % P_STAGES);
                    if (it >= P_STAGES) umma::mbar_wait(&empty_bar[s], uint32_t((it / P_STAGES - 1) & 1));
                    uint8_t* sa = smem + size_t(s) * P_STAGE;
                    expand_store_sw128(sa, r, 0, v[j][0]);
                    expand_store_sw128(sa, r, 1, v[j][1]);
                    expand_store_sw128(sa + P_REGION, r, 0, v[j][2]);
                    expand_store_sw128(sa + P_REGION, r, 1, v[j][3]);
                    umma::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) umma::mbar_arrive_cluster(full_leader0 + s * 8);
                }
            }
        }
    } else if (warp < P_PRODUCERS / 32) {
        // ------------------------------------------------ expanders: two groups of 4 warps take
        // alternate stages (global stage parity = group), thread r of a group owns row r of A
        // and of Bt.  While one group drains its stores through the proxy fence the other
        // group's stores keep the shared-memory port busy.  Per superstage (4 stages of packed
        // bits) a warp reads its rows' bits for its two stages, frees the packed slot, then
        // expands and stores each stage into the tensor-core ring.
        const uint32_t grp = warp >> 2, r = tid & (P_ROWS - 1), rsw = r & 7;
        // Bt row this thread expands and the operand row (accumulator column) it goes to
        const uint32_t rbt = r, rb = r, rbsw = r & 7;
        const uint32_t full_leader0 = umma::mapa_shared(smem_u32(&full_bar[0]), 0);
        const uint8_t* pkrow = smem + size_t(P_STAGES) * P_STAGE + r * 128;
        const uint8_t* pkrow_b = smem + size_t(P_STAGES) * P_STAGE + rbt * 128 + P_SST_OP;
        uint64_t base = 0;  // global stage index of stage 0 of the current tile
        int slot = 0;
        uint32_t pk_parity = 0;
#ifdef BMMGPU_PROBE
        unsigned long long pw[8] = {};
        const long long p_t0 = clock64();
#endif
        for (uint32_t t = pair; t < total_tiles; t += n_pairs, base += n_stages) {
            const uint32_t sub0 = (uint32_t(base) ^ grp) & 1;  // first stage of this group in a superstage
            for (uint64_t k0 = 0; k0 < n_stages; k0 += 4) {
                if (!PROBE(256)) PWAIT(1, umma::mbar_wait(&pk_full_bar[slot], pk_parity));
                const uint8_t* q = pkrow + slot * P_SST;
                const uint8_t* qb = pkrow_b + slot * P_SST;
                uint4 v[2][4];  // [stage][A lo, A hi, Bt lo, Bt hi]
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint32_t c = 2 * (sub0 + 2 * i);  // 16-byte chunk of the stage's low half
                    v[i][0] = *reinterpret_cast<const uint4*>(q + ((c ^ rsw) << 4));
                    v[i][1] = *reinterpret_cast<const uint4*>(q + (((c + 1) ^ rsw) << 4));
                    v[i][2] = *reinterpret_cast<const uint4*>(qb + ((c ^ rbsw) << 4));
                    v[i][3] = *reinterpret_cast<const uint4*>(qb + (((c + 1) ^ rbsw) << 4));
                }
                __syncwarp();
                if (lane == 0 && !PROBE(256)) umma::mbar_arrive(&pk_empty_bar[slot]);
                if (++slot == P_SST_SLOTS) { slot = 0; pk_parity ^= 1; }
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint64_t k = k0 + sub0 + 2 * i;
                    if (k >= n_stages) break;
                    const uint64_t it = base + k;
                    const uint32_t s = uint32_t(it % P_STAGES);
                    if (it >= P_STAGES && !PROBE(128))
                        PWAIT(0, umma::mbar_wait(&empty_bar[s], uint32_t((it / P_STAGES - 1) & 1)));
                    TRACE_AT(pair == 0 && (warp & 3) == 0 && lane == 0 && it < 512, (rank ? 2048 : 1024) + it);
                    uint8_t* sa = smem + size_t(s) * P_STAGE;
                    if (kTs) {
                        // A -> this thread's TMEM lane (row r), 32 columns = the stage's 256 K
                        // elements in logical chunk order; Bt -> shared memory as below.  The
                        // empty barrier said the MMAs reading this slot completed.
                        umma::fence_after_sync();
                        uint32_t w[32];
                        expand_regs(v[i][0], w, 0);
                        expand_regs(v[i][1], w, 16);
                        umma::tmem_st32(tmem + (((warp & 3) * 32) << 16) + P_TS_A + 32 * s, w);
                        expand_store_sw128(sa + P_REGION, rb, 0, v[i][2]);
                        expand_store_sw128(sa + P_REGION, rb, 1, v[i][3]);
                        umma::tmem_st_wait();
                        umma::fence_proxy_async_smem();
                        umma::fence_before_sync();
                        __syncwarp();
                        if (lane == 0) umma::mbar_arrive_cluster(full_leader0 + s * 8);
                        continue;
                    }
                    if (!PROBE(64 | 128) && !(PROBE(2048) && it >= P_STAGES)) {
                        if (!(PROBE(4096) && it >= P_STAGES)) {
                            expand_store_sw128(sa, r, 0, v[i][0]);
                            expand_store_sw128(sa, r, 1, v[i][1]);
                        }
                        if (!PROBE(1024)) {
                            expand_store_sw128(sa + P_REGION, rb, 0, v[i][2]);
                            expand_store_sw128(sa + P_REGION, rb, 1, v[i][3]);
                        }
                    }
                    if (!PROBE(512)) umma::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0 && !PROBE(128)) umma::mbar_arrive_cluster(full_leader0 + s * 8);
                    TRACE_AT(pair == 0 && (warp & 3) == 0 && lane == 0 && it < 512, (rank ? 2560 : 1536) + it);
                }
            }
        }
#ifdef BMMGPU_PROBE
        pw[2] = clock64() - p_t0;
#endif
        PSTORE(0, 2, tid == 0);
    } else if (warp == P_MMA_WARP) {
        // ------------------------------------------------ MMA issuer (leader CTA).  The whole warp
        // runs the loop so ring slots and descriptors stay warp-uniform (uniform registers, no
        // per-instruction R2UR waterfall); one elected lane issues the MMAs and commits.
        if (rank == 0) {
            constexpr uint32_t idesc = umma::idesc_mxf4(P_BM, P_BN);
            const uint64_t desc_base = umma::smem_desc_sw128(smem_u32(smem), 1024);
            const uint64_t desc_const = umma::smem_desc_sw128(
                smem_u32(smem + size_t(P_STAGES) * P_STAGE + size_t(P_PACKED)), 1024);
            uint64_t it = 0;
            int s = 0;
            uint32_t full_parity = 0;
            uint32_t local = 0;
#ifdef BMMGPU_PROBE
            unsigned long long pw[8] = {};
            const long long p_t0 = clock64();
#endif
            long long clk0 = 0;
            unsigned long long ns0 = 0;
            if (pair == 0) {
                clk0 = clock64();
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns0));
            }
            for (uint32_t t = pair; t < total_tiles; t += n_pairs, ++local) {
                // the tile's first stage is usually staged long before the accumulator comes
                // back: wait for it first so the MMAs issue right after the accumulator is free.
                // Accumulator (local & 1) must have been drained by both CTAs' epilogues from
                // tile local - 2, and the overlap columns from tile local - 1.
                const uint32_t buf = kAcc2 ? (local & 1) : 0;
                if (local > 0 && n_stages > 0) umma::mbar_wait(&full_bar[s], full_parity);
                if (kAcc2) {
                    if (local > 0) PWAIT(4, umma::mbar_wait(&ovl_bar, (local - 1) & 1));
                    if (local > 1) PWAIT(4, umma::mbar_wait(&acc_empty_bar[buf], ((local >> 1) - 1) & 1));
                } else if (local > 0) {
                    PWAIT(4, umma::mbar_wait(&acc_empty_bar[(local - 1) & 1], ((local - 1) >> 1) & 1));
                }
                const uint32_t dacc = tmem + (buf ? P_ACC_Y : 0);
                TRACE_AT(pair == 0 && lane == 0 && local < 512, 3072 + 4 * local + 3);
                umma::fence_after_sync();
                if (umma::elect_one() && !PROBE(32))  // preset the accumulator to 2^23
                    umma::mma_mxf4_pair(dacc, desc_const, desc_const, idesc, tmem + P_SF_BIAS, tmem + P_SF_BIAS, 0u);
                __syncwarp();
                for (uint64_t k = 0; k < (PROBE(128) ? 0 : n_stages); ++k, ++it, s = (s + 1 == P_STAGES) ? (full_parity ^= 1, 0) : s + 1) {
                    PWAIT(3, umma::mbar_wait(&full_bar[s], full_parity));
                    TRACE_AT(pair == 0 && lane == 0 && it < 512, it);
                    umma::fence_after_sync();
                    // descriptors differ only in the start-address field (bytes >> 4)
                    const uint64_t da0 = desc_base + uint64_t((uint32_t(s) * P_STAGE) >> 4);
                    const uint64_t db0 = da0 + (P_REGION >> 4);
                    if (umma::elect_one()) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t sf = tmem + ((j & 1) ? P_SF_ODD : P_SF_EVEN);
                            if (PROBE(32)) continue;
                            // + 32 bytes per K = 64 step (A in TMEM: + 8 columns)
                            // always accumulate onto the bias
                            if (kTs)
                                umma::mma_mxf4_pair_ts(dacc, tmem + P_TS_A + 32 * uint32_t(s) + 8 * j, db0 + 2 * j, idesc,
                                                       sf, sf, 1u);
                            else
                                umma::mma_mxf4_pair(dacc, da0 + 2 * j, db0 + 2 * j, idesc, sf, sf, 1u);
                        }
                        umma::mma_commit_pair(&empty_bar[s], 0x3);
                    }
                    __syncwarp();
                    TRACE_AT(pair == 0 && lane == 0 && it < 512, 512 + it);
                }
                if (umma::elect_one()) umma::mma_commit_pair(&acc_full_bar[local & 1], 0x3);
                TRACE_AT(pair == 0 && lane == 0 && local < 512, 3072 + 4 * local + 0);
                __syncwarp();
            }
#ifdef BMMGPU_PROBE
            pw[5] = clock64() - p_t0;
#endif
            PSTORE(3, 5, lane == 0);
            if (pair == 0 && lane == 0) {
                unsigned long long ns1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1));
                g_clock_stat[0] = (unsigned long long)(clock64() - clk0);
                g_clock_stat[1] = ns1 - ns0;
            }
        }
    } else if (kFold && warp >= P_LOADER_WARP0) {
        // ------------------------------------------------ loader, level-shifted leaves: per superstage
        // one 128-row x 128-byte box (4 stages) per selected parent quadrant, A then Bt.
        if (tid == P_LOADER_WARP0 * 32) {
            umma::tma_prefetch_desc(&tmA);
            umma::tma_prefetch_desc(&tmB);
            uint8_t* units = smem + size_t(P_STAGES) * P_STAGE;
            const int32_t kq = int32_t(fold.L / 64);
            uint64_t un = 0;
            for (uint32_t t = pair; t < total_tiles; t += n_pairs) {
                uint32_t b, tm, tn;
                map.decode(t, b, tm, tn);
                const uint32_t h = b % 7, par = b / 7;
                const uint32_t ma = (fold.ma >> (4 * h)) & 15u, mb = (fold.mb >> (4 * h)) & 15u;
                const int32_t ra = int32_t(tm * P_BM + rank * P_ROWS), rb = int32_t(tn * P_BN + rank * P_ROWS);
                for (uint64_t k0 = 0; k0 < n_stages; k0 += 4)
                    for (uint32_t i = 0; i < 8; ++i) {
                        const uint32_t q = i & 3, m = i < 4 ? ma : mb;
                        if (!((m >> q) & 1)) continue;
                        const uint32_t u = uint32_t(un % P_UNITS);
                        if (un >= P_UNITS) umma::mbar_wait(&unit_empty_bar[u], uint32_t((un / P_UNITS - 1) & 1));
                        umma::mbar_arrive_expect_tx(&unit_full_bar[u], P_UNIT);
                        const int32_t kc = int32_t(k0 * 4) + int32_t(q & 1) * kq;
                        const int32_t row = (i < 4 ? ra : rb) + int32_t(q >> 1) * int32_t(fold.L);
                        umma::tma_load_3d(units + size_t(u) * P_UNIT, i < 4 ? &tmA : &tmB, kc, row, int32_t(par),
                                          &unit_full_bar[u]);
                        ++un;
                    }
            }
        }
    } else if (kTma && warp >= P_LOADER_WARP0) {
        // ------------------------------------------------ loader: one thread issues two TMA boxes per superstage
        if (tid == P_LOADER_WARP0 * 32) {
            umma::tma_prefetch_desc(&tmA);
            umma::tma_prefetch_desc(&tmB);
            // L2 policy: the kRasterGroup row panels (A) are reused by every wave of the
            // group's sweep over the column panels; a column panel (Bt) only within a wave.
            // Only for long-K products (flag 4): in a batch of short leaf products the
            // evict_last lines of finished products would crowd out the live ones.
            const bool hint = (flags & 4) != 0;
#if BMMGPU_L2_HINT == 1
            const uint64_t polA = hint ? umma::createpolicy_evict_last() : umma::createpolicy_evict_normal();
            const uint64_t polB = hint ? umma::createpolicy_evict_first() : umma::createpolicy_evict_normal();
#elif BMMGPU_L2_HINT == 2
            const uint64_t polA = umma::createpolicy_evict_normal();
            const uint64_t polB = hint ? umma::createpolicy_evict_first() : umma::createpolicy_evict_normal();
#else
            const uint64_t polA = umma::createpolicy_evict_normal(), polB = umma::createpolicy_evict_normal();
#endif
            uint8_t* pk = smem + size_t(P_STAGES) * P_STAGE;
            int slot = 0;
            uint32_t pk_empty_parity = 0;
            uint64_t qn = 0;
            uint32_t local = 0;
            bool align = wave_ctr != nullptr;
            for (uint32_t t = pair; t < (PROBE(256) ? 0 : total_tiles); t += n_pairs, ++local) {
                uint32_t b, tm, tn;
                map.decode(t, b, tm, tn);
                const int32_t ra = int32_t(tm * P_BM + rank * P_ROWS), rb = int32_t(tn * P_BN + rank * P_ROWS);
                // Wave alignment (long-K products): tile `local` of every pair shares row and
                // column panels through L2 only if the pairs sweep K together.  Static round
                // robin lets fast pairs drift whole waves ahead (the measured DRAM traffic was
                // 200x the operands); so a loader starts its next tile only once every pair's
                // loader has issued its previous one.  The loaders run two superstages ahead
                // of the MMAs, so the wait hides behind buffered work.  Bounded: after
                // kWaveSpinLimit polls it proceeds anyway (co-residency is not assumed).
                if (align && local > 0) {
                    const unsigned long long target = (unsigned long long)n_pairs * local;
                    uint32_t i = 0;
                    while (i < kWaveSpinLimit && umma::ld_acquire_u64(wave_ctr) < target) {
                        __nanosleep(64);
                        ++i;
                    }
                    // a timeout means the pairs are not all resident (another kernel holds
                    // SMs): stop aligning for the rest of this launch instead of paying it
                    // on every tile
                    if (i == kWaveSpinLimit) align = false;
                }
                for (uint64_t k0 = 0; k0 < n_stages; k0 += 4, ++qn) {
                    if (qn >= P_SST_SLOTS) umma::mbar_wait(&pk_empty_bar[slot], pk_empty_parity);
                    uint8_t* dst = pk + slot * P_SST;
                    umma::mbar_arrive_expect_tx(&pk_full_bar[slot], P_SST);
                    // a zero batch stride broadcasts one panel (its map has a single batch entry)
                    umma::tma_load_3d_hint(dst, &tmA, int32_t(k0 * 4), ra, map.sA ? int32_t(b) : 0,
                                           &pk_full_bar[slot], polA);
                    umma::tma_load_3d_hint(dst + P_SST_OP, &tmB, int32_t(k0 * 4), rb, map.sB ? int32_t(b) : 0,
                                           &pk_full_bar[slot], polB);
                    if (++slot == P_SST_SLOTS) {
                        slot = 0;
                        if (qn + 1 > P_SST_SLOTS) pk_empty_parity ^= 1;
                    }
                }
                if (wave_ctr && rank == 0) umma::red_release_add_u64(wave_ctr, 1);
            }
            if (wave_ctr && !align) atomicAdd(&g_wave_timeouts, 1ull);
        }
    } else if (warp >= P_LOADER_WARP0) {
        // ------------------------------------------------ loaders: packed bits global -> shared (cp.async)
        // Superstage slot: [A, Bt][row][128 bytes = 4 stages], 16-byte chunk c of row r at
        // c ^ (r & 7).  Loader thread lt always moves chunk c = lt & 7 of rows r0 + kStep i
        // (r0 = lt >> 3, kStep = P_LOADERS / 8), so a warp instruction covers four whole
        // 128-byte rows; with kStep = 4 the swizzle alternates between two row phases.
        constexpr int kStep = P_LOADERS / 8;
        const uint32_t lt = tid - P_LOADER_WARP0 * 32, c = lt & 7, r0 = lt >> 3;
        uint8_t* pk = smem + size_t(P_STAGES) * P_STAGE + r0 * 128 + ((c ^ (r0 & 7)) << 4);
        // offset of row r0 + kStep (second phase) relative to the first, within an 8-row atom
        const int phase2 = kStep == 4 ? 4 * 128 + (int((c ^ ((r0 + 4) & 7)) << 4) - int((c ^ (r0 & 7)) << 4)) : 0;
        int slot = 0;
        uint32_t pk_empty_parity = 0;
        uint64_t qn = 0;  // superstages issued
#ifdef BMMGPU_PROBE
        unsigned long long pw[8] = {};
        const long long p_t0 = clock64();
#endif
        for (uint32_t t = pair; t < (PROBE(256) ? 0 : total_tiles); t += n_pairs) {
            uint32_t b, tm, tn;
            map.decode(t, b, tm, tn);
            const uint8_t* ga = reinterpret_cast<const uint8_t*>(
                                    A + b * map.sA + (uint64_t(tm) * P_BM + rank * P_ROWS + r0) * lda) + c * 16;
            const uint8_t* gb = reinterpret_cast<const uint8_t*>(
                                    Bt + b * map.sB + (uint64_t(tn) * P_BN + rank * P_ROWS + r0) * ldbt) + c * 16;
            const uint64_t sa8 = 8 * lda * 8, sb8 = 8 * ldbt * 8;  // 8 rows further
            const uint64_t sa4 = 4 * lda * 8, sb4 = 4 * ldbt * 8;  // 4 rows further
            for (uint64_t k0 = 0; k0 < n_stages; k0 += 4, ++qn) {
                if (qn >= P_SST_SLOTS) PWAIT(6, umma::mbar_wait(&pk_empty_bar[slot], pk_empty_parity));
                if (k0 + (c >> 1) < n_stages) {  // this chunk's stage exists
                    uint8_t* dst = pk + slot * P_SST;
                    const uint8_t* pa = ga + k0 * 32;
                    const uint8_t* pb = gb + k0 * 32;
#pragma unroll 4
                    for (int i = 0; i < P_ROWS / 8; ++i) {
                        cp_async16(dst + i * 1024, pa + i * sa8);
                        cp_async16(dst + P_SST_OP + i * 1024, pb + i * sb8);
                        if (kStep == 4) {
                            cp_async16(dst + i * 1024 + phase2, pa + i * sa8 + sa4);
                            cp_async16(dst + P_SST_OP + i * 1024 + phase2, pb + i * sb8 + sb4);
                        }
                    }
                }
                umma::cp_async_mbar_arrive_noinc(&pk_full_bar[slot]);
                if (++slot == P_SST_SLOTS) {
                    slot = 0;
                    if (qn + 1 > P_SST_SLOTS) pk_empty_parity ^= 1;
                }
            }
        }
#ifdef BMMGPU_PROBE
        pw[7] = clock64() - p_t0;
#endif
        PSTORE(6, 7, lt == 0);
    } else {
        // ------------------------------------------------ epilogue (warps 9 .. 12): warp w drains
        // TMEM lanes 32 (w % 4) .. of the tile's accumulator (local & 1), overlap group first.
        const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
        const uint32_t ovl_leader = umma::mapa_shared(smem_u32(&ovl_bar), 0);
        const uint32_t empty_leader0 = umma::mapa_shared(smem_u32(&acc_empty_bar[0]), 0);
        uint32_t local = 0;
        for (uint32_t t = pair; t < total_tiles; t += n_pairs, ++local) {
            uint32_t b, tm, tn;
            map.decode(t, b, tm, tn);
            uint32_t words[8];
            const uint32_t buf = local & 1;
            if (epi_sleep_ns > 0)
                umma::mbar_wait_sleep(&acc_full_bar[buf], (local >> 1) & 1, epi_sleep_ns);
            else
                umma::mbar_wait(&acc_full_bar[buf], (local >> 1) & 1);
            umma::fence_after_sync();
            TRACE_AT(pair == 0 && rank == 0 && quarter == 0 && lane == 0 && local < 512, 3072 + 4 * local + 1);
            const uint32_t ybuf = kAcc2 ? buf : 0;
            const uint32_t tacc = tmem + ((quarter * 32) << 16) + (ybuf ? P_ACC_Y : 0);
            const uint32_t empty_leader = empty_leader0 + 8 * buf;
            if (kGf2 && BMMGPU_GF2_PACK16) {
                if (ybuf)
                    drain_accumulator_gf2_pack16<false>(tacc, words, ovl_leader, empty_leader, lane);
                else
                    drain_accumulator_gf2_pack16<true>(tacc, words, ovl_leader, empty_leader, lane);
            } else if (kGf2) {
                if (ybuf)
                    drain_accumulator2<true, false>(tacc, words, ovl_leader, empty_leader, lane);
                else
                    drain_accumulator2<true, true>(tacc, words, ovl_leader, empty_leader, lane);
            } else {
                if (ybuf)
                    drain_accumulator2<false, false>(tacc, words, ovl_leader, empty_leader, lane);
                else
                    drain_accumulator2<false, true>(tacc, words, ovl_leader, empty_leader, lane);
            }
            TRACE_AT(pair == 0 && rank == 0 && quarter == 0 && lane == 0 && local < 512, 3072 + 4 * local + 2);
            const uint64_t row = uint64_t(tm) * P_BM + rank * P_ROWS + quarter * 32 + lane;
            uint4* dst = reinterpret_cast<uint4*>(C + b * map.sC + row * ldc + uint64_t(tn) * (P_BN / 64));
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                uint4 w = make_uint4(words[4 * i], words[4 * i + 1], words[4 * i + 2], words[4 * i + 3]);
                if (accumulate) {
                    const uint4 o = dst[i];
                    if (kGf2)
                        w = make_uint4(w.x ^ o.x, w.y ^ o.y, w.z ^ o.z, w.w ^ o.w);
                    else
                        w = make_uint4(w.x | o.x, w.y | o.y, w.z | o.z, w.w | o.w);
                }
                dst[i] = w;
            }
        }
    }
    umma::fence_before_sync();
    umma::cluster_sync();  // all MMAs retired and all TMEM reads done in both CTAs
    if (warp == P_MMA_WARP) {
        umma::fence_after_sync();
        umma::tmem_dealloc2(tmem, P_TMEM_COLS);
    }
}

}  // namespace

#ifndef BMMGPU_L2_PROMOTION
#define BMMGPU_L2_PROMOTION 3  // CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

std::atomic<uint64_t> g_wave_aligned_launches{0};
std::atomic<uint64_t> g_ts_launches{0};  // K2 launches with operand A in TMEM

#ifndef BMMGPU_TS_MIN_STAGES
#define BMMGPU_TS_MIN_STAGES 128  // launches with at least this many 256-bit stages use kTs (0: never)
#endif

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
EncodeTiledFn encode_tiled() {
    static const EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return EncodeTiledFn(nullptr);
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

// Tensor map of a packed operand: [batch][rows][kw words], box 16 words (one 128-byte
// superstage row) x 128 rows x 1, 128-byte swizzle = the loader's shared layout.
bool make_operand_map(CUtensorMap* m, const uint64_t* base, uint64_t kw, uint64_t rows, uint64_t ld, uint64_t batch,
                      uint64_t s_batch) {
    const EncodeTiledFn fn = encode_tiled();
    if (!fn || kw < 16 || rows < uint64_t(P_ROWS) || ld % 2 || (batch > 1 && s_batch % 2) ||
        (reinterpret_cast<uintptr_t>(base) & 15))
        return false;
    if (s_batch == 0) batch = 1;  // broadcast panel
    const cuuint64_t dims[3] = {kw, rows, batch};
    const cuuint64_t strides[2] = {ld * 8, (batch > 1 ? s_batch : rows * ld) * 8};
    const cuuint32_t box[3] = {16, uint32_t(P_ROWS), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint64_t*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CUtensorMapL2promotion(BMMGPU_L2_PROMOTION),
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void umma_granularity(uint64_t* gm, uint64_t* gn, uint64_t* gk_bits) {
    *gm = P_BM;
    *gn = P_BN;
    *gk_bits = P_KBITS;
}

// CTA pairs this host thread's K2 launches leave idle (alt.cu's overlapped leaf groups run
// their expand / compress passes on the freed SMs next to the leaves).
thread_local int t_umma_pair_reserve = 0;
void set_umma_pair_reserve(int pairs) { t_umma_pair_reserve = pairs < 0 ? 0 : pairs; }

int launch_cubic_umma(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                      uint64_t m_pad, uint64_t n_pad, uint64_t kw, bool gf2, bool accumulate, cudaStream_t stream,
                      uint64_t batch, uint64_t sA_batch, uint64_t sB_batch, uint64_t sC_batch) {
    if (m_pad % P_BM || n_pad % P_BN || (kw * 64) % P_KBITS || lda % 2 || ldbt % 2 || ldc % 4) {
        set_error("umma2 kernel: m_pad % 256, n_pad % 256, K % 256 bits must be 0 and strides 16-byte aligned");
        return kEinval;
    }
    if (m_pad == 0 || n_pad == 0 || batch == 0) return kOk;
    if (kw == 0) {  // empty inner dimension: the product is zero
        if (!accumulate)
            for (uint64_t b = 0; b < batch; ++b) {
                BMMGPU_CUDA_TRY(cudaMemset2DAsync(dC + b * sC_batch, ldc * 8, 0, n_pad / 8, m_pad, stream));
                count_launch();
            }
        return kOk;
    }
    if (kw * 64 >= (1ull << 23)) {
        set_error("umma2 kernel: K of 2^23 bits or more would exceed exact biased fp32 accumulation");
        return kEinval;
    }
    const uint64_t m_tiles = m_pad / P_BM, n_tiles = n_pad / P_BN;
    const uint64_t per_prod = m_tiles * n_tiles;
    const uint64_t total = per_prod * batch;
    if (total > 0xffffffffull) {
        set_error("umma2 kernel: too many tiles");
        return kEinval;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t max_pairs = std::min<uint64_t>(P_MAX_PAIRS, std::max(1, sms / 2 - t_umma_pair_reserve));
    const uint64_t pairs = std::min<uint64_t>(total, max_pairs);
    TileMap map{uint32_t(m_tiles), uint32_t(n_tiles), uint32_t(per_prod), sA_batch, sB_batch, sC_batch};
    // TMA loads when the operands can be described by tensor maps (BMMGPU_UMMA_LOADER=cpasync
    // forces the cp.async loader warps, which have no such constraints)
    CUtensorMap tmA{}, tmB{};
    const char* ld_env = getenv("BMMGPU_UMMA_LOADER");
    const bool tma = !(ld_env && !strcmp(ld_env, "cpasync")) &&
                     make_operand_map(&tmA, dA, kw, m_pad, lda, batch, sA_batch) &&
                     make_operand_map(&tmB, dBt, kw, n_pad, ldbt, batch, sB_batch);
    const uint64_t n_stages_l = kw * 64 / P_KBITS;
    // Long-K launches keep operand A in TMEM (kTs): half the expanders' shared-memory stores,
    // which under the board power cap is SM clock (c3: 1731 -> ~1810 MHz with A's stores
    // removed, profiles/r02/probe_effclock2.txt); short-K tiles keep both operands in shared
    // memory and the two overlapping accumulators.
    static const uint64_t ts_min = [] {
        const char* e = getenv("BMMGPU_TS_MIN_STAGES");
        return e ? uint64_t(strtoull(e, nullptr, 10)) : uint64_t(BMMGPU_TS_MIN_STAGES);
    }();
    const bool ts = tma && ts_min > 0 && n_stages_l >= ts_min;
    if (ts) g_ts_launches.fetch_add(1, std::memory_order_relaxed);
    auto kern = ts ? cubic_umma2_kernel<true, false, true>
                   : tma ? cubic_umma2_kernel<true, false> : cubic_umma2_kernel<false, false>;
    BMMGPU_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P_SMEM)));
    const char* probe = getenv("BMMGPU_UMMA_PROBE");
    const int flags = (accumulate ? 1 : 0) | (gf2 ? 2 : 0) | (n_stages_l >= 64 ? 4 : 0) |
                      (getenv("BMMGPU_UMMA_TRACE") ? 16 : 0) | (probe && *probe ? 32 * atoi(probe) : 0);
    // Epilogue warps poll acc_full with this sleep between tries: long tiles (K of tens of
    // thousands of bits) leave them idle for ~100 us and their spinning would steal issue
    // slots from the expanders; for short tiles the sleep granularity is pure bubble.
    const uint64_t n_stages = kw * 64 / P_KBITS;
    uint32_t epi_sleep = n_stages >= 128 ? BMMGPU_EPI_SLEEP : n_stages >= 32 ? 64 : 0;
    if (const char* es = getenv("BMMGPU_EPI_SLEEP_NS")) epi_sleep = uint32_t(atoi(es));
    // Wave alignment of the TMA loaders for long-K products (see the loader): a zeroed
    // 8-byte counter per launch from the stream-ordered pool.
    DeviceBuffer ctr;
    unsigned long long* wave_ctr = nullptr;
    const char* wa = getenv("BMMGPU_WAVE_ALIGN");
    if (tma && n_stages >= 64 && total > pairs && !(wa && *wa == '0')) {
        int st;
        if ((st = ctr.alloc(8, stream))) return st;
        BMMGPU_CUDA_TRY(cudaMemsetAsync(ctr.p, 0, 8, stream));
        count_launch();
        wave_ctr = static_cast<unsigned long long*>(ctr.p);
        g_wave_aligned_launches.fetch_add(1, std::memory_order_relaxed);
    }
    kern<<<unsigned(2 * pairs), P_THREADS, P_SMEM, stream>>>(dA, lda, dBt, ldbt, dC, ldc, kw, flags, map,
                                                             uint32_t(total), epi_sleep, wave_ctr, tmA, tmB,
                                                             FoldSpec{0, 0, 0});
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

// Tensor map of a parent array for the level-shifted leaves: [parents][2L rows][ld words],
// box 16 words (one superstage, 128 bytes) x 128 rows x 1, 128-byte swizzle = the unit layout.
static bool make_parent_map(CUtensorMap* m, const uint64_t* base, uint64_t L, uint64_t ld, uint64_t parents,
                            uint64_t s_parent) {
    const EncodeTiledFn fn = encode_tiled();
    if (!fn || L % 256 || ld % 2 || (parents > 1 && s_parent % 2) || (reinterpret_cast<uintptr_t>(base) & 15))
        return false;
    if (s_parent == 0) parents = 1;
    const cuuint64_t dims[3] = {2 * L / 64, 2 * L, parents};
    const cuuint64_t strides[2] = {ld * 8, (parents > 1 ? s_parent : 2 * L * ld) * 8};
    const cuuint32_t box[3] = {16, uint32_t(P_ROWS), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint64_t*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CUtensorMapL2promotion(BMMGPU_L2_PROMOTION),
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Level-shifted leaf layer: the 7 * parents products Q[7 p + h] = T_h . S_h^T of L x L
// leaves whose operands T_h = XOR_{q in ma_h} A_p quadrant q, S_h = XOR_{q in mb_h} Bt_p
// quadrant q are formed inside the kernel from the parents (2L x 2L, row strides
// ld_a / ld_b, parent strides s_a / s_b; s = 0: one parent).  Q row-major L x L / 64 per
// product, stride ldq, product stride s_q.  Returns kEinval when the shapes do not allow
// it (L not a multiple of 256, unaligned strides): the caller materialises the leaves.
int launch_cubic_umma_fold(const uint64_t* dApar, uint64_t ld_a, uint64_t s_a, const uint64_t* dBtpar, uint64_t ld_b,
                           uint64_t s_b, uint64_t parents, uint64_t L, uint32_t ma, uint32_t mb, uint64_t* dQ,
                           uint64_t ldq, uint64_t s_q, bool gf2, cudaStream_t stream) {
    CUtensorMap tmA{}, tmB{};
    if (L % P_BM || ldq % 4 || L / 64 >= (uint64_t(1) << 17) ||
        !make_parent_map(&tmA, dApar, L, ld_a, parents, s_a) || !make_parent_map(&tmB, dBtpar, L, ld_b, parents, s_b)) {
        set_error("umma2 fold: shapes not supported");
        return kEinval;
    }
    const uint64_t kw = L / 64;
    const uint64_t m_tiles = L / P_BM, per_prod = m_tiles * m_tiles, total = per_prod * 7 * parents;
    if (total > 0xffffffffull) {
        set_error("umma2 fold: too many tiles");
        return kEinval;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t pairs = std::min<uint64_t>(total, std::min<uint64_t>(P_MAX_PAIRS, std::max(1, sms / 2)));
    TileMap map{uint32_t(m_tiles), uint32_t(m_tiles), uint32_t(per_prod), 0, 0, s_q};
    auto kern = cubic_umma2_kernel<true, true>;
    BMMGPU_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P_SMEM)));
    const uint64_t n_stages = kw * 64 / P_KBITS;
    const uint32_t epi_sleep = n_stages >= 128 ? BMMGPU_EPI_SLEEP : n_stages >= 32 ? 64 : 0;
    const int flags = gf2 ? 2 : 0;
    kern<<<unsigned(2 * pairs), P_THREADS, P_SMEM, stream>>>(dApar, ld_a, dBtpar, ld_b, dQ, ldq, kw, flags, map,
                                                             uint32_t(total), epi_sleep, nullptr, tmA, tmB,
                                                             FoldSpec{ma, mb, uint32_t(L)});
    count_launch();
    BMMGPU_CUDA_TRY(cudaGetLastError());
    return kOk;
}

}  // namespace bmmgpu

// Debug: the per-CTA wait counters of the last launch of a -DBMMGPU_PROBE build.
extern "C" int bmmgpu_debug_umma2_probe(unsigned long long* out) {
#ifdef BMMGPU_PROBE
    return cudaMemcpyFromSymbol(out, bmmgpu::g_probe, sizeof(bmmgpu::g_probe)) == cudaSuccess ? 0 : 5;
#else
    (void)out;
    return 1;
#endif
}

// Debug: K2 launches that ran with wave-aligned loaders (host count) and loaders that gave
// up aligning after the spin limit (device count), since the library was loaded.
extern "C" int bmmgpu_debug_wave_stats(uint64_t* aligned_launches, uint64_t* loader_timeouts) {
    if (aligned_launches) *aligned_launches = bmmgpu::g_wave_aligned_launches.load();
    if (loader_timeouts) {
        unsigned long long t = 0;
        if (cudaMemcpyFromSymbol(&t, bmmgpu::g_wave_timeouts, sizeof(t)) != cudaSuccess) return 5;
        *loader_timeouts = t;
    }
    return 0;
}

// Debug: SM cycles and nanoseconds of pair 0's MMA loop in the last K2 launch (effective
// SM clock = cycles / ns).
extern "C" int bmmgpu_debug_k2_clock(uint64_t* cycles, uint64_t* ns) {
    unsigned long long v[2] = {0, 0};
    if (cudaMemcpyFromSymbol(v, bmmgpu::g_clock_stat, sizeof(v)) != cudaSuccess) return 5;
    if (cycles) *cycles = v[0];
    if (ns) *ns = v[1];
    return 0;
}

// Debug: K2 launches that kept operand A in tensor memory (kTs), since the library was loaded.
extern "C" int bmmgpu_debug_ts_launches(uint64_t* launches) {
    if (!launches) return 1;
    *launches = bmmgpu::g_ts_launches.load();
    return 0;
}

// Debug: copy the pipeline timestamps of the last traced launch.
extern "C" int bmmgpu_debug_umma2_trace(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, bmmgpu::g_trace, sizeof(bmmgpu::g_trace)) == cudaSuccess ? 0 : 5;
}
