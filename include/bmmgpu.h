/*
 * bmmgpu.h -- C ABI of the B200-native Boolean / GF(2) bit-matrix product.
 *
 * Plain pointers and sizes only.  Every entry point returns a status code;
 * bmmgpu_last_error() gives the message of the last failure on the calling
 * thread.  The C++ drop-in (include/bmm/ headers, libbmm_b200.so) turns the codes
 * back into the reference's exception types:
 *     BMMGPU_EINVAL -> std::invalid_argument   (reference engine.cpp:355-365)
 *     BMMGPU_ESHAPE -> bmm::ShapeError         (reference engine.cpp:134, 359-362)
 *     BMMGPU_ECUDA / BMMGPU_ENODEV -> std::runtime_error (no CPU fallback)
 *
 * Bit layout everywhere is the reference BitMatrix layout
 * (reference include/bmm/bitmatrix.hpp:27-52): row-major, words_per_row =
 * ceil(cols/64) little-endian uint64 words, bit j of row i at bit j%64 of word
 * j/64, pad bits zero.
 */
#ifndef BMMGPU_H
#define BMMGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define BMMGPU_OK 0
#define BMMGPU_EINVAL 1
#define BMMGPU_ESHAPE 3
#define BMMGPU_EFORMAT 4 /* malformed BMM1 file -> bmm::FormatError */
#define BMMGPU_ECUDA 5
#define BMMGPU_ENODEV 6

/* bmm::Semiring order (reference include/bmm/engine.hpp:14) */
#define BMMGPU_BOOLEAN_OR_AND 0
#define BMMGPU_GF2_XOR_AND 1

/* bmm::Algo order (reference include/bmm/engine.hpp:16) */
#define BMMGPU_ALGO_CUBIC 0
#define BMMGPU_ALGO_STRASSEN_WINOGRAD 1
#define BMMGPU_ALGO_ALT_SELF_INVERSE 2
#define BMMGPU_ALGO_ALT_CHAINING 3

/* block-product kernel selection */
#define BMMGPU_KERNEL_AUTO 0
#define BMMGPU_KERNEL_LOP3 1      /* LOP3 AND/XOR|OR word kernel (integer ALU)      */
#define BMMGPU_KERNEL_UMMA_F4 2   /* tcgen05 kind::mxf4 0/1 e2m1, f32 accumulate, persistent CTA pairs */
/* (ids 3 and 4 were the superseded single-CTA and non-persistent CTA-pair forms of the
   tensor-core kernel; their sources are kept under microbench/history/ and the ids are
   rejected with BMMGPU_EINVAL) */

typedef struct bmmgpu_opts {
    uint32_t device_mask; /* bit g = use CUDA device g; 0 = device 0            */
    int32_t kernel;       /* BMMGPU_KERNEL_*                                      */
    int32_t accumulate;   /* 0: C = A.B;  1: C = C (+) A.B  (XOR / OR integration) */
    int32_t leaf_log2;    /* fast algos: log2 of the leaf dimension the recursion stops at
                             and hands to the block-product kernel (>= 6); 0 = auto */
    double* timing_ms;    /* optional out: device time of the product on the slowest device */
    uint64_t device_budget; /* HBM bytes one call may use per device; 0 = what is free.  Products
                               whose operands do not fit run through the out-of-core driver:
                               A row panels resident, B streamed in double-buffered K-chunks
                               from host memory, partial products XOR/OR-integrated on device */
    int32_t force_streaming; /* 0 auto; 1: the out-of-core tile driver (A panels resident, B
                                streamed per column tile); 2: the K-outer pipeline (C resident,
                                A/B K-chunks uploaded while the previous chunk multiplies) */
    int32_t reserved;
} bmmgpu_opts;

/* bmm::LayerPlan (reference include/bmm/plan.hpp:26-44) */
typedef struct bmmgpu_plan {
    int32_t d_host;
    int32_t d_serial;
    int32_t d_parallel;
    int32_t d_inner;
    int32_t workers;
} bmmgpu_plan;

/* ---------------------------------------------------------------- host API */

/* Optional warm-up of the devices in device_mask (0 = device 0): loads every kernel (one
 * tiny product of each kind), fills the stream pool and, with reserve_bytes > 0, grows the
 * device's stream-ordered memory pool by that much, so the first timed call costs what
 * later calls cost.  Calls without it stay correct; they pay the warm-up once. */
int bmmgpu_init(uint32_t device_mask, uint64_t reserve_bytes);

/* C (m x n) = A (m x k) . B (k x n) over the semiring.  Host row-major buffers
 * (A: m*ceil(k/64) words, B: k*ceil(n/64), C: m*ceil(n/64), written in full,
 * pad bits zero).  Any shape, including non-multiples of 64 and empty
 * dimensions.  Replaces bmm::multiply_cubic (reference engine.cpp:132-144 ->
 * cubic_blocked 60-100 / cubic_rowwise 102-128). */
int bmmgpu_cubic(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t m, uint64_t k, uint64_t n,
                 int32_t semiring, const bmmgpu_opts* opts);

/* One 64 x 64 block product in the reference's operand form: out[i] bit k = the GF(2)
 * dot product (parity of popcount) or Boolean dot product of row i of a (64 words, row
 * major) with column k of B given column-major in bt (word k = column k).  One launch
 * and one synchronisation through page-locked mapped memory (no stream lease, no copies
 * beyond the 1.5 KB staging), so callers that loop over blocks pay the launch latency,
 * not a full host-API product.  Replaces bmm::kernel64 (reference engine.cpp:34-56). */
int bmmgpu_kernel64(const uint64_t* a, const uint64_t* bt, uint64_t* out, int32_t semiring);

/* Fast product through a bilinear scheme: square n = 64 * 2^depth, plan.depth()
 * must equal depth.  Cubic algo dispatches to bmmgpu_cubic; Boolean with a fast
 * algo is BMMGPU_EINVAL.  Replaces bmm::multiply (reference engine.cpp:351-382).
 * With several devices in opts->device_mask the top host levels of the recursion
 * (plan.d_host, or an automatic choice when it is 0) are dealt across the devices,
 * one host thread each, and the partial products are XOR-folded slab by slab over
 * peer copies (bmmgpu_dev_multiply_partial).  Operands beyond the device budget (or
 * opts->force_streaming == 1) run out of core.  On one device: the recursion's top
 * plan.d_host levels (0: the fewest that fit the budget) as 7^d_host sub-instances whose
 * operands are generated on the device from pieces of A and B streamed from host memory,
 * each product's Q folded into C by host threads (C must be writable host memory).  On
 * several devices (or with the environment BMMGPU_ALT_OOC=tiles): b x b output tiles
 * (b = 2^17, or n/2), each the XOR of n/b alternative-basis block products of tiles
 * streamed from host memory, row panels of tiles dealt over the devices. */
int bmmgpu_multiply(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int32_t algo,
                    const bmmgpu_plan* plan, int32_t semiring, const bmmgpu_opts* opts);

/* The out-of-core fast product restricted to output row panels [panel_begin, panel_end)
 * of its b x b tiles (b = 2^tile_log2; tile_log2 = 0: the default, 2^17 or n/2): C rows
 * [panel_begin * b, panel_end * b) = those rows of A . B, over the devices of
 * opts->device_mask.  Only those rows of A and C are read / written, all of B is, so
 * ranks of one node can split a product by panels with B in shared host memory. */
int bmmgpu_multiply_panels(const uint64_t* A, const uint64_t* B, uint64_t* C, uint64_t n, int32_t algo,
                           int32_t tile_log2, uint64_t panel_begin, uint64_t panel_end, const bmmgpu_opts* opts);

/* bmm::multiply_alt on interleaved vectors already in the scheme's basis (host
 * buffers of 4^depth * 64 words laid out [4]*depth [4096]; right operand blocks
 * stored transposed, reference bitmatrix.cpp:112-173): c_hat =
 * chi^-1(phi^-1 a_hat . psi^-1 b_hat), computed on one device (the lowest bit of
 * opts->device_mask).  Replaces bmm::multiply_alt (reference engine.cpp:293-349) and
 * is the solve stage of the host pipeline (pipeline.cpp:310). */
int bmmgpu_multiply_alt(const uint64_t* a_hat, const uint64_t* b_hat, uint64_t* c_hat, int32_t depth, int32_t algo,
                        const bmmgpu_opts* opts);

/* In-place basis change of an interleaved vector (host buffer of total_words
 * words laid out [4]*levels ... [inner]): factor 0 phi, 1 psi, 2 chi of the
 * scheme of `algo`; inverse != 0 applies the factor's inverse.  Each level is
 * one in-place pass over [outer][4][inner] (reference engine.cpp:146-172 ->
 * yates.cpp:143-172). */
int bmmgpu_basis_change(uint64_t* words, uint64_t total_words, int32_t levels, int32_t algo, int32_t factor,
                        int32_t inverse);

/* Layout conversions of the bmm:: API (reference bitmatrix.cpp:97-173, the CLI's
 * `transform`, tools/bmm_cli.cpp:210-234) on the device, streamed through it in
 * Morton-aligned super-tiles for host buffers of any size:
 *   BMMGPU_LAYOUT_TRANSPOSE_BLOCKS64: rows x cols (multiples of 64) row-major matrix,
 *     every 64 x 64 block transposed in place (src == dst allowed) -> transpose_blocks64;
 *   BMMGPU_LAYOUT_TO_INTERLEAVED[_RIGHT]: n x n row-major (n = 64 * 2^depth) -> n^2/64
 *     words of 64-word blocks in Morton order (right operand: blocks transposed)
 *     -> to_interleaved(m, plan, Left|Result / Right);
 *   BMMGPU_LAYOUT_FROM_INTERLEAVED[_RIGHT]: the inverse -> from_interleaved.
 * Interleave conversions are out of place.  Errors: BMMGPU_ESHAPE with the reference's
 * messages.  bmmgpu_dev_layout: the same on device buffers, on `stream`. */
#define BMMGPU_LAYOUT_TRANSPOSE_BLOCKS64 0
#define BMMGPU_LAYOUT_TO_INTERLEAVED 1
#define BMMGPU_LAYOUT_TO_INTERLEAVED_RIGHT 2
#define BMMGPU_LAYOUT_FROM_INTERLEAVED 3
#define BMMGPU_LAYOUT_FROM_INTERLEAVED_RIGHT 4
int bmmgpu_layout(const uint64_t* src, uint64_t* dst, uint64_t rows, uint64_t cols, int32_t op,
                  const bmmgpu_opts* opts);

/* BMM1 files (reference bitmatrix.cpp:187-233: "BMM1", rows, cols as LE u64, then
 * rows * ceil(cols/64) LE words) straight between disk and caller storage with parallel
 * positioned I/O (`threads` <= 0: one per host core).  Read into page-locked memory
 * (bmmgpu_host_alloc) the matrix goes to the GPU without a staging copy.  Same checks
 * and messages as the reference reader; malformed files give BMMGPU_EFORMAT.
 * bmmgpu_bmm1_read needs n_words == rows * ceil(cols/64) of the file. */
int bmmgpu_bmm1_info(const char* path, uint64_t* rows, uint64_t* cols);
int bmmgpu_bmm1_read(const char* path, uint64_t* words, uint64_t n_words, int32_t threads);
int bmmgpu_bmm1_write(const char* path, uint64_t rows, uint64_t cols, const uint64_t* words, int32_t threads);

/* -------------------------------------------------------- device-resident API
 * Pointers are device memory on the current CUDA device; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Launch only, no sync. */

/* Padding granularity of the panel product for a kernel: rows of A / Bt a
 * launch tiles by, and the K granule in bits. */
int bmmgpu_dev_granularity(int32_t kernel, uint64_t* m_gran, uint64_t* n_gran, uint64_t* k_gran_bits);

/* Bt (n_pad x kw words, row j = column j of B) from row-major B (k x ceil(n/64)
 * words, row stride ldb words).  Rows j >= n and bits k.. are zero-filled up to
 * n_pad / kw*64.  The 64x64 block transpose is reference bitmatrix.cpp:16-31. */
int bmmgpu_dev_transpose(const uint64_t* dB, uint64_t ldb, uint64_t k, uint64_t n, uint64_t* dBt, uint64_t n_pad,
                         uint64_t kw, void* stream);

/* Panel product on device: dA (m_pad x kw words, row stride lda),
 * dBt (n_pad x kw words, stride ldbt), dC (m_pad x n_pad/64 words, stride ldc).
 * m_pad, n_pad, kw*64 multiples of the kernel granularity.  accumulate != 0
 * XOR/OR-folds into dC (out-of-core K-split integration, reference
 * engine.cpp:81-84). */
int bmmgpu_dev_cubic(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                     uint64_t m_pad, uint64_t n_pad, uint64_t kw, int32_t semiring, int32_t kernel,
                     int32_t accumulate, void* stream);

/* `batch` independent panel products in one persistent launch: product b uses
 * dA + b*sA, dBt + b*sB, dC + b*sC (strides in words; sA or sB = 0 broadcasts
 * one panel to every product), otherwise as bmmgpu_dev_cubic.  The leaf layer of the fast recursion is this call
 * (reference parallel_leaf's 7^d kernel64 calls, engine.cpp:232-272). */
int bmmgpu_dev_cubic_batched(const uint64_t* dA, uint64_t lda, uint64_t sA, const uint64_t* dBt, uint64_t ldbt,
                             uint64_t sB, uint64_t* dC, uint64_t ldc, uint64_t sC, uint64_t batch, uint64_t m_pad,
                             uint64_t n_pad, uint64_t kw, int32_t semiring, int32_t kernel, int32_t accumulate,
                             void* stream);

/* bmmgpu_layout on device buffers (see above), on `stream`. */
int bmmgpu_dev_layout(const uint64_t* d_src, uint64_t* d_dst, uint64_t rows, uint64_t cols, int32_t op,
                      void* stream);

/* dst (+)= src over rows x words (XOR for GF(2), OR for Boolean), device memory,
 * row strides ldd / lds words: the integration of partial products of a K-split or
 * tile-partitioned product (reference cubic_blocked fold, engine.cpp:81-84). */
int bmmgpu_dev_fold(uint64_t* dst, uint64_t ldd, const uint64_t* src, uint64_t lds, uint64_t rows, uint64_t words,
                    int32_t semiring, void* stream);

/* Fast GF(2) product on device, n = 64 * 2^depth: dA (n x n/64 words, stride
 * lda), dBt = Bt of B (n x n/64, stride ldbt; rows padded to 256 in memory),
 * dC (n x n/64, stride ldc).  dA and dBt are only read: the scheme's basis
 * changes are folded into the expand / compress coefficients.  leaf_log2 as in
 * bmmgpu_opts.  Stream-ordered; level buffers come from and return to the
 * device's memory pool as the recursion proceeds. */
int bmmgpu_dev_multiply(uint64_t* dA, uint64_t lda, uint64_t* dBt, uint64_t ldbt, uint64_t* dC, uint64_t ldc,
                        uint64_t n, int32_t algo, int32_t leaf_log2, int32_t kernel, void* stream);

/* The host layer on one device (reference pipeline::coordinate, pipeline.cpp:198-369,
 * with generate_into / aggregate 108-179): the top `host_levels` recursion levels of the
 * fast product are 7^host_levels independent sub-instances; dC (n x n/64, stride ldc,
 * overwritten) = the XOR of the contributions of sub-instances first, first + stride,
 * ... (each generated on the device from dA / dBt, solved by the fast product, folded
 * into its C sub-blocks).  The XOR over first = 0 .. stride-1 is A.B: the multi-device
 * and multi-rank drivers deal sub-instances this way and fold the partials once.
 * 0 <= host_levels <= 4 and at least one recursion level must remain below them
 * (leaf_log2 as in bmmgpu_opts).  dA / dBt are only read. */
int bmmgpu_dev_multiply_partial(const uint64_t* dA, uint64_t lda, const uint64_t* dBt, uint64_t ldbt, uint64_t* dC,
                                uint64_t ldc, uint64_t n, int32_t algo, int32_t host_levels, uint32_t first,
                                uint32_t stride, int32_t leaf_log2, int32_t kernel, void* stream);

/* Host levels the multi-device fast product uses for n on `parts` devices when the
 * plan does not fix them (the most even deal of sub-instances, see capi.cu). */
int bmmgpu_host_levels(uint64_t n, uint32_t parts, int32_t leaf_log2);

/* The output-row slab [begin, end) of part `index` of `parts` (gran-aligned,
 * contiguous, covering [0, m) exactly once).  The single partition rule of the
 * multi-GPU driver (device slabs in bmmgpu_cubic, ranks in bench.py); output
 * slabs are independent, so no exchange step exists.
 * Pure host arithmetic, no device needed. */
int bmmgpu_slab_rows(uint64_t m, uint32_t parts, uint32_t index, uint64_t gran, uint64_t* begin, uint64_t* end);

/* Block-product timer.  bmmgpu_block_timer(1) clears and starts bracketing every
 * block-product launch (cubic, batched, the leaves of the fast recursion, the
 * out-of-core drivers) with CUDA events on its stream; bmmgpu_block_timer(0) stops.
 * bmmgpu_block_timer_read waits for the recorded launches and returns their summed
 * device time and count: the dominant kernel's time inside a longer pipeline
 * (bench.py's roofline).  Off by default. */
int bmmgpu_block_timer(int32_t enable);
int bmmgpu_block_timer_read(double* ms, uint64_t* launches);

/* Number of kernel launches the calling thread's last host-API call made on its
 * devices (plus device-API launches made on this thread since).  Per thread: concurrent
 * calls on other threads do not disturb it. */
uint64_t bmmgpu_last_launch_count(void);

/* Page-locked host memory (cudaHostAlloc, portable across devices) for buffers
 * the host-API calls copy from / into at full link speed: the host pipeline's
 * per-worker sub-instance buffers, callers' operand staging. */
int bmmgpu_host_alloc(uint64_t bytes, void** ptr);
int bmmgpu_host_free(void* ptr);

/* Host->device and device->host bytes the calling thread's last host-API call copied
 * (operands, re-streamed panels, results).  Per thread, like the launch count. */
int bmmgpu_last_copy_bytes(uint64_t* h2d, uint64_t* d2h);

int bmmgpu_device_count(void);
/* Free and total HBM bytes of a device (cudaMemGetInfo). */
int bmmgpu_mem_info(int32_t device, uint64_t* free_bytes, uint64_t* total_bytes);

/* Debug: tensor-core launches that ran with wave-aligned loaders (long-K products with
 * more output tiles than CTA pairs) and loaders that stopped aligning at the spin limit,
 * since the library was loaded (the tests assert the mode runs and never times out). */
int bmmgpu_debug_wave_stats(uint64_t* aligned_launches, uint64_t* loader_timeouts);

/* Debug counter: K2 launches that kept operand A in tensor memory (long-K products,
 * BMMGPU_TS_MIN_STAGES stages or more), since the library was loaded. */
int bmmgpu_debug_ts_launches(uint64_t* launches);

/* Debug: SM clock cycles (clock64) and nanoseconds (globaltimer) of CTA pair 0's MMA loop
 * in the last K2 launch; cycles / ns is the effective SM clock under the power cap. */
int bmmgpu_debug_k2_clock(uint64_t* cycles, uint64_t* ns);
const char* bmmgpu_last_error(void);
const char* bmmgpu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BMMGPU_H */
