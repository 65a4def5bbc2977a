/*
 * fsx.h — C ABI of the B200-native StencilFFT-P periodic solver
 * (libfsx.so, paper_2105_06676_b200/csrc).
 *
 * Drop-in boundary for the reference C++ library's periodic hot path
 * (/root/reference/proj/include/fftstencil/periodic.hpp:43-65 and the
 * spectral/FFT building blocks it is built from).  Plain pointers and sizes;
 * no C++ or torch types.  Every entry point returns an fsx_status; the
 * thread-local message of the last failure is fsx_last_error().
 *
 * Data layout (proj/include/fftstencil/grid.hpp:17-20): a grid of
 * prod(dims) cells x `fields` values, row-major over the dims with the field
 * index innermost, fp64.  Complex arrays are interleaved (re, im) fp64.
 * A stencil kernel is `ntaps` offsets (ntaps x rank int64, row-major) and
 * `ntaps` blocks (ntaps x fields x fields fp64, row-major); repeated offsets
 * accumulate and the taps are used in sorted-offset order
 * (proj/src/kernel.cpp:7-22).
 *
 * Reference error types map to status codes: SpecError -> FSX_ERR_SPEC,
 * NumericError -> FSX_ERR_NUMERIC (proj/include/fftstencil/errors.hpp:9-37).
 */
#ifndef FSX_H_
#define FSX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fsx_status {
    FSX_OK = 0,
    FSX_ERR_SPEC = 1,      /* reference SpecError: invalid shapes, kernels, arguments */
    FSX_ERR_NUMERIC = 2,   /* reference NumericError: non-finite result / residue blow-up */
    FSX_ERR_CUDA = 3,      /* CUDA runtime failure (no device, launch error, ...) */
    FSX_ERR_NCCL = 4,      /* NCCL failure (multi-GPU nccl exchange) */
    FSX_ERR_OOM = 5,       /* device allocation failed */
    FSX_ERR_IO = 6         /* reference IoError: file parsing / reading / writing (errors.hpp:20-24) */
} fsx_status;

#define FSX_MAX_RANK 8

/* GridShape (proj/include/fftstencil/grid.hpp:21-83) */
typedef struct fsx_shape {
    int32_t rank;
    int32_t fields;
    int64_t dims[FSX_MAX_RANK];
} fsx_shape;

/* StencilKernel (proj/include/fftstencil/kernel.hpp:19-56) */
typedef struct fsx_kernel {
    int32_t rank;
    int32_t fields;
    int64_t ntaps;
    const int64_t* offsets; /* ntaps * rank */
    const double* blocks;   /* ntaps * fields * fields */
} fsx_kernel;

/* StageTimings (proj/include/fftstencil/periodic.hpp:14-23): seconds,
 * ACCUMULATED (+=) like the reference's Stopwatch sinks.  On the GPU the
 * stages are CUDA-event intervals on the solve's stream: forward_fft = the
 * forward passes before the fused spectral pass, squaring = the fused pass
 * (last forward line FFT + symbol^T + multiply + first inverse line FFT),
 * hadamard = 0 when fused, inverse_fft = remaining inverse passes, the C2R
 * and the non-finite scan. */
typedef struct fsx_stage_timings {
    double forward_fft;
    double squaring;
    double hadamard;
    double inverse_fft;
    double boundary_recursion;
} fsx_stage_timings;

/* Options (NULL = defaults). */
typedef struct fsx_options {
    int32_t device;     /* CUDA device ordinal (default 0) */
    int32_t path;       /* 0 = auto (fused fast path when eligible), 1 = force general path */
    int32_t stage_events; /* device API: record CUDA events at the stage boundaries of each
                             solve (read back with fsx_last_stage_ms) */
    int32_t spectral_cut; /* 1 = exact spectral cut (2D fused plan, explicit scalar solve): the
                             columns kx whose multipliers lam^T all underflow to 0 (the same
                             |lam|^T < 2^-1100 test the fused pass applies per element, bounded
                             by sum_g |A_g(kx)| on the host) are neither stored by the forward
                             rows nor transformed; the inverse rows read them as 0.  The result
                             is bitwise the full solve's (those columns are exactly 0 there).
                             Default 0: every column moves (the reference's work). */
    void* stream;       /* cudaStream_t to enqueue on (NULL = library stream) */
    /* Multi-GPU (single process; host-pointer fsx_solve_periodic /
     * fsx_solve_periodic_cached of rank-2/3 scalar pow2 grids whose axis 0 (and,
     * in 3D, axis 1) divides by the device count; other problems run on one
     * GPU with the same result contract):
     *   num_gpus  0 = the process default (fsx_set_devices), 1 = one GPU,
     *             P > 1 = slab-decompose axis 0 over P devices;
     *   devices   NULL = ordinals 0..P-1, else P ordinals (a repeated ordinal
     *             runs several ranks on one device: one-GPU emulation);
     *   exchange  FSX_EXCHANGE_AUTO (p2p when every pair has peer access),
     *             FSX_EXCHANGE_P2P (NVLink peer memory: fused into the row
     *             kernels in 2D, chunked copy-engine puts/pulls overlapping
     *             the y passes in 3D), FSX_EXCHANGE_NCCL (grouped
     *             ncclSend/ncclRecv all-to-alls; libnccl.so.2 loaded on use). */
    int32_t num_gpus;
    int32_t exchange;
    const int32_t* devices;
    /* decomp: FSX_DECOMP_AUTO (slabs when axis 0 -- and in 3D axis 1 -- divide
     * by P, else pencils when they apply), FSX_DECOMP_SLAB, FSX_DECOMP_PENCIL
     * (3D only: a Pr x Pc grid; rank (pr, pc) owns planes [pr n0/Pr, ...) and
     * rows [pc n1/Pc, ...) of axis 1; four transposes per solve, over peer
     * memory by the copy engines; pencil_rows = Pr, 0 = the most square
     * factorization of P).  Slabs are pencils with Pr = 1 and need two
     * transposes: they are the better choice whenever they apply. */
    int32_t decomp;
    int32_t pencil_rows;
} fsx_options;

#define FSX_DECOMP_AUTO 0
#define FSX_DECOMP_SLAB 1
#define FSX_DECOMP_PENCIL 2

#define FSX_EXCHANGE_AUTO 0
#define FSX_EXCHANGE_P2P 1
#define FSX_EXCHANGE_NCCL 2

/* Process default device list for host solves whose options leave num_gpus
 * at 0 (the drop-in C++ header passes no options): n = 0 or 1 -> one GPU.
 * The multi-GPU counterpart of the reference's process-wide thread budget
 * (proj/include/fftstencil/parallel.hpp, set_num_threads; parallel.cpp:11-21).
 * devices NULL = ordinals 0..n-1.  Ordinals are validated against the visible
 * devices.  fsx_get_devices copies up to cap ordinals and returns the count. */
fsx_status fsx_set_devices(const int32_t* devices, int32_t n);
int32_t fsx_get_devices(int32_t* devices, int32_t cap);

/* Opaque spectrum/plan cache (proj/include/fftstencil/periodic.hpp:28-35). */
typedef struct fsx_spectrum_cache fsx_spectrum_cache;

/* ---------------------------------------------------------------- solvers
 * Host pointers; `out` may alias `a0`.  T == 0 copies a0 bit-exactly after
 * validation (proj/src/periodic.cpp:78-79). */

/* solve_periodic (proj/src/periodic.cpp:76-86) */
fsx_status fsx_solve_periodic(const fsx_shape* shape, const double* a0, const fsx_kernel* k,
                              uint64_t T, double* out, const fsx_options* opt,
                              fsx_stage_timings* st);

/* solve_periodic_vector (proj/src/periodic.cpp:101-106): requires fields >= 2 */
fsx_status fsx_solve_periodic_vector(const fsx_shape* shape, const double* a0, const fsx_kernel* k,
                                     uint64_t T, double* out, const fsx_options* opt,
                                     fsx_stage_timings* st);

/* solve_periodic_cached + SpectrumCache (proj/src/periodic.cpp:67-99): the
 * cache memoises the device plan (symbol tables, workspaces) by dims, like
 * the reference memoises the spectrum by dims only. */
fsx_spectrum_cache* fsx_spectrum_cache_create(void);
void fsx_spectrum_cache_destroy(fsx_spectrum_cache* cache);
fsx_status fsx_solve_periodic_cached(const fsx_shape* shape, const double* a0, const fsx_kernel* k,
                                     uint64_t T, fsx_spectrum_cache* cache, double* out,
                                     const fsx_options* opt, fsx_stage_timings* st);

/* solve_periodic_implicit (proj/src/periodic.cpp:108-124): scalar q, s */
fsx_status fsx_solve_periodic_implicit(const fsx_shape* shape, const double* a0, const fsx_kernel* q,
                                       const fsx_kernel* s, uint64_t T, double* out,
                                       const fsx_options* opt, fsx_stage_timings* st);

/* Pipelined batch of nbatch independent solves of one shape, kernel and T
 * (host pointers a0s[i] -> outs[i], each may alias).  Two internal lanes keep
 * one solve's D2H, the next one's H2D and the kernels in flight together, so
 * with PINNED host buffers a batch runs at ~max(H2D, D2H, kernels) per solve.
 * Returns synchronized; FSX_ERR_NUMERIC names the first failing item (the
 * other outputs are valid).  Extension for batched slab solves (the
 * aperiodic recursion's rb_run, proj/src/aperiodic.cpp:226-244). */
fsx_status fsx_solve_periodic_batch(const fsx_shape* shape, int64_t nbatch, const double* const* a0s,
                                    const fsx_kernel* k, uint64_t T, double* const* outs, const fsx_options* opt);

/* One recursion level's slab solves (the aperiodic recursion's rb_run, which
 * calls solve_periodic_cached on each of the 2d face slabs of a level in turn,
 * proj/src/aperiodic.cpp:224-228,240-244): nslabs grids of possibly different
 * shapes (shapes[i], host pointers a0s[i] -> outs[i], each may alias), one
 * kernel and T.  Slabs of equal shape are stacked and solved as one batched
 * plan (one launch per pass for all of them, the stack an outer dimension of
 * every pass); different shapes run on the device's two lanes so their
 * copies and kernels overlap.  cache (may be NULL): SpectrumCache semantics of
 * fsx_solve_periodic_cached -- the first kernel seen for a dims vector is used
 * for every later slab with those dims.  Plans stay resident per device
 * (keyed by shape and stack size) across calls.  Returns synchronized;
 * FSX_ERR_NUMERIC names the first failing slab in argument order (the other
 * outputs are valid).  st (may be NULL): the call's wall time is accumulated
 * into boundary_recursion (the reference's stage for the recursion's solves,
 * proj/src/aperiodic.cpp:310-313). */
fsx_status fsx_solve_periodic_slabs(int64_t nslabs, const fsx_shape* shapes, const double* const* a0s,
                                    const fsx_kernel* k, uint64_t T, fsx_spectrum_cache* cache, double* const* outs,
                                    const fsx_options* opt, fsx_stage_timings* st);

/* Device-resident variant: d_a0 / d_out are device pointers (may alias);
 * the work is enqueued on opt->stream and the call returns without
 * synchronizing.  The non-finite check is deferred: fsx_device_check()
 * synchronizes that stream and reports FSX_ERR_NUMERIC if any solve
 * enqueued since the last check produced a non-finite value. */
fsx_status fsx_solve_periodic_device(const fsx_shape* shape, const double* d_a0, const fsx_kernel* k,
                                     uint64_t T, double* d_out, const fsx_options* opt);
fsx_status fsx_device_check(const fsx_options* opt);

/* fp32 mode (north star: an optional fp32 mode at <= 1e-4 relative L2 vs the
 * fp64 reference).  Float grids in and out: half the PCIe traffic of the host
 * entry points and, on the fused 2D/3D plan, half the HBM bytes of the first
 * and last row passes (the row kernels read and write floats directly; the
 * 1D plan's strided first / last column passes do too; other shapes widen /
 * narrow around their fp64 buffers).  The symbol power and the half spectrum
 * stay fp64; for a real (symmetric) symbol on that plan the row FFTs and the
 * fused column pass's FFTs run in fp32 (~1e-7 relative; FSX_F32_COMPUTE=0
 * keeps them fp64, and every other path is fp64 arithmetic: the fp64 solve of
 * the widened input rounded once, ~6e-8).  A result outside the float range raises FSX_ERR_NUMERIC.
 * Same shapes, kernels, T == 0 (bit-exact copy) and error rules as
 * fsx_solve_periodic / fsx_solve_periodic_device / fsx_solve_periodic_batch;
 * no implicit or cached variants.  No reference counterpart (the reference
 * library is fp64 only, proj/include/fftstencil/grid.hpp:86-100). */
fsx_status fsx_solve_periodic_f32(const fsx_shape* shape, const float* a0, const fsx_kernel* k, uint64_t T,
                                  float* out, const fsx_options* opt, fsx_stage_timings* st);
fsx_status fsx_solve_periodic_device_f32(const fsx_shape* shape, const float* d_a0, const fsx_kernel* k,
                                         uint64_t T, float* d_out, const fsx_options* opt);
fsx_status fsx_solve_periodic_batch_f32(const fsx_shape* shape, int64_t nbatch, const float* const* a0s,
                                        const fsx_kernel* k, uint64_t T, float* const* outs,
                                        const fsx_options* opt);

/* Direct-stepping verifier (not the solve path): the reference's naive
 * oracle step_periodic / evolve_periodic_naive (proj/src/oracle.cpp:90-115,
 * oracle.hpp:15-20) on the GPU, bitwise equal to the reference loop (taps in
 * sorted-offset order, products and sums rounded separately).  T direct
 * steps; an independent full-size check of the FFT solver.  Host pointers
 * (returns synchronized) or, for _device, device pointers enqueued on
 * opt->stream.  Ranks 1-8; fields <= 8; for rank <= 3 the axes before the
 * last must be <= 65535. */
fsx_status fsx_step_periodic(const fsx_shape* shape, const double* a, const fsx_kernel* k, double* out,
                             const fsx_options* opt);
fsx_status fsx_evolve_periodic_naive(const fsx_shape* shape, const double* a0, const fsx_kernel* k, uint64_t T,
                                     double* out, const fsx_options* opt);
fsx_status fsx_evolve_periodic_naive_device(const fsx_shape* shape, const double* d_a0, const fsx_kernel* k,
                                            uint64_t T, double* d_out, const fsx_options* opt);

/* Stage durations (ms) of the most recent device solve enqueued with
 * opt->stage_events = 1: ms[0] forward passes, ms[1] the fused spectral
 * pass (plan 1: exactly one kernel, k_fused_r2c), ms[2] inverse passes.
 * Waits for that solve's last stage event. */
fsx_status fsx_last_stage_ms(const fsx_options* opt, double* ms);

/* ---------------------------------------------------------------- slab decomposition
 * Multi-GPU StencilFFT-P for rank-2/3 scalar pow2 grids (plan 1 eligible):
 * rank r of P owns planes [r n0/P, (r+1) n0/P) of axis 0 of the real grid.
 * One solve is
 *     fsx_slab_forward(local a0 -> send)
 *     all_to_all(recv <- send)      equal split: P chunks of xbuf_bytes / P
 *     fsx_slab_spectral(recv, in place)
 *     all_to_all(send <- recv)
 *     fsx_slab_inverse(send -> local out)
 * with the all-to-alls done by the caller (NCCL over NVLink).  The exchange
 * layout needs no pack/unpack in 2D: the R2C rows are written directly as
 * P column blocks, and the received buffer is already the [n0][block] column
 * tile the fused pass transforms (3D packs with 2D copies after the local
 * y pass).  All calls are asynchronous on opt->stream; device pointers; the
 * non-finite check is deferred to fsx_device_check(). */
typedef struct fsx_slab_info {
    int32_t nranks;
    int32_t rank;
    int64_t local_dims[FSX_MAX_RANK]; /* this rank's slab of the real grid */
    int64_t plane_offset;             /* first global index along axis 0 */
    int64_t col_block;                /* 2D: kx columns per rank; 3D: ky rows per rank */
    int64_t xbuf_bytes;               /* size of each exchange buffer (send and receive) */
} fsx_slab_info;
fsx_status fsx_slab_describe(const fsx_shape* global, int32_t nranks, int32_t rank, fsx_slab_info* info);
fsx_status fsx_slab_forward(const fsx_shape* global, int32_t nranks, int32_t rank, const double* d_local_in,
                            double* d_send, const fsx_options* opt);
fsx_status fsx_slab_spectral(const fsx_shape* global, const fsx_kernel* k, uint64_t T, int32_t nranks,
                             int32_t rank, double* d_recv, const fsx_options* opt);
fsx_status fsx_slab_inverse(const fsx_shape* global, int32_t nranks, int32_t rank, const double* d_send,
                            double* d_local_out, const fsx_options* opt);

/* The same decomposition with the exchange fused into the row passes (2D):
 * d_recv_peers is a DEVICE array of nranks device pointers, entry d = rank
 * d's exchange buffer (xbuf_bytes, mapped into this process: NVLink peer
 * memory, e.g. torch symmetric memory's buffer_ptrs_dev).  One solve is
 *     barrier; fsx_slab_forward_p2p   (R2C rows store block d into rank d's buffer)
 *     barrier; fsx_slab_spectral      (own buffer, in place)
 *     barrier; fsx_slab_inverse_p2p   (C2R rows load their blocks from every rank)
 * where "barrier" is a cross-rank device barrier on the same stream.  No
 * all-to-all: the NVLink traffic overlaps the row FFTs inside the kernels. */
fsx_status fsx_slab_forward_p2p(const fsx_shape* global, int32_t nranks, int32_t rank, const double* d_local_in,
                                void* const* d_recv_peers, const fsx_options* opt);
fsx_status fsx_slab_inverse_p2p(const fsx_shape* global, int32_t nranks, int32_t rank, void* const* d_recv_peers,
                                double* d_local_out, const fsx_options* opt);

/* ---------------------------------------------------------------- building blocks
 * (host pointers, complex = interleaved fp64) */

/* multi_fft / multi_ifft (proj/src/fft.cpp:159-192): per-axis DFT, fields
 * transformed independently; inverse carries 1/n per axis. */
fsx_status fsx_multi_fft(const fsx_shape* shape, const double* in, double* out, int32_t inverse);

/* spectrum_from_kernel (proj/src/spectrum.cpp:21-45): cells * m * m blocks */
fsx_status fsx_spectrum_from_kernel(const fsx_shape* shape, const fsx_kernel* k, double* out);

/* pow_spectrum (proj/src/spectrum.cpp:47-83) */
fsx_status fsx_pow_spectrum(const fsx_shape* shape, const double* blocks, uint64_t T, double* out);

/* pseudo_inverse_spectrum (proj/src/spectrum.cpp:85-96), scalar only */
fsx_status fsx_pseudo_inverse_spectrum(const fsx_shape* shape, const double* blocks, double* out);

/* multiply_spectra (proj/src/spectrum.cpp:98-109) */
fsx_status fsx_multiply_spectra(const fsx_shape* shape, const double* a, const double* b, double* out);

/* hadamard (proj/src/spectrum.cpp:111-134): y = lam x per frequency */
fsx_status fsx_hadamard(const fsx_shape* shape, const double* lam, const double* x, double* y);

/* ---------------------------------------------------------------- grid I/O and the bench stage table
 * (proj/include/fftstencil/grid_io.hpp,
 * proj/src/grid_io.cpp, proj/src/runner.cpp:46-115).
 * raw: little-endian float64, row-major dims then field, plus "<path>.meta"
 * ("dims = ...", "fields = m", "dtype = float64", "order = row-major");
 * csv: one line per (cell, field) "i1,...,id,f,value", shortest round-trip
 * decimals.  Reading detects raw by the presence of the sidecar.  Malformed
 * input -> FSX_ERR_IO naming the offending line or byte count. */
#define FSX_GRID_CSV 0
#define FSX_GRID_RAW 1
fsx_status fsx_write_grid(const fsx_shape* shape, const double* data, const char* path, int32_t format);
/* The grid's shape as stored (raw: from the sidecar, validated against the file size). */
fsx_status fsx_read_grid_shape(const char* path, fsx_shape* shape);
/* Host read; `shape` (may be NULL) must equal the stored shape. */
fsx_status fsx_read_grid(const char* path, const fsx_shape* shape, double* out);
/* Raw grid straight into device memory d_out (opt->device): chunked reads into
 * two pinned staging buffers, each chunk's H2D overlapping the next read.
 * Returns after the data is on the device. */
fsx_status fsx_load_grid_device(const char* path, const fsx_shape* shape, double* d_out, const fsx_options* opt);
/* run_bench's stage table (runner.cpp:46-62) for accumulated StageTimings,
 * the call's total seconds and (>= 0) the naive solver's seconds. */
fsx_status fsx_format_stage_table(const fsx_stage_timings* st, double total, double naive_seconds, char* buf,
                                  int64_t buflen);

/* ---------------------------------------------------------------- introspection */
const char* fsx_last_error(void);
/* ABI version: 200 = round 2 (fsx_options grew num_gpus / exchange / devices /
 * decomp / pencil_rows, fsx_plan_info grew sched_bytes / ranks / exchange /
 * decomp / pencil_rows; callers built against 100 must be rebuilt). */
#define FSX_ABI_VERSION 200
int32_t fsx_version(void);
int32_t fsx_device_count(void);

/* Plan description for measurement: which path a problem takes, how many
 * of our kernels one solve launches and the algorithmic HBM bytes of the
 * minimal pass schedule. */
typedef struct fsx_plan_info {
    int32_t path;            /* 1 = fused R2C (rank 2/3), 2 = 1D four-step row-pair, 3 = general */
    int32_t launches;        /* kernels per solve */
    int64_t alg_bytes;       /* algorithmic bytes of the minimal pass schedule */
    int64_t fused_bytes;     /* algorithmic bytes of the dominant (fused) kernel */
    int64_t work_bytes;      /* device workspace of the plan */
    int64_t sched_bytes;     /* bytes the launched pass schedule moves (> alg_bytes when a pass is split,
                                e.g. the 1D plan's two-level column FFT above 8192 columns) */
    int32_t ranks;           /* devices a host solve is decomposed over (1 = single GPU) */
    int32_t exchange;        /* ranks > 1: FSX_EXCHANGE_P2P or FSX_EXCHANGE_NCCL as resolved */
    int32_t decomp;          /* ranks > 1: FSX_DECOMP_SLAB or FSX_DECOMP_PENCIL as resolved */
    int32_t pencil_rows;     /* pencils: Pr (the grid is Pr x ranks / Pr) */
} fsx_plan_info;
/* Columns the exact spectral cut keeps for this solve (kept <= total = L/2 + 1;
 * kept == total when the cut does not apply: other plans, rank 3, T == 1, ...). */
fsx_status fsx_spectral_cut_columns(const fsx_shape* shape, const fsx_kernel* k, uint64_t T, int64_t* kept,
                                    int64_t* total);
fsx_status fsx_plan_describe(const fsx_shape* shape, const fsx_kernel* k, const fsx_options* opt,
                             fsx_plan_info* info);

#ifdef __cplusplus
}
#endif

#endif /* FSX_H_ */
