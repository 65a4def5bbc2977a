// Host-visible launch interface of the sm_100a kernels (fsx_kernels.cu).
// Every launcher enqueues on `stream` and returns the launch error (if any);
// none of them synchronizes.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fsx {

using i64 = long long;
using u64 = unsigned long long;

constexpr int kMaxLine = 8192;      // longest pow2 line one CTA transforms
constexpr int kMaxTwPow2 = 32768;   // global pow2 twiddle tables cover N <= this
constexpr int kMaxRank = 8;
constexpr int kMaxFusedTaps = 64;
constexpr int kMaxGroups = 16;
constexpr int kMaxDirect = 12288;   // direct-DFT line limit (non-pow2 axes)
// Twiddle buffer layout (tw_all, one per device):
//   tw_all[N + x] = exp(-2 pi i x / N)                   pow2 N <= kMaxTwPow2
//   tw_all[kPassTabBase + 16 N + 16 Ns + (u - 1) Ns + k]  LineFFT<N> pass twiddles
//       = exp(-2 pi i u k / (Ns r))  (pass with span Ns and radix r, 1 <= u < r,
//       k < Ns): the same exact values gathered so a warp's loads are contiguous
constexpr long long kPassTabBase = 2LL * kMaxTwPow2;
constexpr long long kTwAllSize = kPassTabBase + 32LL * kMaxLine;

// exp(-2 pi i x / n) for any x in [0, n): lo[x & mask] * hi[x >> shift]
// (shift == 0: a single full table lo[x]).
struct PhaseTable {
    const double2* lo = nullptr;
    const double2* hi = nullptr;
    int shift = 0;
    i64 mask = 0;
    i64 n = 1;
};

// Four-step twiddle applied around a strided pass: W_n^(b * k) with
// b = column / col_div (the "n2" digit) and k the line position.
// Exponent = (c / col_div) * (k * kmul + o * omul) for column c of outer
// block o at line position k (kmul = 1, omul = 0: the plain four-step case).
struct StepTwiddle {
    int mode = 0;  // 0 none, 1 post-multiply (forward), 2 pre-multiply by conj (inverse)
    i64 col_div = 1;
    i64 kmul = 1, omul = 0;
    PhaseTable tab;
};

// Lines along one axis of a complex array.
//   element(o, c, p) = base[o * block + c + p * inner], p in [0, n)
struct AxisGeom {
    i64 n = 1;       // line length
    i64 inner = 1;   // element stride along the line
    i64 outer = 1;   // number of outer blocks
    i64 block = 1;   // element stride between outer blocks
    i64 ncols = 1;   // columns c in [0, ncols) per outer block (ncols <= inner when inner > 1)
};

// Symbol description for the fused half-spectrum (m = 1, R2C) pass along
// axis 0 of a rank-2/3 pow2 grid.  Taps are grouped by their axis-0 offset.
struct FusedSymbol {
    int rank = 2;
    int ntaps = 0;
    int ngroups = 0;
    i64 n0 = 1, n1 = 1, L = 1;   // dims: axis0, axis1 (rank 3 only), last axis (real length)
    i64 P = 1;                   // half-spectrum row pitch (complex)
    i64 M = 1;                   // L / 2
    int group_off[kMaxGroups];   // axis-0 offset of each group
    int group_partner[kMaxGroups] = {};  // complex symbols: for og > 0, 1 + the group of -og (0: none);
                                         // -1: an -og group folded into its partner
    int tap_group[kMaxFusedTaps];
    int tap_o1[kMaxFusedTaps];   // axis-1 offset (rank 3)
    int tap_olast[kMaxFusedTaps];
    double tap_c[kMaxFusedTaps];
    u64 T = 1;
    double scale = 1.0;          // 1 / prod(dims)
    int real = 0;                // taps symmetric under o -> -o: lam is real
    double neg_mag2 = 0.0;       // |lam|^2 below this: |lam|^T < 2^-1100 (power skipped, 0)
    // rank 2: every multiplier of a half-spectrum column kx > kzero is exactly 0 -- the host proved
    // |lam(k0, kx)|^2 < neg_mag2 for every k0 (compute_kcut's column bound) -- so the fused pass
    // takes 0 without evaluating the symbol (same bits as evaluating it); default: no such column
    i64 kzero = 0x7fffffffffffffffLL;
    // implicit solve (solve_periodic_implicit): groups of the mass kernel Q
    // carry group_set = 1; lam = pinv(lamQ) * lamS with the pinv threshold
    // 1e-12 * max |lamQ| (*qmax_bits, filled by launch_fused_qmax first)
    int implicit = 0;
    int group_set[kMaxGroups] = {};
    const unsigned long long* qmax_bits = nullptr;
    i64 c_off = 0;               // slab decomposition: global frequency of local column block start
                                 // (rank 2: kx offset; rank 3: ky offset)
    i64 c_off_x = 0;             // rank 3 pencil decomposition: kx of the local tile's first column
                                 // (the local [ky][kx] tile has pitch P = its kx block width)
};

// Local column c of a fused-pass tile -> global (kx, ky); valid iff kx <= M.
__host__ __device__ inline void fused_col_freqs(const FusedSymbol& s, i64 c, i64& kx, i64& ky) {
    if (s.rank == 3) {
        ky = c / s.P;
        kx = c - ky * s.P + s.c_off_x;
        ky += s.c_off;
    } else {
        ky = 0;
        kx = c + s.c_off;
    }
}

// Row-kernel output/input layout: pitch rows (blk == 0: element (row, k) at
// row * P + k) or the slab all-to-all layout (blk > 0: column block
// d = k / blk of all rows is contiguous: d * nrows * blk + row * blk + k % blk).
//
// Peer layout (peers != nullptr, blk > 0): column block d of every row lives
// directly in rank d's exchange buffer, peers[d] (a device array of P device
// pointers, NVLink peer memory): element (row, k) at
// peers[d][(row_off + row) * blk + k % blk] -- the [n0][blk] column tile rank
// d transforms.  The row kernels then store / load across NVLink themselves,
// fusing the all-to-all into the row passes.
struct RowLayout {
    i64 P = 0;
    i64 blk = 0;
    i64 nrows = 0;
    double2* const* peers = nullptr;
    i64 row_off = 0;
    i64 kcut = -1;  // exact spectral cut: only columns k <= kcut are stored / loaded (-1: all)
    // (k and blk < 2^31: 32-bit division, the 64-bit one is a long software sequence)
    __host__ __device__ i64 at(i64 row, i64 k) const {
        if (blk == 0) return row * P + k;
        const int d = (int)k / (int)blk;
        return (i64)d * nrows * blk + row * blk + (k - (i64)d * blk);
    }
    __device__ double2* ptr(double2* base, i64 row, i64 k) const {
        if (peers) {
            const int d = (int)k / (int)blk;
            return peers[d] + (row_off + row) * blk + (k - (i64)d * blk);
        }
        return base + at(row, k);
    }
    __device__ const double2* ptr(const double2* base, i64 row, i64 k) const {
        return ptr(const_cast<double2*>(base), row, k);
    }
};

// compile-time layout selection for the hot row kernels (pitch: row * P + k)
template <bool BLK>
__host__ __device__ inline i64 row_at(const RowLayout& l, i64 row, i64 k) {
    if constexpr (BLK) return l.at(row, k);
    else return row * l.P + k;
}
template <bool BLK, class Ptr>
__device__ inline Ptr row_ptr(Ptr H, const RowLayout& l, i64 row, i64 k) {
    if constexpr (BLK) return l.ptr(H, row, k);
    else return H + row * l.P + k;
}

// General spectral stage over a full complex spectrum with m fields.
struct GeneralSymbol {
    int rank = 1;
    int m = 1;
    i64 cells = 1;
    i64 dims[kMaxRank];
    i64 split[kMaxRank];         // 0: natural order; else n1 of a four-step split axis
    PhaseTable tab[kMaxRank];    // exp(-2 pi i x / dims[a])
    int ntaps = 0;
    const long long* offsets = nullptr;  // [ntaps * rank]
    const double* blocks = nullptr;      // [ntaps * m * m]
    // implicit (scalar): second tap set, lambda = pinv(lamQ) * lamS
    int implicit = 0;
    int ntaps_q = 0;
    const long long* offsets_q = nullptr;
    const double* blocks_q = nullptr;
    const double* qmax = nullptr;        // device scalar: max |lamQ|
    u64 T = 1;
    double scale = 1.0;
    i64 batch = 1;                       // independent grids stacked [batch][cells][m] (one symbol)
};

// 1D fused row-pair pass (four-step row stage + pairing + spectral + inverse rows).
struct RowPairArgs {
    double2* z;          // [N1][N2] complex in four-step transposed order
    i64 N1 = 1, N2 = 1;  // M = N1 * N2 complex points
    int mode = 0;        // 0: real packing (m = 1, L = 2M reals); 1: two-for-one (m = 2, N = M)
    const double2* tw_all = nullptr;  // pow2 line twiddles
    PhaseTable wk;       // exp(-2 pi i x / L) for the R2C split twiddle (mode 0) and the symbol
    int ntaps = 0;
    int tap_off[kMaxFusedTaps];
    double tap_b[kMaxFusedTaps][4];   // m x m block, row-major (m <= 2)
    u64 T = 1;
    double scale = 1.0;
    int real = 0;        // symmetric taps: the (block) symbol is real
    double neg_mag2 = 0.0;  // scalar symbol: |lam|^2 below this -> |lam|^T < 2^-1100 (power skipped)
    i64 row_split = 0;   // rows stored digit-reversed by a four-step split of N1 (= N1b), 0: natural
};

// Direct stepping verifier (fsx_naive.cu).  rank <= 3: n[] padded to 3 axes
// with leading 1s and the tap offsets padded the same way (stride 3);
// rank 4..8: n[0..rank), offsets stride rank.
constexpr int kMaxNaiveFields = 8;
struct NaiveGeom {
    int rank = 1, m = 1, ntaps = 0;
    i64 n[kMaxRank];
    i64 cells = 1;
};

struct Flags {
    unsigned int nonfinite;
    unsigned int pad;
    unsigned long long max_re_bits;  // max |re| as ordered bits of a nonnegative double
    unsigned long long max_im_bits;
};

// ---------------------------------------------------------------- launchers
// One-time per (kernel, device, smem) setup: the dynamic shared-memory
// opt-in and (threads > 0) the resident CTAs per SM, cached so a launch costs
// no driver attribute/occupancy queries after the first.
int kernel_prepare(const void* fn, size_t smem, int threads = 0);
// Twiddle tables: tw_all[N + x] = exp(-2 pi i x / N) for pow2 N <= kMaxTwPow2.
// flags != nullptr: the output is also scanned for non-finite values
cudaError_t launch_axis_pow2(const double2* in, double2* out, const AxisGeom& g, int sign,
                             const StepTwiddle& st, const double2* tw_all, cudaStream_t s, Flags* flags = nullptr);
cudaError_t launch_axis_direct(const double2* in, double2* out, const AxisGeom& g, int sign,
                               const PhaseTable& tab, cudaStream_t s);
cudaError_t launch_r2c_rows(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& P,
                            const double2* tw_all, cudaStream_t s);
cudaError_t launch_c2r_rows(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& P,
                            const double2* tw_all, Flags* flags, cudaStream_t s);
cudaError_t launch_fused_r2c(double2* H, const AxisGeom& g, const FusedSymbol& sym,
                             const double2* tw_all, cudaStream_t s);
cudaError_t launch_rowpair(const RowPairArgs& a, cudaStream_t s);
cudaError_t launch_promote(const double* x, double2* z, i64 n, cudaStream_t s);
// fp32 storage mode: widen / narrow (non-finite float results flagged), and
// the plan-1 row passes reading / writing floats directly
cudaError_t launch_widen(const float* x, double* y, i64 n, cudaStream_t s);
cudaError_t launch_narrow(const double* x, float* y, i64 n, Flags* flags, cudaStream_t s);
bool rows_f32_ok(i64 L);
bool axis_f32_ok(const AxisGeom& g);
// fp32 mode: plan-1 column passes in fp32 arithmetic (mode 2 fused, real symbols; 0 / 1 the 3D y passes)
bool f32_compute_enabled();
cudaError_t launch_cols_tma_f32(const void* tensor_map, const AxisGeom& g, int mode, const FusedSymbol& sym,
                                const double2* tw_all, const float2* twf_all, cudaStream_t s);
cudaError_t launch_axis_f32(const void* in, void* out, const AxisGeom& g, int sign, const StepTwiddle& st,
                            const double2* tw_all, cudaStream_t s, Flags* flags);
// (twf_all: the float twiddle copy -> the row FFTs in fp32 arithmetic; nullptr -> fp64)
cudaError_t launch_r2c_rows_f32(const float* x, double2* H, i64 nrows, i64 L, const RowLayout& lay,
                                const double2* tw_all, const float2* twf_all, cudaStream_t s);
cudaError_t launch_c2r_rows_f32(const double2* H, float* x, i64 nrows, i64 L, const RowLayout& lay,
                                const double2* tw_all, const float2* twf_all, Flags* flags, cudaStream_t s);
// Bluestein stages for non-pow2 axes (fsx_kernels.cu): gather * chirp into [lines][P],
// pointwise * Bhat, scatter * chirp * scale (conj in / out for the inverse)
cudaError_t launch_blue_pre(const double2* Z, double2* buf, const AxisGeom& g, i64 P, const double2* chirp, int conj_in,
                            cudaStream_t s);
cudaError_t launch_blue_mul(double2* buf, i64 lines, i64 P, const double2* bhat, cudaStream_t s);
cudaError_t launch_blue_post(const double2* buf, double2* Z, const AxisGeom& g, i64 P, const double2* chirp,
                             double scale, int conj_out, cudaStream_t s);
cudaError_t launch_extract(const double2* z, double* x, i64 n, Flags* flags, cudaStream_t s);
cudaError_t launch_scale(double2* z, i64 n, double scale, cudaStream_t s);
cudaError_t launch_finite_check(const double* x, i64 n, Flags* flags, cudaStream_t s);
cudaError_t launch_spectral_general(double2* z, const GeneralSymbol& sym, cudaStream_t s);
cudaError_t launch_symbol_blocks(double2* out, const GeneralSymbol& sym, int which_q, cudaStream_t s);
cudaError_t launch_symbol_absmax(const GeneralSymbol& sym, double* out_max, cudaStream_t s);
cudaError_t launch_pow_blocks(const double2* in, double2* out, i64 cells, int m, u64 T, cudaStream_t s);
cudaError_t launch_pinv(const double2* in, double2* out, i64 n, const double* maxabs, cudaStream_t s);
cudaError_t launch_absmax(const double2* in, i64 n, double* out_max, cudaStream_t s);
cudaError_t launch_block_mul(const double2* a, const double2* b, double2* out, i64 cells, int m, cudaStream_t s);
cudaError_t launch_block_matvec(const double2* lam, const double2* x, double2* y, i64 cells, int m, cudaStream_t s);
// persistent cp.async-pipelined passes (fsx_pipe.cu)
bool pipe_rows_ok(i64 M);
bool pipe_cols_ok(i64 N);
bool pipe_enabled();
cudaError_t launch_r2c_pipe(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& P, const double2* tw_all,
                            cudaStream_t s);
cudaError_t launch_c2r_pipe(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& P, const double2* tw_all,
                            Flags* flags, cudaStream_t s);
cudaError_t launch_cols_pipe(double2* H, const AxisGeom& g, int mode, const FusedSymbol& sym,
                             const double2* tw_all, cudaStream_t s);
int rows_variant();
cudaError_t launch_r2c_bulk(const double* x, double2* H, i64 nrows, i64 L, const RowLayout& lay, const double2* tw_all,
                            cudaStream_t s);
cudaError_t launch_c2r_bulk(const double2* H, double* x, i64 nrows, i64 L, const RowLayout& lay, const double2* tw_all,
                            Flags* flags, cudaStream_t s);
// one direct periodic stencil step out = sum_taps B a[x + off] (verifier)
cudaError_t launch_step_naive(const double* a, double* out, const NaiveGeom& g, const long long* off,
                              const double* blk, cudaStream_t s);
// max |lamQ| over the half spectrum of an implicit fused symbol (bits of a
// nonnegative double; *out zeroed by the caller)
cudaError_t launch_fused_qmax(const FusedSymbol& sym, i64 ncols, unsigned long long* out, const double2* tw_all,
                              cudaStream_t s);
// C2C strided pass with TMA column I/O, four-step twiddles and an optional
// non-finite scan (fsx_tma.cu); cudaErrorNotSupported when not applicable
cudaError_t launch_axis_tma(const double2* in, double2* out, const AxisGeom& g, int sign, const StepTwiddle& st,
                            const double2* tw_all, cudaStream_t s, Flags* flags);
// 8192-point fused pass as two parity halves (fsx_tma.cu)
bool halves_ok(const AxisGeom& g);
int make_cols_tensor_map_par(void* out_map, void* base, const AxisGeom& g);
// base: the half spectrum the map describes (enables the optional L2 strip prefetch), or nullptr
cudaError_t launch_fused_halves(const void* tensor_map2, const AxisGeom& g, const FusedSymbol& sym,
                                const double2* tw_all, cudaStream_t s, const double2* base = nullptr);
// TMA column passes (fsx_tma.cu); tensor_map points at a 64-byte aligned CUtensorMap
bool tma_cols_ok(i64 N);
int tma_cols_width(i64 N);  // columns per TMA tile (the box width the host encodes)
int make_cols_tensor_map(void* out_map, void* base, const AxisGeom& g);
int make_cols_tensor_map_w(void* out_map, void* base, const AxisGeom& g, int W);  // explicit tile width
cudaError_t launch_cols_tma(const void* tensor_map, const AxisGeom& g, int mode, const FusedSymbol& sym,
                            const double2* tw_all, cudaStream_t s);
cudaError_t launch_transpose_split(const double2* in, double2* out, i64 outer, i64 n1, i64 n2, i64 inner,
                                   int to_natural, cudaStream_t s);

}  // namespace fsx
