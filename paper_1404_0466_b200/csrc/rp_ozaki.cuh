// FP64 symmetric rank-K products C = A A^T (or C -= A A^T) on the 5th-generation tensor cores
// (tcgen05, kind::i8) by the Ozaki scheme. Used for the Gram blocks G_b = X_b^T X_b and the
// trailing updates of the blocked Cholesky.
//
// sm_100a has no FP64 tcgen05 MMA: the FP64 path (mma.sync DMMA) peaks at 37 TFLOP/s, while the
// int8 tensor cores run at ~4 POPS. A (M x K, column-major) is cut into fixed-point slices
//
//   per row i:  a_ik = 2^(E_i - 54) * sum_{p<S} d_p(i,k) 256^(S-1-p),   d_p in [-128, 127]
//   (E_i = exponent of max_k |a_ik|; |a| 2^(54 - E_i) < 2^54 truncated to an integer and written
//   as S = 7 balanced base-256 digits), so
//
//   (A A^T)_ij = 2^(E_i+E_j) sum_{g<S} 2^(-8g-12) C_g(i,j),   C_g = sum_{p+q=g} S_p S_q^T
//
// with C_g exact in int32 and the 28 products of weight below 2^(-8S-4) dropped (the order of
// the digit truncation): FP64-level accuracy in the sqrt(C_ii C_jj) norm.
//
// Kernels:
//   oz_rowexp_kernel     E[b][i] + range guard    (one pass over A, row max and sum of squares)
//   oz_gram_prep_*       the same for A = X_b^T, fused with C_b = X_b^T Y_b (one pass over X)
//   oz_slice_kernel      digits, K-major int8 slices [b][p][k / 32][i][32 bytes, swizzled] (oz_slice_offset)
//   oz_syrk_pair_kernel  persistent, warp-specialised, 2-CTA clusters (tcgen05 cta_group::2,
//                        M = 256, N = 128, K = 32): warp 0 of each CTA issues the TMA loads
//                        (SWIZZLE_32B boxes, its own 128 rows of A_I and 64 rows of A_J), warp 1
//                        of the leader issues the MMAs into 4 weight-group accumulators of
//                        128 x 128 int32 (all 512 TMEM columns), warps 2-9 of both CTAs drain TMEM
//                        (tcgen05.ld) into FP64 registers and add the tile into C with a single
//                        read-modify-write that overlaps the next tile's MMAs. Only 4 groups fit in
//                        TMEM, so a tile runs two passes over K: groups 4..6 (all 7 slices), then
//                        0..3 (slices 0..3). K is cut in chunks short enough that no int32
//                        accumulator can overflow (7 pairs x 128^2 x K_chunk < 2^31).
//   oz_dotb_pair_kernel  the Gram-form hold-out w^T T w on the same machinery.
// Every product has a device-side range guard (OZ_RANGE_BITS below) with a gated FP64 DMMA fallback.
#pragma once
#include "rp_common.cuh"

namespace rp {

constexpr int OZ_S = 7;  // slices: balanced base-256 digits of a 54-bit fixed-point value
constexpr int OZ_BM = 128, OZ_BK = 32, OZ_GP = 4;
constexpr int OZ_SYRK_THREADS = 320;  // producer, MMA, 8 epilogue warps (SYRK and hold-out kernels)
constexpr int OZ_SLICE = OZ_BM * OZ_BK;             // bytes of one 128 x 32 slice tile
// Row exponent marking a row with a NaN or infinity: the entries it touches are NaN, as in FP64.
constexpr int OZ_NONFINITE = 0x7fffffff;

inline int64_t oz_kpad(int64_t k) { return (k + 63) / 64 * 64; }

// K-chunk such that S ordered pairs of int8 products never overflow an int32 accumulator.
inline int64_t oz_kchunk(int64_t kpad) {
  int64_t c = (2147483647LL / ((int64_t)OZ_S * 128 * 128)) / OZ_BK * OZ_BK;
  return c < kpad ? c : kpad;
}

struct OzIn {  // A_b: M x K column-major, element (i, k) at A + b * bstride + k * lda + i
  const double* A;
  int64_t lda, bstride, K;
  int M, nbatch;
  int Mpad = 0;  // rows of the slice layout (>= M, multiple of 128; 0 = M); rows >= M are zero
  int tri = 0;   // 1: use T = strict_lower(A) + diag(A)/2 instead of A (A square, lower read only)
  __host__ __device__ int mpad() const { return Mpad ? Mpad : M; }
};

// ------------------------------------------------------------------ preprocessing

// Range guard. Per-row scaling truncates every entry of row i at 2^(E_i - 54), E_i the exponent of
// the row's largest entry: normwise (relative to sqrt(C_ii C_jj)) this is always FP64-level, but an
// entry 2^g below the row max keeps only 54 - g bits, so when the BULK of a row sits far below its
// largest entry (a huge outlier among unit-scale values, heavy tails) the small entries of C --
// and the small-eigenvalue directions a later Cholesky solve depends on -- lose accuracy that
// FP64 keeps. The guard measures that gap as the row's largest exponent minus the mean exponent of
// its nonzero entries (a geometric mean: Gaussian rows ~2.5 bits, sparse rows count only their
// nonzeros) and sets *guard when it exceeds the product's bit budget (OZ_RANGE_BITS for the Gram
// blocks and the Cholesky trailing updates; the hold-out's quadratic form only needs normwise
// accuracy and uses OZ_RANGE_BITS_DOT). Every tensor-core kernel of the call then exits at once and
// the gated FP64 DMMA kernel launched beside it computes the product. Zero and non-finite rows are
// not guarded (zeros are exact; NaN/inf propagate).
constexpr int OZ_RANGE_BITS = 10;
constexpr int OZ_RANGE_BITS_DOT = 24;
RP_DEVINL int oz_biased_exp(double v) { return (int)((__double_as_longlong(v) >> 52) & 0x7ff); }
RP_DEVINL bool oz_out_of_range(double mx, double se, double nz, int bits) {
  return nz > 0.0 && mx > 0.0 && mx <= 1.79769313486231570e308 && (double)oz_biased_exp(mx) - se / nz > (double)bits;
}

// E[b][i]: exponent with max_k |a_ik| < 2^E (0 for an all-zero row, OZ_NONFINITE if any entry is
// NaN or infinite), and the range guard (range_bits).
// One CTA per 32 rows: 8 warps stride over k (each warp reads 32 contiguous rows of A per k:
// coalesced), then a max / sum-of-squares reduction over the warps in shared memory.
// row_mask (optional): out-of-range rows mark their 128-row tile in row_mask[b * mask_tiles + i / 128]
// instead of tripping the guard (the hold-out's W^T rows: only those columns fall back to FP64).
__global__ void __launch_bounds__(256) oz_rowexp_kernel(OzIn in, int* E, int* guard, int range_bits,
                                                        int* row_mask = nullptr, int mask_tiles = 0) {
  __shared__ double smx[8][32], sse[8][32], snz[8][32];
  __shared__ int sfin[8][32];
  const int b = blockIdx.y, lane = threadIdx.x & 31, wk = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const int mp = in.mpad();
  double mx = 0.0, se = 0.0, nz = 0.0;
  bool finite = true;
  const int64_t kend = in.tri ? (i + 1 < in.K ? i + 1 : in.K) : in.K;  // T: columns k <= i
  if (i < in.M) {
    const double* x = in.A + (int64_t)b * in.bstride + i;
#pragma unroll 4
    for (int64_t k = wk; k < kend; k += 8) {
      double v = fabs(__ldcs(x + k * in.lda));
      finite &= (v <= 1.79769313486231570e308);  // false for NaN and inf
      if (in.tri && k == i) v *= 0.5;             // T's diagonal
      mx = fmax(mx, v);
      if (v != 0.0) {
        se += (double)oz_biased_exp(v);
        nz += 1.0;
      }
    }
  }
  smx[wk][lane] = mx;
  sse[wk][lane] = se;
  snz[wk][lane] = nz;
  sfin[wk][lane] = finite ? 1 : 0;
  __syncthreads();
  if (E != nullptr && wk == 0 && i < mp) {
    for (int w = 1; w < 8; ++w) {
      mx = fmax(mx, smx[w][lane]);
      se += sse[w][lane];
      nz += snz[w][lane];
      finite = finite && sfin[w][lane];
    }
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);
    E[(int64_t)b * mp + i] = (i < in.M && !finite) ? OZ_NONFINITE : e;
    if (guard != nullptr && i < in.M && finite && oz_out_of_range(mx, se, nz, range_bits)) {
      if (row_mask != nullptr)
        atomicOr(&row_mask[(int64_t)b * mask_tiles + i / 128], 1);
      else
        atomicOr(guard, 1);
    }
  }
}

// Gram blocks: the row exponents of A_b = X_b^T fused with C_b = X_b^T Y_b (both need one pass
// over X_b; done separately they read X twice more than the slicing does). X_b row-major
// (rows x d, leading dimension ldx), Y_b row-major (rows x m, ldy). CTA = (1024 columns, a chunk
// of rows, block): 256 threads x 4 columns (consecutive threads on consecutive columns, so every
// row read is coalesced and each Y row is one broadcast for 4 columns). Per chunk the rows are
// summed in order; with nchunk > 1 the chunk partials (sums, |max| with +inf marking NaN/inf) go
// to Cp / Mp and oz_gram_prep_reduce_kernel combines them in chunk order, with nchunk == 1 the
// kernel writes C and E itself. E[b][i] as oz_rowexp_kernel (stride mp, rows i >= d get 0;
// E = nullptr: X^T Y only, the FP64 Gram's side stream); C[b][o][i] column-major d x m.
RP_DEVINL int oz_exp_code(double mx) {  // mx = +inf marks a NaN/inf entry
  if (!(mx <= 1.79769313486231570e308)) return OZ_NONFINITE;
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);
  return e;
}

template <int MT>
__global__ void __launch_bounds__(256) oz_gram_prep_kernel(const double* X, int64_t ldx, int64_t rows, int d,
                                                           const double* Y, int64_t ldy, int m, int nchunk,
                                                           double* Cp, double* Mp, int mp, int* E, double* C,
    int* guard) {
  constexpr int MM = MT > 0 ? MT : 1;
  const int b = blockIdx.z, ch = blockIdx.y;
  const int i0 = blockIdx.x * 1024 + threadIdx.x;
  const int64_t r0 = rows * ch / nchunk, r1 = rows * (ch + 1) / nchunk;
  double acc[4][MM], mx[4], se[4], nz[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    mx[j] = se[j] = nz[j] = 0.0;
#pragma unroll
    for (int o = 0; o < MM; ++o) acc[j][o] = 0.0;
  }
  const double* x = X + (int64_t)b * rows * ldx + i0;
  const double* y = Y + (int64_t)b * rows * ldy;
#pragma unroll 2
  for (int64_t r = r0; r < r1; ++r) {
    double yv[MM];
#pragma unroll
    for (int o = 0; o < MM; ++o) yv[o] = __ldg(y + r * ldy + o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i0 + 256 * j < d) {
        const double xv = __ldcs(x + r * ldx + 256 * j);
        const double av = fabs(xv);
        mx[j] = (av <= 1.79769313486231570e308) ? fmax(mx[j], av) : __longlong_as_double(0x7ff0000000000000LL);
        if (av != 0.0) {
          se[j] += (double)oz_biased_exp(av);
          nz[j] += 1.0;
        }
#pragma unroll
        for (int o = 0; o < MM; ++o) acc[j][o] = fma(xv, yv[o], acc[j][o]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = i0 + 256 * j;
    // compile-time bound on o (a runtime bound would index acc dynamically: local memory)
    if (nchunk == 1) {
      if (E != nullptr && i < mp) E[(int64_t)b * mp + i] = i < d ? oz_exp_code(mx[j]) : 0;
      if (guard != nullptr && i < d && oz_out_of_range(mx[j], se[j], nz[j], OZ_RANGE_BITS)) atomicOr(guard, 1);
      if (i < d) {
#pragma unroll
        for (int o = 0; o < MM; ++o)
          if (o < m) C[((int64_t)b * m + o) * d + i] = acc[j][o];
      }
    } else if (i < d) {
      Mp[((int64_t)b * nchunk + ch) * d + i] = mx[j];
      Mp[((int64_t)(gridDim.z + b) * nchunk + ch) * d + i] = se[j];  // exponent sums and nonzero counts
      Mp[((int64_t)(2 * gridDim.z + b) * nchunk + ch) * d + i] = nz[j];  // after the maxima
#pragma unroll
      for (int o = 0; o < MM; ++o)
        if (o < m) Cp[(((int64_t)b * nchunk + ch) * m + o) * d + i] = acc[j][o];
    }
  }
}

// Same computation with the X rows streamed into shared memory by bulk copies (8 KB row segments,
// an 8-deep ring completed on mbarriers): the register-resident version keeps only four loads per
// thread in flight and runs at ~2.3 TB/s, latency-bound. The Y row rides in the same stage.
// Requires 16-byte aligned rows (ldx, d, ldy and m even; X and Y 16-byte aligned).
constexpr int OZ_GP_STAGES = 8;
constexpr int OZ_GP_ROW = 1024 + 16;  // per stage: the X row segment, then the Y row (m <= 16)
constexpr size_t OZ_GP_SMEM = sizeof(double) * OZ_GP_STAGES * OZ_GP_ROW + 2 * OZ_GP_STAGES * sizeof(uint64_t);

template <int MT>
__global__ void __launch_bounds__(256, 2) oz_gram_prep_bulk_kernel(const double* X, int64_t ldx, int64_t rows, int d,
                                                                const double* Y, int64_t ldy, int m, int nchunk,
                                                                double* Cp, double* Mp, int mp, int* E, double* C,
    int* guard) {
  constexpr int MM = MT > 0 ? MT : 1;
  extern __shared__ __align__(16) double gp_smem[];
  double* sx = gp_smem;  // [stage][OZ_GP_ROW]
  uint64_t* full = reinterpret_cast<uint64_t*>(gp_smem + OZ_GP_STAGES * OZ_GP_ROW);
  uint64_t* empty = full + OZ_GP_STAGES;
  const int b = blockIdx.z, ch = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const int c0 = blockIdx.x * 1024, i0 = c0 + tid;
  const int width = d - c0 < 1024 ? d - c0 : 1024;  // columns of this segment
  const int64_t r0 = rows * ch / nchunk, r1 = rows * (ch + 1) / nchunk, nr = r1 - r0;
  const double* xseg = X + (int64_t)b * rows * ldx + c0;
  const double* y = Y + (int64_t)b * rows * ldy;
  if (tid == 0) {
    for (int s2 = 0; s2 < OZ_GP_STAGES; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int64_t rr) {  // row r0 + rr into stage rr % STAGES
    if (tid == 0 && rr < nr) {
      const int st = (int)(rr % OZ_GP_STAGES);
      if (rr >= OZ_GP_STAGES) mbar_wait(&empty[st], (uint32_t)(((rr / OZ_GP_STAGES) + 1) & 1));
      mbar_arrive_expect_tx(&full[st], (uint32_t)((width + m) * 8));
      bulk_g2s(sx + st * OZ_GP_ROW, xseg + (r0 + rr) * ldx, (uint32_t)(width * 8), &full[st]);
      bulk_g2s(sx + st * OZ_GP_ROW + 1024, y + (r0 + rr) * ldy, (uint32_t)(m * 8), &full[st]);
    }
  };
  for (int s2 = 0; s2 < OZ_GP_STAGES - 1; ++s2) issue(s2);
  // Column statistics on the entries' high words (sign cleared): their maximum carries the largest exponent
  // (all the exponent code and the range guard use of the maximum; a NaN or infinity gives >= 0x7ff00000),
  // integer exponent sums and nonzero counts (exact: rows * 2047 < 2^31). Integer work instead of FP64
  // compares keeps the FP64 pipe for the X^T Y products.
  double acc[4][MM];
  unsigned mxh[4];
  int se[4], nz[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    mxh[j] = 0u;
    se[j] = nz[j] = 0;
#pragma unroll
    for (int o = 0; o < MM; ++o) acc[j][o] = 0.0;
  }
  for (int64_t rr = 0; rr < nr; ++rr) {
    issue(rr + OZ_GP_STAGES - 1);
    const int st = (int)(rr % OZ_GP_STAGES);
    mbar_wait(&full[st], (uint32_t)((rr / OZ_GP_STAGES) & 1));
    const double* xr = sx + st * OZ_GP_ROW;
    double yv[MM];
#pragma unroll
    for (int o = 0; o < MM; ++o) yv[o] = (o < m) ? xr[1024 + o] : 0.0;  // broadcast shared-memory reads
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (tid + 256 * j < width) {
        const double xv = xr[tid + 256 * j];
        const unsigned hi = (unsigned)__double2hiint(xv) & 0x7fffffffu;
        mxh[j] = max(mxh[j], hi);
        if ((hi | (unsigned)__double2loint(xv)) != 0u) {
          se[j] += (int)(hi >> 20);
          nz[j] += 1;
        }
#pragma unroll
        for (int o = 0; o < MM; ++o) acc[j][o] = fma(xv, yv[o], acc[j][o]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  double mx[4];  // the maximum as a double: +inf for a non-finite entry, else the high word with a zero low word
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    unsigned h = mxh[j] >= 0x7ff00000u ? 0x7ff00000u : mxh[j];
    if (h == 0u && nz[j] > 0) h = 0x00080000u;  // only subnormal entries: 2^-1023 bounds them like their maximum
    mx[j] = __hiloint2double((int)h, 0);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = i0 + 256 * j;
    if (nchunk == 1) {
      if (E != nullptr && i < mp) E[(int64_t)b * mp + i] = i < d ? oz_exp_code(mx[j]) : 0;
      if (guard != nullptr && i < d && oz_out_of_range(mx[j], (double)se[j], (double)nz[j], OZ_RANGE_BITS)) atomicOr(guard, 1);
      if (i < d) {
#pragma unroll
        for (int o = 0; o < MM; ++o)
          if (o < m) C[((int64_t)b * m + o) * d + i] = acc[j][o];
      }
    } else if (i < d) {
      Mp[((int64_t)b * nchunk + ch) * d + i] = mx[j];
      Mp[((int64_t)(gridDim.z + b) * nchunk + ch) * d + i] = (double)se[j];  // exponent sums and nonzero counts
      Mp[((int64_t)(2 * gridDim.z + b) * nchunk + ch) * d + i] = (double)nz[j];  // after the maxima
#pragma unroll
      for (int o = 0; o < MM; ++o)
        if (o < m) Cp[(((int64_t)b * nchunk + ch) * m + o) * d + i] = acc[j][o];
    }
  }
}

__global__ void oz_gram_prep_reduce_kernel(const double* Cp, const double* Mp, int d, int m, int nchunk, int mp,
                                           int* E, double* C, int nblocks, int* guard) {
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= mp) return;
  if (i >= d) {
    if (E != nullptr) E[(int64_t)b * mp + i] = 0;
    return;
  }
  if (E != nullptr) {
    double mx = 0.0;
    double se = 0.0, nz = 0.0;
    for (int c = 0; c < nchunk; ++c) {
      mx = fmax(mx, Mp[((int64_t)b * nchunk + c) * d + i]);
      se += Mp[((int64_t)(nblocks + b) * nchunk + c) * d + i];
      nz += Mp[((int64_t)(2 * nblocks + b) * nchunk + c) * d + i];
    }
    E[(int64_t)b * mp + i] = oz_exp_code(mx);
    if (guard != nullptr && oz_out_of_range(mx, se, nz, OZ_RANGE_BITS)) atomicOr(guard, 1);
  }
  for (int o = 0; o < m; ++o) {
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s += Cp[(((int64_t)b * nchunk + c) * m + o) * d + i];
    C[((int64_t)b * m + o) * d + i] = s;
  }
}

// Slice layout in global memory: the shared-memory image of the tensor-core operands. For every
// (batch b, slice p, K block kc of 32 bytes) the Mpad rows x 32 bytes are contiguous, each row's two
// 16-byte halves swapped where bit 2 of the row is set (the SWIZZLE_32B pattern of the K-major
// canonical layout, 8-row atoms of 256 bytes). A 128-row operand tile of one K block is therefore one
// contiguous 4 KB run that a TMA box copies as whole 128-byte lines; the former [row][kpad] layout with
// 32-byte box rows kept the SM's L2 request port 95% busy (one request per 32-byte sector) and the tensor
// pipe at 78%. Byte offset of row `row` (its physical half 0) in K block kc:
__host__ __device__ __forceinline__ int64_t oz_slice_offset(int b, int p, int row, int64_t kc, int mp, int64_t kpad) {
  return ((((int64_t)b * OZ_S + p) * (kpad / OZ_BK) + kc) * mp + row) * OZ_BK;
}

// 2 KB row of the tensor-map view (oz_tensor_map) where operand row row0 (a multiple of 64) of K block kc starts
RP_DEVINL int oz_box_row(int b, int p, int row0, int kc, int mp, int nkc) {
  return ((b * OZ_S + p) * nkc + kc) * (mp >> 6) + (row0 >> 6);
}

// Digits of 128 (i) x 256 (k) of A, in four 128 x 64 sub-tiles, written K-major in the layout above.
// Columns past K and rows past M give zero digits. Each
// k of a sub-tile is one 1 KB contiguous read of A (consecutive threads on consecutive rows i);
// a thread loads its 16 values of a half sub-tile before converting any (the kernel is bound by
// load latency otherwise).
constexpr int OZ_SLICE_IW = 128;
constexpr size_t OZ_SLICE_SMEM = sizeof(uint32_t) * OZ_S * OZ_SLICE_IW * 17;
__global__ void __launch_bounds__(256) oz_slice_kernel(OzIn in, const int* E, int8_t* slices, int64_t kpad,
                                                       const int* guard) {
  if (guard != nullptr && *guard) return;  // out of range: the FP64 fallback runs instead
  constexpr int IW = OZ_SLICE_IW;
  extern __shared__ uint32_t oz_dig_raw[];  // dig[p][i][k/4], 4 digits per word, padded rows
  uint32_t(*dig)[IW][17] = reinterpret_cast<uint32_t(*)[IW][17]>(oz_dig_raw);
  const int b = blockIdx.z, i0 = blockIdx.y * IW;
  const double* Ab = in.A + (int64_t)b * in.bstride;
  const int mp = in.mpad();
  const int ii = threadIdx.x & (IW - 1), kqb = threadIdx.x / IW;  // kq = kqb + 2 * u
  const int i = i0 + ii;
  const int ei = (i < in.M) ? E[(int64_t)b * mp + i] : OZ_NONFINITE;
  const double scale = ldexp(1.0, 54 - (ei == OZ_NONFINITE ? 0 : ei));  // |x| < 2^ei -> |v| < 2^54
  for (int sub = 0; sub < 4; ++sub) {
    const int64_t k0 = (int64_t)blockIdx.x * 256 + sub * 64;
    if (k0 >= kpad) break;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      double xs[4][4];
      if (!in.tri && ei != OZ_NONFINITE && k0 + 64 <= in.K) {
        // the whole 64-deep sub-tile is inside the matrix: no per-entry predicates, one pointer walked by lda
        const double* pk = Ab + (k0 + (kqb + 8 * half) * 4) * in.lda + i;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int r = 0; r < 4; ++r) xs[u][r] = __ldcs(pk + r * in.lda);
          pk += 8 * in.lda;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int kq = kqb + 2 * (4 * half + u);
            const int64_t k = k0 + kq * 4 + r;
            xs[u][r] =
                (ei != OZ_NONFINITE && k < in.K && (!in.tri || k <= i)) ? __ldcs(Ab + k * in.lda + i) : 0.0;
          }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kq = kqb + 2 * (4 * half + u);
        uint32_t w[OZ_S];
#pragma unroll
        for (int p = 0; p < OZ_S; ++p) w[p] = 0u;
        if (ei != OZ_NONFINITE) {
          uint32_t lo[4], hi[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int64_t k = k0 + kq * 4 + r;
            double x = xs[u][r];
            if (in.tri && k == i) x *= 0.5;  // exact
            const long long v = (long long)(x * scale);  // truncation toward zero, |v| < 2^54
            // balanced base-256 digits: with uu = v + 0x808080808080, the low six bytes of uu are
            // the digits d_1..d_6 (d in [-128, 127]) offset by 128, and uu >> 48 is the top digit
            // d_0 (|d_0| <= 65). Offsets are removed below by flipping each byte's top bit.
            const unsigned long long uu = (unsigned long long)(v + 0x808080808080LL);
            lo[r] = (uint32_t)uu;
            hi[r] = (uint32_t)(uu >> 32);
          }
          // byte k of the four entries' words gathered into one word (digit word w[p], entry r in byte r): a
          // 4 x 4 byte transpose by byte permutes (d_6..d_3 = bytes 0..3 of lo, d_2, d_1, d_0 = bytes 0..2 of hi)
          const uint32_t a01 = __byte_perm(lo[0], lo[1], 0x5140), a23 = __byte_perm(lo[2], lo[3], 0x5140);
          const uint32_t b01 = __byte_perm(lo[0], lo[1], 0x7362), b23 = __byte_perm(lo[2], lo[3], 0x7362);
          const uint32_t c01 = __byte_perm(hi[0], hi[1], 0x5140), c23 = __byte_perm(hi[2], hi[3], 0x5140);
          const uint32_t d01 = __byte_perm(hi[0], hi[1], 0x7362), d23 = __byte_perm(hi[2], hi[3], 0x7362);
          w[6] = __byte_perm(a01, a23, 0x5410);
          w[5] = __byte_perm(a01, a23, 0x7632);
          w[4] = __byte_perm(b01, b23, 0x5410);
          w[3] = __byte_perm(b01, b23, 0x7632);
          w[2] = __byte_perm(c01, c23, 0x5410);
          w[1] = __byte_perm(c01, c23, 0x7632);
          w[0] = __byte_perm(d01, d23, 0x5410);
#pragma unroll
          for (int p = 1; p < OZ_S; ++p) w[p] ^= 0x80808080u;
        }
#pragma unroll
        for (int p = 0; p < OZ_S; ++p) dig[p][ii][kq] = w[p];
      }
    }
    __syncthreads();
    // consecutive threads write consecutive 16-byte chunks of one (slice, K block): 128 rows x 32 bytes
    // = 4 KB contiguous; physical half h of row ri holds K chunk h ^ ((ri >> 2) & 1) (32-byte swizzle)
    for (int it = threadIdx.x; it < OZ_S * IW * 4; it += 256) {
      const int h = it & 1, ri = (it >> 1) & (IW - 1), kcl = (it >> 8) & 1, p = it / (4 * IW);
      const int row = i0 + ri;
      const int c = kcl * 2 + (h ^ ((ri >> 2) & 1));
      const int64_t k = k0 + c * 16;
      if (row >= mp || k >= kpad) continue;
      uint4 v;
      v.x = dig[p][ri][c * 4 + 0];
      v.y = dig[p][ri][c * 4 + 1];
      v.z = dig[p][ri][c * 4 + 2];
      v.w = dig[p][ri][c * 4 + 3];
      *reinterpret_cast<uint4*>(slices + oz_slice_offset(b, p, row, k0 / OZ_BK + kcl, mp, kpad) + h * 16) = v;
    }
    __syncthreads();
  }
}

inline cudaError_t oz_slice_launch(const OzIn& in, const int* E, int8_t* slices, int64_t kpad, const int* guard,
                                   cudaStream_t st) {
  static const cudaError_t attr =
      cudaFuncSetAttribute(oz_slice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OZ_SLICE_SMEM);
  if (attr != cudaSuccess) return attr;
  const int mp = in.mpad();
  oz_slice_kernel<<<dim3((unsigned)((kpad + 255) / 256), (mp + OZ_SLICE_IW - 1) / OZ_SLICE_IW, in.nbatch), 256,
                    OZ_SLICE_SMEM, st>>>(in, E, slices, kpad, guard);
  return cudaSuccess;  // launch errors are picked up by the caller's RP_LAUNCH_CHECK
}

// ------------------------------------------------------------------ tcgen05 helpers

RP_DEVINL uint64_t oz_desc_sw32(uint32_t saddr) {
  // K-major, SWIZZLE_32B canonical layout: 32-byte rows, 8-row groups 256 B apart (SBO),
  // LBO unused (1), version 1 (sm_100), layout type 6 = SWIZZLE_32B
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}

// kind::i8 instruction descriptor: s32 accumulate, signed A and B, both K-major, M = N = 128
constexpr uint32_t OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) |
                              ((uint32_t)(OZ_BM >> 4) << 24);

// All products S_p S_q^T of one K-step whose weight group g = p + q lies in [G0, G0 + OZ_GP), into
// accumulator slab g - G0. G0 is a compile-time constant so the (p, q) list is fully unrolled
// with constant descriptor offsets, and the issuing warp runs converged so the operands stay in
// uniform registers; one elected lane issues each MMA (the issue loop, not the tensor pipe, bounded
// the kernel while one thread rebuilt the descriptors and branched per MMA: c4 Gram 23.4 -> 19.6
// ms). BSL: bytes between consecutive B slices in shared memory. Call with the whole warp.
template <int G0, int BSL, bool PAIR>
RP_DEVINL void oz_issue_kstep(uint32_t tmem, uint64_t da0, uint64_t db0, uint32_t first) {
#pragma unroll
  for (int p = 0; p < OZ_S; ++p)
#pragma unroll
    for (int q = 0; q < OZ_S - p; ++q) {
      if (p + q < G0 || p + q >= G0 + OZ_GP) continue;
      const uint64_t da = da0 + (uint64_t)(p * (OZ_SLICE >> 4));
      const uint64_t db = db0 + (uint64_t)(q * (BSL >> 4));
      const uint32_t acc = (p == 0) ? (first ? 0u : 1u) : 1u;  // p = 0 starts every group of the pass
      const uint32_t d = tmem + (uint32_t)((p + q - G0) * 128);
      if (PAIR)  // issued by the whole (converged) warp: operands stay warp-uniform, one elected lane issues
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
            "l"(da), "l"(db), "r"((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) |
                                  ((uint32_t)(256 >> 4) << 24)),
            "r"(acc));
      else
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
            "l"(da), "l"(db), "r"(OZ_IDESC), "r"(acc));
    }
}

// Whole-warp variants (the MMA issuer warp runs its loop converged; one elected lane commits).
RP_DEVINL void oz_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
RP_DEVINL void oz_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

RP_DEVINL void oz_tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

RP_DEVINL void oz_tma_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

RP_DEVINL void oz_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

RP_DEVINL uint32_t oz_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

RP_DEVINL void oz_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

RP_DEVINL void oz_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

RP_DEVINL void oz_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

struct OzArgs {
  const int* E;      // [nbatch][Mp]
  double* C;         // C_b at C + b * cstride, column-major, leading dimension ldc
  int64_t ldc, cstride;
  int M, per, total_tiles;
  int Mp = 0;        // rows per (batch, slice) of the slice layout (pair kernel: M rounded up to 256)
  const int* guard = nullptr;  // range guard (oz_rowexp / gram prep): nonzero -> the FP64 fallback runs instead
  int subtract;      // 0: C = A A^T, 1: C -= A A^T
  int64_t kpad, kchunk;
};

// ------------------------------------------------------------------ CTA-pair (cta_group::2) SYRK
// A 2-CTA cluster computes a 256 x 128 block (sub-tile rows 2 I2 and 2 I2 + 1, column tile J) with
// tcgen05.mma.cta_group::2 (M = 256, N = 128, K = 32): each CTA stages its own 128 rows of A and
// half (64 rows) of B_J, so per SM the tensor core reads 6 KB of shared memory per 128 x 128 x 32
// product instead of 8 KB and the TMA writes 25% fewer operand bytes -- the single-CTA kernel is
// bound by shared-memory bandwidth, not by L2 (a 4th stage changed nothing). The leader CTA
// (rank 0) issues the MMAs; both CTAs' TMA loads complete on the leader's full barrier
// (.cta_group::2), the MMA commits are multicast to both CTAs' empty / tfull barriers, and both
// CTAs' epilogue warps release the accumulators on the leader's tempty barrier. Each CTA drains
// and stores its own 128 x 128 sub-tile exactly as the single-CTA epilogue does.

constexpr uint32_t OZ_IDESC_PAIR = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) |
                                   ((uint32_t)(256 >> 4) << 24);

RP_DEVINL uint32_t oz_mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

RP_DEVINL void oz_mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAITC_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

RP_DEVINL void oz_mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}

RP_DEVINL void oz_tma_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

RP_DEVINL void oz_mma_pair(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(OZ_IDESC_PAIR), "r"(accumulate));
}

// (whole warp; one elected lane commits)
RP_DEVINL void oz_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

constexpr int OZ_PSLICE_B = 64 * OZ_BK;                     // bytes of one 64 x 32 B-half slice tile
constexpr int OZ_PSTAGE = OZ_S * (OZ_SLICE + OZ_PSLICE_B);  // A (128 rows) and B half (64 rows), all slices
constexpr int OZ_PSTAGES = 4;
constexpr size_t OZ_PSMEM = 1024 + (size_t)OZ_PSTAGES * OZ_PSTAGE + 128;
constexpr size_t OZ_PSMEM_DOT = OZ_PSMEM + 4 * 128 * 8;  // + the hold-out row reduction

// Pair units of one matrix: sub-tile-row pair I2 (rows 2 I2, 2 I2 + 1), column tiles J <= 2 I2 + 1
// (J < mt): 2 I2 + 2 units per full pair row, I2^2 + I2 before row I2.
RP_DEVINL void oz_pair_unit(int lin, int per, int mt, int& b, int& I2, int& J) {
  b = lin / per;
  const int t = lin - b * per;
  int i = (int)((sqrt(4.0 * t + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) <= t) ++i;
  while (i * (i + 1) > t) --i;
  I2 = i;
  J = t - i * (i + 1);
  (void)mt;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(OZ_SYRK_THREADS, 1)
    oz_syrk_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, OzArgs a) {
  extern __shared__ __align__(1024) uint8_t oz_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OZ_PSTAGES * OZ_PSTAGE);
  uint64_t* empty = full + OZ_PSTAGES;
  uint64_t* tfull = empty + OZ_PSTAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = oz_cluster_rank();
  const int nchunks = (int)((a.kpad + a.kchunk - 1) / a.kchunk);
  const int unit0 = blockIdx.x / 2, ustep = gridDim.x / 2;
  const int mt = a.M / OZ_BM;  // sub-tile rows that exist (rows of the padded pair past mt are zero)
  if (a.guard != nullptr && *a.guard) return;  // out of range: both CTAs leave before any cluster barrier

  if (tid == 0) {
    for (int s = 0; s < OZ_PSTAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's arrive + both CTAs' bytes
      mbar_init(&empty[s], 1);  // the leader's MMA commit (multicast)
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 16);  // 8 epilogue warps of each CTA (used on the leader)
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  oz_fence_before();
  __syncthreads();
  oz_cluster_sync();
  oz_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t full_leader = oz_mapa(smem_u32(full), 0);
  const uint32_t tempty_leader = oz_mapa(smem_u32(tempty), 0);

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: own A rows, own half of B) ----------------
    if (lane == 0) {
      int it = 0;
      for (int u = unit0; u < a.total_tiles; u += ustep) {
        int b, I2, J;
        oz_pair_unit(u, a.per, mt, b, I2, J);
        const int rowA = (2 * I2 + (int)rank) * OZ_BM;
        const int rowB = J * OZ_BM + (int)rank * 64;
        const int nkc = (int)(a.kpad / OZ_BK);
        for (int pass = 1; pass >= 0; --pass) {
          const int ns = pass ? OZ_S : OZ_GP;
          for (int64_t k = 0; k < a.kpad; k += OZ_BK, ++it) {
            const int st = it % OZ_PSTAGES;
            oz_mbar_wait_cluster(&empty[st], ((it / OZ_PSTAGES) & 1) ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[st], (uint32_t)(2 * ns * (OZ_SLICE + OZ_PSLICE_B)));
            uint8_t* sa = smem + st * OZ_PSTAGE;
            uint8_t* sb = sa + OZ_S * OZ_SLICE;
            const uint32_t fb = full_leader + (uint32_t)(st * 8);
            for (int p = 0; p < ns; ++p) {
              oz_tma_2d_pair(sa + p * OZ_SLICE, &tmA, 0, oz_box_row(b, p, rowA, (int)(k / OZ_BK), a.Mp, nkc), fb);
              oz_tma_2d_pair(sb + p * OZ_PSLICE_B, &tmB, 0, oz_box_row(b, p, rowB, (int)(k / OZ_BK), a.Mp, nkc), fb);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only; the whole warp runs the loop, one lane issues) ----------------
    if (rank == 0) {
      int it = 0, item = 0;
      for (int u = unit0; u < a.total_tiles; u += ustep) {
        for (int pass = 1; pass >= 0; --pass) {
          const int g0 = pass * OZ_GP;
          for (int ch = 0; ch < nchunks; ++ch, ++item) {
            oz_mbar_wait_cluster(tempty, (item & 1) ^ 1);  // both CTAs have drained the accumulators
            oz_fence_after();
            const int64_t kb = ch * a.kchunk, ke = (kb + a.kchunk < a.kpad) ? kb + a.kchunk : a.kpad;
            for (int64_t k = kb; k < ke; k += OZ_BK, ++it) {
              const int st = it % OZ_PSTAGES;
              oz_mbar_wait_cluster(&full[st], (it / OZ_PSTAGES) & 1);
              oz_fence_after();
              const uint32_t sa = smem_u32(smem + st * OZ_PSTAGE);
              const uint32_t sb = sa + OZ_S * OZ_SLICE;
              const bool first = (k == kb);
              if (g0) {
                oz_issue_kstep<OZ_GP, OZ_PSLICE_B, true>(tmem, oz_desc_sw32(sa), oz_desc_sw32(sb), first);
              } else {
                oz_issue_kstep<0, OZ_PSLICE_B, true>(tmem, oz_desc_sw32(sa), oz_desc_sw32(sb), first);
              }
              oz_commit_pair(&empty[st]);  // frees the stage in both CTAs once the MMAs have read it
            }
            oz_commit_pair(tfull);
          }
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..9 of both CTAs): this CTA's 128-row sub-tile ----------------
    const int quarter = warp & 3;
    const int chalf = (warp - 2) >> 2;
    const int row_in_tile = quarter * 32 + lane;
    const uint32_t tlane = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(chalf * 64);
    int item = 0;
    for (int u = unit0; u < a.total_tiles; u += ustep) {
      int b, I2, J;
      oz_pair_unit(u, a.per, mt, b, I2, J);
      const int I = 2 * I2 + (int)rank;
      const bool valid = I < mt && J <= I;
      const int i = I * OZ_BM + row_in_tile;
      const int* Eb = a.E + (int64_t)b * a.Mp;
      const int ei = valid ? Eb[i] : 0;
      double acc[64];
#pragma unroll
      for (int c = 0; c < 64; ++c) acc[c] = 0.0;
      for (int pass = 1; pass >= 0; --pass) {
        const int g0 = pass * OZ_GP;
        for (int ch = 0; ch < nchunks; ++ch, ++item) {
          oz_mbar_wait_cluster(tfull, item & 1);
          oz_fence_after();
#pragma unroll
          for (int g = OZ_GP - 1; g >= 0; --g) {  // smallest weights first
            if (g0 + g >= OZ_S) continue;
            const double w = ldexp(1.0, -8 * (g0 + g) - 12);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              uint32_t v[16];
              oz_ld16(tlane + (uint32_t)(g * 128 + q4 * 16), v);
#pragma unroll
              for (int c = 0; c < 16; ++c) acc[q4 * 16 + c] = fma((double)(int)v[c], w, acc[q4 * 16 + c]);
            }
          }
          oz_fence_before();
          __syncwarp();
          if (lane == 0) oz_mbar_arrive_remote(tempty_leader);
        }
      }
      if (!valid) continue;  // above the diagonal, or the zero rows past M
      double* dst0 = a.C + (int64_t)b * a.cstride + (int64_t)(J * OZ_BM + chalf * 64) * a.ldc + i;
      const int* Ej = Eb + J * OZ_BM + chalf * 64;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        double old[16];
        if (a.subtract) {
#pragma unroll
          for (int c = 0; c < 16; ++c) old[c] = __ldcg(dst0 + (int64_t)(q4 * 16 + c) * a.ldc);
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int ej = Ej[q4 * 16 + c];
          double v;
          if (ei == OZ_NONFINITE || ej == OZ_NONFINITE) {
            v = __longlong_as_double(0x7ff8000000000000LL);
          } else {
            v = ldexp(acc[q4 * 16 + c], ei + ej);
            if (a.subtract) v = old[c] - v;
          }
          dst0[(int64_t)(q4 * 16 + c) * a.ldc] = v;
        }
      }
    }
  }
  oz_fence_before();
  __syncthreads();
  oz_cluster_sync();  // no CTA deallocates or exits while its peer may still signal it
  oz_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ------------------------------------------------------------------ host side

inline PFN_cuTensorMapEncodeTiled_v12000 oz_encode_fn() { return tensor_map_encoder(); }

// View of the slice area as rows of 2 KB (256 x 8-byte elements; 64 operand rows x 32 bytes of one K
// block): an operand tile is a box of box_rows / 64 consecutive rows, copied unswizzled (the swizzle is
// already in the layout, see oz_slice_offset). Row coordinate of (b, p, kc, row0): oz_box_row().
inline bool oz_tensor_map(CUtensorMap* m, const int8_t* slices, int64_t kpad, int64_t nrows, int box_rows = OZ_BM) {
  auto enc = oz_encode_fn();
  if (!enc) return false;
  const int64_t total = nrows * kpad;  // bytes (nrows = nbatch * S * Mpad, Mpad a multiple of 64)
  cuuint64_t dims[2] = {256, (cuuint64_t)(total / 2048)};
  cuuint64_t strides[1] = {2048};
  cuuint32_t box[2] = {256, (cuuint32_t)(box_rows / 64)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<int8_t*>(slices), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline size_t oz_eb(int M, int nbatch) { return ((size_t)nbatch * M * sizeof(int) + 1023) / 1024 * 1024; }

// Rows of the SYRK slice layout: M rounded up to the 256-row blocks of the CTA-pair kernel.
inline int oz_mp(int M) { return (M + 255) / 256 * 256; }

// Workspace of one tensor-core product: a 1 KB header (the range guard int), the row exponents
// E[b][mp], then the K-major slices.
constexpr size_t OZ_HDR = 1024;
inline int* oz_guard_of(void* work) { return reinterpret_cast<int*>(work); }

inline size_t oz_workspace_bytes(int M, int64_t K, int nbatch) {
  const int mp = oz_mp(M);
  return OZ_HDR + oz_eb(mp, nbatch) + (size_t)nbatch * OZ_S * mp * (size_t)oz_kpad(K);
}

// Shapes the tensor-core path takes: 128-row tiles, int32 TMA coordinates.
inline bool oz_supported(int M, int64_t K, int nbatch) {
  // (2 KB rows of the slice view)
  return M % OZ_BM == 0 && (int64_t)nbatch * OZ_S * (oz_mp(M) / 64) * (oz_kpad(K) / OZ_BK) < 0x7fffffff &&
         oz_encode_fn() != nullptr;
}

// Exponents (+ range guard with the given bit budget) and K-major slices of a batch of column-major matrices (rows padded
// to in.mpad()). The guard must have been cleared by the caller.
inline int oz_prepare(const OzIn& in, int* E, int8_t* slices, int64_t kpad, int* guard, int range_bits,
                      cudaStream_t st, int* row_mask = nullptr, int mask_tiles = 0) {
  const int mp = in.mpad();
  oz_rowexp_kernel<<<dim3((mp + 31) / 32, in.nbatch), 256, 0, st>>>(in, E, guard, range_bits, row_mask,
                                                                     mask_tiles);
  RP_LAUNCH_CHECK("ozaki rowexp");
  cudaError_t e = oz_slice_launch(in, E, slices, kpad, guard, st);
  if (e != cudaSuccess) return cuda_status(e, "ozaki slice attributes");
  RP_LAUNCH_CHECK("ozaki slice");
  return RP_OK;
}

// C_b (lower 128 x 128 tiles, each complete) = / -= A_b A_b^T for nbatch column-major M x K A_b,
// on 2-CTA clusters. exps_ready: the row exponents and the range guard are already in the
// workspace (oz_gram_prep_kernel), so only the slicing pass runs; otherwise the guard is cleared
// and set here. When the guard is set every kernel of this call exits at once: the caller
// launches the gated FP64 fallback (GemmArgs::run_if_set = oz_guard_of(work)) behind it.
inline int oz_syrk(const OzIn& in, double* C, int64_t ldc, int64_t cstride, bool subtract, void* work,
                   cudaStream_t st, const char* prof_name = "oz_syrk", bool exps_ready = false) {
  OzIn pin = in;
  pin.Mpad = oz_mp(in.M);
  const int mp = pin.Mpad;
  int* guard = oz_guard_of(work);
  int* E = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(work) + OZ_HDR);
  int8_t* slices = reinterpret_cast<int8_t*>(work) + OZ_HDR + oz_eb(mp, in.nbatch);
  const int64_t kpad = oz_kpad(in.K);
  {
    ProfScope prof("oz_prep", st);
    if (exps_ready) {
      cudaError_t e = oz_slice_launch(pin, E, slices, kpad, guard, st);
      if (e != cudaSuccess) return cuda_status(e, "ozaki slice attributes");
      RP_LAUNCH_CHECK("ozaki slice");
    } else {
      cudaError_t e = cudaMemsetAsync(guard, 0, sizeof(int), st);
      if (e != cudaSuccess) return cuda_status(e, "ozaki guard");
      int rc = oz_prepare(pin, E, slices, kpad, guard, OZ_RANGE_BITS, st);
      if (rc) return rc;
    }
  }
  CUtensorMap tm, tmB;
  if (!oz_tensor_map(&tm, slices, kpad, (int64_t)in.nbatch * OZ_S * mp) ||
      !oz_tensor_map(&tmB, slices, kpad, (int64_t)in.nbatch * OZ_S * mp, 64))
    return set_error(RP_ECUDA, "ozaki: cuTensorMapEncodeTiled failed");
  OzArgs a;
  a.E = E;
  a.C = C;
  a.ldc = ldc;
  a.cstride = cstride;
  a.M = in.M;
  a.Mp = mp;
  a.guard = guard;
  const int mt = in.M / OZ_BM;
  a.subtract = subtract ? 1 : 0;
  a.kpad = kpad;
  a.kchunk = oz_kchunk(kpad);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  a.per = 0;
  for (int i2 = 0; i2 < (mt + 1) / 2; ++i2) a.per += (2 * i2 + 2 < mt ? 2 * i2 + 2 : mt);
  a.total_tiles = a.per * in.nbatch;  // pair units
  cudaFuncSetAttribute(oz_syrk_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OZ_PSMEM);
  int pairs = sms / 2;
  if (pairs > a.total_tiles) pairs = a.total_tiles;
  {
    ProfScope prof(prof_name, st);
    oz_syrk_pair_kernel<<<2 * pairs, OZ_SYRK_THREADS, OZ_PSMEM, st>>>(tm, tmB, a);
  }
  RP_LAUNCH_CHECK("ozaki syrk (CTA pairs)");
  return RP_OK;
}

// ------------------------------------------------------------------ Gram-form hold-out
// quad[b][n] = w_n^T T_b w_n with T_b = strict_lower(G_b) + diag(G_b)/2 (so w^T G w = 2 quad),
// for the q*m solution columns w_n of W_b (row-major d x ldw). One 128 x 128 tile (I, J) of
// T_b W_b at a time, K = rows k < 128(I+1) only (T is lower triangular); A = slices of T_b
// (shared by all b when the batch stride of G is 0), B = slices of W_b^T. The epilogue scales
// the tile to FP64, multiplies by W_b(i, n), reduces over the 128 rows (warp reduce-scatter,
// then the 4 row quarters through shared memory) and writes one partial per tile row:
// part[b][I][n], summed in a fixed order by the finish kernel. As in the SYRK, 8 epilogue warps
// drain both passes of a tile into FP64 registers and release TMEM before the reduction.
struct OzDotArgs {
  const int* EA;  // [nA][MpadA]
  const int* EB;  // [nbatch][MpadB]
  const double* W;
  int64_t ldw, w_stride;
  double* part;
  const int* guard;  // range guard: nonzero -> exit (the FP64 fallback runs)
  int d, N, MpadA, MpadB, mtA, ntB, nbatch, a_shared, total_tiles;
  int64_t kpad;
};

// CTA-pair hold-out kernel: a 2-CTA cluster computes sub-tile rows 2 I2
// and 2 I2 + 1 of T_b against the 128 columns J of W_b^T with tcgen05.mma.cta_group::2 (M = 256,
// N = 128); each CTA stages its own 128 rows of T and 64 of the 128 W^T rows (the barrier
// protocol of oz_syrk_pair_kernel). K runs to 128 (2 I2 + 2) for both rows of the pair (T is
// lower triangular, so the even row's extra K block multiplies zeros). Each CTA reduces its own
// sub-tile row into part[b][I][n].
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(OZ_SYRK_THREADS, 1)
    oz_dotb_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        OzDotArgs a) {
  extern __shared__ __align__(1024) uint8_t oz_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OZ_PSTAGES * OZ_PSTAGE);
  uint64_t* empty = full + OZ_PSTAGES;
  uint64_t* tfull = empty + OZ_PSTAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  double* red = reinterpret_cast<double*>(smem + OZ_PSTAGES * OZ_PSTAGE + 128);  // [4][128]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = oz_cluster_rank();
  const int mt2 = (a.mtA + 1) / 2;
  const int per_I = a.nbatch * a.ntB;
  auto decode = [&](int unit, int& b, int& I2, int& J) {  // heaviest (largest I2) first
    const int r = unit / per_I, rem = unit - r * per_I;
    I2 = mt2 - 1 - r;
    b = rem / a.ntB;
    J = rem - b * a.ntB;
  };
  auto ksteps = [&](int I2) {
    const int64_t ke = (int64_t)(2 * I2 + 2) * OZ_BM < a.kpad ? (int64_t)(2 * I2 + 2) * OZ_BM : a.kpad;
    return (int)(ke / OZ_BK);
  };
  const int unit0 = blockIdx.x / 2, ustep = gridDim.x / 2;
  if (a.guard != nullptr && *a.guard) return;  // out of range: both CTAs leave before any cluster barrier

  if (tid == 0) {
    for (int s = 0; s < OZ_PSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 16);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  oz_fence_before();
  __syncthreads();
  oz_cluster_sync();
  oz_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t full_leader = oz_mapa(smem_u32(full), 0);
  const uint32_t tempty_leader = oz_mapa(smem_u32(tempty), 0);

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int u = unit0; u < a.total_tiles; u += ustep) {
        int b, I2, J;
        decode(u, b, I2, J);
        const int ba = a.a_shared ? 0 : b;
        const int rowA = (2 * I2 + (int)rank) * OZ_BM;
        const int rowB = J * OZ_BM + (int)rank * 64;
        const int nkc = (int)(a.kpad / OZ_BK);
        const int nk = ksteps(I2);
        for (int pass = 1; pass >= 0; --pass) {
          const int ns = pass ? OZ_S : OZ_GP;
          for (int kk = 0; kk < nk; ++kk, ++it) {
            const int st = it % OZ_PSTAGES;
            oz_mbar_wait_cluster(&empty[st], ((it / OZ_PSTAGES) & 1) ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[st], (uint32_t)(2 * ns * (OZ_SLICE + OZ_PSLICE_B)));
            uint8_t* sa = smem + st * OZ_PSTAGE;
            uint8_t* sb = sa + OZ_S * OZ_SLICE;
            const uint32_t fb = full_leader + (uint32_t)(st * 8);
            for (int p = 0; p < ns; ++p) {
              oz_tma_2d_pair(sa + p * OZ_SLICE, &tmA, 0, oz_box_row(ba, p, rowA, kk, a.MpadA, nkc), fb);
              oz_tma_2d_pair(sb + p * OZ_PSLICE_B, &tmB, 0, oz_box_row(b, p, rowB, kk, a.MpadB, nkc), fb);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // the whole warp runs the loop, one elected lane issues
      int it = 0, item = 0;
      for (int u = unit0; u < a.total_tiles; u += ustep) {
        int b, I2, J;
        decode(u, b, I2, J);
        const int nk = ksteps(I2);
        for (int pass = 1; pass >= 0; --pass, ++item) {
          oz_mbar_wait_cluster(tempty, (item & 1) ^ 1);
          oz_fence_after();
          for (int kk = 0; kk < nk; ++kk, ++it) {
            const int st = it % OZ_PSTAGES;
            oz_mbar_wait_cluster(&full[st], (it / OZ_PSTAGES) & 1);
            oz_fence_after();
            const uint32_t sa = smem_u32(smem + st * OZ_PSTAGE);
            const uint32_t sb = sa + OZ_S * OZ_SLICE;
            if (pass)
              oz_issue_kstep<OZ_GP, OZ_PSLICE_B, true>(tmem, oz_desc_sw32(sa), oz_desc_sw32(sb), kk == 0);
            else
              oz_issue_kstep<0, OZ_PSLICE_B, true>(tmem, oz_desc_sw32(sa), oz_desc_sw32(sb), kk == 0);
            oz_commit_pair(&empty[st]);
          }
          oz_commit_pair(tfull);
        }
      }
    }
  } else {
    const int quarter = warp & 3, chalf = (warp - 2) >> 2;
    const int row_in_tile = quarter * 32 + lane;
    const uint32_t tlane = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(chalf * 64);
    int item = 0;
    for (int u = unit0; u < a.total_tiles; u += ustep) {
      int b, I2, J;
      decode(u, b, I2, J);
      const int I = 2 * I2 + (int)rank;
      const bool valid = I < a.mtA;
      const int ba = a.a_shared ? 0 : b;
      const int i = I * OZ_BM + row_in_tile;
      const int ei = a.EA[(int64_t)ba * a.MpadA + i];
      const int* EBb = a.EB + (int64_t)b * a.MpadB;
      const double* Wrow = a.W + (int64_t)b * a.w_stride + (int64_t)i * a.ldw;
      double acc[64];
#pragma unroll
      for (int c = 0; c < 64; ++c) acc[c] = 0.0;
      for (int pass = 1; pass >= 0; --pass, ++item) {
        const int g0 = pass * OZ_GP;
        oz_mbar_wait_cluster(tfull, item & 1);
        oz_fence_after();
#pragma unroll
        for (int g = OZ_GP - 1; g >= 0; --g) {
          if (g0 + g >= OZ_S) continue;
          const double w = ldexp(1.0, -8 * (g0 + g) - 12);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t t[16];
            oz_ld16(tlane + (uint32_t)(g * 128 + q4 * 16), t);
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[q4 * 16 + c] = fma((double)(int)t[c], w, acc[q4 * 16 + c]);
          }
        }
        oz_fence_before();
        __syncwarp();
        if (lane == 0) oz_mbar_arrive_remote(tempty_leader);
      }
      const int n0 = J * OZ_BM + chalf * 64;
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        const int n = n0 + c;
        double x = 0.0;
        if (valid && i < a.d && n < a.N) {
          const int en = EBb[n];
          x = (ei == OZ_NONFINITE || en == OZ_NONFINITE) ? __longlong_as_double(0x7ff8000000000000LL)
                                                          : ldexp(acc[c], ei + en) * Wrow[n];
        }
        acc[c] = x;
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
        for (int s2 = 16; s2 >= 1; s2 >>= 1) {
          const bool upper = (lane & s2) != 0;
#pragma unroll
          for (int j = 0; j < s2; ++j) {
            const double send = upper ? acc[hh * 32 + j] : acc[hh * 32 + j + s2];
            const double keep = upper ? acc[hh * 32 + j + s2] : acc[hh * 32 + j];
            acc[hh * 32 + j] = keep + __shfl_xor_sync(0xffffffffu, send, s2);
          }
        }
        red[quarter * 128 + chalf * 64 + hh * 32 + lane] = acc[hh * 32];
      }
      named_bar_sync(1, 256);
      if (quarter == 0 && valid) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int col = chalf * 64 + hh * 32 + lane;
          const double tot = red[col] + red[128 + col] + red[256 + col] + red[384 + col];
          const int n = J * OZ_BM + col;
          if (n < a.N) a.part[((int64_t)b * a.mtA + I) * a.N + n] = tot;
        }
      }
      named_bar_sync(1, 256);
    }
  }
  oz_fence_before();
  __syncthreads();
  oz_cluster_sync();
  oz_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

inline int64_t oz_rup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Workspace of oz_holdout: guard header, exponents and slices of T (nA copies) and of W^T (nbatch).
inline size_t oz_holdout_workspace(int d, int64_t N, int nbatch, bool a_shared) {
  const int64_t mpa = oz_rup(d, 256), mpb = oz_rup(N, OZ_BM), kpad = oz_kpad(d);
  const int na = a_shared ? 1 : nbatch;
  return OZ_HDR + (size_t)oz_rup((int64_t)na * mpa * 4, 1024) + (size_t)oz_rup((int64_t)nbatch * mpb * 4, 1024) +
         (size_t)na * OZ_S * mpa * kpad + (size_t)nbatch * OZ_S * mpb * kpad;
}

inline bool oz_holdout_supported(int d, int64_t N, int nbatch) {
  const int64_t mpa = oz_rup(d, 256), mpb = oz_rup(N, OZ_BM);
  return oz_kpad(d) <= oz_kchunk(oz_kpad(d)) &&
         (int64_t)nbatch * OZ_S * ((mpa > mpb ? mpa : mpb) / 64) * (oz_kpad(d) / OZ_BK) < 0x7fffffff &&
         oz_encode_fn() != nullptr;
}

// part[b][I][n]: partials of w_n^T T_b w_n (sum over the ceil(d/128) entries). The range guard
// covers both operands: a row of T out of range trips it (the kernels exit and the caller's gated
// FP64 fallback runs, as oz_syrk); a row of W^T (one solution vector) out of range only marks its
// 128-column tile in col_mask (zeroed here; nbatch x ceil(N / 128) ints), and the caller's gated
// FP64 product then recomputes just the marked tiles' partials after this kernel.
// side / fork / join (optional): T's exponents and slices are prepared on the side stream beside W's on st
// (two latency-bound passes, ~2 TB/s each alone); st waits for both before the product.
inline int oz_holdout(const double* G, int64_t g_stride, int d, const double* W, int64_t ldw, int64_t w_stride,
                      int64_t N, int nbatch, double* part, void* work, int* col_mask, cudaStream_t st,
                      cudaStream_t side = nullptr, cudaEvent_t fork = nullptr, cudaEvent_t join = nullptr) {
  const bool shared = g_stride == 0;
  const int64_t mpa = oz_rup(d, 256), mpb = oz_rup(N, OZ_BM), kpad = oz_kpad(d);
  const int na = shared ? 1 : nbatch;
  int* guard = oz_guard_of(work);
  uint8_t* w8 = reinterpret_cast<uint8_t*>(work) + OZ_HDR;
  int* EA = reinterpret_cast<int*>(w8);
  w8 += oz_rup((int64_t)na * mpa * 4, 1024);
  int* EB = reinterpret_cast<int*>(w8);
  w8 += oz_rup((int64_t)nbatch * mpb * 4, 1024);
  int8_t* SA = reinterpret_cast<int8_t*>(w8);
  int8_t* SB = SA + (size_t)na * OZ_S * mpa * kpad;
  OzIn ia{G, d, g_stride, d, d, na};
  ia.Mpad = (int)mpa;
  ia.tri = 1;
  OzIn ib{W, ldw, w_stride, d, (int)N, nbatch};  // W_b^T: row n, column k at W + k*ldw + n
  ib.Mpad = (int)mpb;
  const int mask_tiles = (int)((N + 127) / 128);
  cudaError_t e = cudaMemsetAsync(guard, 0, sizeof(int), st);
  if (e == cudaSuccess && col_mask != nullptr)
    e = cudaMemsetAsync(col_mask, 0, sizeof(int) * (size_t)nbatch * mask_tiles, st);
  if (e != cudaSuccess) return cuda_status(e, "ozaki guard");
  const bool two = side != nullptr && fork != nullptr && join != nullptr;
  if (two) {  // the guard and mask are cleared before either preparation starts
    e = cudaEventRecord(fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, fork, 0);
    if (e != cudaSuccess) return cuda_status(e, "ozaki holdout fork");
  }
  int rc = oz_prepare(ia, EA, SA, kpad, guard, OZ_RANGE_BITS_DOT, two ? side : st);
  if (rc) return rc;
  rc = oz_prepare(ib, EB, SB, kpad, guard, OZ_RANGE_BITS_DOT, st, col_mask, mask_tiles);
  if (rc) return rc;
  if (two) {
    e = cudaEventRecord(join, side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, join, 0);
    if (e != cudaSuccess) return cuda_status(e, "ozaki holdout join");
  }
  CUtensorMap ta, tb;
  if (!oz_tensor_map(&ta, SA, kpad, (int64_t)na * OZ_S * mpa) ||
      !oz_tensor_map(&tb, SB, kpad, (int64_t)nbatch * OZ_S * mpb, 64))
    return set_error(RP_ECUDA, "ozaki: cuTensorMapEncodeTiled failed");
  OzDotArgs a;
  a.EA = EA;
  a.EB = EB;
  a.W = W;
  a.ldw = ldw;
  a.w_stride = w_stride;
  a.part = part;
  a.guard = guard;
  a.d = d;
  a.N = (int)N;
  a.MpadA = (int)mpa;
  a.MpadB = (int)mpb;
  a.mtA = (int)(oz_rup(d, OZ_BM) / OZ_BM);
  a.ntB = (int)(mpb / OZ_BM);
  a.nbatch = nbatch;
  a.a_shared = shared ? 1 : 0;
  a.total_tiles = (a.mtA + 1) / 2 * a.ntB * nbatch;
  a.kpad = kpad;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int pairs = sms / 2;
  if (pairs > a.total_tiles) pairs = a.total_tiles;
  cudaFuncSetAttribute(oz_dotb_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OZ_PSMEM_DOT);
  {
    ProfScope prof("oz_holdout", st);
    oz_dotb_pair_kernel<<<2 * pairs, OZ_SYRK_THREADS, OZ_PSMEM_DOT, st>>>(ta, tb, a);
  }
  RP_LAUNCH_CHECK("ozaki holdout");
  return RP_OK;
}

}  // namespace rp
