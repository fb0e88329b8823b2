// FP64 Gram blocks on the 5th-generation tensor cores (tcgen05, kind::i8) by the Ozaki scheme.
//
// sm_100a has no FP64 tcgen05 MMA: the FP64 path (mma.sync DMMA) peaks at 37 TFLOP/s, while the
// int8 tensor cores run at ~4.5 POPS. G_b = X_b^T X_b is computed exactly in integer arithmetic
// on fixed-point slices of X_b and recombined in FP64:
//
//   per column i of the block:  x_ki = 2^E_i * sum_{p<S} d_p(k,i) 2^{-7(p+1)},  d_p in [-127,127]
//   (E_i = exponent of max_k |x_ki|, |x| / 2^E_i < 1 written as S signed 7-bit digits, the tail
//   below 2^{E_i - 7S} truncated), so
//
//   G_ij = 2^{E_i+E_j} sum_{g<S} 2^{-7(g+2)} C_g(i,j),   C_g = sum_{p+q=g} S_p S_q^T  (int32, exact)
//
// with the products of weight below 2^{-7(S+1)} dropped (the same order as the digit truncation).
// Relative to FP64 (u = 2^-53) the result carries an error of about S * 2^{-7S} relative to
// max|x_i| max|x_j| per term: ~1e-15 for S = 7 on Gaussian-like columns.
//
// Kernels:
//   oz_colexp_kernel   E[b][i]                    (one pass over X, column max)
//   oz_slice_kernel    digits, transposed to K-major int8 slices [b][p][i][Kpad]
//   oz_gram_kernel     persistent, warp-specialised: warp 0 issues the TMA loads (SWIZZLE_32B
//                      boxes of 32 k x 128/64 rows, all S slices of A and B per stage), warp 1
//                      allocates TMEM and issues the S(S+1)/2 tcgen05.mma per k-step into S
//                      accumulators of 128 x 64 int32 (one TMEM column block per weight g),
//                      warps 2-5 read TMEM (tcgen05.ld), recombine in FP64 and store the tile.
// K is processed in chunks short enough that no int32 accumulator can overflow
// (S pairs x 127^2 x K_chunk < 2^31); the epilogue carries the FP64 sum across chunks.
#pragma once
#include <cuda.h>

#include "rp_common.cuh"

namespace rp {

constexpr int OZ_BM = 128, OZ_BN = 64, OZ_BK = 32, OZ_STAGES = 4;
constexpr int OZ_SLICES = 8;  // 56-bit fixed point: FP64-level Gram accuracy (7 slices: ~1e-13)
constexpr int OZ_THREADS = 192;  // producer, MMA, 4 epilogue warps

template <int S>
struct OzSmem {
  static constexpr int A_SLICE = OZ_BM * OZ_BK;  // bytes per slice tile
  static constexpr int B_SLICE = OZ_BN * OZ_BK;
  static constexpr int STAGE = S * (A_SLICE + B_SLICE);
  static constexpr size_t BYTES = 1024 + (size_t)OZ_STAGES * STAGE + 256;  // + alignment slack, barriers
};

inline int64_t oz_kpad(int64_t rows) { return (rows + 63) / 64 * 64; }

// K-chunk such that S ordered pairs of int8 products never overflow an int32 accumulator.
inline int64_t oz_kchunk(int S, int64_t kpad) {
  int64_t c = (2147483647LL / ((int64_t)S * 127 * 127)) / OZ_BK * OZ_BK;
  return c < kpad ? c : kpad;
}

// ------------------------------------------------------------------ preprocessing

// Column exponent marking a column with a NaN or infinity: the Gram entries it touches are NaN,
// as they would be in FP64 arithmetic.
constexpr int OZ_NONFINITE = 0x7fffffff;

// E[b][i]: exponent with max_k |x_ki| < 2^E (0 for an all-zero column, OZ_NONFINITE if any entry
// is NaN or infinite).
__global__ void oz_colexp_kernel(const double* X, int64_t ldx, int64_t rows, int d, int* E) {
  const int b = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d) return;
  const double* x = X + (int64_t)b * rows * ldx + i;
  double mx = 0.0;
  bool finite = true;
#pragma unroll 8
  for (int64_t k = 0; k < rows; ++k) {
    const double v = fabs(__ldcs(x + k * ldx));
    finite &= (v <= 1.79769313486231570e308);  // false for NaN and inf
    mx = fmax(mx, v);
  }
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);
  E[(int64_t)b * d + i] = finite ? e : OZ_NONFINITE;
}

// Digits of a 64 (k) x 64 (i) tile of block b, written K-major: slices[((b*S + p)*d + i)*kpad + k].
// Rows past the block (k >= rows) and columns past d give zero digits.
template <int S>
__global__ void __launch_bounds__(256) oz_slice_kernel(const double* X, int64_t ldx, int64_t rows, int d,
                                                       const int* E, int8_t* slices, int64_t kpad) {
  __shared__ uint32_t dig[S][64][17];  // [p][i][k/4], 4 digits per word, padded rows
  const int b = blockIdx.z, i0 = blockIdx.y * 64;
  const int64_t k0 = (int64_t)blockIdx.x * 64;
  const double* Xb = X + (int64_t)b * rows * ldx;
  for (int it = threadIdx.x; it < 64 * 16; it += 256) {
    const int ii = it & 63, kq = it >> 6;  // consecutive threads: consecutive columns
    const int i = i0 + ii;
    uint32_t w[S];
#pragma unroll
    for (int p = 0; p < S; ++p) w[p] = 0u;
    const int ei = (i < d) ? E[(int64_t)b * d + i] : OZ_NONFINITE;
    if (ei != OZ_NONFINITE) {
      const double scale = ldexp(1.0, 7 * S - ei);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t k = k0 + kq * 4 + r;
        const double x = (k < rows) ? Xb[k * ldx + i] : 0.0;
        const unsigned long long u = (unsigned long long)(fabs(x) * scale);  // truncation, < 2^{7S}
        const bool neg = x < 0.0;
#pragma unroll
        for (int p = 0; p < S; ++p) {
          int dv = (int)((u >> (7 * (S - 1 - p))) & 127ull);
          if (neg) dv = -dv;
          w[p] |= ((uint32_t)(dv & 0xff)) << (8 * r);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < S; ++p) dig[p][ii][kq] = w[p];
  }
  __syncthreads();
  for (int it = threadIdx.x; it < S * 64 * 4; it += 256) {
    const int c = it & 3, ii = (it >> 2) & 63, p = it >> 8;
    const int i = i0 + ii;
    const int64_t k = k0 + c * 16;
    if (i >= d || k >= kpad) continue;
    uint4 v;
    v.x = dig[p][ii][c * 4 + 0];
    v.y = dig[p][ii][c * 4 + 1];
    v.z = dig[p][ii][c * 4 + 2];
    v.w = dig[p][ii][c * 4 + 3];
    *reinterpret_cast<uint4*>(slices + (((int64_t)b * S + p) * d + i) * kpad + k) = v;
  }
}

// ------------------------------------------------------------------ tcgen05 helpers

RP_DEVINL uint64_t oz_desc_sw32(uint32_t saddr) {
  // K-major, SWIZZLE_32B canonical layout: 32-byte rows, 8-row groups 256 B apart (SBO),
  // LBO unused (1), version 1 (sm_100), layout type 6 = SWIZZLE_32B
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}

// kind::i8 instruction descriptor: s32 accumulate, signed A and B, both K-major, M=128, N=64
constexpr uint32_t OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
                              ((uint32_t)(OZ_BM >> 4) << 24);

RP_DEVINL void oz_mma(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(OZ_IDESC), "r"(accumulate));
}

RP_DEVINL void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

RP_DEVINL void oz_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
RP_DEVINL void oz_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

RP_DEVINL void oz_tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
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

// Lower tiles (I, J) of one block: 128-row tile I, 64-column tile J <= 2I + 1 (I(I+1) before row I).
RP_DEVINL void oz_tile(int lin, int per_block, int& b, int& I, int& J) {
  b = lin / per_block;
  const int t = lin - b * per_block;
  int i = (int)((sqrt(4.0 * t + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) <= t) ++i;
  while (i * (i + 1) > t) --i;
  I = i;
  J = t - i * (i + 1);
}

struct OzArgs {
  const int* E;      // [nblocks][d]
  double* G;         // [nblocks][d][d] column-major (lower tiles written, tiles complete)
  int d, nblocks, per_block, total_tiles;
  int64_t kpad, kchunk;
};

template <int S>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    oz_gram_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, OzArgs a) {
  using SM = OzSmem<S>;
  extern __shared__ __align__(1024) uint8_t oz_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OZ_STAGES * SM::STAGE);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* tfull = empty + OZ_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nchunks = (int)((a.kpad + a.kchunk - 1) / a.kchunk);

  if (tid == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  oz_fence_before();
  __syncthreads();
  oz_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
        int b, I, J;
        oz_tile(tile, a.per_block, b, I, J);
        const int rowA = b * S * a.d + I * OZ_BM, rowB = b * S * a.d + J * OZ_BN;
        for (int64_t k = 0; k < a.kpad; k += OZ_BK, ++it) {
          const int st = it % OZ_STAGES;
          mbar_wait(&empty[st], ((it / OZ_STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], (uint32_t)SM::STAGE);
          uint8_t* sa = smem + st * SM::STAGE;
          uint8_t* sb = sa + S * SM::A_SLICE;
#pragma unroll
          for (int p = 0; p < S; ++p) {
            oz_tma_2d(sa + p * SM::A_SLICE, &tmA, (int)k, rowA + p * a.d, &full[st]);
            oz_tma_2d(sb + p * SM::B_SLICE, &tmB, (int)k, rowB + p * a.d, &full[st]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int it = 0, item = 0;
      for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
        for (int ch = 0; ch < nchunks; ++ch, ++item) {
          mbar_wait(tempty, (item & 1) ^ 1);  // epilogue has drained the accumulators
          oz_fence_after();
          const int64_t kb = ch * a.kchunk, ke = (kb + a.kchunk < a.kpad) ? kb + a.kchunk : a.kpad;
          for (int64_t k = kb; k < ke; k += OZ_BK, ++it) {
            const int st = it % OZ_STAGES;
            mbar_wait(&full[st], (it / OZ_STAGES) & 1);
            oz_fence_after();
            const uint32_t sa = smem_u32(smem + st * SM::STAGE);
            const uint32_t sb = sa + S * SM::A_SLICE;
            const uint32_t first = (k == kb) ? 1u : 0u;
#pragma unroll
            for (int p = 0; p < S; ++p)
#pragma unroll
              for (int q = 0; q < S - p; ++q)
                // p = 0 writes every weight group first: it starts the group on a chunk's first step
                oz_mma(tmem + (uint32_t)((p + q) * OZ_BN), oz_desc_sw32(sa + p * SM::A_SLICE),
                       oz_desc_sw32(sb + q * SM::B_SLICE), (first && p == 0) ? 0u : 1u);
            oz_commit(&empty[st]);  // frees the stage once these MMAs have read it
          }
          oz_commit(tfull);
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5: TMEM lane quarter = warp % 4) ----------------
    const int quarter = warp & 3;
    const int row_in_tile = quarter * 32 + lane;
    int item = 0;
    for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
      int b, I, J;
      oz_tile(tile, a.per_block, b, I, J);
      double acc[OZ_BN];
#pragma unroll
      for (int c = 0; c < OZ_BN; ++c) acc[c] = 0.0;
      for (int ch = 0; ch < nchunks; ++ch, ++item) {
        mbar_wait(tfull, item & 1);
        oz_fence_after();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double part[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) part[c] = 0.0;
#pragma unroll 1
          for (int g = S - 1; g >= 0; --g) {  // smallest weights first
            uint32_t v[32];
            oz_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(g * OZ_BN + h * 32), v);
            const double w = ldexp(1.0, -7 * (g + 2));
#pragma unroll
            for (int c = 0; c < 32; ++c) part[c] = fma((double)(int)v[c], w, part[c]);
          }
#pragma unroll
          for (int c = 0; c < 32; ++c) acc[h * 32 + c] += part[c];
        }
        oz_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
      }
      const int i = I * OZ_BM + row_in_tile;
      if (i < a.d) {
        const int ei = a.E[(int64_t)b * a.d + i];
        double* Gb = a.G + (int64_t)b * a.d * a.d;
#pragma unroll
        for (int c = 0; c < OZ_BN; ++c) {
          const int j = J * OZ_BN + c;
          if (j < a.d) {
            const int ej = a.E[(int64_t)b * a.d + j];
            Gb[(int64_t)j * a.d + i] =
                (ei == OZ_NONFINITE || ej == OZ_NONFINITE) ? __longlong_as_double(0x7ff8000000000000LL)
                                                           : ldexp(acc[c], ei + ej);
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

}  // namespace rp

// ------------------------------------------------------------------ host side
#include <cudaTypedefs.h>

namespace rp {

inline PFN_cuTensorMapEncodeTiled_v12000 oz_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D int8 view of the slices: inner dim kpad bytes, outer nblocks*S*d rows; SWIZZLE_32B boxes.
inline bool oz_tensor_map(CUtensorMap* m, const int8_t* slices, int64_t kpad, int64_t nrows, int box_rows) {
  auto enc = oz_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)kpad, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {(cuuint64_t)kpad};
  cuuint32_t box[2] = {(cuuint32_t)OZ_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(slices), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline size_t oz_workspace_bytes(int S, int d, int64_t rows, int nblocks) {
  const size_t e = ((size_t)nblocks * d * sizeof(int) + 1023) / 1024 * 1024;
  return e + (size_t)nblocks * S * d * (size_t)oz_kpad(rows);
}

// G[b] = X_b^T X_b (all tiles with J <= 2I+1, i.e. the lower triangle and the diagonal-straddling
// tiles, each complete) for nblocks row blocks of `rows` rows. d % 128 == 0. Returns RP_OK or an error.
template <int S>
inline int oz_gram(const double* X, int64_t ldx, int64_t rows, int nblocks, int d, double* G, void* work,
                   cudaStream_t st) {
  int* E = reinterpret_cast<int*>(work);
  const size_t eb = ((size_t)nblocks * d * sizeof(int) + 1023) / 1024 * 1024;
  int8_t* slices = reinterpret_cast<int8_t*>(work) + eb;
  const int64_t kpad = oz_kpad(rows);
  oz_colexp_kernel<<<dim3((d + 255) / 256, nblocks), 256, 0, st>>>(X, ldx, rows, d, E);
  RP_LAUNCH_CHECK("ozaki colexp");
  oz_slice_kernel<S><<<dim3((unsigned)(kpad / 64), (d + 63) / 64, nblocks), 256, 0, st>>>(X, ldx, rows, d, E, slices,
                                                                                          kpad);
  RP_LAUNCH_CHECK("ozaki slice");
  CUtensorMap ta, tb;
  const int64_t nrows = (int64_t)nblocks * S * d;
  if (!oz_tensor_map(&ta, slices, kpad, nrows, OZ_BM) || !oz_tensor_map(&tb, slices, kpad, nrows, OZ_BN))
    return set_error(RP_ECUDA, "ozaki: cuTensorMapEncodeTiled failed");
  OzArgs a;
  a.E = E;
  a.G = G;
  a.d = d;
  a.nblocks = nblocks;
  const int mt = d / OZ_BM;
  a.per_block = mt * (mt + 1);
  a.total_tiles = a.per_block * nblocks;
  a.kpad = kpad;
  a.kchunk = oz_kchunk(S, kpad);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.total_tiles < sms ? a.total_tiles : sms;
  const size_t smem = OzSmem<S>::BYTES;
  cudaFuncSetAttribute(oz_gram_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  oz_gram_kernel<S><<<grid, OZ_THREADS, smem, st>>>(ta, tb, a);
  RP_LAUNCH_CHECK("ozaki gram");
  return RP_OK;
}

}  // namespace rp
