// FP64 DMMA GEMM for the piCholesky CV path (sm_100a).
//
// C(M x N) = alpha * A(M x K) * B(K x N) + beta * C, batched over blockIdx.y.
//   A layout: KMAJOR  -> A(m, k) at A[k * lda + m]   (X^T of a row-major X; a column-major L)
//             MMAJOR  -> A(m, k) at A[m * lda + k]   (a row-major X_val)
//   B layout: always  -> B(k, n) at B[k * ldb + n]
//   C layout: column-major C(m, n) at C[n * ldc + m]
// Epilogues:
//   EPI_STORE    plain alpha/beta store (Gram blocks, X^T Y, Cholesky SYRK/TRSM updates)
//   EPI_SSE      sum over rows of (acc - Y[m][n % ycols])^2   (direct RMSE hold-out)
//   EPI_MIS      sum over rows of [sign(acc) != sign(Y)]       (direct MISCLASS hold-out)
//   EPI_DOTB     sum over rows of acc * B2[m][n]                (Gram-form hold-out b^T G b)
// The reduction epilogues never write C: they write one partial per (batch, m-tile, n) that a
// second kernel sums over m-tiles in a fixed order (deterministic, no atomics).
//
// Tiling: 256 threads = 8 warps, CTA tile BM x BN, warp tile WM x WN, BK = 16, 3-stage cp.async
// ring. Shared-memory strides are padded so both DMMA fragment reads are 2-wavefront
// (conflict-free) loads: KMAJOR A / B rows padded to (width + 8) doubles, MMAJOR A rows to 20.
#pragma once

#include "rp_common.cuh"

namespace rp {

enum { EPI_STORE = 0, EPI_SSE = 1, EPI_MIS = 2, EPI_DOTB = 3 };
enum { A_KMAJOR = 0, A_MMAJOR = 1 };

struct GemmArgs {
  int M, N, K;
  const double* A;
  int64_t lda, strideA;
  const double* B;
  int64_t ldb, strideB;
  double* C;
  int64_t ldc, strideC;
  double alpha, beta;
  int lower_only;  // square tiles only: compute tiles with tn <= tm (SYRK)
  // warp-specialised kernel only: A is symmetric and only its lower triangle is used, as
  // T = strict_lower(A) + diag(A)/2 (so A = T + T^T): row tile tm runs k < (tm+1)*BM, the
  // diagonal block is masked, and the tiles are walked heaviest first
  int tri_a;
  // reduction epilogues
  const double* Y;  // EPI_SSE/EPI_MIS: Y(m, o) at Y[m * ldy + o];  EPI_DOTB: B2(m, n) at Y[m*ldy+n]
  int64_t ldy, strideY;
  int ycols;
  double* partial;  // [batch][mtiles][N]
  // gated launch (the FP64 fallback of a tensor-core product): when non-null the kernel does its
  // work only if *run_if_set != 0 (the Ozaki range guard tripped), else every CTA exits at once --
  // unless tile_mask is given: then, with the guard clear, it computes only the column tiles whose
  // tile_mask[batch * ntiles + tn] is nonzero (the operand columns out of the tensor-core range)
  const int* run_if_set;
  const int* tile_mask;
};

// Number of gated FP64 fallbacks that ran (tensor-core products whose range guard tripped);
// read by rp_ozaki_fallbacks().
__device__ unsigned long long g_oz_fallbacks = 0;

constexpr int GEMM_BK = 16;
constexpr int GEMM_STAGES = 3;

template <int AL, int BM, int BN>
struct GemmSmem {
  static constexpr int A_STRIDE = (AL == A_KMAJOR) ? (BM + 8) : (GEMM_BK + 4);
  static constexpr int A_ELEMS = (AL == A_KMAJOR) ? GEMM_BK * A_STRIDE : BM * A_STRIDE;
  static constexpr int B_STRIDE = BN + 8;
  static constexpr int B_ELEMS = GEMM_BK * B_STRIDE;
  static constexpr size_t BYTES = sizeof(double) * GEMM_STAGES * (A_ELEMS + B_ELEMS);
};

template <int AL, int BM, int BN, int WM, int WN, int EPI, bool VEC2>
__global__ void __launch_bounds__(256) dgemm_kernel(GemmArgs p) {
  bool all_tiles = true;
  if (p.run_if_set != nullptr) {
    all_tiles = *p.run_if_set != 0;
    if (!all_tiles && p.tile_mask == nullptr) return;
    if (all_tiles && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&g_oz_fallbacks, 1ull);
  }
  constexpr int BK = GEMM_BK;
  constexpr int MT = WM / 8, NT = WN / 8;
  constexpr int WARPS_M = BM / WM;
  static_assert((BM / WM) * (BN / WN) == 8, "8 warps");
  using SM = GemmSmem<AL, BM, BN>;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + GEMM_STAGES * SM::A_ELEMS;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int batch = blockIdx.y;

  const int mtiles = (p.M + BM - 1) / BM;
  int tm, tn;
  if (p.lower_only) {
    int lin = blockIdx.x;
    tm = (int)((sqrt(8.0 * lin + 1.0) - 1.0) * 0.5);
    while ((tm + 1) * (tm + 2) / 2 <= lin) ++tm;
    while (tm * (tm + 1) / 2 > lin) --tm;
    tn = lin - tm * (tm + 1) / 2;
  } else {
    tm = blockIdx.x % mtiles;
    tn = blockIdx.x / mtiles;
  }
  if (!all_tiles && p.tile_mask[(int64_t)batch * ((p.N + BN - 1) / BN) + tn] == 0) return;
  const int m0 = tm * BM, n0 = tn * BN;
  const double* A = p.A + batch * p.strideA;
  const double* B = p.B + batch * p.strideB;

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ktiles = (p.K + BK - 1) / BK;

  auto load_stage = [&](int kt, int st) {
    const int k0 = kt * BK;
    double* dA = sA + st * SM::A_ELEMS;
    double* dB = sB + st * SM::B_ELEMS;
    constexpr int V = VEC2 ? 2 : 1;
    if (AL == A_KMAJOR) {
      constexpr int PER_ROW = BM / V;
      for (int c = tid; c < BK * PER_ROW; c += 256) {
        int kk = c / PER_ROW, mm = (c % PER_ROW) * V;
        int gk = k0 + kk, gm = m0 + mm;
        bool ok = gk < p.K && gm < p.M;
        const double* src = ok ? A + (int64_t)gk * p.lda + gm : A;
        if (VEC2) cp_async16(dA + kk * SM::A_STRIDE + mm, src, ok);
        else cp_async8(dA + kk * SM::A_STRIDE + mm, src, ok);
      }
    } else {
      constexpr int PER_ROW = BK / V;
      for (int c = tid; c < BM * PER_ROW; c += 256) {
        int mm = c / PER_ROW, kk = (c % PER_ROW) * V;
        int gk = k0 + kk, gm = m0 + mm;
        bool ok = gk < p.K && gm < p.M;
        const double* src = ok ? A + (int64_t)gm * p.lda + gk : A;
        if (VEC2) cp_async16(dA + mm * SM::A_STRIDE + kk, src, ok);
        else cp_async8(dA + mm * SM::A_STRIDE + kk, src, ok);
      }
    }
    {
      constexpr int PER_ROW = BN / V;
      for (int c = tid; c < BK * PER_ROW; c += 256) {
        int kk = c / PER_ROW, nn = (c % PER_ROW) * V;
        int gk = k0 + kk, gn = n0 + nn;
        bool ok = gk < p.K && gn < p.N;
        const double* src = ok ? B + (int64_t)gk * p.ldb + gn : B;
        if (VEC2) cp_async16(dB + kk * SM::B_STRIDE + nn, src, ok);
        else cp_async8(dB + kk * SM::B_STRIDE + nn, src, ok);
      }
    }
  };

#pragma unroll
  for (int s = 0; s < GEMM_STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    const int st = kt % GEMM_STAGES;
    {
      int nk = kt + GEMM_STAGES - 1;
      if (nk < ktiles) load_stage(nk, nk % GEMM_STAGES);
      cp_async_commit();
    }
    cp_async_wait<GEMM_STAGES - 1>();
    __syncthreads();
    const double* a_s = sA + st * SM::A_ELEMS;
    const double* b_s = sB + st * SM::B_ELEMS;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + t;
      double af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        int row = wm * WM + i * 8 + g;
        af[i] = (AL == A_KMAJOR) ? a_s[k * SM::A_STRIDE + row] : a_s[row * SM::A_STRIDE + k];
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = b_s[k * SM::B_STRIDE + wn * WN + j * 8 + g];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  if (EPI == EPI_STORE) {
    double* C = p.C + batch * p.strideC;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      int row = m0 + wm * WM + i * 8 + g;
      if (row >= p.M) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int col = n0 + wn * WN + j * 8 + 2 * t + h;
          if (col >= p.N) continue;
          double* c = C + (int64_t)col * p.ldc + row;
          double v = p.alpha * acc[i][j][h];
          if (p.beta != 0.0) v = fma(p.beta, *c, v);
          *c = v;
        }
      }
    }
  } else {
    // Row-reduction epilogues: each lane sums its rows for each of its columns, then the 8
    // lanes sharing t (same columns) reduce over g, then warps sharing wn reduce via smem.
    const double* Yb = p.Y + batch * p.strideY;
    double colsum[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) colsum[j][0] = colsum[j][1] = 0.0;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      int row = m0 + wm * WM + i * 8 + g;
      if (row >= p.M) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int col = n0 + wn * WN + j * 8 + 2 * t + h;
          if (col >= p.N) continue;
          double v;
          if (EPI == EPI_SSE) {
            double y = Yb[(int64_t)row * p.ldy + (col % p.ycols)];
            double e = acc[i][j][h] - y;
            v = e * e;
          } else if (EPI == EPI_MIS) {
            double y = Yb[(int64_t)row * p.ldy + (col % p.ycols)];
            double s_pred = acc[i][j][h] >= 0.0 ? 1.0 : -1.0;
            double s_y = (y > 0.0) ? 1.0 : ((y < 0.0) ? -1.0 : 0.0);
            v = (s_pred != s_y) ? 1.0 : 0.0;
          } else {
            v = acc[i][j][h] * Yb[(int64_t)row * p.ldy + col];
          }
          colsum[j][h] += v;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = colsum[j][h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        colsum[j][h] = v;
      }
    __syncthreads();
    double* red = smem;  // [WARPS_M][BN]
    if (g == 0) {
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) red[wm * BN + wn * WN + j * 8 + 2 * t + h] = colsum[j][h];
    }
    __syncthreads();
    for (int c = tid; c < BN; c += 256) {
      int col = n0 + c;
      if (col >= p.N) continue;
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < WARPS_M; ++w) s += red[w * BN + c];
      p.partial[((int64_t)batch * mtiles + tm) * p.N + col] = s;
    }
  }
}


// ---------------------------------------------------------------------------------------------
// Warp-specialised persistent variant (the default on aligned operands). One CTA per SM walks
// the (batch, tile) list; warp 8 is a producer that moves each 16-deep k-tile with 1-D bulk async
// copies (cp.async.bulk, one per contiguous tile row) into padded shared-memory rows and signals
// a full-mbarrier with the transaction byte count; warps 0-7 only issue LDS + DMMA and release
// the stage through an empty-mbarrier. The stage ring runs continuously across tiles, so the
// producer prefetches the next tile while the consumers run the previous tile's epilogue; there
// is no block-wide barrier in the main loop.
constexpr int WS_STAGES = 4;

template <int AL, int BM, int BN>
struct WsSmem {
  using B = GemmSmem<AL, BM, BN>;
  static constexpr size_t DATA = sizeof(double) * WS_STAGES * (B::A_ELEMS + B::B_ELEMS);
  static constexpr size_t RED = sizeof(double) * 8 * BN;  // reduction epilogue scratch (<= 8 row groups)
  static constexpr size_t BYTES = DATA + RED + 2 * WS_STAGES * sizeof(uint64_t);
};

struct TileCoord {
  int batch, tm, tn;
};

RP_DEVINL TileCoord ws_tile(const GemmArgs& p, int tile, int mtiles, int ntiles, int nbatch) {
  TileCoord c;
  if (p.tri_a) {  // descending row tile (work ~ tm + 1), then batch, then column tile
    const int per_tm = ntiles * nbatch;
    const int rank = tile / per_tm, rem = tile - rank * per_tm;
    c.tm = mtiles - 1 - rank;
    c.batch = rem / ntiles;
    c.tn = rem - c.batch * ntiles;
    return c;
  }
  const int per = p.lower_only ? mtiles * (mtiles + 1) / 2 : mtiles * ntiles;
  c.batch = tile / per;
  int lin = tile - c.batch * per;
  if (p.lower_only) {
    int tm = (int)((sqrt(8.0 * lin + 1.0) - 1.0) * 0.5);
    while ((tm + 1) * (tm + 2) / 2 <= lin) ++tm;
    while (tm * (tm + 1) / 2 > lin) --tm;
    c.tm = tm;
    c.tn = lin - tm * (tm + 1) / 2;
  } else {
    c.tm = lin % mtiles;
    c.tn = lin / mtiles;
  }
  return c;
}

// One 16-deep k-tile of a consumer warp's MT x NT DMMA tile. MASK (triangular A, diagonal block):
// A(row, k) -> 0 above the diagonal and A/2 on it; rk = (global row - global k) of fragment 0.
template <int AL, int MT, int NT, int A_STRIDE, int B_STRIDE, bool MASK>
RP_DEVINL void ws_ktile(double (&acc)[MT][NT][2], const double* a_s, const double* b_s, int arow0, int bcol0, int g,
                        int t, int rk) {
#pragma unroll
  for (int ks = 0; ks < GEMM_BK / 4; ++ks) {
    const int k = ks * 4 + t;
    double af[MT], bf[NT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int row = arow0 + i * 8 + g;
      af[i] = (AL == A_KMAJOR) ? a_s[k * A_STRIDE + row] : a_s[row * A_STRIDE + k];
      if (MASK) {
        const int dr = rk + i * 8 + g - k;  // global row - global k
        af[i] = dr < 0 ? 0.0 : (dr == 0 ? 0.5 * af[i] : af[i]);
      }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) bf[j] = b_s[k * B_STRIDE + bcol0 + j * 8 + g];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
}

template <int AL, int BM, int BN, int WM, int WN, int EPI>
__global__ void __launch_bounds__(288, 1) dgemm_ws_kernel(GemmArgs p, int total_tiles) {
  bool all_tiles = true;
  if (p.run_if_set != nullptr) {
    all_tiles = *p.run_if_set != 0;
    if (!all_tiles && p.tile_mask == nullptr) return;
    if (all_tiles && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&g_oz_fallbacks, 1ull);
  }
  constexpr int BK = GEMM_BK;
  constexpr int MT = WM / 8, NT = WN / 8;
  constexpr int WARPS_M = BM / WM;
  static_assert((BM / WM) * (BN / WN) == 8, "8 consumer warps");
  using SM = GemmSmem<AL, BM, BN>;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + WS_STAGES * SM::A_ELEMS;
  double* red = smem + WS_STAGES * (SM::A_ELEMS + SM::B_ELEMS);
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 8 * BN);
  uint64_t* empty = full + WS_STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mtiles = (p.M + BM - 1) / BM, ntiles = (p.N + BN - 1) / BN;
  const int ktiles_all = (p.K + BK - 1) / BK;
  const int nbatch = total_tiles / (p.lower_only ? mtiles * (mtiles + 1) / 2 : mtiles * ntiles);
  auto skip = [&](const TileCoord& c) {  // tiles outside the mask of a partial fallback
    return !all_tiles && p.tile_mask[(int64_t)c.batch * ntiles + c.tn] == 0;
  };
  auto ktiles_of = [&](int tm) {
    if (EPI != EPI_DOTB || !p.tri_a) return ktiles_all;
    const int kt = ((tm + 1) * BM + BK - 1) / BK;
    return kt < ktiles_all ? kt : ktiles_all;
  };

  if (tid == 0) {
    for (int s = 0; s < WS_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 8) {
    // ---------------- producer ----------------
    int it = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const TileCoord tc = ws_tile(p, tile, mtiles, ntiles, nbatch);
      if (skip(tc)) continue;
      const int m0 = tc.tm * BM, n0 = tc.tn * BN;
      const int mv = min(BM, p.M - m0), nv = min(BN, p.N - n0);
      const double* A = p.A + tc.batch * p.strideA;
      const double* B = p.B + tc.batch * p.strideB;
      const int ktiles = ktiles_of(tc.tm);
      if (EPI == EPI_STORE && p.beta != 0.0) {
        // warm L2 with the C tile the epilogue will read: its loads then hit L2 instead of HBM
        // (with short K the epilogue is a large share of a tile, and the consumers wait on it)
        const double* Ct = p.C + tc.batch * p.strideC + (int64_t)n0 * p.ldc + m0;
        const uint32_t bytes = (uint32_t)(mv * 8);
        if ((bytes & 15) == 0)
          for (int c = lane; c < nv; c += 32) {
            const double* col = Ct + (int64_t)c * p.ldc;
            if (((uintptr_t)col & 15) == 0)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(col), "r"(bytes) : "memory");
          }
      }
      for (int kt = 0; kt < ktiles; ++kt, ++it) {
        const int st = it % WS_STAGES;
        mbar_wait(&empty[st], ((it / WS_STAGES) & 1) ^ 1);
        const int k0 = kt * BK, kv = min(BK, p.K - k0);
        double* dA = sA + st * SM::A_ELEMS;
        double* dB = sB + st * SM::B_ELEMS;
        // zero the out-of-range parts of the stage (edge tiles only)
        if (kv < BK || mv < BM) {
          for (int e = lane; e < BK * BM; e += 32) {
            if (AL == A_KMAJOR) {
              const int kk = e / BM, mm = e % BM;
              if (kk >= kv || mm >= mv) dA[kk * SM::A_STRIDE + mm] = 0.0;
            } else {
              const int mm = e / BK, kk = e % BK;
              if (kk >= kv || mm >= mv) dA[mm * SM::A_STRIDE + kk] = 0.0;
            }
          }
        }
        if (kv < BK || nv < BN)
          for (int e = lane; e < BK * BN; e += 32) {
            const int kk = e / BN, nn = e % BN;
            if (kk >= kv || nn >= nv) dB[kk * SM::B_STRIDE + nn] = 0.0;
          }
        __syncwarp();
        const uint32_t bytesA = (uint32_t)(kv * mv * 8), bytesB = (uint32_t)(kv * nv * 8);
        if (lane == 0) mbar_arrive_expect_tx(&full[st], bytesA + bytesB);
        __syncwarp();
        if (AL == A_KMAJOR) {
          for (int kk = lane; kk < kv; kk += 32)
            bulk_g2s(dA + kk * SM::A_STRIDE, A + (int64_t)(k0 + kk) * p.lda + m0, (uint32_t)(mv * 8), &full[st]);
        } else {
          for (int mm = lane; mm < mv; mm += 32)
            bulk_g2s(dA + mm * SM::A_STRIDE, A + (int64_t)(m0 + mm) * p.lda + k0, (uint32_t)(kv * 8), &full[st]);
        }
        for (int kk = lane; kk < kv; kk += 32)
          bulk_g2s(dB + kk * SM::B_STRIDE, B + (int64_t)(k0 + kk) * p.ldb + n0, (uint32_t)(nv * 8), &full[st]);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  int it = 0;
  for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    const TileCoord tc = ws_tile(p, tile, mtiles, ntiles, nbatch);
    if (skip(tc)) continue;
    const int m0 = tc.tm * BM, n0 = tc.tn * BN;
    const int batch = tc.batch;
    const int ktiles = ktiles_of(tc.tm);
    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < ktiles; ++kt, ++it) {
      const int st = it % WS_STAGES;
      mbar_wait(&full[st], (it / WS_STAGES) & 1);
      const double* a_s = sA + st * SM::A_ELEMS;
      const double* b_s = sB + st * SM::B_ELEMS;
      if (EPI == EPI_DOTB && p.tri_a && kt * BK + BK > m0)  // k-tile in the diagonal block: T's mask
        ws_ktile<AL, MT, NT, SM::A_STRIDE, SM::B_STRIDE, true>(acc, a_s, b_s, wm * WM, wn * WN, g, t,
                                                              m0 + wm * WM - kt * BK);
      else
        ws_ktile<AL, MT, NT, SM::A_STRIDE, SM::B_STRIDE, false>(acc, a_s, b_s, wm * WM, wn * WN, g, t, 0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }

    if (EPI == EPI_STORE) {
      double* C = p.C + batch * p.strideC;
      if (p.beta != 0.0) {
        // issue every C load before any store (stores could alias later loads otherwise,
        // which serialises 64 global round trips per thread)
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int row = m0 + wm * WM + i * 8 + g;
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int col = n0 + wn * WN + j * 8 + 2 * t + h;
              const double old = (row < p.M && col < p.N) ? __ldcg(C + (int64_t)col * p.ldc + row) : 0.0;
              acc[i][j][h] = fma(p.beta, old, p.alpha * acc[i][j][h]);
            }
        }
      } else {
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            acc[i][j][0] *= p.alpha;
            acc[i][j][1] *= p.alpha;
          }
      }
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int row = m0 + wm * WM + i * 8 + g;
        if (row >= p.M) continue;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = n0 + wn * WN + j * 8 + 2 * t + h;
            if (col < p.N) C[(int64_t)col * p.ldc + row] = acc[i][j][h];
          }
        }
      }
    } else {
      const double* Yb = p.Y + batch * p.strideY;
      double colsum[NT][2];
#pragma unroll
      for (int j = 0; j < NT; ++j) colsum[j][0] = colsum[j][1] = 0.0;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        int row = m0 + wm * WM + i * 8 + g;
        if (row >= p.M) continue;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            int col = n0 + wn * WN + j * 8 + 2 * t + h;
            if (col >= p.N) continue;
            double v;
            if (EPI == EPI_SSE) {
              double y = Yb[(int64_t)row * p.ldy + (col % p.ycols)];
              double e = acc[i][j][h] - y;
              v = e * e;
            } else if (EPI == EPI_MIS) {
              double y = Yb[(int64_t)row * p.ldy + (col % p.ycols)];
              double s_pred = acc[i][j][h] >= 0.0 ? 1.0 : -1.0;
              double s_y = (y > 0.0) ? 1.0 : ((y < 0.0) ? -1.0 : 0.0);
              v = (s_pred != s_y) ? 1.0 : 0.0;
            } else {
              v = acc[i][j][h] * Yb[(int64_t)row * p.ldy + col];
            }
            colsum[j][h] += v;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double v = colsum[j][h];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          colsum[j][h] = v;
        }
      named_bar_sync(1, 256);  // previous tile's readers of red are done
      if (g == 0) {
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) red[wm * BN + wn * WN + j * 8 + 2 * t + h] = colsum[j][h];
      }
      named_bar_sync(1, 256);
      for (int c = tid; c < BN; c += 256) {
        int col = n0 + c;
        if (col >= p.N) continue;
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS_M; ++w) s += red[w * BN + c];
        p.partial[((int64_t)batch * mtiles + tc.tm) * p.N + col] = s;
      }
    }
  }
}

}  // namespace rp
