// C-ABI entry points for the piCholesky CV path (everything except the fused eval+solve,
// which lives in rp_solve.cu). See include/ridgepath_b200.h for the contract and the
// reference routine each entry point replaces.
#include <map>
#include <mutex>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rp_common.cuh"
#include "rp_gemm.cuh"
#include "rp_potrf_diag.cuh"
#include "rp_ozaki.cuh"
#include "../../include/ridgepath_b200.h"

namespace rp {

static thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

static std::atomic<long long> g_launches{0};
extern int g_solve_lam;      // rp_solve.cu
extern int g_solve_cluster;  // rp_solve.cu
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static bool g_profile = false;
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
  cudaStream_t st;
};
static std::vector<ProfRec> g_prof;
bool prof_on() { return g_profile; }
cudaEvent_t prof_event() {
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
void prof_push(const char* name, cudaEvent_t a, cudaEvent_t b, cudaStream_t st) { g_prof.push_back({name, a, b, st}); }

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// Path options (rp_set_option; the environment variables set the initial value for A/B runs):
// Gram-form hold-out on the int8 tensor cores (Ozaki, rp_ozaki.cuh oz_holdout) when the workspace
// allows ("holdout_ozaki" 0 / RP_HOLDOUT_OZAKI=0 keeps FP64 DMMA); Gram blocks on FP64 DMMA even
// with a workspace ("gram_dmma" 1 / RP_GRAM_DMMA=1).
static bool env_flag(const char* name, bool dflt) {
  const char* e = getenv(name);
  return e ? e[0] == '1' : dflt;
}
static bool g_holdout_ozaki = env_flag("RP_HOLDOUT_OZAKI", true);
static bool g_gram_dmma = env_flag("RP_GRAM_DMMA", false);

// ------------------------------------------------------------------ GEMM dispatch

// Operands the bulk-copy (warp-specialised) GEMM can stream: 16-byte aligned rows and sizes.
static bool gemm_vec2(const GemmArgs& a, int AL) {
  return aligned16(a.A) && aligned16(a.B) && a.lda % 2 == 0 && a.ldb % 2 == 0 && a.strideA % 2 == 0 &&
         a.strideB % 2 == 0 && a.N % 2 == 0 && (AL == A_KMAJOR ? a.M % 2 == 0 : a.K % 2 == 0);
}

template <int AL, int BM, int BN, int WM, int WN, int EPI>
static int gemm(const GemmArgs& a, int batch, cudaStream_t st, const char* name) {
  if (a.M <= 0 || a.N <= 0 || batch <= 0) return RP_OK;
  bool vec2 = gemm_vec2(a, AL);
  if (a.tri_a && !vec2) return set_error(RP_EINVAL, "%s: triangular A needs the bulk-copy GEMM", name);
  const int mt = (a.M + BM - 1) / BM, nt = (a.N + BN - 1) / BN;
  if (a.lower_only && (BM != BN || a.M != a.N)) return set_error(RP_EINVAL, "%s: lower_only needs square", name);
  dim3 grid(a.lower_only ? mt * (mt + 1) / 2 : mt * nt, batch);
  size_t smem = GemmSmem<AL, BM, BN>::BYTES;
  // bulk-copy (warp-specialised) path: every copied tile row must be 16-byte aligned and sized
  const bool ws = vec2 && a.N % 2 == 0 && (AL == A_KMAJOR ? a.M % 2 == 0 : a.K % 2 == 0);
  if (ws) {
    auto k = dgemm_ws_kernel<AL, BM, BN, WM, WN, EPI>;
    size_t wsm = WsSmem<AL, BM, BN>::BYTES;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
    const int total = (int)grid.x * batch;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ctas = total < sms ? total : sms;  // persistent: one CTA per SM walks the tile list
    k<<<ctas, 288, wsm, st>>>(a, total);
  } else if (vec2) {
    auto k = dgemm_kernel<AL, BM, BN, WM, WN, EPI, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, 256, smem, st>>>(a);
  } else {
    auto k = dgemm_kernel<AL, BM, BN, WM, WN, EPI, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, 256, smem, st>>>(a);
  }
  RP_LAUNCH_CHECK(name);
  return RP_OK;
}

static GemmArgs gemm_args() {
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.alpha = 1.0;
  a.beta = 0.0;
  return a;
}

// ------------------------------------------------------------------ small kernels

// Lower-triangle mirror, 32x32 tiles through shared memory.
__global__ void symmetrize_kernel(double* G, int d, int64_t stride) {
  __shared__ double tile[32][33];
  const int nt = (d + 31) / 32;
  int lin = blockIdx.x;
  int I = (int)((sqrt(8.0 * lin + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= lin) ++I;
  while (I * (I + 1) / 2 > lin) --I;
  int J = lin - I * (I + 1) / 2;
  if (I >= nt) return;
  double* A = G + blockIdx.y * stride;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    int row = I * 32 + tx, col = J * 32 + r;  // element (row, col) of the lower block (I, J)
    tile[r][tx] = (row < d && col < d) ? A[(int64_t)col * d + row] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    // write (J*32 + tx, I*32 + r) = (I*32 + r, J*32 + tx)
    int row = J * 32 + tx, col = I * 32 + r;
    if (row < d && col < d && row < col) A[(int64_t)col * d + row] = tile[tx][r];
  }
}

constexpr int FS_FOLDS = 64, FS_LAMS = 32;  // per launch; rp_fold_systems chunks over more
struct FoldSysArgs {
  int folds[FS_FOLDS];
  double lams[FS_LAMS];
};

// Leave-one-out sums, one pass over the Gram blocks for all folds of the call:
//   A[f][s0 + s] = sum_{b != folds[f]} G_b + lams[s] I  (fixed order b = 0..nblocks-1, lower triangle)
// A[f] holds s_total matrices (a launch covers lambdas s0 .. s0 + s - 1).
// Each element's nblocks values are read once (registers when nblocks <= KB) and every fold's sum
// is formed directly -- no G_total - G_f cancellation, and the sum of a fold is bit-identical
// whether or not its own block is among the nblocks (the streamed path factors the last fold
// before its block has arrived). Column by column so the threads of a block stay on contiguous rows.
template <int KB>
__global__ void fold_shift_kernel(const double* G, int nblocks, int d, int s, int s0, int s_total, int nf,
                                  FoldSysArgs fa, double* A) {
  const int j = blockIdx.x;  // column
  const int64_t n = (int64_t)d * d;
  const double* gj = G + (int64_t)j * d;
  for (int i = j + threadIdx.x; i < d; i += blockDim.x) {
    double g[KB > 0 ? KB : 1];
    if (KB > 0) {
#pragma unroll
      for (int b = 0; b < KB; ++b) g[b] = b < nblocks ? __ldcs(gj + b * n + i) : 0.0;
    }
    for (int f = 0; f < nf; ++f) {
      const int hold = fa.folds[f];
      double v = 0.0;
      if (KB > 0) {
#pragma unroll
        for (int b = 0; b < KB; ++b)
          if (b < nblocks && b != hold) v += g[b];
      } else {
        for (int b = 0; b < nblocks; ++b)
          if (b != hold) v += gj[b * n + i];
      }
      double* out = A + ((int64_t)f * s_total + s0) * n + (int64_t)j * d + i;
      for (int si = 0; si < s; ++si) __stcs(out + si * n, (i == j) ? v + fa.lams[si] : v);
    }
  }
}

// The same sums on row pairs (d even, 16-byte aligned G and A): 16-byte loads and streaming stores halve the
// instruction count of the scalar kernel, which ncu showed issuing 71% of its cycles at 4.5 TB/s. Per entry the
// additions are the scalar kernel's, in the same order. An odd column's diagonal entry is done by one thread
// on its own, so nothing above the diagonal is read or written.
template <int KB>
__global__ void __launch_bounds__(256) fold_shift2_kernel(const double* G, int nblocks, int d, int s, int s0,
                                                          int s_total, int nf, FoldSysArgs fa, double* A) {
  const int j = blockIdx.x;  // column
  const int64_t n = (int64_t)d * d;
  const double* gj = G + (int64_t)j * d;
  if ((j & 1) && threadIdx.x == 0) {  // the diagonal entry of an odd column
    double g[KB];
#pragma unroll
    for (int b = 0; b < KB; ++b) g[b] = b < nblocks ? gj[b * n + j] : 0.0;
    for (int f = 0; f < nf; ++f) {
      const int hold = fa.folds[f];
      double v = 0.0;
#pragma unroll
      for (int b = 0; b < KB; ++b)
        if (b < nblocks && b != hold) v += g[b];
      double* out = A + ((int64_t)f * s_total + s0) * n + (int64_t)j * d + j;
      for (int si = 0; si < s; ++si) out[si * n] = v + fa.lams[si];
    }
  }
  for (int i = j + (j & 1) + 2 * threadIdx.x; i < d; i += 2 * blockDim.x) {
    double2 g[KB];
#pragma unroll
    for (int b = 0; b < KB; ++b)
      g[b] = b < nblocks ? __ldcs(reinterpret_cast<const double2*>(gj + b * n + i)) : make_double2(0.0, 0.0);
    for (int f = 0; f < nf; ++f) {
      const int hold = fa.folds[f];
      double2 v = make_double2(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < KB; ++b)
        if (b < nblocks && b != hold) {
          v.x += g[b].x;
          v.y += g[b].y;
        }
      double* out = A + ((int64_t)f * s_total + s0) * n + (int64_t)j * d + i;
      for (int si = 0; si < s; ++si)
        __stcs(reinterpret_cast<double2*>(out + si * n), make_double2(i == j ? v.x + fa.lams[si] : v.x, v.y));
    }
  }
}

// rhs[f] = sum_{b != folds[f]} C_b (fixed order), row-major dp x m, rows >= d zero.
__global__ void fold_rhs_kernel(const double* C, int nblocks, int d, int dp, int m, FoldSysArgs fa, double* rhs) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;  // over dp*m, row-major (i, o)
  if (e >= dp * m) return;
  const int f = blockIdx.y;
  int i = e / m, o = e % m;
  double v = 0.0;
  if (i < d)
    for (int b = 0; b < nblocks; ++b)
      if (b != fa.folds[f]) v += C[((int64_t)b * m + o) * d + i];
  rhs[(int64_t)f * dp * m + e] = v;
}

// Column sums of squares per fold block: yy[b][o] = sum_rows Y[row][o]^2 (fixed row order per thread
// chunk, then a fixed-order combine).
__global__ void col_sumsq_kernel(const double* Y, int64_t ldy, int64_t rows, int m, double* yy) {
  const int b = blockIdx.x, o = blockIdx.y;
  const double* y = Y + (int64_t)b * rows * ldy + o;
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += 256) {
    double v = y[r * ldy];
    s = fma(v, v, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) yy[b * m + o] = red[0];
}

// ------------------------------------------------------------------ Cholesky

constexpr int CHOL_NB = 128;
static int CHOL_OB = [] {
  const char* e = getenv("RP_CHOL_OB");
  // measured at c4 with DMMA trailing updates: 384 -> 38.3 ms, 512 -> 37.4, 768 -> 36.8, 1024 -> 36.7;
  // with tensor-core trailing updates (evals/s): 768 -> 15442, 1024 -> 15815, 1536 -> 15949, 2048 -> 15919;
  // once the tensor-core SYRK drained both passes before one C read-modify-write (factorize ms):
  // 512 -> 24.3, 640 -> 24.6, 768 -> 22.4-24.0, 896 -> 23.2, 1024 -> 23.0-23.5, 1536 -> 26.1
  int v = e ? atoi(e) : 768;
  return v >= 128 && v % 128 == 0 ? v : 768;
}();

// ------------------------------------------------------------------ fit

struct FitArgs {
  double P[5][32];  // (r+1) x s
  double V[32][5];  // s x (r+1)
};

// theta_p = sum_s P[p][s] L_s for one 64 x 64 tile (I, J) of every fold, written straight into the
// column-major padded tile planes, with the tile's share of ||T - V theta||_F^2. Padding rows (64..67)
// and entries outside the triangle are 0, padded diagonal entries 1 in plane 0.
// HBM-bound (s factor reads + P plane writes per entry): each thread owns pairs of adjacent rows of a
// column (16-byte loads of every factor and 16-byte streaming stores of every plane, coalesced along
// the column), and the kernel is sized for 4 resident CTAs per SM so enough loads are in flight to
// cover the HBM latency.
constexpr int FIT_THREADS = 256;
constexpr int FIT_PAIRS = TILE_PLANE / 2;
#ifndef RP_FIT_IU
#define RP_FIT_IU 1
#endif
constexpr int FIT_IU = RP_FIT_IU;  // interior tiles: columns in flight per thread  // 34 row pairs (64 rows + 4 padding) per column x 64 columns

// Occupancy over unrolling (measured at c4, ms): 4 CTAs x 256 threads per SM, one pair per thread in
// flight 0.95; 2 CTAs with 2 / 3 pairs in flight 1.22 / 1.21; 3 CTAs x 2 pairs 1.10; 5 / 6 / 8 CTAs
// (register-capped) 1.08 / 1.17 / 1.63.
// INTERIOR: the instantiation handles only the interior tiles (fast path) / only the others; both are launched
// over all tiles and a CTA of the wrong kind exits at once.
// PT > 0: compile-time plane count of the interior instantiation (0 in the general one: split = an interior
// instantiation runs beside it and owns the interior tiles).
template <int SMAX, int FIT_UNROLL = 1, bool INTERIOR = false, int PT = 0>
__global__ void __launch_bounds__(FIT_THREADS, SMAX <= 8 ? 4 : 1) fit_tiles_kernel(const double* L, int d, int s, int r,
                                                                int64_t ntiles, int64_t fold_stride, FitArgs fa,
                                                                double* theta, double* partial, int split) {
  const int64_t tile = blockIdx.x;
  const int f = blockIdx.y;
  const int P = PT ? PT : r + 1;
  int I = (int)((sqrt(8.0 * tile + 1.0) - 1.0) * 0.5);
  while ((int64_t)(I + 1) * (I + 2) / 2 <= tile) ++I;
  while ((int64_t)I * (I + 1) / 2 > tile) --I;
  const int J = (int)(tile - (int64_t)I * (I + 1) / 2);
  const int64_t n = (int64_t)d * d;
  const double* Lf = L + (int64_t)f * s * n;
  double* out = theta + f * fold_stride + tile * P * TILE_PLANE;
  const bool vec = (d & 1) == 0 && ((uintptr_t)L & 15) == 0;  // 16-byte aligned row pairs in the factors
  double res = 0.0;
  // Interior tiles (strictly below the diagonal, all 64 rows inside the matrix: the bulk of the triangle) take a
  // path without per-entry predicates or index divisions: a warp owns one column per step (lane = row pair, 512
  // contiguous bytes per factor); the 4 padding rows of every column are zeros.
  // Same arithmetic per entry as the general path below (only the order of the residual's partial sums differs).
  const bool interior = split && vec && I > J && (I + 1) * 64 <= d;
  if (interior != INTERIOR) return;
  if constexpr (INTERIOR) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* src0 = Lf + (int64_t)(J * 64) * d + I * 64 + 2 * lane;
#pragma unroll 1
    for (int j0 = 0; j0 < 64; j0 += FIT_IU * (FIT_THREADS / 32)) {
      double2 T[FIT_IU][SMAX];
#pragma unroll
      for (int u = 0; u < FIT_IU; ++u) {
        const double* src = src0 + (int64_t)(j0 + u * (FIT_THREADS / 32) + warp) * d;
#pragma unroll
        for (int si = 0; si < SMAX; ++si)
          T[u][si] = si < s ? __ldcs(reinterpret_cast<const double2*>(src + si * n)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < FIT_IU; ++u) {
        const int e = (j0 + u * (FIT_THREADS / 32) + warp) * TILE_LD + 2 * lane;
        constexpr int PA = PT ? PT : 5;
        double2 th[PA];
#pragma unroll
        for (int p = 0; p < PA; ++p)
          if (p < P) {
            double v0 = 0.0, v1 = 0.0;
#pragma unroll
            for (int si = 0; si < SMAX; ++si)
              if (si < s) {
                v0 = fma(fa.P[p][si], T[u][si].x, v0);
                v1 = fma(fa.P[p][si], T[u][si].y, v1);
              }
            th[p] = make_double2(v0, v1);
            __stcs(reinterpret_cast<double2*>(out + p * TILE_PLANE + e), th[p]);
          }
#pragma unroll
        for (int si = 0; si < SMAX; ++si)
          if (si < s) {
            double v0 = 0.0, v1 = 0.0;
#pragma unroll
            for (int p = 0; p < PA; ++p)
              if (p < P) {
                v0 = fma(fa.V[si][p], th[p].x, v0);
                v1 = fma(fa.V[si][p], th[p].y, v1);
              }
            const double d0 = T[u][si].x - v0, d1 = T[u][si].y - v1;
            res = fma(d0, d0, res);
            res = fma(d1, d1, res);
          }
      }
    }
    // padding rows 64..67 of the 64 columns: two zero pairs per column and plane
    if (threadIdx.x < 128) {
      const int e = (threadIdx.x >> 1) * TILE_LD + 64 + 2 * (threadIdx.x & 1);
      for (int p = 0; p < P; ++p) __stcs(reinterpret_cast<double2*>(out + p * TILE_PLANE + e), make_double2(0.0, 0.0));
    }
  }
  for (int q0 = threadIdx.x; !INTERIOR && q0 < FIT_PAIRS; q0 += FIT_THREADS * FIT_UNROLL) {
    double2 T[FIT_UNROLL][SMAX];
    int kind[FIT_UNROLL];  // 0: outside the tile, 1: both rows in the triangle, 2: mixed (edge / diagonal)
#pragma unroll
    for (int u = 0; u < FIT_UNROLL; ++u) {
      const int qq = q0 + u * FIT_THREADS;
      const int e = 2 * qq;
      const int j = e / TILE_LD, i = e - j * TILE_LD;  // rows i, i + 1 of column j of the tile
      const int row = I * 64 + i, col = J * 64 + j;
      const bool in0 = qq < FIT_PAIRS && i < 64 && row < d && col < d && row >= col;
      const bool in1 = qq < FIT_PAIRS && i + 1 < 64 && row + 1 < d && col < d && row + 1 >= col;
      kind[u] = (in0 && in1 && vec) ? 1 : ((in0 || in1) ? 2 : 0);
      const double* src = Lf + (int64_t)col * d + row;
#pragma unroll
      for (int si = 0; si < SMAX; ++si) {
        if (si < s && kind[u] == 1) {
          T[u][si] = __ldcs(reinterpret_cast<const double2*>(src + si * n));
        } else if (si < s && kind[u] == 2) {
          T[u][si].x = in0 ? __ldcs(src + si * n) : 0.0;
          T[u][si].y = in1 ? __ldcs(src + si * n + 1) : 0.0;
        } else {
          T[u][si] = make_double2(0.0, 0.0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < FIT_UNROLL; ++u) {
      const int qq = q0 + u * FIT_THREADS;
      if (qq >= FIT_PAIRS) continue;
      const int e = 2 * qq;
      if (kind[u] == 0) {
        const int j = e / TILE_LD, i = e - j * TILE_LD;
        const int row = I * 64 + i, col = J * 64 + j;
        const double d0 = (i < 64 && row == col && row >= d) ? 1.0 : 0.0;
        const double d1 = (i + 1 < 64 && row + 1 == col && row + 1 >= d) ? 1.0 : 0.0;
        for (int p = 0; p < P; ++p)
          __stcs(reinterpret_cast<double2*>(out + p * TILE_PLANE + e), p == 0 ? make_double2(d0, d1)
                                                                             : make_double2(0.0, 0.0));
        continue;
      }
      // rows outside the triangle (mixed pairs) carry T = 0 and get theta = 0 and no residual
      const int j = e / TILE_LD, i = e - j * TILE_LD;
      const int row = I * 64 + i, col = J * 64 + j;
      const bool in0 = i < 64 && row < d && col < d && row >= col;
      const bool in1 = i + 1 < 64 && row + 1 < d && col < d && row + 1 >= col;
      double2 th[5];
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        if (p < P) {
          double v0 = 0.0, v1 = 0.0;
#pragma unroll
          for (int si = 0; si < SMAX; ++si)
            if (si < s) {
              v0 = fma(fa.P[p][si], T[u][si].x, v0);
              v1 = fma(fa.P[p][si], T[u][si].y, v1);
            }
          th[p] = make_double2(v0, v1);
          if (kind[u] == 2) {  // padded diagonal entries below d keep the identity in plane 0
            if (!in0) th[p].x = (p == 0 && i < 64 && row == col && row >= d) ? 1.0 : 0.0;
            if (!in1) th[p].y = (p == 0 && i + 1 < 64 && row + 1 == col && row + 1 >= d) ? 1.0 : 0.0;
          }
          __stcs(reinterpret_cast<double2*>(out + p * TILE_PLANE + e), th[p]);
        }
      }
#pragma unroll
      for (int si = 0; si < SMAX; ++si) {
        if (si < s) {
          double v0 = 0.0, v1 = 0.0;
#pragma unroll
          for (int p = 0; p < 5; ++p)
            if (p < P) {
              v0 = fma(fa.V[si][p], th[p].x, v0);
              v1 = fma(fa.V[si][p], th[p].y, v1);
            }
          if (in0) {
            const double dl = T[u][si].x - v0;
            res = fma(dl, dl, res);
          }
          if (in1) {
            const double dl = T[u][si].y - v1;
            res = fma(dl, dl, res);
          }
        }
      }
    }
  }
  __shared__ double red[FIT_THREADS];
  red[threadIdx.x] = res;
  __syncthreads();
  for (int w = FIT_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(int64_t)f * ntiles + tile] = red[0];
}

// Any number of samples / planes (s > 32 or degree > 4): the same arithmetic with P (P x s) and V
// (s x P) in device memory and the samples re-read per plane (L1-resident); not on the BASELINE path.
__global__ void __launch_bounds__(512) fit_tiles_any_kernel(const double* L, int d, int s, int r, int64_t ntiles,
                                                            int64_t fold_stride, const double* Pd, const double* Vd,
                                                            double* theta, double* partial) {
  const int64_t tile = blockIdx.x;
  const int f = blockIdx.y;
  const int P = r + 1;
  int I = (int)((sqrt(8.0 * tile + 1.0) - 1.0) * 0.5);
  while ((int64_t)(I + 1) * (I + 2) / 2 <= tile) ++I;
  while ((int64_t)I * (I + 1) / 2 > tile) --I;
  const int J = (int)(tile - (int64_t)I * (I + 1) / 2);
  const int64_t n = (int64_t)d * d;
  const double* Lf = L + (int64_t)f * s * n;
  double* out = theta + f * fold_stride + tile * P * TILE_PLANE;
  double res = 0.0;
  for (int e = threadIdx.x; e < TILE_PLANE; e += blockDim.x) {
    const int j = e / TILE_LD, i = e - j * TILE_LD;
    const int row = I * 64 + i, col = J * 64 + j;
    if (i < 64 && row < d && col < d && row >= col) {
      const double* Le = Lf + (int64_t)col * d + row;
      for (int p = 0; p < P; ++p) {
        double v = 0.0;
        for (int si = 0; si < s; ++si) v = fma(Pd[p * s + si], Le[si * n], v);
        out[p * TILE_PLANE + e] = v;
      }
      for (int si = 0; si < s; ++si) {
        double v = 0.0;
        for (int p = 0; p < P; ++p) v = fma(Vd[si * P + p], out[p * TILE_PLANE + e], v);
        const double dlt = Le[si * n] - v;
        res = fma(dlt, dlt, res);
      }
    } else {
      const double diag = (i < 64 && row == col && row >= d) ? 1.0 : 0.0;
      for (int p = 0; p < P; ++p) out[p * TILE_PLANE + e] = (p == 0) ? diag : 0.0;
    }
  }
  __shared__ double red[512];
  red[threadIdx.x] = res;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(int64_t)f * ntiles + tile] = red[0];
}

__global__ void fit_resid_kernel(const double* partial, int64_t ntiles, double* resid) {
  const int f = blockIdx.x;
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < ntiles; i += 256) s += partial[f * ntiles + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) resid[f] = sqrt(red[0]);
}

RP_DEVINL int64_t tile_offset(int row, int col, int P) {
  const int I = row >> 6, J = col >> 6;
  return ((int64_t)I * (I + 1) / 2 + J) * P * TILE_PLANE + (col & 63) * TILE_LD + (row & 63);
}

// pichol.eval_vector's arithmetic exactly (pichol.py:147-150): v = theta_r; v *= t; v += theta_i,
// with separate roundings (no FMA contraction).
RP_DEVINL double horner_ref(const double* th, int P, double t) {
  double v = th[(int64_t)(P - 1) * TILE_PLANE];
  for (int p = P - 2; p >= 0; --p) v = __dadd_rn(__dmul_rn(v, t), th[(int64_t)p * TILE_PLANE]);
  return v;
}

__global__ void materialize_kernel(const double* theta, int d, int P, double t, double* L) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)d * d) return;
  int row = (int)(e % d), col = (int)(e / d);
  L[e] = (row >= col) ? horner_ref(theta + tile_offset(row, col, P), P, t) : 0.0;
}

__global__ void export_kernel(const double* theta, int d, int P, const int64_t* perm, int64_t D, double* out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= D) return;
  int64_t pos = perm ? perm[j] : j;
  int row = (int)(pos % d), col = (int)(pos / d);
  for (int p = 0; p < P; ++p)
    out[p * D + j] = (row >= col) ? theta[tile_offset(row, col, P) + (int64_t)p * TILE_PLANE] : 0.0;
}

__global__ void theta_init_kernel(double* theta, int d, int P, int64_t ntiles) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t half = ntiles * P * TILE_PLANE;
  if (e >= half) return;
  const int64_t w0 = e;
  const int64_t tile = w0 / (P * TILE_PLANE);
  const int rem = (int)(w0 % (P * TILE_PLANE));
  const int p = rem / TILE_PLANE, w = rem % TILE_PLANE;
  int I = (int)((sqrt(8.0 * tile + 1.0) - 1.0) * 0.5);
  while ((int64_t)(I + 1) * (I + 2) / 2 <= tile) ++I;
  while ((int64_t)I * (I + 1) / 2 > tile) --I;
  const int J = (int)(tile - (int64_t)I * (I + 1) / 2);
  const int mj = w / TILE_LD, mn = w % TILE_LD;
  // only the padded diagonal is nonzero
  const int row = I * 64 + mn, col = J * 64 + mj;
  theta[e] = (p == 0 && mn < 64 && row == col && row >= d) ? 1.0 : 0.0;
}

__global__ void import_kernel(const double* vec, int d, int P, const int64_t* perm, int64_t D, int64_t ntiles,
                              double* theta) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= D) return;
  int64_t pos = perm ? perm[j] : j;
  int row = (int)(pos % d), col = (int)(pos / d);
  if (row < col) return;
  const int I = row >> 6, J = col >> 6;
  const int64_t base = ((int64_t)I * (I + 1) / 2 + J) * P * TILE_PLANE;
  for (int p = 0; p < P; ++p) theta[base + (int64_t)p * TILE_PLANE + (col & 63) * TILE_LD + (row & 63)] = vec[p * D + j];
}

// ------------------------------------------------------------------ hold-out reductions

// sse[f][n] = sum_tm partial[f][tm][n] (fixed order), then curves[f][j][o] from it.
// Gram form: n_val * MSE = y^T y - 2 w^T c + w^T G w loses log2((y^T y + |2 w^T c| + w^T G w) / sse)
// bits to cancellation (a near-exact fit, tiny noise). Columns that would lose more than 20 bits
// (relative error above ~1e-10 on the RMSE) are listed in rep_list and recomputed from the direct
// residual by holdout_repair_kernel (cvsearch.py:119-120's arithmetic).
constexpr double HOLDOUT_CANCEL = 1048576.0;  // 2^20
__global__ void holdout_finish_kernel(const double* partial, int mtiles, int N, int m, int64_t n_val, int metric,
                                      const double* yy, const double* bc, double quad_scale, double* curves,
                                      int* rep_count, int* rep_list) {
  const int f = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double s = 0.0;
  for (int tm = 0; tm < mtiles; ++tm) s += partial[((int64_t)f * mtiles + tm) * N + n];
  double out;
  if (yy) {  // Gram form: n_val * MSE = y^T y - 2 w^T c + w^T G w
    const int o = n % m;
    const double yv = yy[f * m + o], b2 = 2.0 * bc[(int64_t)f * N + n], qd = quad_scale * s;
    double sse = yv - b2 + qd;
    if (rep_list != nullptr && !(sse * HOLDOUT_CANCEL >= fabs(yv) + fabs(b2) + fabs(qd)))
      rep_list[atomicAdd(rep_count, 1)] = f * N + n;
    out = sqrt((sse > 0.0 ? sse : 0.0) / (double)n_val);
  } else if (metric == RP_METRIC_RMSE) {
    out = sqrt(s / (double)n_val);
  } else {
    out = s / (double)n_val;
  }
  curves[(int64_t)f * N + n] = out;
}

// Direct residual of the listed Gram-form columns: part[c][chunk] = sum over the chunk's rows of
// (x_row . w - y_row)^2 (rows in order per warp, warps combined in order: deterministic for a
// column whatever its position in the list). w is staged in shared memory when it fits.
constexpr int REP_CHUNKS = 16;
__global__ void __launch_bounds__(256) holdout_repair_kernel(const double* X, int64_t ldx, int64_t fold_stride_rows,
                                                             int64_t n_val, int d, const double* Y, int64_t ldy, int m,
                                                             const double* W, int64_t ldw, int64_t w_fold_stride,
                                                             int N, const int* rep_count, const int* rep_list,
                                                             int w_in_smem, double* part) {
  extern __shared__ double rep_w[];
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int count = *rep_count;
  const int64_t r0 = n_val * blockIdx.x / REP_CHUNKS, r1 = n_val * (blockIdx.x + 1) / REP_CHUNKS;
  for (int c = blockIdx.y; c < count; c += gridDim.y) {
    const int id = rep_list[c], f = id / N, n = id - f * N, o = n % m;
    const double* w = W + f * w_fold_stride + n;
    if (w_in_smem)
      for (int k = threadIdx.x; k < d; k += 256) rep_w[k] = w[(int64_t)k * ldw];
    __syncthreads();
    double acc = 0.0;  // lane 0: this warp's rows
    for (int64_t r = r0 + warp; r < r1; r += 8) {
      const double* x = X + (f * fold_stride_rows + r) * ldx;
      double p = 0.0;
      for (int k = lane; k < d; k += 32) p = fma(x[k], w_in_smem ? rep_w[k] : w[(int64_t)k * ldw], p);
#pragma unroll
      for (int sh = 16; sh > 0; sh >>= 1) p += __shfl_xor_sync(0xffffffffu, p, sh);
      const double e = p - Y[(f * fold_stride_rows + r) * ldy + o];
      acc = fma(e, e, acc);
    }
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < 8; ++i) t += red[i];
      part[(int64_t)c * REP_CHUNKS + blockIdx.x] = t;
    }
    __syncthreads();
  }
}

__global__ void holdout_repair_finish_kernel(const int* rep_count, const int* rep_list, const double* part,
                                             int64_t n_val, double* curves) {
  const int count = *rep_count;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < count; c += gridDim.x * blockDim.x) {
    double sse = 0.0;
    for (int i = 0; i < REP_CHUNKS; ++i) sse += part[(int64_t)c * REP_CHUNKS + i];
    curves[rep_list[c]] = sqrt(sse / (double)n_val);
  }
}

// bc[f][n] = sum_i W[i][n] * C_f[i][o]
// bc[f][n] = sum_i W[i][n] * C_f[i][o]: CTA = 32 columns x 8 row groups (rows i = g mod 8,
// coalesced 256-byte row segments), the 8 partials combined in a fixed order.
__global__ void __launch_bounds__(256) holdout_bc_kernel(const double* W, int64_t ldw, int64_t w_fold_stride,
                                                         const double* Cf, int64_t c_stride, int d, int m, int N,
                                                         double* bc) {
  __shared__ double red[8][32];
  const int f = blockIdx.y, lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int n = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (n < N) {
    const int o = n % m;
    const double* w = W + f * w_fold_stride + n;
    const double* c = Cf + f * c_stride + (int64_t)o * d;
#pragma unroll 4
    for (int i = g; i < d; i += 8) s = fma(w[(int64_t)i * ldw], c[i], s);
  }
  red[g][lane] = s;
  __syncthreads();
  if (g == 0 && n < N) {
    double t = red[0][lane];
    for (int r = 1; r < 8; ++r) t += red[r][lane];
    bc[(int64_t)f * N + n] = t;
  }
}

__global__ void select_kernel(const double* curves, int k, int q, int m, double* mean, int* best) {
  const int N = q * m;
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    double s = 0.0;
    for (int f = 0; f < k; ++f) s += curves[(int64_t)f * N + e];
    mean[e] = s / (double)k;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < m; o += blockDim.x) {
    int bi = 0;
    double bv = mean[o];
    if (!isnan(bv)) {
      for (int j = 1; j < q; ++j) {
        double v = mean[j * m + o];
        if (isnan(v)) {
          bi = j;
          break;
        }
        if (v < bv) {
          bv = v;
          bi = j;
        }
      }
    }
    best[o] = bi;
  }
}

// C_b = X_b^T Y_b for few outputs (m <= 16), optionally with the Ozaki row exponents of X_b^T
// (E != nullptr): oz_gram_prep_kernel, one pass over X. The FP64 (DMMA) Gram runs it on a side
// stream without E, so C is bit-identical whichever Gram path is taken (given the same scratch:
// the row-chunk count depends on it). scratch: nscratch bytes for the chunk partials (the Gram
// workspace's slice area, overwritten by the slicing afterwards), or nullptr for one chunk.
static int gram_prep(const double* X, int64_t ldx, int64_t rows, int nblocks, int d, const double* Y, int64_t ldy,
                     int m, int* E, int mp, double* C, int* guard, void* scratch, size_t nscratch, cudaStream_t st) {
  RP_REQUIRE(m >= 1 && m <= 16, "gram prep: m=%d outside [1, 16]", m);
  // row chunks: ~4 waves of 1024-column CTAs, as many as the scratch holds (per chunk: the m
  // partial sums, the column maxima, exponent sums and nonzero counts of the range guard)
  const size_t per_chunk = sizeof(double) * (size_t)nblocks * (m + 3) * d;
  int nchunk = 32;
  if (rows < 256) nchunk = 1;
  while (nchunk > 1 && (scratch == nullptr || per_chunk * nchunk > nscratch || rows / nchunk < 64)) nchunk /= 2;
  double* Cp = reinterpret_cast<double*>(scratch);
  double* Mp = Cp ? Cp + (size_t)nblocks * nchunk * m * d : nullptr;
  dim3 grid((d + 1023) / 1024, nchunk, nblocks);
  // X rows streamed by bulk copies when every row segment is 16-byte aligned
  const bool bulk = ((uintptr_t)X & 15) == 0 && ldx % 2 == 0 && d % 2 == 0 && ((uintptr_t)Y & 15) == 0 &&
                    ldy % 2 == 0 && m % 2 == 0;
  switch (m) {
#define RP_GPREP(M)                                                                                            \
  case M:                                                                                                      \
    if (bulk) {                                                                                                \
      cudaFuncSetAttribute(oz_gram_prep_bulk_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                           (int)OZ_GP_SMEM);                                                                   \
      oz_gram_prep_bulk_kernel<M><<<grid, 256, OZ_GP_SMEM, st>>>(X, ldx, rows, d, Y, ldy, m, nchunk, Cp, Mp, mp, \
                                                                 E, C, guard);                                      \
    } else {                                                                                                   \
      oz_gram_prep_kernel<M><<<grid, 256, 0, st>>>(X, ldx, rows, d, Y, ldy, m, nchunk, Cp, Mp, mp, E, C, guard); \
    }                                                                                                          \
    break;
    RP_GPREP(1) RP_GPREP(2) RP_GPREP(3) RP_GPREP(4) RP_GPREP(5) RP_GPREP(6) RP_GPREP(7) RP_GPREP(8)
    RP_GPREP(9) RP_GPREP(10) RP_GPREP(11) RP_GPREP(12) RP_GPREP(13) RP_GPREP(14) RP_GPREP(15) RP_GPREP(16)
#undef RP_GPREP
  }
  RP_LAUNCH_CHECK("gram prep");
  if (nchunk > 1) {
    oz_gram_prep_reduce_kernel<<<dim3((mp + 255) / 256, nblocks), 256, 0, st>>>(Cp, Mp, d, m, nchunk, mp, E, C,
                                                                              nblocks, guard);
    RP_LAUNCH_CHECK("gram prep reduce");
  }
  return RP_OK;
}

}  // namespace rp

using namespace rp;

static inline int grid1d(int64_t n, int b = 256) { return (int)((n + b - 1) / b); }

extern "C" {

int rp_version(void) { return 1; }

long long rp_launch_count(void) { return rp::g_launches.load(); }

const char* rp_last_error(void) { return rp::g_last_error.c_str(); }

long long rp_ozaki_fallbacks(void) {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_oz_fallbacks, sizeof(v)) != cudaSuccess) return -1;
  return (long long)v;
}

int64_t rp_tile_count(int d) {
  int64_t nt = (d + 63) / 64;
  return nt * (nt + 1) / 2;
}

int64_t rp_theta_size(int d, int r) {
#ifdef RP_THETA_GAP  // experiment: fold stride with a gap as large as the data
  return 2 * rp_tile_count(d) * (r + 1) * TILE_PLANE;
#else
  return rp_tile_count(d) * (r + 1) * TILE_PLANE;
#endif
}

size_t rp_gram_workspace_size(int d, int64_t rows_per_block, int nblocks) {
  if (d < 1 || rows_per_block < 1 || nblocks < 1) return 0;
  return oz_workspace_bytes(d, rows_per_block, nblocks);
}

// Side streams (and fork/join events) per calling stream, created with the caller's priority:
// work a call forks off (X^T Y beside the Gram, the Cholesky stream groups) stays independent of
// other callers' and keeps the priority of the stream it was issued on.
struct SideStreams {
  cudaStream_t s[8];
  cudaEvent_t fork, join[8];
};

static SideStreams* side_streams(cudaStream_t caller, int tag) {
  static std::mutex mu;
  static std::map<std::pair<cudaStream_t, int>, SideStreams> by_caller;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(caller, tag);
  auto it = by_caller.find(key);
  if (it == by_caller.end()) {
    int prio = 0;
    cudaStreamGetPriority(caller, &prio);
    SideStreams g{};
    cudaEventCreateWithFlags(&g.fork, cudaEventDisableTiming);
    for (int i = 0; i < 8; ++i) {
      cudaStreamCreateWithPriority(&g.s[i], cudaStreamNonBlocking, prio);
      cudaEventCreateWithFlags(&g.join[i], cudaEventDisableTiming);
    }
    it = by_caller.emplace(key, g).first;
  }
  return &it->second;
}

int rp_gram_blocks(const double* X, int64_t ldx, int64_t rows_per_block, int nblocks, int d, const double* Y,
                   int64_t ldy, int m, double* G, double* C, void* work, void* stream) {
  RP_REQUIRE(d >= 1 && nblocks >= 1 && rows_per_block >= 1 && ldx >= d, "rp_gram_blocks: bad sizes");
  RP_REQUIRE(rows_per_block <= 0x7fffffff, "rp_gram_blocks: block too tall");
  RP_REQUIRE(work == nullptr || ((uintptr_t)work & 15) == 0, "rp_gram_blocks: workspace must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  // Ozaki-scheme tensor-core Gram (int8 tcgen05) when a workspace is given ("gram_dmma" forces FP64 DMMA)
  const bool ozaki = work != nullptr && !g_gram_dmma && oz_supported(d, rows_per_block, nblocks);
  GemmArgs a = gemm_args();
  a.M = a.N = d;
  a.K = (int)rows_per_block;
  a.A = a.B = X;
  a.lda = a.ldb = ldx;
  a.strideA = a.strideB = rows_per_block * ldx;
  a.C = G;
  a.ldc = d;
  a.strideC = (int64_t)d * d;
  a.lower_only = 1;
  const bool want_c = m > 0 && C != nullptr;
  if (want_c) RP_REQUIRE(Y != nullptr && ldy >= m, "rp_gram_blocks: Y");
  // C_b = X_b^T Y_b by the one-pass prep kernel (m <= 16), on either Gram path with the same row
  // chunking (the same scratch), so C is bit-identical whichever path computes G
  const bool prep_c = want_c && m <= 16;
  const size_t ws = work ? rp_gram_workspace_size(d, rows_per_block, nblocks) : 0;
  const size_t eb = OZ_HDR + oz_eb(oz_mp(d), nblocks);
  void* scratch = work ? reinterpret_cast<uint8_t*>(work) + eb : nullptr;
  const size_t nscratch = work ? ws - eb : 0;
  // X_b row-major (rows x d) is the column-major d x rows matrix A_b with lda = ldx: G_b = A_b A_b^T
  const OzIn oin{X, ldx, rows_per_block * ldx, rows_per_block, d, nblocks};
  int rc;
  if (ozaki) {
    int* guard = oz_guard_of(work);
    if (prep_c) {
      // one pass over X for the row exponents (+ range guard) of the slicing and C_b = X_b^T Y_b
      ProfScope prof("gram_prep", st);
      cudaError_t e = cudaMemsetAsync(guard, 0, sizeof(int), st);
      if (e != cudaSuccess) return cuda_status(e, "gram guard");
      rc = gram_prep(X, ldx, rows_per_block, nblocks, d, Y, ldy, m,
                     reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(work) + OZ_HDR), oz_mp(d), C, guard, scratch,
                     nscratch, st);
      if (rc) return rc;
    }
    rc = oz_syrk(oin, G, d, (int64_t)d * d, false, work, st, "oz_syrk", prep_c);
    if (rc) return rc;
    a.run_if_set = guard;  // FP64 fallback when a block is outside the Ozaki range
    rc = gemm<A_KMAJOR, 128, 128, 64, 32, EPI_STORE>(a, nblocks, st, "gram syrk (guarded fallback)");
    if (rc) return rc;
  } else {
    cudaStream_t xs = nullptr;
    cudaEvent_t join = nullptr;
    if (prep_c) {  // X^T Y on a side stream that starts from the same point of `st` as the SYRK
      SideStreams* ss = side_streams(st, 0);
      xs = ss->s[0];
      join = ss->join[0];
      cudaError_t e = cudaEventRecord(ss->fork, st);
      if (e != cudaSuccess) return cuda_status(e, "gram fork");
      cudaStreamWaitEvent(xs, ss->fork, 0);
    }
    rc = gemm<A_KMAJOR, 128, 128, 64, 32, EPI_STORE>(a, nblocks, st, "gram syrk");
    if (rc) return rc;
    if (prep_c) {  // launched after the SYRK so its CTAs fill in next to the SYRK's; joined on `st`
      rc = gram_prep(X, ldx, rows_per_block, nblocks, d, Y, ldy, m, nullptr, d, C, nullptr, scratch, nscratch, xs);
      if (rc) return rc;
      cudaEventRecord(join, xs);
      cudaStreamWaitEvent(st, join, 0);
    }
  }
  if (want_c && !prep_c) {
    GemmArgs b = gemm_args();
    b.M = d;
    b.N = m;
    b.K = (int)rows_per_block;
    b.A = X;
    b.lda = ldx;
    b.strideA = rows_per_block * ldx;
    b.B = Y;
    b.ldb = ldy;
    b.strideB = rows_per_block * ldy;
    b.C = C;
    b.ldc = d;
    b.strideC = (int64_t)d * m;
    rc = gemm<A_KMAJOR, 128, 16, 16, 16, EPI_STORE>(b, nblocks, st, "gram xty");
    if (rc) return rc;
  }
  return RP_OK;
}

int rp_symmetrize(double* G, int d, int64_t stride, int nmat, void* stream) {
  RP_REQUIRE(d >= 1 && nmat >= 1, "rp_symmetrize: bad sizes");
  const int nt = (d + 31) / 32;
  dim3 grid(nt * (nt + 1) / 2, nmat);
  symmetrize_kernel<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(G, d, stride);
  RP_LAUNCH_CHECK("symmetrize");
  return RP_OK;
}

int rp_col_sumsq(const double* Y, int64_t ldy, int64_t rows_per_block, int nblocks, int m, double* yy,
                 void* stream) {
  RP_REQUIRE(m >= 1 && nblocks >= 1 && rows_per_block >= 1, "rp_col_sumsq: bad sizes");
  col_sumsq_kernel<<<dim3(nblocks, m), 256, 0, (cudaStream_t)stream>>>(Y, ldy, rows_per_block, m, yy);
  RP_LAUNCH_CHECK("col_sumsq");
  return RP_OK;
}

int rp_fold_systems(const double* G, const double* C, int nblocks, int d, int m, const int* folds_host, int nf,
                    const double* lams_host, int s, double* A, double* rhs, void* stream) {
  RP_REQUIRE(nf >= 1 && s >= 1, "rp_fold_systems: nf=%d, s=%d", nf, s);
  RP_REQUIRE(nblocks >= 1 && d >= 1 && m >= 0, "rp_fold_systems: nblocks=%d d=%d m=%d", nblocks, d, m);
  for (int f = 0; f < nf; ++f) RP_REQUIRE(folds_host[f] >= -1, "rp_fold_systems: fold %d", folds_host[f]);
  cudaStream_t st = (cudaStream_t)stream;
  const int dp = ((d + 63) / 64) * 64;
  // chunks of <= 64 folds x 32 lambdas per launch (kernel-parameter arrays); each element of the
  // Gram blocks is read once per chunk
  for (int f0 = 0; f0 < nf; f0 += FS_FOLDS) {
    const int nfc = nf - f0 < FS_FOLDS ? nf - f0 : FS_FOLDS;
    FoldSysArgs fa;
    for (int f = 0; f < nfc; ++f) fa.folds[f] = folds_host[f0 + f];
    if (A) {
      for (int s0 = 0; s0 < s; s0 += FS_LAMS) {
        const int sc = s - s0 < FS_LAMS ? s - s0 : FS_LAMS;
        for (int i = 0; i < sc; ++i) fa.lams[i] = lams_host[s0 + i];
        double* Ac = A + (int64_t)f0 * s * d * d;
        const bool pairs = (d & 1) == 0 && (((uintptr_t)G | (uintptr_t)Ac) & 15) == 0;
        if (pairs && nblocks <= 8)
          fold_shift2_kernel<8><<<d, 256, 0, st>>>(G, nblocks, d, sc, s0, s, nfc, fa, Ac);
        else if (pairs && nblocks <= 16)
          fold_shift2_kernel<16><<<d, 256, 0, st>>>(G, nblocks, d, sc, s0, s, nfc, fa, Ac);
        else if (nblocks <= 16)
          fold_shift_kernel<16><<<d, 256, 0, st>>>(G, nblocks, d, sc, s0, s, nfc, fa, Ac);
        else
          fold_shift_kernel<0><<<d, 256, 0, st>>>(G, nblocks, d, sc, s0, s, nfc, fa, Ac);
        RP_LAUNCH_CHECK("fold_shift");
      }
    }
    if (rhs && m > 0) {
      fold_rhs_kernel<<<dim3(grid1d((int64_t)dp * m), nfc), 256, 0, st>>>(C, nblocks, d, dp, m, fa,
                                                                         rhs + (int64_t)f0 * dp * m);
      RP_LAUNCH_CHECK("fold_rhs");
    }
  }
  return RP_OK;
}

// The batch is factored as up to CHOL_GROUPS independent groups on their own streams, so one
// group's latency-bound diagonal kernels (one CTA per matrix) and GEMM tails overlap with the
// other groups' GEMMs. Each matrix sees the same operation sequence whatever the grouping.
static int CHOL_GROUPS = [] {
  const char* e = getenv("RP_CHOL_GROUPS");
  int v = e ? atoi(e) : 4;  // measured at c4: 1 -> 36.7 ms, 2 -> 34.5, 4 -> 33.6, 5 -> 33.5
  return v >= 1 && v <= 8 ? v : 4;
}();

// Trailing updates A22 -= L21 L21^T on the int8 tensor cores (Ozaki) instead of FP64 DMMA
// (measured at c4: factorize 36.2 ms DMMA vs 33.3 ms Ozaki). rp_set_option("chol_ozaki", 0) or
// RP_CHOL_OZAKI=0 keeps them on DMMA.
static bool g_chol_ozaki = env_flag("RP_CHOL_OZAKI", true);

// Per-group slice workspace of the tensor-core trailing update (largest update: d - OB rows).
static size_t potrf_oz_group_bytes(int d, int batch) {
  const int groups = batch < CHOL_GROUPS ? batch : CHOL_GROUPS;
  const int per = (batch + groups - 1) / groups;
  const int rem = d - CHOL_OB;
  if (rem <= 0 || !oz_supported(rem, CHOL_OB, per)) return 0;
  return (oz_workspace_bytes(rem, CHOL_OB, per) + 1023) / 1024 * 1024;
}

size_t rp_potrf_workspace_size(int d, int batch) {
  const size_t inv = ((sizeof(double) * (size_t)batch * CHOL_NB * CHOL_NB) + 1023) / 1024 * 1024;
  const int groups = batch < CHOL_GROUPS ? batch : CHOL_GROUPS;
  // sized for the tensor-core trailing updates whatever "chol_ozaki" is now, so a workspace stays
  // valid if the option changes between the query and the call
  return inv + (size_t)groups * potrf_oz_group_bytes(d, batch);
}

double rp_profile_ms(const char* name) {
  cudaDeviceSynchronize();
  double tot = 0.0;
  std::vector<ProfRec> keep;
  // RP_PROF_TIMELINE=<path>: dump every record (name, stream, start, end in ms from the first)
  if (name == nullptr && !g_prof.empty()) {
    if (const char* path = getenv("RP_PROF_TIMELINE")) {
      if (FILE* f = fopen(path, "w")) {
        for (auto& r : g_prof) {
          float t0 = 0.f, t1 = 0.f;
          cudaEventElapsedTime(&t0, g_prof[0].a, r.a);
          cudaEventElapsedTime(&t1, g_prof[0].a, r.b);
          fprintf(f, "%s %p %.4f %.4f\n", r.name.c_str(), (void*)r.st, t0, t1);
        }
        fclose(f);
      }
    }
  }
  for (auto& r : g_prof) {
    if (name == nullptr || r.name == name) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) tot += ms;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    } else {
      keep.push_back(r);
    }
  }
  g_prof.swap(keep);
  return tot;
}

int rp_set_option(const char* name, int value) {
  RP_REQUIRE(name != nullptr, "rp_set_option: name");
  if (strcmp(name, "chol_ozaki") == 0) {
    g_chol_ozaki = value != 0;
    return RP_OK;
  }
  if (strcmp(name, "gram_dmma") == 0) {
    g_gram_dmma = value != 0;
    return RP_OK;
  }
  if (strcmp(name, "holdout_ozaki") == 0) {
    g_holdout_ozaki = value != 0;
    return RP_OK;
  }
  if (strcmp(name, "solve_cluster") == 0) {
    RP_REQUIRE(value >= 0 && value <= 8 && (value & (value - 1)) == 0,
               "rp_set_option: solve_cluster %d (0/1 = off, 2/4/8 = theta multicast clusters)", value);
    g_solve_cluster = value;
    return RP_OK;
  }
  if (strcmp(name, "solve_lam") == 0) {
    RP_REQUIRE(value >= 0 && value <= 16, "rp_set_option: solve_lam %d outside [0, 16]", value);
    g_solve_lam = value;
    return RP_OK;
  }
  if (strcmp(name, "profile") == 0) {
    g_profile = value != 0;
    return RP_OK;
  }
  return set_error(RP_EINVAL, "rp_set_option: unknown option %s", name);
}

static int potrf_group(double* A, int d, int64_t stride, int batch, int* info, double* inv, void* ozws,
                       cudaStream_t st);

int rp_potrf_batched(double* A, int d, int64_t stride, int batch, int* info, void* work, void* stream) {
  RP_REQUIRE(d >= 1 && batch >= 1 && stride >= (int64_t)d * d, "rp_potrf_batched: bad sizes");
  cudaStream_t st = (cudaStream_t)stream;
  double* inv = (double*)work;
  cudaError_t e = cudaMemsetAsync(info, 0, sizeof(int) * batch, st);
  if (e != cudaSuccess) return cuda_status(e, "potrf memset");
  cudaFuncSetAttribute(potrf_diag_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PD_SMEM);
  const int groups = batch < CHOL_GROUPS ? batch : CHOL_GROUPS;
  // tensor-core trailing updates: one slice workspace per group after inv(L11)
  const size_t ozg = g_chol_ozaki ? potrf_oz_group_bytes(d, batch) : 0;
  uint8_t* ozbase = reinterpret_cast<uint8_t*>(work) +
                    ((sizeof(double) * (size_t)batch * CHOL_NB * CHOL_NB) + 1023) / 1024 * 1024;
  if (groups <= 1 || d <= CHOL_NB) return potrf_group(A, d, stride, batch, info, inv, ozg ? ozbase : nullptr, st);
  // group streams per calling stream: factorizations issued concurrently from different streams
  // (the streamed sweep factors its last fold beside the others) stay independent
  SideStreams* grp = side_streams(st, 1);
  cudaStream_t* gs = grp->s;
  cudaEvent_t fork = grp->fork;
  cudaEvent_t* join = grp->join;
  e = cudaEventRecord(fork, st);
  if (e != cudaSuccess) return cuda_status(e, "potrf fork");
  int b0 = 0;
  for (int g = 0; g < groups; ++g) {
    const int nb = batch / groups + (g < batch % groups ? 1 : 0);
    cudaStreamWaitEvent(gs[g], fork, 0);
    int rc = potrf_group(A + (int64_t)b0 * stride, d, stride, nb, info + b0, inv + (int64_t)b0 * CHOL_NB * CHOL_NB,
                         ozg ? ozbase + g * ozg : nullptr, gs[g]);
    if (rc) return rc;
    cudaEventRecord(join[g], gs[g]);
    cudaStreamWaitEvent(st, join[g], 0);
    b0 += nb;
  }
  return RP_OK;
}

static int potrf_group(double* A, int d, int64_t stride, int batch, int* info, double* inv, void* ozws,
                       cudaStream_t st) {
  // Two-level blocked right-looking factorization. Outer panels of CHOL_OB columns are factored
  // left-looking in 128-column blocks (update from the panel's earlier blocks as one DMMA GEMM,
  // shared-memory diagonal factor + inverse, panel TRSM as a DMMA GEMM against the inverse);
  // the trailing matrix then gets one SYRK with K = CHOL_OB (lower tiles only).
  for (int k0 = 0; k0 < d; k0 += CHOL_OB) {
    const int ob = d - k0 < CHOL_OB ? d - k0 : CHOL_OB;
    for (int k1 = k0; k1 < k0 + ob; k1 += CHOL_NB) {
      const int nb = k0 + ob - k1 < CHOL_NB ? k0 + ob - k1 : CHOL_NB;
      if (k1 > k0) {
        // A[k1:d, k1:k1+nb] -= L[k1:d, k0:k1] * L[k1:k1+nb, k0:k1]^T
        GemmArgs u = gemm_args();
        u.M = d - k1;
        u.N = nb;
        u.K = k1 - k0;
        u.A = A + (int64_t)k0 * d + k1;
        u.B = A + (int64_t)k0 * d + k1;
        u.lda = u.ldb = d;
        u.strideA = u.strideB = stride;
        u.C = A + (int64_t)k1 * d + k1;
        u.ldc = d;
        u.strideC = stride;
        u.alpha = -1.0;
        u.beta = 1.0;
        ProfScope prof("chol_update", st);
        int rc = gemm<A_KMAJOR, 128, 128, 64, 32, EPI_STORE>(u, batch, st, "potrf panel update");
        if (rc) return rc;
      }
      {
        ProfScope prof("chol_diag", st);
        potrf_diag_dmma_kernel<<<batch, PD_THREADS, PD_SMEM, st>>>(A, d, stride, k1, inv, info);
        RP_LAUNCH_CHECK("potrf_diag");
      }
      const int rows = d - k1 - nb;
      if (rows > 0) {
        // L[k1+nb:d, k1:k1+nb] = A[...] * inv(L11)^T   (in place: each CTA owns whole rows, BN >= nb)
        double* L21 = A + (int64_t)k1 * d + k1 + nb;
        GemmArgs t = gemm_args();
        t.M = rows;
        t.N = nb;
        t.K = nb;
        t.A = L21;
        t.lda = d;
        t.strideA = stride;
        t.B = inv;
        t.ldb = CHOL_NB;
        t.strideB = CHOL_NB * CHOL_NB;
        t.C = L21;
        t.ldc = d;
        t.strideC = stride;
        ProfScope prof("chol_trsm", st);
        int rc = gemm<A_KMAJOR, 128, 128, 64, 32, EPI_STORE>(t, batch, st, "potrf trsm");
        if (rc) return rc;
      }
    }
    const int rem = d - k0 - ob;
    if (rem <= 0) break;
    // A22 -= L21 L21^T with K = ob (lower tiles)
    const double* L21 = A + (int64_t)k0 * d + k0 + ob;
    const bool ozaki = ozws && oz_supported(rem, ob, batch);
    if (ozaki) {  // on the int8 tensor cores (Ozaki scheme), FP64 fallback below gated on its range guard
      const OzIn oin{L21, d, stride, ob, rem, batch};
      int rc = oz_syrk(oin, A + (int64_t)(k0 + ob) * d + k0 + ob, d, stride, true, ozws, st, "oz_syrk_chol");
      if (rc) return rc;
    }
    GemmArgs u = gemm_args();
    u.run_if_set = ozaki ? oz_guard_of(ozws) : nullptr;
    u.M = u.N = rem;
    u.K = ob;
    u.A = u.B = L21;
    u.lda = u.ldb = d;
    u.strideA = u.strideB = stride;
    u.C = A + (int64_t)(k0 + ob) * d + k0 + ob;
    u.ldc = d;
    u.strideC = stride;
    u.alpha = -1.0;
    u.beta = 1.0;
    u.lower_only = 1;
    int rc = gemm<A_KMAJOR, 128, 128, 64, 32, EPI_STORE>(u, batch, st, "potrf syrk");
    if (rc) return rc;
  }
  return RP_OK;
}

// partials (ntiles x nf), then P and V for the general kernel
size_t rp_fit_workspace_size(int d, int nf, int s, int r) {
  if (d < 1 || nf < 1 || s < 1 || r < 0) return 0;
  return sizeof(double) * ((size_t)rp_tile_count(d) * nf + 2 * (size_t)s * (r + 1));
}

int rp_fit_tiles(const double* L, int d, int s, int nf, int r, const double* P_host, const double* V_host,
                 double* theta, double* resid, void* work, void* stream) {
  RP_REQUIRE(d >= 1 && nf >= 1 && s >= 1 && r >= 0 && s > r, "rp_fit_tiles: bad sizes d=%d nf=%d s=%d r=%d", d, nf,
             s, r);
  RP_REQUIRE(((uintptr_t)theta & 15) == 0, "rp_fit_tiles: theta must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nt = rp_tile_count(d);
  double* partial = (double*)work;
  if (s <= 32 && r <= 4) {
    FitArgs fa;
    memset(&fa, 0, sizeof(fa));
    for (int p = 0; p <= r; ++p)
      for (int i = 0; i < s; ++i) {
        fa.P[p][i] = P_host[p * s + i];
        fa.V[i][p] = V_host[i * (r + 1) + p];
      }
    const dim3 grid((unsigned)nt, nf);
    const int64_t fs = rp_theta_size(d, r);
    // interior tiles on the predicate-free instantiation (degrees 2 and 3: the BASELINE configs), the rest
    // (diagonal tiles, the last tile row of a padded matrix) on the general one
    const int split = (s <= 8 && (r == 2 || r == 3)) ? 1 : 0;
#define RP_FIT_LAUNCH(SM)                                                                                      \
  do {                                                                                                         \
    if (split && r == 2)                                                                                       \
      fit_tiles_kernel<SM, 1, true, 3><<<grid, FIT_THREADS, 0, st>>>(L, d, s, r, nt, fs, fa, theta, partial, 1); \
    else if (split)                                                                                            \
      fit_tiles_kernel<SM, 1, true, 4><<<grid, FIT_THREADS, 0, st>>>(L, d, s, r, nt, fs, fa, theta, partial, 1); \
    fit_tiles_kernel<SM><<<grid, FIT_THREADS, 0, st>>>(L, d, s, r, nt, fs, fa, theta, partial, split);          \
  } while (0)
    if (s <= 4)
      RP_FIT_LAUNCH(4);
    else if (s <= 6)
      RP_FIT_LAUNCH(6);
    else if (s <= 8)
      RP_FIT_LAUNCH(8);
#undef RP_FIT_LAUNCH
    else
      fit_tiles_kernel<32><<<dim3((unsigned)nt, nf), FIT_THREADS, 0, st>>>(L, d, s, r, nt, rp_theta_size(d, r), fa,
                                                                            theta, partial, 0);
  } else {
    double* Pd = partial + (size_t)nt * nf;
    double* Vd = Pd + (size_t)s * (r + 1);
    const size_t pv = sizeof(double) * (size_t)s * (r + 1);
    cudaError_t e = cudaMemcpyAsync(Pd, P_host, pv, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(Vd, V_host, pv, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_status(e, "rp_fit_tiles: P / V upload");
    fit_tiles_any_kernel<<<dim3((unsigned)nt, nf), 512, 0, st>>>(L, d, s, r, nt, rp_theta_size(d, r), Pd, Vd, theta,
                                                                  partial);
  }
  RP_LAUNCH_CHECK("fit_tiles");
  if (resid) {
    fit_resid_kernel<<<nf, 256, 0, st>>>(partial, nt, resid);
    RP_LAUNCH_CHECK("fit_resid");
  }
  return RP_OK;
}

int rp_eval_materialize(const double* theta, int d, int r, double t, double* L, void* stream) {
  RP_REQUIRE(d >= 1 && r >= 0, "rp_eval_materialize: bad sizes");
  materialize_kernel<<<grid1d((int64_t)d * d), 256, 0, (cudaStream_t)stream>>>(theta, d, r + 1, t, L);
  RP_LAUNCH_CHECK("materialize");
  return RP_OK;
}

int rp_theta_export(const double* theta, int d, int r, const int64_t* perm, int64_t D, double* out, void* stream) {
  RP_REQUIRE(d >= 1 && D >= 1 && r >= 0, "rp_theta_export: bad sizes");
  export_kernel<<<grid1d(D), 256, 0, (cudaStream_t)stream>>>(theta, d, r + 1, perm, D, out);
  RP_LAUNCH_CHECK("theta_export");
  return RP_OK;
}

int rp_theta_import(const double* vec, int d, int r, const int64_t* perm, int64_t D, double* theta, void* stream) {
  RP_REQUIRE(d >= 1 && D >= 1 && r >= 0, "rp_theta_import: bad sizes");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = rp_theta_size(d, r);
  theta_init_kernel<<<grid1d(n), 256, 0, st>>>(theta, d, r + 1, rp_tile_count(d));
  RP_LAUNCH_CHECK("theta_init");
  import_kernel<<<grid1d(D), 256, 0, st>>>(vec, d, r + 1, perm, D, rp_tile_count(d), theta);
  RP_LAUNCH_CHECK("theta_import");
  return RP_OK;
}

static int64_t holdout_mt(int64_t n_val, int d) {
  const int64_t mt_direct = (n_val + 127) / 128, mt_gram = 2 * ((d + 127) / 128);  // 2 passes (Ozaki)
  return mt_direct > mt_gram ? mt_direct : mt_gram;
}

// Hold-out workspace: [partials nf x mt x N][bc nf x N] [repair: count, list nf x N, partials
// nf x N x REP_CHUNKS] [Ozaki slices (Gram form on the tensor cores)].
static size_t holdout_base_bytes(int64_t n_val, int d, int64_t N, int nf) {
  return (sizeof(double) * (size_t)(nf * holdout_mt(n_val, d) * N + nf * N) + 1023) / 1024 * 1024;
}
static size_t holdout_rep_list_bytes(int64_t N, int nf) {  // count (16 bytes) + list, 16-byte aligned
  return (16 + sizeof(int) * (size_t)nf * N + 15) / 16 * 16;
}
static size_t holdout_rep_bytes(int64_t N, int nf) {
  return (holdout_rep_list_bytes(N, nf) + sizeof(double) * (size_t)nf * N * REP_CHUNKS + 1023) / 1024 * 1024;
}

// per-fold 128-column tiles whose solution vectors are out of the tensor-core range (Ozaki hold-out)
static size_t holdout_mask_bytes(int64_t N, int nf) {
  return (sizeof(int) * (size_t)nf * ((N + 127) / 128) + 1023) / 1024 * 1024;
}

size_t rp_holdout_workspace_size(int64_t n_val, int d, int q, int m, int nf) {
  const int64_t N = (int64_t)q * m;
  const bool oz = g_holdout_ozaki && oz_holdout_supported(d, N, nf);
  return holdout_base_bytes(n_val, d, N, nf) + holdout_rep_bytes(N, nf) + holdout_mask_bytes(N, nf) +
         (oz ? oz_holdout_workspace(d, N, nf, false) : 0);
}

int rp_holdout_direct(const double* Xval, int64_t ldx, int64_t fold_stride_rows, int64_t n_val, int d,
                      const double* Yval, int64_t ldy, int m, const double* W, int64_t ldw, int64_t w_fold_stride,
                      int q, int nf, int metric, double* curves, void* work, void* stream) {
  RP_REQUIRE(n_val >= 1, "rp_holdout_direct: empty validation set");
  RP_REQUIRE(metric == RP_METRIC_RMSE || metric == RP_METRIC_MISCLASS, "rp_holdout_direct: metric %d", metric);
  RP_REQUIRE(n_val <= 0x7fffffff && (int64_t)q * m <= 0x7fffffff, "rp_holdout_direct: sizes");
  cudaStream_t st = (cudaStream_t)stream;
  const int N = q * m;
  double* partial = (double*)work;
  GemmArgs a = gemm_args();
  a.M = (int)n_val;
  a.N = N;
  a.K = d;
  a.A = Xval;
  a.lda = ldx;
  a.strideA = fold_stride_rows * ldx;
  a.B = W;
  a.ldb = ldw;
  a.strideB = w_fold_stride;
  a.Y = Yval;
  a.ldy = ldy;
  a.strideY = fold_stride_rows * ldy;
  a.ycols = m;
  a.partial = partial;
  int rc = metric == RP_METRIC_RMSE ? gemm<A_MMAJOR, 128, 128, 64, 32, EPI_SSE>(a, nf, st, "holdout sse")
                                    : gemm<A_MMAJOR, 128, 128, 64, 32, EPI_MIS>(a, nf, st, "holdout mis");
  if (rc) return rc;
  const int mtiles = (int)((n_val + 127) / 128);
  holdout_finish_kernel<<<dim3(grid1d(N), nf), 256, 0, st>>>(partial, mtiles, N, m, n_val, metric, nullptr, nullptr,
                                                             1.0, curves, nullptr, nullptr);
  RP_LAUNCH_CHECK("holdout finish");
  return RP_OK;
}

int rp_holdout_gram(double* Gf, int64_t g_stride, const double* Cf, int64_t c_stride, const double* yy,
                    int64_t n_val, int d, int m, const double* W, int64_t ldw, int64_t w_fold_stride, int q, int nf,
                    const double* Xval, int64_t ldx, int64_t fold_stride_rows, const double* Yval, int64_t ldy,
                    double* curves, void* work, void* stream) {
  RP_REQUIRE(n_val >= 1, "rp_holdout_gram: empty validation set");
  RP_REQUIRE(((uintptr_t)work & 15) == 0, "rp_holdout_gram: workspace must be 16-byte aligned");
  RP_REQUIRE(Xval == nullptr || (Yval != nullptr && ldx >= d && ldy >= m), "rp_holdout_gram: Xval / Yval");
  cudaStream_t st = (cudaStream_t)stream;
  const int N = q * m;
  const int mtiles = (d + 127) / 128;
  uint8_t* w8 = reinterpret_cast<uint8_t*>(work);
  double* partial = reinterpret_cast<double*>(w8);
  double* bc = partial + (size_t)nf * holdout_mt(n_val, d) * N;
  w8 += holdout_base_bytes(n_val, d, N, nf);
  int* rep_count = reinterpret_cast<int*>(w8);
  int* rep_list = rep_count + 4;
  double* rep_part = reinterpret_cast<double*>(w8 + holdout_rep_list_bytes(N, nf));
  w8 += holdout_rep_bytes(N, nf);
  int* col_mask = reinterpret_cast<int*>(w8);
  w8 += holdout_mask_bytes(N, nf);
  cudaError_t e = cudaMemsetAsync(rep_count, 0, sizeof(int), st);
  if (e != cudaSuccess) return cuda_status(e, "holdout repair count");

  GemmArgs a = gemm_args();
  a.M = d;
  a.N = N;
  a.K = d;
  a.A = Gf;
  a.lda = d;
  a.strideA = g_stride;
  a.B = W;
  a.ldb = ldw;
  a.strideB = w_fold_stride;
  a.Y = W;
  a.ldy = ldw;
  a.strideY = w_fold_stride;
  a.ycols = N;
  a.partial = partial;
  // w^T G w = 2 w^T T w with T = strict_lower(G) + diag(G)/2: half the GEMM, only G's lower triangle read
  a.tri_a = gemm_vec2(a, A_KMAJOR) ? 1 : 0;
  int rc;
  if (a.tri_a && g_holdout_ozaki && oz_holdout_supported(d, N, nf)) {
    // T W on the int8 tensor cores (partials [f][mtiles][N]); the DMMA product behind it runs in full
    // when T is out of the tensor-core range, and otherwise only for the 128-column tiles holding a
    // solution vector out of range (c5's largest lambdas: ~8% of the columns), overwriting their partials
    SideStreams* ss = side_streams(st, 2);
    rc = oz_holdout(Gf, g_stride, d, W, ldw, w_fold_stride, N, nf, partial, w8, col_mask, st, ss->s[0], ss->fork,
                    ss->join[0]);
    if (rc) return rc;
    a.run_if_set = oz_guard_of(w8);
    a.tile_mask = col_mask;
  } else if (!a.tri_a) {  // the full product reads both triangles: fill G_f's upper triangle first
    const int nt = (d + 31) / 32;
    const int nmat = g_stride == 0 ? 1 : nf;
    symmetrize_kernel<<<dim3(nt * (nt + 1) / 2, nmat), dim3(32, 8), 0, st>>>(Gf, d, g_stride);
    RP_LAUNCH_CHECK("holdout symmetrize");
  }
  {
    ProfScope prof(a.run_if_set ? "holdout_gemm_fallback" : "holdout_gemm", st);
    rc = gemm<A_KMAJOR, 128, 128, 64, 32, EPI_DOTB>(a, nf, st, "holdout gram");
  }
  if (rc) return rc;
  holdout_bc_kernel<<<dim3((N + 31) / 32, nf), 256, 0, st>>>(W, ldw, w_fold_stride, Cf, c_stride, d, m, N, bc);
  RP_LAUNCH_CHECK("holdout bc");
  holdout_finish_kernel<<<dim3(grid1d(N), nf), 256, 0, st>>>(partial, mtiles, N, m, n_val, RP_METRIC_RMSE, yy, bc,
                                                             a.tri_a ? 2.0 : 1.0, curves,
                                                             Xval ? rep_count : nullptr, rep_list);
  RP_LAUNCH_CHECK("holdout gram finish");
  if (Xval != nullptr) {  // cancellation repair (no work unless a column was listed)
    const size_t wsm = sizeof(double) * (size_t)d;
    const int in_smem = wsm <= 192 * 1024 ? 1 : 0;
    if (in_smem)
      cudaFuncSetAttribute(holdout_repair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
    holdout_repair_kernel<<<dim3(REP_CHUNKS, 32), 256, in_smem ? wsm : 0, st>>>(
        Xval, ldx, fold_stride_rows, n_val, d, Yval, ldy, m, W, ldw, w_fold_stride, N, rep_count, rep_list, in_smem,
        rep_part);
    RP_LAUNCH_CHECK("holdout repair");
    holdout_repair_finish_kernel<<<8, 256, 0, st>>>(rep_count, rep_list, rep_part, n_val, curves);
    RP_LAUNCH_CHECK("holdout repair finish");
  }
  return RP_OK;
}

int rp_select(const double* curves, int k, int q, int m, double* mean, int* best, void* stream) {
  RP_REQUIRE(k >= 1 && q >= 1 && m >= 1, "rp_select: bad sizes");
  select_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(curves, k, q, m, mean, best);
  RP_LAUNCH_CHECK("select");
  return RP_OK;
}

}  // extern "C"
