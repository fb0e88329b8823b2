// Warp-specialised fused evaluate + solve (the path the BASELINE shapes take; rp_solve.cuh keeps
// the generic runtime-shaped kernel).
//
// Same mathematics and the same deterministic per-lambda arithmetic as eval_solve_kernel, but:
//  * warp 8 is a producer: it streams every 16-column (fwd) / 16-row (bwd) slab of the
//    coefficient tiles -- including the four slabs of the diagonal tile -- and the matching
//    16 rows of the already solved W through a STAGES-deep ring with 1-D bulk async copies
//    (cp.async.bulk + mbarrier complete_tx). It only waits for W_J when it reaches the first
//    slab that needs it (a row-done mbarrier), so the next row streams in while the consumers
//    finish the current one;
//  * warps 0-7 (4 row groups x 2 lambda groups) only evaluate + DMMA; there is no block-wide
//    barrier in the off-diagonal loop;
//  * the diagonal tile is processed as four 16-row sub-blocks: the owning row group solves its
//    16 x 16 triangle per (lambda, output) column, then the other row groups apply the
//    sub-block to their accumulators with DMMA (B fragments from the solved rows in smem).
#pragma once
#include "rp_solve.cuh"

namespace rp {

RP_DEVINL void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

// acc += L(rows of this warp, slab k) * Wslab(k, cols) for all lambdas of this warp.
// A force-inlined function (not a lambda capturing the accumulator arrays by reference), so the
// accumulators and t values stay in registers.
template <int NT, int REM, int P, int LH, int LC>
RP_DEVINL void ws_slab_update(double (&acc)[LH][2][NT > 0 ? NT : 1][2], double (&accx)[LH][2][REM > 0 ? REM : 1],
                              const double (&tl)[LH], const double* __restrict__ T, const double* __restrict__ wbase,
                              int S, int m, int rg, int lg, int g, int t) {
  constexpr int NTA = NT > 0 ? NT : 1;
  constexpr int REMA = REM > 0 ? REM : 1;
  constexpr bool REM2 = (REM % 2) == 0;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int k = ks * 4 + t;
    double th[2][P];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int row = rg * 16 + mt * 8 + g;
#pragma unroll
      for (int p = 0; p < P; ++p) th[mt][p] = T[p * FWD_SLAB + k * 68 + row];
    }
    const double* wrow = wbase + k * S;
#pragma unroll
    for (int i = 0; i < LH; ++i) {
      const int l = lg * LH + i;
      if (l < LC) {
        double b[NTA];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = wrow[l * m + j * 8 + g];
        double rv[REMA];
        if (REM2) {
#pragma unroll
          for (int c = 0; c < REM; c += 2) {
            const double2 v2 = *reinterpret_cast<const double2*>(wrow + l * m + NT * 8 + c);
            rv[c] = v2.x;
            rv[c + 1] = v2.y;
          }
        } else {
#pragma unroll
          for (int c = 0; c < REM; ++c) rv[c] = wrow[l * m + NT * 8 + c];
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          double av = th[mt][P - 1];
#pragma unroll
          for (int p = P - 2; p >= 0; --p) av = fma(av, tl[i], th[mt][p]);
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma884(acc[i][mt][j][0], acc[i][mt][j][1], av, b[j]);
#pragma unroll
          for (int c = 0; c < REM; ++c) accx[i][mt][c] = fma(av, rv[c], accx[i][mt][c]);
        }
      }
    }
  }
}

template <int NT, int REM, int P, int LC, int STAGES, bool BWD>
// 288 threads = 9 warps: one SM sub-partition holds 3 of them, so the register file caps a thread
// at 168 registers.
__global__ void __launch_bounds__(288, 1) eval_solve_ws_kernel(SolveArgs a) {
  constexpr int LG = 2;
  constexpr int LH = (LC + LG - 1) / LG;
  constexpr int REMA = REM > 0 ? REM : 1;
  constexpr int NTA = NT > 0 ? NT : 1;
  constexpr int STAGE_T = P * FWD_SLAB;  // both directions use the [k][68] slab layout
  extern __shared__ __align__(16) double smem[];
  const int S = a.S, m = a.m;
  const int stageW = 16 * S;
  const int stage = STAGE_T + stageW;
  double* sR = smem + STAGES * stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sR + 64 * S);
  uint64_t* empty = full + STAGES;
  uint64_t* rowbar = empty + STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fold = blockIdx.x / a.chunks, chunk = blockIdx.x % a.chunks;
  const int l0 = min(chunk * LC, a.q - LC);
  const double* theta = a.theta + fold * a.theta_fold_stride;
  double* W = a.W + fold * a.w_fold_stride;
  double* Wc = a.Wc + (int64_t)blockIdx.x * (a.nt * 64) * S;  // this CTA's private rows
  const int cw = LC * m;
  const int64_t wcol0 = (int64_t)l0 * m;
  const int nt = a.nt;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    mbar_init(rowbar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 8) {
    // ================= producer =================
    int it = 0, done = 0;
    auto load = [&](const double* tile, int kq, int J) {  // J < 0: diagonal slab (no W rows)
      const int st = it % STAGES;
      mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
      double* dT = smem + st * stage;
      double* dW = dT + STAGE_T;
      const uint32_t bytes = (uint32_t)(P * FWD_SLAB * 8) + (J >= 0 ? (uint32_t)(16 * S * 8) : 0u);
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[st], bytes);
        // one contiguous copy per plane: 16 columns (fwd, column-major copy) or 16 rows
        // (bwd, row-major copy) of a padded 64 x 68 plane
        for (int p = 0; p < P; ++p)
          bulk_g2s(dT + p * FWD_SLAB, tile + p * TILE_PLANE + kq * 16 * TILE_LD, (uint32_t)(FWD_SLAB * 8), &full[st]);
        if (J >= 0) bulk_g2s(dW, Wc + (int64_t)(J * 64 + kq * 16) * S, (uint32_t)(16 * S * 8), &full[st]);
      }
      __syncwarp();
      ++it;
    };
    const double* thb = theta + (BWD ? a.theta_bwd_off : 0);
    for (int step = 0; step < nt; ++step) {
      const int I = BWD ? (nt - 1 - step) : step;
      const int nJ = BWD ? (nt - 1 - I) : I;
      for (int jj = 0; jj < nJ; ++jj) {
        const int J = BWD ? (I + 1 + jj) : jj;
        const int need = BWD ? (nt - 1 - J) : J;  // completion order index of row J
        while (done <= need) {
          mbar_wait(rowbar, done & 1);
          ++done;
        }
        const double* tile = thb + (int64_t)(BWD ? tile_index(J, I) : tile_index(I, J)) * P * TILE_PLANE;
        for (int kq = 0; kq < 4; ++kq) load(tile, kq, J);
      }
      const double* dtile = thb + (int64_t)tile_index(I, I) * P * TILE_PLANE;
      for (int q = 0; q < 4; ++q) load(dtile, BWD ? 3 - q : q, -1);
    }
    return;
  }

  // ================= consumers =================
  const int g = lane >> 2, t = lane & 3;
  const int rg = warp & 3, lg = warp >> 2;
  double tl[LH];
#pragma unroll
  for (int i = 0; i < LH; ++i) {
    const int l = lg * LH + i;
    tl[i] = (l < LC) ? a.tvals[l0 + l] : 0.0;
  }
  double acc[LH][2][NTA][2];
  double accx[LH][2][REMA];

  int it = 0;
  for (int step = 0; step < nt; ++step) {
    const int I = BWD ? (nt - 1 - step) : step;
    const int nJ = BWD ? (nt - 1 - I) : I;
    const int rowI = I * 64;
#pragma unroll
    for (int i = 0; i < LH; ++i)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
        for (int j = 0; j < NTA; ++j) acc[i][mt][j][0] = acc[i][mt][j][1] = 0.0;
#pragma unroll
        for (int c = 0; c < REMA; ++c) accx[i][mt][c] = 0.0;
      }
    // ---- off-diagonal tiles
    for (int s = 0; s < 4 * nJ; ++s, ++it) {
      const int st = it % STAGES;
      mbar_wait(&full[st], (it / STAGES) & 1);
      const double* T = smem + st * stage;
      ws_slab_update<NT, REM, P, LH, LC>(acc, accx, tl, T, T + STAGE_T, S, m, rg, lg, g, t);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // ---- diagonal tile, four 16-row sub-blocks
    for (int q = 0; q < 4; ++q, ++it) {
      const int kq = BWD ? 3 - q : q;
      const int st = it % STAGES;
      mbar_wait(&full[st], (it / STAGES) & 1);
      const double* T = smem + st * stage;
      if (rg == kq) {
        // R = base - acc for this row group's 16 rows into sR
#pragma unroll
        for (int i = 0; i < LH; ++i) {
          const int l = lg * LH + i;
          if (l < LC) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              const int row = rg * 16 + mt * 8 + g;
#pragma unroll
              for (int c = 0; c < REM; ++c) {
                double v = accx[i][mt][c];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                accx[i][mt][c] = v;
              }
#pragma unroll
              for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const int col = j * 8 + 2 * t + h;
                  const double base = BWD ? Wc[(int64_t)(rowI + row) * S + l * m + col]
                                          : a.rhs[fold * a.rhs_fold_stride + (int64_t)(rowI + row) * m + col];
                  sR[row * S + l * m + col] = base - acc[i][mt][j][h];
                }
              if (t == 0) {
#pragma unroll
                for (int c = 0; c < REM; ++c) {
                  const int col = NT * 8 + c;
                  const double base = BWD ? Wc[(int64_t)(rowI + row) * S + l * m + col]
                                          : a.rhs[fold * a.rhs_fold_stride + (int64_t)(rowI + row) * m + col];
                  sR[row * S + l * m + col] = base - accx[i][mt][c];
                }
              }
            }
          }
        }
      }
      named_bar_sync(1, 256);  // R rows of sub-block kq are in sR
      // 16 x 16 triangular solve, all 256 consumer threads: 4 lanes (t) per (lambda, output)
      // column split the dot products (k = t mod 4) and combine them with two shuffles
      for (int c0 = 0; c0 < cw; c0 += 64) {
        const int c = c0 + (tid >> 2);
        const bool live = c < cw;
        const int cc = live ? c : cw - 1;
        const int l = cc / m;
        const double tv = a.tvals[l0 + l];
        double* x = sR + (kq * 16) * S + cc;
        auto Lval = [&](int i, int k) {  // L(16kq + i, 16kq + k) at lambda l
          // fwd slab: [col - 16kq][row]; bwd slab (transposed copy): [row - 16kq][col]
          const int off = BWD ? i * 68 + kq * 16 + k : k * 68 + kq * 16 + i;
          double v = T[(P - 1) * FWD_SLAB + off];
#pragma unroll
          for (int p = P - 2; p >= 0; --p) v = fma(v, tv, T[p * FWD_SLAB + off]);
          return v;
        };
        double xk[4];  // x_k for k = 4j + t
        bool singular = false;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
          const int i = BWD ? 15 - s : s;
          double part = 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = 4 * j + t;
            const bool use = BWD ? (k > i) : (k < i);
            if (use) part = fma(BWD ? Lval(k, i) : Lval(i, k), xk[j], part);
          }
          part += __shfl_xor_sync(0xffffffffu, part, 1);
          part += __shfl_xor_sync(0xffffffffu, part, 2);
          const double lii = Lval(i, i);
          if (!BWD && rowI + kq * 16 + i < a.d && !(fabs(lii) >= 1e-12)) singular = true;
          const double xi = (x[i * S] - part) / lii;
          if ((i & 3) == t) {
            xk[i >> 2] = xi;
            if (live) x[i * S] = xi;
          }
        }
        if (!BWD && singular && live && t == 0 && (c % m) == 0) a.flags[fold * a.q + l0 + l] = 1;
      }
      named_bar_sync(1, 256);  // the solved 16 rows are visible to every row group
      if (BWD ? (rg < kq) : (rg > kq))
        ws_slab_update<NT, REM, P, LH, LC>(acc, accx, tl, T, sR + (kq * 16) * S, S, m, rg, lg, g, t);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // ---- row I solved: publish W_I rows, then signal the producer
    named_bar_sync(1, 256);
    for (int i = warp; i < 64; i += 8) {
      double* dc = Wc + (int64_t)(rowI + i) * S;
      for (int c = lane; c < cw; c += 32) dc[c] = sR[i * S + c];
      if (BWD) {  // the final solution also goes to the caller's row-major W
        double* dst = W + (int64_t)(rowI + i) * a.ldw + wcol0;
        for (int c = lane; c < cw; c += 32) dst[c] = sR[i * S + c];
      }
    }
    fence_proxy_async_global();
    named_bar_sync(1, 256);
    if (tid == 0) mbar_arrive(rowbar);
  }
}

template <int P, int STAGES, bool BWD>
constexpr size_t solve_ws_smem_doubles(int S) {
  return (size_t)STAGES * (P * FWD_SLAB + 16 * S) + 64 * (size_t)S + 16;
}

template <int NT, int REM, int P, int LC, int STAGES, bool BWD>
int launch_solve_ws_pass(const SolveArgs& a, int grid, cudaStream_t st) {
  auto k = eval_solve_ws_kernel<NT, REM, P, LC, STAGES, BWD>;
  const size_t smem = sizeof(double) * solve_ws_smem_doubles<P, STAGES, BWD>(a.S);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, 288, smem, st>>>(a);
  RP_LAUNCH_CHECK(BWD ? "eval_solve_ws bwd" : "eval_solve_ws fwd");
  return RP_OK;
}

}  // namespace rp
