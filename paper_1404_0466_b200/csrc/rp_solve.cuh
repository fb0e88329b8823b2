// (5) Fused evaluate + solve: for every local fold f and every grid lambda_j,
//       W_f(:, j) = (L_f(t_j) L_f(t_j)^T)^{-1} rhs_f,   L_f(t) = sum_p theta_{f,p} t^p,
// without ever materializing L_f(t_j). Replaces pichol.eval_vector (pichol.py:143-151)
// + trivec.unvectorize (trivec.py:150-162) + the singular check (ridge.py:88-89) +
// linalg.solve_chol (linalg.py:104-128), once per lambda in the reference's q-lambda loop
// (cvsearch.py:232-239).
//
// Design (B200, FP64 = one DMMA/DFMA datapath, 64 MAC/clk/SM):
//  * One CTA owns a chain (fold f, chunk of <= 16 lambdas) and runs the blocked, left-looking
//    forward substitution over 64-row tile rows (kernel BWD=false) and, in a second launch, the
//    backward substitution with the transposed tiles (BWD=true). No inter-CTA dependencies,
//    so the result is deterministic and independent of the grid.
//  * Off-diagonal tiles are streamed as 16-column (fwd) / 16-row (bwd) slabs through a 3-stage
//    cp.async ring together with the matching 16 rows of the already-solved W.
//  * Per slab each warp owns 8 output rows. For each k-step it loads the P coefficient planes
//    of its A fragment once, evaluates L(t_l) for every lambda of the chunk with Horner in
//    registers (DFMA), and feeds it to mma.m8n8k4.f64 against W_J(lambda) (N = 8 outputs per
//    DMMA). The m % 8 leftover outputs are done with DFMA on the same evaluated fragment and
//    reduced across the 4 k-lanes at the end of the row (no N padding waste).
//  * The 64 x 64 diagonal tile is solved in shared memory, one thread per (lambda, output)
//    column, reading its coefficients through the read-only path (uniform addresses ->
//    broadcast). The diagonal pass also raises the SingularInterpolant flag.
#pragma once
#include <cstdio>

#include "rp_common.cuh"

namespace rp {

// RP_SOLVE_PROF (experiments only): per-phase clock64 totals of the diagonal steps of CTA 0,
// printed when the kernel ends.
#ifdef RP_SOLVE_PROF
#define RP_SP_MARK(k)                              \
  do {                                             \
    if (tid == 0) {                                \
      const long long _t = clock64();              \
      sp_acc[k] += _t - sp_last;                   \
      sp_last = _t;                                \
    }                                              \
  } while (0)
#else
#define RP_SP_MARK(k) \
  do {                \
  } while (0)
#endif

constexpr int SOLVE_LC = 16;          // max lambdas per CTA (specialised kernels)
constexpr int SOLVE_LC_GENERIC = 8;   // max lambdas per CTA (generic kernel)
constexpr int SOLVE_PMAX = 5;    // max polynomial planes (degree <= 4)
constexpr int SOLVE_STAGES = 3;
constexpr int FWD_SLAB = 16 * 68;   // per plane: 16 columns x 64 rows (stride 68), one bulk copy
constexpr int BWD_SLAB = 64 * 16;   // per plane: 64 columns x 16 rows, one 2-D TMA box, 128-byte swizzle

struct SolveArgs {
  CUtensorMap tmb;  // backward slabs: 2-D view {68, nf * theta_fold_stride / 68} of the tile layout
  const double* theta;
  int64_t theta_fold_stride;
  const double* rhs;
  int64_t rhs_fold_stride;
  double* W;
  int64_t ldw, w_fold_stride;
  const double* tvals;
  int* flags;
  int flag_stride;  // flags of fold f at flags + f * flag_stride (q unless a caller splits the grid)
  int q, m, d, nt, P, lam_per_cta, chunks, S;
  int chunks_real;  // chunks that cover the grid; chunks (>= chunks_real, a multiple of cl) pads the
                    // last cluster of a fold with copies of its last chunk (bit-identical duplicate writes)
  int cl;           // CTAs per cluster: consecutive chunks of one fold; rank 0 multicasts the theta slabs
  int chunk0;       // first chunk index of this launch (a tail launch covers only a fold's last chunk)
  int njobs;        // (fold, chunk) chains of this launch; CTA b runs jobs b, b + gridDim.x, ... in turn
  double* Wc;      // chunk-private rows of the solution (dp x S per CTA)
  int64_t ntiles;  // 64 x 64 tiles per fold
};

RP_DEVINL int tile_index(int I, int J) { return I * (I + 1) / 2 + J; }

// NT: number of 8-wide DMMA output tiles, REM: leftover outputs (m = 8 NT + REM).
// PT / LCT: compile-time planes / lambdas per CTA (0 = runtime, the generic instantiation).
// With LCT > 0 every chunk is full: the last chunk starts at q - LCT and recomputes a few
// lambdas of its neighbour; per-lambda arithmetic is independent of the chunk, so the
// duplicated writes are bit-identical.
//
// Warp layout: 8 warps = 4 row groups (16 rows = 2 DMMA m-tiles each) x 2 lambda groups, so
// every W fragment loaded from shared memory feeds two DMMAs and every coefficient fragment
// is evaluated for half of the chunk's lambdas.
// Small chunks (LCT <= 4: little arithmetic per slab, e.g. one fold per GPU) add a producer warp that
// streams the slabs, so no compute warp stalls on refills (the per-slab issue cost is not hidden there).
inline constexpr bool solve_pw_lam(int lam) { return lam > 0 && lam <= 4; }
template <int LCT>
constexpr bool solve_pw() {
  return solve_pw_lam(LCT);
}

template <int NT, int REM, int PT, int LCT, int LG, int STG, bool BWD>
__global__ void __launch_bounds__(128 * LG + (solve_pw<LCT>() ? 32 : 0), 1)
    eval_solve_kernel(const __grid_constant__ SolveArgs a) {
  constexpr int NTH = 128 * LG;  // 4 row groups x LG lambda groups of compute warps
  constexpr bool PW = solve_pw<LCT>();
  constexpr int LC = LCT ? LCT : SOLVE_LC_GENERIC;
  constexpr int LH = (LC + LG - 1) / LG;
  constexpr int PM = PT ? PT : SOLVE_PMAX;
  constexpr int REMA = REM > 0 ? REM : 1;
  constexpr int NTA = NT > 0 ? NT : 1;
  constexpr bool REM2 = (REM % 2) == 0;
  extern __shared__ __align__(16) double smem_raw[];
  // backward pass: 1 KB-aligned base, the slabs land with the 128-byte TMA swizzle (8-row atoms of 1 KB)
  // (pointer arithmetic on the shared array, so the compiler keeps shared-memory loads)
  double* smem = BWD ? smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / 8 : smem_raw;
  // diagonal-block helpers (static): packed lower index -> (row, col) of a 16 x 16 block, and the
  // chunk's t values
  __shared__ uint8_t s_pi[136], s_pj[136];
  __shared__ double s_tv[LCT ? LCT : SOLVE_LC_GENERIC];
  const int P = PT ? PT : a.P;
  const int S = a.S, m = a.m;
  const int stageT = P * (BWD ? BWD_SLAB : FWD_SLAB);
  const int stageW = 16 * S;
  double* sT = smem;
  double* sW = smem + STG * stageT;
  const int ring = STG * (stageT + stageW);
  const int LCr = LCT ? LCT : a.lam_per_cta;
  const int diagw = P * TILE_PLANE + LCr * (16 * 17 + 16);  // theta_II + evaluated block + pivots
  double* sR = smem + (ring > diagw ? ring : diagw);
  uint64_t* full = reinterpret_cast<uint64_t*>(sR + 64 * S);  // per stage, + [STG] diagonal tile
  uint64_t* empty = full + STG + 1;                             // per stage: all warps released it
  uint64_t* cempty = empty + STG;  // per stage, used in cluster rank 0: all warps of the cluster released it

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int rg = warp & 3, lg = warp >> 2;  // row group, lambda group
  // tile row of this lane's DMMA row g in m-tile mt (the accumulators follow the A fragments): fwd
  // pairs the two m-tiles' rows (16-byte loads of adjacent rows), bwd spreads the rows of each
  // quarter-warp over both halves of the 128-byte swizzle atom (conflict-free 16-byte loads)
  auto slab_row = [&](int mt) {
    return BWD ? rg * 16 + mt * 8 + (g >> 1) + 4 * (g & 1) : rg * 16 + 2 * g + mt;
  };
  const int cl = a.cl;
  const uint32_t rank = cl > 1 ? cluster_rank() : 0;
  if (tid == 0) {
    for (int i = 0; i <= STG; ++i) mbar_init(&full[i], 1);
    for (int i = 0; i < STG; ++i) mbar_init(&empty[i], NTH / 32);
    for (int i = 0; i < STG; ++i) mbar_init(&cempty[i], NTH / 32 * cl);
    fence_mbar_init();
  }
  __syncthreads();
  if (cl > 1) cluster_sync();  // every CTA's barriers are initialised before any remote arrival
  const uint32_t cempty0 = cl > 1 ? cluster_addr(cempty, 0) : 0;  // rank 0's cluster-release barriers
  int it0 = 0;      // slabs consumed by earlier rows (stage / phase bookkeeping)
  int diag_it = 0;  // diagonal tiles staged so far (phase of full[STG])
  auto csync = [&]() {  // barrier of the compute warps only (the producer warp never joins it)
    if (PW) named_bar_sync(1, NTH);
    else __syncthreads();
  };

#ifdef RP_SOLVE_PROF
  long long sp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, sp_last = clock64();
#endif
  for (int e = tid; e < 136; e += NTH) {
    int i = 0;
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    s_pi[e] = (uint8_t)i;
    s_pj[e] = (uint8_t)(e - i * (i + 1) / 2);
  }
  // A CTA runs its jobs (fold, chunk) one after the other (one job per CTA unless the launch is a tail
  // launch with fewer CTAs than jobs); barrier phases and the ring position carry over.
#pragma unroll 1
  for (int job = blockIdx.x; job < a.njobs; job += gridDim.x) {
  const bool last_job = job + (int)gridDim.x >= a.njobs;
  const int fold = job / a.chunks, chunk = a.chunk0 + min(job % a.chunks, a.chunks_real - 1);
  const int l0 = LCT ? min(chunk * LCT, a.q - LCT) : chunk * a.lam_per_cta;
  const int nl = LCT ? LCT : min(a.lam_per_cta, a.q - l0);
  if (nl <= 0) continue;  // (never: every chunk of a plan holds a lambda)
  const double* theta = a.theta + fold * a.theta_fold_stride;
  double* W = a.W + fold * a.w_fold_stride;
  double* Wc = a.Wc + (int64_t)job * (a.nt * 64) * S;  // this job's private solve rows
  const int cw = nl * m;  // valid chunk columns
  const int64_t wcol0 = (int64_t)l0 * m;
  for (int l = tid; l < nl; l += NTH) s_tv[l] = a.tvals[l0 + l];
  double tl[LH];
#pragma unroll
  for (int i = 0; i < LH; ++i) {
    const int l = lg * LH + i;
    tl[i] = (l < nl) ? a.tvals[l0 + l] : 0.0;
  }

  double acc[LH][2][NTA][2];
  double accx[LH][2][REMA];

  for (int step = 0; step < a.nt; ++step) {
    const int I = BWD ? (a.nt - 1 - step) : step;
    const int nslab = 4 * (BWD ? (a.nt - 1 - I) : I);
    if (tid == 0) {  // warm L2 with this row's diagonal tile: its copy at the end of the row then hits
      const double* dt = theta + (int64_t)tile_index(I, I) * P * TILE_PLANE;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(dt), "r"((uint32_t)(P * TILE_PLANE * 8))
                   : "memory");
    }
#pragma unroll
    for (int i = 0; i < LH; ++i)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
        for (int j = 0; j < NTA; ++j) acc[i][mt][j][0] = acc[i][mt][j][1] = 0.0;
#pragma unroll
        for (int c = 0; c < REMA; ++c) accx[i][mt][c] = 0.0;
      }

    // one thread streams slab s: P contiguous 16-column plane slices (fwd: bulk copies) or P 16-row
    // x 64-column boxes of the transposed operand (bwd: 2-D TMA from the same column-major tiles,
    // 128-byte swizzle) + the 16 already solved rows of this CTA's private W, completion on full[st].
    // A stage is refilled once every warp has released its previous slab (empty[st]); only the
    // issuing thread waits for that, the other warps run ahead as far as the data allows.
    // In a cluster (cl > 1, the CTAs of consecutive lambda chunks of one fold) rank 0 reads each theta
    // slab once and multicasts it into every CTA's stage, after every warp of the cluster released that
    // stage (cempty); each CTA still copies its own W rows.
    auto issue = [&](int s) {
      if ((PW ? tid == NTH : tid == 0) && s < nslab) {
        const int it = it0 + s, st = it % STG;
        if (it >= STG) mbar_wait(&empty[st], ((it / STG) + 1) & 1);
        const int J = BWD ? (I + 1 + (s >> 2)) : (s >> 2);
        const int kq = s & 3;
        const uint32_t bytes = (uint32_t)(stageT * 8 + 16 * S * 8);
        mbar_arrive_expect_tx(&full[st], bytes);
        if (rank == 0) {
          const uint16_t mask = (uint16_t)((1u << cl) - 1u);
          if (cl > 1 && it >= STG) mbar_wait_cluster(&cempty[st], ((it / STG) + 1) & 1);
          if (BWD) {
            const int64_t row0 = fold * a.theta_fold_stride / TILE_LD + (int64_t)tile_index(J, I) * P * 64;
            for (int p = 0; p < P; ++p) {
              if (cl > 1)
                tma_2d_g2s_multicast(sT + st * stageT + p * BWD_SLAB, &a.tmb, kq * 16, (int)(row0 + p * 64),
                                     &full[st], mask);
              else
                tma_2d_g2s(sT + st * stageT + p * BWD_SLAB, &a.tmb, kq * 16, (int)(row0 + p * 64), &full[st]);
            }
          } else {
            const double* tile = theta + (int64_t)tile_index(I, J) * P * TILE_PLANE;
            for (int p = 0; p < P; ++p) {
              if (cl > 1)
                bulk_g2s_multicast(sT + st * stageT + p * FWD_SLAB, tile + p * TILE_PLANE + kq * 16 * TILE_LD,
                                   (uint32_t)(FWD_SLAB * 8), &full[st], mask);
              else
                bulk_g2s(sT + st * stageT + p * FWD_SLAB, tile + p * TILE_PLANE + kq * 16 * TILE_LD,
                         (uint32_t)(FWD_SLAB * 8), &full[st]);
            }
          }
        }
        bulk_g2s(sW + st * stageW, Wc + (int64_t)(J * 64 + kq * 16) * S, (uint32_t)(16 * S * 8), &full[st]);
      }
    };

    // slabs in flight ahead of the consumers: 2 with the 3/4-stage rings of the large chunks (compute
    // per slab hides the copy latency), STG - 2 with the deep rings of small chunks (latency-bound)
    constexpr int AHEAD = STG >= 6 ? STG - 2 : 2;
    if (PW && warp == NTH / 32) {
      // producer warp: the row's slabs as far ahead as the ring allows, then wait until the compute
      // warps are done with the row's diagonal step (it reuses the ring's memory)
#pragma unroll 1
      for (int s = 0; s < nslab; ++s) issue(s);
      __syncwarp();
      it0 += nslab;
      if (step + 1 < a.nt || !last_job) named_bar_sync(2, NTH + 32);
      continue;
    }
    if (!PW) {
#pragma unroll
      for (int s0 = 0; s0 < AHEAD; ++s0) issue(s0);
    }
#pragma unroll 1
    for (int s = 0; s < nslab; ++s) {
      if (!PW) issue(s + AHEAD);
      const int st = (it0 + s) % STG;
      mbar_wait(&full[st], ((it0 + s) / STG) & 1);
      const double* T = sT + st * stageT;
      const double* Wb = sW + st * stageW;
      // Each lane's A fragments come from one 16-byte shared load per (plane, k-step pair):
      //  fwd: the rows of its two m-tiles are adjacent (slab_row), A(row, k), A(row + 1, k) at [k][68];
      //  bwd: its k values of the k-steps 2 kp and 2 kp + 1 are adjacent (k = 8 kp + 2 t + h), one
      //       swizzled 16-byte chunk of row slab_row(mt), chunk index (4 kp + t) ^ (row & 7).
      // Both are bank-conflict free, and the B fragments (W rows k) stay conflict free (S = 12 mod 16).
      // k-step ks (0..3) of the slab, with the coefficient fragments of its two m-tiles in th[mt][plane]
      auto kstep = [&](int ks, const double (&th)[2][PM]) {
        const double* wrow = Wb + (BWD ? 8 * (ks >> 1) + 4 * (ks & 1) + t : ks * 4 + t) * S;
#pragma unroll
        for (int i = 0; i < LH; ++i) {
          const int l = lg * LH + i;
          if (l < nl) {
            double b[NTA];
            double rv[REMA];
#pragma unroll
            for (int j = 0; j < NT; ++j) b[j] = wrow[l * m + j * 8 + g];
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
              // Horner from the top plane: v = theta_{P-1}; v = v*t + theta_p
              double av = 0.0;
#pragma unroll
              for (int p = PM - 1; p >= 0; --p)
                if (p < P) av = (p == P - 1) ? th[mt][p] : fma(av, tl[i], th[mt][p]);
#pragma unroll
              for (int j = 0; j < NT; ++j) dmma884(acc[i][mt][j][0], acc[i][mt][j][1], av, b[j]);
#pragma unroll
              for (int c = 0; c < REM; ++c) accx[i][mt][c] = fma(av, rv[c], accx[i][mt][c]);
            }
          }
        }
      };
      if (!BWD) {
        // forward: one 16-byte load per (k-step, plane) holds both m-tiles' rows; the next k-step's
        // fragments are loaded while this one computes
        auto ldf = [&](int ks, double (&th)[2][PM]) {
#pragma unroll
          for (int p = 0; p < PM; ++p)
            if (p < P) {
              const double2 v =
                  *reinterpret_cast<const double2*>(T + p * FWD_SLAB + (ks * 4 + t) * 68 + slab_row(0));
              th[0][p] = v.x;
              th[1][p] = v.y;
            }
        };
        double tha[2][PM], thb[2][PM];
        ldf(0, tha);
        ldf(1, thb);
        kstep(0, tha);
        ldf(2, tha);
        kstep(1, thb);
        ldf(3, thb);
        kstep(2, tha);
        kstep(3, thb);
      } else {
        // backward: one 16-byte load per (m-tile, plane) holds two k-steps (swizzled row chunk); the
        // second pair is loaded while the first computes
        auto ldb = [&](int kp, double (&th0)[2][PM], double (&th1)[2][PM]) {
#pragma unroll
          for (int p = 0; p < PM; ++p)
            if (p < P) {
#pragma unroll
              for (int mt = 0; mt < 2; ++mt) {
                const int row = slab_row(mt);
                const double2 v = *reinterpret_cast<const double2*>(
                    T + p * BWD_SLAB + row * 16 + (((4 * kp + t) ^ (row & 7)) << 1));
                th0[mt][p] = v.x;
                th1[mt][p] = v.y;
              }
            }
        };
        double th0[2][PM], th1[2][PM], th2[2][PM], th3[2][PM];
        ldb(0, th0, th1);
        ldb(1, th2, th3);
        kstep(0, th0);
        kstep(1, th1);
        kstep(2, th2);
        kstep(3, th3);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[st]);
        if (cl > 1) mbar_arrive_cluster(cempty0 + 8u * st);
      }
    }
    it0 += nslab;
    csync();  // every warp is done with the ring
    RP_SP_MARK(0);    // slabs of the row

    // ---- diagonal tile: stage theta_II (P x 64 x 64, forward copy) into the drained ring,
    //      R = base - acc into sR, then a triangular solve per (lambda, output) column ----
    double* sD = smem;  // union with the ring (idle during the diagonal step)
    if (tid == 0) {
      const double* tile = theta + (int64_t)tile_index(I, I) * P * TILE_PLANE;
      mbar_arrive_expect_tx(&full[STG], (uint32_t)(P * TILE_PLANE * 8));
      bulk_g2s(sD, tile, (uint32_t)(P * TILE_PLANE * 8), &full[STG]);
    }
    const int rowI = I * 64;
#pragma unroll
    for (int i = 0; i < LH; ++i) {
      const int l = lg * LH + i;
      if (l < nl) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int row = slab_row(mt);
#pragma unroll
          for (int c = 0; c < REM; ++c) {
            double v = accx[i][mt][c];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            accx[i][mt][c] = v;
          }
#pragma unroll
          for (int j = 0; j < NT; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int col = j * 8 + 2 * t + h;
              double base = BWD ? Wc[(int64_t)(rowI + row) * S + l * m + col]
                                : a.rhs[fold * a.rhs_fold_stride + (int64_t)(rowI + row) * m + col];
              sR[row * S + l * m + col] = base - acc[i][mt][j][h];
            }
          }
          if (t == 0) {
#pragma unroll
            for (int c = 0; c < REM; ++c) {
              const int col = NT * 8 + c;
              double base = BWD ? Wc[(int64_t)(rowI + row) * S + l * m + col]
                                : a.rhs[fold * a.rhs_fold_stride + (int64_t)(rowI + row) * m + col];
              sR[row * S + l * m + col] = base - accx[i][mt][c];
            }
          }
        }
      }
    }
    mbar_wait(&full[STG], diag_it & 1);
    ++diag_it;
    csync();
    RP_SP_MARK(1);  // R = base - acc, theta_II staged
    // triangular solve of the 64 x 64 diagonal tile, blocked by 16 rows. Per 16 x 16 diagonal
    // block: evaluate it once per lambda into shared memory (with reciprocal pivots and the
    // singular check), then one thread per (lambda, output) column substitutes with its 16 rows in
    // registers (column-oriented, so the serial chain is one FMA + one multiply per row); the
    // block's contribution to the remaining rows of the tile is then applied with DMMA like a slab
    // (A = L(rows, block cols) evaluated from sD, B = the block's solved rows in sR).
    double* sLev = sD + P * TILE_PLANE;  // [nl][16][17] evaluated block (row i, col j <= i)
    double* sRinv = sLev + LCr * 16 * 17;  // [nl][16] reciprocal pivots
    for (int q = 0; q < 4; ++q) {
      const int sb = BWD ? 3 - q : q;
      const int r0 = sb * 16;
      for (int e = tid; e < nl * 136; e += NTH) {
        const int l = e / 136;
        const int ij = e - l * 136;  // packed lower index: row i, col j <= i
        const int i = s_pi[ij], j = s_pj[ij];
        const double tv = s_tv[l];
        const int off = (r0 + j) * TILE_LD + r0 + i;  // L(r0+i, r0+j), forward (column-major) copy
        double v = 0.0;
#pragma unroll
        for (int p = PM - 1; p >= 0; --p)
          if (p < P) v = (p == P - 1) ? sD[p * TILE_PLANE + off] : fma(v, tv, sD[p * TILE_PLANE + off]);
        sLev[(l * 16 + i) * 17 + j] = v;
        if (i == j) {
          sRinv[l * 16 + i] = __drcp_rn(v);  // = 1.0 / v (correctly rounded), without the division path
          if (!BWD && rowI + r0 + i < a.d && !(fabs(v) >= 1e-12)) a.flags[fold * a.flag_stride + l0 + l] = 1;
        }
      }
      csync();
      RP_SP_MARK(2);  // evaluate the 16 x 16 block
      if (tid < cw) {
        const int l = tid / m;
        const double* Lv = sLev + l * 16 * 17;
        const double* ri = sRinv + l * 16;
        double x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = sR[(r0 + i) * S + tid];
        if (!BWD) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            x[i] *= ri[i];
#pragma unroll
            for (int j = i + 1; j < 16; ++j) x[j] = fma(-Lv[j * 17 + i], x[i], x[j]);
          }
        } else {
#pragma unroll
          for (int i = 15; i >= 0; --i) {
            x[i] *= ri[i];
#pragma unroll
            for (int j = 0; j < i; ++j) x[j] = fma(-Lv[i * 17 + j], x[i], x[j]);
          }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) sR[(r0 + i) * S + tid] = x[i];
      }
      csync();
      RP_SP_MARK(3);  // 16-row substitution
      // rows still to solve: after the block (fwd) / before it (bwd)
      if (q < 3 && (BWD ? (rg < sb) : (rg > sb))) {
#pragma unroll
        for (int i = 0; i < LH; ++i)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
            for (int j = 0; j < NTA; ++j) acc[i][mt][j][0] = acc[i][mt][j][1] = 0.0;
#pragma unroll
            for (int c = 0; c < REMA; ++c) accx[i][mt][c] = 0.0;
          }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int k = r0 + ks * 4 + t;
          double th[2][PM];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const int row = slab_row(mt);
            // fwd: L(row, k) (column k of the tile); bwd: L(k, row) (column row)
            const int off = BWD ? row * TILE_LD + k : k * TILE_LD + row;
#pragma unroll
            for (int p = 0; p < PM; ++p)
              if (p < P) th[mt][p] = sD[p * TILE_PLANE + off];
          }
          const double* wrow = sR + k * S;
#pragma unroll
          for (int i = 0; i < LH; ++i) {
            const int l = lg * LH + i;
            if (l < nl) {
              double b[NTA];
#pragma unroll
              for (int j = 0; j < NT; ++j) b[j] = wrow[l * m + j * 8 + g];
              double rv[REMA];
#pragma unroll
              for (int c = 0; c < REM; ++c) rv[c] = wrow[l * m + NT * 8 + c];
#pragma unroll
              for (int mt = 0; mt < 2; ++mt) {
                double av = 0.0;
#pragma unroll
                for (int p = PM - 1; p >= 0; --p)
                  if (p < P) av = (p == P - 1) ? th[mt][p] : fma(av, tl[i], th[mt][p]);
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma884(acc[i][mt][j][0], acc[i][mt][j][1], av, b[j]);
#pragma unroll
                for (int c = 0; c < REM; ++c) accx[i][mt][c] = fma(av, rv[c], accx[i][mt][c]);
              }
            }
          }
        }
        // subtract from this warp's rows (each element owned by exactly one lane)
#pragma unroll
        for (int i = 0; i < LH; ++i) {
          const int l = lg * LH + i;
          if (l < nl) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              const int row = slab_row(mt);
#pragma unroll
              for (int c = 0; c < REM; ++c) {
                double v = accx[i][mt][c];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                if (t == 0) sR[row * S + l * m + NT * 8 + c] -= v;
              }
#pragma unroll
              for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) sR[row * S + l * m + j * 8 + 2 * t + h] -= acc[i][mt][j][h];
            }
          }
        }
      }
      csync();
      RP_SP_MARK(4);  // DMMA update of the rows below
    }
    // publish row I: private rows (read back by later slabs through the async proxy) and, for
    // the backward pass, the caller's row-major W (overlapping chunks write identical values)
    // (the backward pass stores each 16-row group of its private rows in the order its slab loop
    // reads them: logical row 8 kp + 2 t + h at 8 kp + 4 h + t, so the B fragments and the leftover
    // 16-byte loads of lanes t = 0..3 hit consecutive rows -- conflict-free with S = 12 mod 16)
    for (int i = warp; i < 64; i += NTH / 32) {
      const int ip = BWD ? (i & ~15) | (i & 8) | ((i & 1) << 2) | ((i >> 1) & 3) : i;
      double* dc = Wc + (int64_t)(rowI + ip) * S;
      for (int c = lane; c < cw; c += 32) dc[c] = sR[i * S + c];
      if (BWD) {
        double* dst = W + (int64_t)(rowI + i) * a.ldw + wcol0;
        for (int c = lane; c < cw; c += 32) dst[c] = sR[i * S + c];
      }
    }
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    csync();
    // the diagonal step used the ring's memory: rank 0 multicasts the next row's slabs only after every
    // CTA of the cluster is done with it
    if (cl > 1) cluster_sync();
    if (PW && (step + 1 < a.nt || !last_job)) named_bar_arrive(2, NTH + 32);  // the producer may refill the ring
    RP_SP_MARK(5);  // publish
  }
  }  // jobs
#ifdef RP_SOLVE_PROF
  if (tid == 0 && blockIdx.x == 0)
    printf("solve %s phases (Mcycles): slabs %.3f R+stage %.3f eval %.3f subst %.3f update %.3f publish %.3f\n",
           BWD ? "bwd" : "fwd", sp_acc[0] * 1e-6, sp_acc[1] * 1e-6, sp_acc[2] * 1e-6, sp_acc[3] * 1e-6,
           sp_acc[4] * 1e-6, sp_acc[5] * 1e-6);
#endif
}

// Row stride of the W / R tiles: >= lam*m and = 12 (mod 16) doubles, so the DMMA B fragments
// (rows t, cols g) and the 16-byte leftover-column loads (4 rows, one address per row) are both
// bank-conflict free.
inline int solve_stride(int lam, int m) { return ((lam * m + 3) / 16) * 16 + 12; }

// Dynamic shared memory of one pass. The backward pass's slabs are smaller (64 x 16 TMA boxes vs
// 16 x 68 columns) but its ring must start on a 1 KB boundary (128-byte swizzle atoms): + 1 KB slack.
inline size_t solve_smem_bytes(int lam, int m, int P, int stages = SOLVE_STAGES, bool bwd = false) {
  const int S = solve_stride(lam, m);
  size_t per_stage = (size_t)P * (bwd ? BWD_SLAB : FWD_SLAB) + 16 * (size_t)S;
  size_t ring = stages * per_stage;
  // theta_II + the evaluated 16 x 16 diagonal blocks + pivots, in the idle ring during the diagonal step
  size_t diag = (size_t)P * TILE_PLANE + (size_t)lam * (16 * 17 + 16);
  // + mbarriers: full (stages + 1), empty and cluster-empty (stages each)
  return sizeof(double) * ((ring > diag ? ring : diag) + 64 * (size_t)S + 3 * (size_t)stages + 1) + (bwd ? 1024 : 0);
}

inline size_t solve_smem_max(int lam, int m, int P, int stages = SOLVE_STAGES) {
  const size_t f = solve_smem_bytes(lam, m, P, stages, false), b = solve_smem_bytes(lam, m, P, stages, true);
  return f > b ? f : b;
}


template <typename K>
static cudaError_t launch_clustered(K kern, int grid, int threads, size_t smem, int cl, cudaStream_t st,
                                   const SolveArgs& a) {
  if (cl <= 1) {
    kern<<<grid, threads, smem, st>>>(a);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// tail: the launch covers only each fold's last chunk beside a main launch (profiled under its own names)
template <int NT, int REM, int PT, int LCT, int LG = 2, int STG = SOLVE_STAGES>
int launch_solve(const SolveArgs& a, int grid, cudaStream_t st, bool tail = false) {
  auto kf = eval_solve_kernel<NT, REM, PT, LCT, LG, STG, false>;
  auto kb = eval_solve_kernel<NT, REM, PT, LCT, LG, STG, true>;
  const size_t sf = solve_smem_bytes(a.lam_per_cta, a.m, a.P, STG, false);
  const size_t sb = solve_smem_bytes(a.lam_per_cta, a.m, a.P, STG, true);
  cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
  if (a.cl > 8) {
    cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kb, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  {
    ProfScope prof(tail ? "eval_solve_fwd_tail" : "eval_solve_fwd", st);
    cudaError_t e = launch_clustered(kf, grid, 128 * LG + (solve_pw<LCT>() ? 32 : 0), sf, a.cl, st, a);
    if (e != cudaSuccess) return cuda_status(e, "eval_solve fwd launch");
  }
  RP_LAUNCH_CHECK("eval_solve fwd");
  {
    ProfScope prof(tail ? "eval_solve_bwd_tail" : "eval_solve_bwd", st);
    cudaError_t e = launch_clustered(kb, grid, 128 * LG + (solve_pw<LCT>() ? 32 : 0), sb, a.cl, st, a);
    if (e != cudaSuccess) return cuda_status(e, "eval_solve bwd launch");
  }
  RP_LAUNCH_CHECK("eval_solve bwd");
  return RP_OK;
}

// Co-resident clusters of `cl` CTAs (the smaller of the two passes; 0 when the shape cannot be scheduled).
template <int NT, int REM, int PT, int LCT, int LG = 2, int STG = SOLVE_STAGES>
int solve_clusters(int lam, int m, int P, int cl) {
  int best = 1 << 30;
  for (int bwd = 0; bwd < 2; ++bwd) {
    auto k = bwd ? eval_solve_kernel<NT, REM, PT, LCT, LG, STG, true> : eval_solve_kernel<NT, REM, PT, LCT, LG, STG, false>;
    const size_t smem = solve_smem_bytes(lam, m, P, STG, bwd);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cl > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(128 * LG + (solve_pw<LCT>() ? 32 : 0));
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    best = n < best ? n : best;
  }
  return best;
}

// Fast instantiations (rp_solve_fast.cu): returns -2 when (m, P, lam) has none.
int launch_solve_fast(int m, int P, int lam, const SolveArgs& a, int grid, cudaStream_t st, bool tail = false);
bool has_solve_fast(int m, int P, int lam);
int solve_fast_clusters(int m, int P, int lam, int cl);  // solve_clusters of that instantiation

}  // namespace rp
