// Diagonal-block kernel of the blocked Cholesky (rp_potrf_batched): factor the 128 x 128
// diagonal block of every batch matrix in shared memory and produce inv(L11) for the panel
// TRSM (which then runs as a DMMA GEMM). One CTA (16 warps) per matrix.
//
// Both halves are blocked by 16 with the updates on the FP64 tensor pipe (mma.m8n8k4.f64):
//   factor  (left-looking): for each 16-column block jb
//             1a  A[jb:, jb] -= L[jb:, :jb] L[jb, :jb]^T        (DMMA, one m-tile per warp)
//             1b  16 x 16 diagonal factor (LAPACK dpotf2 order) + its inverse D^-1 (warp 0)
//             1c  L[jb+1:, jb] = A[jb+1:, jb] D^-T               (DMMA against D^-1)
//   inverse (LAPACK dtrtri order, in place, last block first):
//             X[jb+1:, jb] = -X[jb+1:, jb+1:] L[jb+1:, jb] D_jb^-1,  X[jb, jb] = D_jb^-1
// Shared layout: the block column-major with a padded column stride of 136 doubles, so both
// DMMA fragment reads (A: rows g, k = t; B: k = t, cols g) are conflict-free 2-wavefront loads.
#pragma once
#include "rp_common.cuh"

namespace rp {

constexpr int PD_NB = 128;
constexpr int PD_LDA = 136;
constexpr int PD_LDD = 24;  // stride of the 16 x 16 inverse blocks
constexpr int PD_THREADS = 512;
constexpr size_t PD_SMEM = sizeof(double) * (PD_NB * PD_LDA + 2 * 8 * 16 * PD_LDD + 16 * 16 * 8);

// Register-resident 16 x 16 dpotf2 step J (lane i < 16 holds row i; column J of L broadcast
// with shuffles), unrolled at compile time so `row` never leaves registers. rinv[J] = 1/L(J,J).
template <int J>
RP_DEVINL void pd_factor_step(double (&row)[16], int ri, int& bad, double* rinv) {
  double ajj = __shfl_sync(0xffffffffu, row[J], J);
  if (!bad && !(ajj > 0.0)) bad = J + 1;  // uniform across the warp
  if (bad) ajj = 1.0;                       // keep the (discarded) arithmetic finite
  const double ljj = sqrt(ajj), rl = __drcp_rn(ljj);  // = 1.0 / ljj (correctly rounded), no division path
  if (ri > J) row[J] *= rl;
  if (ri == J) row[J] = ljj;
  if ((threadIdx.x & 31) == 0) rinv[J] = rl;
#pragma unroll
  for (int c = J + 1; c < 16; ++c) {
    const double lcj = __shfl_sync(0xffffffffu, row[J], c);  // L(c, J)
    if (ri >= c) row[c] = fma(-row[J], lcj, row[c]);
  }
  if constexpr (J + 1 < 16) pd_factor_step<J + 1>(row, ri, bad, rinv);
}

// Row I of column c of D^-1 (forward substitution D x = e_c), x in registers.
template <int I>
RP_DEVINL void pd_inv_step(double (&x)[16], const double* D, const double* rinv, int c) {
  double s = (I == c) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < I; ++k) s = fma(-D[k * PD_LDA + I], x[k], s);
  x[I] = (I < c) ? 0.0 : s * rinv[I];
  if constexpr (I + 1 < 16) pd_inv_step<I + 1>(x, D, rinv, c);
}

__global__ void __launch_bounds__(PD_THREADS, 1) potrf_diag_dmma_kernel(double* A, int d, int64_t stride, int k0,
                                                                       double* inv, int* info) {
  extern __shared__ __align__(16) double sm[];
  double* a = sm;                                // a[c * LDA + r]
  double* dinvT = a + PD_NB * PD_LDA;            // block b: dinvT[b][k][n] = Dinv_b(n, k)
  double* dinvN = dinvT + 8 * 16 * PD_LDD;       // block b: dinvN[b][k][n] = Dinv_b(k, n)
  double* scratch = dinvN + 8 * 16 * PD_LDD;     // per warp 16 x 8 (k-major) staging
  __shared__ int fail;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  if (info[b] != 0) return;  // this matrix already failed in an earlier block
  double* Ab = A + b * stride;
  const int nbv = min(PD_NB, d - k0);
  if (tid == 0) fail = 0;
  for (int e = tid; e < PD_NB * PD_NB; e += PD_THREADS) {
    const int r = e & 127, c = e >> 7;
    double v;
    if (r < nbv && c < nbv) v = (r >= c) ? Ab[(int64_t)(k0 + c) * d + k0 + r] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    a[c * PD_LDA + r] = v;
  }
  __syncthreads();

  // ------------------------------------------------------------ factor
  for (int jb = 0; jb < 8; ++jb) {
    const int b0 = jb * 16;
    if (jb > 0) {  // 1a: block column update, m-tile per warp (rows b0 .. 127)
      const int ntile = 16 - 2 * jb;
      if (warp < ntile) {
        const int r0 = b0 + warp * 8;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        for (int ks = 0; ks < b0 / 4; ++ks) {
          const int k = ks * 4 + t;
          const double av = a[k * PD_LDA + r0 + g];
          const double b0v = a[k * PD_LDA + b0 + g];
          const double b1v = a[k * PD_LDA + b0 + 8 + g];
          dmma884(acc[0][0], acc[0][1], av, b0v);
          dmma884(acc[1][0], acc[1][1], av, b1v);
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = r0 + g, col = b0 + nt * 8 + 2 * t + h;
            if (row >= col) a[col * PD_LDA + row] -= acc[nt][h];
          }
      }
      __syncthreads();
    }
    if (warp == 0) {  // 1b: 16 x 16 factor + inverse
      double* D = a + b0 * PD_LDA + b0;  // D(r, c) = D[c * LDA + r]
      // register-resident 16 x 16 factor: lane i (< 16) holds row i; column j of L is
      // broadcast with shuffles (dpotf2 order: sqrt pivot, scale by the reciprocal, rank-1 update)
      const int ri = lane & 15;
      double* rinv = scratch;  // 16 reciprocal pivots (warp 0's scratch; the inverse phase reuses it later)
      double row[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) row[c] = (c <= ri) ? D[c * PD_LDA + ri] : 0.0;
      int bad = 0;
      pd_factor_step<0>(row, ri, bad, rinv);
      if (bad) {
        if (lane == 0) fail = k0 + b0 + bad;
      } else if (lane < 16) {
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c <= ri) D[c * PD_LDA + ri] = row[c];
      }
      __syncwarp();
      if (fail == 0 && lane < 16) {  // column `lane` of D^-1: solve D x = e_c
        const int c = lane;
        double x[16];
        pd_inv_step<0>(x, D, rinv, c);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          dinvN[(jb * 16 + i) * PD_LDD + c] = x[i];  // Dinv(i, c) at [k=i][n=c]
          dinvT[(jb * 16 + c) * PD_LDD + i] = x[i];  // Dinv(i, c) at [k=c][n=i]
        }
      }
    }
    __syncthreads();
    if (fail) {
      if (tid == 0) info[b] = fail;
      return;
    }
    // 1c: panel rows b0+16 .. 127: X = P D^-T (in place; a warp owns its 8 rows)
    const int np = 14 - 2 * jb;
    if (warp < np) {
      const int r0 = b0 + 16 + warp * 8;
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int k = ks * 4 + t;
        const double av = a[(b0 + k) * PD_LDA + r0 + g];
        const double* bt = dinvT + (jb * 16 + k) * PD_LDD;
        dmma884(acc[0][0], acc[0][1], av, bt[g]);
        dmma884(acc[1][0], acc[1][1], av, bt[8 + g]);
      }
      __syncwarp();
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) a[(b0 + nt * 8 + 2 * t + h) * PD_LDA + r0 + g] = acc[nt][h];
    }
    __syncthreads();
  }
  for (int e = tid; e < PD_NB * PD_NB; e += PD_THREADS) {
    const int r = e & 127, c = e >> 7;
    if (r < nbv && c < nbv && r >= c) Ab[(int64_t)(k0 + c) * d + k0 + r] = a[c * PD_LDA + r];
  }

  // ------------------------------------------------------------ inverse, in place
  double* sc = scratch + warp * 128;  // T1 staging, [k 0..15][r 0..7]
  for (int jb = 7; jb >= 0; --jb) {
    const int b0 = jb * 16;
    const int np = 14 - 2 * jb;  // m-tiles below the diagonal block
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    if (jb < 7 && warp < np) {
      // T1 = X[b0+16:, b0+16:] * L[b0+16:, b0:b0+16] for this warp's 8 rows (X lower: k <= row)
      const int r0 = b0 + 16 + warp * 8;
      const int kend = r0 + 8;
      for (int kb = b0 + 16; kb < kend; kb += 4) {
        const int k = kb + t;
        const double av = a[k * PD_LDA + r0 + g];
        dmma884(acc[0][0], acc[0][1], av, a[(b0 + g) * PD_LDA + k]);
        dmma884(acc[1][0], acc[1][1], av, a[(b0 + 8 + g) * PD_LDA + k]);
      }
    }
    __syncthreads();  // every warp has read the L panel before it is overwritten
    if (jb < 7 && warp < np) {
      const int r0 = b0 + 16 + warp * 8;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) sc[(nt * 8 + 2 * t + h) * 8 + g] = acc[nt][h];
      __syncwarp();
      double o[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int k = ks * 4 + t;
        const double av = sc[k * 8 + g];
        const double* bn = dinvN + (jb * 16 + k) * PD_LDD;
        dmma884(o[0][0], o[0][1], av, bn[g]);
        dmma884(o[1][0], o[1][1], av, bn[8 + g]);
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) a[(b0 + nt * 8 + 2 * t + h) * PD_LDA + r0 + g] = -o[nt][h];
    }
    // X[jb, jb] = D_jb^-1 (lower); the diagonal block is not read by this iteration's products
    for (int e = tid; e < 256; e += PD_THREADS) {
      const int i = e & 15, c = e >> 4;
      a[(b0 + c) * PD_LDA + b0 + i] = (i >= c) ? dinvN[(jb * 16 + i) * PD_LDD + c] : 0.0;
    }
    __syncthreads();
  }
  double* X = inv + (int64_t)b * PD_NB * PD_NB;
  for (int e = tid; e < PD_NB * PD_NB; e += PD_THREADS) {
    const int r = e & 127, c = e >> 7;
    X[e] = (r >= c) ? a[c * PD_LDA + r] : 0.0;  // column-major inv(L11)
  }
}

}  // namespace rp
