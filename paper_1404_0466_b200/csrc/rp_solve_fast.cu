// Specialised instantiations of the fused eval+solve kernel (compile-time polynomial planes
// and full lambda chunks) for the output counts / degrees of the BASELINE configs:
// m = 1 (c1), m = 10 (c2-c4, degree 2), m = 16 (c5, degree 3).
#include "rp_solve.cuh"

#ifndef RP_SOLVE_LG
#define RP_SOLVE_LG 4
#endif

namespace rp {

#define RP_FAST_LIST(X) \
  X(1, 3, 16) X(1, 3, 8) X(10, 3, 4) X(10, 3, 8) X(10, 3, 12) X(10, 3, 16) X(16, 4, 4) X(16, 4, 6) X(16, 4, 8)

bool has_solve_fast(int m, int P, int lam) {
#define RP_HAS(M, PP, L) \
  if (m == M && P == PP && lam == L) return true;
  RP_FAST_LIST(RP_HAS)
#undef RP_HAS
  return false;
}

int launch_solve_fast(int m, int P, int lam, const SolveArgs& a, int grid, size_t smem, cudaStream_t st) {
#define RP_LAUNCH(M, PP, L) \
  if (m == M && P == PP && lam == L) return launch_solve<(M) / 8, (M) % 8, PP, L, RP_SOLVE_LG>(a, grid, smem, st);
  RP_FAST_LIST(RP_LAUNCH)
#undef RP_LAUNCH
  return -2;
}

}  // namespace rp
