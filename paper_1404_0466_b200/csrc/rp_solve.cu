// (5) Fused evaluate + solve: host dispatch of rp_eval_solve and the generic (runtime P and
// chunk size) kernel instantiations. The kernel itself is in rp_solve.cuh; the specialised
// (compile-time P and chunk) instantiations used by the BASELINE configs are in rp_solve_fast.cu.
#include <cstdlib>
#include <map>
#include <mutex>

#include "rp_solve.cuh"
#include "../../include/ridgepath_b200.h"

using namespace rp;

namespace rp {
int g_solve_lam = 0;      // rp_set_option("solve_lam", n): 0 = the planner's choice
int g_solve_cluster = 0;  // rp_set_option("solve_cluster", n): 2/4/8 = theta multicast clusters; 0/1 = none
}

// One side stream (with fork / join events) per calling stream, at the caller's priority.
static bool solve_side_stream(cudaStream_t caller, cudaStream_t* side, cudaEvent_t* fork, cudaEvent_t* join) {
  struct Side {
    cudaStream_t s;
    cudaEvent_t fork, join;
  };
  static std::mutex mu;
  static std::map<cudaStream_t, Side> by_caller;
  std::lock_guard<std::mutex> lock(mu);
  auto it = by_caller.find(caller);
  if (it == by_caller.end()) {
    int prio = 0;
    cudaStreamGetPriority(caller, &prio);
    Side sd{};
    if (cudaStreamCreateWithPriority(&sd.s, cudaStreamNonBlocking, prio) != cudaSuccess ||
        cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming) != cudaSuccess)
      return false;
    it = by_caller.emplace(caller, sd).first;
  }
  *side = it->second.s;
  *fork = it->second.fork;
  *join = it->second.join;
  return true;
}

static int launch_generic(int m, const SolveArgs& a, int grid, cudaStream_t st) {
  switch (m) {
    case 1: return launch_solve<0, 1, 0, 0>(a, grid, st);
    case 2: return launch_solve<0, 2, 0, 0>(a, grid, st);
    case 3: return launch_solve<0, 3, 0, 0>(a, grid, st);
    case 4: return launch_solve<0, 4, 0, 0>(a, grid, st);
    case 5: return launch_solve<0, 5, 0, 0>(a, grid, st);
    case 6: return launch_solve<0, 6, 0, 0>(a, grid, st);
    case 7: return launch_solve<0, 7, 0, 0>(a, grid, st);
    case 8: return launch_solve<1, 0, 0, 0>(a, grid, st);
    case 9: return launch_solve<1, 1, 0, 0>(a, grid, st);
    case 10: return launch_solve<1, 2, 0, 0>(a, grid, st);
    case 11: return launch_solve<1, 3, 0, 0>(a, grid, st);
    case 12: return launch_solve<1, 4, 0, 0>(a, grid, st);
    case 13: return launch_solve<1, 5, 0, 0>(a, grid, st);
    case 14: return launch_solve<1, 6, 0, 0>(a, grid, st);
    case 15: return launch_solve<1, 7, 0, 0>(a, grid, st);
    default: return launch_solve<2, 0, 0, 0>(a, grid, st);
  }
}

struct SolvePlan {
  int lam = 0, chunks = 0, S = 0, P = 0, nt = 0;
  int cl = 1, chunks_pad = 0;  // CTAs per cluster (theta multicast), chunks per fold padded to a multiple of cl
  bool fast = false;
  // Split plan (lam2 > 0): the main launch covers the first chunks * lam lambdas of every fold; a tail launch
  // of tail_ctas CTAs on the SMs the main launch leaves idle covers each fold's last lam2 lambdas (one job
  // per fold, several jobs per CTA when there are fewer idle SMs than folds).
  int lam2 = 0, S2 = 0, tail_ctas = 0;
  size_t work_doubles(int nf) const {
    return (size_t)nf * nt * 64 * ((size_t)chunks_pad * S + (lam2 ? (size_t)S2 : 0));
  }
};

static int generic_clusters(int m, int lam, int P, int cl) {
  switch (m) {
    case 1: return solve_clusters<0, 1, 0, 0>(lam, m, P, cl);
    case 2: return solve_clusters<0, 2, 0, 0>(lam, m, P, cl);
    case 3: return solve_clusters<0, 3, 0, 0>(lam, m, P, cl);
    case 4: return solve_clusters<0, 4, 0, 0>(lam, m, P, cl);
    case 5: return solve_clusters<0, 5, 0, 0>(lam, m, P, cl);
    case 6: return solve_clusters<0, 6, 0, 0>(lam, m, P, cl);
    case 7: return solve_clusters<0, 7, 0, 0>(lam, m, P, cl);
    case 8: return solve_clusters<1, 0, 0, 0>(lam, m, P, cl);
    case 9: return solve_clusters<1, 1, 0, 0>(lam, m, P, cl);
    case 10: return solve_clusters<1, 2, 0, 0>(lam, m, P, cl);
    case 11: return solve_clusters<1, 3, 0, 0>(lam, m, P, cl);
    case 12: return solve_clusters<1, 4, 0, 0>(lam, m, P, cl);
    case 13: return solve_clusters<1, 5, 0, 0>(lam, m, P, cl);
    case 14: return solve_clusters<1, 6, 0, 0>(lam, m, P, cl);
    case 15: return solve_clusters<1, 7, 0, 0>(lam, m, P, cl);
    default: return solve_clusters<2, 0, 0, 0>(lam, m, P, cl);
  }
}

// Cluster size (on request, rp_set_option("solve_cluster", n)): the CTAs of consecutive chunks of one fold
// share each theta slab (read once from L2/HBM by rank 0, multicast into every CTA). Padding a fold's
// chunks to a multiple of cl adds CTAs (copies of the last chunk); the requested size is used when it
// can be scheduled.
static void plan_cluster(SolvePlan& pl, int nf, int m, int sms) {
  pl.cl = 1;
  pl.chunks_pad = pl.chunks;
  if (pl.chunks < 2) return;
  auto clusters = [&](int cl) {
    return pl.fast ? solve_fast_clusters(m, pl.P, pl.lam, cl) : generic_clusters(m, pl.lam, pl.P, cl);
  };
  auto waves = [&](int cl, int active) {
    const long long ctas = (long long)nf * ((pl.chunks + cl - 1) / cl * cl);
    return (ctas + active - 1) / active;
  };
  const long long base = waves(1, sms);
  const int force = g_solve_cluster;
  for (int cl = 8; cl >= 2; cl /= 2) {
    if (force > 0 && cl != force) continue;
    if (cl > pl.chunks) continue;
    const int n = clusters(cl);
    if (n <= 0) continue;
    if (force == 0 && waves(cl, n * cl) > base) continue;
    pl.cl = cl;
    pl.chunks_pad = (pl.chunks + cl - 1) / cl * cl;
    return;
  }
}

// Chunk size: specialised kernels (full chunks, compile-time P) and the generic kernel compete
// on the lowest (waves x chunk) cost, the generic kernel's overhead weighted in.
static SolvePlan plan_solve(int d, int r, int nf, int m, int q) {
  SolvePlan pl;
  pl.P = r + 1;
  pl.nt = (d + 63) / 64;
  int dev = 0, sms = 148, maxsmem = 227 * 1024;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  double best_cost = 1e300;
  for (int lam = SOLVE_LC; lam >= 1; --lam) {
    if (lam * m > 256) continue;  // one thread per (lambda, output) column in the diagonal solve
    if (solve_smem_max(lam, m, pl.P) > (size_t)maxsmem) continue;
    const int chunks = (q + lam - 1) / lam;
    const long long ctas = (long long)nf * chunks;
    const double waves = (double)((ctas + sms - 1) / sms);
    // per-lambda cost grows as chunks shrink (every CTA streams all of its fold's theta and runs
    // all diagonal steps): measured per-lambda time at c5 (m = 16, degree 3) 16.5 / 13.7 / 13.0
    // for 4 / 6 / 8 lambdas per CTA, i.e. ~1 + 0.1 (16 - lam) relative to a full chunk
    const double base = waves * lam * (1.0 + 0.1 * (SOLVE_LC - lam));
    const bool fast_ok = q >= lam && has_solve_fast(m, pl.P, lam) && ((m % 2 == 0) || ((q - lam) % 2 == 0));
    const bool gen_ok = lam <= SOLVE_LC_GENERIC && !((m & 1) && (lam & 1) && q > 1);  // odd m: even chunks
    if (fast_ok && base < best_cost - 1e-9) {
      best_cost = base;
      pl.lam = lam;
      pl.fast = true;
    }
    if (gen_ok && 2.5 * base < best_cost - 1e-9) {
      best_cost = 2.5 * base;
      pl.lam = lam;
      pl.fast = false;
    }
  }
  // rp_set_option("solve_lam", n) (tests): force a specialised chunk size when it exists
  const int lam_force = g_solve_lam;
  if (lam_force > 0 && q >= lam_force && has_solve_fast(m, pl.P, lam_force) &&
      ((m % 2 == 0) || ((q - lam_force) % 2 == 0)) && solve_smem_max(lam_force, m, pl.P) <= (size_t)maxsmem) {
    pl.lam = lam_force;
    pl.fast = true;
  }
  if (pl.lam > 0) {
    pl.chunks = (q + pl.lam - 1) / pl.lam;
    pl.S = solve_stride(pl.lam, m);
    // clusters only on request: measured slower at every shape tried (c4 fwd 15.6 -> 18.1 ms at 2 CTAs,
    // one fold per GPU 14.8 -> 17.7-18.4 ms at 2/4/8): the lockstep refills and the per-row cluster
    // barrier cost more than the L2/HBM reads they save (the solve is not bandwidth-bound)
    // (the small-chunk kernels run a producer warp outside the per-row cluster barrier: no clusters)
    if (g_solve_cluster > 1 && !(pl.fast && solve_pw_lam(pl.lam))) plan_cluster(pl, nf, m, sms);
    else pl.chunks_pad = pl.chunks;
  }
  // One wave that leaves SMs idle (c4: 8 folds x 17 chunks of 12 lambdas = 136 CTAs on 148 SMs): a smaller
  // main chunk with floor(q / lam) chunks per fold, and each fold's few remaining lambdas as a short tail job
  // on the idle SMs (c4: 144 CTAs of 11 lambdas + 4 CTAs x 2 folds x 2 lambdas). Every CTA's chain is then
  // shorter; a chain costs ~3.35 + lam in units of one lambda's arithmetic (c4: 2 / 4 / 12 lambdas per CTA
  // take 10.8 / 14.7 / 30.5 ms for both passes), which is what the tail must fit under.
  if (pl.lam > 0 && pl.fast && lam_force == 0 && g_solve_cluster <= 1 && m % 2 == 0 &&
      (long long)nf * pl.chunks <= sms) {
    auto cost = [](int lam) { return 3.35 + lam; };
    double best = cost(pl.lam);
    for (int l1 = pl.lam - 1; l1 >= 5 && l1 >= pl.lam - 3; --l1) {
      if (!has_solve_fast(m, pl.P, l1) || solve_pw_lam(l1)) continue;
      const int c1 = q / l1, rem = q - c1 * l1;
      const int idle = sms - nf * c1;
      if (c1 < 1 || rem == 0 || idle < 1) continue;
      int l2 = 0;
      for (int l = rem; l <= 4 && l <= q; ++l)
        if (has_solve_fast(m, pl.P, l)) {
          l2 = l;
          break;
        }
      if (l2 == 0) continue;
      const int tail_ctas = nf < idle ? nf : idle;
      const int jobs = (nf + tail_ctas - 1) / tail_ctas;
      if (jobs * cost(l2) > cost(l1) || cost(l1) >= best - 1e-9) continue;
      best = cost(l1);
      pl.lam = l1;
      pl.chunks = pl.chunks_pad = c1;
      pl.S = solve_stride(l1, m);
      pl.lam2 = l2;
      pl.S2 = solve_stride(l2, m);
      pl.tail_ctas = tail_ctas;
    }
  }
  return pl;
}

// Degree > SOLVE_PMAX - 1 (not on the BASELINE path): each lambda's factor L(t_j) is evaluated into a
// one-plane tile buffer (the same Horner arithmetic) and solved as a degree-0 "model".
__global__ void theta_eval_kernel(const double* theta, int64_t fold_stride, int P, int64_t plane_elems,
                                  const double* tval, double* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // element of one plane set
  const int f = blockIdx.y;
  if (e >= plane_elems) return;
  const int64_t tile = e / TILE_PLANE, w = e - tile * TILE_PLANE;
  const double* th = theta + f * fold_stride + tile * P * TILE_PLANE + w;
  const double t = *tval;
  double v = th[(int64_t)(P - 1) * TILE_PLANE];
  for (int p = P - 2; p >= 0; --p) v = fma(v, t, th[(int64_t)p * TILE_PLANE]);
  out[(int64_t)f * plane_elems + e] = v;
}

__global__ void copy_cols_kernel(const double* src, int64_t lds, int64_t src_fold, double* dst, int64_t ldd,
                                 int64_t dst_fold, int rows, int m) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int f = blockIdx.y;
  if (e >= (int64_t)rows * m) return;
  const int64_t i = e / m;
  const int o = (int)(e - i * m);
  dst[f * dst_fold + i * ldd + o] = src[f * src_fold + i * lds + o];
}

static int eval_solve_planned(const double* theta, int d, int r, int nf, const double* rhs, int m, const double* tvals,
                              int q, double* W, int64_t ldw, int* flags, int flag_stride, void* work,
                              cudaStream_t st);

extern "C" size_t rp_eval_solve_workspace_size(int d, int r, int nf, int m, int q) {
  if (d < 1 || nf < 1 || m < 1 || m > 16 || q < 1 || r < 0) return 0;
  if (r + 1 > SOLVE_PMAX)  // one-plane tiles + a column block of solutions + the degree-0 solve's rows
    return sizeof(double) * (size_t)nf * (rp_theta_size(d, 0) + (size_t)((d + 63) / 64 * 64) * (m + (m & 1))) +
           rp_eval_solve_workspace_size(d, 0, nf, m, 1);
  const SolvePlan pl = plan_solve(d, r, nf, m, q);
  if (pl.lam == 0) return 0;
  return sizeof(double) * pl.work_doubles(nf);
}

extern "C" int rp_eval_solve_plan(int d, int r, int nf, int m, int q, int* plan) {
  RP_REQUIRE(plan != nullptr, "rp_eval_solve_plan: plan");
  RP_REQUIRE(d >= 1 && nf >= 1 && q >= 1 && r >= 0 && m >= 1 && m <= 16, "rp_eval_solve_plan: bad sizes");
  const bool high = r + 1 > SOLVE_PMAX;  // per-lambda degree-0 solves
  const SolvePlan pl = plan_solve(d, high ? 0 : r, nf, m, high ? 1 : q);
  plan[0] = pl.lam;
  plan[1] = pl.chunks_pad;
  plan[2] = pl.lam2;
  plan[3] = pl.lam2 ? pl.tail_ctas : 0;
  return RP_OK;
}

extern "C" int rp_eval_solve(const double* theta, int d, int r, int nf, const double* rhs, int m,
                             const double* tvals, int q, double* W, int64_t ldw, int* flags, void* work,
                             void* stream) {
  RP_REQUIRE(d >= 1 && nf >= 1 && q >= 1, "rp_eval_solve: bad sizes d=%d nf=%d q=%d", d, nf, q);
  RP_REQUIRE(r >= 0, "rp_eval_solve: degree %d", r);
  RP_REQUIRE(m >= 1 && m <= 16, "rp_eval_solve: %d outputs per call (max 16)", m);
  RP_REQUIRE(ldw >= (int64_t)q * m && ldw % 2 == 0, "rp_eval_solve: ldw=%lld must be even and >= q*m",
             (long long)ldw);
  RP_REQUIRE(((uintptr_t)theta & 15) == 0 && ((uintptr_t)W & 15) == 0, "rp_eval_solve: 16-byte alignment");
  RP_REQUIRE(work != nullptr && ((uintptr_t)work & 15) == 0, "rp_eval_solve: workspace (16-byte aligned)");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)nf * q, st);
  if (e != cudaSuccess) return cuda_status(e, "rp_eval_solve memset");
  if (r + 1 <= SOLVE_PMAX) return eval_solve_planned(theta, d, r, nf, rhs, m, tvals, q, W, ldw, flags, q, work, st);
  // high degree: per lambda, L(t_j) into a one-plane tile buffer, then a degree-0 solve of that column block
  const int dp = (d + 63) / 64 * 64, mp = m + (m & 1);
  double* th0 = (double*)work;
  const int64_t plane = rp_theta_size(d, 0);
  double* wcol = th0 + (size_t)nf * plane;  // nf x dp x mp
  void* work2 = wcol + (size_t)nf * dp * mp;
  for (int j = 0; j < q; ++j) {
    theta_eval_kernel<<<dim3((unsigned)((plane + 255) / 256), nf), 256, 0, st>>>(theta, rp_theta_size(d, r), r + 1,
                                                                                 plane, tvals + j, th0);
    RP_LAUNCH_CHECK("theta_eval");
    int rc = eval_solve_planned(th0, d, 0, nf, rhs, m, tvals + j, 1, wcol, mp, flags + j, q, work2, st);
    if (rc) return rc;
    copy_cols_kernel<<<dim3((unsigned)(((int64_t)dp * m + 255) / 256), nf), 256, 0, st>>>(
        wcol, mp, (int64_t)dp * mp, W + (int64_t)j * m, ldw, (int64_t)dp * ldw, dp, m);
    RP_LAUNCH_CHECK("solve column copy");
  }
  return RP_OK;
}

static int eval_solve_planned(const double* theta, int d, int r, int nf, const double* rhs, int m, const double* tvals,
                              int q, double* W, int64_t ldw, int* flags, int flag_stride, void* work,
                              cudaStream_t st) {
  RP_REQUIRE(((uintptr_t)W & 15) == 0, "rp_eval_solve: 16-byte alignment of the W column block");
  const SolvePlan pl = plan_solve(d, r, nf, m, q);
  RP_REQUIRE(pl.lam >= 1, "rp_eval_solve: no chunk size fits shared memory");
  const int P = pl.P, nt = pl.nt;
  SolveArgs a{};
  a.theta = theta;
  a.theta_fold_stride = rp_theta_size(d, r);
  a.ntiles = rp_tile_count(d);
  {  // backward slabs: 2-D FP64 view of all folds' tiles, inner dim = the 68-padded column
    auto enc = tensor_map_encoder();
    RP_REQUIRE(enc != nullptr, "rp_eval_solve: cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)TILE_LD, (cuuint64_t)(nf * a.theta_fold_stride / TILE_LD)};
    cuuint64_t strides[1] = {(cuuint64_t)TILE_LD * sizeof(double)};
    cuuint32_t box[2] = {16, 64};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&a.tmb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(theta), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
#ifndef RP_SOLVE_PROMO
#define RP_SOLVE_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_128B
#endif
                      RP_SOLVE_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return set_error(RP_ECUDA, "rp_eval_solve: tensor map (CUresult %d)", (int)cr);
  }
  a.rhs = rhs;
  a.rhs_fold_stride = (int64_t)nt * 64 * m;
  a.W = W;
  a.ldw = ldw;
  a.w_fold_stride = (int64_t)nt * 64 * ldw;
  a.tvals = tvals;
  a.flags = flags;
  a.flag_stride = flag_stride;
  a.q = q;
  a.m = m;
  a.d = d;
  a.nt = nt;
  a.P = P;
  a.lam_per_cta = pl.lam;
  a.chunks = pl.chunks_pad;
  a.chunks_real = pl.chunks;
  a.cl = pl.cl;
  a.S = pl.S;
  a.Wc = (double*)work;
  const int grid = nf * a.chunks;
  a.chunk0 = 0;
  a.njobs = grid;
  if (!pl.fast) return launch_generic(m, a, grid, st);
  if (pl.lam2 == 0) return launch_solve_fast(m, P, pl.lam, a, grid, st);
  // split plan: the tail launch runs on a side stream, on the SMs the main launch leaves idle (main and
  // tail CTAs together fit the device, so neither waits for the other; each stream orders its own two
  // passes, and the caller's stream joins the side stream at the end)
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  RP_REQUIRE(solve_side_stream(st, &side, &fork, &join), "rp_eval_solve: side stream");
  cudaError_t e = cudaEventRecord(fork, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(side, fork, 0);
  if (e != cudaSuccess) return cuda_status(e, "rp_eval_solve fork");
  int rc = launch_solve_fast(m, P, pl.lam, a, grid, st);
  if (rc) return rc;
  SolveArgs t = a;
  t.lam_per_cta = pl.lam2;
  t.S = pl.S2;
  t.chunks = t.chunks_real = 1;
  t.chunk0 = (q + pl.lam2 - 1) / pl.lam2 - 1;  // the fold's last chunk: lambdas q - lam2 .. q - 1
  t.njobs = nf;
  t.Wc = a.Wc + (size_t)grid * nt * 64 * pl.S;
  rc = launch_solve_fast(m, P, pl.lam2, t, pl.tail_ctas, side, true);
  if (rc) return rc;
  e = cudaEventRecord(join, side);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, join, 0);
  if (e != cudaSuccess) return cuda_status(e, "rp_eval_solve join");
  return RP_OK;
}
