// Shared device helpers for the piCholesky CV path on B200 (sm_100a).
//
// FP64 on sm_100a: tcgen05 has no f64 kind, so the FP64 tensor path is the
// warp-level mma.sync m8n8k4 f64 (SASS DMMA.8x8x4). Measured on this pool's
// B200 (tools/fp64_peaks.cu, profiles/r01_fp64_peaks.json): DMMA 37.0 TFLOP/s,
// DFMA 33.6 TFLOP/s, and the two share one FP64 datapath (mixed 31.6 + 4.0).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define RP_DEVINL __device__ __forceinline__

namespace rp {

// D = A(8x4, row) * B(4x8, col) + D.  Fragment ownership per lane
// (g = lane >> 2, t = lane & 3):  a = A[g][t], b = B[t][g], d0/d1 = D[g][2t], D[g][2t+1].
RP_DEVINL void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

RP_DEVINL uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte async copy global -> shared, zero-filled when !valid.
RP_DEVINL void cp_async8(void* smem, const void* gmem, bool valid) {
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(n));
}

// 16-byte async copy (L2 only), zero-filled when !valid.
RP_DEVINL void cp_async16(void* smem, const void* gmem, bool valid) {
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(n));
}

RP_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
RP_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- mbarrier + bulk async copy (Hopper/Blackwell async proxy) ----
RP_DEVINL void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

RP_DEVINL void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

RP_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar))
               : "memory");
}

RP_DEVINL void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

RP_DEVINL void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Contiguous global -> shared bulk copy (16-byte aligned, size % 16 == 0), completion on `bar`.
RP_DEVINL void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// 2-D TMA load (tensor map in param / const / global space), completion on `bar`.
RP_DEVINL void tma_2d_g2s(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed).
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

// ---- thread-block clusters: rank, barrier, remote mbarrier arrive, multicast bulk copies ----
RP_DEVINL uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

// Full cluster barrier (every thread of every CTA arrives; release/acquire at cluster scope).
RP_DEVINL void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Address of `p` (this CTA's shared memory) in CTA `rank` of the cluster.
RP_DEVINL uint32_t cluster_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

RP_DEVINL void mbar_arrive_cluster(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster_addr) : "memory");
}

// Wait on a local mbarrier whose arrivals come from other CTAs of the cluster.
RP_DEVINL void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
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

// Bulk copy into the same shared-memory offset of every CTA in `mask`; each destination CTA's
// mbarrier at `bar`'s offset receives the byte count.
RP_DEVINL void bulk_g2s_multicast(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
      "%4;\n" ::"r"(smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

RP_DEVINL void tma_2d_g2s_multicast(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                    uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
      "{%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

RP_DEVINL void named_bar_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

RP_DEVINL void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

}  // namespace rp

// Coefficient tile layout (include/ridgepath_b200.h): 64 x 64 column-major planes with a padded
// leading dimension of 68, so a 16-column slab (forward substitution) is one contiguous bulk copy
// that lands in a conflict-free shared layout, and a 16-row slab (backward substitution, the
// transposed operand) is one 2-D TMA box {16 rows, 64 columns} with the 128-byte swizzle.
constexpr int TILE_LD = 68;
constexpr int TILE_PLANE = 64 * TILE_LD;

// Status codes of the C ABI (include/ridgepath_b200.h).
#define RP_OK 0
#define RP_EINVAL (-1)
#define RP_ECUDA 1

// ---- host-side error plumbing shared by the C-ABI translation units ----
namespace rp {
int set_error(int code, const char* fmt, ...);  // records rp_last_error(), returns code
void count_launch();                             // rp_launch_count() bookkeeping
inline int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return RP_OK;
  return set_error((int)e, "%s: %s", where, cudaGetErrorString(e));
}

// Kernel timing for the bench's roofline (rp_set_option("profile", 1)): CUDA events recorded on
// the launching stream around selected kernels, summed by rp_profile_ms(name).
bool prof_on();
void prof_push(const char* name, cudaEvent_t a, cudaEvent_t b, cudaStream_t st);
cudaEvent_t prof_event();
struct ProfScope {
  const char* name;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
    if (prof_on()) {
      a = prof_event();
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event();
      cudaEventRecord(b, st);
      prof_push(name, a, b, st);
    }
  }
};
}  // namespace rp

#define RP_LAUNCH_CHECK(where)                          \
  do {                                                  \
    rp::count_launch();                                 \
    cudaError_t _e = cudaGetLastError();                \
    if (_e != cudaSuccess) return rp::cuda_status(_e, where); \
  } while (0)

#define RP_REQUIRE(cond, ...)                                  \
  do {                                                         \
    if (!(cond)) return rp::set_error(RP_EINVAL, __VA_ARGS__); \
  } while (0)
