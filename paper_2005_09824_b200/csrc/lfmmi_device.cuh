// Device-side helpers shared by the LF-MMI kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "lfmmi_internal.h"

namespace lfmmi {

constexpr unsigned kFull = 0xffffffffu;

// Frames of item b as the kernels see them: a length outside [1, T_max] (a
// caller mistake such as pre-subsampling lengths) makes the item a failed
// zero-length item instead of an out-of-bounds write.
__device__ __forceinline__ int item_frames(const int *lengths, int b, int T_max) {
  const int T = lengths[b];
  return (T >= 1 && T <= T_max) ? T : 0;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// NaN-propagating maximum: the reference takes row maxima with numpy
// (forward_backward.py:126), where a NaN anywhere in a valid frame makes the
// shift NaN, every emission of the frame NaN and the utterance fail in both
// graphs.  IEEE fmax would drop the NaN and only poison that one pdf.
__device__ __forceinline__ float nan_max(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ double nan_max(double a, double b) {
  return (a != a || b != b) ? (a + b) : fmax(a, b);
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nan_max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// Sum of the first n (<= 32) entries of v, identical in every lane.
template <typename T>
__device__ __forceinline__ T lane_sum_n(const T *v, int n, int lane) {
  T x = lane < n ? v[lane] : T(0);
  return warp_sum(x);
}

template <typename Real>
__device__ __forceinline__ const Real *pick(const float *f, const double *d);
template <>
__device__ __forceinline__ const float *pick<float>(const float *f, const double *) { return f; }
template <>
__device__ __forceinline__ const double *pick<double>(const float *, const double *d) { return d; }

__device__ __forceinline__ float exp_r(float x) { return expf(x); }
// Correctly rounded reciprocal (== 1 / x in IEEE round-to-nearest), no division subroutine.
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }
// One MUFU.RCP (rel. error ~2^-23, subnormals kept) for per-frame normalisers
// of the split kernel: a column scaled by (1 + e) / t instead of 1 / t is
// renormalised by the next frame's sum, so the forward log-probability (sum of
// log t) picks up sum log(1 + e) <= T 2^-23 (~4e-5 absolute at T = 300, far
// inside the fp32 objective bar), and posteriors, divided by their frame total
// Z, do not see the backward normaliser at all.
__device__ __forceinline__ float rcp_fast(float x) {
  float y;
  asm("rcp.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double exp_r(double x) { return exp(x); }

// ---- cp.async (LDGSTS) -----------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async_elem(float *dst, const float *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_elem(double *dst, const double *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- TMA bulk copies (cp.async.bulk, UBLKCP) completing on an mbarrier ---------
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
// Make initialised barriers visible to the async (TMA) proxy.
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// Order this thread's earlier generic-proxy shared accesses before later
// async-proxy writes (a slot is refilled by TMA after it was read with LDS).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// One elected thread: expect `bytes` on `bar` and start a global -> shared bulk copy.
__device__ __forceinline__ void bulk_copy_g2s(void *dst, const void *src, unsigned bytes,
                                              unsigned long long *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long *bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// The same on 32-bit shared-window addresses (no generic -> shared conversion).
__device__ __forceinline__ void bulk_copy_g2s(uint32_t dst, const void *src, unsigned bytes,
                                              uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
// 32-bit shared-memory integer reduction (RED, no return value).
__device__ __forceinline__ void red_add_shared(uint32_t addr, unsigned v) {
  asm volatile("red.shared.add.u32 [%0], %1;\n" ::"r"(addr), "r"(v));
}
// ... skipped (predicated, no branch) when v == 0.
__device__ __forceinline__ void red_add_shared_nz(uint32_t addr, unsigned v) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p red.shared.add.u32 [%0], %1;\n}\n" ::"r"(
          addr),
      "r"(v));
}

__host__ __device__ inline int pad4(int x) { return (x + 3) & ~3; }

// Kernel arguments shared by the fused kernels.
template <typename Real>
struct FBArgs {
  DevGraphs g;
  const int64_t *row_map;
  int B, T_max, D, S_max, S_pad, D_pad, NC_pad, T_pad;
  const Real *L;
  const int *lengths;
  Real leak;
  Real floor_eff;
  const Real *leak_pi;
  Real *work;
  Real *post;
  int mode;
  const int *other_fail;
  double *logp;
  int *fail;
  double *scale_logs;
  int I_pad;  // tile kernel: per-arc scratch (posterior slots)
  int rep_r, r_stride, rep_e, e_stride;  // tile kernel: gather-vector replication
  int packed;  // 1: L / posteriors are ragged (sum_b T_b, D), item b at row sum_{j<b} T_j
  long long sc_off;    // tile kernel: per-frame scales at work + sc_off + item_off,
  long long sc_total;  //   row maxima sc_total Reals further (ragged, like the trellis)
  int sc_smem;         //   ... or in shared memory (1; set by the launcher when they fit)
  long long *prof;     // split kernel debug timestamps (LFMMI_PROFILE_SPLIT), normally NULL
  // Emissions computed once per step by emit_kernel (chain loss): E = exp(L - m)
  // in L's layout and the row maxima m ((B, T_max) padded / (sum T) packed), or NULL.
  const Real *E;
  const Real *Em;
  int reserve_sms;  // split den kernel: SMs to leave to the concurrent numerator pass (0: default)
  int persist;      // tile den kernel: > 0 = that many persistent CTAs, utterances by in-kernel LPT
};

}  // namespace lfmmi
