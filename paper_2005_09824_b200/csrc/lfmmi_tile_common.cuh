// Shared-memory helpers of the tile kernels (fb_tile_kernel, fb_split_kernel):
// explicitly scheduled fp32 arc loops over byte-offset slot words.
#pragma once

#include <type_traits>

#include "lfmmi_device.cuh"

namespace lfmmi {

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// Slot storage per phase: fp32 -> uint2 (word, prob bits) [+ u16 xslot];
// fp64 -> u32 word + f64 prob [+ u16 xslot].

// Sum of n4 groups of 4 consecutive values (16/32-byte aligned), 4 accumulators.
__device__ __forceinline__ float sum_groups4(const float *x, int n4) {
  const float4 *q = reinterpret_cast<const float4 *>(x);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  for (int i = 0; i < n4; ++i) {
    const float4 v = q[i];
    s0 += v.x;
    s1 += v.y;
    s2 += v.z;
    s3 += v.w;
  }
  return (s0 + s1) + (s2 + s3);
}
__device__ __forceinline__ double sum_groups4(const double *x, int n4) {
  const double2 *q = reinterpret_cast<const double2 *>(x);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int i = 0; i < n4; ++i) {
    const double2 v = q[2 * i], w = q[2 * i + 1];
    s0 += v.x;
    s1 += v.y;
    s2 += w.x;
    s3 += w.y;
  }
  return (s0 + s1) + (s2 + s3);
}

template <int BLOCK>
__device__ __forceinline__ void copy16(void *dst, const void *src, size_t bytes, int tid) {
  const int4 *s = static_cast<const int4 *>(src);
  int4 *d = static_cast<int4 *>(dst);
  const int n = int(bytes >> 4);
  for (int c = tid; c < n; c += BLOCK) cp_async_16(d + c, s + c);
}

// Sum of the NW (<= 32) per-warp partials in v, identical in every lane.
template <int NW, typename Real>
__device__ __forceinline__ Real lane_sum(const Real *v, int lane) {
  if constexpr (NW == 1) {
    return v[0];
  } else {
    Real x = lane < NW ? v[lane] : Real(0);
    return warp_sum(x);
  }
}

// Sum over the G (power of 2) adjacent lanes that share one state of a tile
// pack (kTileG); every lane of the group gets the same value.
template <typename Real>
__device__ __forceinline__ Real group_sum(Real v, int G) {
  for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

struct SlotF32 {
  const uint2 *wp;
  __device__ __forceinline__ void load(int slot, unsigned &w, float &p) const {
    const uint2 v = wp[slot];
    w = ((v.x & 0xFFFFu) >> 2) | ((v.x >> 18) << 16);  // byte offsets -> indices
    p = __uint_as_float(v.y);
  }
};
struct SlotF64 {
  const unsigned *w;
  const double *p;
  __device__ __forceinline__ void load(int slot, unsigned &ww, double &pp) const {
    ww = w[slot];
    pp = p[slot];
  }
};
template <typename Real>
struct SlotOf;
template <>
struct SlotOf<float> { using type = SlotF32; };
template <>
struct SlotOf<double> { using type = SlotF64; };

// ---- 32-bit shared-space accessors (explicitly scheduled fp32 inner loops) ----
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_h(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];\n" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_v2(uint32_t a, uint2 v) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(a), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void sts_f(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(a), "f"(v));
}

// Pairwise sum of N terms ((t0 + t1) + (t2 + t3) for N = 4: the order the
// 4-row loops always used, so N = 4 builds are bit-identical to before).
template <int N>
__device__ __forceinline__ float pair_sum(const float *t) {
  if constexpr (N == 1) {
    return t[0];
  } else {
    return pair_sum<N / 2>(t) + pair_sum<N / 2>(t + N / 2);
  }
}

// Slot rows per unrolled step of the arc loops below: every step issues all of
// its slot-word loads, then all emission / column gathers, then the math, so a
// warp keeps 3 x kSlotRows shared loads in flight (build-time: -DLFMMI_SLOT_ROWS).
#ifndef LFMMI_SLOT_ROWS
#define LFMMI_SLOT_ROWS 4
#endif
constexpr int kSlotRows = LFMMI_SLOT_ROWS;
static_assert(kSlotRows == 4 || kSlotRows == 8, "slot rows per step: 4 or 8");

// Runs body<N>(row offset) over `trips` slot rows: steps of kSlotRows, then the
// remainder as at most one 4-, one 2- and one 1-row step (no remainder loop).
template <typename F>
__device__ __forceinline__ void slot_rows(int trips, F &&body) {
  int j = 0;
#pragma unroll 1
  for (; j + kSlotRows <= trips; j += kSlotRows) body(j, std::integral_constant<int, kSlotRows>{});
  if constexpr (kSlotRows > 4) {
    if (j + 4 <= trips) {
      body(j, std::integral_constant<int, 4>{});
      j += 4;
    }
  }
  if (j + 2 <= trips) {
    body(j, std::integral_constant<int, 2>{});
    j += 2;
  }
  if (j < trips) body(j, std::integral_constant<int, 1>{});
}

// Forward arc sums of one tile lane, fp32 (slots hold byte-offset words):
// A = sum p e[pdf] r[src], Bs = sum p e[pdf] (leak mass, uniform pi).
template <bool LEAKY>
__device__ __forceinline__ void fwd_tile_f32(uint32_t sb, int trips, uint32_t e32, uint32_t r32,
                                             float &A, float &Bs) {
  slot_rows(trips, [&](int j, auto n) {
    constexpr int N = decltype(n)::value;
    uint2 w[N];
    float e[N], r[N];
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = lds_v2(sb + uint32_t(j + i) * 256u);
#pragma unroll
    for (int i = 0; i < N; ++i) e[i] = lds_f(e32 + (w[i].x >> 16));
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = lds_f(r32 + (w[i].x & 0xFFFFu));
    float q[N];
#pragma unroll
    for (int i = 0; i < N; ++i) q[i] = __uint_as_float(w[i].y) * e[i];
#pragma unroll
    for (int i = 0; i < N; ++i) A = fmaf(q[i], r[i], A);
    if (LEAKY) Bs += pair_sum<N>(q);
  });
}

// Backward arc sums of one tile lane, fp32: term = p e[pdf] (b[dst] + ld);
// A = sum term, posterior slot xs <- as * term.
__device__ __forceinline__ float bwd_tile_f32(uint32_t sb, uint32_t xb, int trips, uint32_t e32,
                                              uint32_t b32, uint32_t x32, float ld, float as) {
  float A = 0.f;
  slot_rows(trips, [&](int j, auto n) {
    constexpr int N = decltype(n)::value;
    uint2 w[N];
    uint32_t x[N];
    float e[N], bb[N], t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = lds_v2(sb + uint32_t(j + i) * 256u);
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = lds_h(xb + uint32_t(j + i) * 64u);
#pragma unroll
    for (int i = 0; i < N; ++i) e[i] = lds_f(e32 + (w[i].x >> 16));
#pragma unroll
    for (int i = 0; i < N; ++i) bb[i] = lds_f(b32 + (w[i].x & 0xFFFFu));
#pragma unroll
    for (int i = 0; i < N; ++i) t[i] = __uint_as_float(w[i].y) * e[i] * (bb[i] + ld);
    A += pair_sum<N>(t);
#pragma unroll
    for (int i = 0; i < N; ++i) sts_f(x32 + 4 * x[i], as * t[i]);
  });
  return A;
}

// Forward arc sums with posterior slots (fb_split_kernel, second half of the
// forward CTA): term = p e[pdf] (r[src] + lu); A = sum term; slot xs <- cb * term
// (cb = beta(dst) / scale, one value per lane).
__device__ __forceinline__ float fwd_post_tile_f32(uint32_t sb, uint32_t xb, int trips,
                                                   uint32_t e32, uint32_t r32, uint32_t x32,
                                                   float lu, float cb) {
  float A = 0.f;
  slot_rows(trips, [&](int j, auto n) {
    constexpr int N = decltype(n)::value;
    uint2 w[N];
    uint32_t x[N];
    float e[N], r[N], t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = lds_v2(sb + uint32_t(j + i) * 256u);
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = lds_h(xb + uint32_t(j + i) * 64u);
#pragma unroll
    for (int i = 0; i < N; ++i) e[i] = lds_f(e32 + (w[i].x >> 16));
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = lds_f(r32 + (w[i].x & 0xFFFFu));
#pragma unroll
    for (int i = 0; i < N; ++i) t[i] = __uint_as_float(w[i].y) * e[i] * (r[i] + lu);
    A += pair_sum<N>(t);
#pragma unroll
    for (int i = 0; i < N; ++i) sts_f(x32 + 4 * x[i], cb * t[i]);
  });
  return A;
}

// Backward arc sums without posterior slots (fb_split_kernel, first half of the
// backward CTA): A = sum p e[pdf] (b[dst] + ld).
__device__ __forceinline__ float bwd_plain_tile_f32(uint32_t sb, int trips, uint32_t e32,
                                                    uint32_t b32, float ld) {
  float A = 0.f;
  slot_rows(trips, [&](int j, auto n) {
    constexpr int N = decltype(n)::value;
    uint2 w[N];
    float e[N], bb[N], t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = lds_v2(sb + uint32_t(j + i) * 256u);
#pragma unroll
    for (int i = 0; i < N; ++i) e[i] = lds_f(e32 + (w[i].x >> 16));
#pragma unroll
    for (int i = 0; i < N; ++i) bb[i] = lds_f(b32 + (w[i].x & 0xFFFFu));
#pragma unroll
    for (int i = 0; i < N; ++i) t[i] = __uint_as_float(w[i].y) * e[i] * (bb[i] + ld);
    A += pair_sum<N>(t);
  });
  return A;
}

}  // namespace lfmmi
