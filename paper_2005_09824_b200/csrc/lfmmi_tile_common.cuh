// Shared-memory helpers of the tile kernels (fb_tile_kernel, fb_split_kernel):
// explicitly scheduled fp32 arc loops over byte-offset slot words.
#pragma once

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
__device__ __forceinline__ void sts_f(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(a), "f"(v));
}

// Forward arc sums of one tile lane, fp32 (slots hold byte-offset words):
// A = sum p e[pdf] r[src], Bs = sum p e[pdf] (leak mass, uniform pi).
template <bool LEAKY>
__device__ __forceinline__ void fwd_tile_f32(uint32_t sb, int trips, uint32_t e32, uint32_t r32,
                                             float &A, float &Bs) {
  int j = 0;
#pragma unroll 1
  for (; j + 4 <= trips; j += 4, sb += 4 * 256) {
    const uint2 w0 = lds_v2(sb), w1 = lds_v2(sb + 256), w2 = lds_v2(sb + 512),
                w3 = lds_v2(sb + 768);
    const float e0 = lds_f(e32 + (w0.x >> 16)), e1 = lds_f(e32 + (w1.x >> 16)),
                e2 = lds_f(e32 + (w2.x >> 16)), e3 = lds_f(e32 + (w3.x >> 16));
    const float r0 = lds_f(r32 + (w0.x & 0xFFFFu)), r1 = lds_f(r32 + (w1.x & 0xFFFFu)),
                r2 = lds_f(r32 + (w2.x & 0xFFFFu)), r3 = lds_f(r32 + (w3.x & 0xFFFFu));
    const float q0 = __uint_as_float(w0.y) * e0, q1 = __uint_as_float(w1.y) * e1,
                q2 = __uint_as_float(w2.y) * e2, q3 = __uint_as_float(w3.y) * e3;
    A = fmaf(q0, r0, A);
    A = fmaf(q1, r1, A);
    A = fmaf(q2, r2, A);
    A = fmaf(q3, r3, A);
    if (LEAKY) Bs += (q0 + q1) + (q2 + q3);
  }
  // Remainder (trips % 4 rows) without a loop: at most one pair and one single.
  if (j + 2 <= trips) {
    const uint2 w0 = lds_v2(sb), w1 = lds_v2(sb + 256);
    const float e0 = lds_f(e32 + (w0.x >> 16)), e1 = lds_f(e32 + (w1.x >> 16));
    const float r0 = lds_f(r32 + (w0.x & 0xFFFFu)), r1 = lds_f(r32 + (w1.x & 0xFFFFu));
    const float q0 = __uint_as_float(w0.y) * e0, q1 = __uint_as_float(w1.y) * e1;
    A = fmaf(q0, r0, A);
    A = fmaf(q1, r1, A);
    if (LEAKY) Bs += q0 + q1;
    j += 2;
    sb += 2 * 256;
  }
  if (j < trips) {
    const uint2 w = lds_v2(sb);
    const float q = __uint_as_float(w.y) * lds_f(e32 + (w.x >> 16));
    A = fmaf(q, lds_f(r32 + (w.x & 0xFFFFu)), A);
    if (LEAKY) Bs += q;
  }
}

// Backward arc sums of one tile lane, fp32: term = p e[pdf] (b[dst] + ld);
// A = sum term, posterior slot xs <- as * term.
__device__ __forceinline__ float bwd_tile_f32(uint32_t sb, uint32_t xb, int trips, uint32_t e32,
                                              uint32_t b32, uint32_t x32, float ld, float as) {
  float A = 0.f;
  int j = 0;
#pragma unroll 1
  for (; j + 4 <= trips; j += 4, sb += 4 * 256, xb += 4 * 64) {
    const uint2 w0 = lds_v2(sb), w1 = lds_v2(sb + 256), w2 = lds_v2(sb + 512),
                w3 = lds_v2(sb + 768);
    const uint32_t x0 = lds_h(xb), x1 = lds_h(xb + 64), x2 = lds_h(xb + 128),
                   x3 = lds_h(xb + 192);
    const float e0 = lds_f(e32 + (w0.x >> 16)), e1 = lds_f(e32 + (w1.x >> 16)),
                e2 = lds_f(e32 + (w2.x >> 16)), e3 = lds_f(e32 + (w3.x >> 16));
    const float b0 = lds_f(b32 + (w0.x & 0xFFFFu)), b1 = lds_f(b32 + (w1.x & 0xFFFFu)),
                b2 = lds_f(b32 + (w2.x & 0xFFFFu)), b3 = lds_f(b32 + (w3.x & 0xFFFFu));
    const float t0 = __uint_as_float(w0.y) * e0 * (b0 + ld),
                t1 = __uint_as_float(w1.y) * e1 * (b1 + ld),
                t2 = __uint_as_float(w2.y) * e2 * (b2 + ld),
                t3 = __uint_as_float(w3.y) * e3 * (b3 + ld);
    A += (t0 + t1) + (t2 + t3);
    sts_f(x32 + 4 * x0, as * t0);
    sts_f(x32 + 4 * x1, as * t1);
    sts_f(x32 + 4 * x2, as * t2);
    sts_f(x32 + 4 * x3, as * t3);
  }
  if (j + 2 <= trips) {
    const uint2 w0 = lds_v2(sb), w1 = lds_v2(sb + 256);
    const uint32_t x0 = lds_h(xb), x1 = lds_h(xb + 64);
    const float e0 = lds_f(e32 + (w0.x >> 16)), e1 = lds_f(e32 + (w1.x >> 16));
    const float b0 = lds_f(b32 + (w0.x & 0xFFFFu)), b1 = lds_f(b32 + (w1.x & 0xFFFFu));
    const float t0 = __uint_as_float(w0.y) * e0 * (b0 + ld),
                t1 = __uint_as_float(w1.y) * e1 * (b1 + ld);
    A += t0 + t1;
    sts_f(x32 + 4 * x0, as * t0);
    sts_f(x32 + 4 * x1, as * t1);
    j += 2;
    sb += 2 * 256;
    xb += 2 * 64;
  }
  if (j < trips) {
    const uint2 w = lds_v2(sb);
    const uint32_t x = lds_h(xb);
    const float t = __uint_as_float(w.y) * lds_f(e32 + (w.x >> 16)) *
                    (lds_f(b32 + (w.x & 0xFFFFu)) + ld);
    A += t;
    sts_f(x32 + 4 * x, as * t);
  }
  return A;
}

// Forward arc sums with posterior slots (fb_split_kernel, second half of the
// forward CTA): term = p e[pdf] (r[src] + lu); A = sum term; slot xs <- cb * term
// (cb = beta(dst) / scale, one value per lane).
__device__ __forceinline__ float fwd_post_tile_f32(uint32_t sb, uint32_t xb, int trips,
                                                   uint32_t e32, uint32_t r32, uint32_t x32,
                                                   float lu, float cb) {
  float A = 0.f;
  int j = 0;
#pragma unroll 1
  for (; j + 4 <= trips; j += 4, sb += 4 * 256, xb += 4 * 64) {
    const uint2 w0 = lds_v2(sb), w1 = lds_v2(sb + 256), w2 = lds_v2(sb + 512),
                w3 = lds_v2(sb + 768);
    const uint32_t x0 = lds_h(xb), x1 = lds_h(xb + 64), x2 = lds_h(xb + 128),
                   x3 = lds_h(xb + 192);
    const float e0 = lds_f(e32 + (w0.x >> 16)), e1 = lds_f(e32 + (w1.x >> 16)),
                e2 = lds_f(e32 + (w2.x >> 16)), e3 = lds_f(e32 + (w3.x >> 16));
    const float r0 = lds_f(r32 + (w0.x & 0xFFFFu)), r1 = lds_f(r32 + (w1.x & 0xFFFFu)),
                r2 = lds_f(r32 + (w2.x & 0xFFFFu)), r3 = lds_f(r32 + (w3.x & 0xFFFFu));
    const float t0 = __uint_as_float(w0.y) * e0 * (r0 + lu),
                t1 = __uint_as_float(w1.y) * e1 * (r1 + lu),
                t2 = __uint_as_float(w2.y) * e2 * (r2 + lu),
                t3 = __uint_as_float(w3.y) * e3 * (r3 + lu);
    A += (t0 + t1) + (t2 + t3);
    sts_f(x32 + 4 * x0, cb * t0);
    sts_f(x32 + 4 * x1, cb * t1);
    sts_f(x32 + 4 * x2, cb * t2);
    sts_f(x32 + 4 * x3, cb * t3);
  }
  if (j + 2 <= trips) {
    const uint2 w0 = lds_v2(sb), w1 = lds_v2(sb + 256);
    const uint32_t x0 = lds_h(xb), x1 = lds_h(xb + 64);
    const float e0 = lds_f(e32 + (w0.x >> 16)), e1 = lds_f(e32 + (w1.x >> 16));
    const float r0 = lds_f(r32 + (w0.x & 0xFFFFu)), r1 = lds_f(r32 + (w1.x & 0xFFFFu));
    const float t0 = __uint_as_float(w0.y) * e0 * (r0 + lu),
                t1 = __uint_as_float(w1.y) * e1 * (r1 + lu);
    A += t0 + t1;
    sts_f(x32 + 4 * x0, cb * t0);
    sts_f(x32 + 4 * x1, cb * t1);
    j += 2;
    sb += 2 * 256;
    xb += 2 * 64;
  }
  if (j < trips) {
    const uint2 w = lds_v2(sb);
    const uint32_t x = lds_h(xb);
    const float t = __uint_as_float(w.y) * lds_f(e32 + (w.x >> 16)) *
                    (lds_f(r32 + (w.x & 0xFFFFu)) + lu);
    A += t;
    sts_f(x32 + 4 * x, cb * t);
  }
  return A;
}

// Backward arc sums without posterior slots (fb_split_kernel, first half of the
// backward CTA): A = sum p e[pdf] (b[dst] + ld).
__device__ __forceinline__ float bwd_plain_tile_f32(uint32_t sb, int trips, uint32_t e32,
                                                    uint32_t b32, float ld) {
  float A = 0.f;
  int j = 0;
#pragma unroll 1
  for (; j + 4 <= trips; j += 4, sb += 4 * 256) {
    const uint2 w0 = lds_v2(sb), w1 = lds_v2(sb + 256), w2 = lds_v2(sb + 512),
                w3 = lds_v2(sb + 768);
    const float e0 = lds_f(e32 + (w0.x >> 16)), e1 = lds_f(e32 + (w1.x >> 16)),
                e2 = lds_f(e32 + (w2.x >> 16)), e3 = lds_f(e32 + (w3.x >> 16));
    const float b0 = lds_f(b32 + (w0.x & 0xFFFFu)), b1 = lds_f(b32 + (w1.x & 0xFFFFu)),
                b2 = lds_f(b32 + (w2.x & 0xFFFFu)), b3 = lds_f(b32 + (w3.x & 0xFFFFu));
    A += (__uint_as_float(w0.y) * e0 * (b0 + ld) + __uint_as_float(w1.y) * e1 * (b1 + ld)) +
         (__uint_as_float(w2.y) * e2 * (b2 + ld) + __uint_as_float(w3.y) * e3 * (b3 + ld));
  }
  if (j + 2 <= trips) {
    const uint2 w0 = lds_v2(sb), w1 = lds_v2(sb + 256);
    const float e0 = lds_f(e32 + (w0.x >> 16)), e1 = lds_f(e32 + (w1.x >> 16));
    const float b0 = lds_f(b32 + (w0.x & 0xFFFFu)), b1 = lds_f(b32 + (w1.x & 0xFFFFu));
    A += __uint_as_float(w0.y) * e0 * (b0 + ld) + __uint_as_float(w1.y) * e1 * (b1 + ld);
    j += 2;
    sb += 2 * 256;
  }
  if (j < trips) {
    const uint2 w = lds_v2(sb);
    A += __uint_as_float(w.y) * lds_f(e32 + (w.x >> 16)) * (lds_f(b32 + (w.x & 0xFFFFu)) + ld);
  }
  return A;
}

}  // namespace lfmmi
