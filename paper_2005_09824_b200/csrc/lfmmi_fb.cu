// B200-native LF-MMI forward-backward (sm_100a).
//
// Production path: ONE launch per graph batch, one CTA per utterance, the
// whole time loop on chip (no per-frame launches).  Per frame the CTA does a
// single block barrier:
//   forward  (replaces _kernels.py:54-122): gather over CSR-by-destination,
//            per-frame normaliser by warp-shuffle + fixed-order cross-warp sum,
//            leaky-HMM correction folded into the *next* frame's gather
//            (deferred normalisation), finals at the item's own last frame;
//   backward (replaces _kernels.py:125-191): gather over CSR-by-source with
//            the leak adjoint deferred the same way;
//   posterior + grad (replaces _kernels.py:194-224 and loss.py:67-69): fused
//            into the backward frame loop as a deterministic per-pdf chunked
//            gather, written straight into the gradient row (num pass writes,
//            den pass subtracts).
// Emissions exp(L - max L) (forward_backward.py:120-130) are computed on the
// fly from log-likelihood rows staged two frames ahead with cp.async; the
// scaled alpha column of every frame is spilled to a caller-provided HBM
// workspace during the forward and streamed back (cp.async, double buffer)
// during the backward.
//
// Parity path (f64): lfmmi_{forward,backward,posterior}_kernel mirror the
// numba kernels argument-for-argument with the reference's exact operation
// order (no FMA contraction), for bit-level parity with the reference tests.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdint>
#include <string>

#include "lfmmi_internal.h"

namespace lfmmi {

constexpr unsigned kFull = 0xffffffffu;

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

template <typename Real>
__device__ __forceinline__ const Real *pick(const float *f, const double *d);
template <>
__device__ __forceinline__ const float *pick<float>(const float *f, const double *) { return f; }
template <>
__device__ __forceinline__ const double *pick<double>(const float *, const double *d) { return d; }

__device__ __forceinline__ float exp_r(float x) { return expf(x); }
__device__ __forceinline__ double exp_r(double x) { return exp(x); }

// ---- cp.async (LDGSTS) helpers -------------------------------------------
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
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---- shared-memory layout of the fused kernel ----------------------------
struct SmemLayout {
  int rbuf, ebuf, stage, aring, slots, scales, shifts, part, mpart, reals;
};
constexpr int kScratchBytes = 512;  // 32 doubles + 32 int64

__host__ __device__ inline int pad4(int x) { return (x + 3) & ~3; }

__host__ __device__ inline SmemLayout make_layout(int S_pad, int D_pad, int NC_pad, int T_pad,
                                                  int NW) {
  SmemLayout l;
  int o = 0;
  l.rbuf = o;   o += 2 * S_pad;   // alpha / beta columns (ping-pong)
  l.aring = o;  o += 2 * S_pad;   // alpha columns streamed back from HBM
  l.ebuf = o;   o += 2 * D_pad;   // exp'd emission rows
  l.stage = o;  o += 2 * D_pad;   // raw log-likelihood rows (cp.async)
  l.slots = o;  o += 2 * NC_pad;  // per-chunk posterior partials
  l.scales = o; o += T_pad;       // per-frame normalisers
  l.shifts = o; o += T_pad;       // per-frame max shifts
  l.part = o;   o += pad4(2 * NW);
  l.mpart = o;  o += pad4(2 * NW);
  l.reals = o;
  return l;
}

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
};

// Fused forward + backward + posterior/grad for one utterance per CTA.
template <typename Real, int BLOCK>
__global__ void __launch_bounds__(BLOCK, 1) fb_fused_kernel(const FBArgs<Real> a) {
  constexpr int NW = BLOCK / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *dscr = reinterpret_cast<double *>(smem_raw);
  long long *lscr = reinterpret_cast<long long *>(smem_raw + 256);
  Real *sm = reinterpret_cast<Real *>(smem_raw + kScratchBytes);
  const SmemLayout lay = make_layout(a.S_pad, a.D_pad, a.NC_pad, a.T_pad, NW);
  Real *rbuf = sm + lay.rbuf;
  Real *aring = sm + lay.aring;
  Real *ebuf = sm + lay.ebuf;
  Real *stage = sm + lay.stage;
  Real *slots = sm + lay.slots;
  Real *scales = sm + lay.scales;
  Real *shifts = sm + lay.shifts;
  Real *part = sm + lay.part;
  Real *mpart = sm + lay.mpart;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const int T = a.lengths[b];
  const int D = a.D;
  const int S_pad = a.S_pad, D_pad = a.D_pad, NC_pad = a.NC_pad;
  const int row = int(a.row_map[b]);
  const int *desc = a.g.desc + row * kDescInts;
  const int S = desc[kS], init = desc[kInit], nch = desc[kNumChunks];
  const int aoff = desc[kArcOff], poff = desc[kPtrOff];
  const int *in_ptr = a.g.in_ptr + poff;
  const int *in_src = a.g.in_src + aoff;
  const int *in_pdf = a.g.in_pdf + aoff;
  const Real *in_p = pick<Real>(a.g.in_p32, a.g.in_p64) + aoff;
  const int *out_ptr = a.g.out_ptr + poff;
  const int *out_dst = a.g.out_dst + aoff;
  const int *out_pdf = a.g.out_pdf + aoff;
  const Real *out_p = pick<Real>(a.g.out_p32, a.g.out_p64) + aoff;
  const int *pa_src = a.g.pa_src + aoff;
  const int *pa_dst = a.g.pa_dst + aoff;
  const Real *pa_p = pick<Real>(a.g.pa_p32, a.g.pa_p64) + aoff;
  const int *ch_begin = a.g.chunk_begin + desc[kChunkOff];
  const int *ch_end = a.g.chunk_end + desc[kChunkOff];
  const int *ch_pdf = a.g.chunk_pdf + desc[kChunkOff];
  const int *pdf_cptr = a.g.pdf_chunk_ptr + desc[kPdfPtrOff];
  const Real *fin = pick<Real>(a.g.fin32, a.g.fin64) + desc[kStateOff];
  const Real *Lb = a.L + size_t(b) * a.T_max * D;
  Real *post_b = a.post + size_t(b) * a.T_max * D;
  const bool subtract = a.mode == LFMMI_POST_SUBTRACT;
  const bool other_failed = a.other_fail != nullptr && a.other_fail[b] >= 0;

  // Item offset into the ragged alpha trellis: sum of earlier lengths.
  long long off = 0;
  for (int j = tid; j < b; j += BLOCK) off += a.lengths[j];
  off = warp_sum(off);
  if (lane == 0) lscr[warp] = off;
  // Leak distribution: uniform 1/S_g (forward_backward.py:133-141) or custom.
  const Real *pi = a.leak_pi ? a.leak_pi + size_t(row) * a.S_max : nullptr;
  const Real upi = Real(1.0 / double(S));
  const Real lam = a.leak;
  double psum_d = 0.0;
  if (pi)
    for (int s = tid; s < S; s += BLOCK) psum_d += double(pi[s]);
  psum_d = warp_sum(psum_d);
  if (lane == 0) dscr[warp] = psum_d;
  __syncthreads();
  long long item_off = 0;
  double pisum_d = 0.0;
  for (int w = 0; w < NW; ++w) {
    item_off += lscr[w];
    pisum_d += dscr[w];
  }
  const Real pisum = pi ? Real(pisum_d) : Real(1);
  Real *trellis = a.work + item_off * S_pad;

  if (!subtract) {
    // Padded rows of the posterior output are zero (forward_backward.py:89-92).
    const size_t n = size_t(a.T_max - T) * D;
    for (size_t i = tid; i < n; i += BLOCK) post_b[size_t(T) * D + i] = Real(0);
  }

  // ---- prologue: alpha_0 = onehot(init); emission rows 0 and 1 -------------
  for (int s = tid; s < S; s += BLOCK) rbuf[s] = (s == init) ? Real(1) : Real(0);
  auto issue_row = [&](int t, Real *dst) {
    const Real *src = Lb + size_t(t) * D;
    for (int d = tid; d < D; d += BLOCK) cp_async_elem(dst + d, src + d);
  };
  auto row_max_part = [&](const Real *src, Real *mp) {
    Real m = -INFINITY;
    for (int d = tid; d < D; d += BLOCK) m = fmax(m, src[d]);
    m = warp_max(m);
    if (lane == 0) mp[warp] = m;
  };
  auto block_max = [&](const Real *mp) {
    Real m = -INFINITY;
    for (int w = 0; w < NW; ++w) m = fmax(m, mp[w]);
    return m;
  };
  issue_row(0, stage);
  if (T > 1) issue_row(1, stage + D_pad);
  cp_async_commit();
  cp_async_wait_all();
  row_max_part(stage, mpart);
  if (T > 1) row_max_part(stage + D_pad, mpart + NW);
  __syncthreads();
  {
    const Real m0 = block_max(mpart);
    for (int d = tid; d < D; d += BLOCK) ebuf[d] = exp_r(stage[d] - m0);
    if (tid == 0) shifts[0] = m0;
  }
  __syncthreads();

  // ---- forward: one barrier per frame ---------------------------------------
  Real inv2 = Real(1), leakc = Real(0);
  int fail_at = -1;
  for (int k = 0; k < T; ++k) {
    const int cur = k & 1, nxt = cur ^ 1;
    if (k > 0) {
      Real t0 = Real(0);
      for (int w = 0; w < NW; ++w) t0 += part[cur * NW + w];
      Real t2 = t0;
      leakc = Real(0);
      if (lam > Real(0) && t0 > Real(0)) {
        leakc = lam * t0;
        t2 = t0 + leakc * pisum;
      }
      if (!(t2 >= a.floor_eff) || isinf(t2)) {
        fail_at = k - 1;
        break;
      }
      inv2 = Real(1) / t2;
      if (tid == 0) scales[k - 1] = t2;
    }
    // alpha_k (scaled, leak applied) -> HBM trellis for the backward phase.
    {
      const Real *r = rbuf + cur * S_pad;
      Real *arow = trellis + size_t(k) * S_pad;
      for (int s = tid; s < S; s += BLOCK)
        arow[s] = (r[s] + leakc * (pi ? pi[s] : upi)) * inv2;
    }
    // e_{k+1} from the row staged last frame.
    if (k + 1 < T) {
      const Real m = block_max(mpart + nxt * NW);
      for (int d = tid; d < D; d += BLOCK) ebuf[nxt * D_pad + d] = exp_r(stage[nxt * D_pad + d] - m);
      if (tid == 0) shifts[k + 1] = m;
    }
    if (k + 2 < T) issue_row(k + 2, stage + cur * D_pad);
    cp_async_commit();
    // Gather over in-arcs: raw_{k+1}[s] = sum p * alpha_k[src] * e_k[pdf].
    {
      const Real *e = ebuf + cur * D_pad;
      const Real *r = rbuf + cur * S_pad;
      Real *rn = rbuf + nxt * S_pad;
      const bool last = (k + 1 == T);
      Real psum = Real(0);
      for (int s = tid; s < S; s += BLOCK) {
        const int lo = in_ptr[s], hi = in_ptr[s + 1];
        Real A = Real(0), Bs = Real(0);
        if (leakc != Real(0)) {
          for (int i = lo; i < hi; ++i) {
            const int src = __ldg(in_src + i);
            const Real w = __ldg(in_p + i) * e[__ldg(in_pdf + i)];
            A = fma(w, r[src], A);
            Bs = pi ? fma(w, pi[src], Bs) : Bs + w;
          }
        } else {
          for (int i = lo; i < hi; ++i) {
            const int src = __ldg(in_src + i);
            const Real w = __ldg(in_p + i) * e[__ldg(in_pdf + i)];
            A = fma(w, r[src], A);
          }
        }
        Real raw = inv2 * (A + leakc * (pi ? Bs : upi * Bs));
        if (last) raw *= fin[s];
        rn[s] = raw;
        psum += raw;
      }
      psum = warp_sum(psum);
      if (lane == 0) part[nxt * NW + warp] = psum;
    }
    cp_async_wait_all();
    if (k + 2 < T) row_max_part(stage + cur * D_pad, mpart + cur * NW);
    __syncthreads();
  }
  if (fail_at < 0) {
    Real t0 = Real(0);
    for (int w = 0; w < NW; ++w) t0 += part[(T & 1) * NW + w];
    Real t2 = t0;
    if (lam > Real(0) && t0 > Real(0)) t2 = t0 + lam * t0 * pisum;
    if (!(t2 >= a.floor_eff) || isinf(t2))
      fail_at = T - 1;
    else if (tid == 0)
      scales[T - 1] = t2;
  }
  // Failed items: remaining scales are 1, remaining shifts are still the row
  // maxima (the reference computes emissions for every valid frame).
  if (fail_at >= 0) {
    const int first = fail_at + 1;  // shifts[0..fail_at] were computed in-loop
    for (int k = first + warp; k < T; k += NW) {
      Real m = -INFINITY;
      for (int d = lane; d < D; d += 32) m = fmax(m, Lb[size_t(k) * D + d]);
      m = warp_max(m);
      if (lane == 0) shifts[k] = m;
    }
    for (int k = fail_at + tid; k < T; k += BLOCK) scales[k] = Real(1);
  }
  __syncthreads();

  // log P = sum_t log(scale_t) + shift_t   (forward_backward.py:206-212), in f64.
  {
    double acc = 0.0;
    for (int k = tid; k < T; k += BLOCK) {
      const double v = log(double(scales[k])) + double(shifts[k]);
      acc += v;
      if (a.scale_logs) a.scale_logs[size_t(b) * a.T_max + k] = v;
    }
    if (a.scale_logs)
      for (int k = T + tid; k < a.T_max; k += BLOCK) a.scale_logs[size_t(b) * a.T_max + k] = 0.0;
    acc = warp_sum(acc);
    if (lane == 0) dscr[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < NW; ++w) tot += dscr[w];
      a.logp[b] = fail_at >= 0 ? NAN : tot;
      a.fail[b] = fail_at;
    }
  }

  if (fail_at >= 0 || other_failed) {
    // Failed rows contribute zero gradient (loss.py:67-69, _kernels.py:214).
    const size_t n = size_t(T) * D;
    for (size_t i = tid; i < n; i += BLOCK) post_b[i] = Real(0);
    return;
  }

  // ---- backward + fused posterior / grad write-back --------------------------
  auto write_post = [&](int t, int d, Real g) {
    Real *p = post_b + size_t(t) * D + d;
    *p = subtract ? (*p - g) : g;
  };
  auto issue_alpha = [&](int k, Real *dst) {
    const char *src = reinterpret_cast<const char *>(trellis + size_t(k) * S_pad);
    char *d = reinterpret_cast<char *>(dst);
    const int chunks = S_pad * int(sizeof(Real)) / 16;
    for (int c = tid; c < chunks; c += BLOCK) cp_async_16(d + 16 * c, src + 16 * c);
  };
  auto flush_post = [&](int t, const Real *sl) {
    for (int d = tid; d < D; d += BLOCK) {
      Real g = Real(0);
      const int c1 = pdf_cptr[d + 1];
      for (int c = pdf_cptr[d]; c < c1; ++c) g += sl[c];
      write_post(t, d, g);
    }
  };

  // column T: b_T = final * (1 + leak), leak add 0, inv = 1/scale_{T-1}  (_kernels.py:152-158)
  for (int s = tid; s < S; s += BLOCK) rbuf[(T & 1) * S_pad + s] = fin[s] * (Real(1) + lam);
  issue_alpha(T - 1, aring + ((T - 1) & 1) * S_pad);
  issue_row(T - 1, stage + ((T - 1) & 1) * D_pad);
  if (T >= 2) issue_row(T - 2, stage + ((T - 2) & 1) * D_pad);
  cp_async_commit();
  cp_async_wait_all();
  row_max_part(stage + ((T - 1) & 1) * D_pad, mpart + ((T - 1) & 1) * NW);
  if (T >= 2) row_max_part(stage + ((T - 2) & 1) * D_pad, mpart + ((T - 2) & 1) * NW);
  __syncthreads();
  {
    const int c = (T - 1) & 1;
    const Real m = block_max(mpart + c * NW);
    for (int d = tid; d < D; d += BLOCK) ebuf[c * D_pad + d] = exp_r(stage[c * D_pad + d] - m);
  }
  __syncthreads();

  for (int t = T; t >= 1; --t) {
    const int ct = t & 1, cp = ct ^ 1;
    Real ld = Real(0);
    if (t < T && lam > Real(0)) {
      Real dot = Real(0);
      for (int w = 0; w < NW; ++w) dot += part[ct * NW + w];
      ld = lam * dot;
    }
    const Real inv = Real(1) / scales[t - 1];
    if (t < T) flush_post(t, slots + ct * NC_pad);
    if (t - 2 >= 0) {
      const Real m = block_max(mpart + ct * NW);
      for (int d = tid; d < D; d += BLOCK) ebuf[ct * D_pad + d] = exp_r(stage[ct * D_pad + d] - m);
    }
    if (t - 2 >= 0) issue_alpha(t - 2, aring + ct * S_pad);
    if (t - 3 >= 0) issue_row(t - 3, stage + cp * D_pad);
    cp_async_commit();

    const Real *bt = rbuf + ct * S_pad;
    const Real *e = ebuf + cp * D_pad;
    // (a) beta gather over out-arcs: b_{t-1}[s] = sum p e[pdf] beta_t[dst]
    {
      Real *bn = rbuf + cp * S_pad;
      Real dp = Real(0);
      for (int s = tid; s < S; s += BLOCK) {
        const int lo = out_ptr[s], hi = out_ptr[s + 1];
        Real A = Real(0), C = Real(0);
        for (int i = lo; i < hi; ++i) {
          const Real w = __ldg(out_p + i) * e[__ldg(out_pdf + i)];
          A = fma(w, bt[__ldg(out_dst + i)], A);
          C += w;
        }
        const Real v = inv * (A + ld * C);
        bn[s] = v;
        dp = fma(pi ? pi[s] : upi, v, dp);
      }
      dp = warp_sum(dp);
      if (lane == 0) part[cp * NW + warp] = dp;
    }
    // (b) posterior chunks of frame t-1: e[d]/scale * sum alpha[src] p beta_t[dst]
    {
      const Real *al = aring + cp * S_pad;
      Real *sl = slots + cp * NC_pad;
      for (int c = tid; c < nch; c += BLOCK) {
        const int lo = ch_begin[c], hi = ch_end[c];
        Real P = Real(0), Q = Real(0);
        for (int i = lo; i < hi; ++i) {
          const Real x = al[__ldg(pa_src + i)] * __ldg(pa_p + i);
          P = fma(x, bt[__ldg(pa_dst + i)], P);
          Q += x;
        }
        sl[c] = e[ch_pdf[c]] * inv * (P + ld * Q);
      }
    }
    cp_async_wait_all();
    if (t - 3 >= 0) row_max_part(stage + cp * D_pad, mpart + cp * NW);
    __syncthreads();
  }
  flush_post(0, slots);
}

// ---- f64 parity kernels (exact reference operation order) -----------------
// _kernels.py:54-122.  One CTA per item; per-state sums in CSR order, column
// sums sequential in state order, no FMA contraction.
__global__ void fwd_parity_kernel(DevGraphs g, const int64_t *row_map, int B, int T_max, int D,
                                  int S_max, const double *expl, const int *lengths, double leak,
                                  const double *leak_pi, double floor, double *alpha,
                                  double *scales, int64_t *fail) {
  const int b = blockIdx.x;
  const int row = int(row_map[b]);
  const int *desc = g.desc + row * kDescInts;
  const int S = desc[kS];
  const int *ptr = g.in_ptr + desc[kPtrOff];
  const int *src = g.in_src + desc[kArcOff];
  const int *pdf = g.in_pdf + desc[kArcOff];
  const double *p = g.in_p64 + desc[kArcOff];
  const double *fin = g.fin64 + desc[kStateOff];
  const double *pi = leak_pi + size_t(row) * S_max;
  const int T = lengths[b];
  const size_t T1 = size_t(T_max) + 1;
  __shared__ double s_total;
  __shared__ int s_fail;
  double *al = alpha + size_t(b) * T1 * S_max;
  if (threadIdx.x == 0) {
    al[desc[kInit]] = 1.0;
    s_fail = -1;
  }
  __syncthreads();
  for (int t = 1; t <= T; ++t) {
    const double *prev = al + size_t(t - 1) * S_max;
    double *col = al + size_t(t) * S_max;
    const double *e = expl + (size_t(b) * T_max + (t - 1)) * D;
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
      double acc = 0.0;
      for (int i = ptr[s]; i < ptr[s + 1]; ++i)
        acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(p[i], prev[src[i]]), e[pdf[i]]));
      if (t == T) acc = __dmul_rn(acc, fin[s]);
      col[s] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double total = 0.0;
      for (int s = 0; s < S_max; ++s) total = __dadd_rn(total, col[s]);
      s_total = total;
    }
    __syncthreads();
    double total = s_total;
    if (leak > 0.0 && total > 0.0) {
      for (int s = threadIdx.x; s < S_max; s += blockDim.x)
        col[s] = __dadd_rn(col[s], __dmul_rn(__dmul_rn(leak, pi[s]), total));
      __syncthreads();
      if (threadIdx.x == 0) {
        double t2 = 0.0;
        for (int s = 0; s < S_max; ++s) t2 = __dadd_rn(t2, col[s]);
        s_total = t2;
      }
      __syncthreads();
      total = s_total;
    }
    if (!(total >= floor) || total == INFINITY) {
      for (int s = threadIdx.x; s < S_max; s += blockDim.x) col[s] = 0.0;
      if (threadIdx.x == 0) s_fail = t - 1;
      __syncthreads();
      break;
    }
    const double inv = 1.0 / total;
    for (int s = threadIdx.x; s < S_max; s += blockDim.x) col[s] = __dmul_rn(col[s], inv);
    if (threadIdx.x == 0) scales[size_t(b) * T_max + t - 1] = total;
    __syncthreads();
  }
  if (threadIdx.x == 0) fail[b] = s_fail;
}

// _kernels.py:125-191.
__global__ void bwd_parity_kernel(DevGraphs g, const int64_t *row_map, int B, int T_max, int D,
                                  int S_max, const double *expl, const int *lengths,
                                  const double *scales, double leak, const double *leak_pi,
                                  const int64_t *fail, double *beta) {
  const int b = blockIdx.x;
  if (fail[b] >= 0) return;
  const int row = int(row_map[b]);
  const int *desc = g.desc + row * kDescInts;
  const int S = desc[kS];
  const int *ptr = g.out_ptr + desc[kPtrOff];
  const int *dst = g.out_dst + desc[kArcOff];
  const int *pdf = g.out_pdf + desc[kArcOff];
  const double *p = g.out_p64 + desc[kArcOff];
  const double *fin = g.fin64 + desc[kStateOff];
  const double *pi = leak_pi + size_t(row) * S_max;
  const int T = lengths[b];
  const size_t T1 = size_t(T_max) + 1;
  double *be = beta + size_t(b) * T1 * S_max;
  __shared__ double s_dot;
  {
    const double factor = (1.0 + leak) / scales[size_t(b) * T_max + T - 1];
    for (int s = threadIdx.x; s < S_max; s += blockDim.x)
      be[size_t(T) * S_max + s] = __dmul_rn(s < S ? fin[s] : 0.0, factor);
  }
  __syncthreads();
  for (int t = T; t >= 1; --t) {
    const double *nxt = be + size_t(t) * S_max;
    double *col = be + size_t(t - 1) * S_max;
    const double *e = expl + (size_t(b) * T_max + (t - 1)) * D;
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
      double acc = 0.0;
      for (int i = ptr[s]; i < ptr[s + 1]; ++i)
        acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(p[i], e[pdf[i]]), nxt[dst[i]]));
      col[s] = acc;
    }
    __syncthreads();
    if (t - 1 >= 1) {
      if (leak > 0.0) {
        if (threadIdx.x == 0) {
          double dot = 0.0;
          for (int s = 0; s < S_max; ++s) dot = __dadd_rn(dot, __dmul_rn(pi[s], col[s]));
          s_dot = dot;
        }
        __syncthreads();
        const double add = __dmul_rn(leak, s_dot);
        for (int s = threadIdx.x; s < S_max; s += blockDim.x) col[s] = __dadd_rn(col[s], add);
        __syncthreads();
      }
      const double inv = 1.0 / scales[size_t(b) * T_max + t - 2];
      for (int s = threadIdx.x; s < S_max; s += blockDim.x) col[s] = __dmul_rn(col[s], inv);
      __syncthreads();
    }
  }
}

// _kernels.py:194-224.  One thread per (item, frame); arcs in forward_* order.
__global__ void post_parity_kernel(DevGraphs g, const int64_t *row_map, int B, int T_max, int D,
                                   int S_max, const double *expl, const int *lengths,
                                   const double *alpha, const double *beta, const int64_t *fail,
                                   double *gamma) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= B * T_max) return;
  const int b = u / T_max, t = u % T_max;
  if (t >= lengths[b] || fail[b] >= 0) return;
  const int row = int(row_map[b]);
  const int *desc = g.desc + row * kDescInts;
  const int I = desc[kI];
  const int *ptr = g.out_ptr + desc[kPtrOff];
  const int *dst = g.out_dst + desc[kArcOff];
  const int *pdf = g.out_pdf + desc[kArcOff];
  const double *p = g.out_p64 + desc[kArcOff];
  const size_t T1 = size_t(T_max) + 1;
  const double *at = alpha + (size_t(b) * T1 + t) * S_max;
  const double *bt = beta + (size_t(b) * T1 + t + 1) * S_max;
  const double *e = expl + (size_t(b) * T_max + t) * D;
  double *gm = gamma + (size_t(b) * T_max + t) * D;
  // The out-CSR is the reference forward_* order; recover from-states by row.
  int s = 0;
  for (int i = 0; i < I; ++i) {
    while (ptr[s + 1] <= i) ++s;
    const int d = pdf[i];
    gm[d] = __dadd_rn(gm[d], __dmul_rn(__dmul_rn(__dmul_rn(at[s], p[i]), e[d]), bt[dst[i]]));
  }
}

// Batch totals for chain_loss (loss.py:61-72), fixed-order reduction.
__global__ void totals_kernel(int B, const int *lengths, const double *num_lp, const double *den_lp,
                              const int *num_fail, const int *den_fail, double *totals) {
  __shared__ double so[256], sf[256], sn[256];
  double o = 0.0, f = 0.0, n = 0.0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    if (num_fail[b] < 0 && den_fail[b] < 0) {
      o += num_lp[b] - den_lp[b];
      f += double(lengths[b]);
    } else {
      n += 1.0;
    }
  }
  so[threadIdx.x] = o;
  sf[threadIdx.x] = f;
  sn[threadIdx.x] = n;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) {
      so[threadIdx.x] += so[threadIdx.x + w];
      sf[threadIdx.x] += sf[threadIdx.x + w];
      sn[threadIdx.x] += sn[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    totals[0] = so[0];
    totals[1] = sf[0];
    totals[2] = sn[0];
  }
}

// ---- launch helpers ---------------------------------------------------------
template <typename Real, int BLOCK>
int launch_fused(const FBArgs<Real> &a, size_t smem, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    int rc = check_cuda(cudaFuncSetAttribute(fb_fused_kernel<Real, BLOCK>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024),
                        "cudaFuncSetAttribute");
    if (rc) return rc;
    configured = true;
  }
  fb_fused_kernel<Real, BLOCK><<<a.B, BLOCK, smem, st>>>(a);
  return check_cuda(cudaGetLastError(), "fb_fused_kernel launch");
}

inline int choose_block(const lfmmi_graphs *g) {
  const int want = std::max(g->max_states, g->max_chunks / 2);
  if (want <= 128) return 128;
  if (want <= 256) return 256;
  if (want <= 512) return 512;
  return 1024;
}

template <typename Real>
int run_fused(const lfmmi_graphs *graphs, const int64_t *row_map, int B, int T_max, int D,
              const void *L, const int *lengths, double leak, double floor, const void *leak_pi,
              void *work, size_t work_bytes, void *post, int mode, const int *other_fail,
              double *logp, int *fail, double *scale_logs, cudaStream_t st) {
  FBArgs<Real> a{};
  a.g = graphs->dev;
  a.row_map = row_map;
  a.B = B;
  a.T_max = T_max;
  a.D = D;
  a.S_max = graphs->max_states;
  a.S_pad = pad4(graphs->max_states);
  a.D_pad = pad4(D);
  a.NC_pad = pad4(std::max(1, graphs->max_chunks));
  a.T_pad = pad4(T_max);
  a.L = static_cast<const Real *>(L);
  a.lengths = lengths;
  a.leak = Real(leak);
  a.floor_eff = std::is_same<Real, float>::value ? Real(std::max(floor, double(FLT_MIN)))
                                                 : Real(floor);
  a.leak_pi = static_cast<const Real *>(leak_pi);
  a.work = static_cast<Real *>(work);
  a.post = static_cast<Real *>(post);
  a.mode = mode;
  a.other_fail = other_fail;
  a.logp = logp;
  a.fail = fail;
  a.scale_logs = scale_logs;
  const int block = choose_block(graphs);
  const SmemLayout lay = make_layout(a.S_pad, a.D_pad, a.NC_pad, a.T_pad, block / 32);
  const size_t smem = kScratchBytes + size_t(lay.reals) * sizeof(Real);
  if (smem > 227 * 1024)
    return set_error(LFMMI_ERR_UNSUPPORTED,
                     "graph/utterance too large for the on-chip path: needs " +
                         std::to_string(smem) + " bytes of shared memory");
  if (work_bytes < 16 && B > 0)
    return set_error(LFMMI_ERR_INVALID, "workspace too small");
  switch (block) {
    case 128: return launch_fused<Real, 128>(a, smem, st);
    case 256: return launch_fused<Real, 256>(a, smem, st);
    case 512: return launch_fused<Real, 512>(a, smem, st);
    default: return launch_fused<Real, 1024>(a, smem, st);
  }
}

}  // namespace lfmmi

using namespace lfmmi;

extern "C" size_t lfmmi_workspace_size(int32_t max_states, int64_t total_frames,
                                       int32_t precision) {
  const size_t es = precision == LFMMI_F64 ? 8 : 4;
  return size_t(pad4(std::max(1, int(max_states)))) * size_t(std::max<int64_t>(total_frames, 1)) *
             es + 256;
}

static int check_common(const lfmmi_graphs *graphs, int32_t batch, int32_t max_frames,
                        int32_t num_pdfs, int32_t precision) {
  if (!graphs) return set_error(LFMMI_ERR_INVALID, "graph handle is NULL");
  if (batch < 1 || max_frames < 1) return set_error(LFMMI_ERR_INVALID, "empty batch");
  if (num_pdfs != graphs->num_pdfs)
    return set_error(LFMMI_ERR_INVALID,
                     "pdf dimension mismatch: batch has " + std::to_string(num_pdfs) +
                         ", graphs have " + std::to_string(graphs->num_pdfs));
  if (precision != LFMMI_F32 && precision != LFMMI_F64)
    return set_error(LFMMI_ERR_INVALID, "precision must be LFMMI_F32 or LFMMI_F64");
  return LFMMI_OK;
}

extern "C" int lfmmi_forward_backward(const lfmmi_graphs *graphs, const int64_t *row_map,
                                      int32_t batch, int32_t max_frames, int32_t num_pdfs,
                                      int32_t precision, const void *loglikes,
                                      const int32_t *lengths, double leak, double scale_floor,
                                      const void *leak_pi, void *workspace,
                                      size_t workspace_bytes, void *posteriors,
                                      int32_t post_mode, const int32_t *other_fail,
                                      double *log_probs, int32_t *fail_frames,
                                      double *scale_logs, void *stream) {
  int rc = check_common(graphs, batch, max_frames, num_pdfs, precision);
  if (rc) return rc;
  if (!row_map || !loglikes || !lengths || !workspace || !posteriors || !log_probs || !fail_frames)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_forward_backward: NULL device pointer");
  if (!(leak >= 0.0) || !(scale_floor > 0.0))
    return set_error(LFMMI_ERR_INVALID, "leak must be >= 0 and scale_floor > 0");
  auto st = static_cast<cudaStream_t>(stream);
  if (precision == LFMMI_F64)
    return run_fused<double>(graphs, row_map, batch, max_frames, num_pdfs, loglikes, lengths, leak,
                             scale_floor, leak_pi, workspace, workspace_bytes, posteriors,
                             post_mode, other_fail, log_probs, fail_frames, scale_logs, st);
  return run_fused<float>(graphs, row_map, batch, max_frames, num_pdfs, loglikes, lengths, leak,
                          scale_floor, leak_pi, workspace, workspace_bytes, posteriors, post_mode,
                          other_fail, log_probs, fail_frames, scale_logs, st);
}

extern "C" int lfmmi_chain_loss(const lfmmi_graphs *numerators, const int64_t *num_row_map,
                                const lfmmi_graphs *denominator, const int64_t *den_row_map,
                                int32_t batch, int32_t max_frames, int32_t num_pdfs,
                                int32_t precision, const void *loglikes, const int32_t *lengths,
                                double leak, double scale_floor, const void *num_leak_pi,
                                const void *den_leak_pi, void *workspace, size_t workspace_bytes,
                                void *grad, double *num_log_probs, double *den_log_probs,
                                int32_t *num_fail, int32_t *den_fail, double *totals,
                                void *stream) {
  int rc = lfmmi_forward_backward(numerators, num_row_map, batch, max_frames, num_pdfs, precision,
                                  loglikes, lengths, leak, scale_floor, num_leak_pi, workspace,
                                  workspace_bytes, grad, LFMMI_POST_WRITE, nullptr, num_log_probs,
                                  num_fail, nullptr, stream);
  if (rc) return rc;
  rc = lfmmi_forward_backward(denominator, den_row_map, batch, max_frames, num_pdfs, precision,
                              loglikes, lengths, leak, scale_floor, den_leak_pi, workspace,
                              workspace_bytes, grad, LFMMI_POST_SUBTRACT, num_fail, den_log_probs,
                              den_fail, nullptr, stream);
  if (rc) return rc;
  if (totals) {
    totals_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        batch, lengths, num_log_probs, den_log_probs, num_fail, den_fail, totals);
    rc = check_cuda(cudaGetLastError(), "totals_kernel launch");
  }
  return rc;
}

extern "C" int lfmmi_forward_kernel(const lfmmi_graphs *graphs, const int64_t *row_map,
                                    int32_t batch, int32_t max_frames, int32_t num_pdfs,
                                    const double *expl, const int32_t *lengths, double leak,
                                    const double *leak_pi, double scale_floor, double *alpha,
                                    double *scales, int64_t *fail_frames, void *stream) {
  int rc = check_common(graphs, batch, max_frames, num_pdfs, LFMMI_F64);
  if (rc) return rc;
  if (!leak_pi) return set_error(LFMMI_ERR_INVALID, "parity kernels need an explicit leak_pi");
  fwd_parity_kernel<<<batch, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      graphs->dev, row_map, batch, max_frames, num_pdfs, graphs->max_states, expl, lengths, leak,
      leak_pi, scale_floor, alpha, scales, fail_frames);
  return check_cuda(cudaGetLastError(), "fwd_parity_kernel launch");
}

extern "C" int lfmmi_backward_kernel(const lfmmi_graphs *graphs, const int64_t *row_map,
                                     int32_t batch, int32_t max_frames, int32_t num_pdfs,
                                     const double *expl, const int32_t *lengths,
                                     const double *scales, double leak, const double *leak_pi,
                                     const int64_t *fail_frames, double *beta, void *stream) {
  int rc = check_common(graphs, batch, max_frames, num_pdfs, LFMMI_F64);
  if (rc) return rc;
  if (!leak_pi) return set_error(LFMMI_ERR_INVALID, "parity kernels need an explicit leak_pi");
  bwd_parity_kernel<<<batch, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      graphs->dev, row_map, batch, max_frames, num_pdfs, graphs->max_states, expl, lengths, scales,
      leak, leak_pi, fail_frames, beta);
  return check_cuda(cudaGetLastError(), "bwd_parity_kernel launch");
}

extern "C" int lfmmi_posterior_kernel(const lfmmi_graphs *graphs, const int64_t *row_map,
                                      int32_t batch, int32_t max_frames, int32_t num_pdfs,
                                      const double *expl, const int32_t *lengths,
                                      const double *alpha, const double *beta,
                                      const int64_t *fail_frames, double *gamma, void *stream) {
  int rc = check_common(graphs, batch, max_frames, num_pdfs, LFMMI_F64);
  if (rc) return rc;
  const int n = batch * max_frames;
  post_parity_kernel<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      graphs->dev, row_map, batch, max_frames, num_pdfs, graphs->max_states, expl, lengths, alpha,
      beta, fail_frames, gamma);
  return check_cuda(cudaGetLastError(), "post_parity_kernel launch");
}
