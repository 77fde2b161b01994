// Linear-chain forward-backward: the numerator pass.
//
// The reference's numerator graphs are linear chains (build_numerator,
// /root/reference/pkg/src/chainloss/toy_builder.py:218-265): state 0 enters
// phone 1, state k has one self-loop and one arc to k+1.  For such a graph
// the sparse recursion of _kernels.py:54-191 collapses to a two-term stencil
//
//   raw_{t+1}[s] = w_self_t[s] * alpha_t[s] + w_in_t[s] * alpha_t[s-1]
//   X_{t-1}[s]   = w_self_t[s] * beta_t[s]  + w_in_t[s+1] * beta_t[s+1]
//
// (w = p * exp(L[t, pdf] - max_d L[t, d])), so one warp runs an utterance with
// its states in registers: lane l owns states [l K, l K + K), the s-1 / s+1
// neighbours crossing a lane boundary come from one shuffle, and the only
// cross-lane reductions are the per-frame normaliser (forward) and the
// leaky-HMM dot product (backward).  Both are deferred (the stencil runs on
// the unnormalised column and the scalars are folded in afterwards), so a
// frame's critical path is one warp reduction plus a few FMAs.  No block
// barrier, no arc tables in shared memory.
//
// Semantics follow the reference exactly: finals at t == T (:97-98), uniform
// leak pi = 1/S (forward_backward.py:133-166 default) re-normalised by
// tot = R (1 + leak) (:108-113), failure when !(tot >= floor) or tot == inf
// (:114-118), beta_T = final (1 + leak) / scale_{T-1} (:152-158), the leak
// adjoint and 1/scale_{t-2} in the backward (:177-191), and posteriors
// gamma[t, d] = sum_{pdf_i = d} alpha_t[src] p_i e[t, d] beta_{t+1}[dst]
// (:211-224), accumulated per frame in a per-warp shared-memory histogram as
// 2^-28 fixed-point integers (order-independent => deterministic).
//
// Log-likelihood rows are staged by cp.async kRing-1 frames ahead (coalesced
// 16-byte chunks), alpha rows of the backward likewise; the row maximum is
// taken from the staged row (NaN-propagating, forward_backward.py:126).
#include "lfmmi_device.cuh"
#include "lfmmi_kernels.h"
#include "lfmmi_options.h"

#include <algorithm>

namespace lfmmi {
namespace {

constexpr int kRing = 4;                       // cp.async stages (frames in flight + 1)
constexpr float kFix = 268435456.0f;           // 2^28: posterior fixed-point scale
constexpr float kUnfix = 1.0f / 268435456.0f;

struct LinLayout {
  int T4, Dr, stage;  // floats
  size_t bytes;
};

__host__ __device__ inline LinLayout lin_layout(int T_max, int D, int K) {
  LinLayout l;
  l.T4 = pad4(T_max);
  l.Dr = pad4(D);
  l.stage = l.Dr + 32 * K;
  // scales[T4] | shifts[T4] | histogram[Dr] (u32) | ring[kRing][stage]
  l.bytes = size_t(2 * l.T4 + l.Dr + kRing * l.stage) * 4;
  return l;
}

// K of one utterance: lanes own K states each, the smallest power of two with
// 32 K >= S.  Chosen per utterance (not per batch), so an utterance's result
// never depends on its batch-mates (bitwise batch independence).
__device__ __forceinline__ int k_of(int S) {
  return S <= 32 ? 1 : S <= 64 ? 2 : S <= 128 ? 4 : S <= 256 ? 8 : 16;
}

// PRE: the step's emissions E = exp(L - m) and row maxima come from emit_kernel
// (chain loss), so a frame stages the E row and gathers it — no row maximum,
// no exp; otherwise both are computed here from the staged L row.
template <int K, bool PRE>
__device__ __forceinline__ void linear_item(const FBArgs<float> &a, float *lsm,
                                            const LinLayout &lay, int b) {
  const int lane = threadIdx.x;
  const int D = a.D, T_max = a.T_max;
  float *scl = lsm;                    // per-frame scales (forward normalisers)
  float *shf = lsm + lay.T4;           // per-frame row maxima
  unsigned *hist = reinterpret_cast<unsigned *>(lsm + 2 * lay.T4);
  float *ring = lsm + 2 * lay.T4 + lay.Dr;
  const int mode = a.mode;
  const bool reads_post = mode == kPostAdd || mode == kPostSubtract;

  // Row offset of this item in the ragged trellis (and in L / post when packed).
  long long off = 0;
  for (int j = lane; j < b; j += 32) off += a.packed ? a.lengths[j] : item_frames(a.lengths, j, T_max);
  off = warp_sum(off);
  const int T = item_frames(a.lengths, b, T_max);
  const size_t row0 = a.packed ? size_t(off) : size_t(b) * T_max;
  const float *Lb = (PRE ? a.E : a.L) + row0 * D;
  const float *Emb = PRE ? a.Em + (a.packed ? size_t(off) : size_t(b) * T_max) : nullptr;
  float *post_b = a.post + row0 * D;
  if (!reads_post && !a.packed)  // padded rows of this item
    for (size_t i = lane; i < size_t(T_max - T) * D; i += 32) post_b[size_t(T) * D + i] = 0.f;
  if (T <= 0) {  // zero-length (or out-of-range) item: failed, no frames touched
    if (a.scale_logs && !a.packed)
      for (int k = lane; k < T_max; k += 32) a.scale_logs[size_t(b) * T_max + k] = 0.0;
    if (lane == 0) {
      a.logp[b] = NAN;
      a.fail[b] = 0;
    }
    return;
  }
  const int ld = (a.S_max + 31) & ~31;  // trellis row stride (lfmmi_workspace_size)
  float *tr = a.work + size_t(off) * ld;
  const bool own_row = lane * K < ld;

  // ---- graph: two arcs per state, in registers ----------------------------------
  const int4 item = a.g.lin_item[a.row_map[b]];
  const int S = item.y, init = item.z;
  const uint4 *rec = a.g.lin_state + item.x;
  float ps[K], pin[K], fin[K];
  unsigned pdp[K];  // self pdf | entry pdf << 16
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int s = lane * K + k;
    const uint4 v = s < S ? rec[s] : make_uint4(0u, 0u, 0u, 0u);
    ps[k] = __uint_as_float(v.x);
    pin[k] = __uint_as_float(v.y);
    pdp[k] = v.z;
    fin[k] = __uint_as_float(v.w);
  }
  // arc (lane K + K - 1) -> (lane K + K): the entry arc of the next lane's first state
  float po_last = __shfl_down_sync(kFull, pin[0], 1);
  unsigned pdo_last = __shfl_down_sync(kFull, pdp[0], 1) >> 16;
  if (lane == 31) {
    po_last = 0.f;
    pdo_last = 0u;
  }
  const float leak = a.leak;
  const float vleak = leak > 0.f ? leak / (float(S) * (1.f + leak)) : 0.f;  // leak * pi / (1 + leak)

  const bool vec16 = (D & 3) == 0 && ((reinterpret_cast<uintptr_t>(Lb) & 15) == 0);
  auto stage = [&](int t) { return ring + (t % kRing) * lay.stage; };
  auto issue_row = [&](int t) {
    float *dst = stage(t);
    const float *src = Lb + size_t(t) * D;
    if (vec16) {
      for (int c = lane; c < (D >> 2); c += 32) cp_async_16(dst + 4 * c, src + 4 * c);
    } else {
      for (int d = lane; d < D; d += 32) cp_async_elem(dst + d, src + d);
    }
  };
  auto issue_alpha = [&](int t) {  // alpha row t (this lane's K states) behind the L row
    if (!own_row) return;
    float *dst = stage(t) + lay.Dr + lane * K;
    const float *src = tr + size_t(t) * ld + lane * K;
    if constexpr (K >= 4) {
#pragma unroll
      for (int c = 0; c < K; c += 4) cp_async_16(dst + c, src + c);
    } else {
#pragma unroll
      for (int c = 0; c < K; ++c) cp_async_elem(dst + c, src + c);
    }
  };
  auto emission = [&](const float *Lt, unsigned pdf, float m) {
    if constexpr (PRE) {
      (void)m;
      return Lt[pdf];
    } else {
      return expf(Lt[pdf] - m);
    }
  };

  // ---- forward (_kernels.py:54-122) ---------------------------------------------
  float r[K];  // unnormalised column: alpha_0 (one-hot) at t = 0, raw_t after
#pragma unroll
  for (int k = 0; k < K; ++k) r[k] = (lane * K + k == init) ? 1.f : 0.f;
  int fail_at = -1;
#pragma unroll
  for (int p = 0; p < kRing - 1; ++p) {
    if (p < T) issue_row(p);
    cp_async_commit();
  }
  for (int t = 0; t < T; ++t) {
    __syncwarp();  // stage of frame t-1 fully consumed before it is refilled
    if (t + kRing - 1 < T) issue_row(t + kRing - 1);
    cp_async_commit();
    cp_async_wait<kRing - 1>();
    __syncwarp();
    const float *Lt = stage(t);
    // normaliser of column t (t >= 1); runs beside the stencil below
    float R = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) R += r[k];
    // unnormalised stencil on column t
    float prev = __shfl_up_sync(kFull, r[K - 1], 1);
    if (lane == 0) prev = 0.f;
    float m = 0.f;
    if constexpr (!PRE) {
      m = -INFINITY;
      for (int d = lane; d < D; d += 32) m = nan_max(m, Lt[d]);
      m = warp_max(m);
    }
    R = warp_sum(R);
    float A[K], Bv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float ws = ps[k] * emission(Lt, pdp[k] & 0xffffu, m);
      const float wi = pin[k] * emission(Lt, pdp[k] >> 16, m);
      A[k] = ws * r[k] + wi * (k ? r[k - 1] : prev);
      Bv[k] = ws + wi;
    }
    float u = 1.f, v = 0.f;
    if (t > 0) {
      float tot = R;
      if (leak > 0.f && R > 0.f) {
        tot = R + leak * R;
        v = vleak;
      }
      if (!(tot >= a.floor_eff) || tot == INFINITY) {
        fail_at = t - 1;
        break;
      }
      u = rcp_rn(tot);
      if (lane == 0) scl[t - 1] = tot;
    }
    // (PRE: the row maxima are read once at the end, not per frame — a global
    // load feeding a store here would stall the warp every frame)
    if constexpr (!PRE) {
      if (lane == 0) shf[t] = m;
    }
    // normalised alpha_t -> trellis row t (posteriors of frame t in the backward)
    if (own_row) {
      float al[K];
#pragma unroll
      for (int k = 0; k < K; ++k) al[k] = lane * K + k < S ? fmaf(r[k], u, v) : 0.f;
      float *dst = tr + size_t(t) * ld + lane * K;
      if constexpr (K >= 4) {
#pragma unroll
        for (int c = 0; c < K; c += 4)
          *reinterpret_cast<float4 *>(dst + c) = make_float4(al[c], al[c + 1], al[c + 2], al[c + 3]);
      } else {
#pragma unroll
        for (int c = 0; c < K; ++c) dst[c] = al[c];
      }
    }
    // raw_{t+1} = W (r u + v) = u (W r) + v (W 1)
#pragma unroll
    for (int k = 0; k < K; ++k) r[k] = fmaf(u, A[k], v * Bv[k]);
    if (t + 1 == T) {
#pragma unroll
      for (int k = 0; k < K; ++k) r[k] *= fin[k];  // finals at the last frame (:97-98)
    }
  }
  cp_async_wait<0>();
  if (fail_at < 0) {  // column T
    float R = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) R += r[k];
    R = warp_sum(R);
    const float tot = (leak > 0.f && R > 0.f) ? R + leak * R : R;
    if (!(tot >= a.floor_eff) || tot == INFINITY)
      fail_at = T - 1;
    else if (lane == 0)
      scl[T - 1] = tot;
  }
  if (fail_at >= 0) {
    // scales stay 1 from the failing frame on; the shifts of the frames the loop
    // did not reach are still reported (forward_backward.py:184,206)
    for (int k = fail_at; k < T; ++k) {
      if (k > fail_at) {
        if constexpr (!PRE) {
          float m = -INFINITY;
          for (int d = lane; d < D; d += 32) m = nan_max(m, Lb[size_t(k) * D + d]);
          m = warp_max(m);
          if (lane == 0) shf[k] = m;
        }
      }
      if (lane == 0) scl[k] = 1.f;
    }
  }
  __syncwarp();
  {
    double acc = 0.0;
    for (int k = lane; k < T; k += 32) {
      const double v = log(double(scl[k])) + double(PRE ? Emb[k] : shf[k]);
      acc += v;
      if (a.scale_logs) a.scale_logs[size_t(b) * T_max + k] = v;
    }
    if (a.scale_logs)
      for (int k = T + lane; k < T_max; k += 32) a.scale_logs[size_t(b) * T_max + k] = 0.0;
    acc = warp_sum(acc);
    if (lane == 0) {
      a.logp[b] = fail_at >= 0 ? NAN : acc;
      a.fail[b] = fail_at;
    }
  }
  const bool other_failed = a.other_fail != nullptr && a.other_fail[b] >= 0;
  if (fail_at >= 0 || other_failed) {
    for (size_t i = lane; i < size_t(T) * D; i += 32) post_b[i] = 0.f;
    return;
  }

  // ---- backward + posteriors (_kernels.py:125-224) --------------------------------
  // beta_t = Y_t / scale_{t-1} + z_t, z_t = leak (pi . Y_t) / scale_{t-1} (t < T).
  for (int d = lane; d < lay.Dr; d += 32) hist[d] = 0u;
  float Y[K];
#pragma unroll
  for (int k = 0; k < K; ++k) Y[k] = fin[k] * (1.f + leak);
#pragma unroll
  for (int p = 0; p < kRing - 1; ++p) {
    const int e = T - 1 - p;
    if (e >= 0) {
      issue_row(e);
      issue_alpha(e);
    }
    cp_async_commit();
  }
  const bool vflush = (D & 3) == 0 && ((reinterpret_cast<uintptr_t>(post_b) & 15) == 0);
  for (int t = T; t >= 1; --t) {
    const int e = t - 1;  // emission frame
    __syncwarp();         // stage + histogram of frame e+1 consumed
    {
      const int en = e - (kRing - 1);
      if (en >= 0) {
        issue_row(en);
        issue_alpha(en);
      }
      cp_async_commit();
    }
    cp_async_wait<kRing - 1>();
    __syncwarp();
    const float *Lt = stage(e);
    const float *al = Lt + lay.Dr + lane * K;
    const float m = PRE ? 0.f : shf[e];
    const float q = rcp_rn(scl[t - 1]);
    float sY = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) sY += Y[k];
    float ynext = __shfl_down_sync(kFull, Y[0], 1);
    if (lane == 31) ynext = 0.f;
    float ws[K], wo[K];
#pragma unroll
    for (int k = 0; k < K; ++k) ws[k] = ps[k] * emission(Lt, pdp[k] & 0xffffu, m);
#pragma unroll
    for (int k = 0; k < K - 1; ++k) wo[k] = pin[k + 1] * emission(Lt, pdp[k + 1] >> 16, m);
    wo[K - 1] = po_last * emission(Lt, pdo_last, m);
    float A[K], Bv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      A[k] = ws[k] * Y[k] + wo[k] * (k + 1 < K ? Y[k + 1] : ynext);
      Bv[k] = ws[k] + wo[k];
    }
    float z = 0.f;
    if (leak > 0.f && t < T) z = leak * q * (warp_sum(sY) / float(S));
    // posterior terms of frame e: alpha_e[src] * p e * beta_t[dst]
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float a_s = own_row ? al[k] : 0.f;
      const float bs = fmaf(Y[k], q, z);
      const float bn = fmaf(k + 1 < K ? Y[k + 1] : ynext, q, z);
      const float gs = a_s * ws[k] * bs;
      const float go = a_s * wo[k] * bn;
      if (gs > 0.f) atomicAdd(hist + (pdp[k] & 0xffffu), __float2uint_rn(gs * kFix));
      const unsigned pdo = k + 1 < K ? (pdp[k + 1] >> 16) : pdo_last;
      if (go > 0.f) atomicAdd(hist + pdo, __float2uint_rn(go * kFix));
    }
    // X_{t-1} = Y_{t-1}: the next column (reference beta_{t-1} before leak / scale)
#pragma unroll
    for (int k = 0; k < K; ++k) Y[k] = fmaf(q, A[k], z * Bv[k]);
    __syncwarp();
    // flush gamma row e into the posterior output (mode), clearing the histogram
    float *prow = post_b + size_t(e) * D;
    if (vflush) {
      uint4 *h4 = reinterpret_cast<uint4 *>(hist);
      float4 *p4 = reinterpret_cast<float4 *>(prow);
      for (int c = lane; c < (D >> 2); c += 32) {
        const uint4 hv = h4[c];
        h4[c] = make_uint4(0u, 0u, 0u, 0u);
        float4 g = make_float4(float(hv.x) * kUnfix, float(hv.y) * kUnfix, float(hv.z) * kUnfix,
                               float(hv.w) * kUnfix);
        if (mode == kPostNegate) {
          g = make_float4(-g.x, -g.y, -g.z, -g.w);
        } else if (reads_post) {
          const float4 o = p4[c];
          const float sg = mode == kPostAdd ? 1.f : -1.f;
          g = make_float4(o.x + sg * g.x, o.y + sg * g.y, o.z + sg * g.z, o.w + sg * g.w);
        }
        p4[c] = g;
      }
    } else {
      for (int d = lane; d < D; d += 32) {
        float g = float(hist[d]) * kUnfix;
        hist[d] = 0u;
        if (mode == kPostNegate) g = -g;
        else if (mode == kPostAdd) g = prow[d] + g;
        else if (mode == kPostSubtract) g = prow[d] - g;
        prow[d] = g;
      }
    }
  }
  cp_async_wait<0>();
}

// ---- forward | backward split: two warps per utterance ------------------------
//
// Warp 0 runs the forward recursion over frames 0..T-1, warp 1 the backward one
// over T-1..0, concurrently, meeting at h ~ T/2 (the fb_split_kernel scheme on
// one SM): the forward warp stores alpha rows 0..h-1 and does the posteriors of
// frames >= h, the backward warp (its own normalisers inv_t) stores beta' rows
// h..T-1 and does the posteriors of frames < h.  The fixed-point posterior bins
// need each frame's arc terms scaled to sum to 1 before the frame: with B_t the
// backward column t in its own scale (raw + leak), kappa_t = sum over arcs of
// alpha_{t-1} p e_{t-1} B_t obeys kappa_{t-1} = inv_t kappa_t scale_{t-2}
// exactly (reference recursions), kappa_h is one dot product at the midpoint,
// and the forward frame k >= h normalises by kappa_k / scale_{k-1}.  Emissions
// from emit_kernel (PRE) only; K <= 8.
struct LinSplitLayout {
  int T4, Dr, SK, nwd;
  size_t bytes;
};

// nwd: warps per direction (1, or 2 for the K = 16 class: 64 lanes x 8 states).
__host__ __device__ inline LinSplitLayout lin_split_layout(int T_max, int D, int K, int nwd = 1) {
  LinSplitLayout l;
  l.T4 = pad4(T_max);
  l.Dr = pad4(D);
  l.SK = 32 * K;
  l.nwd = nwd;
  // scales | shifts | inv (T4 + 4) | B_h (32 K) | hist[2][Dr] | ring[2 nwd][kRing][Dr] |
  // kappa + partials (4 doubles) | exchange slots (32 floats)
  l.bytes = size_t(3 * l.T4 + 4 + l.SK + 2 * l.Dr + 2 * nwd * kRing * l.Dr) * 4 + 32 + 128;
  return l;
}

// The two directions of a split utterance meet at different code locations (the
// forward warps inside their frame loop, the backward warps at their midpoint),
// so they use the non-aligned named barrier 1 (all 64 NWD threads), not
// __syncthreads; the two warps of one direction (NWD = 2) use barrier 2 / 3.
template <int NWD>
__device__ __forceinline__ void pair_sync() {
  asm volatile("barrier.sync 1, %0;\n" ::"n"(64 * NWD) : "memory");
}

// NWD = 1: one warp per direction, lane l owns states [l K, l K + K).  NWD = 2
// (the K = 16 class as 64 lanes x 8 states): the two warps of a direction
// exchange the column sum and the boundary state through shared memory once
// per frame (one 64-thread named barrier), share the posterior bins, and split
// the gradient-row flush.
template <int K, int NWD = 1>
__device__ __forceinline__ void linear_item_split(const FBArgs<float> &a, float *lsm,
                                                  const LinSplitLayout &lay, int b) {
  constexpr int NG = 32 * NWD;  // lanes per direction
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wrole = warp / NWD, half = warp % NWD;  // 0 forward, 1 backward; warp within it
  const int gl = half * 32 + lane;                  // lane within the direction
  const int D = a.D, T_max = a.T_max;
  float *scl = lsm;                 // forward scales (tot of column t+1 at [t])
  float *invs = lsm + 2 * lay.T4;   // backward normalisers n_t = 1 / inv_t at [t]
                                    // (lsm + T4: the row-maxima slot, unused with E rows)
  float *Bh = invs + lay.T4 + 4;    // backward column B_h at the midpoint
  unsigned *hist = reinterpret_cast<unsigned *>(Bh + lay.SK) + wrole * lay.Dr;
  const uint32_t hist32 = smem_u32(hist);
  float *ring = reinterpret_cast<float *>(Bh + lay.SK + 2 * lay.Dr) + warp * kRing * lay.Dr;
  double *kap = reinterpret_cast<double *>(Bh + lay.SK + 2 * lay.Dr + 2 * NWD * kRing * lay.Dr);
  // exchange slots (NWD = 2): [wrole][frame parity][4] | [wrole][2] | boundary arcs [wrole][2]
  float *xch = reinterpret_cast<float *>(kap + 4);
  auto group_sync = [&]() {
    if constexpr (NWD == 1)
      __syncwarp();
    else
      asm volatile("barrier.sync %0, 64;\n" ::"r"(2 + wrole) : "memory");
  };
  // sum over the direction's lanes (identical in every lane); slot: 2 floats
  auto group_sum = [&](float v, float *slot) {
    v = warp_sum(v);
    if constexpr (NWD > 1) {
      if (lane == 0) slot[half] = v;
      group_sync();
      v = slot[0] + slot[1];
    }
    return v;
  };
  const int mode = a.mode;
  const bool reads_post = mode == kPostAdd || mode == kPostSubtract;

  long long off = 0;
  for (int j = lane; j < b; j += 32) off += a.packed ? a.lengths[j] : item_frames(a.lengths, j, T_max);
  off = warp_sum(off);
  const int T = item_frames(a.lengths, b, T_max);
  const size_t row0 = a.packed ? size_t(off) : size_t(b) * T_max;
  const float *Lb = a.E + row0 * D;
  const float *Emb = a.Em + row0;
  float *post_b = a.post + row0 * D;
  if (wrole == 0 && !reads_post && !a.packed)
    for (size_t i = gl; i < size_t(T_max - T) * D; i += NG) post_b[size_t(T) * D + i] = 0.f;
  if (T <= 0) {
    if (wrole == 0) {
      if (a.scale_logs && !a.packed)
        for (int k = gl; k < T_max; k += NG) a.scale_logs[size_t(b) * T_max + k] = 0.0;
      if (gl == 0) {
        a.logp[b] = NAN;
        a.fail[b] = 0;
      }
    }
    return;  // every warp: no barriers for this item
  }
  const int ldt = (a.S_max + 31) & ~31;
  float *tr = a.work + size_t(off) * ldt;
  const bool own_row = gl * K < ldt;
  const int h = T == 1 ? 1 : min(T - 1, max(1, (T * 33 + 32) >> 6));

  const int4 item = a.g.lin_item[a.row_map[b]];
  const int S = item.y, init = item.z;
  const uint4 *rec = a.g.lin_state + item.x;
  float ps[K], pin[K], fin[K];
  unsigned pdp[K];
  bool valid[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int s = gl * K + k;
    valid[k] = s < S;
    const uint4 v = valid[k] ? rec[s] : make_uint4(0u, 0u, 0u, 0u);
    ps[k] = __uint_as_float(v.x);
    pin[k] = __uint_as_float(v.y);
    pdp[k] = v.z;
    fin[k] = __uint_as_float(v.w);
  }
  float po_last = __shfl_down_sync(kFull, pin[0], 1);
  unsigned pdo_last = __shfl_down_sync(kFull, pdp[0], 1) >> 16;
  if constexpr (NWD > 1) {  // the first state of the next warp of this direction
    float *xb = xch + 24 + 2 * wrole;
    if (half == 1 && lane == 0) {
      xb[0] = pin[0];
      xb[1] = __uint_as_float(pdp[0] >> 16);
    }
    group_sync();
    if (half == 0 && lane == 31) {
      po_last = xb[0];
      pdo_last = __float_as_uint(xb[1]);
    }
  }
  if (gl == NG - 1) {
    po_last = 0.f;
    pdo_last = 0u;
  }
  const float leak = a.leak;
  const float vleak = leak > 0.f ? leak / (float(S) * (1.f + leak)) : 0.f;
  const bool vec16 = (D & 3) == 0 && ((reinterpret_cast<uintptr_t>(Lb) & 15) == 0);
  auto stage = [&](int t) { return ring + (t % kRing) * lay.Dr; };
  auto issue_row = [&](int t) {
    float *dst = stage(t);
    const float *src = Lb + size_t(t) * D;
    if (vec16) {
      for (int c = lane; c < (D >> 2); c += 32) cp_async_16(dst + 4 * c, src + 4 * c);
    } else {
      for (int d = lane; d < D; d += 32) cp_async_elem(dst + d, src + d);
    }
  };
  auto load_row_k = [&](int t, float *v) {  // this lane's K entries of trellis row t
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = 0.f;
    if (!own_row || t < 0 || t >= T) return;
    const float *src = tr + size_t(t) * ldt + gl * K;
    if constexpr (K >= 4) {
#pragma unroll
      for (int c = 0; c < K; c += 4) {
        const float4 q = *reinterpret_cast<const float4 *>(src + c);
        v[c] = q.x;
        v[c + 1] = q.y;
        v[c + 2] = q.z;
        v[c + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < K; ++c) v[c] = src[c];
    }
  };
  auto store_row_k = [&](int t, const float *v) {
    if (!own_row) return;
    float *dst = tr + size_t(t) * ldt + gl * K;
    if constexpr (K >= 4) {
#pragma unroll
      for (int c = 0; c < K; c += 4)
        *reinterpret_cast<float4 *>(dst + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
    } else {
#pragma unroll
      for (int c = 0; c < K; ++c) dst[c] = v[c];
    }
  };
  const bool vflush = (D & 3) == 0 && ((reinterpret_cast<uintptr_t>(post_b) & 15) == 0);
  auto flush = [&](int e) {  // this warp's bins -> gradient row e (mode), cleared
    float *prow = post_b + size_t(e) * D;
    if (vflush) {
      uint4 *h4 = reinterpret_cast<uint4 *>(hist);
      float4 *p4 = reinterpret_cast<float4 *>(prow);
      for (int c = gl; c < (D >> 2); c += NG) {
        const uint4 hv = h4[c];
        h4[c] = make_uint4(0u, 0u, 0u, 0u);
        float4 g = make_float4(float(hv.x) * kUnfix, float(hv.y) * kUnfix, float(hv.z) * kUnfix,
                               float(hv.w) * kUnfix);
        if (mode == kPostNegate) {
          g = make_float4(-g.x, -g.y, -g.z, -g.w);
        } else if (reads_post) {
          const float4 o = p4[c];
          const float sg = mode == kPostAdd ? 1.f : -1.f;
          g = make_float4(o.x + sg * g.x, o.y + sg * g.y, o.z + sg * g.z, o.w + sg * g.w);
        }
        p4[c] = g;
      }
    } else {
      for (int d = gl; d < D; d += NG) {
        float g = float(hist[d]) * kUnfix;
        hist[d] = 0u;
        if (mode == kPostNegate) g = -g;
        else if (mode == kPostAdd) g = prow[d] + g;
        else if (mode == kPostSubtract) g = prow[d] - g;
        prow[d] = g;
      }
    }
  };
  for (int d = gl; d < lay.Dr; d += NG) hist[d] = 0u;
  const bool other_failed = a.other_fail != nullptr && a.other_fail[b] >= 0;

  if (wrole == 0) {
    // ======================= forward warp =========================================
    float r[K];
#pragma unroll
    for (int k = 0; k < K; ++k) r[k] = (gl * K + k == init) ? 1.f : 0.f;
    int fail_at = -1;
    bool mid_done = false;
    double kappa = 0.0;
    float bcur[K];  // beta'_{t+1} of this lane's states (posterior frames)
#pragma unroll
    for (int k = 0; k < K; ++k) bcur[k] = 0.f;
    auto midpoint = [&](const float *raw) {  // kappa_h = sum raw_h B_h
      pair_sync<NWD>();  // B_h, backward rows >= h and inv_t are written
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (valid[k]) acc += double(raw[k]) * double(Bh[gl * K + k]);
      acc = warp_sum(acc);
      if constexpr (NWD > 1) {
        if (lane == 0) kap[2 + half] = acc;
        group_sync();
        acc = kap[2] + kap[3];
      }
      if (gl == 0) kap[0] = acc;
      kappa = acc;
      mid_done = true;
      pair_sync<NWD>();  // kappa_h delivered
    };
#pragma unroll
    for (int p = 0; p < kRing - 1; ++p) {
      if (p < T) issue_row(p);
      cp_async_commit();
    }
    for (int t = 0; t < T; ++t) {
      __syncwarp();
      if (t + kRing - 1 < T) issue_row(t + kRing - 1);
      cp_async_commit();
      if (t == h) {
        midpoint(r);
        load_row_k(t, bcur);  // row t holds beta'_{t+1}
      }
      cp_async_wait<kRing - 1>();
      __syncwarp();
      const float *Lt = stage(t);
      float R = 0.f;
#pragma unroll
      for (int k = 0; k < K; ++k) R += r[k];
      float prev = __shfl_up_sync(kFull, r[K - 1], 1);
      {
        float *x = xch + (wrole * 2 + (t & 1)) * 4;
        if constexpr (NWD > 1)
          if (half == 0 && lane == 31) x[2] = r[K - 1];  // published by the group_sum barrier
        R = group_sum(R, x);
        if constexpr (NWD > 1)
          if (half == 1 && lane == 0) prev = x[2];
      }
      if (gl == 0) prev = 0.f;
      float ws[K], wi[K], A[K], Bv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ws[k] = ps[k] * Lt[pdp[k] & 0xffffu];
        wi[k] = pin[k] * Lt[pdp[k] >> 16];
        A[k] = ws[k] * r[k] + wi[k] * (k ? r[k - 1] : prev);
        Bv[k] = ws[k] + wi[k];
      }
      float u = 1.f, v = 0.f, tot = 1.f;
      if (t > 0) {
        tot = R;
        if (leak > 0.f && R > 0.f) {
          tot = R + leak * R;
          v = vleak;
        }
        if (!(tot >= a.floor_eff) || tot == INFINITY) {
          fail_at = t - 1;
          break;
        }
        u = rcp_rn(tot);
        if (gl == 0) scl[t - 1] = tot;
      }
      if (t < h) {  // alpha_t for the backward warp's posteriors
        float al[K];
#pragma unroll
        for (int k = 0; k < K; ++k) al[k] = valid[k] ? fmaf(r[k], u, v) : 0.f;
        store_row_k(t, al);
      }
      if (t >= h && !other_failed) {  // posteriors of frame t: terms / Z_t, Z_t = kappa_t / scale_{t-1}
        // (no double divisions on the frame's path: u = 1 / scale_{t-1} and the
        // backward normaliser n_{t+1} = 1 / inv_{t+1} are at hand)
        const double zt = kappa * double(u);
        const float zs = (zt > 1e-37 && zt < 1e37) ? __frcp_rn(float(zt)) : 0.f;
        const float vprev = (gl * K > 0 && gl * K - 1 < S) ? v : 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const float a_s = valid[k] ? fmaf(r[k], u, v) : 0.f;
          const float a_p = (k ? (valid[k - 1] ? fmaf(r[k - 1], u, v) : 0.f) : fmaf(prev, u, vprev));
          const float gs = a_s * ws[k] * bcur[k] * zs;
          const float gi = a_p * wi[k] * bcur[k] * zs;
          // predicated REDs (no branch per term; zero / negative / NaN terms quantise to 0)
          red_add_shared_nz(hist32 + ((pdp[k] & 0xffffu) << 2), __float2uint_rn(gs * kFix));
          red_add_shared_nz(hist32 + ((pdp[k] >> 16) << 2), __float2uint_rn(gi * kFix));
        }
        group_sync();  // every warp's bins of frame t are in
        flush(t);
        __syncwarp();  // (the next frame's group_sum barrier orders the clears)
        kappa = zt * double(invs[t + 1]);  // kappa_{t+1} = Z_t / inv_{t+1} (invs holds n = 1 / inv)
        if (t + 1 < T) load_row_k(t + 1, bcur);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) r[k] = fmaf(u, A[k], v * Bv[k]);
      if (t + 1 == T) {
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] *= fin[k];
      }
    }
    cp_async_wait<0>();
    if (fail_at < 0) {
      float R = 0.f;
#pragma unroll
      for (int k = 0; k < K; ++k) R += r[k];
      R = group_sum(R, xch + 16 + 2 * wrole);
      const float tot = (leak > 0.f && R > 0.f) ? R + leak * R : R;
      if (!(tot >= a.floor_eff) || tot == INFINITY)
        fail_at = T - 1;
      else if (gl == 0)
        scl[T - 1] = tot;
    }
    if (!mid_done) {  // T == 1 (kappa_1 = scale_0) or failed before the midpoint
      __syncwarp();
      pair_sync<NWD>();
      if (gl == 0) kap[0] = fail_at < 0 ? double(scl[T - 1]) : 1.0;
      pair_sync<NWD>();
    }
    if (fail_at >= 0 && gl == 0)
      for (int k = fail_at; k < T; ++k) scl[k] = 1.f;
    pair_sync<NWD>();  // end: the backward warps' posterior rows (and scl) are written
    if (half == 0) {
      double acc = 0.0;
      for (int k = lane; k < T; k += 32) {
        const double val = log(double(scl[k])) + double(Emb[k]);
        acc += val;
        if (a.scale_logs) a.scale_logs[size_t(b) * T_max + k] = val;
      }
      if (a.scale_logs)
        for (int k = T + lane; k < T_max; k += 32) a.scale_logs[size_t(b) * T_max + k] = 0.0;
      acc = warp_sum(acc);
      if (lane == 0) {
        a.logp[b] = fail_at >= 0 ? NAN : acc;
        a.fail[b] = fail_at;
      }
    }
    if (fail_at >= 0 || other_failed)
      for (size_t i = gl; i < size_t(T) * D; i += NG) post_b[i] = 0.f;
  } else {
    // ======================= backward warp ========================================
    float Y[K];  // pre-leak column t in this warp's own scale; B_t = Y + ld_t
#pragma unroll
    for (int k = 0; k < K; ++k) Y[k] = fin[k] * (1.f + leak);
    double kappa = 0.0;
    float al[K];  // alpha of the current posterior frame (this lane's states)
#pragma unroll
    for (int p = 0; p < kRing - 1; ++p) {
      const int e = T - 1 - p;
      if (e >= 0) issue_row(e);
      cp_async_commit();
    }
    for (int t = T; t >= 1; --t) {
      const int e = t - 1;
      __syncwarp();
      {
        const int en = e - (kRing - 1);
        if (en >= 0) issue_row(en);
        cp_async_commit();
      }
      if (t == h) {  // midpoint: B_h for the forward warp, then kappa_h
        float sY = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) sY += Y[k];
        sY = group_sum(sY, xch + 16 + 2 * wrole);
        const float ldh = (t < T && leak > 0.f) ? leak * sY / float(S) : 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) Bh[gl * K + k] = valid[k] ? Y[k] + ldh : 0.f;
        __threadfence_block();
        pair_sync<NWD>();  // forward warps compute kappa_h
        pair_sync<NWD>();
        kappa = kap[0];
        load_row_k(e, al);
      }
      cp_async_wait<kRing - 1>();
      __syncwarp();
      const float *Lt = stage(e);
      const bool post = t <= h && !other_failed;
      float sY = 0.f;
#pragma unroll
      for (int k = 0; k < K; ++k) sY += Y[k];
      float ynext = __shfl_down_sync(kFull, Y[0], 1);
      {
        float *xf = xch + (wrole * 2 + (t & 1)) * 4;
        if constexpr (NWD > 1)
          if (half == 1 && lane == 0) xf[2] = Y[0];  // published by the group_sum barrier
        sY = group_sum(sY, xf);
        if constexpr (NWD > 1)
          if (half == 0 && lane == 31) ynext = xf[2];
      }
      if (gl == NG - 1) ynext = 0.f;
      float ws[K], wo[K], A[K], Bv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) ws[k] = ps[k] * Lt[pdp[k] & 0xffffu];
#pragma unroll
      for (int k = 0; k < K - 1; ++k) wo[k] = pin[k + 1] * Lt[pdp[k + 1] >> 16];
      wo[K - 1] = po_last * Lt[pdo_last];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        A[k] = ws[k] * Y[k] + wo[k] * (k + 1 < K ? Y[k + 1] : ynext);
        Bv[k] = ws[k] + wo[k];
      }
      const float ld = (t < T && leak > 0.f) ? leak * sY / float(S) : 0.f;
      const float n = sY + ld * float(S);
      const float inv = (n > 0.f && n < INFINITY) ? rcp_rn(n) : 1.f;
      if (gl == 0) invs[t] = (n > 0.f && n < INFINITY) ? n : 1.f;  // n_t = 1 / inv_t
      if (!post) {  // beta'_t = B_t inv_t -> row e (the forward warp's posteriors)
        if (t > h) {
          float bb[K];
#pragma unroll
          for (int k = 0; k < K; ++k) bb[k] = valid[k] ? (Y[k] + ld) * inv : 0.f;
          store_row_k(e, bb);
        }
      } else {  // posteriors of frame e: alpha_e p e B_t / kappa_t
        const float zinv = (kappa > 1e-37 && kappa < 1e37) ? __frcp_rn(float(kappa)) : 0.f;
        const bool nvalid = gl * K + K < S;  // state gl K + K exists
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const float bs = valid[k] ? Y[k] + ld : 0.f;
          const float bn = k + 1 < K ? (valid[k + 1] ? Y[k + 1] + ld : 0.f)
                                     : (nvalid ? ynext + ld : 0.f);
          const float gs = al[k] * ws[k] * bs * zinv;
          const float go = al[k] * wo[k] * bn * zinv;
          red_add_shared_nz(hist32 + ((pdp[k] & 0xffffu) << 2), __float2uint_rn(gs * kFix));
          const unsigned pdo = k + 1 < K ? (pdp[k + 1] >> 16) : pdo_last;
          red_add_shared_nz(hist32 + (pdo << 2), __float2uint_rn(go * kFix));
        }
        group_sync();  // every warp's bins of frame e are in
        flush(e);
        __syncwarp();  // (the next frame's group_sum barrier orders the clears)
        if (t >= 2) kappa = double(inv) * kappa * double(scl[t - 2]);  // kappa_{t-1}
        load_row_k(e - 1, al);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) Y[k] = inv * fmaf(ld, Bv[k], A[k]);
    }
    cp_async_wait<0>();
    pair_sync<NWD>();  // end
  }
}

// One warp per utterance; this launch runs the utterances whose K lies in
// [KLO, KHI] (the K = 16 variant needs ~2x the registers of the others, so it
// is a separate launch that only batches with S > 256 pay for).  Shared-memory
// strides follow the batch's largest K (`kstage`).
template <int KLO, int KHI, bool PRE>
__global__ void __launch_bounds__(32) fb_linear_kernel(const FBArgs<float> a, int kstage) {
  extern __shared__ __align__(16) float lsm[];
  const int b = blockIdx.x;
  const int K = k_of(a.g.lin_item[a.row_map[b]].y);
  if (K < KLO || K > KHI) return;
  const LinLayout lay = lin_layout(a.T_max, a.D, kstage);
  switch (K) {
    case 1: if constexpr (KLO <= 1 && 1 <= KHI) linear_item<1, PRE>(a, lsm, lay, b); break;
    case 2: if constexpr (KLO <= 2 && 2 <= KHI) linear_item<2, PRE>(a, lsm, lay, b); break;
    case 4: if constexpr (KLO <= 4 && 4 <= KHI) linear_item<4, PRE>(a, lsm, lay, b); break;
    case 8: if constexpr (KLO <= 8 && 8 <= KHI) linear_item<8, PRE>(a, lsm, lay, b); break;
    default: if constexpr (KHI >= 16) linear_item<16, PRE>(a, lsm, lay, b); break;
  }
}

// Two warps per utterance (forward | backward) for the utterances with K in
// [KLO, KHI]: instantiated for the batch's largest K <= 8 (registers follow that
// K), plus a K = 16 launch (254 registers) only when the batch has S > 256.
template <int KLO, int KHI>
__global__ void __launch_bounds__(64) fb_linear_split_kernel(const FBArgs<float> a, int kstage) {
  extern __shared__ __align__(16) float lsm[];
  const int b = blockIdx.x;
  const int K = k_of(a.g.lin_item[a.row_map[b]].y);
  if (K < KLO || K > KHI) return;
  const LinSplitLayout lay = lin_split_layout(a.T_max, a.D, kstage);
  switch (K) {
    case 1: if constexpr (KLO <= 1) linear_item_split<1>(a, lsm, lay, b); break;
    case 2: if constexpr (KLO <= 2 && KHI >= 2) linear_item_split<2>(a, lsm, lay, b); break;
    case 4: if constexpr (KLO <= 4 && KHI >= 4) linear_item_split<4>(a, lsm, lay, b); break;
    case 8: if constexpr (KLO <= 8 && KHI >= 8) linear_item_split<8>(a, lsm, lay, b); break;
    default: if constexpr (KHI >= 16) linear_item_split<16>(a, lsm, lay, b); break;
  }
}

// The K = 16 class (S in (256, 512]) as two warps per direction (64 lanes x 8
// states, 128 threads): half the per-lane chain of the one-warp K = 16 variant
// (254 registers), one 64-thread barrier per frame for the column sum and the
// warp-boundary state.
__global__ void __launch_bounds__(128) fb_linear_split2_kernel(const FBArgs<float> a, int kstage) {
  extern __shared__ __align__(16) float lsm[];
  const int b = blockIdx.x;
  if (k_of(a.g.lin_item[a.row_map[b]].y) != 16) return;
  const LinSplitLayout lay = lin_split_layout(a.T_max, a.D, kstage, 2);
  linear_item_split<8, 2>(a, lsm, lay, b);
}

int launch_split2(const FBArgs<float> &a, int ks, cudaStream_t st) {
  const size_t ssm = lin_split_layout(a.T_max, a.D, ks, 2).bytes;
  if (ssm > size_t(kMaxSmem)) return LFMMI_ERR_UNSUPPORTED;
  if (ssm > 48 * 1024) {
    const int rc = check_cuda(cudaFuncSetAttribute(fb_linear_split2_kernel,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   int(ssm)),
                              "cudaFuncSetAttribute(linear split2)");
    if (rc) return rc;
  }
  fb_linear_split2_kernel<<<a.B, 128, ssm, st>>>(a, ks);
  return check_cuda(cudaGetLastError(), "fb_linear_split2_kernel launch");
}

template <int KLO, int KHI>
int launch_split_k(const FBArgs<float> &a, int ks, size_t ssm, cudaStream_t st) {
  if (ssm > 48 * 1024) {
    const int rc = check_cuda(cudaFuncSetAttribute(fb_linear_split_kernel<KLO, KHI>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   int(ssm)),
                              "cudaFuncSetAttribute(linear split)");
    if (rc) return rc;
  }
  fb_linear_split_kernel<KLO, KHI><<<a.B, 64, ssm, st>>>(a, ks);
  return check_cuda(cudaGetLastError(), "fb_linear_split_kernel launch");
}

template <int KLO, int KHI, bool PRE>
int launch_range(const FBArgs<float> &a, int kstage, size_t smem, cudaStream_t st) {
  if (smem > 48 * 1024) {
    const int rc = check_cuda(cudaFuncSetAttribute(fb_linear_kernel<KLO, KHI, PRE>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   int(smem)),
                              "cudaFuncSetAttribute(linear)");
    if (rc) return rc;
  }
  fb_linear_kernel<KLO, KHI, PRE><<<a.B, 32, smem, st>>>(a, kstage);
  return check_cuda(cudaGetLastError(), "fb_linear_kernel launch");
}

}  // namespace

int launch_linear(const FBArgs<float> &a, const lfmmi_graphs *g, cudaStream_t st) {
  if (!g->linear || a.leak_pi != nullptr || a.D > 65536) return LFMMI_ERR_UNSUPPORTED;
  const int S = g->max_states;
  if (S > 512) return LFMMI_ERR_UNSUPPORTED;
  const int kstage = S <= 32 ? 1 : S <= 64 ? 2 : S <= 128 ? 4 : S <= 256 ? 8 : 16;
  const size_t smem = lin_layout(a.T_max, a.D, kstage).bytes;
  if (smem > size_t(kMaxSmem)) return LFMMI_ERR_UNSUPPORTED;
  const bool pre = a.E != nullptr;
  if (pre && options().linear_split) {  // forward | backward warps
    const size_t ssm = lin_split_layout(a.T_max, a.D, kstage).bytes;
    if (ssm <= size_t(kMaxSmem)) {
      note_kernel("fb_linear_split_kernel (forward | backward warps)");
      // K = 16 in the batch: a K <= 8 launch followed by a K = 16 one (252
      // registers only for the long transcripts), or (option linear_k16 = 1)
      // one launch for every K.  Sweep at B = 128 (the 8-GPU per-rank load):
      // step 4.00 vs 4.31 ms; at B = 1024: 28.6 vs 28.2 ms.
      if (kstage > 8 && options().linear_k16) return launch_split_k<1, 16>(a, kstage, ssm, st);
      int rc = kstage == 1   ? launch_split_k<1, 1>(a, kstage, ssm, st)
               : kstage == 2 ? launch_split_k<1, 2>(a, kstage, ssm, st)
               : kstage == 4 ? launch_split_k<1, 4>(a, kstage, ssm, st)
                             : launch_split_k<1, 8>(a, kstage, ssm, st);
      if (rc || kstage <= 8) return rc;
      if (options().linear_k16w == 2) {
        const int rc2 = launch_split2(a, kstage, st);
        if (rc2 != LFMMI_ERR_UNSUPPORTED) return rc2;
      }
      return launch_split_k<16, 16>(a, kstage, ssm, st);
    }
  }
  note_kernel(kstage <= 8 ? (pre ? "fb_linear_kernel<1..8> (emissions pre-pass)"
                                 : "fb_linear_kernel<1..8>")
                          : (pre ? "fb_linear_kernel<1..8> + <16> (emissions pre-pass)"
                                 : "fb_linear_kernel<1..8> + <16>"));
  int rc = pre ? launch_range<1, 8, true>(a, kstage, smem, st)
               : launch_range<1, 8, false>(a, kstage, smem, st);
  if (rc || kstage <= 8) return rc;
  return pre ? launch_range<16, 16, true>(a, kstage, smem, st)
             : launch_range<16, 16, false>(a, kstage, smem, st);
}

}  // namespace lfmmi
