// fb_streamsplit_kernel — the meet-in-the-middle split (lfmmi_split.cu) for
// graphs whose arc packs live in L2 (lfmmi_stream.cu): configs 3/4.
//
// One 2-CTA cluster per utterance slot, persistent over an in-kernel LPT
// assignment of the batch: CTA 0 runs the forward recursion over frames
// 0..T-1, CTA 1 the backward recursion over T-1..0, concurrently, each with
// the full columns in its own shared memory and the stream packs (32-state
// tiles, bank-scheduled rows) streamed from L2 through the per-warp TMA slot
// ring (lfmmi_ring.cuh) when it fits beside the columns, else read per row from
// L2.  They meet at h (~T/2):
//
//   forward  frames 0..h-1 : alpha, spilled to trellis rows 0..h-1 (backward-pack order)
//            frames h..T-1 : alpha + posteriors of those frames (using beta' rows)
//   backward frames T-1..h : beta' with its OWN normalisers inv_t, spilled to rows
//                            h..T-1 (forward-pack order: row f holds beta'_{f+1})
//            frames h-1..0 : beta' + posteriors of those frames (using alpha rows)
//
// so an utterance costs ~T frames of latency instead of 2T.  Posteriors are
// 2^-28 fixed-point per-pdf bins (native shared-memory integer atomics,
// deterministic), which needs every frame's arc terms scaled to sum to ~1
// BEFORE the arc loop.  With B_t = the backward column t in its own scale
// (raw + leak), kappa_t = sum over arcs of alpha_{t-1}(src) p e_{t-1} B_t(dst) is
// the posterior normaliser of frame t-1, and (reference recursions,
// _kernels.py:54-191) it obeys, exactly,
//
//   kappa_{t-1} = inv_t * kappa_t * scale_{t-2}     (scale = forward normaliser)
//
// The CTAs compute kappa_h once at the midpoint (a dot product of the forward
// raw column h with the backward column B_h read through distributed shared
// memory) and then walk the recursion in their own direction, reading the
// other CTA's per-frame scalars (scales / inv) through DSMEM:
//   forward frame k >= h : Z_k = kappa_{k+1} inv_{k+1} = kappa_k / scale_{k-1}
//   backward frame t-1 < h: Z = kappa_t
// Log-probability, scales and failure frames come from the forward CTA exactly
// as in fb_stream_kernel (reference forward_backward.py:206-212).
#include <cooperative_groups.h>

#include <algorithm>
#include <string>

#include "lfmmi_device.cuh"
#include "lfmmi_kernels.h"
#include "lfmmi_lpt.cuh"
#include "lfmmi_options.h"
#include "lfmmi_ring.cuh"
#include "lfmmi_tile_common.cuh"

namespace cg = cooperative_groups;

namespace lfmmi {
namespace {

constexpr int kNT = 1024, kNW = kNT / 32;
constexpr int kMaxD = 2048, kEPT = (kMaxD + kNT - 1) / kNT;  // log-likelihood elements per thread
constexpr float kPostScale = 268435456.f;        // 2^28
constexpr int kMaxItems = kLptMaxItems;          // utterances per cluster
#ifndef LFMMI_L2_ROWS
#define LFMMI_L2_ROWS 8
#endif
constexpr int kL2Rows = LFMMI_L2_ROWS;  // slot-row loads in flight per lane (L2 path)
// TMA slot ring (as fb_stream_kernel): 2 chunks of 8 slot rows per warp
using Ring = SlotRing<2, 8, 64>;

struct SSLayout {
  unsigned vec, ebuf, bins, scales, invs, shifts, part, mpart, misc, items, ring, bars, ctab, total;
};

__host__ __device__ inline SSLayout ss_layout(int S32, int D_pad, int T_pad, bool ring) {
  SSLayout l;
  unsigned o = 512;  // scratch: 32 doubles + 32 int64
  auto take = [&](unsigned bytes) {
    const unsigned at = o;
    o = (o + bytes + 15u) & ~15u;
    return at;
  };
  l.vec = take(2u * S32 * 4u);
  l.ebuf = take(2u * D_pad * 4u);
  l.bins = take(2u * D_pad * 4u);
  l.scales = take(unsigned(T_pad) * 4u);  // forward: per-frame scales (read by the backward CTA)
  l.invs = take(unsigned(T_pad + 4) * 4u);  // backward: own normalisers inv_t (read by the forward)
  l.shifts = take(unsigned(T_pad) * 4u);
  l.part = take(2u * 32u * 4u);
  l.mpart = take(2u * 32u * 4u);
  l.misc = take(64u);  // [0] kappa_h (double), [8] ld_h (float), [12] fail flag (int)
  l.items = take(unsigned(kMaxItems + 4) * 4u);
  l.ring = take(ring ? Ring::slot_bytes(kNW) : 0u);
  l.bars = take(ring ? Ring::bar_bytes(kNW) : 0u);
  l.ctab = take(ring ? Ring::table_bytes(kNW) : 0u);
  l.total = o;
  return l;
}

__device__ __forceinline__ uint2 ldg_slot(const uint2 *p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];\n"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void cluster_sync_rows() {
  __threadfence();  // trellis rows in global memory before the arrive
  cg::this_cluster().sync();
}

}  // namespace

template <bool RING>
__global__ void __launch_bounds__(kNT, 1)
    fb_streamsplit_kernel(const FBArgs<float> a, int S32, const SSLayout lay, int nclusters,
                          int hnum) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  cg::cluster_group cl = cg::this_cluster();
  const int role = int(cl.block_rank());  // 0 forward, 1 backward
  const bool fwd = role == 0;
  const int cluster = blockIdx.x >> 1;
  double *dscr = reinterpret_cast<double *>(smem);
  float *vec = reinterpret_cast<float *>(smem + lay.vec);
  float *ebuf = reinterpret_cast<float *>(smem + lay.ebuf);
  unsigned *bins = reinterpret_cast<unsigned *>(smem + lay.bins);
  float *scales = reinterpret_cast<float *>(smem + lay.scales);
  float *invs = reinterpret_cast<float *>(smem + lay.invs);
  float *shifts = reinterpret_cast<float *>(smem + lay.shifts);
  float *part = reinterpret_cast<float *>(smem + lay.part);
  float *mpart = reinterpret_cast<float *>(smem + lay.mpart);
  unsigned char *misc = smem + lay.misc;
  int *items = reinterpret_cast<int *>(smem + lay.items);
  // the partner CTA's buffers (distributed shared memory)
  const float *vec_p = cl.map_shared_rank(vec, role ^ 1);
  const float *scales_p = cl.map_shared_rank(scales, role ^ 1);
  const float *invs_p = cl.map_shared_rank(invs, role ^ 1);
  unsigned char *misc_p = cl.map_shared_rank(misc, role ^ 1);
  const int D = a.D, D_pad = a.D_pad;
  const float lam = a.leak;
  const bool negate = a.mode == kPostNegate;

  // ---- LPT assignment of the batch over the clusters (identical in every CTA) ----
  lpt_assign<kNT>(a.lengths, a.B, a.T_max, nclusters, cluster, 2, reinterpret_cast<int *>(vec),
                  items);
  const int nitems = items[0];
  Ring ring;
  if constexpr (RING) {
    ring.init(smem + lay.ring, smem + lay.bars, smem + lay.ctab, warp);
    Ring::init_barriers(smem + lay.bars, kNW, tid);
    __syncthreads();
  }

  for (int it = 0; it < nitems; ++it) {
    const int b = items[4 + it];
    const int T = item_frames(a.lengths, b, a.T_max);
    if (T <= 0) {  // zero-length item: failed, no frames touched, no barriers
      if (fwd) {
        if (!a.packed)
          for (size_t i = tid; i < size_t(a.T_max) * D; i += kNT)
            a.post[size_t(b) * a.T_max * D + i] = 0.f;
        if (tid == 0) {
          a.logp[b] = NAN;
          a.fail[b] = 0;
        }
      }
      continue;
    }
    const int row = int(a.row_map[b]);
    const int *desc = a.g.desc + row * kDescInts;
    const int S = desc[kS], init = desc[kInit];
    const int ntiles = desc[kSTiles], stoff = desc[kSTileOff];
    const float *fin = a.g.fin32 + desc[kStateOff];
    const int *finfo = a.g.sf_info + size_t(stoff) * 32, *binfo = a.g.sb_info + size_t(stoff) * 32;
    const int *trips_arr = (fwd ? a.g.sf_trips : a.g.sb_trips) + stoff;
    const int *base_arr = (fwd ? a.g.sf_base : a.g.sb_base) + stoff;
    const uint2 *wp = fwd ? a.g.sf_wp + desc[kSfSlotOff] : a.g.sb_wp + desc[kSbSlotOff];
    const float upi = float(1.0 / double(S));
    // midpoint: 1 <= h <= T - 1 (T >= 2); T = 1: h = 1 (the backward CTA does frame 0)
    const int h = T == 1 ? 1 : min(T - 1, max(1, (T * hnum + 32) >> 6));
    const bool other_failed = a.other_fail != nullptr && a.other_fail[b] >= 0;

    long long off = 0;
    for (int j = tid; j < b; j += kNT) off += a.lengths[j];
    off = warp_sum(off);
    __syncthreads();  // previous item's readers of the scratch are done
    if (lane == 0) reinterpret_cast<long long *>(smem + 256)[warp] = off;
    __syncthreads();
    long long item_off = 0;
    for (int w = 0; w < kNW; ++w) item_off += reinterpret_cast<long long *>(smem + 256)[w];
    float *trellis = a.work + item_off * S32;
    const float *Lb = a.L + size_t(b) * a.T_max * D;
    float *post_b = a.post + size_t(b) * a.T_max * D;
    if (a.packed) {
      Lb = a.L + size_t(item_off) * D;
      post_b = a.post + size_t(item_off) * D;
    }

    // ---- log-likelihood rows in registers (two frames ahead) -------------------------
    float rn[kEPT], rn2[kEPT];
    auto load_row = [&](int t, float *r) {
#pragma unroll
      for (int j = 0; j < kEPT; ++j) {
        const int d = tid + j * kNT;
        r[j] = (t >= 0 && t < T && d < D) ? __ldg(Lb + size_t(t) * D + d) : -INFINITY;
      }
    };
    auto max_part = [&](int t, const float *r) {
      float m = r[0];
#pragma unroll
      for (int j = 1; j < kEPT; ++j) m = nan_max(m, r[j]);
      m = warp_max(m);
      if (lane == 0) mpart[(t & 1) * 32 + warp] = m;
    };
    auto compute_e = [&](int t, const float *r, bool record) {
      float m = lane < kNW ? mpart[(t & 1) * 32 + lane] : -INFINITY;
      m = warp_max(m);
#pragma unroll
      for (int j = 0; j < kEPT; ++j) {
        const int d = tid + j * kNT;
        if (d < D) ebuf[(t & 1) * D_pad + d] = expf(r[j] - m);
      }
      if (record && tid == 0) shifts[t] = m;
    };
    auto part_total = [&](const float *v) {
      float x = lane < kNW ? v[lane] : 0.f;
      return warp_sum(x);
    };
    // fixed-point bins of one frame -> its gradient row (then cleared)
    auto flush = [&](int f, int slot) {
      unsigned *bn = bins + slot * D_pad;
      float *prow = post_b + size_t(f) * D;
      for (int d = tid; d < D; d += kNT) {
        const float g = float(double(bn[d]) * (1.0 / double(kPostScale)));
        prow[d] = negate ? -g : g;
        bn[d] = 0u;
      }
    };
    // this warp's tiles: warp, warp + 32, ...; lane i keeps tile i's trips / base
    const int ntw = warp < ntiles ? (ntiles - warp + kNW - 1) / kNW : 0;
    const int my_trips = lane < ntw ? __ldg(trips_arr + warp + kNW * lane) : 0;
    const int my_base = lane < ntw ? __ldg(base_arr + warp + kNW * lane) : 0;
    for (int d = tid; d < 2 * D_pad; d += kNT) bins[d] = 0u;
    // Arc rows of one tile: body(w) per slot word, from the ring or from L2.
    auto tile_rows = [&](const uint2 *sp, int trips, auto &&body) {
      if constexpr (RING) {
        ring.rows(trips, body);
      } else {
        // 8 slot-row loads in flight per lane before their arc bodies (L2 latency)
        int j = 0;
        for (; j + kL2Rows <= trips; j += kL2Rows) {
          uint2 w[kL2Rows];
#pragma unroll
          for (int r = 0; r < kL2Rows; ++r) w[r] = ldg_slot(sp + 32 * (j + r));
#pragma unroll
          for (int r = 0; r < kL2Rows; ++r) body(w[r]);
        }
        for (; j < trips; ++j) body(ldg_slot(sp + 32 * j));
      }
    };
    // this CTA's arc-loop frames of the item: forward T (fewer only on a
    // failure, which drains the ring), backward T - h (+ h posterior frames)
    if constexpr (RING)
      ring.begin(wp, ntw, my_trips, my_base, fwd ? T : (other_failed ? T - h : T));

    if (fwd) {
      // ======================= forward CTA ==============================================
      if (!a.packed)
        for (size_t i = tid; i < size_t(a.T_max - T) * D; i += kNT) post_b[size_t(T) * D + i] = 0.f;
      for (int s = tid; s < S32; s += kNT) vec[s] = (s == init) ? 1.f : 0.f;
      {
        float r0[kEPT];
        load_row(0, r0);
        load_row(1, rn);
        load_row(2, rn2);
        max_part(0, r0);
        max_part(1, rn);
        __syncthreads();
        compute_e(0, r0, true);
        __syncthreads();
      }
      float inv2 = 1.f, leakc = 0.f, scale_prev = 1.f;
      int fail_at = -1;
      double kappa = 0.0;  // kappa_k during the posterior frames
      bool mid_done = false;
      auto midpoint = [&](const float *raw_h) {  // both barriers + kappa_h
        cluster_sync_rows();  // backward half done: rows >= h, inv_t, B_h, ld_h ready
        mid_done = true;
        const float ld_h = *reinterpret_cast<const float *>(misc_p + 8);
        const float *bh = vec_p + (h & 1) * S32;
        double acc = 0.0;
        for (int s = tid; s < S; s += kNT) acc += double(raw_h[s]) * double(bh[s] + ld_h);
        acc = warp_sum(acc);
        if (lane == 0) dscr[warp] = acc;
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < kNW; ++w) tot += dscr[w];
        if (tid == 0) *reinterpret_cast<double *>(misc_p) = tot;  // to the backward CTA
        kappa = tot;
        cl.sync();  // kappa_h delivered
      };
      for (int k = 0; k < T; ++k) {
        const int cur = k & 1, nxt = cur ^ 1;
        if (k == h && !mid_done) midpoint(vec + cur * S32);
        if (k > 0) {
          const float t0 = part_total(part + cur * 32);
          float t2 = t0;
          leakc = 0.f;
          if (lam > 0.f && t0 > 0.f) {
            leakc = lam * t0;
            t2 = t0 + leakc;
          }
          if (!(t2 >= a.floor_eff) || isinf(t2)) {
            fail_at = k - 1;
            if constexpr (RING) ring.drain();
            break;
          }
          inv2 = __frcp_rn(t2);
          scale_prev = t2;
          if (tid == 0) scales[k - 1] = t2;
        }
        const float lu = leakc * upi;
        if (k < h) {  // alpha_k for the backward CTA's posteriors (backward-pack order)
          const float *r = vec + cur * S32;
          float *arow = trellis + size_t(k) * S32;
          for (int q = tid; q < ntiles * 32; q += kNT) {
            const int s = __ldg(binfo + q);
            if (s >= 0) arow[q] = (r[s] + lu) * inv2;
          }
        }
        const bool post = k >= h && !other_failed;
        // Z_k = kappa_k / scale_{k-1}; terms scaled by 1 / Z_k sum to 1
        float zs = 0.f;
        const double zk = post ? kappa / double(scale_prev) : 0.0;
        if (post) zs = (zk > 0.0 && zk < 1e38) ? float(1.0 / zk) : 0.f;
        if (k + 1 < T) compute_e(k + 1, rn, true);
#pragma unroll
        for (int j = 0; j < kEPT; ++j) rn[j] = rn2[j];
        load_row(k + 3, rn2);
        if (post && k > h) flush(k - 1, (k - 1) & 1);
        {
          const uint32_t e32 = smem_u32(ebuf + cur * D_pad), r32 = smem_u32(vec + cur * S32);
          float *rnew = vec + nxt * S32;
          const float *brow = trellis + size_t(k) * S32;  // beta'_{k+1} (forward-pack order)
          const uint32_t bn32 = smem_u32(bins + cur * D_pad);
          const bool last = (k + 1 == T);
          float psum = 0.f;
          int s_next = ntw > 0 ? __ldg(finfo + warp * 32 + lane) : -1;
          float b_next = (post && ntw > 0) ? brow[warp * 32 + lane] : 0.f;
          for (int i = 0; i < ntw; ++i) {
            const int tile = warp + kNW * i;
            const int s = s_next;
            const float cb = s >= 0 ? b_next * inv2 * zs : 0.f;
            if (i + 1 < ntw) {
              s_next = __ldg(finfo + (tile + kNW) * 32 + lane);
              if (post) b_next = brow[(tile + kNW) * 32 + lane];
            }
            const int trips = __shfl_sync(kFull, my_trips, i);
            const uint2 *sp = wp + __shfl_sync(kFull, my_base, i) + lane;
            float A = 0.f, Bs = 0.f;
            if (post) {
              tile_rows(sp, trips, [&](const uint2 w) {
                const uint32_t pdf4 = (w.x >> 15) << 2;
                const float q = __uint_as_float(w.y) * lds_f(e32 + pdf4);
                const float rs = lds_f(r32 + ((w.x & 0x7FFFu) << 2));
                A = fmaf(q, rs, A);
                Bs += q;
                red_add_shared_nz(bn32 + pdf4, __float2uint_rn(q * (rs + lu) * cb * kPostScale));
              });
            } else {
              tile_rows(sp, trips, [&](const uint2 w) {
                const float q = __uint_as_float(w.y) * lds_f(e32 + ((w.x >> 15) << 2));
                A = fmaf(q, lds_f(r32 + ((w.x & 0x7FFFu) << 2)), A);
                Bs += q;
              });
            }
            if (s >= 0) {
              float raw = inv2 * (A + lu * Bs);
              if (last) raw *= fin[s];
              rnew[s] = raw;
              psum += raw;
            }
          }
          psum = warp_sum(psum);
          if (lane == 0) part[nxt * 32 + warp] = psum;
        }
        max_part(k + 2, rn);
        __syncthreads();
        if (post) kappa = zk / double(invs_p[k + 1]);  // kappa_{k+1} = Z_k / inv_{k+1}
      }
      if (fail_at < 0) {
        const float t0 = part_total(part + (T & 1) * 32);
        float t2 = t0;
        if (lam > 0.f && t0 > 0.f) t2 = t0 + lam * t0;
        if (!(t2 >= a.floor_eff) || isinf(t2))
          fail_at = T - 1;
        else if (tid == 0)
          scales[T - 1] = t2;
        if (T - 1 >= h && !other_failed) flush(T - 1, (T - 1) & 1);
      }
      __syncthreads();
      if (!mid_done) {  // failed before the midpoint, or T == 1 (h == T)
        // T == 1: the backward CTA's only frame needs kappa_1 = scale_0
        if (tid == 0) {
          *reinterpret_cast<double *>(misc_p) = fail_at < 0 ? double(scales[T - 1]) : 1.0;
        }
        cluster_sync_rows();
        cl.sync();
      }
      if (fail_at >= 0) {
        for (int k = fail_at + 1 + warp; k < T; k += kNW) {
          float m = -INFINITY;
          for (int d = lane; d < D; d += 32) m = nan_max(m, Lb[size_t(k) * D + d]);
          m = warp_max(m);
          if (lane == 0) shifts[k] = m;
        }
        for (int k = fail_at + tid; k < T; k += kNT) scales[k] = 1.f;
      }
      __syncthreads();
      {
        double acc = 0.0;
        for (int k = tid; k < T; k += kNT) {
          const double v = log(double(scales[k])) + double(shifts[k]);
          acc += v;
          if (a.scale_logs) a.scale_logs[size_t(b) * a.T_max + k] = v;
        }
        if (a.scale_logs)
          for (int k = T + tid; k < a.T_max; k += kNT) a.scale_logs[size_t(b) * a.T_max + k] = 0.0;
        acc = warp_sum(acc);
        if (lane == 0) dscr[warp] = acc;
        __syncthreads();
        if (tid == 0) {
          double tot = 0.0;
          for (int w = 0; w < kNW; ++w) tot += dscr[w];
          a.logp[b] = fail_at >= 0 ? NAN : tot;
          a.fail[b] = fail_at;
        }
      }
      cluster_sync_rows();  // end: the backward CTA's posterior rows are written
      if (fail_at >= 0 || other_failed)
        for (size_t i = tid; i < size_t(T) * D; i += kNT) post_b[i] = 0.f;
    } else {
      // ======================= backward CTA =============================================
      // B_t = b_t + ld_t (own scale); column T: fin (1 + leak)
      for (int s = tid; s < S32; s += kNT) vec[(T & 1) * S32 + s] = s < S ? fin[s] * (1.f + lam) : 0.f;
      {
        float dp = 0.f;
        for (int s = tid; s < S; s += kNT) dp = fmaf(upi, fin[s] * (1.f + lam), dp);
        dp = warp_sum(dp);
        if (lane == 0) part[(T & 1) * 32 + warp] = dp;
        float r0[kEPT];
        load_row(T - 1, r0);
        load_row(T - 2, rn);
        load_row(T - 3, rn2);
        max_part(T - 1, r0);
        max_part(T - 2, rn);
        __syncthreads();
        compute_e(T - 1, r0, false);
        __syncthreads();
      }
      double kappa = 0.0;
      // iteration t: arcs of frame f = t - 1, column t (raw b_t) in vec[t & 1]
      auto bframe = [&](int t, bool post) {
        const int ct = t & 1, cp = ct ^ 1;
        const int f = t - 1;
        const float t0 = part_total(part + ct * 32);  // mean of b_t
        const float ld = (t < T && lam > 0.f) ? lam * t0 : 0.f;
        const float n = float(S) * (t0 + ld);
        const float inv = (n > 0.f && !isinf(n)) ? __frcp_rn(n) : 1.f;
        if (tid == 0) invs[t] = inv;
        if (!post) {  // beta'_t = B_t inv_t -> row f (forward-pack order)
          const float *bt = vec + ct * S32;
          float *brow = trellis + size_t(f) * S32;
          for (int q = tid; q < ntiles * 32; q += kNT) {
            const int s = __ldg(finfo + q);
            if (s >= 0) brow[q] = (bt[s] + ld) * inv;
          }
        }
        if (post && t < h) flush(t, t & 1);  // frame t (previous iteration)
        if (t - 2 >= 0) compute_e(t - 2, rn, false);
#pragma unroll
        for (int j = 0; j < kEPT; ++j) rn[j] = rn2[j];
        load_row(t - 4, rn2);
        const float zinv = post ? ((kappa > 0.0 && kappa < 1e38) ? float(1.0 / kappa) : 0.f) : 0.f;
        {
          const uint32_t b32 = smem_u32(vec + ct * S32), e32 = smem_u32(ebuf + cp * D_pad);
          float *bnew = vec + cp * S32;
          const float *arow = trellis + size_t(f) * S32;  // alpha_f, backward-pack order
          const uint32_t bn32 = smem_u32(bins + (f & 1) * D_pad);
          float dq = 0.f;
          int s_next = -1;
          float a_next = 0.f;
          if (ntw > 0) {
            s_next = __ldg(binfo + warp * 32 + lane);
            if (post) a_next = arow[warp * 32 + lane];
          }
          for (int i = 0; i < ntw; ++i) {
            const int tile = warp + kNW * i;
            const int s = s_next;
            const float as = s >= 0 ? a_next * zinv : 0.f;
            if (i + 1 < ntw) {
              s_next = __ldg(binfo + (tile + kNW) * 32 + lane);
              if (post) a_next = arow[(tile + kNW) * 32 + lane];
            }
            const int trips = __shfl_sync(kFull, my_trips, i);
            const uint2 *sp = wp + __shfl_sync(kFull, my_base, i) + lane;
            float A = 0.f;
            if (post) {
              tile_rows(sp, trips, [&](const uint2 w) {
                const uint32_t pdf4 = (w.x >> 15) << 2;
                const float term = __uint_as_float(w.y) * lds_f(e32 + pdf4) *
                                   (lds_f(b32 + ((w.x & 0x7FFFu) << 2)) + ld);
                A += term;
                red_add_shared_nz(bn32 + pdf4, __float2uint_rn(as * term * kPostScale));
              });
            } else {
              tile_rows(sp, trips, [&](const uint2 w) {
                A += __uint_as_float(w.y) * lds_f(e32 + ((w.x >> 15) << 2)) *
                     (lds_f(b32 + ((w.x & 0x7FFFu) << 2)) + ld);
              });
            }
            if (s >= 0) {
              const float v = inv * A;
              bnew[s] = v;
              dq = fmaf(upi, v, dq);
            }
          }
          dq = warp_sum(dq);
          if (lane == 0) part[cp * 32 + warp] = dq;
        }
        if (t - 3 >= 0) max_part(t - 3, rn);
        __syncthreads();
        if (post && t >= 2) kappa = double(inv) * kappa * double(scales_p[t - 2]);  // kappa_{t-1}
      };
      for (int t = T; t > h; --t) bframe(t, false);
      // midpoint: B_h's leak term for the forward CTA's kappa_h, then two cluster barriers
      if (warp == 0) {
        const float t0 = part_total(part + (h & 1) * 32);  // mean of b_h
        if (lane == 0) *reinterpret_cast<float *>(misc + 8) = (h < T && lam > 0.f) ? lam * t0 : 0.f;
      }
      cluster_sync_rows();
      cl.sync();  // kappa_h written by the forward CTA
      kappa = *reinterpret_cast<const double *>(misc);
      if (!other_failed)
        for (int t = h; t >= 1; --t) bframe(t, true);
      __syncthreads();
      if (!other_failed) flush(0, 0);
      cluster_sync_rows();  // end
    }
  }
}

int launch_stream_split(const FBArgs<float> &a, const lfmmi_graphs *g, cudaStream_t st) {
  if (!g->streamable) return set_error(LFMMI_ERR_UNSUPPORTED, "graph has no stream pack");
  if (a.leak_pi) return set_error(LFMMI_ERR_UNSUPPORTED, "stream split: uniform leak only");
  if (a.D > kMaxD) return set_error(LFMMI_ERR_UNSUPPORTED, "stream split: D > 2048");
  if (a.mode != kPostWrite && a.mode != kPostNegate)
    return set_error(LFMMI_ERR_UNSUPPORTED, "stream split: WRITE / NEGATE modes only");
  const int S32 = (g->max_states + 31) & ~31;
  if (2 * S32 < 2 * a.B || g->max_stiles > 32 * kNW)
    return set_error(LFMMI_ERR_UNSUPPORTED, "stream split: batch / graph shape");
  const Options &opt = options();
  // TMA ring when its table holds a warp's chunks and it fits next to the columns
  const int tiles_per_warp = (g->max_stiles + kNW - 1) / kNW;
  const int max_deg = std::max(g->max_in_deg, g->max_out_deg);
  // (option ssplit_ring: the TMA slot ring; off by default since the L2 path
  // with 8 row loads in flight per lane measured faster: biphone 7.09 vs 7.68 ms)
  bool ring = opt.ssplit_ring != 0 && ring_chunks_needed(tiles_per_warp, max_deg, 8) <= 64 &&
              ss_layout(S32, a.D_pad, a.T_pad, true).total <= unsigned(kMaxSmem);
  const SSLayout lay = ss_layout(S32, a.D_pad, a.T_pad, ring);
  if (lay.total > unsigned(kMaxSmem))
    return set_error(LFMMI_ERR_UNSUPPORTED,
                     "stream split needs " + std::to_string(lay.total) + " B shared memory");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // every SM pair: the numerators (0.85 ms alone at biphone) run in the
  // denominator's tail (biphone step 7.10 / 7.04 ms with 72 / 74 clusters)
  int nc = opt.split_clusters > 0 ? opt.split_clusters : std::min(a.B, sms / 2);
  nc = std::max(1, std::min(nc, std::min(96, sms / 2)));
  nc = std::max(nc, (a.B + kMaxItems - 1) / kMaxItems);
  if (nc > std::min(96, sms / 2))
    return set_error(LFMMI_ERR_UNSUPPORTED, "stream split: too many utterances per cluster");
  auto kern = ring ? fb_streamsplit_kernel<true> : fb_streamsplit_kernel<false>;
  static bool configured[2] = {false, false};
  if (!configured[ring]) {
    const int rc = check_cuda(
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem),
        "cudaFuncSetAttribute(stream split)");
    if (rc) return rc;
    configured[ring] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * nc);
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = lay.total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_den_kernel(ring ? "fb_streamsplit_kernel (2-CTA cluster: forward | backward, TMA slot ring)"
                       : "fb_streamsplit_kernel (2-CTA cluster: forward | backward, L2 packs)");
  const int hnum = std::max(1, std::min(63, opt.split_h64));
  return check_cuda(cudaLaunchKernelEx(&cfg, kern, a, S32, lay, nc, hnum),
                    "fb_streamsplit_kernel launch");
}

}  // namespace lfmmi
