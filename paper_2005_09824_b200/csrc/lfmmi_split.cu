// Denominator forward-backward split across a 2-CTA thread-block cluster
// ("meet in the middle"): CTA 0 runs the forward recursion over frames 0..T-1,
// CTA 1 the backward recursion over frames T-1..0, concurrently, on two SMs.
//
//   CTA 0 (forward)  frames 0..h-1: alpha columns, spilled to the trellis rows 0..h-1
//                    frames h..T-1: alpha + arc posteriors, using the beta rows
//   CTA 1 (backward) frames T-1..h: beta columns (own per-frame normalisers),
//                                   spilled to the trellis rows h..T-1
//                    frames h-1..0: beta + arc posteriors, using the alpha rows
//
// with one cluster barrier at the midpoint h = T/2 (each half only needs the
// other CTA's finished first half) and one at the end of the utterance.  The
// critical path of an utterance is T frames of one recursion instead of 2T,
// and the batch is load-balanced over the clusters (LPT on the utterance
// lengths, computed identically by every CTA), so the step is ~sum(T)/(2 x
// clusters) frames instead of max(T) — the fix for the WSJ-mono batch (128
// utterances of 150-300 frames on 148 SMs), whose step was bound by its
// longest utterance.
//
// Posteriors: the arc terms of frame f are alpha'_{f-1}(src) p e_f(pdf)
// beta'_f(dst) in each CTA's own normalisation; their sum Z_f is the same for
// every frame in exact arithmetic (forward-backward identity, leaky HMM
// included), so gamma_f = slots / Z_f equals the reference's
// alpha-beta-with-forward-scales posterior (forward_backward.py:240-307) up to
// rounding.  Objective, scales and failure frames come from the forward CTA
// exactly as in fb_tile_kernel.
//
// fp32, uniform leak distribution, WRITE / NEGATE posterior modes, arc packs in
// shared memory; everything else stays on fb_tile_kernel.
#include <cooperative_groups.h>

#include "lfmmi_device.cuh"
#include "lfmmi_kernels.h"
#include "lfmmi_lpt.cuh"
#include "lfmmi_options.h"
#include "lfmmi_schedule.h"
#include "lfmmi_tile_common.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

namespace cg = cooperative_groups;

namespace lfmmi {

namespace {

constexpr int kNW = 16, kNT = 32 * kNW;
constexpr int kMaxClusters = 96;              // clusters (LPT bins) per launch
constexpr int kRowAhead = 4, kStageRing = 8;  // log-likelihood row pipeline (as fb_tile_kernel)
constexpr int kRing = 3, kRingAhead = 2;      // other CTA's trellis rows: issued 2 frames ahead
constexpr int kWait = 1;                      // groups still in flight at the end of a frame
constexpr int kMaxItems = kLptMaxItems;       // utterances per cluster (launcher guarantees)

struct SplitLayout {
  size_t wp, xs, tinfo, ttrips, tbase, wlist, wtab, wlist2, wtab2, pdfptr, xterm, rbuf, ring, ebuf, stage,
      scales, shifts, part, partz, mpart, items, total;
};

__host__ __device__ inline SplitLayout split_layout(int F, int nt, int D, int X_pad, int S_pad,
                                                    int D_pad, int T_pad, int RB, int EB,
                                                    bool smem_scales) {
  SplitLayout l;
  size_t o = 512;  // scratch: 32 doubles + 32 int64
  l.wp = o;      o = al16(o + size_t(F) * 8);
  l.xs = o;      o = al16(o + size_t(F) * 2);
  l.tinfo = o;   o = al16(o + size_t(nt) * 128);
  l.ttrips = o;  o = al16(o + size_t(pad4(nt)) * 4);
  l.tbase = o;   o = al16(o + size_t(pad4(nt)) * 4);
  l.wlist = o;   o = al16(o + size_t(pad4(nt)) * 4);
  l.wtab = o;    o = al16(o + size_t(kWarpTable) * 4);
  l.wlist2 = o;  o = al16(o + size_t(pad4(nt)) * 4);  // forward CTA, posterior half
  l.wtab2 = o;   o = al16(o + size_t(kWarpTable) * 4);
  l.pdfptr = o;  o = al16(o + size_t(D + 1) * 4);
  l.xterm = o;   o = al16(o + size_t(2) * X_pad * 4);
  l.rbuf = o;    o = al16(o + size_t(2) * RB * 4);
  l.ring = o;    o = al16(o + size_t(kRing) * S_pad * 4);
  l.ebuf = o;    o = al16(o + size_t(2) * EB * 4);
  l.stage = o;   o = al16(o + size_t(kStageRing) * D_pad * 4);
  l.scales = o;  o = al16(o + (smem_scales ? size_t(T_pad) * 4 : 0));
  l.shifts = o;  o = al16(o + (smem_scales ? size_t(T_pad) * 4 : 0));
  l.part = o;    o += 2 * 32 * 4;
  l.partz = o;   o += 2 * 32 * 4;
  l.mpart = o;   o += 2 * 32 * 4;
  l.items = o;   o = al16(o + size_t(kMaxItems + 4) * 4);
  l.total = o;
  return l;
}

__device__ __forceinline__ void cluster_barrier() {
  __threadfence();  // trellis rows written to global memory before the arrive
  cg::this_cluster().sync();
}

}  // namespace

// kGrp: some row's tile packs have G > 1 lanes per state (partial sums over G
// lanes); compiled out otherwise.  (A 4-warp variant for small graphs — one
// cluster per utterance, several per SM — measured slower on the 43-state hmm
// den: 0.77 vs 0.61 ms.)
template <bool kGrp>
__global__ void __launch_bounds__(kNT, 1)
    fb_split_kernel(const FBArgs<float> a, int Fmax, int ntiles_max, int X_pad, int nclusters,
                    int hnum) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ctid = kNT - 1 - tid, cwarp = ctid >> 5;  // chores on the last warps
  const int role = int(cg::this_cluster().block_rank());  // 0 forward, 1 backward
  const int cluster = blockIdx.x >> 1;
  const int RB = pad4(a.rep_r * a.r_stride), EB = a.rep_e * a.e_stride;
  const SplitLayout lay = split_layout(Fmax, ntiles_max, a.D, X_pad, a.S_pad, a.D_pad, a.T_pad,
                                       RB, EB, a.sc_smem != 0);
  double *dscr = reinterpret_cast<double *>(smem);
  long long *lscr = reinterpret_cast<long long *>(smem + 256);
  int *pdfptr = reinterpret_cast<int *>(smem + lay.pdfptr);
  float *xterm = reinterpret_cast<float *>(smem + lay.xterm);
  float *rbuf = reinterpret_cast<float *>(smem + lay.rbuf);
  float *ring = reinterpret_cast<float *>(smem + lay.ring);
  float *ebuf = reinterpret_cast<float *>(smem + lay.ebuf);
  float *stage = reinterpret_cast<float *>(smem + lay.stage);
  float *part = reinterpret_cast<float *>(smem + lay.part);
  float *mpart = reinterpret_cast<float *>(smem + lay.mpart);
  int *items = reinterpret_cast<int *>(smem + lay.items);
  const uint32_t wp32 = smem_u32(smem + lay.wp), xs32 = smem_u32(smem + lay.xs);
  const unsigned *tinfo = reinterpret_cast<const unsigned *>(smem + lay.tinfo);
  const int *ttrips = reinterpret_cast<const int *>(smem + lay.ttrips);
  const int *tbase = reinterpret_cast<const int *>(smem + lay.tbase);
  const int *wl1 = reinterpret_cast<const int *>(smem + lay.wlist);
  const int *wt1 = reinterpret_cast<const int *>(smem + lay.wtab);
  const int *wl2 = reinterpret_cast<const int *>(smem + lay.wlist2);
  const int *wt2 = reinterpret_cast<const int *>(smem + lay.wtab2);
  const int D = a.D, S_pad = a.S_pad, D_pad = a.D_pad;
  const float lam = a.leak;
  const bool fwd = role == 0;

  // ---- this cluster's utterances: LPT over the clusters, longest first (every CTA
  // computes the same assignment; lengths / order staged in the slot buffers)
  lpt_assign<kNT>(a.lengths, a.B, a.T_max, nclusters, cluster, 4,
                  reinterpret_cast<int *>(xterm), items);
  const int nitems = items[0];

  // ---- the arc pack of this CTA's direction (reloaded only when the row changes) -----
  int bound_row = -1;
  auto bind = [&](int row) {
    const int *desc = a.g.desc + row * kDescInts;
    const int so = desc[fwd ? kTfSlotOff : kTbSlotOff], nsl = desc[fwd ? kTfSlots : kTbSlots];
    const int ntiles = desc[kNTiles], toff = desc[kTileOff];
    copy16<kNT>(smem + lay.wp, (fwd ? a.g.tf_wp : a.g.tb_wp) + so, size_t(nsl) * 8, tid);
    copy16<kNT>(smem + lay.xs, (fwd ? a.g.tf_xslot : a.g.tb_xslot) + so, size_t(nsl) * 2, tid);
    copy16<kNT>(smem + lay.tinfo, (fwd ? a.g.tf_info : a.g.tb_info) + size_t(toff) * 32,
                size_t(ntiles) * 128, tid);
    copy16<kNT>(smem + lay.ttrips, (fwd ? a.g.tf_trips : a.g.tb_trips) + toff,
                size_t(pad4(ntiles)) * 4, tid);
    copy16<kNT>(smem + lay.tbase, (fwd ? a.g.tf_base : a.g.tb_base) + toff,
                size_t(pad4(ntiles)) * 4, tid);
    copy16<kNT>(smem + lay.wlist, (fwd ? a.g.tf_wlist : a.g.tb_wlist) + toff,
                size_t(pad4(ntiles)) * 4, tid);
    copy16<kNT>(smem + lay.wtab, (fwd ? a.g.tf_wtab : a.g.tb_wtab) + desc[kWTabOff],
                size_t(kWarpTable) * 4, tid);
    if (fwd) {
      copy16<kNT>(smem + lay.wlist2, a.g.tp_wlist + toff, size_t(pad4(ntiles)) * 4, tid);
      copy16<kNT>(smem + lay.wtab2, a.g.tp_wtab + desc[kWTabOff], size_t(kWarpTable) * 4, tid);
    }
    const int *pp = a.g.pdf_arc_ptr + desc[kPdfPtrOff2];
    for (int d = tid; d <= D; d += kNT) pdfptr[d] = pp[d];
    // padding slots of the per-pdf groups are never written: zero them once per
    // pack (the buffers also held the scheduling scratch)
    for (int i = tid; i < 2 * X_pad; i += kNT) xterm[i] = 0.f;
    cp_async_commit();
    cp_async_wait<0>();
    bound_row = row;
  };

  // gamma_t[d] = (sum of pdf d's slots) / Z_t: SPL chore lanes per pdf.
  int spl = 1, spl_log = 0;
  while (spl < 32 && D * spl * 2 <= kNT) {
    spl <<= 1;
    ++spl_log;
  }
  const bool flusher = cwarp * 32 < D * spl;
  const bool negate = a.mode == kPostNegate;
  const bool rep2 = a.rep_r > 1;
  const int rstride = a.r_stride;

  for (int it = 0; it < nitems; ++it) {
    const int b = items[4 + it];
    const int T = item_frames(a.lengths, b, a.T_max);
    if (T <= 0) {  // zero-length item (host APIs reject it): failed, no frames touched
      if (fwd) {
        if (!a.packed)
          for (size_t i = tid; i < size_t(a.T_max) * D; i += kNT)
            a.post[size_t(b) * a.T_max * D + i] = 0.f;
        if (tid == 0) {
          a.logp[b] = NAN;
          a.fail[b] = 0;
        }
      }
      continue;  // no barriers: both CTAs skip it
    }
    const int row = int(a.row_map[b]);
    const int *desc = a.g.desc + row * kDescInts;
    const int S = desc[kS], init = desc[kInit];
    const int G = desc[kTileG];  // lanes per state: partial sums over G adjacent lanes
    const bool lead = (lane & (G - 1)) == 0;
    const float *fin = a.g.fin32 + desc[kStateOff];
    const float upi = float(1.0 / double(S));
    // forward CTA: posteriors of frames >= h; backward CTA: < h.  The forward
    // posterior frame costs ~7% more than the backward one (measured, WSJ-mono),
    // so the forward CTA takes slightly fewer: h = T * hnum / 64, <= T - 1.
    const int h = min(T - 1, (T * hnum + 32) >> 6);
    const bool other_failed = a.other_fail != nullptr && a.other_fail[b] >= 0;

    if (a.prof != nullptr && tid == 0)
      a.prof[(size_t(blockIdx.x) * kMaxItems + it) * 8] = clock64();
    long long off = 0;
    for (int j = tid; j < b; j += kNT) off += a.lengths[j];
    off = warp_sum(off);
    __syncthreads();  // previous item's readers of the scratch are done
    if (lane == 0) lscr[warp] = off;
    if (row != bound_row) bind(row);
    __syncthreads();
    long long item_off = 0;
    for (int w = 0; w < kNW; ++w) item_off += lscr[w];
    float *trellis = a.work + item_off * S_pad;
    float *scales, *shifts;
    if (a.sc_smem) {
      scales = reinterpret_cast<float *>(smem + lay.scales);
      shifts = reinterpret_cast<float *>(smem + lay.shifts);
    } else {
      scales = a.work + a.sc_off + item_off;
      shifts = scales + a.sc_total;
    }
    // With the emissions pre-pass (chain loss), the staged rows are E = exp(L - m)
    // and the row maxima come precomputed: the chore warps only copy rows.
    const bool pre = a.E != nullptr;
    const float *Lb = (pre ? a.E : a.L) + size_t(b) * a.T_max * D;
    const float *Emb = pre ? a.Em + size_t(b) * a.T_max : nullptr;
    float *post_b = a.post + size_t(b) * a.T_max * D;
    if (a.packed) {
      Lb = (pre ? a.E : a.L) + size_t(item_off) * D;
      if (pre) Emb = a.Em + size_t(item_off);
      post_b = a.post + size_t(item_off) * D;
    }
    // forward CTA: LPT lists without / with the flush chore (first / second half)
    const int *wl = wl1;
    int wlo = wt1[warp], whi = wt1[warp + 1];

    const int nrw = (D + 31) / 32 < kNW ? (D + 31) / 32 : kNW;  // chore warps (row elements)
    auto issue_row = [&](int t) {
      if (t < 0 || t >= T || cwarp >= nrw) return;
      const float *src = Lb + size_t(t) * D;
      float *dst = stage + (t & (kStageRing - 1)) * D_pad;
      for (int d = ctid; d < D; d += kNT) cp_async_elem(dst + d, src + d);
    };
    auto row_max_part = [&](int t) {
      if (pre || t < 0 || t >= T || cwarp >= nrw) return;
      const float *src = stage + (t & (kStageRing - 1)) * D_pad;
      float m = -INFINITY;
      for (int d = ctid; d < D; d += kNT) m = nan_max(m, src[d]);
      m = warp_max(m);
      if (lane == 0) mpart[(t & 1) * 32 + cwarp] = m;
    };
    auto compute_e = [&](int t, bool record_shift) {
      if (cwarp >= nrw) return;
      const float *src = stage + (t & (kStageRing - 1)) * D_pad;
      float *dst = ebuf + (t & 1) * EB;
      if (pre) {  // staged row already holds exp(L - m)
        for (int d = ctid; d < D; d += kNT) {
          const float v = src[d];
          for (int c = 0; c < a.rep_e; ++c) dst[c * a.e_stride + d] = v;
        }
        (void)record_shift;  // row maxima read once at the end (no per-frame global load)
        return;
      }
      const float *mp = mpart + (t & 1) * 32;
      float m = lane < nrw ? mp[lane] : -INFINITY;
      m = warp_max(m);
      for (int d = ctid; d < D; d += kNT) {
        const float v = exp_r(src[d] - m);
        for (int c = 0; c < a.rep_e; ++c) dst[c * a.e_stride + d] = v;
      }
      if (record_shift && ctid == 0) shifts[t] = m;
    };
    auto issue_trellis = [&](int k) {  // the other CTA's row k -> ring
      if (k < 0 || k >= T) return;
      copy16<kNT>(ring + (k % kRing) * S_pad, trellis + size_t(k) * S_pad,
                  size_t(S_pad) * sizeof(float), ctid);
    };
    auto put_vec = [&](float *v, int s, float x) {
      v[s] = x;
      if (rep2) v[rstride + s] = x;
    };
    auto flush_post = [&](int t, const float *xsrc) {
      float *prow = post_b + size_t(t) * D;
      const int sub = ctid & (spl - 1);
      for (int base_i = 0; base_i < D * spl; base_i += kNT) {
        const int idx = base_i + ctid;
        const int d = idx >> spl_log;
        float g = 0.f;
        if (d < D) {
          const int lo = pdfptr[d] >> 2, hi = pdfptr[d + 1] >> 2;
          for (int q = lo + sub; q < hi; q += spl) g += sum_groups4(xsrc + 4 * q, 1);
        }
        for (int o = 1; o < spl; o <<= 1) g += __shfl_xor_sync(kFull, g, o);
        if (d < D && sub == 0) prow[d] = negate ? -g : g;
      }
    };
    // Posterior rows [f0, f1) of this CTA: divide by Z_f = |sum of the row| (the
    // sum of all arc terms of frame f), one warp per row, after the last flush.
    auto normalize_rows = [&](int f0, int f1) {
      for (int f = f0 + warp; f < f1; f += kNW) {
        float *prow = post_b + size_t(f) * D;
        float z = 0.f;
        for (int d = lane; d < D; d += 32) z += prow[d];
        z = warp_sum(z);
        const float iz = rcp_rn(fabsf(z));
        for (int d = lane; d < D; d += 32) prow[d] *= iz;
      }
    };
    bool mid_done = false;
    auto stamp = [&](int j) {
      if (a.prof != nullptr && tid == 0) {
        long long *pr = a.prof + (size_t(blockIdx.x) * kMaxItems + it) * 8;
        pr[j] = clock64();
        pr[6] = T;
        pr[7] = h;
      }
    };

    if (fwd) {
      // ================= forward CTA ===================================================
      if (!a.packed) {
        const size_t n = size_t(a.T_max - T) * D;
        for (size_t i = tid; i < n; i += kNT) post_b[size_t(T) * D + i] = 0.f;
      }
      for (int i = tid; i < 2 * RB; i += kNT) rbuf[i] = 0.f;
      __syncthreads();
      for (int s = tid; s < S; s += kNT) put_vec(rbuf, s, (s == init) ? 1.f : 0.f);
      for (int j = 0; j < kRowAhead; ++j) {
        issue_row(j);
        cp_async_commit();
      }
      cp_async_wait<kWait>();
      row_max_part(0);
      row_max_part(1);
      __syncthreads();
      compute_e(0, true);
      __syncthreads();

      float inv2 = 1.f, leakc = 0.f;
      int fail_at = -1;
      // One forward frame; POST (compile-time) adds the posterior slots.  Returns
      // false when the frame's input column fails the scale floor.
      auto fframe = [&](int k, auto postc) -> bool {
        constexpr bool POST = decltype(postc)::value;
        const int cur = k & 1, nxt = cur ^ 1;
        if (k > 0) {
          const float t0 = lane_sum<kNW>(part + cur * 32, lane);
          float t2 = t0;
          leakc = 0.f;
          if (lam > 0.f && t0 > 0.f) {
            leakc = lam * t0;
            t2 = t0 + leakc;  // uniform pi: sum(pi) = 1
          }
          if (!(t2 >= a.floor_eff) || isinf(t2)) {
            fail_at = k - 1;
            return false;
          }
          inv2 = rcp_fast(t2);
          if (tid == 0) scales[k - 1] = t2;
        }
        const float lu = leakc * upi;
        if (k < h) {  // alpha'_{k-1} for the backward CTA's posteriors
          const float4 *r4 = reinterpret_cast<const float4 *>(rbuf + cur * RB);
          float4 *a4 = reinterpret_cast<float4 *>(trellis + size_t(k) * S_pad);
          for (int q = tid; q < (S_pad >> 2); q += kNT) {
            float4 v = r4[q];
            v.x = (v.x + lu) * inv2;
            v.y = (v.y + lu) * inv2;
            v.z = (v.z + lu) * inv2;
            v.w = (v.w + lu) * inv2;
            a4[q] = v;
          }
        }
        if (POST && k - 1 >= h && flusher) flush_post(k - 1, xterm + ((k - 1) & 1) * X_pad);
        if (k + 1 < T) compute_e(k + 1, true);
        issue_row(k + kRowAhead);
        if (POST) issue_trellis(k + kRingAhead);
        cp_async_commit();
        {
          const uint32_t e32 = smem_u32(ebuf + cur * EB), r32 = smem_u32(rbuf + cur * RB);
          float *rn = rbuf + nxt * RB;
          const bool last = (k + 1 == T);
          float psum = 0.f;
          for (int rr = wlo; rr < whi; ++rr) {
            const int tile = wl[rr];
            const unsigned info = tinfo[tile * 32 + lane];
            const int trips = ttrips[tile];
            const int base = tbase[tile] + lane;
            const int s = int(info & 0xFFFFu);
            float raw;
            if constexpr (POST) {
              const float *bet = ring + (k % kRing) * S_pad;
              const float cb = s != 0xFFFF ? inv2 * bet[s] : 0.f;
              const float A = fwd_post_tile_f32(wp32 + uint32_t(base) * 8u,
                                                xs32 + uint32_t(base) * 2u, trips, e32, r32,
                                                smem_u32(xterm + (k & 1) * X_pad), lu, cb);
              raw = inv2 * A;
            } else {
              float A = 0.f, Bs = 0.f;
              if (leakc != 0.f)
                fwd_tile_f32<true>(wp32 + uint32_t(base) * 8u, trips, e32, r32, A, Bs);
              else
                fwd_tile_f32<false>(wp32 + uint32_t(base) * 8u, trips, e32, r32, A, Bs);
              raw = inv2 * (A + lu * Bs);
            }
            if constexpr (kGrp) raw = group_sum(raw, G);
            if (s != 0xFFFF && (!kGrp || lead)) {
              if (last) raw *= fin[s];
              put_vec(rn, s, raw);
              psum += raw;
            }
          }
          psum = warp_sum(psum);
          if (lane == 0) part[nxt * 32 + warp] = psum;
        }
        // plain frames: log-likelihood rows only, two frames of slack; posterior
        // frames: the trellis row issued last frame must land too
        if constexpr (POST)
          cp_async_wait<kWait>();
        else
          cp_async_wait<kRowAhead - 2>();
        row_max_part(k + 2);
        __syncthreads();
        return true;
      };
      stamp(1);
      bool ok = true;
      for (int k = 0; k < h && ok; ++k) ok = fframe(k, std::false_type{});
      if (ok) {
        stamp(2);
        cluster_barrier();
        mid_done = true;
        if (!other_failed) {
          for (int q = 0; q < kRingAhead; ++q) issue_trellis(h + q);
          cp_async_commit();
          cp_async_wait<0>();
          __syncthreads();
          wl = wl2;
          wlo = wt2[warp];
          whi = wt2[warp + 1];
        }
        stamp(3);
        if (!other_failed)
          for (int k = h; k < T && ok; ++k) ok = fframe(k, std::true_type{});
        else
          for (int k = h; k < T && ok; ++k) ok = fframe(k, std::false_type{});
      }
      if (fail_at < 0) {
        const float t0 = lane_sum<kNW>(part + (T & 1) * 32, lane);
        float t2 = t0;
        if (lam > 0.f && t0 > 0.f) t2 = t0 + lam * t0;
        if (!(t2 >= a.floor_eff) || isinf(t2))
          fail_at = T - 1;
        else if (tid == 0)
          scales[T - 1] = t2;
        if (!other_failed) {  // frame T-1 (h <= T-1 always), then rows h..T-1
          if (flusher) flush_post(T - 1, xterm + ((T - 1) & 1) * X_pad);
          __syncthreads();
          normalize_rows(h, T);
        }
      }
      if (!mid_done) cluster_barrier();  // failed before the midpoint
      if (fail_at >= 0) {
        // remaining shifts are row maxima, remaining scales 1 (forward_backward.py:184,206)
        for (int k = fail_at + 1 + warp; k < T; k += kNW) {
          if (!pre) {
            float m = -INFINITY;
            for (int d = lane; d < D; d += 32) m = nan_max(m, Lb[size_t(k) * D + d]);
            m = warp_max(m);
            if (lane == 0) shifts[k] = m;
          }
        }
        for (int k = fail_at + tid; k < T; k += kNT) scales[k] = 1.f;
      }
      __syncthreads();
      {
        double acc = 0.0;
        for (int k = tid; k < T; k += kNT) {
          const double v = log(double(scales[k])) + double(pre ? Emb[k] : shifts[k]);
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
      stamp(4);
      cluster_barrier();  // end: the backward CTA's posterior rows are written
      stamp(5);
      if (fail_at >= 0 || other_failed) {
        const size_t n = size_t(T) * D;
        for (size_t i = tid; i < n; i += kNT) post_b[i] = 0.f;
      }
    } else {
      // ================= backward CTA ==================================================
      if (!other_failed) {
        for (int i = tid; i < 2 * RB; i += kNT) rbuf[i] = 0.f;
        __syncthreads();
        float dp = 0.f;
        for (int s = tid; s < S; s += kNT) {
          const float v = fin[s] * (1.f + lam);
          put_vec(rbuf + (T & 1) * RB, s, v);
          dp = fmaf(upi, v, dp);
        }
        dp = warp_sum(dp);
        if (lane == 0) part[(T & 1) * 32 + warp] = dp;
        for (int u = T + kRowAhead; u > T; --u) {
          if (u - 1 - kRowAhead < T) issue_row(u - 1 - kRowAhead);
          cp_async_commit();
        }
        cp_async_wait<0>();
        row_max_part(T - 1);
        row_max_part(T - 2);
        __syncthreads();
        compute_e(T - 1, false);
        __syncthreads();

        // iteration t: arcs of frame f = t-1; beta column "t" (raw) in rbuf[t & 1]
        auto bframe = [&](int t, auto postc) {
          constexpr bool POST = decltype(postc)::value;
          const int ct = t & 1, cpar = ct ^ 1;
          const int f = t - 1;
          const float t0 = lane_sum<kNW>(part + ct * 32, lane);  // mean of the raw column
          const float ld = (t < T && lam > 0.f) ? lam * t0 : 0.f;
          const float n = float(S) * t0;
          const float inv = (n > 0.f && !isinf(n)) ? rcp_fast(n) : 1.f;
          if constexpr (!POST) {  // beta'_f for the forward CTA's posteriors
            const float4 *r4 = reinterpret_cast<const float4 *>(rbuf + ct * RB);
            float4 *b4 = reinterpret_cast<float4 *>(trellis + size_t(f) * S_pad);
            for (int q = tid; q < (S_pad >> 2); q += kNT) {
              float4 v = r4[q];
              v.x = (v.x + ld) * inv;
              v.y = (v.y + ld) * inv;
              v.z = (v.z + ld) * inv;
              v.w = (v.w + ld) * inv;
              b4[q] = v;
            }
          }
          if (POST && t < h && flusher)  // frame t (posterior, previous iteration)
            flush_post(t, xterm + (t & 1) * X_pad);
          if (t - 2 >= 0) compute_e(t - 2, false);
          issue_row(t - 1 - kRowAhead);
          if (POST) issue_trellis(f - kRingAhead);
          cp_async_commit();
          {
            const uint32_t e32 = smem_u32(ebuf + cpar * EB), b32 = smem_u32(rbuf + ct * RB);
            float *bn = rbuf + cpar * RB;
            float dq = 0.f;
            for (int rr = wlo; rr < whi; ++rr) {
              const int tile = wl[rr];
              const unsigned info = tinfo[tile * 32 + lane];
              const int trips = ttrips[tile];
              const int base = tbase[tile] + lane;
              const int s = int(info & 0xFFFFu);
              float A;
              if constexpr (POST) {
                const float *al = ring + (f % kRing) * S_pad;  // alpha'_{f-1} = trellis row f
                const float as = s != 0xFFFF ? al[s] : 0.f;
                A = bwd_tile_f32(wp32 + uint32_t(base) * 8u, xs32 + uint32_t(base) * 2u, trips,
                                 e32, b32, smem_u32(xterm + (f & 1) * X_pad), ld, as);
              } else {
                A = bwd_plain_tile_f32(wp32 + uint32_t(base) * 8u, trips, e32, b32, ld);
              }
              if constexpr (kGrp) A = group_sum(A, G);
              if (s != 0xFFFF && (!kGrp || lead)) {
                const float v = inv * A;
                put_vec(bn, s, v);
                dq = fmaf(upi, v, dq);
              }
            }
            dq = warp_sum(dq);
            if (lane == 0) part[cpar * 32 + warp] = dq;
          }
          if constexpr (POST)
            cp_async_wait<kWait>();
          else
            cp_async_wait<kRowAhead - 2>();
          row_max_part(t - 3);
          __syncthreads();
        };
        stamp(1);
        for (int t = T; t > h; --t) bframe(t, std::false_type{});
        if (h >= 1) {  // first posterior frame h-1: the forward CTA's alpha rows are final
          stamp(2);
          cluster_barrier();
          mid_done = true;
          for (int q = 0; q < kRingAhead; ++q) issue_trellis(h - 1 - q);
          cp_async_commit();
          cp_async_wait<0>();
          __syncthreads();
          stamp(3);
          for (int t = h; t >= 1; --t) bframe(t, std::true_type{});
        }
        if (h >= 1) {
          if (flusher) flush_post(0, xterm);
          __syncthreads();
          normalize_rows(0, h);
        }
      }
      if (!mid_done) cluster_barrier();
      stamp(4);
      cluster_barrier();  // end
      stamp(5);
    }
  }
}

template <>
int launch_split<float>(const FBArgs<float> &a, const lfmmi_graphs *g, cudaStream_t st) {
  if (!g->tileable) return set_error(LFMMI_ERR_UNSUPPORTED, "split: graph not tileable");
  if (a.leak_pi) return set_error(LFMMI_ERR_UNSUPPORTED, "split: uniform leak only");
  if (a.mode != kPostWrite && a.mode != kPostNegate)
    return set_error(LFMMI_ERR_UNSUPPORTED, "split: WRITE / NEGATE modes only");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const Options &opt = options();
  if (opt.split == 0) return set_error(LFMMI_ERR_UNSUPPORTED, "split: disabled");
  if (opt.split != 1 && a.B > 2 * sms)
    return set_error(LFMMI_ERR_UNSUPPORTED, "split: batch fills the SMs");
  const int Fmax = std::max(g->max_tf_slots, g->max_tb_slots);
  const int X_pad = pad4(std::max(4, g->max_xpad));
  const int RB = pad4(a.rep_r * a.r_stride), EB = a.rep_e * a.e_stride;
  FBArgs<float> b = a;
  b.sc_smem = 1;
  SplitLayout lay = split_layout(Fmax, g->max_tiles, a.D, X_pad, a.S_pad, a.D_pad, a.T_pad, RB,
                                 EB, true);
  if (lay.total > size_t(kMaxSmem)) {
    b.sc_smem = 0;
    lay = split_layout(Fmax, g->max_tiles, a.D, X_pad, a.S_pad, a.D_pad, a.T_pad, RB, EB, false);
  }
  if (opt.debug)
    std::fprintf(stderr, "[lfmmi] split layout %zu B (limit %d)\n", lay.total, kMaxSmem);
  // scheduling scratch (lengths + order) lives in the posterior slot buffers
  if (lay.total > size_t(kMaxSmem) || size_t(2) * a.B * 4 > size_t(2) * X_pad * 4)
    return set_error(LFMMI_ERR_UNSUPPORTED,
                     "split kernel needs " + std::to_string(lay.total) + " B shared memory");
  // Clusters: one per utterance while they fit, leaving 6 SMs to the numerator
  // pass that runs beside this one (the linear-chain kernel: 0.43 ms alone,
  // hidden behind the ~1.06 ms denominator; WSJ-mono step 1.111 / 1.101 / 1.088
  // / 1.083 / 1.082 / 1.082 ms with 66 / 68 / 69 / 70 / 71 / 72 clusters, 1.19 ms
  // with 74 — numerators then wait for free SMs); beyond that LPT pairs long
  // with short utterances.  Option split_clusters overrides.
  const int reserve = a.reserve_sms > 0 ? a.reserve_sms : 6;
  const int cap = std::min(kMaxClusters, sms / 2);
  int nc = opt.split_clusters > 0 ? opt.split_clusters : std::min(a.B, (sms - reserve) / 2);
  nc = std::max(1, std::min(nc, cap));
  nc = std::max(nc, (a.B + kMaxItems - 1) / kMaxItems);
  if (nc > cap) return set_error(LFMMI_ERR_UNSUPPORTED, "split: too many utterances per cluster");
  const bool grp = g->max_tile_g > 1;
  auto kern = grp ? fb_split_kernel<true> : fb_split_kernel<false>;
  static bool configured[2] = {false, false};
  if (!configured[grp]) {
    int rc = check_cuda(
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem),
        "cudaFuncSetAttribute(split)");
    if (rc) return rc;
    configured[grp] = true;
  }
  const int hnum = std::max(0, std::min(64, opt.split_h64));  // midpoint in 64ths of T
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
  if (opt.debug) {
    int maxc = -1;
    cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg);
    std::fprintf(stderr, "[lfmmi] split: %d clusters (max active %d), smem %zu (scales %s)\n", nc,
                 maxc, lay.total, b.sc_smem ? "smem" : "hbm");
  }
  note_den_kernel("fb_split_kernel (2-CTA cluster: forward | backward)");
  if (opt.profile != "split")
    return check_cuda(cudaLaunchKernelEx(&cfg, kern, b, Fmax, g->max_tiles, X_pad, nc, hnum),
                      "fb_split_kernel launch");
  // Debug: per-item section timestamps of both CTAs, summarised on stderr.
  const size_t n = size_t(2 * nc) * kMaxItems * 8;
  long long *d = nullptr;
  int rc = check_cuda(cudaMalloc(&d, n * sizeof(long long)), "cudaMalloc(split prof)");
  if (rc) return rc;
  cudaMemsetAsync(d, 0, n * sizeof(long long), st);
  b.prof = d;
  rc = check_cuda(cudaLaunchKernelEx(&cfg, kern, b, Fmax, g->max_tiles, X_pad, nc, hnum),
                  "fb_split_kernel launch");
  std::vector<long long> hp(n);
  cudaStreamSynchronize(st);
  cudaMemcpy(hp.data(), d, n * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  double acc[2][6] = {}, fr[2][2] = {};
  long long span[2] = {0, 0};
  for (int blk = 0; blk < 2 * nc; ++blk) {
    const int r = blk & 1;
    long long first = 0, lastt = 0;
    for (int i = 0; i < kMaxItems; ++i) {
      const long long *p = &hp[(size_t(blk) * kMaxItems + i) * 8];
      if (p[5] == 0) continue;
      if (!first) first = p[0];
      lastt = p[5];
      const long long T = p[6], h = p[7];
      for (int j = 0; j < 5; ++j) acc[r][j] += double(p[j + 1] - p[j]);
      fr[r][0] += double(r == 0 ? h : T - h);
      fr[r][1] += double(r == 0 ? T - h : h);
    }
    span[r] = std::max(span[r], lastt - first);
  }
  for (int r = 0; r < 2; ++r)
    std::fprintf(stderr,
                 "[lfmmi split prof] %s: prologue %.0f  first half %.0f/frame  mid wait %.0f  "
                 "second half %.0f/frame  end wait %.0f (cycles, totals over items: %.0f / %.0f "
                 "frames)  max CTA span %lld\n",
                 r ? "backward" : "forward ", acc[r][0] / (nc), acc[r][1] / fr[r][0],
                 acc[r][2] / nc, acc[r][3] / fr[r][1], acc[r][4] / nc, fr[r][0], fr[r][1],
                 span[r]);
  return rc;
}

template <>
int launch_split<double>(const FBArgs<double> &, const lfmmi_graphs *, cudaStream_t) {
  return set_error(LFMMI_ERR_UNSUPPORTED, "split kernel is fp32-only");
}

}  // namespace lfmmi
