// Tile kernels: the LF-MMI hot path for both graph classes.
//
//   fb_tile_kernel<Real, 512, 1, true, .>  — denominator: one 512-thread CTA
//       per utterance; the arc layout of the current phase is resident in
//       shared memory (CSR-by-destination for the forward, CSR-by-source for
//       the backward).
//   fb_tile_kernel<Real, 32, IPC, ., .> — numerators: one warp per
//       utterance (IPC utterances per CTA, __syncwarp only); the tiny
//       per-utterance arc packs are read through L1.
//
// Layout: states sorted by degree into 32-lane tiles; tile w stores slot j of
// lane l at base_w + 32 j + l, so every arc-data load is one coalesced
// 256-byte row (word | fp32 prob interleaved) and the only random accesses
// are the alpha/beta and emission gathers.  Padded slots carry probability 0
// (and a dummy posterior slot), so the inner loops are branch-free.  Each
// warp owns whole tiles: a state's sum is accumulated by one thread in CSR
// order — deterministic, no atomics.
//
// Whole time loop on chip, one group barrier per frame:
//   forward  (_kernels.py:54-122): deferred normalisation — column k+1 is
//     gathered from the unnormalised column k and the normaliser / leaky-HMM
//     correction of column k is applied inside the gather;
//   backward (_kernels.py:125-191): same deferral for the leak adjoint;
//   posterior + gradient (_kernels.py:194-224, loss.py:67-69): the backward
//     pass already forms every arc term p * e[pdf] * beta_t[dst]; it stores
//     alpha_{t-1}[src] * term into an owned per-arc slot grouped by pdf, and
//     the next frame sums each pdf's slots (float4 loads) into the gradient.
// Emissions exp(L - max_d L) (forward_backward.py:120-130) are computed on
// the fly from log-likelihood rows staged by cp.async two frames ahead; the
// alpha column of every frame is spilled to an HBM workspace and streamed
// back during the backward.
#include "lfmmi_device.cuh"
#include "lfmmi_kernels.h"
#include "lfmmi_lpt.cuh"
#include "lfmmi_options.h"
#include "lfmmi_tile_common.cuh"
#include "lfmmi_schedule.h"

#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

namespace lfmmi {

// cp.async pipelines, one commit group per frame: log-likelihood rows are
// issued kTileRowAhead frames before their row maximum is taken, alpha rows
// (backward) kTileAlphaAhead frames before use (3-slot ring, indexed mod 3), so
// a short frame (numerators) never waits on HBM latency.
constexpr int kTileRowAhead = 4, kTileStageRing = 8;
constexpr int kTileAlphaAhead = 2, kTileAlphaRing = 3;
constexpr int kTileFwdWait = kTileRowAhead - 2;   // row k+2 complete at the end of frame k
constexpr int kTileBwdWait = kTileAlphaAhead - 1; // alpha t-2 / row t-3 at the end of frame t
static_assert(kTileBwdWait <= kTileRowAhead - 2, "row pipeline must be at least as deep");

// Numerator-sized CTAs (<= 128 threads): registers capped (<= 72) so that 7
// utterances share an SM — the numerator pass runs on the 20 SMs the split
// denominator leaves free, and 128 numerators must be resident at once (at 75
// registers only 6 fit: the pass grew from 1.04 to ~1.13 ms).
#ifndef LFMMI_NUM_MIN_BLOCKS
#define LFMMI_NUM_MIN_BLOCKS 7
#endif
constexpr int kNumMinBlocks = LFMMI_NUM_MIN_BLOCKS;

struct TileLayout {  // byte offsets of one utterance's slice of shared memory
  size_t wp, xs, tinfo, ttrips, tbase, wlist, wtab, pdfptr, xterm, rbuf, aring, ebuf, stage,
      gstage, scales, shifts, part, mpart, items, total;
};

__host__ __device__ inline TileLayout tile_layout(bool smem_graph, int Fmax, int ntiles, int D,
                                                  int X_pad, int S_pad, int D_pad, int T_pad,
                                                  int RB, int EB, int real, int nx = 1,
                                                  bool smem_scales = true) {
  TileLayout l;
  size_t o = 512;  // scratch: 32 doubles + 32 int64
  const size_t F = smem_graph ? size_t(Fmax) : 0;
  const size_t nt = smem_graph ? size_t(ntiles) : 0;
  l.wp = o;      o = al16(o + (real == 4 ? F * 8 : al16(F * 4) + F * 8));
  l.xs = o;      o = al16(o + F * 2);
  l.tinfo = o;   o = al16(o + nt * 32 * 4);
  l.ttrips = o;  o = al16(o + size_t(pad4(int(nt))) * 4);
  l.tbase = o;   o = al16(o + size_t(pad4(int(nt))) * 4);
  l.wlist = o;   o = al16(o + (nx > 1 ? size_t(pad4(int(nt))) * 4 + kWarpTable * 4 : 0));
  l.wtab = l.wlist + (nx > 1 ? size_t(pad4(int(nt))) * 4 : 0);
  l.pdfptr = o;  o = al16(o + size_t(D + 1) * 4);
  l.xterm = o;   o = al16(o + size_t(nx) * X_pad * real); // posterior slots (nx frames)
  l.rbuf = o;    o = al16(o + size_t(2) * RB * real);     // alpha/beta columns x copies
  l.aring = o;   o = al16(o + size_t(kTileAlphaRing) * S_pad * real);
  l.ebuf = o;    o = al16(o + size_t(2) * EB * real);     // emission rows x copies
  l.stage = o;   o = al16(o + size_t(kTileStageRing) * D_pad * real);
  l.gstage = o;  o = al16(o + size_t(2) * D_pad * real);
  // per-frame scales / row maxima: shared memory when they fit (smem_scales),
  // else the HBM workspace (ragged, like the trellis)
  l.scales = o;  o = al16(o + (smem_scales ? size_t(T_pad) * real : 0));
  l.shifts = o;  o = al16(o + (smem_scales ? size_t(T_pad) * real : 0));
  l.part = o;    o = al16(o + size_t(2) * 32 * real);
  l.mpart = o;   o = al16(o + size_t(2) * 32 * real);
  l.items = o;   o = al16(o + (nx > 1 ? size_t(kLptMaxItems + 4) * 4 : 0));  // persistent: LPT list
  l.total = o;
  return l;
}

template <int GROUP, int IPC>
__device__ __forceinline__ void tsync() {
  if constexpr (GROUP == 32) {
    __syncwarp();
  } else {
    static_assert(IPC == 1, "CTA-sized groups run one utterance per CTA");
    __syncthreads();
  }
}

// XDB (denominator, fp32, when shared memory allows): two posterior slot
// buffers, so the gradient row of frame t is flushed by the top warps at the
// start of the next backward iteration — overlapped with the other warps' arc
// work — instead of between two extra barriers; tiles then follow the host's
// LPT warp lists, which give the flushing warps fewer arcs.
template <typename Real, int GROUP, int IPC, bool SMEM_GRAPH, bool CUSTOM_PI, bool XDB = false>
__global__ void __launch_bounds__(GROUP *IPC, GROUP *IPC <= 128 ? kNumMinBlocks : 1)
    fb_tile_kernel(const FBArgs<Real> a, int Fmax, int ntiles_max, int X_pad) {
  static_assert(!XDB || (GROUP == 32 * kTableNW && IPC == 1 && SMEM_GRAPH),
                "XDB uses the 16-warp LPT lists");
  constexpr int NW = GROUP / 32;
  using Slot = typename SlotOf<Real>::type;
  extern __shared__ __align__(16) unsigned char smem_all[];
  const int gid = threadIdx.x / GROUP;
  const int tid = threadIdx.x % GROUP, lane = tid & 31, warp = tid >> 5;
  // Per-frame chores (emission rows, prefetch, posterior flush) run on the
  // *last* warps, which the snake tile order gives the lightest arc tiles.
  const int ctid = GROUP - 1 - tid, cwarp = ctid >> 5;
  const int ntile_rounds_max = (ntiles_max + NW - 1) / NW;
  (void)ntile_rounds_max;
  const int RB = pad4(a.rep_r * a.r_stride), EB = a.rep_e * a.e_stride;  // 16-byte buffers
  const TileLayout lay = tile_layout(SMEM_GRAPH, Fmax, ntiles_max, a.D, X_pad, a.S_pad, a.D_pad,
                                     a.T_pad, RB, EB, int(sizeof(Real)), XDB ? 2 : 1,
                                     a.sc_smem != 0);
  unsigned char *smem = smem_all + lay.total * gid;
  double *dscr = reinterpret_cast<double *>(smem);
  long long *lscr = reinterpret_cast<long long *>(smem + 256);
  int *pdfptr = reinterpret_cast<int *>(smem + lay.pdfptr);
  Real *xterm = reinterpret_cast<Real *>(smem + lay.xterm);
  Real *rbuf = reinterpret_cast<Real *>(smem + lay.rbuf);
  Real *aring = reinterpret_cast<Real *>(smem + lay.aring);
  Real *ebuf = reinterpret_cast<Real *>(smem + lay.ebuf);
  Real *stage = reinterpret_cast<Real *>(smem + lay.stage);
  Real *gstage = reinterpret_cast<Real *>(smem + lay.gstage);
  Real *scales = nullptr, *shifts = nullptr;  // set once item_off is known
  Real *part = reinterpret_cast<Real *>(smem + lay.part);
  Real *mpart = reinterpret_cast<Real *>(smem + lay.mpart);
  auto gsync = [] { tsync<GROUP, IPC>(); };
  // fp32 + shared-memory arc pack: explicitly scheduled loops on byte-offset words.
  constexpr bool FAST = std::is_same<Real, float>::value && SMEM_GRAPH && !CUSTOM_PI;
  const uint32_t wp32 = smem_u32(smem + lay.wp), xs32 = smem_u32(smem + lay.xs);
  (void)wp32;
  (void)xs32;

  // One utterance (index b) of this group.
  auto run_item = [&](const int b) {
    const int T = item_frames(a.lengths, b, a.T_max);
    if (T <= 0) {  // zero-length item (host APIs reject it): failed, no frames touched
      if (a.mode != kPostAdd && a.mode != kPostSubtract && !a.packed)
        for (size_t i = tid; i < size_t(a.T_max) * a.D; i += GROUP)
          a.post[size_t(b) * a.T_max * a.D + i] = Real(0);
      if (tid == 0) {
        a.logp[b] = NAN;
        a.fail[b] = 0;
      }
      return;
    }
    const int D = a.D;
    const int S_pad = a.S_pad, D_pad = a.D_pad;
    const int row = int(a.row_map[b]);
    const int *desc = a.g.desc + row * kDescInts;
    const int S = desc[kS], init = desc[kInit];
    const int ntiles = desc[kNTiles];
    const int G = desc[kTileG];  // lanes per state: partial sums over G adjacent lanes
    const bool lead = (lane & (G - 1)) == 0;
    const int toff = desc[kTileOff];
    const Real *fin = pick<Real>(a.g.fin32, a.g.fin64) + desc[kStateOff];
    const Real *Lb = a.L + size_t(b) * a.T_max * D;
    Real *post_b = a.post + size_t(b) * a.T_max * D;
    const int mode = a.mode;
    const bool reads_post = mode == kPostAdd || mode == kPostSubtract;
    const bool other_failed = a.other_fail != nullptr && a.other_fail[b] >= 0;
    const int nrw = (D + 31) / 32 < NW ? (D + 31) / 32 : NW;  // chore warps holding row elements
    const int nrounds = (ntiles + NW - 1) / NW;
    // Snake order: round r gives warp w tile r*NW + w (r even) or r*NW + NW-1-w
    // (r odd), pairing heavy and light tiles (tiles are sorted by degree).
    auto tile_of = [&](int r) { return r * NW + ((r & 1) ? NW - 1 - warp : warp); };
    // XDB: this warp's tiles are wl[wlo..whi) (host LPT lists, staged per phase).
    const int *wl = reinterpret_cast<const int *>(smem + lay.wlist);
    const int *wt = reinterpret_cast<const int *>(smem + lay.wtab);
    int wlo = 0, whi = nrounds;
    auto read_warps = [&] {
      if constexpr (XDB) {
        wlo = wt[warp];
        whi = wt[warp + 1];
      }
    };
    auto tile_at = [&](int i) { return XDB ? wl[i] : tile_of(i); };

    // Arc-pack views of the current phase: shared memory (denominator) or L1 (numerators).
    const unsigned *tinfo;
    const int *ttrips, *tbase;
    Slot slot;
    const unsigned short *XS;
    auto bind_phase = [&](bool fwd) {
      const int so = desc[fwd ? kTfSlotOff : kTbSlotOff], nsl = desc[fwd ? kTfSlots : kTbSlots];
      const uint2 *gwp = (fwd ? a.g.tf_wp : a.g.tb_wp) + so;
      const unsigned *gw = (fwd ? a.g.tf_word : a.g.tb_word) + so;
      const double *gp = (fwd ? a.g.tf_p64 : a.g.tb_p64) + so;
      const unsigned *gi = (fwd ? a.g.tf_info : a.g.tb_info) + size_t(toff) * 32;
      const int *gt = (fwd ? a.g.tf_trips : a.g.tb_trips) + toff;
      const int *gb = (fwd ? a.g.tf_base : a.g.tb_base) + toff;
      const unsigned short *gx = a.g.tb_xslot + so;
      if constexpr (SMEM_GRAPH) {
        unsigned char *wpb = smem + lay.wp;
        if constexpr (sizeof(Real) == 4) {
          copy16<GROUP>(wpb, gwp, size_t(nsl) * 8, tid);
          slot.wp = reinterpret_cast<const uint2 *>(wpb);
        } else {
          unsigned *w = reinterpret_cast<unsigned *>(wpb);
          double *p = reinterpret_cast<double *>(wpb + al16(size_t(Fmax) * 4));
          copy16<GROUP>(w, gw, size_t(nsl) * 4, tid);
          copy16<GROUP>(p, gp, size_t(nsl) * 8, tid);
          slot.w = w;
          slot.p = p;
        }
        unsigned short *xs = reinterpret_cast<unsigned short *>(smem + lay.xs);
        if (!fwd) copy16<GROUP>(xs, gx, size_t(nsl) * 2, tid);
        XS = xs;
        unsigned *ti = reinterpret_cast<unsigned *>(smem + lay.tinfo);
        int *tt = reinterpret_cast<int *>(smem + lay.ttrips);
        int *tb = reinterpret_cast<int *>(smem + lay.tbase);
        copy16<GROUP>(ti, gi, size_t(ntiles) * 128, tid);
        copy16<GROUP>(tt, gt, size_t(pad4(ntiles)) * 4, tid);
        copy16<GROUP>(tb, gb, size_t(pad4(ntiles)) * 4, tid);
        if constexpr (XDB) {
          copy16<GROUP>(smem + lay.wlist, (fwd ? a.g.tf_wlist : a.g.tb_wlist) + toff,
                        size_t(pad4(ntiles)) * 4, tid);
          copy16<GROUP>(smem + lay.wtab, (fwd ? a.g.tf_wtab : a.g.tb_wtab) + desc[kWTabOff],
                        size_t(kWarpTable) * 4, tid);
        }
        tinfo = ti;
        ttrips = tt;
        tbase = tb;
      } else {
        if constexpr (sizeof(Real) == 4) {
          slot.wp = gwp;
        } else {
          slot.w = gw;
          slot.p = gp;
        }
        XS = gx;
        tinfo = gi;
        ttrips = gt;
        tbase = gb;
      }
    };
    bind_phase(true);

    long long off = 0;
    for (int j = tid; j < b; j += GROUP) off += a.lengths[j];
    off = warp_sum(off);
    const Real *pi = CUSTOM_PI ? a.leak_pi + size_t(row) * a.S_max : nullptr;
    double psum_d = 0.0;
    if (pi)
      for (int s = tid; s < S; s += GROUP) psum_d += double(pi[s]);
    psum_d = warp_sum(psum_d);
    if (lane == 0) {
      lscr[warp] = off;
      dscr[warp] = psum_d;
    }
    gsync();
    long long item_off = 0;
    double pisum_d = 0.0;
    for (int w = 0; w < NW; ++w) {
      item_off += lscr[w];
      pisum_d += dscr[w];
    }
    const Real upi = Real(1.0 / double(S));
    const Real pisum = pi ? Real(pisum_d) : Real(1);
    const Real lam = a.leak;
    Real *trellis = a.work + item_off * S_pad;
    if (a.sc_smem) {
      scales = reinterpret_cast<Real *>(smem + lay.scales);
      shifts = reinterpret_cast<Real *>(smem + lay.shifts);
    } else {
      scales = a.work + a.sc_off + item_off;
      shifts = scales + a.sc_total;
    }
    if (a.packed) {  // ragged layout: item b's rows start at sum_{j<b} T_j
      Lb = a.L + size_t(item_off) * D;
      post_b = a.post + size_t(item_off) * D;
    }

    if (!reads_post && !a.packed) {
      const size_t n = size_t(a.T_max - T) * D;
      for (size_t i = tid; i < n; i += GROUP) post_b[size_t(T) * D + i] = Real(0);
    }

    auto issue_row = [&](int t) {
      if (t < 0 || t >= T || cwarp >= nrw) return;
      const Real *src = Lb + size_t(t) * D;
      Real *dst = stage + (t & (kTileStageRing - 1)) * D_pad;
      for (int d = ctid; d < D; d += GROUP) cp_async_elem(dst + d, src + d);
    };
    auto row_max_part = [&](int t) {
      if (t < 0 || t >= T || cwarp >= nrw) return;
      const Real *src = stage + (t & (kTileStageRing - 1)) * D_pad;
      Real m = -INFINITY;
      for (int d = ctid; d < D; d += GROUP) m = nan_max(m, src[d]);
      m = warp_max(m);
      if (lane == 0) mpart[(t & 1) * 32 + cwarp] = m;
    };
    auto compute_e = [&](int t, bool record_shift) {
      if (cwarp >= nrw) return;
      const Real *mp = mpart + (t & 1) * 32;
      Real m;
      if constexpr (NW == 1) {
        m = mp[0];
      } else {
        m = lane < nrw ? mp[lane] : Real(-INFINITY);
        m = warp_max(m);
      }
      const Real *src = stage + (t & (kTileStageRing - 1)) * D_pad;
      Real *dst = ebuf + (t & 1) * EB;
      for (int d = ctid; d < D; d += GROUP) {
        const Real v = exp_r(src[d] - m);
        for (int c = 0; c < a.rep_e; ++c) dst[c * a.e_stride + d] = v;
      }
      if (record_shift && ctid == 0) shifts[t] = m;
    };

    // alpha/beta columns are replicated (rep_r copies, see lfmmi_schedule.cpp)
    // (rep_r is 1 or 2, make_gather_layout; hoisted so no per-store param reloads)
    const bool rep2 = a.rep_r > 1;
    const int rstride = a.r_stride;
    auto put_vec = [&](Real *v, int s, Real x) {
      v[s] = x;
      if (rep2) v[rstride + s] = x;
    };
    // ---- prologue -----------------------------------------------------------------
    for (int i = tid; i < 2 * RB; i += GROUP) rbuf[i] = Real(0);  // padding lanes stay 0
    gsync();
    for (int s = tid; s < S; s += GROUP) put_vec(rbuf, s, (s == init) ? Real(1) : Real(0));
    for (int j = 0; j < kTileRowAhead; ++j) {  // group j holds row j (+ the staged packs in 0)
      issue_row(j);
      cp_async_commit();
    }
    cp_async_wait<kTileFwdWait>();
    row_max_part(0);
    row_max_part(1);
    gsync();
    compute_e(0, true);
    gsync();
    read_warps();

    // debug section timestamps (LFMMI_PROFILE_TILE): fwd start/end, bwd start/end
    auto stamp = [&](int j) {
      if (a.prof != nullptr && tid == 0) {
        a.prof[size_t(b) * 8 + j] = clock64();
        a.prof[size_t(b) * 8 + 6] = T;
      }
    };
    stamp(0);
    // ---- forward: one barrier per frame ------------------------------------------------
    Real inv2 = Real(1), leakc = Real(0);
    int fail_at = -1;
    for (int k = 0; k < T; ++k) {
      const int cur = k & 1, nxt = cur ^ 1;
      if (k > 0) {
        const Real t0 = lane_sum<NW>(part + cur * 32, lane);
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
        inv2 = rcp_rn(t2);
        if (tid == 0) scales[k - 1] = t2;
      }
      {
        const Real *r = rbuf + cur * RB;
        Real *arow = trellis + size_t(k) * S_pad;
        if constexpr (CUSTOM_PI) {
          for (int s = tid; s < S; s += GROUP) arow[s] = (r[s] + leakc * pi[s]) * inv2;
        } else if constexpr (FAST) {  // float4: S_pad and both row bases are 16-byte multiples
          const float4 *r4 = reinterpret_cast<const float4 *>(r);
          float4 *a4 = reinterpret_cast<float4 *>(arow);
          const float lu = leakc * upi;
          for (int q = tid; q < (S_pad >> 2); q += GROUP) {
            float4 v = r4[q];
            v.x = (v.x + lu) * inv2;
            v.y = (v.y + lu) * inv2;
            v.z = (v.z + lu) * inv2;
            v.w = (v.w + lu) * inv2;
            a4[q] = v;
          }
        } else {
          const Real lu = leakc * upi;
          for (int s = tid; s < S; s += GROUP) arow[s] = (r[s] + lu) * inv2;
        }
      }
      if (k + 1 < T) compute_e(k + 1, true);
      issue_row(k + kTileRowAhead);
      cp_async_commit();
      {
        const Real *e = ebuf + cur * EB;
        const Real *r = rbuf + cur * RB;
        Real *rn = rbuf + nxt * RB;
        const bool last = (k + 1 == T);
        const uint32_t e32 = smem_u32(e), r32 = smem_u32(r);
        (void)e32;
        (void)r32;
        Real psum = Real(0);
        // G lanes per state (kTileG) only for small graphs: the partial-sum
        // shuffles and the group-leader test compiled out of the G = 1 loop
        auto tiles = [&](auto grp) {
          constexpr bool GRP = decltype(grp)::value;
          for (int rr = wlo; rr < whi; ++rr) {
            const int tile = tile_at(rr);
            if (!XDB && tile >= ntiles) continue;
            const unsigned info = tinfo[tile * 32 + lane];
            const int trips = ttrips[tile];
            const int base = tbase[tile] + lane;
            Real A = Real(0), Bs = Real(0);
            if constexpr (FAST) {
              const uint32_t sb = wp32 + uint32_t(base) * 8u;
              if (leakc != Real(0))
                fwd_tile_f32<true>(sb, trips, e32, r32, A, Bs);
              else
                fwd_tile_f32<false>(sb, trips, e32, r32, A, Bs);
            } else if (leakc != Real(0)) {
    #pragma unroll 4
              for (int j = 0; j < trips; ++j) {
                unsigned wd;
                Real p;
                slot.load(base + 32 * j, wd, p);
                const Real w = p * e[wd >> 16];
                const int src = int(wd & 0xFFFFu);
                A = fma(w, r[src], A);
                if constexpr (CUSTOM_PI)  // gather index may name copy 1 (rep_r <= 2)
                  Bs = fma(w, pi[src >= a.r_stride ? src - a.r_stride : src], Bs);
                else
                  Bs += w;
              }
            } else {
    #pragma unroll 4
              for (int j = 0; j < trips; ++j) {
                unsigned wd;
                Real p;
                slot.load(base + 32 * j, wd, p);
                A = fma(p * e[wd >> 16], r[wd & 0xFFFFu], A);
              }
            }
            const int s = int(info & 0xFFFFu);
            if constexpr (GRP) {
              A = group_sum(A, G);
              Bs = group_sum(Bs, G);
            }
            if (s != 0xFFFF && (!GRP || lead)) {
              Real raw = inv2 * (A + leakc * (CUSTOM_PI ? Bs : upi * Bs));
              if (last) raw *= fin[s];
              put_vec(rn, s, raw);
              psum += raw;
            }
          }
        };
        if (G > 1)
          tiles(std::true_type{});
        else
          tiles(std::false_type{});
        psum = warp_sum(psum);
        if (lane == 0) part[nxt * 32 + warp] = psum;
      }
      cp_async_wait<kTileFwdWait>();  // row k + 2
      row_max_part(k + 2);
      gsync();
    }
    stamp(1);
    if (fail_at < 0) {
      const Real t0 = lane_sum<NW>(part + (T & 1) * 32, lane);
      Real t2 = t0;
      if (lam > Real(0) && t0 > Real(0)) t2 = t0 + lam * t0 * pisum;
      if (!(t2 >= a.floor_eff) || isinf(t2))
        fail_at = T - 1;
      else if (tid == 0)
        scales[T - 1] = t2;
    }
    if (fail_at >= 0) {
      // The reference exponentiates every valid frame: remaining shifts are row
      // maxima, remaining scales stay 1 (forward_backward.py:184,206).
      for (int k = fail_at + 1 + warp; k < T; k += NW) {
        Real m = -INFINITY;
        for (int d = lane; d < D; d += 32) m = nan_max(m, Lb[size_t(k) * D + d]);
        m = warp_max(m);
        if (lane == 0) shifts[k] = m;
      }
      for (int k = fail_at + tid; k < T; k += GROUP) scales[k] = Real(1);
    }
    gsync();
    {
      double acc = 0.0;
      for (int k = tid; k < T; k += GROUP) {
        const double v = log(double(scales[k])) + double(shifts[k]);
        acc += v;
        if (a.scale_logs) a.scale_logs[size_t(b) * a.T_max + k] = v;
      }
      if (a.scale_logs)
        for (int k = T + tid; k < a.T_max; k += GROUP) a.scale_logs[size_t(b) * a.T_max + k] = 0.0;
      acc = warp_sum(acc);
      if (lane == 0) dscr[warp] = acc;
      gsync();
      if (tid == 0) {
        double tot = 0.0;
        for (int w = 0; w < NW; ++w) tot += dscr[w];
        a.logp[b] = fail_at >= 0 ? NAN : tot;
        a.fail[b] = fail_at;
      }
    }
    if (fail_at >= 0 || other_failed) {
      const size_t n = size_t(T) * D;
      for (size_t i = tid; i < n; i += GROUP) post_b[i] = Real(0);
      return;
    }

    // ---- backward + fused posterior / gradient ---------------------------------------
    bind_phase(false);
    {
      const int *pp = a.g.pdf_arc_ptr + desc[kPdfPtrOff2];
      for (int d = tid; d <= D; d += GROUP) pdfptr[d] = pp[d];
      // Padding slots of the per-pdf groups are never written: zero them once.
      for (int i = tid; i < (XDB ? 2 : 1) * X_pad; i += GROUP) xterm[i] = Real(0);
    }
    auto issue_alpha = [&](int k) {
      if (k < 0) return;
      copy16<GROUP>(aring + (k % kTileAlphaRing) * S_pad, trellis + size_t(k) * S_pad,
                    size_t(S_pad) * sizeof(Real), ctid);
    };
    auto issue_post = [&](int t) {
      if (!reads_post || t < 0 || t >= T) return;
      const Real *src = post_b + size_t(t) * D;
      Real *dst = gstage + (t & 1) * D_pad;
      for (int d = ctid; d < D; d += GROUP) cp_async_elem(dst + d, src + d);
    };
    // gamma_t[d] = sum of pdf d's slots: SPL chore lanes per pdf, each summing
    // float4 groups, combined by a shuffle within the SPL-lane segment.
    int spl = 1, spl_log = 0;  // lanes per pdf in the flush (power of two)
    while (spl < 32 && D * spl * 2 <= GROUP) {
      spl <<= 1;
      ++spl_log;
    }
    auto flush_post = [&](int t, const Real *xsrc) {
      Real *prow = post_b + size_t(t) * D;
      const Real *old = gstage + (t & 1) * D_pad;
      const int sub = ctid & (spl - 1);
      for (int base_i = 0; base_i < D * spl; base_i += GROUP) {
        const int idx = base_i + ctid;
        const int d = idx >> spl_log;
        Real g = Real(0);
        if (d < D) {
          const int lo = pdfptr[d] >> 2, hi = pdfptr[d + 1] >> 2;
          for (int q = lo + sub; q < hi; q += spl) g += sum_groups4(xsrc + 4 * q, 1);
        }
        for (int o = 1; o < spl; o <<= 1) g += __shfl_xor_sync(kFull, g, o);
        if (d < D && sub == 0) {
          switch (mode) {
            case kPostNegate: prow[d] = -g; break;
            case kPostAdd: prow[d] = old[d] + g; break;
            case kPostSubtract: prow[d] = old[d] - g; break;
            default: prow[d] = g;
          }
        }
      }
    };

    for (int s = tid; s < S; s += GROUP) put_vec(rbuf + (T & 1) * RB, s, fin[s] * (Real(1) + lam));
    // Backward pipeline: "iteration" u issues row u-1-kTileRowAhead, alpha
    // u-1-kTileAlphaAhead (and, ADD/SUBTRACT modes, gradient row u-1); the virtual
    // iterations T+kTileRowAhead .. T+1 fill it, one group each.
    for (int u = T + kTileRowAhead; u > T; --u) {
      if (u - 1 - kTileRowAhead < T) issue_row(u - 1 - kTileRowAhead);
      if (u - 1 - kTileAlphaAhead < T) issue_alpha(u - 1 - kTileAlphaAhead);
      if (u - 1 < T) issue_post(u - 1);
      cp_async_commit();
    }
    cp_async_wait<0>();
    row_max_part(T - 1);
    row_max_part(T - 2);
    gsync();
    compute_e(T - 1, false);
    gsync();
    read_warps();

    const bool flusher = cwarp * 32 < D * spl;
    Real sc_cur = scales[T - 1];
    stamp(2);
    for (int t = T; t >= 1; --t) {
      const int ct = t & 1, cp = ct ^ 1;
      Real ld = Real(0);
      if (t < T && lam > Real(0)) ld = lam * lane_sum<NW>(part + ct * 32, lane);
      // scales[t-1] was read one iteration ahead (global, off the critical path)
      const Real inv = rcp_rn(sc_cur);
      sc_cur = t >= 2 ? scales[t - 2] : Real(1);
      // XDB: slots of frame t-1 go to buffer (t & 1); flush frame t (the other one) now.
      const int xb = XDB ? ct : 0;
      if (XDB && t < T && flusher) flush_post(t, xterm + (xb ^ 1) * X_pad);
      if (t - 2 >= 0) compute_e(t - 2, false);
      issue_row(t - 1 - kTileRowAhead);
      issue_alpha(t - 1 - kTileAlphaAhead);
      issue_post(t - 1);
      cp_async_commit();
      {
        const Real *bt = rbuf + ct * RB;
        const Real *e = ebuf + cp * EB;
        const Real *al = aring + ((t - 1) % kTileAlphaRing) * S_pad;  // alpha_{t-1}
        Real *bn = rbuf + cp * RB;
        Real *xt = xterm + xb * X_pad;
        Real dp = Real(0);
        // G lanes per state (kTileG) only for small graphs: the partial-sum
        // shuffles and the group-leader test compiled out of the G = 1 loop
        auto tiles = [&](auto grp) {
          constexpr bool GRP = decltype(grp)::value;
          for (int rr = wlo; rr < whi; ++rr) {
            const int tile = tile_at(rr);
            if (!XDB && tile >= ntiles) continue;
            const unsigned info = tinfo[tile * 32 + lane];
            const int trips = ttrips[tile];
            const int base = tbase[tile] + lane;
            const int s = int(info & 0xFFFFu);
            const Real as = (s != 0xFFFF) ? al[s] * inv : Real(0);
            Real A = Real(0);
            if constexpr (FAST) {
              A = bwd_tile_f32(wp32 + uint32_t(base) * 8u, xs32 + uint32_t(base) * 2u, trips,
                               smem_u32(e), smem_u32(bt), smem_u32(xt), ld, as);
            } else {
    #pragma unroll 4
              for (int j = 0; j < trips; ++j) {
                unsigned wd;
                Real p;
                slot.load(base + 32 * j, wd, p);
                const Real term = p * e[wd >> 16] * (bt[wd & 0xFFFFu] + ld);
                A += term;
                xt[XS[base + 32 * j]] = as * term;
              }
            }
            if constexpr (GRP) A = group_sum(A, G);
            if (s != 0xFFFF && (!GRP || lead)) {
              const Real v = inv * A;
              put_vec(bn, s, v);
              dp = fma(CUSTOM_PI ? pi[s] : upi, v, dp);
            }
          }
        };
        if (G > 1)
          tiles(std::true_type{});
        else
          tiles(std::false_type{});
        dp = warp_sum(dp);
        if (lane == 0) part[cp * 32 + warp] = dp;
      }
      if (reads_post)
        cp_async_wait<0>();  // the gradient row read by the next flush is this group's
      else
        cp_async_wait<kTileBwdWait>();  // alpha t-2 and row t-3
      row_max_part(t - 3);
      gsync();
      if (!XDB) {
        // The posterior slots of frame t-1 are complete: write its gradient row,
        // then release the (single) slot buffer for the next frame.
        if (flusher) flush_post(t - 1, xterm);
        gsync();
      }
    }
    if (XDB && flusher) flush_post(0, xterm + X_pad);  // frame 0: written at t = 1
    stamp(3);
  };
  if constexpr (XDB) {
    if (a.persist > 0) {
      // Persistent CTAs (batch larger than the SMs): this CTA's utterances from
      // the in-kernel LPT (lfmmi_lpt.cuh), so the den never releases an SM to a
      // numerator CTA mid-batch; the numerator pass keeps the SMs left over.
      int *items = reinterpret_cast<int *>(smem + lay.items);
      lpt_assign<GROUP>(a.lengths, a.B, a.T_max, a.persist, int(blockIdx.x), 4,
                        reinterpret_cast<int *>(xterm), items);
      const int n = items[0];
      for (int i = 0; i < n; ++i) {
        if (i > 0) {  // previous utterance's copies and readers done before reuse
          cp_async_wait<0>();
          gsync();
        }
        run_item(items[4 + i]);
      }
      return;
    }
  }
  const int b = blockIdx.x * IPC + gid;
  if (b >= a.B) return;  // whole group exits together (no CTA-wide barriers for IPC > 1)
  run_item(b);
}

constexpr int kDenGroupC = 512;

template <typename Real, int GROUP, int IPC, bool SMEM_GRAPH, bool CUSTOM_PI, bool XDB = false>
static int launch_tile_impl2(const FBArgs<Real> &a, const lfmmi_graphs *g, size_t per_item,
                             cudaStream_t st) {
  static bool configured = false;
  auto kern = fb_tile_kernel<Real, GROUP, IPC, SMEM_GRAPH, CUSTOM_PI, XDB>;
  if (!configured) {
    int rc = check_cuda(
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem),
        "cudaFuncSetAttribute(tile)");
    if (rc) return rc;
    configured = true;
  }
  const int grid = (XDB && a.persist > 0) ? a.persist : (a.B + IPC - 1) / IPC;
  const int Fmax = std::max(g->max_tf_slots, g->max_tb_slots);
  if (GROUP != kDenGroupC || options().profile != "tile") {
    kern<<<grid, GROUP * IPC, per_item * IPC, st>>>(a, Fmax, g->max_tiles,
                                                    pad4(std::max(4, g->max_xpad)));
    return check_cuda(cudaGetLastError(), "fb_tile_kernel launch");
  }
  // Debug: forward / backward cycles per frame (mean over utterances) on stderr.
  FBArgs<Real> ap = a;
  long long *d = nullptr;
  cudaMalloc(&d, size_t(a.B) * 8 * sizeof(long long));
  cudaMemsetAsync(d, 0, size_t(a.B) * 8 * sizeof(long long), st);
  ap.prof = d;
  kern<<<grid, GROUP * IPC, per_item * IPC, st>>>(ap, Fmax, g->max_tiles,
                                                  pad4(std::max(4, g->max_xpad)));
  const int rc = check_cuda(cudaGetLastError(), "fb_tile_kernel launch");
  std::vector<long long> hp(size_t(a.B) * 8);
  cudaStreamSynchronize(st);
  cudaMemcpy(hp.data(), d, hp.size() * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  double fw = 0, bw = 0, fr = 0;
  for (int i = 0; i < a.B; ++i) {
    const long long *p = &hp[size_t(i) * 8];
    if (!p[3]) continue;
    fw += double(p[1] - p[0]);
    bw += double(p[3] - p[2]);
    fr += double(p[6]);
  }
  std::fprintf(stderr, "[lfmmi tile prof] forward %.0f  backward %.0f cycles/frame\n", fw / fr,
               bw / fr);
  return rc;
}

template <typename Real, int GROUP, int IPC, bool SMEM_GRAPH>
static int launch_tile_impl(const FBArgs<Real> &a, const lfmmi_graphs *g, size_t per_item,
                            cudaStream_t st) {
  if (a.leak_pi) return launch_tile_impl2<Real, GROUP, IPC, SMEM_GRAPH, true>(a, g, per_item, st);
  return launch_tile_impl2<Real, GROUP, IPC, SMEM_GRAPH, false>(a, g, per_item, st);
}

// Threads per utterance for the shared-memory (denominator) tile kernel.
constexpr int kDenGroup = 512;

template <typename Real>
int launch_tile(const FBArgs<Real> &a, const lfmmi_graphs *g, bool warp_per_item,
                cudaStream_t st) {
  if (!g->tileable) return set_error(LFMMI_ERR_UNSUPPORTED, "graph not tileable");
  const int Fmax = std::max(g->max_tf_slots, g->max_tb_slots);
  const int X_pad = pad4(std::max(4, g->max_xpad));
  const int real = int(sizeof(Real));
  if (warp_per_item) {
    const int RB = pad4(a.rep_r * a.r_stride), EB = a.rep_e * a.e_stride;  // 16-byte buffers
    const size_t per = tile_layout(false, Fmax, g->max_tiles, a.D, X_pad, a.S_pad, a.D_pad,
                                   a.T_pad, RB, EB, real).total;
    // Several utterances per CTA, but keep at least ~one CTA per SM busy.
    const size_t per_s = tile_layout(true, Fmax, g->max_tiles, a.D, X_pad, a.S_pad, a.D_pad,
                                     a.T_pad, RB, EB, real).total;
    note_kernel("fb_tile_kernel<Real,{128,64,32},*> (numerator-sized graphs)");
    const bool many = a.B >= 8 * 148;
    // Utterances fewer than SMs: more threads per numerator shorten its
    // per-frame latency chain (it runs next to the denominator pass).
    // 4 warps per numerator at every batch size: sweep (B = 1024) num pass
    // 7.8 ms vs 16.0 ms with one warp per utterance.
    const int want = options().num_group;
    if (want == 128 && per_s <= size_t(kMaxSmem))
      return launch_tile_impl<Real, 128, 1, true>(a, g, per_s, st);
    if (want == 64 && per_s <= size_t(kMaxSmem))
      return launch_tile_impl<Real, 64, 1, true>(a, g, per_s, st);
    if (many && per_s * 8 <= size_t(kMaxSmem))
      return launch_tile_impl<Real, 32, 8, true>(a, g, per_s, st);
    if (per_s * 2 <= size_t(kMaxSmem) && a.B >= 2 * 148)
      return launch_tile_impl<Real, 32, 2, true>(a, g, per_s, st);
    if (per_s <= size_t(kMaxSmem)) return launch_tile_impl<Real, 32, 1, true>(a, g, per_s, st);
    if (per <= size_t(kMaxSmem)) return launch_tile_impl<Real, 32, 1, false>(a, g, per, st);
    return set_error(LFMMI_ERR_UNSUPPORTED, "numerator slice exceeds shared memory");
  }
  const size_t per = tile_layout(true, Fmax, g->max_tiles, a.D, X_pad, a.S_pad, a.D_pad,
                                 a.T_pad, pad4(a.rep_r * a.r_stride), a.rep_e * a.e_stride, real).total;
  if constexpr (std::is_same<Real, float>::value) {
    // Fewer utterances than ~2x SMs: forward and backward of each utterance on
    // two SMs (cluster), load-balanced over the batch (lfmmi_split.cu).
    const int rc = launch_split<float>(a, g, st);
    if (rc != LFMMI_ERR_UNSUPPORTED) return rc;
    // Double-buffered slots first; per-frame scales in shared memory if they
    // still fit (short utterances), else in the HBM workspace.
    FBArgs<float> b = a;
    b.sc_smem = 1;
    size_t per2 = tile_layout(true, Fmax, g->max_tiles, a.D, X_pad, a.S_pad, a.D_pad, a.T_pad,
                              pad4(a.rep_r * a.r_stride), a.rep_e * a.e_stride, real, 2, true)
                      .total;
    if (per2 > size_t(kMaxSmem)) {
      b.sc_smem = 0;
      per2 = tile_layout(true, Fmax, g->max_tiles, a.D, X_pad, a.S_pad, a.D_pad, a.T_pad,
                         pad4(a.rep_r * a.r_stride), a.rep_e * a.e_stride, real, 2, false)
                 .total;
    }
    if (options().debug)
      std::fprintf(stderr, "[lfmmi] den tile smem single=%zu double=%zu limit=%d\n", per, per2,
                   kMaxSmem);
    if (!a.leak_pi && per2 <= size_t(kMaxSmem) && options().tile_xdb) {
      // More utterances than SMs: persistent CTAs (SMs minus the numerator
      // reserve) over an in-kernel LPT of the batch instead of one CTA per
      // utterance, whose waves let the concurrent numerator CTAs take SMs a
      // 200 KB denominator CTA then cannot use until they finish.
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int reserve = a.reserve_sms > 0 ? a.reserve_sms : 6;
      const int np = std::min(kLptMaxBins, sms - reserve);
      const int want = options().tile_persist;  // 0 off, 1 auto, >= 2 force that many CTAs
      b.persist = 0;
      if (want == 1 && a.B > sms && np > 0 && a.B <= np * kLptMaxItems && a.B <= X_pad)
        b.persist = np;
      if (want >= 2 && a.B <= std::min(want, kLptMaxBins) * kLptMaxItems && a.B <= X_pad)
        b.persist = std::min(want, kLptMaxBins);
      note_den_kernel(b.persist ? "fb_tile_kernel<float,512,1,1,0,1> (XDB, persistent)"
                                : "fb_tile_kernel<float,512,1,1,0,1> (XDB)");
      return launch_tile_impl2<float, kDenGroup, 1, true, false, true>(b, g, per2, st);
    }
  }
  if (per > size_t(kMaxSmem))
    return set_error(LFMMI_ERR_UNSUPPORTED,
                     "tile pack needs " + std::to_string(per) + " B shared memory");
  note_den_kernel("fb_tile_kernel<Real,512,1,1,*> (single slot buffer)");
  return launch_tile_impl<Real, kDenGroup, 1, true>(a, g, per, st);
}

template int launch_tile<float>(const FBArgs<float> &, const lfmmi_graphs *, bool, cudaStream_t);
template int launch_tile<double>(const FBArgs<double> &, const lfmmi_graphs *, bool,
                                 cudaStream_t);

}  // namespace lfmmi
