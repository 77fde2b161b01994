// fb_chain_kernel — the whole LF-MMI loss + gradient of one utterance in ONE
// CTA (fp32, uniform leak distribution): denominator and numerator recursions
// advance in lock-step, frame by frame, sharing one staged log-likelihood row
// and one exp'd emission row per frame, and the backward phase writes
// grad[t] = gamma_num[t] - gamma_den[t] exactly once.  One launch per batch:
// the last CTA to finish its forward also reduces the batch totals.
//
// Reference semantics (chainloss 0.1.0, /root/reference/pkg/src/chainloss):
//   emissions      forward_backward.py:120-130   (row max + exp, on the fly)
//   forward        _kernels.py:54-122            (scaled leaky alpha, finals at T_b)
//   log-prob       forward_backward.py:206-212   (sum ln scale + shift, fp64)
//   backward       _kernels.py:125-191           (leak adjoint, reuse of scales)
//   posteriors     _kernels.py:194-224           (per-arc slot + per-pdf gather)
//   chain_loss     loss.py:58-72                 (num - den, failed rows zeroed, totals)
// Numerator and denominator are independent recursions (each fails on its
// own and keeps its own normaliser); if either fails the backward is skipped
// and the utterance's gradient rows are zero, as loss.py:67-69 demands.
//
// Shared-memory residency per utterance: the arc pack of the current phase
// of BOTH graphs (denominator tiles of ~10k arcs + the numerator's few
// hundred), alpha/beta columns (replicated copies, see lfmmi_schedule.cpp),
// two emission rows, a 4-row log-likelihood ring, per-frame scales, and the
// per-arc posterior slots of one frame.  The alpha columns are spilled to the
// HBM workspace in the forward and streamed back two frames ahead.
#include "lfmmi_device.cuh"
#include "lfmmi_kernels.h"
#include "lfmmi_tile_common.cuh"

#include <cstdio>
#include <vector>
#include <algorithm>
#include <cstdlib>
#include <string>

#include "lfmmi_schedule.h"

namespace lfmmi {

// cp.async pipelines (one commit group per frame): log-likelihood rows are
// issued kRowAhead frames before their row maximum is taken, alpha rows (bwd)
// kAlphaAhead frames before use, so a frame never waits on HBM latency.
constexpr int kRowAhead = 4, kStageRing = 8;     // ring >= kRowAhead + 2, power of two
constexpr int kAlphaAhead = 2, kAlphaRing = 4;   // ring >= kAlphaAhead + 2, power of two
constexpr int kFwdWait = kRowAhead - 2;          // groups allowed in flight at frame end
constexpr int kBwdWait = (kRowAhead - 2 < kAlphaAhead - 1) ? kRowAhead - 2 : kAlphaAhead - 1;

// Byte offsets of one CTA's shared memory; computed on the host and passed by
// value, so every offset is a constant-bank operand in the kernel (no
// registers, no per-frame recomputation).
struct ChainLayout {
  unsigned wpd, xsd, tid_, ttd, tbd, wld, wtd, ppd, xtd, rbd, ard;
  unsigned wpn, xsn, tin, ttn, tbn, ppn, xtn, rbn, arn;
  unsigned ebuf, stage, scd, scn, shifts, partd, partn, mpart, flag, total;
};

__host__ __device__ inline ChainLayout chain_layout(const ChainDims &m, int D, int D_pad,
                                                    int T_pad, int RBd, int RBn, int EB,
                                                    int Sd_pad, int Sn_pad, bool xdb) {
  const size_t nx = xdb ? 2 : 1;  // posterior slot buffers (double-buffered when they fit)
  ChainLayout l;
  size_t o = 512;  // scratch: 32 doubles + 32 int64
  auto take = [&](size_t bytes) {
    const unsigned at = unsigned(o);
    o = al16(o + bytes);
    return at;
  };
  l.wpd = take(size_t(m.Fd) * 8);
  l.xsd = take(size_t(m.Fd) * 2);
  l.tid_ = take(size_t(m.ntd) * 128);
  l.ttd = take(size_t(pad4(m.ntd)) * 4);
  l.tbd = take(size_t(pad4(m.ntd)) * 4);
  l.wld = take(size_t(pad4(m.ntd)) * 4);
  l.wtd = take(size_t(kWarpTable) * 4);
  l.ppd = take(size_t(D + 1) * 4);
  l.xtd = take(nx * m.Xd * 4);
  l.rbd = take(size_t(2) * RBd * 4);
  l.ard = take(size_t(kAlphaRing) * Sd_pad * 4);
  l.wpn = take(size_t(m.Fn) * 8);
  l.xsn = take(size_t(m.Fn) * 2);
  l.tin = take(size_t(m.ntn) * 128);
  l.ttn = take(size_t(pad4(m.ntn)) * 4);
  l.tbn = take(size_t(pad4(m.ntn)) * 4);
  l.ppn = take(size_t(D + 1) * 4);
  l.xtn = take(nx * m.Xn * 4);
  l.rbn = take(size_t(2) * RBn * 4);
  l.arn = take(size_t(kAlphaRing) * Sn_pad * 4);
  l.ebuf = take(size_t(2) * EB * 4);
  l.stage = take(size_t(kStageRing) * D_pad * 4);
  l.scd = take(size_t(T_pad) * 4);
  l.scn = take(size_t(T_pad) * 4);
  l.shifts = take(size_t(T_pad) * 4);
  l.partd = take(size_t(2) * 32 * 4);
  l.partn = take(size_t(2) * 32 * 4);
  l.mpart = take(size_t(2) * 32 * 4);
  l.flag = take(16);
  l.total = unsigned(o);
  return l;
}

// One graph's view for a phase: tile pack staged in shared memory.
struct PhaseView {
  uint32_t wp, xs;  // shared addresses of the slot words / posterior slot ids
  const unsigned *tinfo;
  const int *ttrips, *tbase;
};

template <int GROUP>
__device__ __forceinline__ PhaseView stage_phase(const DevGraphs &g, const int *desc, bool fwd,
                                                 unsigned char *smem, size_t wp_off,
                                                 size_t xs_off, size_t ti_off, size_t tt_off,
                                                 size_t tb_off, int tid) {
  const int so = desc[fwd ? kTfSlotOff : kTbSlotOff], nsl = desc[fwd ? kTfSlots : kTbSlots];
  const int toff = desc[kTileOff];
  const int ntiles = (desc[kS] + 31) / 32;
  copy16<GROUP>(smem + wp_off, (fwd ? g.tf_wp : g.tb_wp) + so, size_t(nsl) * 8, tid);
  if (!fwd) copy16<GROUP>(smem + xs_off, g.tb_xslot + so, size_t(nsl) * 2, tid);
  copy16<GROUP>(smem + ti_off, (fwd ? g.tf_info : g.tb_info) + size_t(toff) * 32,
                size_t(ntiles) * 128, tid);
  copy16<GROUP>(smem + tt_off, (fwd ? g.tf_trips : g.tb_trips) + toff, size_t(pad4(ntiles)) * 4,
                tid);
  copy16<GROUP>(smem + tb_off, (fwd ? g.tf_base : g.tb_base) + toff, size_t(pad4(ntiles)) * 4,
                tid);
  PhaseView v;
  v.wp = smem_u32(smem + wp_off);
  v.xs = smem_u32(smem + xs_off);
  v.tinfo = reinterpret_cast<const unsigned *>(smem + ti_off);
  v.ttrips = reinterpret_cast<const int *>(smem + tt_off);
  v.tbase = reinterpret_cast<const int *>(smem + tb_off);
  return v;
}

// XDB: two posterior slot buffers — the gradient row of frame t is flushed by
// the chore warps at the start of the next backward iteration, overlapped
// with the other warps' arc work (one barrier per frame).  Without XDB the
// flush sits between two barriers.
// PROF (debug, LFMMI_PROFILE=1): lane 0 of every warp accumulates clock64()
// deltas per code section into a.prof[b][warp][section].
constexpr int kProfSections = 16;

template <int GROUP, bool XDB, bool PROF>
__global__ void __launch_bounds__(GROUP, 1)
    fb_chain_kernel(const ChainArgs a, const ChainDims m, const ChainLayout lay) {
  constexpr int NW = GROUP / 32;
  static_assert(NW == kTableNW, "denominator warp lists are scheduled for 16 warps");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Per-frame chores (emission rows, prefetch, gradient flush) run on the last
  // warps; the numerator tiles go to the first warps.
  const int ctid = GROUP - 1 - tid, cwarp = ctid >> 5;
  const int b = blockIdx.x;
  long long pacc[PROF ? kProfSections : 1] = {};
  long long plast = PROF ? clock64() : 0;
  // Debug ablations (PROF only): bit0 den tiles, bit1 num tiles, bit2 alpha spill,
  // bit3 normaliser reduction, bit4 gradient flush, bit5 emission rows, bit6 row
  // prefetch + row max, bit7 alpha prefetch.
  const int abl = PROF ? a.ablate : 0;
  auto skip = [&](int bit) { return PROF && (abl & (1 << bit)); };
  auto mark = [&](int sec) {
    if constexpr (PROF) {
      const long long now = clock64();
      pacc[sec] += now - plast;
      plast = now;
    }
  };
  const int RBd = pad4(a.rep_rd * a.r_strided), RBn = pad4(a.rep_rn * a.r_striden);
  const int EB = a.rep_e * a.e_stride;
  double *dscr = reinterpret_cast<double *>(smem);
  long long *lscr = reinterpret_cast<long long *>(smem + 256);
  float *rbd = reinterpret_cast<float *>(smem + lay.rbd);
  float *rbn = reinterpret_cast<float *>(smem + lay.rbn);
  float *ard = reinterpret_cast<float *>(smem + lay.ard);
  float *arn = reinterpret_cast<float *>(smem + lay.arn);
  float *xtd = reinterpret_cast<float *>(smem + lay.xtd);
  float *xtn = reinterpret_cast<float *>(smem + lay.xtn);
  int *ppd = reinterpret_cast<int *>(smem + lay.ppd);
  int *ppn = reinterpret_cast<int *>(smem + lay.ppn);
  float *ebuf = reinterpret_cast<float *>(smem + lay.ebuf);
  float *stage = reinterpret_cast<float *>(smem + lay.stage);
  float *scd = reinterpret_cast<float *>(smem + lay.scd);
  float *scn = reinterpret_cast<float *>(smem + lay.scn);
  float *shifts = reinterpret_cast<float *>(smem + lay.shifts);
  float *partd = reinterpret_cast<float *>(smem + lay.partd);
  float *partn = reinterpret_cast<float *>(smem + lay.partn);
  float *mpart = reinterpret_cast<float *>(smem + lay.mpart);
  int *flag = reinterpret_cast<int *>(smem + lay.flag);
  const int *wl = reinterpret_cast<const int *>(smem + lay.wld);
  const int *wt = reinterpret_cast<const int *>(smem + lay.wtd);

  const int T = a.lengths[b];
  const int D = a.D, D_pad = a.D_pad;
  const int *descd = a.den.desc + int(a.den_row_map[b]) * kDescInts;
  const int *descn = a.num.desc + int(a.num_row_map[b]) * kDescInts;
  const int Sd = descd[kS], Sn = descn[kS];
  const int ntd = (Sd + 31) / 32, ntn = (Sn + 31) / 32;
  const float *find = a.den.fin32 + descd[kStateOff];
  const float *finn = a.num.fin32 + descn[kStateOff];
  const float *Lb = a.L + size_t(b) * a.T_max * D;
  float *gb = a.grad + size_t(b) * a.T_max * D;
  const int nrw = (D + 31) / 32 < NW ? (D + 31) / 32 : NW;  // chore warps holding row elements
  int wlo = 0, whi = 0, nrank = 0;  // this warp's den tile range, numerator tile rank
  bool numw = false, nwriter = false;
  int nt_id = 0;
  auto read_warps = [&] {
    wlo = wt[warp];
    whi = wt[warp + 1];
    for (int j = 0; j < NW; ++j)
      if (wt[NW + 1 + j] == warp) nrank = j;
    numw = nrank < (ntn < NW ? ntn : NW);
    nwriter = numw && nrank == 0 && lane == 0;
    nt_id = nrank * 32 + lane;
  };
  auto gsync = [] { __syncthreads(); };

  // Denominator tiles per warp: host LPT schedule (lfmmi_schedule.cpp warp_lists).
  auto stage_warps = [&](bool fwd) {
    copy16<GROUP>(smem + lay.wld, (fwd ? a.den.tf_wlist : a.den.tb_wlist) + descd[kTileOff],
                  size_t(pad4(ntd)) * 4, tid);
    copy16<GROUP>(smem + lay.wtd, (fwd ? a.den.tf_wtab : a.den.tb_wtab) + descd[kWTabOff],
                  size_t(kWarpTable) * 4, tid);
  };
  PhaseView vd = stage_phase<GROUP>(a.den, descd, true, smem, lay.wpd, lay.xsd, lay.tid_, lay.ttd,
                                    lay.tbd, tid);
  stage_warps(true);
  PhaseView vn = stage_phase<GROUP>(a.num, descn, true, smem, lay.wpn, lay.xsn, lay.tin, lay.ttn,
                                    lay.tbn, tid);

  long long off = 0;
  for (int j = tid; j < b; j += GROUP) off += a.lengths[j];
  off = warp_sum(off);
  if (lane == 0) lscr[warp] = off;
  gsync();
  long long item_off = 0;
  for (int w = 0; w < NW; ++w) item_off += lscr[w];
  const float upid = float(1.0 / double(Sd)), upin = float(1.0 / double(Sn));
  const float lam = a.leak;
  float *trd = a.trellis_d + item_off * a.Sd_pad;
  float *trn = a.trellis_n + item_off * a.Sn_pad;
  if (a.packed) {  // ragged layout: item b's rows start at sum_{j<b} T_j
    Lb = a.L + size_t(item_off) * D;
    gb = a.grad + size_t(item_off) * D;
  }

  if (!a.packed)
    for (size_t i = tid; i < size_t(a.T_max - T) * D; i += GROUP) gb[size_t(T) * D + i] = 0.f;

  auto issue_row = [&](int t) {
    if (t < 0 || t >= T || cwarp >= nrw || skip(6)) return;
    const float *src = Lb + size_t(t) * D;
    float *dst = stage + (t & (kStageRing - 1)) * D_pad;
    for (int d = ctid; d < D; d += GROUP) cp_async_elem(dst + d, src + d);
  };
  auto row_max_part = [&](int t) {
    if (t < 0 || t >= T || cwarp >= nrw || skip(6)) return;
    const float *src = stage + (t & (kStageRing - 1)) * D_pad;
    float mx = -INFINITY;
    for (int d = ctid; d < D; d += GROUP) mx = nan_max(mx, src[d]);
    mx = warp_max(mx);
    if (lane == 0) mpart[(t & 1) * 32 + cwarp] = mx;
  };
  auto compute_e = [&](int t, bool record_shift) {
    if (cwarp >= nrw) return;
    const float *mp = mpart + (t & 1) * 32;
    float mx = lane < nrw ? mp[lane] : -INFINITY;
    mx = warp_max(mx);
    const float *src = stage + (t & (kStageRing - 1)) * D_pad;
    float *dst = ebuf + (t & 1) * EB;
    for (int d = ctid; d < D; d += GROUP) {
      const float v = expf(src[d] - mx);
      for (int c = 0; c < a.rep_e; ++c) dst[c * a.e_stride + d] = v;
    }
    if (record_shift && ctid == 0) shifts[t] = mx;
  };
  const int rep_rd = a.rep_rd, rsd = a.r_strided, rep_rn = a.rep_rn, rsn = a.r_striden;
  auto put_d = [&](float *v, int s, float x) {
    v[s] = x;
    if (rep_rd > 1) v[rsd + s] = x;
  };
  auto put_n = [&](float *v, int s, float x) {
    v[s] = x;
    if (rep_rn > 1) v[rsn + s] = x;
  };

  // ---- prologue -----------------------------------------------------------------
  {
    const int init_d = descd[kInit], init_n = descn[kInit];
    for (int s = tid; s < Sd; s += GROUP) put_d(rbd, s, s == init_d ? 1.f : 0.f);
    for (int s = tid; s < Sn; s += GROUP) put_n(rbn, s, s == init_n ? 1.f : 0.f);
    if (tid < 4) flag[tid] = -1;
  }
  for (int j = 0; j < kRowAhead; ++j) {  // one group per row: group j holds row j
    issue_row(j);
    cp_async_commit();
  }
  cp_async_wait<kFwdWait>();  // rows 0, 1 (and the staged phase packs) have landed
  row_max_part(0);
  row_max_part(1);
  gsync();
  compute_e(0, true);
  gsync();
  read_warps();

  // ---- forward: both graphs, one barrier per frame -------------------------------------
  float inv_d = 1.f, inv_n = 1.f, lcd = 0.f, lcn = 0.f;
  int fail_d = -1, fail_n = -1;
  // Numerator recursion state lives on the nwn "numerator warps" only (the
  // warps the host schedule left lightest, see read_warps); they alone reduce
  // its partial sums.  Its failure status reaches every warp through flag[]
  // (double-buffered by frame parity; one frame late is harmless).
  const int nwn = ntn < NW ? ntn : NW;
  auto part_sum = [&](const float *v, int n) {
    float x = lane < n ? v[lane] : 0.f;
    return warp_sum(x);
  };
  auto normaliser = [&](const float *part, int n, bool writer, int k, float &inv, float &lc,
                        int &fail, float *sc) {
    const float t0 = (skip(0) || skip(3)) ? 1.f : part_sum(part, n);
    float t2 = t0;
    lc = 0.f;
    if (lam > 0.f && t0 > 0.f) {
      lc = lam * t0;
      t2 = t0 + lc;  // uniform pi sums to 1
    }
    if (!(t2 >= a.floor_eff) || isinf(t2)) {
      fail = k;
      return;
    }
    inv = __frcp_rn(t2);  // == 1.f / t2 (both IEEE round-to-nearest)
    if (writer) sc[k] = t2;
  };
  mark(15);
  for (int k = 0; k < T; ++k) {
    const int cur = k & 1, nxt = cur ^ 1;
    if (k > 0) {
      if (fail_d < 0) normaliser(partd + cur * 32, NW, tid == 0, k - 1, inv_d, lcd, fail_d, scd);
      if (numw && fail_n < 0)
        normaliser(partn + cur * 32, nwn, nwriter, k - 1, inv_n, lcn, fail_n, scn);
      if (nwriter) flag[2 + cur] = fail_n;
      if (fail_d >= 0 && flag[2 + (cur ^ 1)] >= 0) break;  // uniform: previous frame's flag
    }
    const bool alive_d = fail_d < 0, alive_n = numw && fail_n < 0;
    if (alive_d && !skip(2)) {
      const float *r = rbd + cur * RBd;
      float *row = trd + size_t(k) * a.Sd_pad;
      const float lu = lcd * upid;
      for (int s = tid; s < Sd; s += GROUP) row[s] = (r[s] + lu) * inv_d;
    }
    if (alive_n && !skip(2)) {
      const float *r = rbn + cur * RBn;
      float *row = trn + size_t(k) * a.Sn_pad;
      const float lu = lcn * upin;
      for (int s = nt_id; s < Sn; s += nwn * 32) row[s] = (r[s] + lu) * inv_n;
    }
    mark(0);
    if (k + 1 < T && !skip(5)) compute_e(k + 1, true);
    issue_row(k + kRowAhead);
    cp_async_commit();
    mark(1);
    const bool last = (k + 1 == T);
    const uint32_t e32 = smem_u32(ebuf + cur * EB);
    float psd = 0.f, psn = 0.f;
    if (alive_d && !skip(0)) {
      const uint32_t r32 = smem_u32(rbd + cur * RBd);
      float *rn = rbd + nxt * RBd;
      for (int i = wlo; i < whi; ++i) {
        const int tile = wl[i];
        const unsigned info = vd.tinfo[tile * 32 + lane];
        const uint32_t sb = vd.wp + uint32_t(vd.tbase[tile] + lane) * 8u;
        float A = 0.f, Bs = 0.f;
        if (lcd != 0.f)
          fwd_tile_f32<true>(sb, vd.ttrips[tile], e32, r32, A, Bs);
        else
          fwd_tile_f32<false>(sb, vd.ttrips[tile], e32, r32, A, Bs);
        const int s = int(info & 0xFFFFu);
        if (s != 0xFFFF) {
          float raw = inv_d * (A + lcd * upid * Bs);
          if (last) raw *= find[s];
          put_d(rn, s, raw);
          psd += raw;
        }
      }
    }
    mark(2);
    if (alive_n && !skip(1)) {
      const uint32_t r32 = smem_u32(rbn + cur * RBn);
      float *rn = rbn + nxt * RBn;
      for (int tile = nrank; tile < ntn; tile += NW) {
        const unsigned info = vn.tinfo[tile * 32 + lane];
        const uint32_t sb = vn.wp + uint32_t(vn.tbase[tile] + lane) * 8u;
        float A = 0.f, Bs = 0.f;
        if (lcn != 0.f)
          fwd_tile_f32<true>(sb, vn.ttrips[tile], e32, r32, A, Bs);
        else
          fwd_tile_f32<false>(sb, vn.ttrips[tile], e32, r32, A, Bs);
        const int s = int(info & 0xFFFFu);
        if (s != 0xFFFF) {
          float raw = inv_n * (A + lcn * upin * Bs);
          if (last) raw *= finn[s];
          put_n(rn, s, raw);
          psn += raw;
        }
      }
    }
    mark(3);
    psd = warp_sum(psd);
    if (lane == 0) partd[nxt * 32 + warp] = psd;
    if (numw) {
      psn = warp_sum(psn);
      if (lane == 0) partn[nxt * 32 + nrank] = psn;
    }
    mark(4);
    cp_async_wait<kFwdWait>();  // row k + 2
    row_max_part(k + 2);
    mark(5);
    gsync();
    mark(6);
  }
  // Normaliser of the last column (the loop ends before consuming it).
  if (fail_d < 0) normaliser(partd + (T & 1) * 32, NW, tid == 0, T - 1, inv_d, lcd, fail_d, scd);
  if (numw && fail_n < 0)
    normaliser(partn + (T & 1) * 32, nwn, nwriter, T - 1, inv_n, lcn, fail_n, scn);
  if (nwriter) flag[1] = fail_n;
  gsync();
  fail_n = flag[1];  // CTA-uniform from here on
  {
    // logP = sum_k ln(scale_k) + shift_k (forward_backward.py:206-212), fp64.
    double acd = 0.0, acn = 0.0;
    for (int k = tid; k < T; k += GROUP) {
      const double sh = double(shifts[k]);
      if (fail_d < 0) acd += log(double(scd[k])) + sh;
      if (fail_n < 0) acn += log(double(scn[k])) + sh;
    }
    acd = warp_sum(acd);
    acn = warp_sum(acn);
    if (lane == 0) {
      dscr[warp] = acd;
      dscr[16 + warp] = acn;
    }
    gsync();
    if (tid == 0) {
      double td = 0.0, tn = 0.0;
      for (int w = 0; w < NW; ++w) {
        td += dscr[w];
        tn += dscr[16 + w];
      }
      a.den_lp[b] = fail_d >= 0 ? NAN : td;
      a.num_lp[b] = fail_n >= 0 ? NAN : tn;
      a.den_fail[b] = fail_d;
      a.num_fail[b] = fail_n;
      int last_cta = 0;
      if (a.totals) {
        __threadfence();
        last_cta = atomicAdd(a.counter, 1u) == unsigned(a.B - 1);
      }
      flag[0] = last_cta;
    }
    gsync();
    if (flag[0]) {
      // Batch totals (loss.py:61-72) in a fixed order: {sum_ok(num - den), sum_ok T_b, #failed}.
      __threadfence();
      double o = 0.0, f = 0.0, n = 0.0;
      for (int j = tid; j < a.B; j += GROUP) {
        const int nf = *((volatile int *)(a.num_fail + j)), df = *((volatile int *)(a.den_fail + j));
        if (nf < 0 && df < 0) {
          o += *((volatile double *)(a.num_lp + j)) - *((volatile double *)(a.den_lp + j));
          f += double(a.lengths[j]);
        } else {
          n += 1.0;
        }
      }
      o = warp_sum(o);
      f = warp_sum(f);
      n = warp_sum(n);
      gsync();
      if (lane == 0) {
        dscr[warp] = o;
        dscr[16 + warp] = f;
        lscr[warp] = (long long)n;
      }
      gsync();
      if (tid == 0) {
        double to = 0.0, tf = 0.0, tn = 0.0;
        for (int w = 0; w < NW; ++w) {
          to += dscr[w];
          tf += dscr[16 + w];
          tn += double(lscr[w]);
        }
        a.totals[0] = to;
        a.totals[1] = tf;
        a.totals[2] = tn;
      }
    }
  }
  if (fail_d >= 0 || fail_n >= 0) {
    for (size_t i = tid; i < size_t(T) * D; i += GROUP) gb[i] = 0.f;
    return;
  }

  // ---- backward + fused posterior / gradient ----------------------------------------
  gsync();  // all forward reads of the phase packs are done
  vd = stage_phase<GROUP>(a.den, descd, false, smem, lay.wpd, lay.xsd, lay.tid_, lay.ttd, lay.tbd,
                          tid);
  stage_warps(false);
  vn = stage_phase<GROUP>(a.num, descn, false, smem, lay.wpn, lay.xsn, lay.tin, lay.ttn, lay.tbn,
                          tid);
  {
    const int *pd = a.den.pdf_arc_ptr + descd[kPdfPtrOff2];
    const int *pn = a.num.pdf_arc_ptr + descn[kPdfPtrOff2];
    for (int d = tid; d <= D; d += GROUP) {
      ppd[d] = pd[d];
      ppn[d] = pn[d];
    }
    // Padding slots of the per-pdf groups are never written: zero them once.
    for (int i = tid; i < (XDB ? 2 : 1) * m.Xd; i += GROUP) xtd[i] = 0.f;
    for (int i = tid; i < (XDB ? 2 : 1) * m.Xn; i += GROUP) xtn[i] = 0.f;
  }
  auto issue_alpha = [&](int k) {
    if (k < 0 || skip(7)) return;
    copy16<GROUP>(ard + (k & (kAlphaRing - 1)) * a.Sd_pad, trd + size_t(k) * a.Sd_pad,
                  size_t(a.Sd_pad) * 4,
                  ctid);
    copy16<GROUP>(arn + (k & (kAlphaRing - 1)) * a.Sn_pad, trn + size_t(k) * a.Sn_pad,
                  size_t(a.Sn_pad) * 4,
                  ctid);
  };
  int spl = 1;  // lanes per pdf in the gradient flush (power of two, all chore warps)
  while (spl < 32 && D * spl * 2 <= GROUP) spl <<= 1;
  auto flush = [&](int t, const float *xd, const float *xn) {
    float *prow = gb + size_t(t) * D;
    const int sub = ctid & (spl - 1);
    for (int base_i = 0; base_i < D * spl; base_i += GROUP) {
      const int idx = base_i + ctid;
      const int d = idx / spl;
      float gd = 0.f, gn = 0.f;
      if (d < D) {
        const int lo = ppd[d] >> 2, hi = ppd[d + 1] >> 2;
        for (int q = lo + sub; q < hi; q += spl) gd += sum_groups4(xd + 4 * q, 1);
        const int lo2 = ppn[d] >> 2, hi2 = ppn[d + 1] >> 2;
        for (int q = lo2 + sub; q < hi2; q += spl) gn += sum_groups4(xn + 4 * q, 1);
      }
      for (int o = 1; o < spl; o <<= 1) {
        gd += __shfl_xor_sync(kFull, gd, o);
        gn += __shfl_xor_sync(kFull, gn, o);
      }
      if (d < D && sub == 0) prow[d] = gn - gd;
    }
  };

  {
    const float fl = 1.f + lam;
    for (int s = tid; s < Sd; s += GROUP) put_d(rbd + (T & 1) * RBd, s, find[s] * fl);
    for (int s = tid; s < Sn; s += GROUP) put_n(rbn + (T & 1) * RBn, s, finn[s] * fl);
  }
  // Backward pipeline: "iteration" u issues row u-1-kRowAhead and alpha u-1-kAlphaAhead;
  // the virtual iterations T+kRowAhead .. T+1 fill it (one group each).
  for (int u = T + kRowAhead; u > T; --u) {
    if (u - 1 - kRowAhead < T) issue_row(u - 1 - kRowAhead);
    if (u - 1 - kAlphaAhead < T) issue_alpha(u - 1 - kAlphaAhead);
    cp_async_commit();
  }
  cp_async_wait<kBwdWait>();  // rows T-1, T-2, alpha T-1, phase packs
  row_max_part(T - 1);
  row_max_part(T - 2);
  gsync();
  compute_e(T - 1, false);
  gsync();
  read_warps();

  const bool flusher = cwarp * 32 < D * spl;
  for (int t = T; t >= 1; --t) {
    const int ct = t & 1, cp = ct ^ 1;
    // Slot buffer written this iteration (frame t-1); XDB: flush frame t (written
    // last iteration into the other buffer) while the other warps start their arcs.
    const int xb = XDB ? ct : 0;
    mark(14);
    if (XDB && t < T && flusher && !skip(4)) flush(t, xtd + (xb ^ 1) * m.Xd, xtn + (xb ^ 1) * m.Xn);
    mark(7);
    const uint32_t xd32 = smem_u32(xtd + xb * m.Xd), xn32 = smem_u32(xtn + xb * m.Xn);
    float ldd = 0.f, ldn = 0.f;
    if (t < T && lam > 0.f && !skip(3)) {
      ldd = lam * lane_sum<NW>(partd + ct * 32, lane);
      if (numw) ldn = lam * part_sum(partn + ct * 32, nwn);
    }
    const float ivd = __frcp_rn(scd[t - 1]), ivn = numw ? __frcp_rn(scn[t - 1]) : 0.f;
    if (t - 2 >= 0 && !skip(5)) compute_e(t - 2, false);
    issue_row(t - 1 - kRowAhead);
    issue_alpha(t - 1 - kAlphaAhead);
    cp_async_commit();
    mark(8);
    const uint32_t e32 = smem_u32(ebuf + cp * EB);
    float dpd = 0.f, dpn = 0.f;
    if (!skip(0)) {
      const uint32_t b32 = smem_u32(rbd + ct * RBd);
      const float *al = ard + ((t - 1) & (kAlphaRing - 1)) * a.Sd_pad;  // alpha_{t-1}
      float *bn = rbd + cp * RBd;
      for (int i = wlo; i < whi; ++i) {
        const int tile = wl[i];
        const unsigned info = vd.tinfo[tile * 32 + lane];
        const int base = vd.tbase[tile] + lane;
        const int s = int(info & 0xFFFFu);
        const float as = (s != 0xFFFF) ? al[s] * ivd : 0.f;
        const float A = bwd_tile_f32(vd.wp + uint32_t(base) * 8u, vd.xs + uint32_t(base) * 2u,
                                     vd.ttrips[tile], e32, b32, xd32, ldd, as);
        if (s != 0xFFFF) {
          const float v = ivd * A;
          put_d(bn, s, v);
          dpd = fmaf(upid, v, dpd);
        }
      }
    }
    mark(9);
    if (numw && !skip(1)) {
      const uint32_t b32 = smem_u32(rbn + ct * RBn);
      const float *al = arn + ((t - 1) & (kAlphaRing - 1)) * a.Sn_pad;
      float *bn = rbn + cp * RBn;
      for (int tile = nrank; tile < ntn; tile += NW) {
        const unsigned info = vn.tinfo[tile * 32 + lane];
        const int base = vn.tbase[tile] + lane;
        const int s = int(info & 0xFFFFu);
        const float as = (s != 0xFFFF) ? al[s] * ivn : 0.f;
        const float A = bwd_tile_f32(vn.wp + uint32_t(base) * 8u, vn.xs + uint32_t(base) * 2u,
                                     vn.ttrips[tile], e32, b32, xn32, ldn, as);
        if (s != 0xFFFF) {
          const float v = ivn * A;
          put_n(bn, s, v);
          dpn = fmaf(upin, v, dpn);
        }
      }
    }
    mark(10);
    dpd = warp_sum(dpd);
    if (lane == 0) partd[cp * 32 + warp] = dpd;
    if (numw) {
      dpn = warp_sum(dpn);
      if (lane == 0) partn[cp * 32 + nrank] = dpn;
    }
    mark(11);
    cp_async_wait<kBwdWait>();  // row t-3 and alpha t-2
    row_max_part(t - 3);
    gsync();
    mark(12);
    if (!XDB) {
      // Posterior slots of frame t-1 are complete: write grad[t-1] = gamma_num -
      // gamma_den, then release the slot buffer for the next frame.
      if (flusher && !skip(4)) flush(t - 1, xtd, xtn);
      gsync();
    }
    mark(13);
  }
  if (XDB && flusher) flush(0, xtd + 1 * m.Xd, xtn + 1 * m.Xn);  // frame 0: written at t = 1
  if constexpr (PROF) {
    if (lane == 0)
      for (int i = 0; i < kProfSections; ++i)
        a.prof[(size_t(b) * NW + warp) * kProfSections + i] = pacc[i];
  }
}

template <bool XDB>
static int launch_profiled(const ChainArgs &a0, const ChainDims &m, const ChainLayout &lay,
                           cudaStream_t st);

template <bool XDB, bool PROF = false>
static int launch_chain_impl(const ChainArgs &a, const ChainDims &m, const ChainLayout &lay,
                             cudaStream_t st) {
  const size_t smem = lay.total;
  constexpr int G = 512;
  if (!PROF && std::getenv("LFMMI_PROFILE")) return launch_profiled<XDB>(a, m, lay, st);
  static bool configured = false;
  if (!configured) {
    const int rc = check_cuda(cudaFuncSetAttribute(fb_chain_kernel<G, XDB, PROF>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   kMaxSmem),
                              "cudaFuncSetAttribute(chain)");
    if (rc) return rc;
    configured = true;
  }
  fb_chain_kernel<G, XDB, PROF><<<a.B, G, smem, st>>>(a, m, lay);
  return check_cuda(cudaGetLastError(), "fb_chain_kernel launch");
}

// Debug: one instrumented launch, per-section cycles per frame printed to stderr.
template <bool XDB>
static int launch_profiled(const ChainArgs &a0, const ChainDims &m, const ChainLayout &lay,
                           cudaStream_t st) {
  constexpr int NW = 16;
  ChainArgs a = a0;
  const size_t n = size_t(a.B) * NW * kProfSections;
  long long *d = nullptr;
  int rc = check_cuda(cudaMalloc(&d, n * sizeof(long long)), "cudaMalloc(prof)");
  if (rc) return rc;
  a.prof = d;
  a.ablate = std::getenv("LFMMI_ABLATE") ? std::atoi(std::getenv("LFMMI_ABLATE")) : 0;
  rc = launch_chain_impl<XDB, true>(a, m, lay, st);
  if (rc) return rc;
  std::vector<long long> h(n);
  std::vector<int> len(a.B);
  cudaStreamSynchronize(st);
  cudaMemcpy(h.data(), d, n * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaMemcpy(len.data(), a.lengths, a.B * sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(d);
  static const char *names[kProfSections] = {
      "F normaliser+spill", "F emis+issue", "F den tiles", "F num tiles", "F warp sums",
      "F wait+rowmax", "F barrier", "B flush(XDB)", "B emis+issue", "B den tiles", "B num tiles",
      "B warp sums", "B wait+rowmax+barrier", "B flush+barrier(1x)", "B top", "prologue"};
  std::fprintf(stderr, "[lfmmi prof] XDB=%d ablate=%d cycles per frame (mean over CTAs): warp0 / "
               "warp15 / mean / max over warps\n", int(XDB), a.ablate);
  {
    double fwd = 0, bwd = 0;
    for (int b = 0; b < a.B; ++b) {
      const double T = std::max(1, len[b]);
      long long f = 0, g = 0;
      for (int s = 0; s <= 6; ++s) f += h[(size_t(b) * NW) * kProfSections + s];
      for (int s = 7; s <= 14; ++s) g += h[(size_t(b) * NW) * kProfSections + s];
      fwd += f / T / a.B;
      bwd += g / T / a.B;
    }
    std::fprintf(stderr, "[lfmmi prof] TOTAL per frame: fwd %.0f  bwd %.0f  cycles\n", fwd, bwd);
  }
  for (int s = 0; s < kProfSections; ++s) {
    double w0 = 0, w15 = 0, mean = 0, mx = 0;
    for (int b = 0; b < a.B; ++b) {
      const double T = std::max(1, len[b]);
      double bm = 0, bx = 0;
      for (int w = 0; w < NW; ++w) {
        const double v = double(h[(size_t(b) * NW + w) * kProfSections + s]) / T;
        bm += v / NW;
        bx = std::max(bx, v);
        if (w == 0) w0 += v / a.B;
        if (w == NW - 1) w15 += v / a.B;
      }
      mean += bm / a.B;
      mx += bx / a.B;
    }
    std::fprintf(stderr, "[lfmmi prof] %-24s %8.0f %8.0f %8.0f %8.0f\n", names[s], w0, w15, mean,
                 mx);
  }
  return LFMMI_OK;
}

int launch_chain(const ChainArgs &a, const ChainDims &m, cudaStream_t st) {
  note_den_kernel("fb_chain_kernel<512> (num+den+grad, one launch)");
  const int RBd = pad4(a.rep_rd * a.r_strided), RBn = pad4(a.rep_rn * a.r_striden),
            EB = a.rep_e * a.e_stride;
  const ChainLayout l2 =
      chain_layout(m, a.D, a.D_pad, a.T_pad, RBd, RBn, EB, a.Sd_pad, a.Sn_pad, true);
  const ChainLayout l1 =
      chain_layout(m, a.D, a.D_pad, a.T_pad, RBd, RBn, EB, a.Sd_pad, a.Sn_pad, false);
  const size_t s2 = l2.total, s1 = l1.total;
  static bool told = false;
  if (std::getenv("LFMMI_DEBUG") && !told) {
    told = true;
    std::fprintf(stderr,
                 "[lfmmi] chain layout: smem single=%zu double=%zu limit=%d | Fd=%d ntd=%d Xd=%d "
                 "Fn=%d ntn=%d Xn=%d RBd=%d RBn=%d EB=%d T_pad=%d\n",
                 s1, s2, kMaxSmem, m.Fd, m.ntd, m.Xd, m.Fn, m.ntn, m.Xn, RBd, RBn, EB, a.T_pad);
  }
  if (s2 <= size_t(kMaxSmem) && !std::getenv("LFMMI_CHAIN_SINGLE_X"))
    return launch_chain_impl<true>(a, m, l2, st);
  if (s1 <= size_t(kMaxSmem)) return launch_chain_impl<false>(a, m, l1, st);
  return set_error(LFMMI_ERR_UNSUPPORTED,
                   "fused chain kernel needs " + std::to_string(s1) + " B shared memory");
}

}  // namespace lfmmi
