// Group-generic fused forward-backward: one thread GROUP (a warp, or a
// CTA of up to 1024 threads) per utterance, whole time loop on chip, one
// group barrier per frame.  Arc lists are read from the global graph pack
// (L1/L2 resident); used for numerator graphs (GROUP = 32, several
// utterances per CTA, __syncwarp only) and as the general fallback for graphs
// the tile kernel cannot stage in shared memory.
//
// Semantics follow the reference recursions exactly:
//   forward  _kernels.py:54-122, backward _kernels.py:125-191,
//   posterior _kernels.py:194-224, emissions forward_backward.py:120-130,
//   log-probability forward_backward.py:206-212, num-minus-den loss.py:67-69.
// Deferred normalisation: column k+1 is gathered from the *unnormalised*
// column k and its normaliser/leak are applied inside the gather, so a frame
// needs one barrier instead of three.
#include "lfmmi_device.cuh"
#include "lfmmi_kernels.h"

namespace lfmmi {

template <int GROUP, int GPC>
__device__ __forceinline__ void group_sync(int gid) {
  if constexpr (GROUP == 32) {
    __syncwarp();
  } else if constexpr (GPC == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(gid + 1), "n"(GROUP) : "memory");
  }
}

struct GroupLayout {
  int rbuf, aring, ebuf, stage, gstage, slots, scales, shifts, part, mpart, reals;
};

// LARGE (graphs whose state vectors leave no room for the alpha ring, e.g.
// 20k states): alpha_{t-1} is read straight from the HBM/L2 trellis, the
// gradient is never read back (WRITE / NEGATE modes only) and the per-chunk
// posterior partials are single-buffered (one extra barrier per frame).
__host__ __device__ inline GroupLayout group_layout(int S_pad, int D_pad, int NC_pad, int T_pad,
                                                    int NW, bool large = false) {
  GroupLayout l;
  int o = 0;
  l.rbuf = o;   o += 2 * S_pad;                  // alpha / beta columns (ping-pong)
  l.aring = o;  o += large ? 0 : 3 * S_pad;      // alpha columns streamed back from HBM
  l.ebuf = o;   o += 2 * D_pad;                  // exp'd emission rows
  l.stage = o;  o += 4 * D_pad;                  // raw log-likelihood rows (cp.async ring)
  l.gstage = o; o += large ? 0 : 3 * D_pad;      // existing gradient rows (ADD / SUBTRACT modes)
  l.slots = o;  o += (large ? 1 : 2) * NC_pad;   // per-chunk posterior partials
  l.scales = o; o += T_pad;
  l.shifts = o; o += T_pad;
  l.part = o;   o += pad4(2 * NW);
  l.mpart = o;  o += pad4(2 * NW);
  l.reals = o;
  return l;
}

constexpr int kGroupScratch = 512;

template <typename Real>
size_t group_smem_bytes(int S_pad, int D_pad, int NC_pad, int T_pad, int group,
                        bool large = false) {
  const GroupLayout l = group_layout(S_pad, D_pad, NC_pad, T_pad, group / 32, large);
  return (kGroupScratch + size_t(l.reals) * sizeof(Real) + 15) & ~size_t(15);
}

template <typename Real, int GROUP, int GPC, bool LARGE>
__global__ void __launch_bounds__(GROUP *GPC, 1) fb_group_kernel(const FBArgs<Real> a) {
  constexpr int NW = GROUP / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gid = threadIdx.x / GROUP;
  const int tid = threadIdx.x % GROUP, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x * GPC + gid;
  if (b >= a.B) return;  // whole group exits together

  const GroupLayout lay = group_layout(a.S_pad, a.D_pad, a.NC_pad, a.T_pad, NW, LARGE);
  const size_t gbytes = (kGroupScratch + size_t(lay.reals) * sizeof(Real) + 15) & ~size_t(15);
  unsigned char *base = smem_raw + gbytes * gid;
  double *dscr = reinterpret_cast<double *>(base);
  long long *lscr = reinterpret_cast<long long *>(base + 256);
  Real *sm = reinterpret_cast<Real *>(base + kGroupScratch);
  Real *rbuf = sm + lay.rbuf;
  Real *aring = sm + lay.aring;
  Real *ebuf = sm + lay.ebuf;
  Real *stage = sm + lay.stage;
  Real *gstage = sm + lay.gstage;
  Real *slots = sm + lay.slots;
  Real *scales = sm + lay.scales;
  Real *shifts = sm + lay.shifts;
  Real *part = sm + lay.part;
  Real *mpart = sm + lay.mpart;
  auto gsync = [&]() { group_sync<GROUP, GPC>(gid); };

  const int T = item_frames(a.lengths, b, a.T_max);
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
  const int mode = a.mode;
  const bool reads_post = mode == kPostAdd || mode == kPostSubtract;
  const bool other_failed = a.other_fail != nullptr && a.other_fail[b] >= 0;

  // Ragged alpha-trellis offset = sum of earlier lengths; custom leak mass.
  long long off = 0;
  for (int j = tid; j < b; j += GROUP) off += a.lengths[j];
  off = warp_sum(off);
  const Real *pi = a.leak_pi ? a.leak_pi + size_t(row) * a.S_max : nullptr;
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
  if (a.packed) {  // ragged layout: item b's rows start at sum_{j<b} T_j
    Lb = a.L + size_t(item_off) * D;
    post_b = a.post + size_t(item_off) * D;
  }

  if (!reads_post && !a.packed) {
    const size_t n = size_t(a.T_max - T) * D;
    for (size_t i = tid; i < n; i += GROUP) post_b[size_t(T) * D + i] = Real(0);
  }

  auto issue_row = [&](int t) {
    if (t < 0 || t >= T) return;
    const Real *src = Lb + size_t(t) * D;
    Real *dst = stage + (t & 3) * D_pad;
    for (int d = tid; d < D; d += GROUP) cp_async_elem(dst + d, src + d);
  };
  auto row_max_part = [&](int t) {
    if (t < 0 || t >= T) return;
    const Real *src = stage + (t & 3) * D_pad;
    Real m = -INFINITY;
    for (int d = tid; d < D; d += GROUP) m = nan_max(m, src[d]);
    m = warp_max(m);
    if (lane == 0) mpart[(t & 1) * NW + warp] = m;
  };
  auto block_max = [&](int t) {
    Real m = -INFINITY;
    for (int w = 0; w < NW; ++w) m = nan_max(m, mpart[(t & 1) * NW + w]);
    return m;
  };
  auto compute_e = [&](int t, bool record_shift) {  // e_t -> ebuf[t & 1]
    const Real m = block_max(t);
    const Real *src = stage + (t & 3) * D_pad;
    Real *dst = ebuf + (t & 1) * D_pad;
    for (int d = tid; d < D; d += GROUP) dst[d] = exp_r(src[d] - m);
    if (record_shift && tid == 0) shifts[t] = m;
  };

  // ---- prologue -------------------------------------------------------------
  for (int s = tid; s < S; s += GROUP) rbuf[s] = (s == init) ? Real(1) : Real(0);
  issue_row(0);
  issue_row(1);
  cp_async_commit();
  issue_row(2);
  cp_async_commit();
  cp_async_wait<1>();
  row_max_part(0);
  row_max_part(1);
  gsync();
  compute_e(0, true);
  gsync();

  // ---- forward: one group barrier per frame -----------------------------------
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
    {
      const Real *r = rbuf + cur * S_pad;
      Real *arow = trellis + size_t(k) * S_pad;
      for (int s = tid; s < S; s += GROUP) arow[s] = (r[s] + leakc * (pi ? pi[s] : upi)) * inv2;
    }
    if (k + 1 < T) compute_e(k + 1, true);
    issue_row(k + 3);
    cp_async_commit();
    {
      const Real *e = ebuf + cur * D_pad;
      const Real *r = rbuf + cur * S_pad;
      Real *rn = rbuf + nxt * S_pad;
      const bool last = (k + 1 == T);
      Real psum = Real(0);
      for (int s = tid; s < S; s += GROUP) {
        const int lo = __ldg(in_ptr + s), hi = __ldg(in_ptr + s + 1);
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
            const Real w = __ldg(in_p + i) * e[__ldg(in_pdf + i)];
            A = fma(w, r[__ldg(in_src + i)], A);
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
    cp_async_wait<1>();
    row_max_part(k + 2);
    gsync();
  }
  cp_async_wait<0>();
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
  if (fail_at >= 0) {
    // Remaining shifts are the row maxima (the reference exponentiates every
    // valid frame); remaining scales stay 1 (forward_backward.py:184,206).
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

  // ---- backward + fused posterior / gradient ------------------------------------
  auto issue_alpha = [&](int k) {
    if (LARGE || k < 0) return;
    const char *src = reinterpret_cast<const char *>(trellis + size_t(k) * S_pad);
    char *d = reinterpret_cast<char *>(aring + (k % 3) * S_pad);
    const int chunks = S_pad * int(sizeof(Real)) / 16;
    for (int c = tid; c < chunks; c += GROUP) cp_async_16(d + 16 * c, src + 16 * c);
  };
  // Existing gradient rows are prefetched two frames ahead (cp.async) so the
  // read-modify-write never exposes global-memory latency.
  auto issue_post = [&](int t) {
    if (!reads_post || t < 0 || t >= T) return;
    const Real *src = post_b + size_t(t) * D;
    Real *dst = gstage + (t % 3) * D_pad;
    for (int d = tid; d < D; d += GROUP) cp_async_elem(dst + d, src + d);
  };
  auto flush_post = [&](int t, const Real *sl) {
    Real *prow = post_b + size_t(t) * D;
    const Real *old = gstage + (t % 3) * D_pad;
    for (int d = tid; d < D; d += GROUP) {
      Real g = Real(0);
      const int c1 = pdf_cptr[d + 1];
      for (int c = pdf_cptr[d]; c < c1; ++c) g += sl[c];
      switch (mode) {
        case kPostNegate: prow[d] = -g; break;
        case kPostAdd: prow[d] = old[d] + g; break;
        case kPostSubtract: prow[d] = old[d] - g; break;
        default: prow[d] = g;
      }
    }
  };

  for (int s = tid; s < S; s += GROUP) rbuf[(T & 1) * S_pad + s] = fin[s] * (Real(1) + lam);
  issue_row(T - 1);
  issue_row(T - 2);
  issue_alpha(T - 1);
  issue_post(T - 1);
  cp_async_commit();
  issue_row(T - 3);
  issue_alpha(T - 2);
  cp_async_commit();
  cp_async_wait<1>();
  row_max_part(T - 1);
  row_max_part(T - 2);
  gsync();
  compute_e(T - 1, false);
  gsync();

  for (int t = T; t >= 1; --t) {
    const int ct = t & 1, cp = ct ^ 1;
    Real ld = Real(0);
    if (t < T && lam > Real(0)) {
      Real dot = Real(0);
      for (int w = 0; w < NW; ++w) dot += part[ct * NW + w];
      ld = lam * dot;
    }
    const Real inv = Real(1) / scales[t - 1];
    if (t < T) flush_post(t, slots + (LARGE ? 0 : ct * NC_pad));
    if (LARGE) gsync();  // single slot buffer: flush before the next frame's partials
    if (t - 2 >= 0) compute_e(t - 2, false);
    issue_row(t - 4);
    issue_alpha(t - 3);
    issue_post(t - 2);
    cp_async_commit();

    const Real *bt = rbuf + ct * S_pad;
    const Real *e = ebuf + cp * D_pad;
    {
      Real *bn = rbuf + cp * S_pad;
      Real dp = Real(0);
      for (int s = tid; s < S; s += GROUP) {
        const int lo = __ldg(out_ptr + s), hi = __ldg(out_ptr + s + 1);
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
    {
      const Real *al = LARGE ? trellis + size_t(t - 1) * S_pad : aring + ((t - 1) % 3) * S_pad;
      Real *sl = slots + (LARGE ? 0 : cp * NC_pad);
      for (int c = tid; c < nch; c += GROUP) {
        const int lo = __ldg(ch_begin + c), hi = __ldg(ch_end + c);
        Real P = Real(0), Q = Real(0);
        for (int i = lo; i < hi; ++i) {
          const Real x = al[__ldg(pa_src + i)] * __ldg(pa_p + i);
          P = fma(x, bt[__ldg(pa_dst + i)], P);
          Q += x;
        }
        sl[c] = e[__ldg(ch_pdf + c)] * inv * (P + ld * Q);
      }
    }
    cp_async_wait<1>();
    row_max_part(t - 3);
    gsync();
  }
  cp_async_wait<0>();
  flush_post(0, slots);
}

// ---- host-side launcher --------------------------------------------------------
template <typename Real, int GROUP, int GPC, bool LARGE = false>
static int launch_group_impl(const FBArgs<Real> &a, cudaStream_t st) {
  const size_t per = group_smem_bytes<Real>(a.S_pad, a.D_pad, a.NC_pad, a.T_pad, GROUP, LARGE);
  const size_t smem = per * GPC;
  if (smem > size_t(kMaxSmem))
    return set_error(LFMMI_ERR_UNSUPPORTED, "utterance/graph too large for the group kernel (" +
                                                std::to_string(smem) + " B shared memory)");
  static bool configured = false;
  if (!configured) {
    int rc = check_cuda(cudaFuncSetAttribute(fb_group_kernel<Real, GROUP, GPC, LARGE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem),
                        "cudaFuncSetAttribute(group)");
    if (rc) return rc;
    configured = true;
  }
  const int grid = (a.B + GPC - 1) / GPC;
  fb_group_kernel<Real, GROUP, GPC, LARGE><<<grid, GROUP * GPC, smem, st>>>(a);
  return check_cuda(cudaGetLastError(), "fb_group_kernel launch");
}

template <typename Real>
int launch_group(const FBArgs<Real> &a, int group, cudaStream_t st) {
  switch (group) {
    case 32: {
      // Several utterances per CTA; fall back to fewer if shared memory is short.
      const size_t per = group_smem_bytes<Real>(a.S_pad, a.D_pad, a.NC_pad, a.T_pad, 32);
      if (per * 4 <= size_t(kMaxSmem)) return launch_group_impl<Real, 32, 4>(a, st);
      return launch_group_impl<Real, 32, 1>(a, st);
    }
    case 64: return launch_group_impl<Real, 64, 1>(a, st);
    case 128: return launch_group_impl<Real, 128, 1>(a, st);
    case 256: return launch_group_impl<Real, 256, 1>(a, st);
    case 512: return launch_group_impl<Real, 512, 1>(a, st);
    default: {
      const int rc = launch_group_impl<Real, 1024, 1>(a, st);
      // Graphs too large for the alpha ring (config 4: 20k states) stream alpha
      // from L2 instead; the gradient is then written, never read back.
      const bool reads_post = a.mode == kPostAdd || a.mode == kPostSubtract;
      if (rc == LFMMI_ERR_UNSUPPORTED && !reads_post)
        return launch_group_impl<Real, 1024, 1, true>(a, st);
      return rc;
    }
  }
}

template int launch_group<float>(const FBArgs<float> &, int, cudaStream_t);
template int launch_group<double>(const FBArgs<double> &, int, cudaStream_t);

}  // namespace lfmmi
