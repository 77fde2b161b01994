// fb_stream_kernel — forward-backward for graphs whose arc packs do not fit in
// shared memory (20k states / 200k arcs / 2000 pdfs;
// config 3: 3k states / 30k arcs).  One 1024-thread CTA — or a 2-CTA thread
// block cluster on two SMs (CL = 2, when the batch leaves SMs idle) — per
// utterance, whole time loop on chip, one (cluster) barrier per frame.
// With CL = 2 each CTA owns every other state tile; new alpha/beta values,
// normaliser partials and posterior bins are exchanged through distributed
// shared memory (st.shared::cluster), so both CTAs hold full columns.
//
//   shared memory : alpha/beta columns (ping-pong, fp32), two emission rows,
//                   two per-pdf posterior accumulators, scales, row maxima;
//   L2 (shared by every CTA, the graph is broadcast) : the stream packs —
//                   32-state tiles sorted by degree, slot j of lane l at
//                   base + 32 j + l as {index | pdf << 15, fp32 prob}, so each
//                   warp-wide slot load is one coalesced 256-byte request;
//   registers     : the next two log-likelihood rows (2 values per thread for
//                   D <= 2048), prefetched one frame ahead;
//   HBM           : the alpha trellis, spilled in the BACKWARD pack's state
//                   order so the backward reads it back coalesced.
//
// Semantics are those of the reference: forward
// _kernels.py:54-122, backward _kernels.py:125-191, posteriors
// _kernels.py:194-224 (here: every arc term alpha*p*e*beta in [0, 1] is
// quantised to 2^-28 and added to its pdf's bin with a native 32-bit
// shared-memory integer atomic — integer sums are order-independent, so the
// result is deterministic; the absolute error is <= n * 2^-29 for a pdf with
// n arcs, e.g. ~2e-7 at 100 arcs/pdf, far inside the 1e-4 gradient bar;
// fp32 atomicAdd would compile to a CAS loop on sm_100a),
// emissions forward_backward.py:120-130, log-probability
// forward_backward.py:206-212.  Uniform leak distribution only.
#include "lfmmi_device.cuh"
#include "lfmmi_kernels.h"
#include "lfmmi_options.h"
#include "lfmmi_ring.cuh"
#include "lfmmi_tile_common.cuh"

#include <cooperative_groups.h>

#include <cstdlib>
#include <string>

namespace cg = cooperative_groups;

namespace lfmmi {

namespace {

constexpr int kMaxD = 2048;  // log-likelihood row held in registers: kMaxD / NT per thread
constexpr float kPostScale = 268435456.f;  // 2^28: posterior bins in uint32 fixed point
constexpr int kRingRows = 8;               // slot rows per TMA chunk (8 x 256 B = 2 KB)
constexpr int kRingSlots = 2;              // chunks per warp in flight / being read
constexpr int kRingChunks = 64;            // chunk table entries per warp (per frame)

struct StreamLayout {
  unsigned vec, ebuf, bins, scales, shifts, part, mpart, ring, bars, ctab, total;
  int nslot;  // TMA ring slots per warp (0: slot rows read straight from L2)
};

__host__ __device__ inline StreamLayout stream_layout(int S32, int D_pad, int T_pad, int NW = 0,
                                                      int nslot = 0) {
  StreamLayout l;
  l.nslot = nslot;
  unsigned o = 512;  // scratch: 32 doubles + 32 int64
  auto take = [&](unsigned bytes) {
    const unsigned at = o;
    o = (o + bytes + 15u) & ~15u;
    return at;
  };
  l.vec = take(2u * S32 * 4u);
  l.ebuf = take(2u * D_pad * 4u);
  l.bins = take(2u * D_pad * 4u);  // uint32 fixed point (kPostScale)
  l.scales = take(unsigned(T_pad) * 4u);
  l.shifts = take(unsigned(T_pad) * 4u);
  l.part = take(2u * 64u * 4u);
  l.mpart = take(2u * 32u * 4u);
  l.ring = take(unsigned(NW) * unsigned(nslot) * kRingRows * 256u);
  l.bars = take(unsigned(NW) * unsigned(nslot) * 8u);
  l.ctab = take(nslot ? unsigned(NW) * kRingChunks * 8u : 0u);
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

}  // namespace

template <int NT, int CL, bool RING>
__global__ void __launch_bounds__(NT, 1024 / NT)
    fb_stream_kernel(const FBArgs<float> a, int S32, const StreamLayout lay) {
  constexpr int NW = NT / 32;
  constexpr int kEPT = kMaxD / NT;  // log-likelihood elements per thread
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x / CL;
  const int rank = CL > 1 ? int(cg::this_cluster().block_rank()) : 0;
  double *dscr = reinterpret_cast<double *>(smem);
  long long *lscr = reinterpret_cast<long long *>(smem + 256);
  float *vec = reinterpret_cast<float *>(smem + lay.vec);
  float *ebuf = reinterpret_cast<float *>(smem + lay.ebuf);
  unsigned *bins = reinterpret_cast<unsigned *>(smem + lay.bins);
  float *scales = reinterpret_cast<float *>(smem + lay.scales);
  float *shifts = reinterpret_cast<float *>(smem + lay.shifts);
  float *part = reinterpret_cast<float *>(smem + lay.part);
  float *mpart = reinterpret_cast<float *>(smem + lay.mpart);
  // Peer CTA's copies (CL = 2); with CL = 1 they alias our own buffers.
  float *vec_p = vec, *part_p = part;
  unsigned *bins_p = bins;
  if constexpr (CL > 1) {
    cg::cluster_group cl = cg::this_cluster();
    vec_p = cl.map_shared_rank(vec, rank ^ 1);
    part_p = cl.map_shared_rank(part, rank ^ 1);
    bins_p = cl.map_shared_rank(bins, rank ^ 1);
  }

  const int T = item_frames(a.lengths, b, a.T_max);
  if (T <= 0) {  // zero-length item (host APIs reject it): failed, no frames touched
    if (rank == 0) {
      if (!a.packed)
        for (size_t i = threadIdx.x; i < size_t(a.T_max) * a.D; i += NT)
          a.post[size_t(b) * a.T_max * a.D + i] = 0.f;
      if (threadIdx.x == 0) {
        a.logp[b] = NAN;
        a.fail[b] = 0;
      }
    }
    return;  // both CTAs of a cluster see the same T
  }
  const int D = a.D, D_pad = a.D_pad;
  const int row = int(a.row_map[b]);
  const int *desc = a.g.desc + row * kDescInts;
  const int S = desc[kS], init = desc[kInit];
  const int ntiles = desc[kSTiles], stoff = desc[kSTileOff];
  const float *fin = a.g.fin32 + desc[kStateOff];
  const float *Lb = a.L + size_t(b) * a.T_max * D;
  float *post_b = a.post + size_t(b) * a.T_max * D;
  const bool negate = a.mode == kPostNegate;
  const bool other_failed = a.other_fail != nullptr && a.other_fail[b] >= 0;
  const int *finfo = a.g.sf_info + size_t(stoff) * 32, *binfo = a.g.sb_info + size_t(stoff) * 32;
  const int *ftrips = a.g.sf_trips + stoff, *fbase = a.g.sf_base + stoff;
  const int *btrips = a.g.sb_trips + stoff, *bbase = a.g.sb_base + stoff;
  const uint2 *fwp = a.g.sf_wp + desc[kSfSlotOff], *bwp = a.g.sb_wp + desc[kSbSlotOff];
  auto gsync = [] { __syncthreads(); };
  auto csync = [] {  // frame barrier: CTA, or cluster with release/acquire on DSMEM
    if constexpr (CL > 1)
      cg::this_cluster().sync();
    else
      __syncthreads();
  };
  auto put2 = [&](float *own, float *peer, int i, float v) {
    own[i] = v;
    if (CL > 1) peer[i] = v;
  };

  // Sum of the per-warp partials of every CTA of the cluster, same order in each.
  auto part_total = [&](const float *v) {
    float x = lane < NW ? v[lane] : 0.f;
    if (CL > 1) x += lane < NW ? v[32 + lane] : 0.f;
    return warp_sum(x);
  };
  long long off = 0;
  for (int j = tid; j < b; j += NT) off += a.lengths[j];
  off = warp_sum(off);
  if (lane == 0) lscr[warp] = off;
  gsync();
  long long item_off = 0;
  for (int w = 0; w < NW; ++w) item_off += lscr[w];
  float *trellis = a.work + item_off * S32;  // rows in backward-pack state order
  if (a.packed) {  // ragged layout: item b's rows start at sum_{j<b} T_j
    Lb = a.L + size_t(item_off) * D;
    post_b = a.post + size_t(item_off) * D;
  }
  const float upi = float(1.0 / double(S));
  const float lam = a.leak;

  if (!a.packed)
    for (size_t i = tid; i < size_t(a.T_max - T) * D; i += NT) post_b[size_t(T) * D + i] = 0.f;

  // ---- log-likelihood rows in registers (two frames ahead) ----------------------
  float rn[kEPT], rn2[kEPT];
  auto load_row = [&](int t, float *r) {
#pragma unroll
    for (int j = 0; j < kEPT; ++j) {
      const int d = tid + j * NT;
      r[j] = (t >= 0 && t < T && d < D) ? __ldg(Lb + size_t(t) * D + d) : -INFINITY;
    }
  };
  auto max_part = [&](int t, const float *r) {  // warp maxima of row t -> mpart[t & 1]
    float m = r[0];
#pragma unroll
    for (int j = 1; j < kEPT; ++j) m = nan_max(m, r[j]);
    m = warp_max(m);
    if (lane == 0) mpart[(t & 1) * 32 + warp] = m;
  };
  auto compute_e = [&](int t, const float *r, bool record) {
    float m = lane < NW ? mpart[(t & 1) * 32 + lane] : -INFINITY;
    m = warp_max(m);
#pragma unroll
    for (int j = 0; j < kEPT; ++j) {
      const int d = tid + j * NT;
      if (d < D) ebuf[(t & 1) * D_pad + d] = expf(r[j] - m);
    }
    if (record && tid == 0) shifts[t] = m;
  };

  // This warp's tiles are rank + CL*warp + CL*NW*i, i < ntw; lane i keeps tile i's
  // slot count and base (read once per phase, broadcast by shuffles per tile).
  const int tile0 = rank + CL * warp, tstep = CL * NW;
  const int ntw = tile0 < ntiles ? (ntiles - tile0 + tstep - 1) / tstep : 0;
  int my_trips = 0, my_base = 0;
  auto load_meta = [&](const int *trips_arr, const int *base_arr) {
    const int tl = tile0 + tstep * lane;
    my_trips = lane < ntw ? __ldg(trips_arr + tl) : 0;
    my_base = lane < ntw ? __ldg(base_arr + tl) : 0;
  };

  // ---- TMA slot ring (RING): lfmmi_ring.cuh ---------------------------------------
  SlotRing<kRingSlots, kRingRows, kRingChunks> ring;
  auto begin_phase = [&](const uint2 *pk, int frames) {
    if constexpr (RING) ring.begin(pk, ntw, my_trips, my_base, frames);
  };
  auto drain = [&]() {  // wait for copies still in flight (early exit of a phase)
    if constexpr (RING) ring.drain();
  };
  // Arc rows [0, trips) of one tile: body(w) per slot word (this lane's arc).
  auto tile_rows = [&](const uint2 *sp, int trips, auto &&body) {
    if constexpr (RING) {
      ring.rows(trips, body);
    } else {
      // 8 slot-row loads in flight per lane before their arc bodies (L2 latency)
      int j = 0;
      for (; j + 8 <= trips; j += 8) {
        uint2 w[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) w[r] = ldg_slot(sp + 32 * (j + r));
#pragma unroll
        for (int r = 0; r < 8; ++r) body(w[r]);
      }
      for (; j < trips; ++j) body(ldg_slot(sp + 32 * j));
    }
  };
  if constexpr (RING) {
    ring.init(smem + lay.ring, smem + lay.bars, smem + lay.ctab, warp);
    decltype(ring)::init_barriers(smem + lay.bars, NW, tid);
    gsync();
  }

  // ---- forward ---------------------------------------------------------------------
  load_meta(ftrips, fbase);
  begin_phase(fwp, T);
  for (int s = tid; s < S32; s += NT) vec[s] = (s == init) ? 1.f : 0.f;
  {
    float r0[kEPT];
    load_row(0, r0);
    load_row(1, rn);
    load_row(2, rn2);
    max_part(0, r0);
    max_part(1, rn);
    gsync();
    compute_e(0, r0, true);
    csync();
  }
  float inv2 = 1.f, leakc = 0.f;
  int fail_at = -1;
  for (int k = 0; k < T; ++k) {
    const int cur = k & 1, nxt = cur ^ 1;
    if (k > 0) {
      const float t0 = part_total(part + cur * 64);
      float t2 = t0;
      leakc = 0.f;
      if (lam > 0.f && t0 > 0.f) {
        leakc = lam * t0;
        t2 = t0 + leakc;
      }
      if (!(t2 >= a.floor_eff) || isinf(t2)) {
        fail_at = k - 1;
        drain();
        break;
      }
      inv2 = __frcp_rn(t2);
      if (tid == 0) scales[k - 1] = t2;
    }
    {  // spill the normalised alpha_k in backward-pack order (coalesced both ways)
      const float *r = vec + cur * S32;
      float *arow = trellis + size_t(k) * S32;
      const float lu = leakc * upi;
      for (int q = tid; q < ntiles * 32; q += NT) {  // this CTA's tiles: q / 32 == rank mod CL
        const int p = CL > 1 ? ((q >> 5) * CL + rank) * 32 + (q & 31) : q;
        if (p >= ntiles * 32) break;
        const int s = __ldg(binfo + p);
        if (s >= 0) arow[p] = (r[s] + lu) * inv2;
      }
    }
    if (k + 1 < T) compute_e(k + 1, rn, true);
#pragma unroll
    for (int j = 0; j < kEPT; ++j) rn[j] = rn2[j];
    load_row(k + 3, rn2);
    {
      const uint32_t e32 = smem_u32(ebuf + cur * D_pad), r32 = smem_u32(vec + cur * S32);
      float *rnew = vec + nxt * S32, *rnew_p = vec_p + nxt * S32;
      const bool last = (k + 1 == T);
      float psum = 0.f;
      int s_next = ntw > 0 ? __ldg(finfo + tile0 * 32 + lane) : -1;
      for (int i = 0; i < ntw; ++i) {
        const int tile = tile0 + tstep * i;
        const int s = s_next;
        if (i + 1 < ntw) s_next = __ldg(finfo + (tile + tstep) * 32 + lane);
        const int trips = __shfl_sync(kFull, my_trips, i);
        const uint2 *sp = fwp + __shfl_sync(kFull, my_base, i) + lane;
        float A = 0.f, Bs = 0.f;
        tile_rows(sp, trips, [&](const uint2 w) {
          const float q = __uint_as_float(w.y) * lds_f(e32 + ((w.x >> 15) << 2));
          A = fmaf(q, lds_f(r32 + ((w.x & 0x7FFFu) << 2)), A);
          Bs += q;
        });
        if (s >= 0) {
          float raw = inv2 * (A + leakc * upi * Bs);
          if (last) raw *= fin[s];
          put2(rnew, rnew_p, s, raw);
          psum += raw;
        }
      }
      psum = warp_sum(psum);
      if (lane == 0) put2(part, part_p, nxt * 64 + rank * 32 + warp, psum);
    }
    max_part(k + 2, rn);
    csync();
  }
  if (fail_at < 0) {
    const float t0 = part_total(part + (T & 1) * 64);
    float t2 = t0;
    if (lam > 0.f && t0 > 0.f) t2 = t0 + lam * t0;
    if (!(t2 >= a.floor_eff) || isinf(t2))
      fail_at = T - 1;
    else if (tid == 0)
      scales[T - 1] = t2;
  }
  if (fail_at >= 0) {
    for (int k = fail_at + 1 + warp; k < T; k += NW) {
      float m = -INFINITY;
      for (int d = lane; d < D; d += 32) m = nan_max(m, Lb[size_t(k) * D + d]);
      m = warp_max(m);
      if (lane == 0) shifts[k] = m;
    }
    for (int k = fail_at + tid; k < T; k += NT) scales[k] = 1.f;
  }
  gsync();
  {
    double acc = 0.0;
    for (int k = tid; k < T; k += NT) {
      const double v = log(double(scales[k])) + double(shifts[k]);
      acc += v;
      if (a.scale_logs && rank == 0) a.scale_logs[size_t(b) * a.T_max + k] = v;
    }
    if (a.scale_logs && rank == 0)
      for (int k = T + tid; k < a.T_max; k += NT) a.scale_logs[size_t(b) * a.T_max + k] = 0.0;
    acc = warp_sum(acc);
    if (lane == 0) dscr[warp] = acc;
    gsync();
    if (tid == 0 && rank == 0) {
      double tot = 0.0;
      for (int w = 0; w < NW; ++w) tot += dscr[w];
      a.logp[b] = fail_at >= 0 ? NAN : tot;
      a.fail[b] = fail_at;
    }
  }
  if (fail_at >= 0 || other_failed) {
    for (size_t i = tid + size_t(rank) * NT; i < size_t(T) * D; i += size_t(NT) * CL)
      post_b[i] = 0.f;
    csync();  // no CTA leaves while its peer may still address its shared memory
    return;
  }

  // ---- backward + posteriors ------------------------------------------------------
  load_meta(btrips, bbase);
  begin_phase(bwp, T);
  for (int d = tid; d < 2 * D_pad; d += NT) bins[d] = 0u;
  for (int s = tid; s < S32; s += NT) vec[(T & 1) * S32 + s] = s < S ? fin[s] * (1.f + lam) : 0.f;
  csync();  // peers' bins are zero before anyone accumulates
  {
    float r0[kEPT];
    load_row(T - 1, r0);
    load_row(T - 2, rn);
    load_row(T - 3, rn2);
    max_part(T - 1, r0);
    max_part(T - 2, rn);
    gsync();
    compute_e(T - 1, r0, false);
    gsync();
  }
  auto flush = [&](int t) {  // gamma_t -> gradient row, then clear the bins
    unsigned *bn = bins + (t & 1) * D_pad, *bnp = bins_p + (t & 1) * D_pad;
    float *prow = post_b + size_t(t) * D;
    for (int d = tid * CL + rank; d < D; d += NT * CL) {  // this CTA's pdfs
      const unsigned q = CL > 1 ? bn[d] + bnp[d] : bn[d];
      const float g = float(double(q) * (1.0 / double(kPostScale)));
      prow[d] = negate ? -g : g;
      bn[d] = 0u;
      if (CL > 1) bnp[d] = 0u;
    }
  };
  for (int t = T; t >= 1; --t) {
    const int ct = t & 1, cp = ct ^ 1;
    float ld = 0.f;
    if (t < T && lam > 0.f) ld = lam * part_total(part + ct * 64);
    const float inv = __frcp_rn(scales[t - 1]);
    if (t < T) flush(t);  // bins of frame t (filled last iteration; other buffer than this one)
    if (t - 2 >= 0) compute_e(t - 2, rn, false);
#pragma unroll
    for (int j = 0; j < kEPT; ++j) rn[j] = rn2[j];
    load_row(t - 4, rn2);
    {
      const uint32_t b32 = smem_u32(vec + ct * S32), e32 = smem_u32(ebuf + cp * D_pad);
      float *bnew = vec + cp * S32, *bnew_p = vec_p + cp * S32;
      const float *arow = trellis + size_t(t - 1) * S32;  // alpha_{t-1}, backward-pack order
      const uint32_t bn32 = smem_u32(bins + cp * D_pad);
      float dp = 0.f;
      int s_next = -1;
      float a_next = 0.f;
      if (ntw > 0) {
        s_next = __ldg(binfo + tile0 * 32 + lane);
        a_next = arow[tile0 * 32 + lane];
      }
      for (int i = 0; i < ntw; ++i) {
        const int tile = tile0 + tstep * i;
        const int s = s_next;
        const float as = s >= 0 ? a_next * inv : 0.f;
        if (i + 1 < ntw) {  // next tile's state and alpha, one tile ahead
          s_next = __ldg(binfo + (tile + tstep) * 32 + lane);
          a_next = arow[(tile + tstep) * 32 + lane];
        }
        const int trips = __shfl_sync(kFull, my_trips, i);
        const uint2 *sp = bwp + __shfl_sync(kFull, my_base, i) + lane;
        float A = 0.f;
        tile_rows(sp, trips, [&](const uint2 w) {
          const float pr = __uint_as_float(w.y);
          const uint32_t pdf4 = (w.x >> 15) << 2;
          const float term = pr * lds_f(e32 + pdf4) * (lds_f(b32 + ((w.x & 0x7FFFu) << 2)) + ld);
          A += term;
          const unsigned q = __float2uint_rn(as * term * kPostScale);
          red_add_shared_nz(bn32 + pdf4, q);
        });
        if (s >= 0) {
          const float v = inv * A;
          put2(bnew, bnew_p, s, v);
          dp = fmaf(upi, v, dp);
        }
      }
      dp = warp_sum(dp);
      if (lane == 0) put2(part, part_p, cp * 64 + rank * 32 + warp, dp);
    }
    if (t - 3 >= 0) max_part(t - 3, rn);
    csync();
  }
  flush(0);
  csync();
}

template <typename Real>
int launch_stream(const FBArgs<Real> &, const lfmmi_graphs *, cudaStream_t) {
  return set_error(LFMMI_ERR_UNSUPPORTED, "stream kernel is fp32-only");
}

template <int NT, int CL, bool RING>
static int launch_stream_impl2(const FBArgs<float> &a, int S32, const StreamLayout &lay,
                               cudaStream_t st) {
  auto kern = fb_stream_kernel<NT, CL, RING>;
  note_den_kernel(NT == 1024 ? (CL == 2 ? (RING ? "fb_stream_kernel<1024,2> (TMA slot ring)"
                                                : "fb_stream_kernel<1024,2>")
                                        : (RING ? "fb_stream_kernel<1024,1> (TMA slot ring)"
                                                : "fb_stream_kernel<1024,1>"))
                             : (RING ? "fb_stream_kernel<512,2> (TMA slot ring)"
                                     : "fb_stream_kernel<512,2>"));
  static bool configured = false;
  if (!configured) {
    int rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kMaxSmem),
                        "cudaFuncSetAttribute(stream)");
    if (rc) return rc;
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.B * CL);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = lay.total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return check_cuda(cudaLaunchKernelEx(&cfg, kern, a, S32, lay), "fb_stream_kernel launch");
}

// TMA ring when its kRingSlots x 2 KB per warp fit next to the columns, else
// slot rows straight from L2.
template <int NT, int CL>
static int launch_stream_impl(const FBArgs<float> &a, const lfmmi_graphs *g, int S32,
                              const StreamLayout &base, cudaStream_t st) {
  constexpr int NW = NT / 32;
  // per warp and frame: <= ceil(tiles / (CL NW)) tiles of <= max_deg rows
  const int tiles_per_warp = (g->max_stiles + CL * NW - 1) / (CL * NW);
  const int max_deg = std::max(g->max_in_deg, g->max_out_deg);
  const bool fits = ring_chunks_needed(tiles_per_warp, max_deg, kRingRows) <= kRingChunks;
  if (options().stream_ring && fits) {
    const StreamLayout lay = stream_layout(S32, a.D_pad, a.T_pad, NW, kRingSlots);
    if (lay.total <= unsigned(kMaxSmem)) return launch_stream_impl2<NT, CL, true>(a, S32, lay, st);
  }
  return launch_stream_impl2<NT, CL, false>(a, S32, base, st);
}

template <>
int launch_stream<float>(const FBArgs<float> &a, const lfmmi_graphs *g, cudaStream_t st) {
  if (!g->streamable) return set_error(LFMMI_ERR_UNSUPPORTED, "graph has no stream pack");
  if (a.leak_pi) return set_error(LFMMI_ERR_UNSUPPORTED, "stream kernel: uniform leak only");
  if (a.D > kMaxD) return set_error(LFMMI_ERR_UNSUPPORTED, "stream kernel: D > 2048");
  if (a.mode != kPostWrite && a.mode != kPostNegate)
    return set_error(LFMMI_ERR_UNSUPPORTED, "stream kernel: WRITE / NEGATE modes only");
  const int S32 = (g->max_states + 31) & ~31;
  const StreamLayout lay = stream_layout(S32, a.D_pad, a.T_pad);
  if (lay.total > unsigned(kMaxSmem))
    return set_error(LFMMI_ERR_UNSUPPORTED,
                     "stream kernel needs " + std::to_string(lay.total) + " B shared memory");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Two SMs per utterance (2-CTA cluster of 1024-thread CTAs) while the batch
  // leaves SMs idle, else one 1024-thread CTA per utterance.  ("512x2" — two
  // half-utterance CTAs per SM — measured slower on biphone: 14.1 vs 12.4 ms.)
  // "split" (the default when it applies): the forward | backward split
  // (lfmmi_streamsplit.cu), slot rows from L2 with 8 row loads in flight per
  // lane — biphone 7.09 ms (split + TMA ring 7.68, 1024x1 + ring 8.42), large
  // 23.6 ms (1024x2 27.1).
  const std::string &want = options().stream_mode;
  if (want == "split") return launch_stream_split(a, g, st);
  if (want == "auto") {
    const int rc = launch_stream_split(a, g, st);
    if (rc != LFMMI_ERR_UNSUPPORTED) return rc;
  }
  std::string mode = want != "auto" ? want : (2 * a.B <= sms ? "1024x2" : "1024x1");
  if (mode == "1024x2") return launch_stream_impl<1024, 2>(a, g, S32, lay, st);
  if (mode == "512x2") return launch_stream_impl<512, 2>(a, g, S32, lay, st);
  return launch_stream_impl<1024, 1>(a, g, S32, lay, st);
}

template int launch_stream<double>(const FBArgs<double> &, const lfmmi_graphs *, cudaStream_t);

}  // namespace lfmmi
