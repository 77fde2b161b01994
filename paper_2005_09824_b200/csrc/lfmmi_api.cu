// C-ABI entry points (include/lfmmi.h) + the f64 parity kernels.
//
// Dispatch of the fused forward-backward:
//   * graphs that fit the on-chip tile pack (the denominator) -> fb_tile_kernel
//     (one 1024-thread CTA per utterance, arc layout resident in shared memory);
//   * small graphs (numerators) -> fb_group_kernel with a warp-sized group;
//   * anything else -> fb_group_kernel with a CTA-sized group (arcs via L1/L2).
// chain_loss = denominator pass (grad = -gamma_den) + numerator pass
// (grad += gamma_num, zero rows if either side failed) + totals reduction.
//
// Parity path (f64): lfmmi_{forward,backward,posterior}_kernel mirror the
// numba kernels argument-for-argument with the reference's exact operation
// order (no FMA contraction) for bit-level parity with the reference tests.
#include <algorithm>
#include <string>
#include <type_traits>

#include "lfmmi_device.cuh"
#include "lfmmi_kernels.h"
#include "lfmmi_options.h"

namespace lfmmi {

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
  const int T = item_frames(lengths, b, T_max);
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
  const int T = item_frames(lengths, b, T_max);
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
  if (t >= item_frames(lengths, b, T_max) || fail[b] >= 0) return;
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

// Batch totals for chain_loss (loss.py:61-72), fixed-order reduction by one
// 256-thread block (block (0, 0) of combine_kernel).
__device__ void batch_totals(int B, const int *lengths, const double *num_lp,
                             const double *den_lp, const int *num_fail, const int *den_fail,
                             double *totals) {
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

inline int choose_group(int max_states) {
  const int want = (max_states + 2) / 3;
  int g = 32;
  while (g < want && g < 1024) g <<= 1;
  return g;
}

template <typename Real>
int run_fused(const lfmmi_graphs *graphs, const int64_t *row_map, int B, int T_max, int D,
              const void *L, const int *lengths, double leak, double floor, const void *leak_pi,
              void *work, size_t work_bytes, void *post, int mode, const int *other_fail,
              double *logp, int *fail, double *scale_logs, cudaStream_t st, bool packed,
              int64_t total_frames, const Real *E = nullptr, const Real *Em = nullptr,
              int reserve_sms = 0) {
  FBArgs<Real> a{};
  a.reserve_sms = reserve_sms;
  a.E = E;
  a.Em = Em;
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
  a.I_pad = pad4(std::max(1, graphs->max_arcs));
  a.packed = packed ? 1 : 0;
  {
    const long long tf = std::max<long long>(total_frames, 1);
    const long long stride = (std::max(1, int(graphs->max_states)) + 31) & ~31;
    a.sc_off = stride * tf;  // after the (round32-strided) trellis region
    a.sc_total = tf;
    a.sc_smem = 1;  // default: shared memory (the den XDB launcher may move them to HBM)
  }
  if (std::is_same<Real, float>::value) {  // f32 tile slots address replicated vectors
    a.rep_r = graphs->rep_r;
    a.r_stride = graphs->r_stride;
    a.rep_e = graphs->rep_e;
    a.e_stride = graphs->e_stride;
  } else {  // f64 tile slots use plain indices
    a.rep_r = 1;
    a.r_stride = a.S_pad;
    a.rep_e = 1;
    a.e_stride = a.D_pad;
  }
  if (work_bytes < size_t(a.S_pad) * sizeof(Real))
    return set_error(LFMMI_ERR_INVALID, "workspace too small");
  // Numerator-sized graphs (chains and thin lattices: few states, in-degree
  // <= 4): a warp group per utterance.  Larger or denser graphs — a 43-state
  // phone-bigram den (~1850 arcs), the 50-state toy den (in-degree up to 10) —
  // take the den kernels (forward | backward split: toy step 0.156 -> 0.069 ms).
  // The choice depends only on the graph batch's shape.
  const Options &opt = options();
  const bool small = graphs->max_states <= 512 && graphs->max_arcs <= opt.small_arcs &&
                     graphs->max_in_deg <= opt.small_indeg;
  if constexpr (std::is_same<Real, float>::value) {
    if (graphs->linear && opt.linear) {  // the reference's numerators: linear chains
      const int rc = launch_linear(a, graphs, st);
      if (rc != LFMMI_ERR_UNSUPPORTED) return rc;
    }
  }
  if (graphs->linear_only)
    return set_error(LFMMI_ERR_INVALID,
                     "a linear-chain graph handle (lfmmi_graphs_create_linear) runs in fp32 with "
                     "the uniform leak distribution and the linear option enabled");
  if (opt.tile) {
    const int rc = launch_tile<Real>(a, graphs, small, st);
    if (rc != LFMMI_ERR_UNSUPPORTED) return rc;
  }
  // Arc packs too large for shared memory: stream them from L2 (coalesced tiles).
  if (!small && opt.stream) {
    const int rc = launch_stream<Real>(a, graphs, st);
    if (rc != LFMMI_ERR_UNSUPPORTED) return rc;
  }
  if (!small) note_den_kernel("fb_group_kernel<1024>");
  return launch_group<Real>(a, small ? choose_group(graphs->max_states) : 1024, st);
}

}  // namespace lfmmi

using namespace lfmmi;

extern "C" size_t lfmmi_workspace_size(int32_t max_states, int64_t total_frames,
                                       int32_t precision) {
  const size_t es = precision == LFMMI_F64 ? 8 : 4;
  // Row stride round32(S): the stream kernel spills alpha in 32-state tile order;
  // + 2 Reals per frame for the per-frame scales and row maxima (tile kernel).
  const size_t stride = size_t((std::max(1, int(max_states)) + 31) & ~31);
  return (stride + 2) * size_t(std::max<int64_t>(total_frames, 1)) * es + 256;
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

static int forward_backward_impl(const lfmmi_graphs *graphs, const int64_t *row_map,
                                      int32_t batch, int32_t max_frames, int32_t num_pdfs,
                                      int32_t precision, const void *loglikes,
                                      const int32_t *lengths, double leak, double scale_floor,
                                      const void *leak_pi, int64_t total_frames, void *workspace,
                                      size_t workspace_bytes, void *posteriors,
                                      int32_t post_mode, const int32_t *other_fail,
                                      double *log_probs, int32_t *fail_frames,
                                      double *scale_logs, void *stream, bool packed,
                                      const float *E = nullptr, const float *Em = nullptr,
                                      int reserve_sms = 0) {
  int rc = check_common(graphs, batch, max_frames, num_pdfs, precision);
  if (rc) return rc;
  if (!row_map || !loglikes || !lengths || !workspace || !posteriors || !log_probs || !fail_frames)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_forward_backward: NULL device pointer");
  if (total_frames < 1 ||
      workspace_bytes < lfmmi_workspace_size(graphs->max_states, total_frames, precision))
    return set_error(LFMMI_ERR_INVALID, "workspace smaller than lfmmi_workspace_size(S_max, "
                                        "total_frames, precision)");
  if (post_mode < LFMMI_POST_WRITE || post_mode > LFMMI_POST_NEGATE)
    return set_error(LFMMI_ERR_INVALID, "unknown post_mode");
  if (!(leak >= 0.0) || !(scale_floor > 0.0))
    return set_error(LFMMI_ERR_INVALID, "leak must be >= 0 and scale_floor > 0");
  auto st = static_cast<cudaStream_t>(stream);
  if (precision == LFMMI_F64)
    return run_fused<double>(graphs, row_map, batch, max_frames, num_pdfs, loglikes, lengths, leak,
                             scale_floor, leak_pi, workspace, workspace_bytes, posteriors,
                             post_mode, other_fail, log_probs, fail_frames, scale_logs, st,
                             packed, total_frames);
  return run_fused<float>(graphs, row_map, batch, max_frames, num_pdfs, loglikes, lengths, leak,
                          scale_floor, leak_pi, workspace, workspace_bytes, posteriors, post_mode,
                          other_fail, log_probs, fail_frames, scale_logs, st, packed,
                          total_frames, E, Em, reserve_sms);
}


#define LFMMI_FB_PARAMS                                                                         \
  const lfmmi_graphs *graphs, const int64_t *row_map, int32_t batch, int32_t max_frames,      \
      int32_t num_pdfs, int32_t precision, const void *loglikes, const int32_t *lengths,      \
      double leak, double scale_floor, const void *leak_pi, int64_t total_frames,             \
      void *workspace, size_t workspace_bytes, void *posteriors, int32_t post_mode,           \
      const int32_t *other_fail, double *log_probs, int32_t *fail_frames, double *scale_logs, \
      void *stream
#define LFMMI_FB_ARGS                                                                        \
  graphs, row_map, batch, max_frames, num_pdfs, precision, loglikes, lengths, leak,          \
      scale_floor, leak_pi, total_frames, workspace, workspace_bytes, posteriors, post_mode, \
      other_fail, log_probs, fail_frames, scale_logs, stream

extern "C" int lfmmi_forward_backward(LFMMI_FB_PARAMS) {
  return forward_backward_impl(LFMMI_FB_ARGS, false);
}

extern "C" int lfmmi_forward_backward_packed(LFMMI_FB_PARAMS) {
  return forward_backward_impl(LFMMI_FB_ARGS, true);
}

// Bytes of workspace for lfmmi_chain_loss: both alpha trellises (the two
// passes run concurrently) + the numerator posteriors.
static size_t chain_ws_parts(const lfmmi_graphs *num, const lfmmi_graphs *den, int32_t batch,
                             int32_t max_frames, int32_t num_pdfs, int64_t total_frames,
                             int32_t precision, size_t *den_off, size_t *num_off,
                             size_t *gam_off, size_t *e_off = nullptr) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t es = precision == LFMMI_F64 ? 8 : 4;
  const size_t tf = size_t(std::max<int64_t>(total_frames, 1));
  const size_t den_b = al(lfmmi_workspace_size(den ? den->max_states : 1, int64_t(tf), precision));
  const size_t num_b = al(lfmmi_workspace_size(num ? num->max_states : 1, int64_t(tf), precision));
  const size_t gam_b = al(size_t(batch) * size_t(max_frames) * size_t(num_pdfs) * es);
  // fp32: the step's emissions E = exp(L - m) + row maxima (emit_kernel), sized
  // for the padded layout (>= the packed one)
  const size_t rows = std::max(size_t(batch) * size_t(max_frames), tf);
  const size_t e_b = precision == LFMMI_F32 ? al(rows * size_t(num_pdfs) * 4) + al(rows * 4) : 0;
  if (den_off) *den_off = 0;
  if (num_off) *num_off = den_b;
  if (gam_off) *gam_off = den_b + num_b;
  if (e_off) *e_off = den_b + num_b + gam_b;
  return den_b + num_b + gam_b + e_b + 256;
}

extern "C" size_t lfmmi_chain_loss_workspace_size(const lfmmi_graphs *numerators,
                                                  const lfmmi_graphs *denominator, int32_t batch,
                                                  int32_t max_frames, int32_t num_pdfs,
                                                  int64_t total_frames, int32_t precision) {
  return chain_ws_parts(numerators, denominator, batch, max_frames, num_pdfs, total_frames,
                        precision, nullptr, nullptr, nullptr);
}

// grad = (ok ? grad + gamma_num : 0) over valid rows; padded rows were zeroed
// by the denominator pass.  Float4-vectorised grid-stride loop.
template <typename Real>
__global__ void combine_kernel(bool packed, int B, int T_max, int D, const int *lengths,
                               const int *num_fail, const int *den_fail,
                               const Real *__restrict__ gnum, Real *__restrict__ grad,
                               const double *num_lp, const double *den_lp, double *totals) {
  if (totals != nullptr && blockIdx.x == 0 && blockIdx.y == 0)  // one launch for both
    batch_totals(B, lengths, num_lp, den_lp, num_fail, den_fail, totals);
  const size_t row_elems = size_t(T_max) * D;
  for (int b = blockIdx.y; b < B; b += gridDim.y) {
    const size_t n = size_t(item_frames(lengths, b, T_max)) * D;
    const bool ok = num_fail[b] < 0 && den_fail[b] < 0;
    size_t base = size_t(b) * row_elems;
    if (packed) {  // ragged rows: item b starts at sum_{j<b} T_j
      base = 0;
      for (int j = 0; j < b; ++j) base += size_t(lengths[j]) * D;
    }
    Real *g = grad + base;
    const Real *q = gnum + base;
    if constexpr (sizeof(Real) == 4) {
      // every item's rows start 16-byte aligned when D % 4 == 0 (and the bases are)
      if ((D & 3) == 0 && ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(q)) & 15) == 0) {
        float4 *g4 = reinterpret_cast<float4 *>(g);
        const float4 *q4 = reinterpret_cast<const float4 *>(q);
        for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (n >> 2);
             i += size_t(gridDim.x) * blockDim.x) {
          float4 v = g4[i];
          const float4 u = q4[i];
          if (ok) {
            v.x += u.x;
            v.y += u.y;
            v.z += u.z;
            v.w += u.w;
          } else {
            v = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          g4[i] = v;
        }
        continue;
      }
    }
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
      g[i] = ok ? g[i] + q[i] : Real(0);
  }
}

// Emissions of one step (forward_backward.py:120-130): per valid row
// m = max_d L (NaN-propagating) and E = exp(L - m), one warp per row.  The
// passes that take E gather it instead of recomputing row maxima and exps
// every frame of every recursion.
__global__ void __launch_bounds__(256) emit_kernel(const float *__restrict__ L, const int *lengths,
                                                   int T_max, int D, int packed, long long rows,
                                                   float *__restrict__ E, float *__restrict__ Em) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += nw) {
    if (!packed && int(r % T_max) >= item_frames(lengths, int(r / T_max), T_max)) continue;
    const float *x = L + r * D;
    float *e = E + r * D;
    float m = -INFINITY;
    if ((D & 3) == 0) {
      const float4 *x4 = reinterpret_cast<const float4 *>(x);
      for (int c = lane; c < (D >> 2); c += 32) {
        const float4 v = x4[c];
        m = nan_max(nan_max(m, v.x), nan_max(nan_max(v.y, v.z), v.w));
      }
      m = warp_max(m);
      float4 *e4 = reinterpret_cast<float4 *>(e);
      for (int c = lane; c < (D >> 2); c += 32) {
        const float4 v = x4[c];
        e4[c] = make_float4(expf(v.x - m), expf(v.y - m), expf(v.z - m), expf(v.w - m));
      }
    } else {
      for (int d = lane; d < D; d += 32) m = nan_max(m, x[d]);
      m = warp_max(m);
      for (int d = lane; d < D; d += 32) e[d] = expf(x[d] - m);
    }
    if (lane == 0) Em[r] = m;
  }
}

int lfmmi::launch_emit(const float *L, const int *lengths, int B, int T_max, int D, bool packed,
                       int64_t rows, float *E, float *Em, cudaStream_t st) {
  (void)B;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long want = (rows + 7) / 8;  // 8 rows (warps) per 256-thread block
  const int grid = int(std::max<long long>(1, std::min<long long>(want, 8LL * sms)));
  emit_kernel<<<grid, 256, 0, st>>>(L, lengths, T_max, D, packed ? 1 : 0, rows, E, Em);
  return check_cuda(cudaGetLastError(), "emit_kernel launch");
}

namespace {
thread_local int32_t g_launches = 0;
struct AuxStream {
  cudaStream_t aux = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
// One auxiliary stream + fork/join events per (host thread, device): concurrent
// lfmmi_chain_loss calls from different threads never share event objects.
AuxStream &aux_for_device() {
  static thread_local AuxStream per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  AuxStream &a = per_dev[dev & 63];
  if (!a.aux) {
    cudaStreamCreateWithFlags(&a.aux, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming);
  }
  return a;
}
}  // namespace

extern "C" int32_t lfmmi_last_launch_count(void) { return g_launches; }

namespace {
thread_local const char *g_den_kernel = "";
thread_local const char *g_kernel = "";
}
void lfmmi::note_kernel(const char *name) { g_kernel = name; }
void lfmmi::note_den_kernel(const char *name) { g_den_kernel = g_kernel = name; }
extern "C" const char *lfmmi_last_den_kernel(void) { return g_den_kernel; }
extern "C" const char *lfmmi_last_kernel(void) { return g_kernel; }

static int chain_loss_impl(const lfmmi_graphs *numerators, const int64_t *num_row_map,
                                const lfmmi_graphs *denominator, const int64_t *den_row_map,
                                int32_t batch, int32_t max_frames, int32_t num_pdfs,
                                int32_t precision, const void *loglikes, const int32_t *lengths,
                                double leak, double scale_floor, const void *num_leak_pi,
                                const void *den_leak_pi, int64_t total_frames, void *workspace,
                                size_t workspace_bytes, void *grad, double *num_log_probs,
                                double *den_log_probs,
                                int32_t *num_fail, int32_t *den_fail, double *totals,
                                void *stream, bool packed) {
  if (!numerators || !denominator)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_chain_loss: NULL graph handle");
  size_t den_off, num_off, gam_off, e_off;
  if (total_frames < 1 ||
      workspace_bytes < chain_ws_parts(numerators, denominator, batch, max_frames, num_pdfs,
                                       total_frames, precision, &den_off, &num_off, &gam_off,
                                       &e_off))
    return set_error(LFMMI_ERR_INVALID, "workspace smaller than lfmmi_chain_loss_workspace_size");
  char *ws = static_cast<char *>(workspace);
  const size_t num_bytes = gam_off - num_off, den_bytes = num_off - den_off;
  const float *E = nullptr, *Em = nullptr;
  auto st = static_cast<cudaStream_t>(stream);
  int rc = check_common(denominator, batch, max_frames, num_pdfs, precision);
  if (rc) return rc;
  rc = check_common(numerators, batch, max_frames, num_pdfs, precision);
  if (rc) return rc;
  if (!num_row_map || !den_row_map || !loglikes || !lengths || !grad || !num_log_probs ||
      !den_log_probs || !num_fail || !den_fail)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_chain_loss: NULL device pointer");
  if (!(leak >= 0.0) || !(scale_floor > 0.0))
    return set_error(LFMMI_ERR_INVALID, "leak must be >= 0 and scale_floor > 0");
  AuxStream &ax = aux_for_device();
  // Numerator pass beside the denominator pass (auxiliary stream): the split
  // denominator leaves it 6 SMs; when the denominator batch fills every SM
  // (sweep: 1024 utterances) the numerator warps run in its tail, which still
  // measured better than running them first (sweep step 30.6 vs 31.4 ms).
  // Option serial: 0 concurrent (default), 1 numerators first, -1 serial only
  // when B > 2 x SMs.
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // SMs the split denominator leaves to the concurrent numerator pass, by the
  // numerators' size (their per-utterance latency grows with the states per
  // lane).  Sweep at B = 128 (S up to 501): step 5.54 / 5.18 / 4.00 / 4.23 /
  // 4.55 ms with 71 / 68 / 64 / 60 / 56 clusters (6 / 12 / 20 / 28 / 36 SMs left).
  const int ns = numerators->max_states;
  const int num_reserve = ns <= 128 ? 6 : ns <= 256 ? 10 : 20;
  const int ser_opt = options().serial;
  const bool serial = ser_opt > 0 || (ser_opt < 0 && batch > 2 * sms);
  // Emissions once per step, shared by the passes that take them (the linear
  // numerator kernel and the split denominator kernel).  Option emit: 1 (auto)
  // skips it when the denominator's arc pack cannot sit in shared memory (its
  // L2-streamed kernels exponentiate their own rows; the numerators then take
  // the one-warp linear kernel, in the den's tail: biphone step 7.04 -> 6.79
  // ms), 2 always, 0 never.
  const int emit_opt = options().emit;
  const bool den_smem =
      denominator->tileable &&
      size_t(std::max(denominator->max_tf_slots, denominator->max_tb_slots)) * 10 <=
          size_t(kMaxSmem);
  if (precision == LFMMI_F32 && (emit_opt >= 2 || (emit_opt == 1 && den_smem))) {
    const size_t rows = packed ? size_t(total_frames) : size_t(batch) * size_t(max_frames);
    float *e = reinterpret_cast<float *>(ws + e_off);
    float *em = e + ((rows * size_t(num_pdfs) * 4 + 255) & ~size_t(255)) / 4;
    rc = launch_emit(static_cast<const float *>(loglikes), lengths, batch, max_frames, num_pdfs,
                     packed, int64_t(rows), e, em, st);
    if (rc) return rc;
    E = e;
    Em = em;
  }
  auto num_pass = [&](cudaStream_t s) {
    return forward_backward_impl(numerators, num_row_map, batch, max_frames, num_pdfs, precision,
                                 loglikes, lengths, leak, scale_floor, num_leak_pi, total_frames,
                                 ws + num_off, num_bytes, ws + gam_off, LFMMI_POST_WRITE, nullptr,
                                 num_log_probs, num_fail, nullptr, s, packed, E, Em);
  };
  auto den_pass = [&](cudaStream_t s) {
    const int rc = forward_backward_impl(
        denominator, den_row_map, batch, max_frames, num_pdfs, precision, loglikes, lengths, leak,
        scale_floor, den_leak_pi, total_frames, ws + den_off, den_bytes, grad, LFMMI_POST_NEGATE,
        nullptr, den_log_probs, den_fail, nullptr, s, packed, E, Em, num_reserve);
    note_den_kernel(g_kernel);  // whichever family the denominator took (incl. small dens)
    return rc;
  };
  if (serial) {
    rc = num_pass(st);
    if (rc) return rc;
    rc = den_pass(st);
    if (rc) return rc;
  } else {
    // The denominator is launched first so its CTAs claim whole SMs; the
    // numerator warps fill the SMs it leaves free.  (A highest-priority stream
    // for the denominator measured no better at B = 1024 and worse at B = 128:
    // sweep 28.83 vs 28.76 ms, sweep B = 128 4.33 vs 3.89 ms.)
    rc = check_cuda(cudaEventRecord(ax.fork, st), "cudaEventRecord(fork)");
    if (rc) return rc;
    rc = den_pass(st);
    if (rc) return rc;
    rc = check_cuda(cudaStreamWaitEvent(ax.aux, ax.fork, 0), "cudaStreamWaitEvent(fork)");
    if (rc) return rc;
    rc = num_pass(ax.aux);
    if (rc) return rc;
    rc = check_cuda(cudaEventRecord(ax.join, ax.aux), "cudaEventRecord(join)");
    if (rc) return rc;
    rc = check_cuda(cudaStreamWaitEvent(st, ax.join, 0), "cudaStreamWaitEvent(join)");
    if (rc) return rc;
  }
  {
    const dim3 grid(std::max(1, std::min(32, (max_frames * num_pdfs + 4095) / 4096)),
                    std::min(batch, 4096));
    if (precision == LFMMI_F64)
      combine_kernel<double><<<grid, 256, 0, st>>>(packed, batch, max_frames, num_pdfs, lengths, num_fail,
                                                   den_fail,
                                                   reinterpret_cast<const double *>(ws + gam_off),
                                                   static_cast<double *>(grad), num_log_probs,
                                                   den_log_probs, totals);
    else
      combine_kernel<float><<<grid, 256, 0, st>>>(packed, batch, max_frames, num_pdfs, lengths, num_fail,
                                                  den_fail,
                                                  reinterpret_cast<const float *>(ws + gam_off),
                                                  static_cast<float *>(grad), num_log_probs,
                                                  den_log_probs, totals);
    rc = check_cuda(cudaGetLastError(), "combine_kernel launch");
    if (rc) return rc;
  }
  g_launches = rc == LFMMI_OK ? (E ? 4 : 3) : 0;  // [emit,] den, num, combine (+ totals)
  return rc;
}


#define LFMMI_CL_PARAMS                                                                        \
  const lfmmi_graphs *numerators, const int64_t *num_row_map, const lfmmi_graphs *denominator, \
      const int64_t *den_row_map, int32_t batch, int32_t max_frames, int32_t num_pdfs,         \
      int32_t precision, const void *loglikes, const int32_t *lengths, double leak,            \
      double scale_floor, const void *num_leak_pi, const void *den_leak_pi,                    \
      int64_t total_frames, void *workspace, size_t workspace_bytes, void *grad,               \
      double *num_log_probs, double *den_log_probs, int32_t *num_fail, int32_t *den_fail,      \
      double *totals, void *stream
#define LFMMI_CL_ARGS                                                                         \
  numerators, num_row_map, denominator, den_row_map, batch, max_frames, num_pdfs, precision,  \
      loglikes, lengths, leak, scale_floor, num_leak_pi, den_leak_pi, total_frames, workspace, \
      workspace_bytes, grad, num_log_probs, den_log_probs, num_fail, den_fail, totals, stream

extern "C" int lfmmi_chain_loss(LFMMI_CL_PARAMS) { return chain_loss_impl(LFMMI_CL_ARGS, false); }

extern "C" int lfmmi_chain_loss_packed(LFMMI_CL_PARAMS) {
  return chain_loss_impl(LFMMI_CL_ARGS, true);
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
