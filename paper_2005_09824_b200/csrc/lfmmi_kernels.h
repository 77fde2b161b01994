// Internal launcher declarations (host side).
#pragma once

#include "lfmmi_device.cuh"

namespace lfmmi {

constexpr int kMaxSmem = 227 * 1024;

// Extra posterior write modes used internally by chain_loss (see lfmmi.h).
constexpr int kPostWrite = LFMMI_POST_WRITE;        // p  = g
constexpr int kPostSubtract = LFMMI_POST_SUBTRACT;  // p -= g
constexpr int kPostAdd = LFMMI_POST_ADD;            // p += g
constexpr int kPostNegate = LFMMI_POST_NEGATE;      // p  = -g

template <typename Real>
int launch_group(const FBArgs<Real> &a, int group, cudaStream_t st);

// Returns LFMMI_ERR_UNSUPPORTED (without launching) when the graph batch does
// not fit the on-chip tile path, so the caller can fall back.
template <typename Real>
int launch_tile(const FBArgs<Real> &a, const lfmmi_graphs *graphs, bool warp_per_item,
                cudaStream_t st);

// Denominator forward-backward split over a 2-CTA cluster (forward CTA +
// backward CTA meeting at the midpoint; lfmmi_split.cu).  fp32, uniform leak,
// WRITE / NEGATE; LFMMI_ERR_UNSUPPORTED (without launching) when not applicable.
template <typename Real>
int launch_split(const FBArgs<Real> &a, const lfmmi_graphs *graphs, cudaStream_t st);

// L2-streamed forward-backward for graphs too large for the on-chip packs
// (lfmmi_stream.cu; fp32, uniform leak, WRITE/NEGATE).  LFMMI_ERR_UNSUPPORTED
// (without launching) when not applicable.
template <typename Real>
int launch_stream(const FBArgs<Real> &a, const lfmmi_graphs *graphs, cudaStream_t st);

// Fused LF-MMI loss (lfmmi_chain.cu): numerator + denominator + gradient in one CTA.
struct ChainArgs {
  DevGraphs den, num;
  const int64_t *den_row_map, *num_row_map;
  int B, T_max, D, D_pad, T_pad;
  int Sd_pad, Sn_pad;  // trellis row strides
  int rep_rd, r_strided, rep_rn, r_striden, rep_e, e_stride;
  const float *L;
  const int *lengths;
  float leak, floor_eff;
  float *trellis_d, *trellis_n;
  float *grad;
  double *num_lp, *den_lp;
  int *num_fail, *den_fail;
  double *totals;
  unsigned *counter;
  long long *prof;  // debug section timers (LFMMI_PROFILE), normally NULL
  int ablate;       // debug ablation bits (LFMMI_ABLATE, profiled launches only)
  int packed;       // ragged (sum_b T_b, D) loglikes / grad
};

struct ChainDims {
  int Fd, ntd, Xd;  // denominator: max slots per phase, tiles, posterior slots
  int Fn, ntn, Xn;  // numerator
};

int launch_chain(const ChainArgs &a, const ChainDims &m, cudaStream_t st);

}  // namespace lfmmi
