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

// Linear-chain graphs (every arc s -> s or s -> s+1, <= 1 of each per state;
// the reference's numerators): one warp per utterance, states in registers
// (lfmmi_linear.cu).  fp32, uniform leak; LFMMI_ERR_UNSUPPORTED (without
// launching) when not applicable.
int launch_linear(const FBArgs<float> &a, const lfmmi_graphs *g, cudaStream_t st);

// Forward | backward split of the L2-streamed kernel (lfmmi_streamsplit.cu):
// fp32, uniform leak, WRITE / NEGATE; LFMMI_ERR_UNSUPPORTED when not applicable.
int launch_stream_split(const FBArgs<float> &a, const lfmmi_graphs *g, cudaStream_t st);

// Emissions pre-pass (lfmmi_api.cu emit_kernel): E = exp(L - m), Em = m per valid row.
int launch_emit(const float *L, const int *lengths, int B, int T_max, int D, bool packed,
                int64_t rows, float *E, float *Em, cudaStream_t st);

}  // namespace lfmmi
