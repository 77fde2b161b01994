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

}  // namespace lfmmi
