// In-kernel longest-processing-time (LPT) assignment of a batch's utterances to
// persistent CTAs / clusters (fb_split_kernel, fb_streamsplit_kernel, the
// persistent fb_tile_kernel).  Every CTA computes the same assignment from the
// lengths alone, so no host sort, no atomics and no inter-CTA traffic: the
// utterances are ranked by length (longest first, ties by index) and each goes
// to the bin with the least load so far (load = frames + a per-item overhead),
// ties to the lowest bin.  Results never depend on the assignment (every
// utterance is computed the same way wherever it runs).
#pragma once

#include "lfmmi_device.cuh"

namespace lfmmi {

constexpr int kLptMaxBins = 160;  // >= SMs of a B200 (persistent tile kernel)
constexpr int kLptMaxItems = 64;  // utterances per bin (launchers guarantee B <= bins * this)

// All NT threads of the CTA call it.  scratch: 2 B ints of shared memory (free
// for the duration of the call); items: kLptMaxItems + 4 ints of shared memory,
// on return items[0] = count and items[4 + k] = the k-th utterance of bin
// `mine` in assignment order (longest first).
template <int NT>
__device__ void lpt_assign(const int *lengths, int B, int T_max, int nbins, int mine,
                           int overhead, int *scratch, int *items) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int *lens = scratch;
  int *order = scratch + B;
  for (int i = tid; i < B; i += NT) lens[i] = item_frames(lengths, i, T_max);
  __syncthreads();
  for (int i = tid; i < B; i += NT) {  // rank = #(longer) + #(equal, lower index)
    const int ti = lens[i];
    int r = 0;
    for (int j = 0; j < B; ++j) {
      const int tj = lens[j];
      r += (tj > ti) | ((tj == ti) & (j < i));
    }
    order[r] = i;
  }
  __syncthreads();
  if (warp == 0) {
    constexpr int W = (kLptMaxBins + 31) / 32;
    unsigned load[W] = {};
    int cnt[W] = {};
    int m = 0;
    for (int r = 0; r < B; ++r) {
      const int i = order[r];
      unsigned key = 0xFFFFFFFFu;  // (load << 8) | bin: least load, then lowest bin
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const int bin = lane + 32 * q;
        if (bin < nbins && cnt[q] < kLptMaxItems) key = min(key, (load[q] << 8) | unsigned(bin));
      }
      const int bin = int(__reduce_min_sync(kFull, key) & 255u);
#pragma unroll
      for (int q = 0; q < W; ++q)
        if (lane + 32 * q == bin) {
          load[q] += unsigned(lens[i] + overhead);
          ++cnt[q];
        }
      if (bin == mine) {
        if (lane == 0) items[4 + m] = i;
        ++m;
      }
    }
    if (lane == 0) items[0] = m;
  }
  __syncthreads();
}

}  // namespace lfmmi
