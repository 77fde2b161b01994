// Process-wide dispatch / debug options of the library: ONE struct, parsed once
// from LFMMI_OPTIONS ("split=0,stream_mode=1024x1,...") on first use and
// changeable at run time through lfmmi_set_option (include/lfmmi.h).  Nothing
// else in the library reads the environment.
#pragma once

#include <string>

namespace lfmmi {

struct Options {
  // kernel families the dispatcher may pick (1 = allowed)
  int tile = 1;           // on-chip tile / split kernels
  int stream = 1;         // L2-streamed kernel (graphs beyond shared memory)
  int linear = 1;         // linear-chain numerator kernel
  int linear_split = 1;   // ... with forward | backward warps (chain loss, fp32)
  int linear_k16w = 2;    // ... the K = 16 class: warps per direction (2: 64 lanes x 8 states, 1: one warp)
  int linear_k16 = 0;     // ... batches with S > 256: 1 = one launch for every K, 0 = K <= 8 then K = 16
  int split = -1;         // denominator split kernel: -1 auto (B <= 2 x SMs), 0 off, 1 force
  int split_clusters = 0; // 0 = auto
  int split_h64 = 33;     // split midpoint in 64ths of T
  std::string stream_mode = "auto";  // "auto" | "1024x1" | "1024x2" | "512x2"
  int ssplit_ring = 0;   // stream split kernel: TMA slot ring (L2 rows measured faster)
  int stream_ring = 1;    // stream kernel: TMA slot ring when it fits (biphone 9.45 vs 9.96 ms)
  int num_group = 128;    // threads per utterance of the generic (tile) numerator kernel
  int small_arcs = 1024;  // graphs with <= 512 states, <= this many arcs per row AND in-degree
  int small_indeg = 4;    // <= small_indeg take the numerator-sized kernels; denser ones the den path
  int tile_persist = 0;  // den tile kernel, B > SMs: persistent CTAs over an in-kernel LPT
                         // (0 off, >= 2: force that many CTAs — tests)
  int tile_xdb = 1;       // den tile kernel: double-buffered posterior slots
  int serial = 0;         // chain_loss: numerator pass before the den pass (-1 auto: B > 2 x SMs)
  int emit = 1;           // chain_loss (fp32): emissions pre-pass shared by the passes
                          // (1 auto: not for dens beyond shared memory; 2 always; 0 never)
  int sched_iters = -1;   // bank-conflict local search moves per slot row (-1 auto)
  int chore_bias = 16;    // den warp lists: extra slot rows charged to the chore warps (pack time)
  int tile_g = 0;         // tile packs: lanes per state (0 auto, else forced power of 2; pack time)
  int debug = 0;          // layout / dispatch notes on stderr
  std::string profile;    // "" | "split" | "tile": per-frame cycle counters on stderr
};

// The current options (initialised from LFMMI_OPTIONS on first call).
Options &options();

}  // namespace lfmmi
