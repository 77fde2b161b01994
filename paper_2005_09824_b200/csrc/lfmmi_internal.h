// Internal declarations shared by the graph packer and the kernels.
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "lfmmi.h"

namespace lfmmi {

// Per-row descriptor ints (device array desc[num_rows * kDescInts]).
enum DescField : int {
  kS = 0,          // number of states
  kI = 1,          // number of arcs
  kInit = 2,       // initial state
  kStateOff = 3,   // offset into per-state arrays (finals)
  kPtrOff = 4,     // offset into in_ptr / out_ptr (S + 1 entries per row)
  kArcOff = 5,     // offset into every per-arc array
  kChunkOff = 6,   // offset into chunk arrays
  kNumChunks = 7,  // number of pdf chunks in this row
  kPdfPtrOff = 8,  // offset into pdf_chunk_ptr (D + 1 entries per row)
  kMaxInDeg = 9,
  kMaxOutDeg = 10,
  // tile packs (fb_tile_kernel): states sorted by degree into 32-lane tiles,
  // arc slots stored slot-major per tile (slot j of lane l at base + 32 j + l)
  kTileOff = 11,     // offset into per-tile arrays (trips/base), kNTiles tiles
  kTfSlotOff = 12,   // forward (by destination) slot offset
  kTfSlots = 13,     // forward slot count (multiple of 32)
  kTbSlotOff = 14,   // backward (by source) slot offset
  kTbSlots = 15,     // backward slot count
  kPdfPtrOff2 = 16,  // offset into pdf_arc_ptr (D + 1 per row): posterior slot groups
  kTileable = 17,    // 1 if indices fit the 16-bit tile encoding
  kXPad = 18,        // posterior slot count incl. per-pdf padding + dummy slot (multiple of 4)
  kWTabOff = 19,     // offset into the per-phase warp tables (kWarpTable ints per row)
  // stream packs (fb_stream_kernel, L2-resident graphs): 32-state tiles by degree,
  // slots {index | pdf << 15, fp32 prob} read straight from global memory
  kSTileOff = 20,    // offset into s*_info (x32) / s*_trips / s*_base
  kSTiles = 21,      // tiles per phase (0 = no stream pack for this row)
  kSfSlotOff = 22,   // forward (by destination) slot offset
  kSbSlotOff = 23,   // backward (by source) slot offset
  kNTiles = 24,      // tile packs: tiles per phase = ceil(S * kTileG / 32)
  kTileG = 25,       // tile packs: lanes per state (power of 2; a state's arcs split
                     // over G adjacent lanes, summed with xor shuffles; 1 = one lane)
  kDescInts = 26
};

// Device-side view of a packed graph batch (passed by value to kernels).
struct DevGraphs {
  const int *desc;
  // CSR by destination state (reference "backward_*" layout, graph.py:150-154)
  const int *in_ptr, *in_src, *in_pdf;
  const float *in_p32;
  const double *in_p64;
  // CSR by source state (reference "forward_*" layout, graph.py:144-148)
  const int *out_ptr, *out_dst, *out_pdf;
  const float *out_p32;
  const double *out_p64;
  // arcs grouped by pdf, cut into chunks (new: deterministic posterior gather)
  const int *pa_src, *pa_dst;
  const float *pa_p32;
  const double *pa_p64;
  const int *chunk_begin, *chunk_end, *chunk_pdf, *pdf_chunk_ptr;
  const float *fin32;
  const double *fin64;
  // tile packs
  const unsigned *tf_info, *tb_info;  // per tile lane: state | degree << 16
  const int *tf_trips, *tf_base, *tb_trips, *tb_base;
  const int *tf_wlist, *tb_wlist;     // tile ids grouped by warp (16-warp LPT schedule)
  const int *tf_wtab, *tb_wtab;       // per-warp ranges + warps by ascending load
  const int *tp_wlist, *tp_wtab;      // forward lists with flush chores (split kernel)
  const unsigned *tf_word, *tb_word;  // src|pdf<<16 (forward), dst|pdf<<16 (backward)
  const float *tf_p32, *tb_p32;
  const double *tf_p64, *tb_p64;
  const unsigned short *tb_xslot;     // posterior slot of each backward arc
  const unsigned short *tf_xslot;     // ... of each forward arc (same slot groups)
  const int *pdf_arc_ptr;             // posterior slot range per pdf (16-byte aligned)
  const uint2 *tf_wp, *tb_wp;         // interleaved (word, fp32 prob bits) slots
  const int *sf_info, *sb_info;       // stream packs: state per tile lane (-1 = none)
  const int *sf_trips, *sf_base, *sb_trips, *sb_base;
  const uint2 *sf_wp, *sb_wp;         // {index | pdf << 15, fp32 prob bits}
  // linear-chain pack (fb_linear_kernel): per row {state offset, S, initial, 0};
  // per state {fp32 self-loop prob, fp32 entry prob (arc s-1 -> s),
  // self pdf | entry pdf << 16, fp32 final prob}
  const int4 *lin_item;
  const uint4 *lin_state;
};

}  // namespace lfmmi

struct lfmmi_graphs {
  int32_t num_rows = 0, max_states = 0, max_arcs = 0, num_pdfs = 0;
  int32_t max_chunks = 0, max_in_deg = 0, max_out_deg = 0;
  int32_t max_tiles = 0, max_tf_slots = 0, max_tb_slots = 0, max_xpad = 0;
  bool tileable = false;
  bool streamable = false;  // every row has a stream pack (fb_stream_kernel)
  bool linear = false;      // every row is a linear chain (fb_linear_kernel pack present)
  bool linear_only = false; // lfmmi_graphs_create_linear: nothing but the linear pack
  int32_t max_stiles = 0;
  int32_t max_tile_g = 1;   // largest kTileG of the rows (1: one lane per state everywhere)
  int32_t rep_r = 1, r_stride = 0, rep_e = 1, e_stride = 0;  // gather-vector replication
  void *device_block = nullptr;
  size_t device_bytes = 0;
  lfmmi::DevGraphs dev{};
};

namespace lfmmi {
int set_error(int code, const std::string &msg);
int check_cuda(cudaError_t err, const char *what);
// Records the kernel of the last denominator-sized launch (lfmmi_last_den_kernel).
void note_den_kernel(const char *name);
// Records the kernel of the last forward-backward launch of any size (lfmmi_last_kernel).
void note_kernel(const char *name);
}  // namespace lfmmi
