// Host-side tile scheduling (see lfmmi_schedule.cpp).
#pragma once

#include <vector>

namespace lfmmi {

// Replication of the shared-memory gather vectors: copy c of the alpha/beta
// column sits at c * r_stride, copy c of the emission row at c * e_stride
// (floats), strides chosen so every copy is shifted by a fixed bank offset.
struct GatherLayout {
  int rep_r = 1, r_stride = 0, rep_e = 1, e_stride = 0;
};

GatherLayout make_gather_layout(int max_states, int num_pdfs);

struct TileSchedule {
  std::vector<unsigned> info;      // per tile lane: state | degree << 16 (0xFFFF = none)
  std::vector<int> trips, base;    // per tile
  std::vector<int> arc;            // per slot: CSR arc index (-1 = padding)
  std::vector<unsigned> word_idx;  // gidx | pdf << 16 (plain indices; f64 path)
  std::vector<unsigned> word_b32;  // byte offsets incl. the chosen copies (f32 path)
  std::vector<double> prob;        // 0 on padding
};

// ptr: CSR row pointers (S + 1) of the layout; gidx/pdf/prob per CSR arc.
// iters_per_row < 0: the default local-search budget (option sched_iters / auto).
// lanes_per_state G (power of 2 <= 32): state k of the degree order owns lanes
// [kG, kG + G) of the lane sequence, lane j of them the arcs j, j + G, ... of
// its CSR row; tiles = ceil(S G / 32).  G > 1 splits the long in/out lists of a
// small dense graph (a phone-bigram den: 43 states, ~44 arcs each) over lanes.
TileSchedule schedule_tiles(int S, const int *ptr, const int *gidx, const int *pdf,
                            const double *prob, const GatherLayout &gl, bool optimize,
                            int iters_per_row = -1, int lanes_per_state = 1);

// Lanes per state of a row's tile packs: the largest power of 2 with at most
// 512 lanes in all (one 16-warp CTA) and >= 4 arcs per lane on the longest
// list; 1 for every graph with more than 256 states.  force > 0 overrides.
int tile_lanes_per_state(int S, int max_deg, int force);

// Posterior slot of every backward tile slot: pdf groups (16-byte aligned,
// `slack` spare positions each), conflict-avoiding positions per slot row,
// padding slots -> one trailing dummy slot.  pdf_of_arc is indexed by CSR arc.
void assign_xslots(const TileSchedule &tb, const int *pdf_of_arc, int num_pdfs, int num_arcs,
                   int slack, std::vector<int> &pdf_ptr, std::vector<int> &xslot_of_slot,
                   int &xpad);

// Longest-processing-time assignment of the tiles of one phase to the NW
// warps of a CTA-per-utterance kernel (kWarpTable ints per row and phase):
//   table[0..NW]        per-warp ranges into `list` (CSR),
//   table[NW+1..2NW]    warps in ascending final load (numerator tiles go to
//                       the lightest warps first),
// list: tile ids grouped by warp, each warp's tiles in descending trips.
// `bias[w]` is the extra per-frame work warp w already carries (chores).
constexpr int kTableNW = 16;
constexpr int kWarpTable = 36;
void warp_lists(const std::vector<int> &trips, const std::vector<int> &bias,
                std::vector<int> &table, std::vector<int> &list);

}  // namespace lfmmi
