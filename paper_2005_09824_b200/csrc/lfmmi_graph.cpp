// Host-side graph ingestion: reference padded ChainGraphBatch arrays ->
// device-resident packed CSR layouts (one cudaMalloc per graph batch).
//
// Replaces ChainGraphBatch._build (/root/reference/pkg/src/chainloss/graph.py:236-301)
// plus the device upload the reference never needed.  Three arc orders are
// materialised per graph row:
//   in_*  : CSR by destination state — the reference's backward_* order
//           (graph.py:150-154), consumed by the forward recursion;
//   out_* : CSR by source state — the reference's forward_* order
//           (graph.py:144-148), consumed by the backward recursion;
//   pa_*  : arcs grouped by pdf id and cut into chunks of <= chunk_len arcs,
//           consumed by the fused posterior gather (replaces the reference's
//           scatter over all arcs, _kernels.py:211-224, by a deterministic
//           per-pdf gather).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "lfmmi_internal.h"
#include "lfmmi_schedule.h"
#include "lfmmi_options.h"

namespace lfmmi {

static thread_local std::string g_last_error;

int set_error(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

int check_cuda(cudaError_t err, const char *what) {
  if (err == cudaSuccess) return LFMMI_OK;
  return set_error(LFMMI_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(err));
}

}  // namespace lfmmi

using namespace lfmmi;

extern "C" const char *lfmmi_last_error(void) { return g_last_error.c_str(); }

extern "C" const char *lfmmi_version(void) { return "paper_2005_09824_b200 lfmmi 0.1.0 (sm_100a)"; }

namespace {

struct HostPack {
  std::vector<int> desc;
  std::vector<int> in_ptr, in_src, in_pdf;
  std::vector<float> in_p32;
  std::vector<double> in_p64;
  std::vector<int> out_ptr, out_dst, out_pdf;
  std::vector<float> out_p32;
  std::vector<double> out_p64;
  std::vector<int> pa_src, pa_dst;
  std::vector<float> pa_p32;
  std::vector<double> pa_p64;
  std::vector<int> chunk_begin, chunk_end, chunk_pdf, pdf_chunk_ptr;
  std::vector<float> fin32;
  std::vector<double> fin64;
  std::vector<unsigned> tf_info, tb_info, tf_word, tb_word;
  std::vector<int> tf_trips, tf_base, tb_trips, tb_base, pdf_arc_ptr;
  std::vector<int> tf_wlist, tb_wlist, tf_wtab, tb_wtab, tp_wlist, tp_wtab;
  std::vector<int> sf_info, sb_info, sf_trips, sf_base, sb_trips, sb_base;
  std::vector<uint2> sf_wp, sb_wp;
  std::vector<float> tf_p32, tb_p32;
  std::vector<double> tf_p64, tb_p64;
  std::vector<unsigned short> tb_xslot, tf_xslot;
  std::vector<uint2> tf_wp, tb_wp;
  std::vector<int> lin_item;         // 4 per row: state offset, S, initial, 0
  std::vector<unsigned> lin_state;   // 4 per state (fb_linear_kernel record)
};

// Linear-chain record of one graph row (fb_linear_kernel): every arc is a
// self-loop s -> s or an entry arc s-1 -> s, at most one of each per state —
// the shape of the reference's numerators (toy_builder.py:218-265).  Returns
// false (and leaves `out` untouched) for any other graph.
bool linear_records(int S, int I, const uint32_t *from, const uint32_t *to, const uint32_t *pdf,
                    const double *prob, const double *finals, std::vector<unsigned> &out) {
  if (S > 512) return false;
  std::vector<unsigned> rec(size_t(S) * 4, 0u);
  std::vector<char> has_self(S, 0), has_in(S, 0);
  for (int i = 0; i < I; ++i) {
    const uint32_t f = from[i], t = to[i], d = pdf[i];
    if (d > 0xffffu) return false;
    const float p = float(prob[i]);
    unsigned bits;
    std::memcpy(&bits, &p, 4);
    if (t == f) {
      if (has_self[t]) return false;
      has_self[t] = 1;
      rec[4 * t + 0] = bits;
      rec[4 * t + 2] |= d;
    } else if (t == f + 1) {
      if (has_in[t]) return false;
      has_in[t] = 1;
      rec[4 * t + 1] = bits;
      rec[4 * t + 2] |= d << 16;
    } else {
      return false;
    }
  }
  for (int s = 0; s < S; ++s) {
    const float f = float(finals[s]);
    std::memcpy(&rec[4 * s + 3], &f, 4);
  }
  out.insert(out.end(), rec.begin(), rec.end());
  return true;
}

// Chunk length for the pdf-grouped posterior gather: aim for about one chunk
// per thread of the largest block (1024), never longer than needed.
int chunk_len_for(int num_arcs) { return std::max(2, (num_arcs + 1023) / 1024); }

template <typename T>
size_t align_up(size_t x) {
  (void)sizeof(T);
  return (x + 255) & ~size_t(255);
}

}  // namespace

extern "C" int lfmmi_graphs_create(int32_t num_rows, int32_t max_states, int32_t max_arcs,
                                   int32_t num_pdfs, const int64_t *row_num_states,
                                   const int64_t *row_num_arcs, const uint32_t *fw_from,
                                   const uint32_t *fw_to, const uint32_t *fw_pdf,
                                   const double *fw_prob, const uint32_t *bw_from,
                                   const uint32_t *bw_to, const uint32_t *bw_pdf,
                                   const double *bw_prob, const double *final_probs,
                                   const uint32_t *initial_states, lfmmi_graphs **out) {
  if (!out) return set_error(LFMMI_ERR_INVALID, "lfmmi_graphs_create: out is NULL");
  *out = nullptr;
  if (num_rows < 1 || max_states < 1 || max_arcs < 0 || num_pdfs < 1)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_graphs_create: bad sizes");
  if (!row_num_states || !row_num_arcs || !fw_from || !fw_to || !fw_pdf || !fw_prob ||
      !final_probs || !initial_states)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_graphs_create: NULL input array");
  const bool have_bw = bw_from && bw_to && bw_pdf && bw_prob;

  HostPack h;
  h.desc.resize(size_t(num_rows) * kDescInts, 0);
  const GatherLayout gl = make_gather_layout(max_states, num_pdfs);
  int max_chunks = 0, max_in = 0, max_out = 0;
  int max_tiles = 0, max_tf = 0, max_tb = 0, max_xpad = 0, max_tile_g = 1;
  bool all_tileable = true;
  bool all_streamable = true;
  bool all_linear = true;
  int max_stiles = 0;
  for (int r = 0; r < num_rows; ++r) {
    const int S = int(row_num_states[r]);
    const int I = int(row_num_arcs[r]);
    if (S < 1 || S > max_states || I < 0 || I > max_arcs)
      return set_error(LFMMI_ERR_INVALID, "lfmmi_graphs_create: row " + std::to_string(r) +
                                              " has out-of-range state/arc count");
    const size_t base = size_t(r) * size_t(max_arcs);
    for (int i = 0; i < I; ++i) {
      if (fw_from[base + i] >= uint32_t(S) || fw_to[base + i] >= uint32_t(S) ||
          fw_pdf[base + i] >= uint32_t(num_pdfs))
        return set_error(LFMMI_ERR_INVALID, "lfmmi_graphs_create: row " + std::to_string(r) +
                                                " arc " + std::to_string(i) + " out of range");
    }
    if (initial_states[r] >= uint32_t(S))
      return set_error(LFMMI_ERR_INVALID, "lfmmi_graphs_create: initial state out of range");

    int *d = &h.desc[size_t(r) * kDescInts];
    d[kS] = S;
    d[kI] = I;
    d[kInit] = int(initial_states[r]);
    d[kStateOff] = int(h.fin64.size());
    d[kPtrOff] = int(h.in_ptr.size());
    d[kArcOff] = int(h.in_src.size());
    d[kChunkOff] = int(h.chunk_begin.size());
    d[kPdfPtrOff] = int(h.pdf_chunk_ptr.size());

    for (int s = 0; s < S; ++s) {
      const double f = final_probs[size_t(r) * max_states + s];
      h.fin64.push_back(f);
      h.fin32.push_back(float(f));
    }

    if (all_linear) {
      h.lin_item.insert(h.lin_item.end(), {int(h.lin_state.size() / 4), S, d[kInit], 0});
      all_linear = linear_records(S, I, fw_from + base, fw_to + base, fw_pdf + base, fw_prob + base,
                                  final_probs + size_t(r) * max_states, h.lin_state);
    }

    // out-CSR: the reference forward_* order is already sorted by source.
    std::vector<int> cnt_out(S + 1, 0), cnt_in(S + 1, 0);
    for (int i = 0; i < I; ++i) cnt_out[fw_from[base + i] + 1]++;
    // in-CSR: reference backward_* order when given, else stable sort by destination.
    std::vector<int> in_order(I);
    if (have_bw) {
      for (int i = 0; i < I; ++i) cnt_in[bw_to[base + i] + 1]++;
    } else {
      for (int i = 0; i < I; ++i) cnt_in[fw_to[base + i] + 1]++;
      std::iota(in_order.begin(), in_order.end(), 0);
      std::stable_sort(in_order.begin(), in_order.end(), [&](int x, int y) {
        return fw_to[base + x] < fw_to[base + y];
      });
    }
    int mi = 0, mo = 0;
    for (int s = 0; s < S; ++s) {
      mi = std::max(mi, cnt_in[s + 1]);
      mo = std::max(mo, cnt_out[s + 1]);
    }
    for (int s = 0; s < S; ++s) {
      cnt_in[s + 1] += cnt_in[s];
      cnt_out[s + 1] += cnt_out[s];
    }
    d[kMaxInDeg] = mi;
    d[kMaxOutDeg] = mo;
    max_in = std::max(max_in, mi);
    max_out = std::max(max_out, mo);
    for (int s = 0; s <= S; ++s) {
      h.in_ptr.push_back(cnt_in[s]);
      h.out_ptr.push_back(cnt_out[s]);
    }
    for (int i = 0; i < I; ++i) {
      h.out_dst.push_back(int(fw_to[base + i]));
      h.out_pdf.push_back(int(fw_pdf[base + i]));
      h.out_p64.push_back(fw_prob[base + i]);
      h.out_p32.push_back(float(fw_prob[base + i]));
      if (have_bw) {
        h.in_src.push_back(int(bw_from[base + i]));
        h.in_pdf.push_back(int(bw_pdf[base + i]));
        h.in_p64.push_back(bw_prob[base + i]);
        h.in_p32.push_back(float(bw_prob[base + i]));
      } else {
        const int j = in_order[i];
        h.in_src.push_back(int(fw_from[base + j]));
        h.in_pdf.push_back(int(fw_pdf[base + j]));
        h.in_p64.push_back(fw_prob[base + j]);
        h.in_p32.push_back(float(fw_prob[base + j]));
      }
    }

    // pdf-grouped arcs (stable by the forward_* order) cut into chunks.
    std::vector<int> pa(I);
    std::iota(pa.begin(), pa.end(), 0);
    std::stable_sort(pa.begin(), pa.end(),
                     [&](int x, int y) { return fw_pdf[base + x] < fw_pdf[base + y]; });
    for (int i = 0; i < I; ++i) {
      const int j = pa[i];
      h.pa_src.push_back(int(fw_from[base + j]));
      h.pa_dst.push_back(int(fw_to[base + j]));
      h.pa_p64.push_back(fw_prob[base + j]);
      h.pa_p32.push_back(float(fw_prob[base + j]));
    }
    const int clen = chunk_len_for(I);
    int nchunks = 0;
    int i = 0;
    for (int pdf = 0; pdf < num_pdfs; ++pdf) {
      h.pdf_chunk_ptr.push_back(nchunks);
      int j = i;
      while (j < I && int(fw_pdf[base + pa[j]]) == pdf) ++j;
      for (int c = i; c < j; c += clen) {
        h.chunk_begin.push_back(c);
        h.chunk_end.push_back(std::min(j, c + clen));
        h.chunk_pdf.push_back(pdf);
        ++nchunks;
      }
      i = j;
    }
    h.pdf_chunk_ptr.push_back(nchunks);
    d[kNumChunks] = nchunks;
    max_chunks = std::max(max_chunks, nchunks);

    // ---- stream packs (fb_stream_kernel): graphs too large for the on-chip packs ----
    d[kSTileOff] = int(h.sf_trips.size());
    d[kSTiles] = 0;
    d[kSfSlotOff] = int(h.sf_wp.size());
    d[kSbSlotOff] = int(h.sb_wp.size());
    const bool want_stream = S > 512 && S <= 32767 && num_pdfs <= 131071;
    if (want_stream) {
      const size_t a0 = size_t(d[kArcOff]);
      const int *iptr = &h.in_ptr[h.in_ptr.size() - (S + 1)];
      const int *optr = &h.out_ptr[h.out_ptr.size() - (S + 1)];
      const int nt = (S + 31) / 32;
      auto pack = [&](const int *ptr, const int *gidx, const int *pdf, const double *prob,
                      std::vector<int> &info, std::vector<int> &trips, std::vector<int> &base,
                      std::vector<uint2> &wp) {
        std::vector<int> order(S);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
          return (ptr[x + 1] - ptr[x]) > (ptr[y + 1] - ptr[y]);
        });
        int b = 0;
        for (int t = 0; t < nt; ++t) {
          int tr = 0;
          for (int l = 0; l < 32; ++l) {
            const int k = 32 * t + l;
            info.push_back(k < S ? order[k] : -1);
            if (k < S) tr = std::max(tr, ptr[order[k] + 1] - ptr[order[k]]);
          }
          trips.push_back(tr);
          base.push_back(b);
          for (int j = 0; j < tr; ++j)
            for (int l = 0; l < 32; ++l) {
              const int k = 32 * t + l;
              uint2 v{0u, 0u};
              if (k < S) {
                const int s = order[k];
                if (j < ptr[s + 1] - ptr[s]) {
                  const int a = ptr[s] + j;
                  const float f = float(prob[a]);
                  v.x = unsigned(gidx[a]) | (unsigned(pdf[a]) << 15);
                  std::memcpy(&v.y, &f, 4);
                }
              }
              wp.push_back(v);
            }
          b += 32 * tr;
        }
        while (trips.size() % 4) {  // 16-byte aligned per-row tile arrays
          trips.push_back(0);
          base.push_back(0);
          for (int l = 0; l < 32; ++l) info.push_back(-1);
        }
      };
      // Bank-scheduled rows: the stream kernel gathers plain (unreplicated)
      // columns, so each row's arcs are chosen to spread the 32 lanes' column
      // and emission addresses over the banks (greedy + a bounded local search:
      // ~4M row evaluations per direction at most).
      const GatherLayout plain{1, 0, 1, 0};
      const int rows_est = std::max(1, I / 32 + nt);
      const int iters = std::min(1500, int(4000000 / rows_est));
      auto emit = [&](const TileSchedule &ts, const int *gidx, const int *pdf, const double *prob,
                      std::vector<int> &info, std::vector<int> &trips, std::vector<int> &base,
                      std::vector<uint2> &wp) {
        int b = 0;
        for (size_t t = 0; t < ts.trips.size(); ++t) {
          for (int l = 0; l < 32; ++l) {
            const unsigned v = ts.info[32 * t + l];
            info.push_back((v & 0xFFFFu) == 0xFFFFu ? -1 : int(v & 0xFFFFu));
          }
          trips.push_back(ts.trips[t]);
          base.push_back(b);
          for (int j = 0; j < ts.trips[t]; ++j) {
            // idle lanes re-read an address of an active lane (free broadcast), prob 0
            const int *row = &ts.arc[size_t(ts.base[t]) + 32 * j];
            unsigned pad = 0u;
            for (int l = 0; l < 32; ++l)
              if (row[l] >= 0) {
                pad = unsigned(gidx[row[l]]) | (unsigned(pdf[row[l]]) << 15);
                break;
              }
            for (int l = 0; l < 32; ++l) {
              const int arc = row[l];
              uint2 v{pad, 0u};
              if (arc >= 0) {
                const float f = float(prob[arc]);
                v.x = unsigned(gidx[arc]) | (unsigned(pdf[arc]) << 15);
                std::memcpy(&v.y, &f, 4);
              }
              wp.push_back(v);
            }
          }
          b += 32 * ts.trips[t];
        }
        while (trips.size() % 4) {  // 16-byte aligned per-row tile arrays
          trips.push_back(0);
          base.push_back(0);
          for (int l = 0; l < 32; ++l) info.push_back(-1);
        }
      };
      if (S <= 0xFFFE) {  // schedule info packs states in 16 bits
        const TileSchedule sf = schedule_tiles(S, iptr, &h.in_src[a0], &h.in_pdf[a0],
                                               &h.in_p64[a0], plain, true, iters);
        const TileSchedule sb = schedule_tiles(S, optr, &h.out_dst[a0], &h.out_pdf[a0],
                                               &h.out_p64[a0], plain, true, iters);
        emit(sf, &h.in_src[a0], &h.in_pdf[a0], &h.in_p64[a0], h.sf_info, h.sf_trips, h.sf_base,
             h.sf_wp);
        emit(sb, &h.out_dst[a0], &h.out_pdf[a0], &h.out_p64[a0], h.sb_info, h.sb_trips,
             h.sb_base, h.sb_wp);
      } else {
        pack(iptr, &h.in_src[a0], &h.in_pdf[a0], &h.in_p64[a0], h.sf_info, h.sf_trips,
             h.sf_base, h.sf_wp);
        pack(optr, &h.out_dst[a0], &h.out_pdf[a0], &h.out_p64[a0], h.sb_info, h.sb_trips,
             h.sb_base, h.sb_wp);
      }
      d[kSTiles] = nt;
      max_stiles = std::max(max_stiles, nt);
    } else {
      all_streamable = false;
    }

    // ---- tile packs (scheduled, 16-bit state / pdf / posterior-slot encoding) ----
    bool tileable = S <= 16383 && num_pdfs <= 16383 && I <= 65535 && mi < 65536 && mo < 65536;
    d[kTileG] = 1;
    d[kNTiles] = 0;
    d[kTileOff] = int(h.tf_trips.size());
    d[kTfSlotOff] = int(h.tf_word.size());
    d[kTbSlotOff] = int(h.tb_word.size());
    d[kPdfPtrOff2] = int(h.pdf_arc_ptr.size());
    if (tileable) {
      const size_t a0 = size_t(d[kArcOff]);
      const int *iptr = &h.in_ptr[h.in_ptr.size() - (S + 1)];
      const int *optr = &h.out_ptr[h.out_ptr.size() - (S + 1)];
      // small dense graphs: a state's arc list over G adjacent lanes (both packs)
      const int G = tile_lanes_per_state(S, std::max(mi, mo), options().tile_g);
      TileSchedule tf = schedule_tiles(S, iptr, &h.in_src[a0], &h.in_pdf[a0], &h.in_p64[a0], gl,
                                       true, -1, G);
      TileSchedule tb = schedule_tiles(S, optr, &h.out_dst[a0], &h.out_pdf[a0], &h.out_p64[a0],
                                       gl, true, -1, G);
      d[kTileG] = G;
      max_tile_g = std::max(max_tile_g, G);
      d[kNTiles] = int(tf.trips.size());
      std::vector<int> pptr, xslot;
      int xpad = 0;
      assign_xslots(tb, &h.out_pdf[a0], num_pdfs, I, 4, pptr, xslot, xpad);
      // Forward-pack posterior slots (fb_split_kernel: the forward CTA writes the
      // posteriors of the second half of the utterance).  The per-pdf slot
      // groups depend only on the pdf counts, so both packs share pdf_arc_ptr.
      std::vector<int> pptr_f, xslot_f;
      int xpad_f = 0;
      assign_xslots(tf, &h.in_pdf[a0], num_pdfs, I, 4, pptr_f, xslot_f, xpad_f);
      tileable = xpad <= 65536 && pptr_f == pptr && xpad_f == xpad;
      if (tileable) {
        d[kXPad] = xpad;
        h.pdf_arc_ptr.insert(h.pdf_arc_ptr.end(), pptr.begin(), pptr.end());
        for (size_t k = 0; k < tf.trips.size(); ++k) {
          h.tf_trips.push_back(tf.trips[k]);
          h.tf_base.push_back(tf.base[k]);
          h.tb_trips.push_back(tb.trips[k]);
          h.tb_base.push_back(tb.base[k]);
        }
        {
          // Warp lists for the 16-warp CTA kernels: the last warps carry the
          // per-frame emission-row chores, so they start with a small bias.
          std::vector<int> bias(kTableNW, 0), tab, lst;
          const int chore = std::min(kTableNW, (num_pdfs + 31) / 32);
          // (a frame's chores are latency chains — row max, exp, prefetch — worth
          // ~16 slot rows of arc work; measured: bias 2 -> 16, den 1.419 -> 1.294 ms)
          const int chore_bias = options().chore_bias;
          for (int w = kTableNW - chore; w < kTableNW; ++w) bias[w] = chore_bias;
          d[kWTabOff] = int(h.tf_wtab.size());
          warp_lists(tf.trips, bias, tab, lst);
          h.tf_wtab.insert(h.tf_wtab.end(), tab.begin(), tab.end());
          h.tf_wlist.insert(h.tf_wlist.end(), lst.begin(), lst.end());
          // Backward: the top warps also flush the gradient row of the previous
          // frame (fb_tile_kernel, spl lanes per pdf, ~5 instructions per float4
          // of posterior slots vs ~14 per arc-slot row).
          int spl = 1;
          while (spl < 32 && num_pdfs * spl * 2 <= 32 * kTableNW) spl <<= 1;
          const int lanes = num_pdfs * spl;
          const int chore_bias_bwd = chore_bias;
          for (int w = kTableNW - chore; w < kTableNW; ++w) bias[w] = chore_bias_bwd;
          if (lanes < 32 * kTableNW) {
            const int fw = (lanes + 31) / 32;
            const int per_lane = (xpad / 4 + lanes - 1) / lanes;
            // (flush-bias scale 50-300% measured as slow or slower: DESIGN.md §3.3)
            const int fb = (per_lane * 5 + 13) / 14;
            for (int w = kTableNW - fw; w < kTableNW; ++w) bias[w] += fb;
          }
          warp_lists(tb.trips, bias, tab, lst);
          h.tb_wtab.insert(h.tb_wtab.end(), tab.begin(), tab.end());
          h.tb_wlist.insert(h.tb_wlist.end(), lst.begin(), lst.end());
          // forward with posteriors (fb_split_kernel, second half): same chores as
          // the backward (emission row + gradient-row flush)
          warp_lists(tf.trips, bias, tab, lst);
          h.tp_wtab.insert(h.tp_wtab.end(), tab.begin(), tab.end());
          h.tp_wlist.insert(h.tp_wlist.end(), lst.begin(), lst.end());
        }
        h.tf_info.insert(h.tf_info.end(), tf.info.begin(), tf.info.end());
        h.tb_info.insert(h.tb_info.end(), tb.info.begin(), tb.info.end());
        while (h.tf_trips.size() % 4) {  // keep per-row tile arrays 16-byte aligned
          h.tf_wlist.push_back(0);
          h.tp_wlist.push_back(0);
          h.tb_wlist.push_back(0);
          h.tf_trips.push_back(0);
          h.tf_base.push_back(0);
          h.tb_trips.push_back(0);
          h.tb_base.push_back(0);
          for (int l = 0; l < 32; ++l) {  // info is indexed by tile * 32 + lane
            h.tf_info.push_back(0xFFFFu);
            h.tb_info.push_back(0xFFFFu);
          }
        }
        h.tf_word.insert(h.tf_word.end(), tf.word_idx.begin(), tf.word_idx.end());
        h.tb_word.insert(h.tb_word.end(), tb.word_idx.begin(), tb.word_idx.end());
        auto push_wp = [](std::vector<uint2> &dst, const TileSchedule &ts) {
          for (size_t k = 0; k < ts.prob.size(); ++k) {
            const float f = float(ts.prob[k]);
            unsigned bits;
            std::memcpy(&bits, &f, 4);
            dst.push_back({ts.word_b32[k], bits});
          }
        };
        push_wp(h.tf_wp, tf);
        push_wp(h.tb_wp, tb);
        for (double p : tf.prob) {
          h.tf_p64.push_back(p);
          h.tf_p32.push_back(float(p));
        }
        for (double p : tb.prob) {
          h.tb_p64.push_back(p);
          h.tb_p32.push_back(float(p));
        }
        for (int x : xslot) h.tb_xslot.push_back((unsigned short)x);
        for (int x : xslot_f) h.tf_xslot.push_back((unsigned short)x);
        max_xpad = std::max(max_xpad, xpad);
        d[kTfSlots] = int(tf.word_idx.size());
        d[kTbSlots] = int(tb.word_idx.size());
        max_tiles = std::max(max_tiles, int(tf.trips.size()));
        max_tf = std::max(max_tf, d[kTfSlots]);
        max_tb = std::max(max_tb, d[kTbSlots]);
      }
    }
    d[kTileable] = tileable ? 1 : 0;
    if (!tileable) {
      all_tileable = false;
    }
  }

  // One device allocation, 256-byte aligned sub-buffers.
  struct Piece {
    const void *src;
    size_t bytes;
    const void **dst;
  };
  auto *g = new lfmmi_graphs();
  g->num_rows = num_rows;
  g->max_states = max_states;
  g->max_arcs = max_arcs;
  g->num_pdfs = num_pdfs;
  g->max_chunks = max_chunks;
  g->max_in_deg = max_in;
  g->max_out_deg = max_out;
  g->max_tiles = max_tiles;
  g->max_tile_g = max_tile_g;
  g->max_tf_slots = max_tf;
  g->max_tb_slots = max_tb;
  g->tileable = all_tileable;
  g->streamable = all_streamable;
  g->max_stiles = max_stiles;
  g->max_xpad = max_xpad;
  g->linear = all_linear;
  if (!all_linear) {
    h.lin_item.clear();
    h.lin_state.clear();
  }
  g->rep_r = gl.rep_r;
  g->r_stride = gl.r_stride;
  g->rep_e = gl.rep_e;
  g->e_stride = gl.e_stride;
  DevGraphs &dv = g->dev;
  std::vector<Piece> pieces;
  auto add = [&](const auto &vec, const auto **dst) {
    using T = typename std::decay_t<decltype(vec)>::value_type;
    pieces.push_back({vec.data(), vec.size() * sizeof(T), reinterpret_cast<const void **>(dst)});
  };
  add(h.desc, &dv.desc);
  add(h.in_ptr, &dv.in_ptr);
  add(h.in_src, &dv.in_src);
  add(h.in_pdf, &dv.in_pdf);
  add(h.in_p32, &dv.in_p32);
  add(h.in_p64, &dv.in_p64);
  add(h.out_ptr, &dv.out_ptr);
  add(h.out_dst, &dv.out_dst);
  add(h.out_pdf, &dv.out_pdf);
  add(h.out_p32, &dv.out_p32);
  add(h.out_p64, &dv.out_p64);
  add(h.pa_src, &dv.pa_src);
  add(h.pa_dst, &dv.pa_dst);
  add(h.pa_p32, &dv.pa_p32);
  add(h.pa_p64, &dv.pa_p64);
  add(h.chunk_begin, &dv.chunk_begin);
  add(h.chunk_end, &dv.chunk_end);
  add(h.chunk_pdf, &dv.chunk_pdf);
  add(h.pdf_chunk_ptr, &dv.pdf_chunk_ptr);
  add(h.fin32, &dv.fin32);
  add(h.fin64, &dv.fin64);
  add(h.tf_info, &dv.tf_info);
  add(h.tb_info, &dv.tb_info);
  add(h.tf_trips, &dv.tf_trips);
  add(h.sf_info, &dv.sf_info);
  add(h.sb_info, &dv.sb_info);
  add(h.sf_trips, &dv.sf_trips);
  add(h.sf_base, &dv.sf_base);
  add(h.sb_trips, &dv.sb_trips);
  add(h.sb_base, &dv.sb_base);
  add(h.sf_wp, &dv.sf_wp);
  add(h.sb_wp, &dv.sb_wp);
  add(h.tf_wlist, &dv.tf_wlist);
  add(h.tp_wlist, &dv.tp_wlist);
  add(h.tp_wtab, &dv.tp_wtab);
  add(h.tb_wlist, &dv.tb_wlist);
  add(h.tf_wtab, &dv.tf_wtab);
  add(h.tb_wtab, &dv.tb_wtab);
  add(h.tf_base, &dv.tf_base);
  add(h.tb_trips, &dv.tb_trips);
  add(h.tb_base, &dv.tb_base);
  add(h.tf_word, &dv.tf_word);
  add(h.tb_word, &dv.tb_word);
  add(h.tf_p32, &dv.tf_p32);
  add(h.tb_p32, &dv.tb_p32);
  add(h.tf_p64, &dv.tf_p64);
  add(h.tb_p64, &dv.tb_p64);
  add(h.tb_xslot, &dv.tb_xslot);
  add(h.tf_xslot, &dv.tf_xslot);
  add(h.pdf_arc_ptr, &dv.pdf_arc_ptr);
  add(h.tf_wp, &dv.tf_wp);
  add(h.tb_wp, &dv.tb_wp);
  add(h.lin_item, &dv.lin_item);
  add(h.lin_state, &dv.lin_state);
  size_t total = 0;
  std::vector<size_t> offs;
  for (auto &p : pieces) {
    offs.push_back(total);
    total += align_up<char>(std::max<size_t>(p.bytes, 16));
  }
  std::vector<char> staging(total, 0);
  for (size_t k = 0; k < pieces.size(); ++k)
    if (pieces[k].bytes) std::memcpy(staging.data() + offs[k], pieces[k].src, pieces[k].bytes);
  void *dev = nullptr;
  int rc = check_cuda(cudaMalloc(&dev, total), "cudaMalloc(graph pack)");
  if (rc) {
    delete g;
    return rc;
  }
  rc = check_cuda(cudaMemcpy(dev, staging.data(), total, cudaMemcpyHostToDevice),
                  "cudaMemcpy(graph pack)");
  if (rc) {
    cudaFree(dev);
    delete g;
    return rc;
  }
  for (size_t k = 0; k < pieces.size(); ++k)
    *pieces[k].dst = static_cast<const char *>(dev) + offs[k];
  g->device_block = dev;
  g->device_bytes = total;
  *out = g;
  return LFMMI_OK;
}

extern "C" int lfmmi_graphs_create_linear(int32_t num_rows, int32_t max_states, int32_t num_pdfs,
                                          const int32_t *items, const uint32_t *states,
                                          lfmmi_graphs **out) {
  if (!out) return set_error(LFMMI_ERR_INVALID, "lfmmi_graphs_create_linear: out is NULL");
  *out = nullptr;
  if (num_rows < 1 || max_states < 1 || max_states > 512 || num_pdfs < 1 || num_pdfs > 65536)
    return set_error(LFMMI_ERR_INVALID,
                     "lfmmi_graphs_create_linear: need 1 <= max_states <= 512, 1 <= num_pdfs <= 65536");
  if (!items || !states)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_graphs_create_linear: NULL device array");
  auto *g = new lfmmi_graphs();
  g->num_rows = num_rows;
  g->max_states = max_states;
  g->max_arcs = 2 * max_states;
  g->num_pdfs = num_pdfs;
  g->linear = true;
  g->linear_only = true;
  g->dev.lin_item = reinterpret_cast<const int4 *>(items);
  g->dev.lin_state = reinterpret_cast<const uint4 *>(states);
  *out = g;  // device_block stays NULL: the caller owns the arrays
  return LFMMI_OK;
}

extern "C" int lfmmi_graphs_destroy(lfmmi_graphs *graphs) {
  if (!graphs) return LFMMI_OK;
  int rc = LFMMI_OK;
  if (graphs->device_block) rc = check_cuda(cudaFree(graphs->device_block), "cudaFree(graph pack)");
  delete graphs;
  return rc;
}

extern "C" int lfmmi_graphs_info(const lfmmi_graphs *graphs, int32_t *num_rows,
                                 int32_t *max_states, int32_t *max_arcs, int32_t *num_pdfs) {
  if (!graphs) return set_error(LFMMI_ERR_INVALID, "lfmmi_graphs_info: NULL handle");
  if (num_rows) *num_rows = graphs->num_rows;
  if (max_states) *max_states = graphs->max_states;
  if (max_arcs) *max_arcs = graphs->max_arcs;
  if (num_pdfs) *num_pdfs = graphs->num_pdfs;
  return LFMMI_OK;
}
