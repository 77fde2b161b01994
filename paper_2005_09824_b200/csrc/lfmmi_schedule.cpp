// Offline, bank-conflict-aware scheduling of the tile packs (host side).
//
// A tile packs 32 states (one per lane, sorted by degree); slot row j of the
// tile is one warp-wide step: lane l processes one of its state's arcs.  Each
// step gathers vec[gidx] (alpha column in the forward, beta column in the
// backward) and e[pdf] from shared memory, and the backward additionally
// stores one posterior term.  A warp-wide shared access costs one wavefront
// per distinct address in its busiest bank, so random gathers cost ~3.5x the
// ideal.  Three free choices remove most of that:
//   * the order of each lane's arcs across slot rows (any permutation is
//     valid: the per-state sum just changes order);
//   * which copy of a replicated gather vector an arc reads (the kernel keeps
//     rep_r copies of the alpha/beta column and rep_e copies of the emission
//     row at strides that shift every copy by a fixed number of banks);
//   * where in its pdf group each posterior term is stored.
// The greedy below fills each slot row lane by lane (fewest remaining arcs
// first), picking the arc and copies that add the fewest new addresses to
// already-used banks.  Broadcasts (same address) are free.
#include "lfmmi_schedule.h"
#include "lfmmi_options.h"

#include <algorithm>
#include <atomic>
#include <thread>
#include <cstdint>
#include <array>
#include <random>
#include <cstdlib>
#include <numeric>
#include <functional>
#include <cstdio>

namespace lfmmi {

namespace {

struct BankSet {  // distinct addresses per bank within one slot row
  int n[32];
  int addr[32][8];
  void clear() { std::fill(n, n + 32, 0); }
  int cost(int a) const {
    const int b = a & 31;
    for (int k = 0; k < n[b]; ++k)
      if (addr[b][k] == a) return 0;
    return n[b];
  }
  void add(int a) {
    const int b = a & 31;
    for (int k = 0; k < n[b]; ++k)
      if (addr[b][k] == a) return;
    if (n[b] < 8) addr[b][n[b]] = a;
    n[b] = std::min(n[b] + 1, 8);
  }
};

}  // namespace

// Local-search moves per slot row (option sched_iters; 0 = greedy only).  Auto:
// 1500 for denominator-sized graphs; none for numerator-sized ones (<= 512
// states), whose kernels are latency-bound at a few per cent of SMEM
// bandwidth — the search cost ~7 ms of host time per numerator for nothing.
static int local_search_iters(int S) {
  const int o = options().sched_iters;
  if (o >= 0) return o;
  return S > 512 ? 1500 : 0;
}

GatherLayout make_gather_layout(int max_states, int num_pdfs) {
  GatherLayout gl;
  auto round32 = [](int x) { return (x + 31) & ~31; };
  // copy 1 of the gather column sits r_off banks over (LFMMI_R_OFF overrides)
  // (9: the two candidate banks of an address form a ring rather than 16
  // disjoint pairs, which the row matching exploits better — offline: 1.87 ->
  // 1.66 wavefronts per warp-wide gather with the local search)
  gl.r_stride = round32(max_states) + 9;
  gl.rep_r = (2 * gl.r_stride <= 16383) ? 2 : 1;
  if (gl.rep_r == 1) gl.r_stride = (max_states + 3) & ~3;
  gl.e_stride = round32(num_pdfs) + 8;  // copies shift by 8 banks
  gl.rep_e = 4;
  while (gl.rep_e > 1 && gl.rep_e * gl.e_stride > 16383) gl.rep_e >>= 1;
  if (gl.rep_e == 1) gl.e_stride = (num_pdfs + 3) & ~3;
  return gl;
}

// ---- exact per-row copy assignment + local search over slot rows ---------------
//
// For one slot row, the wavefront count of a gather is the largest number of
// distinct addresses any bank must serve.  Given the row's arcs, choosing the
// copy (hence the bank) of every distinct address is a bipartite b-matching:
// addresses -> banks with capacity k; the smallest feasible k is the row's cost
// (computed exactly by augmenting paths; <= 32 addresses).  A local search then
// swaps a lane's arcs between slot rows of its tile (any permutation of a
// lane's arcs is valid) and keeps swaps that do not raise the summed cost.
namespace {

struct RowSolver {
  int na = 0;
  int addr[32];
  int cand[32][4];
  int ncand = 1;
  int slot_owner[32][8];  // bank -> addresses holding its slots
  int slot_n[32];
  int choice[32];

  bool try_assign(int a, int k, uint32_t &seen) {
    for (int c = 0; c < ncand; ++c) {
      const int b = cand[a][c];
      if (seen & (1u << b)) continue;
      seen |= 1u << b;
      if (slot_n[b] < k) {
        slot_owner[b][slot_n[b]++] = a;
        choice[a] = c;
        return true;
      }
      for (int q = 0; q < slot_n[b]; ++q) {
        const int other = slot_owner[b][q];
        if (try_assign(other, k, seen)) {
          slot_owner[b][q] = a;
          choice[a] = c;
          return true;
        }
      }
    }
    return false;
  }

  // addresses (distinct) with candidate banks; returns min k and fills choice[]
  int solve() {
    // lower bound: ceil(na / 32) and the pigeonhole bound of a single candidate
    for (int k = (na + 31) / 32; k <= 8; ++k) {
      std::fill(slot_n, slot_n + 32, 0);
      bool ok = true;
      for (int a = 0; a < na && ok; ++a) {
        uint32_t seen = 0;
        ok = try_assign(a, k, seen);
      }
      if (ok) return k;
    }
    return 8;
  }
};

// Cost of one row: r-gather k + e-gather k; copies chosen per distinct address.
struct RowEval {
  int cost = 0;
  int rcopy[32], ecopy[32];  // per lane (-1 if idle)
};

RowEval eval_row(const int *arcs, const int *gidx, const int *pdf, const GatherLayout &gl) {
  RowEval ev;
  RowSolver rs, es;
  rs.ncand = gl.rep_r;
  es.ncand = gl.rep_e;
  int rlane_addr[32], elane_addr[32];
  for (int l = 0; l < 32; ++l) {
    ev.rcopy[l] = ev.ecopy[l] = -1;
    rlane_addr[l] = elane_addr[l] = -1;
    const int a = arcs[l];
    if (a < 0) continue;
    auto add = [](RowSolver &r, int v) {
      for (int i = 0; i < r.na; ++i)
        if (r.addr[i] == v) return i;
      r.addr[r.na] = v;
      return r.na++;
    };
    rlane_addr[l] = add(rs, gidx[a]);
    elane_addr[l] = add(es, pdf[a]);
  }
  for (int i = 0; i < rs.na; ++i)
    for (int c = 0; c < rs.ncand; ++c) rs.cand[i][c] = (c * gl.r_stride + rs.addr[i]) & 31;
  for (int i = 0; i < es.na; ++i)
    for (int c = 0; c < es.ncand; ++c) es.cand[i][c] = (c * gl.e_stride + es.addr[i]) & 31;
  const int kr = rs.na ? rs.solve() : 0;
  const int ke = es.na ? es.solve() : 0;
  ev.cost = kr + ke;
  for (int l = 0; l < 32; ++l) {
    if (rlane_addr[l] >= 0) ev.rcopy[l] = rs.choice[rlane_addr[l]];
    if (elane_addr[l] >= 0) ev.ecopy[l] = es.choice[elane_addr[l]];
  }
  return ev;
}

}  // namespace

int tile_lanes_per_state(int S, int max_deg, int force) {
  if (force > 0) {
    int g = 1;
    while (g < 32 && g * 2 <= force) g *= 2;
    return g;
  }
  int g = 1;
  while (g < 32 && S * g * 2 <= 512 && max_deg >= 8 * g) g *= 2;
  return g;
}

TileSchedule schedule_tiles(int S, const int *ptr, const int *gidx, const int *pdf,
                            const double *prob, const GatherLayout &gl, bool optimize,
                            int iters_per_row, int lanes_per_state) {
  const int ls_iters = iters_per_row >= 0 ? iters_per_row : local_search_iters(S);
  const int G = lanes_per_state;
  std::vector<int> sorted(S);
  std::iota(sorted.begin(), sorted.end(), 0);
  std::stable_sort(sorted.begin(), sorted.end(), [&](int x, int y) {
    return (ptr[x + 1] - ptr[x]) > (ptr[y + 1] - ptr[y]);
  });
  // Bank-balanced tiles: a tile's 32 lanes write their states' column entries
  // (and, backward, read alpha[state]) in one warp-wide access, conflict-free
  // iff the states have distinct residues mod 32.  States of equal degree are
  // interchangeable in the degree-sorted order (trips and padding unchanged),
  // so each lane position takes an unused state of the degree it needs whose
  // residue the tile does not hold yet, when one exists.
  std::vector<int> order;
  order.reserve(S);
  if (optimize && G == 1) {
    // per degree: pool of states bucketed by residue
    std::vector<int> deg_of(S);
    int maxdeg = 0;
    for (int st = 0; st < S; ++st) maxdeg = std::max(maxdeg, deg_of[st] = ptr[st + 1] - ptr[st]);
    std::vector<std::array<std::vector<int>, 32>> pool(maxdeg + 1);
    for (int i = S - 1; i >= 0; --i) pool[deg_of[sorted[i]]][sorted[i] & 31].push_back(sorted[i]);
    std::vector<int> left(maxdeg + 1, 0);
    for (int st = 0; st < S; ++st) left[deg_of[st]]++;
    for (size_t t0 = 0; t0 < size_t(S); t0 += 32) {
      int cnt[32] = {0};
      const size_t t1 = std::min(size_t(S), t0 + 32);
      for (size_t k = t0; k < t1; ++k) {
        const int dg = deg_of[sorted[k]];  // the degree this sorted position needs
        // least-used residue in this tile; ties -> the largest remaining pool
        int pick = -1;
        for (int r = 0; r < 32; ++r) {
          if (pool[dg][r].empty()) continue;
          if (pick < 0 || cnt[r] < cnt[pick] ||
              (cnt[r] == cnt[pick] && pool[dg][r].size() > pool[dg][pick].size()))
            pick = r;
        }
        const int st = pool[dg][pick].back();
        pool[dg][pick].pop_back();
        cnt[st & 31]++;
        order.push_back(st);
      }
    }
  } else {
    order = sorted;
  }
  const int ntiles = (S * G + 31) / 32;
  // Tiles are independent: schedule them in parallel into per-tile fragments
  // (each with its own RNG seed, so the result does not depend on threading).
  auto do_tile = [&](int w, TileSchedule &ts) {
    const int base = 0;
    BankSet rb, eb;
    std::vector<std::vector<int>> rem(32);
    int trips = 0;
    for (int l = 0; l < 32; ++l) {
      const int k = (32 * w + l) / G, sub = (32 * w + l) % G;
      if (k >= S) {
        ts.info.push_back(0xFFFFu);
        continue;
      }
      const int s = order[k];
      for (int a = ptr[s] + sub; a < ptr[s + 1]; a += G) rem[l].push_back(a);
      const int deg = int(rem[l].size());
      ts.info.push_back(unsigned(s) | (unsigned(deg) << 16));
      trips = std::max(trips, deg);
    }
    ts.trips.push_back(trips);
    ts.base.push_back(base);
    const size_t start = ts.arc.size();
    ts.arc.resize(start + size_t(32) * trips, -1);
    ts.word_idx.resize(start + size_t(32) * trips, 0u);
    ts.word_b32.resize(start + size_t(32) * trips, 0u);
    ts.prob.resize(start + size_t(32) * trips, 0.0);
    std::vector<int> lanes;
    for (int j = 0; j < trips; ++j) {
      rb.clear();
      eb.clear();
      lanes.clear();
      for (int l = 0; l < 32; ++l)
        if (!rem[l].empty()) lanes.push_back(l);
      std::stable_sort(lanes.begin(), lanes.end(),
                       [&](int x, int y) { return rem[x].size() < rem[y].size(); });
      unsigned pad_idx = 0, pad_b32 = 0;
      bool have_pad = false;
      for (int l : lanes) {
        int best = 0, best_cost = 1 << 30, best_cr = 0, best_ce = 0;
        const int ncand = optimize ? int(rem[l].size()) : 1;
        for (int c = 0; c < ncand; ++c) {
          const int a = rem[l][c];
          int rc = 1 << 20, cr_best = 0;
          for (int cr = 0; cr < gl.rep_r; ++cr) {
            const int v = rb.cost(cr * gl.r_stride + gidx[a]);
            if (v < rc) {
              rc = v;
              cr_best = cr;
            }
          }
          int ec = 1 << 20, ce_best = 0;
          for (int ce = 0; ce < gl.rep_e; ++ce) {
            const int v = eb.cost(ce * gl.e_stride + pdf[a]);
            if (v < ec) {
              ec = v;
              ce_best = ce;
            }
          }
          if (!optimize) rc = ec = 0, cr_best = ce_best = 0;
          if (rc + ec < best_cost) {
            best_cost = rc + ec;
            best = c;
            best_cr = cr_best;
            best_ce = ce_best;
          }
        }
        const int a = rem[l][best];
        rem[l].erase(rem[l].begin() + best);
        const int ra = best_cr * gl.r_stride + gidx[a];
        const int ea = best_ce * gl.e_stride + pdf[a];
        rb.add(ra);
        eb.add(ea);
        const size_t slot = start + size_t(32) * j + l;
        ts.arc[slot] = a;
        ts.prob[slot] = prob[a];
        ts.word_idx[slot] = unsigned(gidx[a]) | (unsigned(pdf[a]) << 16);
        ts.word_b32[slot] = (unsigned(ra) << 2) | ((unsigned(ea) << 2) << 16);
        if (!have_pad) {
          pad_idx = ts.word_idx[slot];
          pad_b32 = ts.word_b32[slot];
          have_pad = true;
        }
      }
      // Idle lanes re-read an address already used in this row (a free
      // broadcast) with probability 0.
      for (int l = 0; l < 32; ++l) {
        const size_t slot = start + size_t(32) * j + l;
        if (ts.arc[slot] < 0) {
          ts.word_idx[slot] = pad_idx;
          ts.word_b32[slot] = pad_b32;
        }
      }
    }
    if (optimize && trips > 1 && ls_iters > 0) {
      // slots[j][l] = CSR arc at row j, lane l (-1 idle); search over lane permutations.
      std::vector<std::array<int, 32>> slots(trips);
      for (int j = 0; j < trips; ++j)
        for (int l = 0; l < 32; ++l) slots[j][l] = ts.arc[start + size_t(32) * j + l];
      std::vector<int> cost(trips);
      for (int j = 0; j < trips; ++j) cost[j] = eval_row(slots[j].data(), gidx, pdf, gl).cost;
      std::mt19937 rng(12345u + unsigned(w));
      const int iters = ls_iters * trips;
      for (int it = 0; it < iters; ++it) {
        const int l = int(rng() % 32u);
        const int j1 = int(rng() % unsigned(trips)), j2 = int(rng() % unsigned(trips));
        if (j1 == j2 || (slots[j1][l] < 0 && slots[j2][l] < 0)) continue;
        std::swap(slots[j1][l], slots[j2][l]);
        const int c1 = eval_row(slots[j1].data(), gidx, pdf, gl).cost;
        const int c2 = eval_row(slots[j2].data(), gidx, pdf, gl).cost;
        if (c1 + c2 <= cost[j1] + cost[j2]) {
          cost[j1] = c1;
          cost[j2] = c2;
        } else {
          std::swap(slots[j1][l], slots[j2][l]);
        }
      }
      for (int j = 0; j < trips; ++j) {
        const RowEval ev = eval_row(slots[j].data(), gidx, pdf, gl);
        unsigned pad_idx = 0, pad_b32 = 0;
        bool have_pad = false;
        for (int l = 0; l < 32; ++l) {
          const size_t slot = start + size_t(32) * j + l;
          const int a = slots[j][l];
          ts.arc[slot] = a;
          if (a < 0) continue;
          const int ra = ev.rcopy[l] * gl.r_stride + gidx[a];
          const int ea = ev.ecopy[l] * gl.e_stride + pdf[a];
          ts.prob[slot] = prob[a];
          ts.word_idx[slot] = unsigned(gidx[a]) | (unsigned(pdf[a]) << 16);
          ts.word_b32[slot] = (unsigned(ra) << 2) | ((unsigned(ea) << 2) << 16);
          if (!have_pad) {
            pad_idx = ts.word_idx[slot];
            pad_b32 = ts.word_b32[slot];
            have_pad = true;
          }
        }
        for (int l = 0; l < 32; ++l) {
          const size_t slot = start + size_t(32) * j + l;
          if (ts.arc[slot] < 0) {
            ts.prob[slot] = 0.0;
            ts.word_idx[slot] = pad_idx;
            ts.word_b32[slot] = pad_b32;
          }
        }
      }
    }
  };
  std::vector<TileSchedule> parts(ntiles);
  const int nthreads = std::max(1, std::min<int>(ntiles, int(std::thread::hardware_concurrency())));
  std::atomic<int> next{0};
  auto worker = [&] {
    for (int w = next++; w < ntiles; w = next++) do_tile(w, parts[w]);
  };
  if (nthreads == 1 || ntiles < 4) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int i = 0; i < nthreads; ++i) pool.emplace_back(worker);
    for (auto &t : pool) t.join();
  }
  TileSchedule ts;
  for (const TileSchedule &p : parts) {
    const int off = int(ts.arc.size());
    ts.info.insert(ts.info.end(), p.info.begin(), p.info.end());
    ts.trips.push_back(p.trips[0]);
    ts.base.push_back(off);
    ts.arc.insert(ts.arc.end(), p.arc.begin(), p.arc.end());
    ts.word_idx.insert(ts.word_idx.end(), p.word_idx.begin(), p.word_idx.end());
    ts.word_b32.insert(ts.word_b32.end(), p.word_b32.begin(), p.word_b32.end());
    ts.prob.insert(ts.prob.end(), p.prob.begin(), p.prob.end());
  }
  return ts;
}

void assign_xslots(const TileSchedule &tb, const int *pdf_of_arc, int num_pdfs, int num_arcs,
                   int slack, std::vector<int> &pdf_ptr, std::vector<int> &xslot_of_slot,
                   int &xpad) {
  std::vector<int> cnt(num_pdfs, 0);
  for (int a = 0; a < num_arcs; ++a) cnt[pdf_of_arc[a]]++;
  pdf_ptr.assign(num_pdfs + 1, 0);
  for (int p = 0; p < num_pdfs; ++p)
    pdf_ptr[p + 1] = pdf_ptr[p] + (cnt[p] ? ((cnt[p] + slack + 3) & ~3) : 0);
  const int dummy = pdf_ptr[num_pdfs];
  xpad = (dummy + 1 + 3) & ~3;
  // free positions per (pdf, bank)
  std::vector<std::vector<int>> freel(size_t(num_pdfs) * 32);
  for (int p = 0; p < num_pdfs; ++p)
    for (int pos = pdf_ptr[p + 1] - 1; pos >= pdf_ptr[p]; --pos)
      freel[size_t(p) * 32 + (pos & 31)].push_back(pos);
  xslot_of_slot.assign(tb.arc.size(), dummy);
  constexpr bool greedy_only = false;  // (bipartite matching: 1.13 -> 1.00 wavefronts/row)
  long waves = 0, rows = 0;
  for (size_t w = 0; w < tb.trips.size(); ++w) {
    for (int j = 0; j < tb.trips[w]; ++j) {
      const size_t row = size_t(tb.base[w]) + size_t(32) * j;
      // Each lane's store goes to a bank where its pdf still has a free
      // position; a row costs one wavefront per store in its busiest bank.
      // Maximum bipartite matching lanes -> banks (augmenting paths, lanes with
      // the fewest candidate banks first, banks with the most free positions
      // first), then the unmatched lanes go to their roomiest bank.
      int bank_of[32], lane_of_bank[32], order[32], nopt[32];
      std::fill(bank_of, bank_of + 32, -1);
      std::fill(lane_of_bank, lane_of_bank + 32, -1);
      bool used_dummy = false;
      int nl = 0;
      for (int l = 0; l < 32; ++l) {
        const int a = tb.arc[row + l];
        if (a < 0) {
          used_dummy = true;
          continue;
        }
        const int p = pdf_of_arc[a];
        nopt[l] = 0;
        for (int b = 0; b < 32; ++b) nopt[l] += !freel[size_t(p) * 32 + b].empty();
        order[nl++] = l;
      }
      if (used_dummy) lane_of_bank[dummy & 31] = 32;  // padding lanes' store (dummy slot)
      std::stable_sort(order, order + nl, [&](int x, int y) { return nopt[x] < nopt[y]; });
      auto pdf_l = [&](int l) { return pdf_of_arc[tb.arc[row + l]]; };
      auto cands = [&](int l, int *bs) {  // candidate banks, most free positions first
        const int p = pdf_l(l);
        int n = 0;
        for (int b = 0; b < 32; ++b)
          if (!freel[size_t(p) * 32 + b].empty()) bs[n++] = b;
        std::stable_sort(bs, bs + n, [&](int x, int y) {
          return freel[size_t(p) * 32 + x].size() > freel[size_t(p) * 32 + y].size();
        });
        return n;
      };
      if (!greedy_only) {
        for (int k = 0; k < nl; ++k) {
          const int l0 = order[k];
          bool seen[32] = {false};
          // DFS augmenting path from l0
          std::function<bool(int)> aug = [&](int l) -> bool {
            int bs[32];
            const int n = cands(l, bs);
            for (int q = 0; q < n; ++q) {
              const int b = bs[q];
              if (seen[b]) continue;
              seen[b] = true;
              const int o = lane_of_bank[b];
              if (o == 32) continue;  // reserved for the padding lanes
              if (o < 0 || aug(o)) {
                lane_of_bank[b] = l;
                bank_of[l] = b;
                return true;
              }
            }
            return false;
          };
          aug(l0);
        }
      }
      int mult[32] = {0};
      if (used_dummy) mult[dummy & 31] = 1;
      for (int k = 0; k < nl; ++k) {
        const int l = order[k];
        const int p = pdf_l(l);
        int b = bank_of[l];
        if (b < 0 || freel[size_t(p) * 32 + b].empty()) {  // unmatched: least-loaded bank
          int best = -1;
          for (int c = 0; c < 32; ++c) {
            if (freel[size_t(p) * 32 + c].empty()) continue;
            if (best < 0 || mult[c] < mult[best] ||
                (mult[c] == mult[best] &&
                 freel[size_t(p) * 32 + c].size() > freel[size_t(p) * 32 + best].size()))
              best = c;
          }
          b = best;
        }
        auto &fl = freel[size_t(p) * 32 + b];
        xslot_of_slot[row + l] = fl.back();
        fl.pop_back();
        ++mult[b];
      }
      waves += *std::max_element(mult, mult + 32);
      ++rows;
    }
  }
  if (options().debug)
    std::fprintf(stderr, "[lfmmi] xslot stores: %ld rows, %.3f wavefronts/row (%s)\n", rows,
                 rows ? double(waves) / double(rows) : 0.0, greedy_only ? "greedy" : "matching");
}

void warp_lists(const std::vector<int> &trips, const std::vector<int> &bias,
                std::vector<int> &table, std::vector<int> &list) {
  const int nw = kTableNW, nt = int(trips.size());
  std::vector<int> order(nt);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return trips[x] > trips[y]; });
  std::vector<long> load(nw, 0);
  for (int w = 0; w < nw; ++w) load[w] = w < int(bias.size()) ? bias[w] : 0;
  std::vector<std::vector<int>> per(nw);
  for (int t : order) {
    int best = 0;
    for (int w = 1; w < nw; ++w)
      if (load[w] < load[best]) best = w;
    per[best].push_back(t);
    load[best] += trips[t];
  }
  table.assign(kWarpTable, 0);
  list.clear();
  for (int w = 0; w < nw; ++w) {
    table[w] = int(list.size());
    list.insert(list.end(), per[w].begin(), per[w].end());
  }
  table[nw] = int(list.size());
  std::vector<int> by_load(nw);
  std::iota(by_load.begin(), by_load.end(), 0);
  std::stable_sort(by_load.begin(), by_load.end(),
                   [&](int x, int y) { return load[x] < load[y]; });
  for (int w = 0; w < nw; ++w) table[nw + 1 + w] = by_load[w];
}

}  // namespace lfmmi
