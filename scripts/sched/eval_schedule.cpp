// Offline evaluation of the tile schedule's bank conflicts (max distinct addresses per bank per row).
#include <cstdio>
#include <vector>
#include <algorithm>
#include <numeric>
#include "lfmmi_schedule.h"
using namespace lfmmi;
int main() {
  FILE *f = fopen("/tmp/sched/den.bin", "rb");
  int hdr[3]; fread(hdr, 4, 3, f);
  int S = hdr[0], D = hdr[1], I = hdr[2];
  std::vector<int> src(I), dst(I), pdf(I); std::vector<double> prob(I);
  fread(src.data(), 4, I, f); fread(dst.data(), 4, I, f); fread(pdf.data(), 4, I, f); fread(prob.data(), 8, I, f);
  // CSR by destination (forward pack) in stable order
  std::vector<int> ord(I); std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b){ return dst[a] < dst[b]; });
  std::vector<int> ptr(S + 1, 0), g(I), pd(I); std::vector<double> pr(I);
  for (int i = 0; i < I; ++i) { ptr[dst[ord[i]] + 1]++; g[i] = src[ord[i]]; pd[i] = pdf[ord[i]]; pr[i] = prob[ord[i]]; }
  for (int s = 0; s < S; ++s) ptr[s + 1] += ptr[s];
  GatherLayout gl = make_gather_layout(S, D);
  for (int opt = 0; opt < 2; ++opt) {
    TileSchedule ts = schedule_tiles(S, ptr.data(), g.data(), pd.data(), pr.data(), gl, opt);
    long rows = 0, wr = 0, we = 0;
    for (size_t t = 0; t < ts.trips.size(); ++t)
      for (int j = 0; j < ts.trips[t]; ++j) {
        std::vector<std::vector<int>> rb(32), eb(32);
        for (int l = 0; l < 32; ++l) {
          unsigned w = ts.word_b32[ts.base[t] + 32 * j + l];
          int ra = (w & 0xFFFF) >> 2, ea = (w >> 16) >> 2;
          auto addu = [](std::vector<int> &v, int a) { if (std::find(v.begin(), v.end(), a) == v.end()) v.push_back(a); };
          addu(rb[ra & 31], ra); addu(eb[ea & 31], ea);
        }
        size_t mr = 0, me = 0;
        for (int b = 0; b < 32; ++b) { mr = std::max(mr, rb[b].size()); me = std::max(me, eb[b].size()); }
        rows++; wr += mr; we += me;
      }
    printf("optimize=%d rows=%ld r-gather wavefronts=%ld (%.2f/row) e-gather=%ld (%.2f/row)\n", opt, rows, wr, double(wr)/rows, we, double(we)/rows);
    if (opt) {  // posterior-slot stores (LFMMI_DEBUG_XSLOT prints wavefronts/row)
      std::vector<int> pp, xs; int xpad = 0;
      assign_xslots(ts, pd.data(), D, I, 4, pp, xs, xpad);
    }
  }
}
