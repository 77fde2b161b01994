// Native text-FST ingestion: parse the reference's
// acceptor text format straight into arc / final-weight arrays that
// lfmmi_graphs_create (and ChainGraph) consume.
//
// Format (same contract as /root/reference/pkg/src/chainloss/fst_io.py:1-17,
// 53-110): arc lines "src dst label [weight]" with label = pdf + 1 (0 is
// epsilon and rejected), final lines "state [weight]", weight = -ln(prob)
// defaulting to 0, '#' comments and blank lines ignored.  States are densely
// re-indexed in order of first appearance, so the first-mentioned state is 0
// (the start state).  Errors carry 1-based line numbers.
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "lfmmi_internal.h"

using namespace lfmmi;

namespace {

struct Parsed {
  std::vector<uint32_t> src, dst, pdf;
  std::vector<double> prob;
  std::vector<double> finals;  // per dense state, 0 = not final
  std::vector<char> is_final;
};

bool parse_uint(const char *b, const char *e, int64_t &out) {
  if (b == e) return false;
  bool neg = false;
  if (*b == '-' || *b == '+') {
    neg = *b == '-';
    ++b;
  }
  if (b == e) return false;
  int64_t v = 0;
  for (; b < e; ++b) {
    if (*b < '0' || *b > '9') return false;
    v = v * 10 + (*b - '0');
    if (v > (int64_t(1) << 40)) return false;
  }
  out = neg ? -v : v;
  return true;
}

bool parse_double(const char *b, const char *e, double &out) {
  std::string s(b, e);
  char *end = nullptr;
  errno = 0;
  out = std::strtod(s.c_str(), &end);
  return end == s.c_str() + s.size() && !s.empty();
}

int parse(const char *text, size_t len, int32_t num_pdfs, Parsed &p) {
  if (num_pdfs < 1) return set_error(LFMMI_ERR_INVALID, "num_pdfs must be >= 1");
  std::unordered_map<int64_t, uint32_t> dense;
  auto index_of = [&](int64_t id) {
    auto it = dense.find(id);
    if (it != dense.end()) return it->second;
    const uint32_t k = uint32_t(dense.size());
    dense.emplace(id, k);
    p.finals.push_back(0.0);
    p.is_final.push_back(0);
    return k;
  };
  size_t pos = 0;
  long lineno = 0;
  while (pos < len) {
    size_t end = pos;
    while (end < len && text[end] != '\n') ++end;
    ++lineno;
    const char *fld[5];
    const char *fle[5];
    int nf = 0;
    size_t i = pos;
    while (i < end) {
      while (i < end && (text[i] == ' ' || text[i] == '\t' || text[i] == '\r')) ++i;
      if (i >= end) break;
      const size_t s = i;
      while (i < end && text[i] != ' ' && text[i] != '\t' && text[i] != '\r') ++i;
      if (nf < 5) {
        fld[nf] = text + s;
        fle[nf] = text + i;
      }
      ++nf;
    }
    pos = end + 1;
    if (nf == 0 || fld[0][0] == '#') continue;
    const std::string at = "line " + std::to_string(lineno) + ": ";
    auto field_str = [&](int k) { return std::string(fld[k], fle[k]); };
    auto get_state = [&](int k, const char *what, int64_t &v) {
      if (!parse_uint(fld[k], fle[k], v))
        return set_error(LFMMI_ERR_INVALID, at + what + " is not an integer: '" + field_str(k) + "'");
      if (v < 0)
        return set_error(LFMMI_ERR_INVALID,
                         at + what + " must be non-negative, got " + std::to_string(v));
      return LFMMI_OK;
    };
    auto get_weight = [&](int k, double &w) {
      if (!parse_double(fld[k], fle[k], w))
        return set_error(LFMMI_ERR_INVALID, at + "weight is not a number: '" + field_str(k) + "'");
      if (!std::isfinite(w))
        return set_error(LFMMI_ERR_INVALID, at + "weight must be finite, got '" + field_str(k) + "'");
      return LFMMI_OK;
    };
    if (nf == 1 || nf == 2) {
      int64_t st;
      int rc = get_state(0, "state", st);
      if (rc) return rc;
      double w = 0.0;
      if (nf == 2 && (rc = get_weight(1, w))) return rc;
      const uint32_t s = index_of(st);
      if (p.is_final[s])
        return set_error(LFMMI_ERR_INVALID,
                         at + "duplicate final line for state " + field_str(0));
      p.is_final[s] = 1;
      p.finals[s] = std::exp(-w);
    } else if (nf == 3 || nf == 4) {
      int64_t a, b, lab;
      int rc = get_state(0, "src state", a);
      if (rc) return rc;
      if ((rc = get_state(1, "dst state", b))) return rc;
      if ((rc = get_state(2, "label", lab))) return rc;
      if (lab == 0) return set_error(LFMMI_ERR_INVALID, at + "label 0 is reserved for epsilon");
      if (lab > num_pdfs)
        return set_error(LFMMI_ERR_INVALID, at + "label " + std::to_string(lab) +
                                                " exceeds num_pdfs=" + std::to_string(num_pdfs));
      double w = 0.0;
      if (nf == 4 && (rc = get_weight(3, w))) return rc;
      const uint32_t s = index_of(a), d = index_of(b);
      p.src.push_back(s);
      p.dst.push_back(d);
      p.pdf.push_back(uint32_t(lab - 1));
      p.prob.push_back(std::exp(-w));
    } else {
      return set_error(LFMMI_ERR_INVALID, at + "expected 1-2 (final) or 3-4 (arc) fields, got " +
                                              std::to_string(nf));
    }
  }
  if (dense.empty()) return set_error(LFMMI_ERR_INVALID, "empty FST: no states mentioned");
  bool any_final = false;
  for (char f : p.is_final) any_final |= f != 0;
  if (!any_final) return set_error(LFMMI_ERR_INVALID, "no final state in FST");
  return LFMMI_OK;
}

}  // namespace

extern "C" int lfmmi_fst_text_size(const char *text, size_t length, int32_t num_pdfs,
                                   int64_t *num_states, int64_t *num_arcs) {
  if (!text || !num_states || !num_arcs)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_fst_text_size: NULL argument");
  Parsed p;
  const int rc = parse(text, length, num_pdfs, p);
  if (rc) return rc;
  *num_states = int64_t(p.finals.size());
  *num_arcs = int64_t(p.src.size());
  return LFMMI_OK;
}

extern "C" int lfmmi_fst_text_parse(const char *text, size_t length, int32_t num_pdfs,
                                    int64_t num_states, int64_t num_arcs, uint32_t *src,
                                    uint32_t *dst, uint32_t *pdf, double *prob,
                                    double *final_probs) {
  if (!text || (num_arcs && (!src || !dst || !pdf || !prob)) || !final_probs)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_fst_text_parse: NULL argument");
  Parsed p;
  const int rc = parse(text, length, num_pdfs, p);
  if (rc) return rc;
  if (int64_t(p.finals.size()) != num_states || int64_t(p.src.size()) != num_arcs)
    return set_error(LFMMI_ERR_INVALID, "lfmmi_fst_text_parse: sizes differ from lfmmi_fst_text_size");
  std::memcpy(src, p.src.data(), p.src.size() * 4);
  std::memcpy(dst, p.dst.data(), p.dst.size() * 4);
  std::memcpy(pdf, p.pdf.data(), p.pdf.size() * 4);
  std::memcpy(prob, p.prob.data(), p.prob.size() * 8);
  std::memcpy(final_probs, p.finals.data(), p.finals.size() * 8);
  return LFMMI_OK;
}
