// lfmmi_options.h: one options struct for the whole library.
#include "lfmmi_options.h"

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "lfmmi_internal.h"

namespace lfmmi {
namespace {

struct Field {
  const char *name;
  int Options::*i;
  std::string Options::*s;
};

const Field kFields[] = {
    {"tile", &Options::tile, nullptr},
    {"stream", &Options::stream, nullptr},
    {"linear", &Options::linear, nullptr},
    {"linear_split", &Options::linear_split, nullptr},
    {"linear_k16", &Options::linear_k16, nullptr},
    {"linear_k16w", &Options::linear_k16w, nullptr},
    {"split", &Options::split, nullptr},
    {"split_clusters", &Options::split_clusters, nullptr},
    {"split_h64", &Options::split_h64, nullptr},
    {"stream_mode", nullptr, &Options::stream_mode},
    {"stream_ring", &Options::stream_ring, nullptr},
    {"ssplit_ring", &Options::ssplit_ring, nullptr},
    {"num_group", &Options::num_group, nullptr},
    {"small_arcs", &Options::small_arcs, nullptr},
    {"small_indeg", &Options::small_indeg, nullptr},
    {"tile_xdb", &Options::tile_xdb, nullptr},
    {"tile_persist", &Options::tile_persist, nullptr},
    {"serial", &Options::serial, nullptr},
    {"emit", &Options::emit, nullptr},
    {"sched_iters", &Options::sched_iters, nullptr},
    {"chore_bias", &Options::chore_bias, nullptr},
    {"tile_g", &Options::tile_g, nullptr},
    {"debug", &Options::debug, nullptr},
    {"profile", nullptr, &Options::profile},
};

const Field *find(const char *name) {
  for (const Field &f : kFields)
    if (std::strcmp(f.name, name) == 0) return &f;
  return nullptr;
}

int set(Options &o, const char *name, const char *value) {
  const Field *f = find(name);
  if (!f) return set_error(LFMMI_ERR_INVALID, std::string("unknown option '") + name + "'");
  if (f->s) {
    o.*(f->s) = value ? value : "";
    return LFMMI_OK;
  }
  char *end = nullptr;
  const long v = std::strtol(value ? value : "", &end, 10);
  if (!value || !*value || *end)
    return set_error(LFMMI_ERR_INVALID, std::string("option '") + name + "' needs an integer");
  o.*(f->i) = int(v);
  return LFMMI_OK;
}

}  // namespace

Options &options() {
  static Options opts;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *env = std::getenv("LFMMI_OPTIONS");
    if (!env) return;
    std::string s(env);
    size_t pos = 0;
    while (pos <= s.size()) {
      const size_t comma = std::min(s.find(',', pos), s.size());
      const std::string kv = s.substr(pos, comma - pos);
      const size_t eq = kv.find('=');
      if (eq != std::string::npos)
        set(opts, kv.substr(0, eq).c_str(), kv.substr(eq + 1).c_str());
      pos = comma + 1;
    }
  });
  return opts;
}

}  // namespace lfmmi

using namespace lfmmi;

extern "C" int lfmmi_set_option(const char *name, const char *value) {
  if (!name) return set_error(LFMMI_ERR_INVALID, "lfmmi_set_option: NULL name");
  return set(options(), name, value);
}

extern "C" int lfmmi_get_option(const char *name, char *buf, size_t len) {
  if (!name || !buf || !len) return set_error(LFMMI_ERR_INVALID, "lfmmi_get_option: bad buffer");
  const Field *f = find(name);
  if (!f) return set_error(LFMMI_ERR_INVALID, std::string("unknown option '") + name + "'");
  const Options &o = options();
  const std::string v = f->s ? o.*(f->s) : std::to_string(o.*(f->i));
  std::strncpy(buf, v.c_str(), len - 1);
  buf[len - 1] = '\0';
  return LFMMI_OK;
}

extern "C" int lfmmi_reset_options(void) {
  options() = Options{};
  return LFMMI_OK;
}
