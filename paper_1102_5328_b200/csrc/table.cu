// table.cu -- the installed decision table of the autotuner and its lookup
// ("discretization of the space",
// "interpolation ... the closest point", "the pre-built
// decision tree is used" when the user calls the library).
//
// The table is the JSON file tools/autotune.py writes (atomically) after
// running tileqr_tune over the (N, ngpus) grid:
//   {"entries": [{"n": 2048, "ngpus": 1, "nb": 64, "ib": 32, ...}, ...]}
// found at $TILEQR_TUNED_TABLE, else as tuned_table.json beside
// libtileqr.so.  Lookup is per-axis nearest point, ties toward the larger
// grid value (R13), on the axes (order, ngpus); the order of an
// M x N problem is the square order with the same useful flop count,
// (3/4 * flops(M, N))^(1/3) (R19; = N for square matrices).
#include <dlfcn.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace tileqr {
namespace {

struct Entry {
  long long n;
  int ngpus, nb, ib;
};

std::mutex g_tab_mu;
std::vector<Entry> g_tab;
std::string g_tab_path;
bool g_tab_loaded = false;

std::string table_path() {
  if (const char* e = getenv("TILEQR_TUNED_TABLE")) return e;
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&table_path), &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    const size_t s = p.rfind('/');
    return (s == std::string::npos ? std::string(".") : p.substr(0, s)) + "/tuned_table.json";
  }
  return "tuned_table.json";
}

// integer value of "key": inside [b, e), or false
bool int_field(const std::string& s, size_t b, size_t e, const char* key, long long* out) {
  const std::string k = std::string("\"") + key + "\"";
  size_t p = s.find(k, b);
  if (p == std::string::npos || p >= e) return false;
  p = s.find(':', p + k.size());
  if (p == std::string::npos || p >= e) return false;
  char* end = nullptr;
  const long long v = strtoll(s.c_str() + p + 1, &end, 10);
  if (end == s.c_str() + p + 1) return false;
  *out = v;
  return true;
}

// Parse the entries of the table file; false if unreadable or empty.
bool load(const std::string& path, std::vector<Entry>* out) {
  FILE* f = fopen(path.c_str(), "rb");
  if (!f) return false;
  std::string s;
  char buf[4096];
  size_t n;
  while ((n = fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, n);
  fclose(f);
  size_t p = s.find("\"entries\"");
  if (p == std::string::npos) return false;
  p = s.find('[', p);
  const size_t end = p == std::string::npos ? p : s.find(']', p);
  if (end == std::string::npos) return false;
  std::vector<Entry> v;
  for (size_t b = s.find('{', p); b != std::string::npos && b < end; b = s.find('{', b + 1)) {
    const size_t e = s.find('}', b);
    if (e == std::string::npos) break;
    long long nn = 0, g = 0, nb = 0, ib = 0;
    if (int_field(s, b, e, "n", &nn) && int_field(s, b, e, "ngpus", &g) && int_field(s, b, e, "nb", &nb) &&
        int_field(s, b, e, "ib", &ib) && valid_nb_ib((int)nb, (int)ib) && nn > 0 && g > 0)
      v.push_back({nn, (int)g, (int)nb, (int)ib});
    b = e;
  }
  if (v.empty()) return false;
  *out = v;
  return true;
}

template <class T>
T nearest(const std::vector<T>& vals, double x) {
  T best = vals[0];
  for (T v : vals) {
    const double d = fabs((double)v - x), db = fabs((double)best - x);
    if (d < db || (d == db && v > best)) best = v;
  }
  return best;
}

}  // namespace

// Built-in pair when no table is installed: the tuner's pick at N = 10000 on
// the B200 (profiles/tune_r01_s3.json).
constexpr int kDefaultNB = 128, kDefaultIB = 16;

int lookup_pair(int64_t M, int64_t N, int ngpus, int* NB, int* IB, bool* from_table) {
  std::lock_guard<std::mutex> lock(g_tab_mu);
  const std::string path = table_path();
  if (!g_tab_loaded || path != g_tab_path) {
    g_tab.clear();
    load(path, &g_tab);
    g_tab_path = path;
    g_tab_loaded = true;
  }
  *NB = kDefaultNB;
  *IB = kDefaultIB;
  *from_table = false;
  if (g_tab.empty()) return 0;
  const double flops = (M >= N) ? 2.0 * M * (double)N * N - 2.0 * (double)N * N * N / 3.0
                                : 2.0 * N * (double)M * M - 2.0 * (double)M * M * M / 3.0;
  const double order = cbrt(0.75 * flops);
  std::vector<long long> ns;
  std::vector<int> gs;
  for (const Entry& e : g_tab) {
    ns.push_back(e.n);
    gs.push_back(e.ngpus);
  }
  const long long n0 = nearest(ns, order);
  const int g0 = nearest(gs, (double)ngpus);
  for (const Entry& e : g_tab)
    if (e.n == n0 && e.ngpus == g0) {
      *NB = e.nb;
      *IB = e.ib;
      *from_table = true;
      return 0;
    }
  // the grid is not a full product: nearest entry in (order, ngpus), order first
  const Entry* best = &g_tab[0];
  for (const Entry& e : g_tab) {
    const double d = fabs((double)e.n - order), db = fabs((double)best->n - order);
    if (d < db || (d == db && abs(e.ngpus - ngpus) < abs(best->ngpus - ngpus))) best = &e;
  }
  *NB = best->nb;
  *IB = best->ib;
  *from_table = true;
  return 0;
}

}  // namespace tileqr

extern "C" {

int tileqr_lookup(int64_t M, int64_t N, int ngpus, int* h_NB, int* h_IB) {
  if (M < 0) return -1;
  if (N < 0) return -2;
  if (ngpus < 1) return -3;
  if (!h_NB) return -4;
  if (!h_IB) return -5;
  bool found = false;
  tileqr::lookup_pair(M, N, ngpus, h_NB, h_IB, &found);
  if (!found) {
    tileqr::set_error("tileqr_lookup: no decision table (tuned_table.json beside libtileqr.so or "
                      "$TILEQR_TUNED_TABLE); built-in default returned");
    return TILEQR_ERR_NOT_INIT;
  }
  return 0;
}

}  // extern "C"
