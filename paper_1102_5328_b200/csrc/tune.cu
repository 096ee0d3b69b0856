// tune.cu -- tileqr_tune: the paper's two-step empirical tuning of (NB, IB)
// on the GPU.
//
//   Step 1: benchmark the dominant kernel, SSRFB, for every
//     (NB, IB) of the grid: one warm-up then 50 back-to-back batched launches
//     on the same buffers ("No Flush"), timed at once with
//     CUDA events; rate = 50 * batch * 4 NB^3 / t (nominal flops).
//   Pre-selection: Property 1 (orthogonal pruning), upper
//     convex hull (Property 2 / Heuristic 0), Heuristic 1
//     (steepness) or 2 (iso-segments), cap 8.
//   Step 2: factorizations on a ladder of matrix orders
//     ascending to N, 6 runs per candidate (median), P =
//     4/3 N^3 / t; after each rung Property 3 ("prune as you go") drops NB2
//     when some NB1 > NB2 is strictly faster.
// Readings of the unclear points (tie rules, first hull point, iso-segment
// count) are DESIGN.md R13/R14.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "internal.h"

namespace tileqr {
namespace {

struct Pt {
  int nb, ib;
  double g;
};

// Property 1: per NB the IB of the highest rate; every IB within tie_rel of
// that rate counts as tied and the largest tied IB is kept (R13,
// R18), with its own rate.
std::vector<Pt> orthogonal_prune(const std::vector<Pt>& in, double tie_rel) {
  std::map<int, double> gmax;
  for (const Pt& p : in) {
    auto it = gmax.find(p.nb);
    if (it == gmax.end() || p.g > it->second) gmax[p.nb] = p.g;
  }
  std::map<int, Pt> best;
  for (const Pt& p : in) {
    if (!(p.g >= gmax[p.nb] * (1.0 - tie_rel))) continue;
    auto it = best.find(p.nb);
    if (it == best.end() || p.ib > it->second.ib || (p.ib == it->second.ib && p.g > it->second.g)) best[p.nb] = p;
  }
  std::vector<Pt> out;
  for (auto& kv : best) out.push_back(kv.second);
  return out;  // sorted by nb
}

// upper hull, strictly decreasing slopes (collinear interior points dropped)
std::vector<Pt> upper_hull(const std::vector<Pt>& pts) {
  std::vector<Pt> h;
  for (const Pt& q : pts) {
    while (h.size() >= 2) {
      const Pt& o = h[h.size() - 2];
      const Pt& a = h[h.size() - 1];
      const long double cross = (long double)(a.nb - o.nb) * ((long double)q.g - o.g) -
                                ((long double)a.g - o.g) * (long double)(q.nb - o.nb);
      if (cross >= 0) h.pop_back();
      else break;
    }
    h.push_back(q);
  }
  return h;
}

// incoming steepness; the first hull point's segment starts at the origin (R13)
long double slope_in(const std::vector<Pt>& h, size_t i) {
  if (i == 0) return (long double)h[0].g / (long double)h[0].nb;
  return ((long double)h[i].g - h[i - 1].g) / (long double)(h[i].nb - h[i - 1].nb);
}

std::vector<Pt> heuristic1(const std::vector<Pt>& h, int cap) {
  std::vector<size_t> idx;
  for (size_t i = 0; i < h.size(); ++i) idx.push_back(i);
  std::stable_sort(idx.begin(), idx.end(), [&](size_t x, size_t y) {
    const long double sx = slope_in(h, x), sy = slope_in(h, y);
    if (sx != sy) return sx > sy;
    return h[x].nb < h[y].nb;
  });
  if ((int)idx.size() > cap) idx.resize(cap);
  std::sort(idx.begin(), idx.end());
  std::vector<Pt> out;
  for (size_t i : idx) out.push_back(h[i]);
  return out;
}

std::vector<Pt> heuristic2(const std::vector<Pt>& h, int cap) {
  if (h.size() <= 1) return h;
  const long double x0 = h.front().nb, x1 = h.back().nb;
  const long double width = (x1 - x0) / cap;
  std::map<int, size_t> best;  // segment -> hull index
  for (size_t i = 0; i < h.size(); ++i) {
    int seg = (h[i].nb == h.back().nb) ? cap - 1 : (int)((h[i].nb - x0) / width);
    if (seg >= cap) seg = cap - 1;
    auto it = best.find(seg);
    if (it == best.end() || slope_in(h, i) > slope_in(h, it->second)) best[seg] = i;
  }
  std::vector<size_t> idx;
  for (auto& kv : best) idx.push_back(kv.second);
  std::sort(idx.begin(), idx.end());
  std::vector<Pt> out;
  for (size_t i : idx) out.push_back(h[i]);
  return out;
}

std::vector<Pt> preselect(const std::vector<Pt>& samples, int heuristic, int cap, double tie_rel) {
  std::vector<Pt> hull = upper_hull(orthogonal_prune(samples, tie_rel));
  if (heuristic == 1) return heuristic1(hull, cap);
  if (heuristic == 2) return heuristic2(hull, cap);
  return hull;
}

std::string pts_json(const std::vector<Pt>& v) {
  std::string s = "[";
  char buf[128];
  for (size_t i = 0; i < v.size(); ++i) {
    snprintf(buf, sizeof buf, "%s{\"nb\": %d, \"ib\": %d, \"gflops\": %.17g}", i ? ", " : "", v[i].nb,
             v[i].ib, v[i].g);
    s += buf;
  }
  return s + "]";
}

#define TQ_TRY(call)                 \
  do {                               \
    int rc_ = (call);                \
    if (rc_) { cleanup(); return rc_; } \
  } while (0)

}  // namespace
}  // namespace tileqr

using namespace tileqr;

extern "C" {

int tileqr_preselect(int n, const int* h_nb, const int* h_ib, const double* h_gflops, int heuristic,
                     int cap, int* h_out_nb, int* h_out_ib, double* h_out_gflops, int* n_out) {
  return tileqr_preselect_tie(n, h_nb, h_ib, h_gflops, heuristic, cap, 0.0, h_out_nb, h_out_ib, h_out_gflops,
                              n_out);
}

int tileqr_preselect_tie(int n, const int* h_nb, const int* h_ib, const double* h_gflops, int heuristic,
                         int cap, double tie_rel, int* h_out_nb, int* h_out_ib, double* h_out_gflops,
                         int* n_out) {
  if (n < 1) { set_error("tileqr_preselect: empty dataset"); return -1; }
  if (!h_nb) return -2;
  if (!h_ib) return -3;
  if (!h_gflops) return -4;
  if (heuristic < 0 || heuristic > 2) return -5;
  if (cap < 1) return -6;
  if (!(tie_rel >= 0.0 && tie_rel < 1.0)) return -7;
  if (!h_out_nb || !h_out_ib || !h_out_gflops || !n_out) return -8;
  std::vector<Pt> s;
  for (int i = 0; i < n; ++i) s.push_back({h_nb[i], h_ib[i], h_gflops[i]});
  std::vector<Pt> out = preselect(s, heuristic, cap, tie_rel);
  for (size_t i = 0; i < out.size(); ++i) {
    h_out_nb[i] = out[i].nb;
    h_out_ib[i] = out[i].ib;
    h_out_gflops[i] = out[i].g;
  }
  *n_out = (int)out.size();
  return 0;
}

int tileqr_payg_prune(int n, const int* h_nb, const double* h_gflops, int* h_keep) {
  if (n < 0) return -1;
  if (!h_nb && n) return -2;
  if (!h_gflops && n) return -3;
  if (!h_keep && n) return -4;
  for (int i = 0; i < n; ++i) {
    h_keep[i] = 1;
    for (int j = 0; j < n; ++j)
      if (h_nb[j] > h_nb[i] && h_gflops[j] > h_gflops[i]) h_keep[i] = 0;
  }
  return 0;
}

int tileqr_tune(int64_t M, int64_t N, int ngpus, int heuristic, int payg, int* h_NB, int* h_IB,
                const char* report_json_path) {
  static const char* fn = "tileqr_tune";
  char msg[256];
  if (M < 1) { snprintf(msg, sizeof msg, "%s: M < 1", fn); set_error(msg); return -1; }
  if (N < 1) { snprintf(msg, sizeof msg, "%s: N < 1", fn); set_error(msg); return -2; }
  int P = 1, me = 0;
  if (ngpus < 1) { snprintf(msg, sizeof msg, "%s: ngpus < 1", fn); set_error(msg); return -3; }
  if (ngpus > 1 && M != N) { snprintf(msg, sizeof msg, "%s: ngpus > 1 tunes square problems", fn); set_error(msg); return -3; }
  if (ngpus > 1) {  // collective over the ranks of tileqr_dist_init: Step 2 times tileqr_dist_factor
    if (dist_ranks(&P, &me) || P != ngpus) {
      snprintf(msg, sizeof msg, "%s: ngpus = %d needs tileqr_dist_init with as many ranks", fn, ngpus);
      set_error(msg);
      return -3;
    }
  }
  // TILEQR_TUNE_DIST=1 (with tileqr_dist_init done): Step 2 through tileqr_dist_factor even on one
  // rank -- the ngpus > 1 code path on a single GPU (tests)
  bool use_dist = P > 1;
  if (const char* e = getenv("TILEQR_TUNE_DIST"))
    if (e[0] == '1' && dist_ranks(&P, &me) == 0 && P == ngpus) use_dist = true;
  if (heuristic < 0 || heuristic > 2) { set_error("tileqr_tune: heuristic not in {0,1,2}"); return -4; }
  if (!h_NB) return -6;
  if (!h_IB) return -7;

  const char* e_batch = getenv("TILEQR_TUNE_BATCH");
  const int batch = e_batch ? atoi(e_batch) : 4096;
  const char* e_small = getenv("TILEQR_TUNE_SMALL_IB");
  const int ib_min = (e_small && e_small[0] == '1') ? 1 : 8;
  const char* e_reps = getenv("TILEQR_TUNE_REPS");
  const int reps = e_reps ? atoi(e_reps) : 50;
  const int nb_grid[] = {64, 96, 128, 160, 192, 224, 256};
  // TILEQR_TUNE_FLUSH=1: Step 1 with an L2 flush before every timed call
  const char* e_flush = getenv("TILEQR_TUNE_FLUSH");
  const bool flush = e_flush && e_flush[0] == '1';
  const size_t flush_bytes = (size_t)512 << 20;  // 4x the 126 MB L2
  void* flushbuf = nullptr;
  const int nbmax = 256;

  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  double* buf = nullptr;
  double** ptrs = nullptr;
  double* pkbuf = nullptr;  // packed reflector tiles of the step-1 batch
  double** pkp = nullptr;
  size_t pk_cap = 0;
  double* A0 = nullptr;
  double* A = nullptr;
  double* T = nullptr;
  int* dinfo = nullptr;
  auto cleanup = [&]() {
    if (s) cudaStreamSynchronize(s);
    cudaFree(buf); cudaFree(ptrs); cudaFree(pkbuf); cudaFree(pkp); cudaFree(flushbuf); cudaFree(A0); cudaFree(A); cudaFree(T); cudaFree(dinfo);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
  };
  TQ_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
  if (flush) TQ_TRY(cudaMalloc(&flushbuf, flush_bytes) == cudaSuccess ? 0 : TILEQR_ERR_ALLOC);
  TQ_TRY(cudaEventCreate(&e0) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
  TQ_TRY(cudaEventCreate(&e1) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);

  // ---- Step 1: SSRFB sweep ---------------------------------------------------
  const size_t tile_max = (size_t)nbmax * nbmax;
  if (cudaMalloc(&buf, (size_t)batch * (4 * tile_max + tile_max) * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ptrs, (size_t)batch * 5 * sizeof(double*)) != cudaSuccess ||
      cudaMalloc(&pkp, (size_t)batch * sizeof(double*)) != cudaSuccess) {
    cudaGetLastError();
    set_error("tileqr_tune: step-1 allocation failed");
    cleanup();
    return TILEQR_ERR_ALLOC;
  }
  std::vector<Pt> samples;
  std::vector<double*> hp(5 * (size_t)batch);
  for (int nb : nb_grid) {
    const size_t tile = (size_t)nb * nb;
    for (int i = 0; i < batch; ++i) {
      double* base = buf + (size_t)i * 5 * tile;
      hp[i] = base;                        // R (top)
      hp[batch + i] = base + tile;         // V2 (TSQRT bottom)
      hp[2 * batch + i] = base + 2 * tile; // C1
      hp[3 * batch + i] = base + 3 * tile; // C2
      hp[4 * batch + i] = base + 4 * tile; // T (IB x NB <= NB x NB)
    }
    TQ_TRY(cudaMemcpy(ptrs, hp.data(), hp.size() * sizeof(double*), cudaMemcpyHostToDevice) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
    TQ_TRY(launch_rng_uniform((int64_t)tile, (int64_t)batch * 5, buf, (int64_t)tile, 2, 0, s));
    for (int ib = ib_min; ib <= nb; ++ib) {
      if (nb % ib) continue;
      // V2, T from a TSQRT of (top, bottom); fresh bottoms each time are not
      // needed for timing: the reflector values only scale the data.
      // Time the kernel tileqr_factor runs for this (NB, IB): the packed-
      // reflector update (operands packed once, outside the timing) where
      // available -- at IBe = lcm(IB, 8) for the IB it runs that way (DESIGN.md
      // R23; a tie with IBe itself then goes to IBe, the larger) -- else the
      // staged DMMA / SIMT update.  IB > 64 keeps its own (generic) kernel
      // here: timed at its divisor IBs it would tie with IBs and, as the larger
      // IB, take Property 1's tie (R18) for a blocking whose T is assembled
      // after the factorization.
      const int ibk = ib > 64 ? ib : effective_ib(nb, ib);
      const bool pk = v2_supported(nb, ibk);
      TQ_TRY(launch_tsqrt(nb, pk ? ibk : ib, batch, ptrs, ptrs + batch, ptrs + 4 * batch, s));
      if (pk) {
        const size_t pd = v2_pk_doubles(nb, ibk);
        if (pd > pk_cap) {
          cudaFree(pkbuf);
          pkbuf = nullptr;
          if (cudaMalloc(&pkbuf, pd * batch * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            set_error("tileqr_tune: step-1 packed buffer allocation failed");
            cleanup();
            return TILEQR_ERR_ALLOC;
          }
          pk_cap = pd;
        }
        TQ_TRY(launch_fill_ptrs(pkp, pkbuf, pd, batch, s));
        TQ_TRY(launch_pack(false, nb, ibk, batch, ptrs + batch, ptrs + 4 * batch, pkp, s));
      }
      auto one = [&]() -> int {
        if (pk) return launch_update_pk(false, nb, ibk, batch, pkp, ptrs + 2 * batch, ptrs + 3 * batch, s);
        return launch_ssrfb(true, nb, ib, batch, ptrs + batch, ptrs + 4 * batch, ptrs + 2 * batch,
                            ptrs + 3 * batch, nb, s);
      };
      TQ_TRY(one());  // warm-up
      float ms = 0.f;
      if (!flush) {  // No Flush: reps back-to-back calls timed at once
        TQ_TRY(cudaEventRecord(e0, s) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
        for (int r = 0; r < reps; ++r) TQ_TRY(one());
        TQ_TRY(cudaEventRecord(e1, s) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
        TQ_TRY(cudaEventSynchronize(e1) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
        cudaEventElapsedTime(&ms, e0, e1);
      } else {  // flushed (the MultCallFlushLRU idea): every call
                // timed alone after overwriting a buffer larger than L2
        for (int r = 0; r < reps; ++r) {
          TQ_TRY(cudaMemsetAsync(flushbuf, r & 0xff, flush_bytes, s) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
          TQ_TRY(cudaEventRecord(e0, s) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
          TQ_TRY(one());
          TQ_TRY(cudaEventRecord(e1, s) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
          TQ_TRY(cudaEventSynchronize(e1) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
          float m1 = 0.f;
          cudaEventElapsedTime(&m1, e0, e1);
          ms += m1;
        }
      }
      const double g = (double)reps * batch * 4.0 * nb * nb * (double)nb / (ms * 1e-3) / 1e9;
      samples.push_back({nb, ib, g});
      // keep magnitudes bounded across the repeated in-place updates
      TQ_TRY(launch_rng_uniform((int64_t)tile, (int64_t)batch * 5, buf, (int64_t)tile, 2, 0, s));
    }
  }
  cudaFree(buf);
  buf = nullptr;
  cudaFree(pkbuf);
  pkbuf = nullptr;
  cudaFree(pkp);
  pkp = nullptr;
  if (use_dist) {  // every rank decides on rank 0's Step-1 data set (identical candidates everywhere)
    std::vector<double> g(samples.size());
    for (size_t i = 0; i < samples.size(); ++i) g[i] = samples[i].g;
    TQ_TRY(dist_host_collective(g.data(), (int)g.size(), 0));
    for (size_t i = 0; i < samples.size(); ++i) samples[i].g = g[i];
  }
  // Property-1 ties within the Step-1 timing's repeatability (R18;
  // TILEQR_TUNE_TIE overrides the relative width)
  double tie_rel = 0.005;
  if (const char* e = getenv("TILEQR_TUNE_TIE")) tie_rel = atof(e);
  if (!(tie_rel >= 0.0 && tie_rel < 1.0)) tie_rel = 0.005;
  std::vector<Pt> cand = preselect(samples, heuristic, 8, tie_rel);

  // ---- Step 2: factorizations on a ladder ascending to N --------------------
  std::vector<int64_t> ladder;
  for (int64_t d : {4, 2, 1}) {
    const int64_t n = std::max<int64_t>(64, N / d);
    if (ladder.empty() || n > ladder.back()) ladder.push_back(n);
  }
  const double ratio = (double)M / (double)N;
  std::string step2 = "[";
  std::vector<Pt> alive = cand;
  std::vector<Pt> last;
  for (size_t li = 0; li < ladder.size(); ++li) {
    const int64_t n = ladder[li];
    const int64_t m = std::max<int64_t>(1, (int64_t)(ratio * n + 0.5));
    cudaFree(A0); cudaFree(A); cudaFree(T); cudaFree(dinfo);
    A0 = A = T = nullptr;
    dinfo = nullptr;
    size_t tn = 0;
    tileqr_t_size(m, n, 8, 8, &tn);
    size_t tmax = 0;
    for (const Pt& p : alive) {
      size_t t = 0;
      tileqr_t_size(m, n, p.nb, p.ib, &t);
      tmax = std::max(tmax, t);
    }
    const size_t nmat = use_dist ? 1 : (size_t)m * n;  // ngpus > 1: per-candidate local buffers below
    if (cudaMalloc(&A0, nmat * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&A, nmat * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&T, (use_dist ? 1 : std::max<size_t>(tmax, 1)) * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&dinfo, sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      set_error("tileqr_tune: step-2 allocation failed");
      cleanup();
      return TILEQR_ERR_ALLOC;
    }
    if (!use_dist) TQ_TRY(launch_rng_uniform(m, n, A0, m, 3, 0, s));
    std::vector<Pt> res;
    for (const Pt& p : alive) {
      std::vector<float> times;
      if (use_dist) {  // tileqr_dist_factor on every rank; each run's time is the max over ranks
        int nloc = 0;
        TQ_TRY(tileqr_dist_local_cols(n, p.nb, &nloc));
        const int64_t mt = (m + p.nb - 1) / p.nb;
        double *dA0 = nullptr, *dA = nullptr, *dT = nullptr;
        const size_t na = std::max<size_t>(1, (size_t)nloc * mt * p.nb * p.nb), nt = std::max<size_t>(1, (size_t)nloc * mt * p.ib * p.nb);
        if (cudaMalloc(&dA0, na * 8) != cudaSuccess || cudaMalloc(&dA, na * 8) != cudaSuccess ||
            cudaMalloc(&dT, nt * 8) != cudaSuccess) {
          cudaGetLastError();
          cudaFree(dA0); cudaFree(dA); cudaFree(dT);
          set_error("tileqr_tune: step-2 allocation failed");
          cleanup();
          return TILEQR_ERR_ALLOC;
        }
        int rc2 = tileqr_dist_fill_uniform(m, n, p.nb, dA0, 3, (tileqr_stream_t)s);
        std::vector<double> tm(7, 0.0);
        for (int r = 0; r < 7 && !rc2; ++r) {
          cudaMemcpyAsync(dA, dA0, na * 8, cudaMemcpyDeviceToDevice, s);
          cudaEventRecord(e0, s);
          rc2 = tileqr_dist_factor(m, n, dA, p.nb, p.ib, dT, dinfo, (tileqr_stream_t)s);
          cudaEventRecord(e1, s);
          cudaEventSynchronize(e1);
          float ms = 0.f;
          cudaEventElapsedTime(&ms, e0, e1);
          tm[r] = ms;
        }
        if (!rc2) rc2 = dist_host_collective(tm.data(), 7, 1);
        cudaFree(dA0); cudaFree(dA); cudaFree(dT);
        TQ_TRY(rc2);
        for (int r = 1; r < 7; ++r) times.push_back((float)tm[r]);
      } else {
      for (int r = 0; r < 7; ++r) {  // 1 warm-up + 6 timed runs
        TQ_TRY(cudaMemcpyAsync(A, A0, (size_t)m * n * sizeof(double), cudaMemcpyDeviceToDevice, s) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
        TQ_TRY(cudaEventRecord(e0, s) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
        TQ_TRY(tileqr_factor(m, n, A, m, p.nb, p.ib, T, dinfo, (tileqr_stream_t)s));
        TQ_TRY(cudaEventRecord(e1, s) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
        TQ_TRY(cudaEventSynchronize(e1) == cudaSuccess ? 0 : TILEQR_ERR_CUDA);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0) times.push_back(ms);
      }
      {  // this candidate's workspace is not needed again at this N
        int dev = 0;
        cudaGetDevice(&dev);
        release_ws(dev, m, n, p.nb, p.ib);
      }
      }  // single GPU
      std::sort(times.begin(), times.end());
      const double med = 0.5 * (times[2] + times[3]);
      const double flops = (m >= n) ? 2.0 * m * (double)n * n - 2.0 * (double)n * n * n / 3.0
                                    : 2.0 * n * (double)m * m - 2.0 * (double)m * m * m / 3.0;
      const double g = flops / (med * 1e-3) / 1e9;
      res.push_back({p.nb, p.ib, g});
      char b[256];
      snprintf(b, sizeof b, "%s{\"n\": %lld, \"nb\": %d, \"ib\": %d, \"median_ms\": %.6f, \"gflops\": %.17g}",
               step2.size() > 1 ? ", " : "", (long long)n, p.nb, p.ib, med, g);
      step2 += b;
    }
    last = res;
    if (payg) {  // Property 3
      std::vector<Pt> keep;
      for (const Pt& q : res) {
        bool drop = false;
        for (const Pt& o : res)
          if (o.nb > q.nb && o.g > q.g) drop = true;
        if (!drop) keep.push_back(q);
      }
      alive = keep;
    }
  }
  step2 += "]";
  Pt best = last.front();
  for (const Pt& p : last)
    if (p.g > best.g) best = p;
  *h_NB = best.nb;
  *h_IB = best.ib;
  if (report_json_path) {
    FILE* f = fopen(report_json_path, "w");
    if (f) {
      fprintf(f, "{\"M\": %lld, \"N\": %lld, \"heuristic\": %d, \"payg\": %d, \"batch\": %d, \"reps\": %d, \"step1_timing\": \"%s\", \"tie_rel\": %.17g, \"ngpus\": %d,\n",
              (long long)M, (long long)N, heuristic, payg, batch, reps, flush ? "flush" : "no_flush", tie_rel, P);
      fprintf(f, " \"step1\": %s,\n \"candidates\": %s,\n \"step2\": %s,\n \"best\": {\"nb\": %d, \"ib\": %d, \"gflops\": %.17g}}\n",
              pts_json(samples).c_str(), pts_json(cand).c_str(), step2.c_str(), best.nb, best.ib, best.g);
      fclose(f);
    }
  }
  cleanup();
  return 0;
}

}  // extern "C"
