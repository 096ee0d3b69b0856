// panel_fast.cuh -- device body of the low-latency GEQRT / TSQRT (
// SURVEY §8(a) rows a2, a4) for NB % 32 == 0, NB <= 256, IB in {8, 16, 24, 32}.
// Used by the batched panel kernel (kernels_panel_fast.cu) and by the
// dataflow DAG kernel (dag.cuh).  Every other (NB, IB) uses the generic
// panel kernel (kernels_panel.cu).
//
// One CTA of 8 warps per task.  For each inner panel p (IB columns):
//  1. Factor: the NB x IB panel lives in registers, lane l holding column l
//     and warp w rows [w*NB/8, (w+1)*NB/8).  Per column j ONE pass of partial
//     dot products gives sigma = ||x2||^2 and every d_c = x2 . P(:,c) (the
//     pivot column is broadcast with warp shuffles), one CTA barrier combines
//     the 8 warp partials (double-buffered, so no second barrier), and every
//     thread forms beta/tau (R1) and applies the rank-1 update to
//     its own registers.
//  2. T_p: the Gram matrix V_p^T V_p on DMMA (mma.sync.m8n8k4.f64) from the
//     staged panel, then the forward recurrence
//     T[0:i,i] = -tau_i T[0:i,0:i] G[0:i,i], one thread per row of T.
//  3. Trailing columns: each warp takes 8-column blocks, holds them for all
//     NB rows in registers (transposed accumulator) and applies
//     W = [R_p; C]^T-part ... exactly the SSRFB/LARFB steps A/B/C of
//     kernels_update.cu on DMMA, reading V_p (swizzled) and T_p from smem.
// TSQRT never writes the strict lower part of R (read concurrently by the
// LARFB of the same DAG level).  Global loads bypass L1
// (ld.global.cg): the persistent DAG kernel runs two CTAs per SM whose items
// hand tiles to other SMs, and L2 is the coherence point.
#pragma once

#include <math.h>

#include <type_traits>

#include "dmma.cuh"
#include "internal.h"
#include "update_v2.cuh"

#ifdef TILEQR_PANEL_PROF  // phase-cycle diagnostics: only kernels_panel_fast.cu is built with it
namespace tileqr { static __device__ unsigned long long g_panel_prof[16]; }  // per translation unit
#endif

namespace tileqr {
namespace pf {

constexpr int LDV = 40;   // >= 32, == 8 mod 16
constexpr int LDT = 36;   // == 4 mod 16
constexpr int LDW = 36;
constexpr int LDG = 33;
constexpr int LDR = 33;

template <int NB, int kWarps>
struct FastSmem {
  double Vs[NB * LDV];
  double Ts[32 * LDT];
  double Gs[32 * LDG];
  double Rin[32 * LDR];
  double Rout[32 * LDR];
  double red[2][kWarps][32];
  double rowj[2][32];
  double tau[32];
  double Ws[kWarps][8 * LDW];
  double Tsv[32 * LDT];  // T_p of the sub-task's earlier inner panels (step 3)
};

// Inner panels c0 = cbeg, cbeg+IB, ... < cend (the whole tile by default; the
// DAG kernel runs a TSQRT / GEQRT as several sub-tasks of consecutive inner
// panels, every state between them lives in global memory).
//
// TT (with TS): the TTQRT of the tree variant -- B is upper
// triangular: reflector j uses rows 0..j of column j of B, V2 is written to
// B's upper triangle (diagonal included) only, and rows of B below a
// column's diagonal are never read or written (they hold the GEQRT V of that
// tile, read by other kernels).  Its zeros enter the register panel, so the
// step loop, the Gram product and the packed copy are the TSQRT ones.
template <bool TS, int NB, int kWarps, int IB, bool TT = false>
__device__ __forceinline__ void panel_fast_body(double* const R, double* const Bx, double* const Tg,
                                                unsigned char* smem_raw, double* const Vpk = nullptr,
                                                int cbeg = 0, int cend = NB) {
  static_assert(IB % 8 == 0 && IB <= 32 && NB % IB == 0, "fast panel geometry");
  static_assert(TS || !TT, "TT is a TS variant");
  constexpr int TR = IB / kWarps > 0 ? IB / kWarps : 1;  // GEQRT: top rows per warp
  constexpr int kThreads = kWarps * 32;
  constexpr int RW = NB / kWarps;  // rows per warp in the factorization
  constexpr int RB = NB / 8;       // 8-row blocks in the trailing update
  // IB <= 16: HL lane groups of IB lanes share a column (group h holds rows
  // [w*RW + h*RL, w*RW + (h+1)*RL)), so no lane idles and the step issues
  // RW/HL instead of RW shuffles and FMAs per warp; their partial dots are
  // combined with shfl_xor (symmetric: every lane of a column gets the same
  // bits).  GEQRT's top-row slots live in group 0.
#ifdef TILEQR_GEQRT_HL1  // diagnostic: GEQRT with one column per lane (round 1)
  constexpr int HL = (TS && IB <= 16 && 32 % IB == 0) ? 32 / IB : 1;
#else
  // GEQRT too (round 2): at 2048^2 GEQRT sub-tasks were 62 % of the critical
  // path (tools/critical_path.py) with half the lanes idle at IB = 16; the
  // top-row slots (rows leaving the reflector) live in lane group 0 only
  constexpr int HL = (IB <= 16 && 32 % IB == 0) ? 32 / IB : 1;
#endif
  constexpr int RL = RW / HL;      // rows per lane
  FastSmem<NB, kWarps>& S = *reinterpret_cast<FastSmem<NB, kWarps>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a = lane & 3, g = lane >> 2;
  const int col = HL > 1 ? (lane % IB) : lane;  // the lane's panel column (>= IB: none)
  const int hg = HL > 1 ? (lane / IB) : 0;      // its lane group
  const int rbase = warp * RW + hg * RL;        // first row it holds
  double* const B = TS ? Bx : R;  // TSQRT: R tile + square tile B; GEQRT: the tile

  for (int e = tid; e < 32 * LDT; e += kThreads) S.Ts[e] = 0.0;  // zero padding for the T merges
  for (int e = tid; e < 32 * LDG; e += kThreads) S.Gs[e] = 0.0;
#ifdef TILEQR_PANEL_PROF
  long long tp0 = clock64(), tp1;
#define TQ_PHASE(k) do { if (tid == 0) { tp1 = clock64(); atomicAdd(&g_panel_prof[(k) + (TS ? 0 : 8)], (unsigned long long)(tp1 - tp0)); tp0 = tp1; } } while (0)
#else
#define TQ_PHASE(k) do { } while (0)
#endif
  const bool fuse = cend - cbeg > IB && cend - cbeg <= 32 && 32 % IB == 0;  // see step 3
  // Panel element idx (of NB * IB) in the order the stage and write-out loops
  // use: each warp instruction covers an 8-row x 4-column block, every 4 lanes
  // one 32-byte sector of a column (coalesced in global memory), every half
  // warp 16 distinct bank pairs of the swizzled Vs.  (Column-major order, 32
  // rows of one column per instruction, hit 4 bank pairs: 8-way conflicts.)
  // GEQRT only: for TSQRT the column-major order measured faster (batched
  // TSQRT +0.3-1.4 %, 10000^2 at IB = 32 +1.8 %; GEQRT -2 to -7 %,
  // profiles/r02z_panel_order_ab.log, r02z2_panel_order_geqrt_only_ab.log)
  auto prow = [](int idx) {
    return TS ? idx % NB : 8 * ((idx >> 5) % (NB / 8)) + (idx & 3) + ((idx >> 4) & 1) * 4;
  };
  auto pcol = [](int idx) { return TS ? idx / NB : 4 * ((idx >> 5) / (NB / 8)) + ((idx >> 2) & 3); };
  for (int c0 = cbeg; c0 < cend; c0 += IB) {
    // ---- stage the panel (coalesced) and, for TSQRT, the R block -------------
    // trailing columns of this inner panel -> L2 while the panel is factored
#ifndef TILEQR_NO_PANEL_PREFETCH
    if (tid == 0 && c0 + IB < NB)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(B + (size_t)(c0 + IB) * NB),
                   "r"((uint32_t)((NB - c0 - IB) * NB * sizeof(double)))
                   : "memory");
#endif
    if constexpr (IB <= 16) {
      // panel columns (and for TSQRT the R block): up to 16 + 2 loads in flight
      // per thread before the shared stores -- the stage is one L2 round trip
      constexpr int UV = (NB * IB + kThreads - 1) / kThreads < 16 ? (NB * IB + kThreads - 1) / kThreads : 16;
      constexpr int UR = (IB * IB + kThreads - 1) / kThreads;
      for (int idx0 = tid; idx0 < NB * IB; idx0 += UV * kThreads) {
        double v[UV];
#pragma unroll
        for (int u = 0; u < UV; ++u) {
          const int idx = idx0 + u * kThreads;
          // GEQRT: rows above c0 are R rows of earlier inner panels that a
          // concurrent TSQRT sub-task may be rewriting -- never read them (a
          // stale line could even land in the L1 another CTA of this SM reads
          // after its acquire); their operand entries are 0 anyway
          const int r = prow(idx), c = pcol(idx);
          v[u] = (idx < NB * IB && (TS || r >= c0) && (!TT || r <= c0 + c))
                     ? __ldcg(&B[r + (size_t)(c0 + c) * NB]) : 0.0;
        }
        double rv[UR];
        if (TS && idx0 == tid) {
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            const int idx = tid + u * kThreads, c = idx / IB, i = idx - c * IB;
            rv[u] = (idx < IB * IB && i <= c) ? __ldcg(&R[(c0 + i) + (size_t)(c0 + c) * NB]) : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < UV; ++u) {
          const int idx = idx0 + u * kThreads;
          if (idx < NB * IB) S.Vs[vsw(prow(idx), pcol(idx), LDV)] = v[u];
        }
        if (TS && idx0 == tid) {
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            const int idx = tid + u * kThreads, c = idx / IB, i = idx - c * IB;
            if (idx < IB * IB) S.Rin[i * LDR + c] = rv[u];
          }
        }
      }
    } else {  // IB > 16: 8 loads in flight, R block after (same-box A/B: the batched stage is slower here)
      // panel columns: 8 loads in flight per thread before the shared stores
      for (int idx0 = tid; idx0 < NB * IB; idx0 += 8 * kThreads) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = idx0 + u * kThreads;
          const int r = prow(idx), c = pcol(idx);
          v[u] = (idx < NB * IB && (TS || r >= c0) && (!TT || r <= c0 + c))
                     ? __ldcg(&B[r + (size_t)(c0 + c) * NB]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = idx0 + u * kThreads;
          if (idx < NB * IB) S.Vs[vsw(prow(idx), pcol(idx), LDV)] = v[u];
        }
      }
      if (TS) {
        for (int idx = tid; idx < IB * IB; idx += kThreads) {
          const int c = idx / IB, i = idx - c * IB;
          S.Rin[i * LDR + c] = (i <= c) ? __ldcg(&R[(c0 + i) + (size_t)(c0 + c) * NB]) : 0.0;
        }
      }
    }
    __syncthreads();
    // Registers: lane = column, warp w holds rows [w*RW, (w+1)*RW) in x[].
    // GEQRT: the IB rows [c0, c0+IB) of the diagonal block -- the rows that
    // leave the reflector one per step -- are held separately, row c0+i in
    // top[i / W] of warp i % W (a warp's rows leave in order: slot 0 is always
    // the next one, see the step); x[] holds only the rows below, which stay in
    // every reflector of the panel.
    double x[RL];
#pragma unroll
    for (int q = 0; q < RL; ++q)
      x[q] = (col < IB && (TS || rbase + q >= c0 + IB)) ? S.Vs[vsw(rbase + q, col, LDV)] : 0.0;
    double top[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      const int i = t * kWarps + warp;
      top[t] = (!TS && lane < IB && i < IB) ? S.Vs[vsw(c0 + i, lane, LDV)] : 0.0;
    }

    double myscal = 1.0;  // 1 / (alpha - beta) of the lane's own column, once its step ran
    TQ_PHASE(0);
    // ---- 1. factor the panel column by column --------------------------------
    auto step = [&](const int jj) {
      const int buf = jj & 1;
      double vj[RL];
      double pp[4] = {0.0, 0.0, 0.0, 0.0};  // 4 independent chains
#pragma unroll
      for (int q = 0; q < RL; ++q) {
        vj[q] = __shfl_sync(0xffffffffu, x[q], jj + hg * IB);
        pp[q & 3] = fma(vj[q], x[q], pp[q & 3]);
      }
      // (after the x rows' shuffles, which do not depend on it: the owner's
      // stores overlap their latency)
      if (!TS && warp == jj % kWarps) {
        // row j leaves the reflector: its owner publishes it (alpha, R(j, c))
        // and stores its final V entries (lanes < j; the rest is R, written
        // from Rout), then shifts its remaining top rows down one slot, so
        // every slot always holds a row below j (no dynamic register index)
        S.rowj[buf][lane] = top[0];
        // columns >= IB: kept panels (step 3), or for IB = 24 the zero padding
        // the packed copy takes
        // (lanes < j: V entries, scaled by their column's deferred scal; the
        // entries from lane j on are R, written from Rout)
        if (lane < IB || 32 % IB != 0) S.Vs[vsw(c0 + jj, lane, LDV)] = lane < IB ? top[0] * myscal : 0.0;
#pragma unroll
        for (int t = 0; t + 1 < TR; ++t) top[t] = top[t + 1];
        top[TR - 1] = 0.0;
      }
      double vt[TR];
      if (!TS) {  // top rows below row j (warp-uniform predicate per slot)
#pragma unroll
        for (int t = 0; t < TR; ++t) {
          vt[t] = __shfl_sync(0xffffffffu, top[t], jj);
          pp[t & 3] = fma(vt[t], top[t], pp[t & 3]);
        }
      }
      double part = (pp[0] + pp[1]) + (pp[2] + pp[3]);
#pragma unroll
      for (int o = IB; o < 32 && HL > 1; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (hg == 0) S.red[buf][warp][lane] = part;
      __syncthreads();
      double ps[kWarps], pd[kWarps];
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        ps[w] = S.red[buf][w][jj];
        pd[w] = S.red[buf][w][col];
      }
#pragma unroll
      for (int h = kWarps / 2; h > 0; h >>= 1)  // pairwise tree (fixed order: deterministic)
#pragma unroll
        for (int w = 0; w < h; ++w) {
          ps[w] += ps[w + h];
          pd[w] += pd[w + h];
        }
      const double sigma = ps[0], d = pd[0];
      const double alpha = TS ? S.Rin[jj * LDR + jj] : S.rowj[buf][jj];
      const double rjl = TS ? S.Rin[jj * LDR + col] : S.rowj[buf][col];
      double tau, scal, beta;
      {  // branch-free: sigma == 0 (R1: tau = 0, v = 0, beta = alpha) is selected at the end
        // Reflector rule (R1) from one reciprocal square root and one
        // reciprocal: with s = alpha^2 + sigma, rs = 1/sqrt(s), nrm = s*rs,
        //   beta = -sgn(alpha) nrm,  tau = (beta - alpha)/beta = 1 + |alpha| rs,
        //   scal = 1/(alpha - beta) = sgn(alpha) / (|alpha| + nrm).
        const double s2 = fma(alpha, alpha, sigma);
        const double aa = fabs(alpha);
        const double sg = (alpha >= 0.0) ? 1.0 : -1.0;
        // One higher-order step each (round 1: two Newton steps each; the
        // shorter dependent chain gives -2.5 % at 2048^2, same-box A/B in
        // profiles/r02y_panel_step_ab.log): with y ~ 1/sqrt(s), r = 1 - s y^2,
        //   1/sqrt(s) = y (1 - r)^(-1/2) = y (1 + q),  q = r/2 + 3r^2/8,
        // and sqrt(s) = (s y)(1 + q) from the same q; with c ~ 1/den,
        // e = 1 - den c: 1/den = c (1 + e + e^2).  The approximations' measured
        // relative error is 2^-20 on sm_100a (tools/approx_err.cu, 2^26
        // log-uniform inputs), so |r| <~ 2^-19 and the truncation errors
        // 5 r^3 / 16 and e^3 stay below 2^-58, under the rounding of the
        // steps themselves.
        double y, c;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s2));
        const double n0 = s2 * y;
        const double r = fma(-s2, y * y, 1.0);
        const double q = r * fma(0.375, r, 0.5);
        const double rs = fma(y, q, y);
        const double nrm = fma(n0, q, n0);
        const double den = aa + nrm;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(c) : "d"(den));
        const double e = fma(-den, c, 1.0), sc = sg * c;
        const bool refl = sigma != 0.0;  // (s2 = 0 makes the values above inf / nan: not selected)
        beta = refl ? -sg * nrm : alpha;
        tau = refl ? fma(aa, rs, 1.0) : 0.0;
        scal = refl ? fma(sc, fma(e, e, e), sc) : 0.0;
      }
      const double w = fma(scal, d, rjl);
      const double tw = col < IB ? tau * w : 0.0;
      // rank-1 update of the reflector rows, x = x + coef * vj (coef = 0 for
      // lanes <= jj).  The pivot lane's column becomes v2 = x2 * scal: it is
      // never read again in this panel, so the scaling is deferred to the
      // write-out (myscal, one rounding as before: bitwise the same values)
      // instead of a multiply of every lane's rows in every step.  (Round 1
      // folded the pivot lane into one fma with coef = scal - 1; the rounding
      // of scal - 1 costs |scal|^-1 ulps, i.e. all of v2 once the column norm
      // reaches ~2^50 -- tests/test_gpu_parity.py scaled inputs.)
      const double coef = (col > jj && col < IB) ? -(tau * scal) * w : 0.0;  // tau*scal beside w
      myscal = (col == jj) ? scal : myscal;
#pragma unroll
      for (int q = 0; q < RL; ++q) x[q] = fma(coef, vj[q], x[q]);
      if (!TS) {
        const double coefT = hg == 0 ? coef : 0.0;
#pragma unroll
        for (int t = 0; t < TR; ++t) top[t] = fma(coefT, vt[t], top[t]);  // (other groups' slots stay 0)
      }
      // row j of R: beta on the diagonal, R(j, c) - tau w_c to its right
      if (warp == 0 && hg == 0 && col >= jj && col < IB) S.Rout[jj * LDR + col] = (col == jj) ? beta : rjl - tw;
      if (tid == 0) S.tau[jj] = tau;
    };
    // TSQRT: unrolled for IB <= 16; for IB >= 24 the unrolled loop's code
    // size costs more than the loop (same-box A/B of the whole 10000^2
    // factorization: IB=32 rolled 51.3 ms, unrolled 52.8; IB=16 rolled 52.9,
    // unrolled 52.7)
#ifdef TILEQR_TSQRT_ROLLED  // diagnostic variant: TSQRT's step loop rolled for every IB
    constexpr bool kUnrolled = false;
#else
    constexpr bool kUnrolled = TS && IB <= 16;
#endif
    if constexpr (kUnrolled) {
#pragma unroll
      for (int jj = 0; jj < IB; ++jj) step(jj);
    } else {
      // GEQRT runs on one SM at a time while every other SM runs update code:
      // its instructions are cold in the SM's instruction caches, and a fully
      // unrolled step loop (~55 KB of SASS) stalled it on instruction fetch
      // about half of the time (ncu source view, stall_no_instruction) -- keep
      // the loop rolled so it is fetched once per inner panel
#pragma unroll 1
      for (int jj = 0; jj < IB; ++jj) step(jj);
    }
    __syncthreads();  // everyone done reading Vs (panel values) and red
    TQ_PHASE(1);

    // ---- write the factored panel: registers -> smem -> global (coalesced) ----
#pragma unroll
    for (int q = 0; q < RL; ++q)  // GEQRT: the top rows were stored by the step loop
      if ((col < IB || 32 % IB != 0) && (TS || rbase + q >= c0 + IB))
        S.Vs[vsw(rbase + q, col, LDV)] = col < IB ? x[q] * myscal : 0.0;
    __syncthreads();  // GEQRT: the top rows were stored as they left the reflector
    // (GEQRT: rows from c0 only -- above it Vs holds the stage's zeros, and
    // the R rows of earlier inner panels are not this panel's to write)
    for (int idx = TS ? tid : (c0 / 8) * IB * 8 + tid; idx < NB * IB; idx += kThreads) {
      const int c = TS ? idx / NB : 4 * ((idx >> 5) % (IB / 4)) + ((idx >> 2) & 3);
      const int r = TS ? idx % NB : 8 * ((idx >> 5) / (IB / 4)) + (idx & 3) + ((idx >> 4) & 1) * 4;
      double* p = &S.Vs[vsw(r, c, LDV)];
      const double v = *p;
      if (TS) {
        if (!TT || r <= c0 + c) B[r + (size_t)(c0 + c) * NB] = v;  // V2 (TT: the upper triangle only)
      } else {
        // GEQRT: V strictly below the diagonal (registers), R on/above it (Rout)
        if (r > c0 + c) B[r + (size_t)(c0 + c) * NB] = v;
        else if (r >= c0) B[r + (size_t)(c0 + c) * NB] = S.Rout[(r - c0) * LDR + c];
        // the DMMA operand is the unit lower trapezoid V_p (same thread, no hazard)
        *p = (r == c0 + c) ? 1.0 : (r > c0 + c ? v : 0.0);
      }
    }
    if (TS) {
      for (int idx = tid; idx < IB * IB; idx += kThreads) {
        const int c = idx / IB, i = idx - c * IB;
        if (i <= c) R[(c0 + i) + (size_t)(c0 + c) * NB] = S.Rout[i * LDR + c];
      }
    }

    __syncthreads();  // GEQRT rewrote Vs in place: complete before the Gram product
    TQ_PHASE(2);
    // ---- 2. T_p: G = V_p^T V_p (DMMA), recurrence ---------------------------
    {
      const int nbk = IB / 8;
      int blk = 0;
      for (int mb = 0; mb < nbk; ++mb)
        for (int nb = mb; nb < nbk; ++nb, ++blk) {
          if (blk % kWarps != warp) continue;
          double g0 = 0.0, g1 = 0.0;
          const int k0 = TS ? 0 : (c0 & ~3);
          for (int k4 = k0; k4 < NB; k4 += 4) {
            const int r = k4 + a;
            dmma(g0, g1, S.Vs[vsw(r, 8 * mb + g, LDV)], S.Vs[vsw(r, 8 * nb + g, LDV)]);
          }
          S.Gs[(8 * mb + g) * LDG + 8 * nb + 2 * a] = g0;
          S.Gs[(8 * mb + g) * LDG + 8 * nb + 2 * a + 1] = g1;
        }
    }
    __syncthreads();
    TQ_PHASE(5);
    // T_p in parallel: 8x8 diagonal blocks by the column recurrence, then
    // pairwise merges T12 = -T11 G12 T22 (Q1 Q2 = I - [V1 V2] [T11 T12; 0 T22]
    // [V1 V2]^T), log2(IB/8) levels.
    if (tid < IB) {
      // thread r: row r of its 8x8 diagonal block, fully unrolled in registers
      // (the G and tau loads do not depend on the recurrence and are hoisted)
      const int b0 = tid & ~7, rr = tid & 7;
      double tr[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < i; ++l)
          if (l >= rr) acc = fma(tr[l], S.Gs[(b0 + l) * LDG + b0 + i], acc);
        const double ti = S.tau[b0 + i];
        tr[i] = (i < rr) ? 0.0 : (i == rr ? ti : -ti * acc);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) S.Ts[tid + (b0 + i) * LDT] = tr[i];
    }
    __syncthreads();
    TQ_PHASE(6);
    // merges: Ts/Gs are zero outside the computed blocks (zero-filled at kernel
    // start), so every dot runs over the full block width with no bounds
    auto merge = [&](auto sz) {
      constexpr int SZ = decltype(sz)::value;
      const int npair = (IB + SZ - 1) / (2 * SZ);  // pairs with a non-empty right block
      for (int e = tid; e < npair * SZ * SZ; e += kThreads) {  // X = G12 T22
        const int p = e / (SZ * SZ), il = (e / SZ) % SZ, kl = e % SZ, st = p * 2 * SZ;
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < SZ; ++l)
          acc = fma(S.Gs[(st + il) * LDG + st + SZ + l], S.Ts[(st + SZ + l) + (st + SZ + kl) * LDT], acc);
        S.Rin[(st + il) * LDR + st + SZ + kl] = acc;  // Rin is free after the factorization
      }
      __syncthreads();
      for (int e = tid; e < npair * SZ * SZ; e += kThreads) {  // T12 = -T11 X
        const int p = e / (SZ * SZ), il = (e / SZ) % SZ, kl = e % SZ, st = p * 2 * SZ;
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < SZ; ++l)
          acc = fma(S.Ts[(st + il) + (st + l) * LDT], S.Rin[(st + l) * LDR + st + SZ + kl], acc);
        S.Ts[(st + il) + (st + SZ + kl) * LDT] = -acc;
      }
      __syncthreads();
    };
    if (IB > 8) merge(std::integral_constant<int, 8>{});
    if (IB > 16) merge(std::integral_constant<int, 16>{});
    TQ_PHASE(7);
    for (int e = tid; e < IB * IB; e += kThreads) {
      const int i = e / IB, r = e - i * IB;
      Tg[(size_t)(c0 + i) * IB + r] = (r <= i) ? S.Ts[r + i * LDT] : 0.0;
    }
    if (Vpk) {  // packed copy of V_p / T_p for the barrier-free update (update_v2.cuh)
      auto vf = [&](int r, int i) { return S.Vs[vsw(r, i, LDV)]; };
      auto tf = [&](int l, int i) { return S.Ts[l + i * LDT]; };
      v2::pack_panel<NB, IB, kThreads>(Vpk, c0 / IB, vf, tf);
    }
    __syncthreads();
    TQ_PHASE(3);
    // ---- 3. trailing columns: 8-column blocks per warp ------------------------
    // A sub-task of NPS <= 32/IB inner panels (the DAG kernel) updates, after
    // panel j, only its own later columns [c0+IB, cend) ("near"); the columns
    // [cend, NB) get all NPS panels in one pass after the last one ("far"):
    // each column block crosses L2 once instead of NPS times, with the same
    // operations in the same order (bitwise the per-panel result).  The
    // earlier panels' V_p and T_p are kept for it in Vs columns
    // [32 - IB(j+1), 32 - IB j) and Tsv rows [j IB, (j+1) IB).
    const int jc = (c0 - cbeg) / IB;  // this panel's index in the sub-task
    const bool last = c0 + IB >= cend;
    if (fuse && !last) {  // read after later barriers only
      const int off = 32 - IB * (jc + 1);
      for (int e = tid; e < NB * IB; e += kThreads) {
        const int r = e / IB, i = e - r * IB;
        S.Vs[vsw(r, off + i, LDV)] = S.Vs[vsw(r, i, LDV)];
      }
      for (int e = tid; e < IB * IB; e += kThreads) {
        const int r = e % IB, i = e / IB;
        S.Tsv[jc * IB + r + i * LDT] = S.Ts[r + i * LDT];
      }
    }
    // apply panels j0..j1 of the sub-task, in order, to columns [lo, hi)
    auto trailing = [&](const int lo, const int hi, const int j0, const int j1) {
      double* Wsw = S.Ws[warp];
      const int nbi = IB / 8;
      const int rlo = cbeg + j0 * IB;
      for (int cb = lo + 8 * warp; cb < hi; cb += 8 * kWarps) {
        const int cc = cb + g;
        // GEQRT: rows above the first applied panel of the trailing columns
        // are R rows of earlier inner panels -- never loaded or stored here
        // (a concurrent TSQRT sub-task of the DAG kernel may own them)
        double acc[RB][2];
#pragma unroll
        // TT: V2 of the applied panels is zero below row rhi: rows >= rhi are
        // neither needed nor touched (below a column's diagonal they hold V)
        const int rhi = TT ? cbeg + (j1 + 1) * IB : NB;
        for (int rb = 0; rb < RB; ++rb) {
          if ((!TS && 8 * rb + 7 < rlo) || (TT && 8 * rb >= rhi)) { acc[rb][0] = acc[rb][1] = 0.0; continue; }
          const double2 v = __ldcg(reinterpret_cast<const double2*>(B + 8 * rb + 2 * a + (size_t)cc * NB));
          acc[rb][0] = v.x;
          acc[rb][1] = v.y;
        }
#pragma unroll 1
        for (int j = j0; j <= j1; ++j) {
          const int pc0 = cbeg + j * IB;
          const int voff = (j == jc) ? 0 : 32 - IB * (j + 1);
          const double* Tj = (j == jc) ? S.Ts : S.Tsv + j * IB;
          // step A: W^T(col, i) = [TS: R(pc0+i, col)] + sum_r C^T(col, r) V_p(r, i);
          // two partial sums (k rows 2a and 2a+1) per output block
          double wacc[4][2], wacc2[4][2], rk[4][2];  // rk: the R rows, reused by step B
#pragma unroll
          for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              rk[nb][jj] = (TS && nb < nbi) ? __ldcg(&R[(pc0 + 8 * nb + 2 * a + jj) + (size_t)cc * NB]) : 0.0;
              wacc[nb][jj] = rk[nb][jj];
              wacc2[nb][jj] = 0.0;
            }
#pragma unroll
          for (int rb = 0; rb < RB; ++rb) {
            if (!TS && 8 * rb + 7 < pc0) continue;
            if (TT && 8 * rb >= pc0 + IB) continue;
#pragma unroll
            for (int nb = 0; nb < 4; ++nb)
              if (nb < nbi) {
                dmma(wacc[nb][0], wacc[nb][1], acc[rb][0], S.Vs[vsw(8 * rb + 2 * a, voff + 8 * nb + g, LDV)]);
                dmma(wacc2[nb][0], wacc2[nb][1], acc[rb][1], S.Vs[vsw(8 * rb + 2 * a + 1, voff + 8 * nb + g, LDV)]);
              }
          }
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) {
            wacc[nb][0] += wacc2[nb][0];
            wacc[nb][1] += wacc2[nb][1];
          }
#pragma unroll
          for (int nb = 0; nb < 4; ++nb)
            if (nb < nbi) {
              Wsw[g * LDW + 8 * nb + 2 * a] = wacc[nb][0];
              Wsw[g * LDW + 8 * nb + 2 * a + 1] = wacc[nb][1];
            }
          __syncwarp();
          // step B: W'^T = W^T T_p (descending blocks, in place); TS: R(pc0+i, col) -= W'
          if constexpr (IB <= 16) {  // unrolled: the R rows come from rk (registers)
#pragma unroll
            for (int nb = 3; nb >= 0; --nb) {
              if (nb >= nbi) continue;
              double o0 = 0.0, o1 = 0.0;
#pragma unroll
              for (int k4 = 0; k4 < 8 * nb + 8; k4 += 4)
                dmma(o0, o1, Wsw[g * LDW + k4 + a], Tj[(k4 + a) + (8 * nb + g) * LDT]);
              __syncwarp();
              Wsw[g * LDW + 8 * nb + 2 * a] = -o0;
              Wsw[g * LDW + 8 * nb + 2 * a + 1] = -o1;
              if (TS) {  // R(pc0+i, col) -= W'  (this warp owns the column)
                double* r0 = &R[(pc0 + 8 * nb + 2 * a) + (size_t)cc * NB];
                *reinterpret_cast<double2*>(r0) = make_double2(rk[nb][0] - o0, rk[nb][1] - o1);
              }
              __syncwarp();
            }
          } else {  // IB > 16: rolled (code size; same-box A/B), R rows reloaded
            for (int nb = nbi - 1; nb >= 0; --nb) {
              double o0 = 0.0, o1 = 0.0;
              for (int k4 = 0; k4 < 8 * nb + 8; k4 += 4)
                dmma(o0, o1, Wsw[g * LDW + k4 + a], Tj[(k4 + a) + (8 * nb + g) * LDT]);
              __syncwarp();
              Wsw[g * LDW + 8 * nb + 2 * a] = -o0;
              Wsw[g * LDW + 8 * nb + 2 * a + 1] = -o1;
              if (TS) {
                double* r0 = &R[(pc0 + 8 * nb + 2 * a) + (size_t)cc * NB];
                r0[0] = __ldcg(r0) - o0;
                r0[1] = __ldcg(r0 + 1) - o1;
              }
              __syncwarp();
            }
          }
          // step C: C^T(col, r) += (-W'^T)(col, i) V_p(r, i)
          for (int k4 = 0; k4 < IB; k4 += 4) {
            const double af = Wsw[g * LDW + k4 + a];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
              if (!TS && 8 * rb + 7 < pc0) continue;
              if (TT && 8 * rb >= pc0 + IB) continue;
              dmma(acc[rb][0], acc[rb][1], af, S.Vs[vsw(8 * rb + g, voff + k4 + a, LDV)]);
            }
          }
          __syncwarp();
        }
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          if ((!TS && 8 * rb + 7 < rlo) || (TT && 8 * rb >= rhi)) continue;
          *reinterpret_cast<double2*>(B + 8 * rb + 2 * a + (size_t)cc * NB) = make_double2(acc[rb][0], acc[rb][1]);
        }
        __syncwarp();
      }
    };
    trailing(c0 + IB, fuse ? cend : NB, jc, jc);
    if (fuse && last) trailing(cend, NB, 0, jc);  // the kept panels were written before earlier barriers
    __syncthreads();  // trailing writes visible before the next panel is staged
    TQ_PHASE(4);
  }
#undef TQ_PHASE
  if (Vpk) v2::fence_proxy_async();  // packed tile is read by TMA (async proxy) on other SMs
}

}  // namespace pf
}  // namespace tileqr
