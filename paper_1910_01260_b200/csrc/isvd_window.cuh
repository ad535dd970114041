// Window projections of the streaming incremental SVD (window-mode ingestion).
//
// The per-snapshot pass of isvd_kernels.cuh reads all of U for every snapshot,
// also to project the next one.  In window mode one pass projects kWB
// snapshots at once, G = U^T [x_t .. x_{t+kWB-1}] plus their Gram XX, and the
// per-snapshot pass (PASS_RESID) runs only for snapshots that enter U
// (independent ones; basis.py:139).  Columns appended inside the window get
// their rows of G from XX (window_row, isvd_kernels.cuh).  Bytes per snapshot
// drop from 8 n (c + 3) to 8 n ((c + kWB) / kWB + [independent] (c + 2)).
//
// k_wproj: one CTA per SM (minus the core step's), a warp of bulk-copy
// producers and 8 consumer warps.  Each 64-row stage holds the c live U column
// segments and the kWB x segments, each copied into a 68-double slot so the
// DMMA fragment loads (8 columns x 4 rows per load) hit distinct banks.  The
// contraction G_cta += U_tile^T X_tile is DMMA m8n8k4 (M = U columns, N = the
// window, K = rows); per-CTA partials are summed by k_wreduce in a fixed order.
#pragma once

#include "isvd_kernels.cuh"
#include "runtime.cuh"

namespace strom {

constexpr int kWLd = kStageRows + 4;  // 68: padded column slot in a window stage
constexpr int kWConsumers = 8;
constexpr int kWThreads = 32 * (kWConsumers + 1);
constexpr int kWMaxStages = 4;

struct WprojArgs {
  const double* U;
  int64_t ldu, n, ccap;
  const PipeCtl* ctl;
  const double* xs[kWB];
  int32_t nw;     // window columns (<= kWB)
  int32_t xbulk;  // every xs[j] 16-byte aligned and n even: stage x by bulk copy
  double* part;   // per-CTA partials, pstride doubles each: [i * kWB + j] G, then kWB^2 XX
  int32_t pstride;
  unsigned long long* prof;
  long long* trace;
};

template <int MT>  // m-tiles (8 U columns) per consumer warp: c <= 64 MT
__global__ void __launch_bounds__(kWThreads, 1) k_wproj(WprojArgs a, int nstages) {
  extern __shared__ __align__(128) double wst[];
  __shared__ __align__(8) uint64_t full[kWMaxStages];
  __shared__ __align__(8) uint64_t empty[kWMaxStages];
  pdl_enter();
  trace_stamp(a.trace, 14);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int c = a.ctl->c, base = a.ctl->base;
  const int c8 = (c + 7) & ~7;
  const int cs = c8 + kWB;
  const size_t stage_elems = (size_t)cs * kWLd;
  const int64_t tstride = (int64_t)kUTile * a.ccap;
  if (a.prof && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(a.prof + P_WPROJ, 8ull * (unsigned long long)a.n * (unsigned long long)(c + a.nw));
  const int64_t ntiles = a.ldu / kStageRows;
  const int64_t per = ceil_div(ntiles, gridDim.x);
  const int64_t t0 = blockIdx.x * per;
  const int64_t nt = max((int64_t)0, min(ntiles, t0 + per) - t0);
  // U padding columns c..c8-1 are never copied: zero them once in every stage
  for (int st = 0; st < nstages; ++st)
    for (int idx = threadIdx.x; idx < (c8 - c) * kWLd; idx += blockDim.x)
      wst[st * stage_elems + (size_t)c * kWLd + idx] = 0.0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < nstages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kWConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wid == 0) {
    // ---------------- producers: lane 0 arms the stage, all lanes issue copies
    for (int64_t i = 0; i < nt; ++i) {
      const int st = (int)(i % nstages);
      const int64_t use = i / nstages;
      if (use > 0) mbar_wait(&empty[st], (unsigned)((use - 1) & 1));
      const int64_t row0 = (t0 + i) * kStageRows;
      const int valid = (int)max((int64_t)0, min((int64_t)kStageRows, a.n - row0));
      const unsigned xb = a.xbulk ? (unsigned)valid * 8u : 0u;
      if (lane == 0) mbar_expect_tx(&full[st], (unsigned)c * kStageRows * 8u + xb * (unsigned)a.nw);
      __syncwarp();
      double* dst = wst + (size_t)st * stage_elems;
      const double* src = a.U + (t0 + i) * tstride + (int64_t)base * kUTile;
      for (int col = lane; col < c; col += 32)
        bulk_g2s(dst + (size_t)col * kWLd, src + (int64_t)col * kUTile, kStageRows * 8u, &full[st]);
      if (xb)
        for (int j = lane; j < a.nw; j += 32) bulk_g2s(dst + (size_t)(c8 + j) * kWLd, a.xs[j] + row0, xb, &full[st]);
    }
  } else {
    // ---------------- consumers: warp cw owns m-tiles cw, cw + 8, ...
    const int cw = wid - 1;
    double acc[MT][2];
#pragma unroll
    for (int q = 0; q < MT; ++q) acc[q][0] = acc[q][1] = 0.0;
    double xa0 = 0.0, xa1 = 0.0;
    const double* xg = (g < a.nw) ? a.xs[g] : nullptr;
    for (int64_t i = 0; i < nt; ++i) {
      const int st = (int)(i % nstages);
      const int64_t use = i / nstages;
      mbar_wait(&full[st], (unsigned)(use & 1));
      const double* tile = wst + (size_t)st * stage_elems;
      const int64_t row0 = (t0 + i) * kStageRows;
      const int valid = (int)max((int64_t)0, min((int64_t)kStageRows, a.n - row0));
#pragma unroll 4
      for (int ks = 0; ks < kStageRows / 4; ++ks) {
        const int kr = 4 * ks + t;
        double b;
        if (a.xbulk) b = (xg && kr < valid) ? tile[(size_t)(c8 + g) * kWLd + kr] : 0.0;
        else b = (xg && kr < valid) ? __ldg(xg + row0 + kr) : 0.0;
#pragma unroll
        for (int q = 0; q < MT; ++q) {
          const int mt = cw + kWConsumers * q;
          if (8 * mt < c) {
            const double av = tile[(size_t)(8 * mt + g) * kWLd + kr];
            dmma884(acc[q][0], acc[q][1], av, b);
          }
        }
        if (cw == 0) dmma884(xa0, xa1, b, b);  // XX = X^T X (A = X^T: a = X(kr, g) = b)
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    double* mypart = a.part + (int64_t)blockIdx.x * a.pstride;
#pragma unroll
    for (int q = 0; q < MT; ++q) {
      const int i = 8 * (cw + kWConsumers * q) + g;
      if (i < c) {
        mypart[i * kWB + 2 * t] = acc[q][0];
        mypart[i * kWB + 2 * t + 1] = acc[q][1];
      }
    }
    if (cw == 0) {
      double* xp = mypart + (int64_t)c8 * kWB;
      xp[g * kWB + 2 * t] = xa0;
      xp[g * kWB + 2 * t + 1] = xa1;
    }
  }
}

// Sum the per-CTA partials in CTA order (fixed: deterministic) into
// G (c x nw, ld ldg) and XX (kWB x kWB).  32 outputs per CTA, 8 warps split
// the partials, lanes = outputs (coalesced).
__global__ void __launch_bounds__(256) k_wreduce(const double* part, int nparts, int pstride, const PipeCtl* ctl,
                                                 int nw, double* G, int ldg, double* XX) {
  __shared__ double red[8][33];
  pdl_enter();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c = ctl->c, c8 = (c + 7) & ~7;
  const int nout = c8 * kWB + kWB * kWB;
  const int o = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (o < nout)
    for (int b = wid; b < nparts; b += 8) s += part[(int64_t)b * pstride + o];
  red[wid][lane] = s;
  __syncthreads();
  if (wid == 0 && o < nout) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][lane];
    if (o < c8 * kWB) {
      const int i = o / kWB, j = o % kWB;
      if (i < c && j < nw) G[(int64_t)j * ldg + i] = v;
    } else {
      XX[o - c8 * kWB] = v;
    }
  }
}

// First snapshot of a window: tvec = L^{-1} G[:, 0], gt = L^{-T} tvec, xx = XX[0, 0]
// (prep_next with the window's column 0 as "next": the caller passes wcol = -1).
__global__ void __launch_bounds__(kDecideThreads) k_prep_w(Pipe pp, IsvdParams P) {
  extern __shared__ double part[];
  pdl_enter();
  prep_next(P, pp, part);
  trace_stamp(P.trace, 15);
}

}  // namespace strom
