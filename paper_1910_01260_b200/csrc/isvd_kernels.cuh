// Device kernels of the streaming incremental SVD (reference basis.py:105-184).
//
// Representation: the reference keeps the n x r left
// basis Phi explicitly and rewrites it every snapshot (Phi' = [Phi j] W_bar,
// basis.py:155-156).  Here Phi = Q_U N with
//   U    n x c_cap  append-only column store in HBM (column-major, ld = ldu)
//   G  = U^T U = L L^T, L and L^{-1} kept exactly, indexed by PHYSICAL column
//        (the live block of a state starts at (base, base)); append-only like U
//   Q_U  = U L^{-T} (never formed): an orthonormal basis of span(U)
//   N    c x r      Phi's coordinates in Q_U (small); Phi^T Phi = N^T N.
//
// One snapshot x_t costs ONE pass over U (k_pass, kind FUSED): it forms the
// residual r1 = x_t - U G^{-1} U^T x_t into the next free column, measures
// e = U^T r1 and |r1|^2 for the exact Gram extension, and -- reading the same
// U tile -- the projection U^T x_{t+1} of the NEXT snapshot.  The decision
// chain (k_decide, optional re-orthogonalisation pass + k_decide2) is a few
// microseconds of one-CTA work; the bordered core SVD, N rotation, truncation
// and drift QR (k_step_b) and the V update run on a second stream, overlapped
// with the next snapshot's pass.
#pragma once

#include "bulk.cuh"
#include "common.cuh"
#include "core_svd.cuh"
#include "dmma.cuh"
#include "small_dense.cuh"

namespace strom {

// -------- per-state header (lives in the state's small block) --------------
struct IsvdHdr {
  int32_t r;       // rank = sigma.size
  int32_t c;       // logical columns of U in use
  int32_t base;    // physical column of logical column 0
  int32_t status;  // 0 ok, 1 non-finite input
  int32_t n_rejected, n_dependent, n_truncated, n_restarts;
  int32_t flags;   // decision bits of the update that produced this state
  int32_t pad0;
  double p;        // Pythagorean residual norm of that update
  double drift;    // |phi_0 . phi_last| of that update
  double xnorm;    // ||x|| of that update
  double p_sq;     // unclamped x.x - ell.ell of that update
};

enum : int32_t {
  F_DEPENDENT = 1, F_TRUNCATED = 2, F_QR = 4, F_RESTART = 8, F_REJECTED = 16,
  F_APPENDED = 32, F_FOLDED = 64, F_ERROR = 128,
};

enum : int32_t { M_NORMAL_DEP = 0, M_NORMAL_INDEP = 1, M_RESTART_ACCEPT = 2, M_REJECT = 3, M_ERROR = 4 };

// -------- pipeline control (device) ----------------------------------------
// The columns (c, base) of the most recently DECIDED state: the passes read
// them, so the host never needs to know the device-side decisions.
struct PipeCtl {
  int32_t c, base;
  int32_t reorth;   // 0 none, 1 DGKS pass requested, 2 restart copy requested
  int32_t bdone;    // core steps (k_step_b) completed since the sequence started
  int32_t decided;  // decision chains (k_decide + k_decide2) completed since then
  int32_t resid;    // window mode: the residual pass of this snapshot is needed
  int32_t adone;    // window mode: first-half decisions (k_decide_a) completed
  int32_t a_inline; // window mode: d_expect of the snapshot whose first half k_step_b already ran
  int32_t slow_step;  // k_new of the update whose shared-memory core step handed over to the global-memory one
  int32_t pad_;
  double xx;        // x.x of the snapshot about to be decided
};

// Cross-stream completion counters: one thread spins (acquire) until *ctr >= target.
__device__ inline void wait_counter(const int32_t* ctr, int32_t target) {
  if (target < 0) return;
  if (threadIdx.x == 0) {
    const volatile int32_t* v = ctr;
    while (*v < target) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}
__device__ inline void signal_counter(int32_t* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1);
  }
}

// One update's decisions (double-buffered by update parity: k_step_b of update
// t reads record t%2 while the decision kernels of t+1 write the other one).
struct IsvdStep {
  int32_t mode, restart, action, dep;  // action: 0 none (dependent), 1 append, 2 fold
  int32_t c, cn, base_new, slot;       // U columns before / after, new base, write slot
  int32_t m, mkeep, pad0, pad1;        // set by k_step_b for k_vupdate
  double xx, rho2, p, p_sq, norm, lam;
};

// Outputs of one pass: e (c), gn (c + 1: U^T x_next, [c] = r . x_next),
// scal[0] = r.r, scal[1] = x_next.x_next, scal[2] = r.x_next
struct PassOut {
  double* e;
  double* gn;
  double* scal;
  double* gw;  // window mode: r . x_j for the window's later snapshots (measured on the stored r)
};

// What k_vupdate needs from k_step_b, in a record of its own: in window mode
// the V update runs on a third stream and may trail the decisions.
struct VRec {
  int32_t mode, m, mkeep, pad;
};

struct Pipe {
  PipeCtl* ctl;
  IsvdStep* step[2];
  VRec* vrec[2];
  double* ell[2];  // r_cap + 2: Phi^T x
  double* nj[2];   // c_cap + 1: the new N column (x - Phi ell)/p in Q_U coordinates
  double* tvec;    // L^{-1} g: x's coordinates in Q_U
  double* gt;      // G^{-1} g = L^{-T} tvec
  double* y;       // tvec - N ell
  double* l1;      // L^{-1} e of the first residual
  double* h;       // DGKS coefficients G^{-1} e, later l2
  double* tmp;     // c_cap scratch (L^{-1} g' of the next snapshot)
  double* w;       // c_cap scratch (L^{-T} l of an appended column)
  PassOut fo;      // the fused pass
  PassOut ro;      // the second (re-orthogonalisation / restart) pass
  double* vbar;    // (r_cap+2)^2 sorted, sign-fixed V_bar of the core
  double* work;    // global fallback workspace of the one-CTA kernels
  double* T;       // c_cap x (r_cap+1) compaction transform
  double* part;    // per-CTA partial sums of the passes
  unsigned* counter;
};

struct StateView {
  IsvdHdr* hdr;
  double* N;      // c_cap x (r_cap + 1), ld = ldn   (Phi = U L^{-T} N)
  double* sigma;  // r_cap + 1
  double* V;      // k_cap x (r_cap + 1), ld = ldv
  double* L;      // store: c_cap x c_cap lower (physical columns), ld = ldl
  double* Li;     // store: L^{-1}
  int32_t ldn, ldl;
  int64_t ldv;
};

struct IsvdParams {
  int64_t n, ldu;
  int32_t ccap, rcap;
  double tol_svd, tol_sv;
  int32_t r_max;     // -1: no cap
  int32_t cap_mode;  // 0 restart, 1 truncate
  int64_t k_new;     // column counter after this update
  int32_t pstride;   // stride of one CTA's partial row
  int32_t work_stride;
  int32_t parity;    // which IsvdStep / ell / nj record this update uses
  int32_t has_next;  // the fused pass also projected the next snapshot
  int32_t b_expect;  // k_decide waits for ctl->bdone >= b_expect (-1: stream order suffices)
  int32_t d_expect;  // k_step_b waits for ctl->decided >= d_expect (-1: stream order suffices)
  double* L;         // store pointers (physical indexing), ld = ccap
  double* Li;
  unsigned long long* prof;  // device byte counters (runtime.cuh ProfKind) or null
  long long* tprobe;         // phase timestamps of step B (diagnostics) or null
  long long* trace;          // per-update globaltimer trace (diagnostics, strom_debug_trace) or null
  // window mode (wn > 0): projections of the window's snapshots onto U,
  // G[i + j ldg] = U_i . x_j (logical columns i), and their Gram XX[i kWB + j];
  // wcol is this snapshot's column.  pp.fo.gn then points at column wcol + 1.
  double* wG;
  const double* wXX;
  int32_t ldg, wcol, wn;
  int32_t inline_next;  // window mode: k_step_b also runs the next snapshot's first-half decision
  int32_t stage_doubles;  // k_decide_b: doubles of shared memory behind its partials for L^{-1} and N (0: none)
  // Core step when the CAPACITY's work area exceeds shared memory (an uncapped state whose rank
  // capacity has grown): 1 = the shared-memory kernel, launched with step_smem_doubles of room,
  // runs if the CURRENT rank's work area fits and otherwise hands over (ctl->slow_step = k_new)
  // to the global-memory kernel queued behind it (2), which runs only then.  0: no hand-over.
  int32_t step_try;
  int32_t step_smem_doubles;
};

constexpr int kWB = 8;  // window width: snapshots projected by one pass over U

// x.x of the next snapshot: the pass's scal[1], or the window Gram's diagonal
__device__ __forceinline__ double next_xx(const IsvdParams& P, const Pipe& pp) {
  return P.wn > 0 ? P.wXX[(P.wcol + 1) * (kWB + 1)] : pp.fo.scal[1];
}

// Programmatic dependent launch: let the next kernel of the stream launch now
// (it waits for us itself), and wait for the previous one before reading its
// results.  Both are no-ops for a kernel launched without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_trigger();
  pdl_wait();
}

// Diagnostics trace: globaltimer stamp into row[k] by thread 0 of CTA 0.
__device__ __forceinline__ void trace_stamp(long long* row, int k) {
  if (row && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    row[k] = (long long)t;
  }
}

#define STROM_TPROBE(P, k)                                  \
  do {                                                      \
    if ((P).tprobe && threadIdx.x == 0) (P).tprobe[k] = clock64(); \
  } while (0)

constexpr int kPassRows = 32;       // rows per pass tile (one per lane)
constexpr int kPassConsumers = 8;                        // consumer warps of the pass
constexpr int kPassThreads = 32 * (kPassConsumers + 1);  // + one TMA producer warp; one CTA per SM
constexpr int kStageRows = kUTile;                       // rows per pipeline stage = one U tile
constexpr int kSubRows = kUTile;                         // rows per consumer step (2 per lane)
constexpr int kSmallThreads = 512;  // one-CTA kernels: 128 registers per thread (no spills)
constexpr int kDecideThreads = 512;
constexpr int kTileRows = 64;       // legacy tile of the helpers below

// Deterministic grid finish: the last CTA to arrive sums the per-CTA partials
// in CTA order.  Returns true in that CTA (after the counter is reset).
__device__ inline bool last_cta_arrives(unsigned* counter, int* s_is_last) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    *s_is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (*s_is_last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;
    return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// The pass over U (HBM-bound; one per snapshot).
//   PROJ   : gn = U^T xn, scal[1] = xn.xn                           (first snapshot)
//   FUSED  : r = x - U coef -> U[:, base + c]; e = U^T r; scal[0] = r.r;
//            gn[0..c) = U^T xn, gn[c] = r.xn, scal[1] = xn.xn, scal[2] = r.xn
//   SECOND : only if ctl->reorth: 1 = DGKS, r = r1 - U h in place; 2 = restart
//            copy, r = x (no U columns read); e, scal[0], scal[2]
// 32-row tiles, lane = row; warp w owns columns w + 8q.  U streams through a
// multi-stage shared-memory ring filled by bulk async copies (mbarrier tx).  Row dots of r reduce
// across warps through a double-buffered shared array (one barrier per tile);
// column dots stay in registers until a deterministic last-CTA reduction.
// Reference: basis.py:135-139 (projection, Pythagorean p) and 150-156 (j).
// ---------------------------------------------------------------------------
enum : int32_t { PASS_PROJ = 0, PASS_FUSED = 1, PASS_SECOND = 2, PASS_RESID = 3 };
// PASS_RESID (window mode): FUSED without the next projection, and only when
// k_decide_a found the snapshot independent (ctl->resid); a no-op otherwise.

struct PassArgs {
  double* U;  // row-tiled store (kUTile-row tiles of ccap column segments)
  int64_t ldu, n;
  int64_t ccap;
  int32_t dbg;  // diagnostics: 1 = consumers only wait/release (bandwidth probe)
  int32_t x_bulk, xn_bulk;  // x / xn may be staged by bulk copy (16-byte aligned, n even)
  // decision tail run by the last-arriving CTA: 0 none, 1 decide (FUSED), 2 decide2 (SECOND)
  int32_t tail;
  int32_t b_expect;  // decide waits until ctl->bdone >= b_expect (-1: no wait)
  StateView dsrc;
  Pipe dpp;
  IsvdParams dP;
  const PipeCtl* ctl;
  int32_t kind;
  int32_t pstride;
  int32_t pld;  // partials are stored output-major: (CTA b, output o) at part[o * pld + b]
  const double* x;
  const double* coef;
  const double* xn;
  PassOut out;
  double* part;
  unsigned* counter;
  unsigned long long* prof;
  long long* trace;  // diagnostics: this update's trace row, or null
  // window mode: dots of the new column r with these later snapshots of the
  // window (consumer warp w takes column w); one more read of nxw columns
  const double* xw[kWB - 1];
  int32_t nxw;
  int32_t xw_bulk;  // every xw[j] 16-byte aligned and n even: staged with U
};

constexpr int kPassMaxStages = 8;


// The pass: lane 0 of warp 0 streams U (kStageRows rows x c columns per stage:
// the tile's live column segments are contiguous, so ONE 1-D bulk copy,
// cp.async.bulk, plus one per x / x_next / window segment) into a ring of
// shared-memory stages (full/empty mbarriers); the kPassConsumers consumer warps process every stage together
// -- warp w owns columns w + 8q, lane l rows 2l, 2l+1 -- and exchange row-dot
// partials through a double-buffered shared array with ONE consumer-only named
// barrier per stage.  Column dots stay in registers until a deterministic
// last-CTA reduction.
// ---------------------------------------------------------------------------
// Small-space helpers of the decision kernels
// ---------------------------------------------------------------------------
// Bordered extension of G's factors by the appended column (physical row c of
// the block at (base, base)):  L' = [[L, 0], [l^T, lam]],
// L'^{-1} = [[L^{-1}, 0], [-(L^{-T} l)^T / lam, 1 / lam]].
__device__ inline void append_factor_row(double* Lb, double* Lib, int ldl, int c, const double* l, double lam,
                                         double* tmpv) {
  cta_gemv_t_cm(Lib, ldl, c, c, l, tmpv, true);  // tmpv = L^{-T} l
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    Lb[(int64_t)j * ldl + c] = l[j];
    Lib[(int64_t)j * ldl + c] = -tmpv[j] / lam;
  }
  if (threadIdx.x == 0) {
    Lb[(int64_t)c * ldl + c] = lam;
    Lib[(int64_t)c * ldl + c] = 1.0 / lam;
  }
  __syncthreads();
}

// Coefficients of the next snapshot's residual: tvec = L^{-1} g, gt = L^{-T} tvec.
__device__ inline void prep_next(const IsvdParams& P, const Pipe& pp, double* part) {
  __syncthreads();  // ctl may have been written by thread 0 of this CTA
  const int c = *(volatile const int32_t*)&pp.ctl->c, base = *(volatile const int32_t*)&pp.ctl->base;
  const double* Lib = P.Li + (int64_t)base * (P.ccap + 1);
  if (c > 0) {
    cta_gemv_cm<8>(Lib, P.ccap, c, c, pp.fo.gn, 1.0, nullptr, pp.tvec, part, true);
    cta_gemv_t_cm(Lib, P.ccap, c, c, pp.tvec, pp.gt, true);
  }
  if (threadIdx.x == 0) pp.ctl->xx = next_xx(P, pp);
}

// A (first snapshot of a sequence, or after a compaction): prepare from a PROJ pass.
__global__ void __launch_bounds__(kDecideThreads) k_prep(Pipe pp, IsvdParams P) {
  extern __shared__ double part[];
  pdl_enter();
  prep_next(P, pp, part);
}

// ctl <- the columns of a state (start of a sequence / after a compaction)
__global__ void k_init_ctl(PipeCtl* ctl, const IsvdHdr* h) {
  ctl->c = h->c;
  ctl->base = h->base;
  ctl->reorth = 0;
  ctl->bdone = 0;
  ctl->decided = 0;
  ctl->resid = 0;
  ctl->adone = 0;
  ctl->a_inline = -1;
  ctl->slow_step = 0;
}

constexpr double kFoldTau = 1e-3;  // append r1 only if its out-of-span part is >= tau |r1|

// Window mode: row `row` of the window projections for the snapshots after
// this one, for a U column r = x_t - U (coef + coef2) (coef null: r = x_t):
//   G[row, j] = x_t . x_j - (coef + coef2)^T G[:c, j]      (j = wcol+1 .. wn-1)
// Only used with coef null (the slot holds x_t itself: its dots ARE the
// window Gram); a residual's row is measured by its pass (window_row_measured):
// the algebraic form loses all relative accuracy when r is rounding-level.
// Row `row` of the window projections from a pass's measured dots gw[j - wcol - 1].
__device__ inline void window_row_measured(const IsvdParams& P, int row, const double* gw) {
  __syncthreads();
  for (int j = P.wcol + 1 + (int)threadIdx.x; j < P.wn; j += blockDim.x)
    P.wG[(int64_t)j * P.ldg + row] = gw[j - P.wcol - 1];
  __syncthreads();
}

__device__ inline void window_row(const IsvdParams& P, int row, int c, const double* coef, const double* coef2) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  for (int j = P.wcol + 1 + wid; j < P.wn; j += nw) {
    double* gcol = P.wG + (int64_t)j * P.ldg;
    double s = 0.0;
    if (coef)
      for (int i = lane; i < c; i += 32) s = fma(coef[i] + (coef2 ? coef2[i] : 0.0), gcol[i], s);
    s = warp_sum(s);
    if (lane == 0) gcol[row] = P.wXX[P.wcol * kWB + j] - s;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// D: every decision of update t (basis.py:112-139 and the U bookkeeping):
//   restart / reject (basis.py:112-133), ell = Phi^T x = N^T L^{-1} g, the
//   Pythagorean p (basis.py:136-138), the dependent test, and for an
//   independent snapshot how r1 enters U: l = L^{-1} e, lambda^2 = |r1|^2 -
//   |l|^2 (its out-of-span part in the G metric); append when lambda >= tau |r1|
//   (extending L, L^{-1} in the store), else request one DGKS pass (k_decide2
//   finishes).  Without a follow-up pass it also prepares the next snapshot.
// ---------------------------------------------------------------------------
__device__ inline void decide_body(const StateView& src, const Pipe& pp, const IsvdParams& P, double* part,
                                   double* red) {
  const IsvdHdr h = *src.hdr;
  IsvdStep* st = pp.step[P.parity];
  double* ell = pp.ell[P.parity];
  double* nj = pp.nj[P.parity];
  const int c = h.c, base = h.base, r = h.r;
  const int ldl = P.ccap;
  double* Lb = P.L + (int64_t)base * (ldl + 1);
  double* Lib = P.Li + (int64_t)base * (ldl + 1);
  const double xx = pp.ctl->xx;
  const double rho2 = pp.fo.scal[0];
  const int slot = base + c;
  int mode = -1, restart = 0, action = 0, dep = 0, cn = c, base_new = base, reorth = 0;
  double p = 0.0, p_sq = 0.0, lam = 0.0;
  if (h.status != 0 || !isfinite(xx)) {
    mode = M_ERROR;
  } else {
    const bool at_cap = P.r_max >= 0 && h.r >= P.r_max;
    if (r == 0 || (at_cap && P.cap_mode == 0)) {
      restart = at_cap ? 1 : 0;
      if (sqrt(xx) > P.tol_svd) {
        mode = M_RESTART_ACCEPT;
        if (c == 0) {  // the pass read no U columns: the slot already holds x
          lam = sqrt(rho2);
          cn = 1;
          base_new = slot;
        } else {
          reorth = 2;  // copy x into the slot (second pass), k_decide2 finishes
        }
      } else {
        mode = M_REJECT;
        cn = 0;
        base_new = base + c;
      }
    }
  }
  bool prepped = false;  // coefficients of the next snapshot already written
  if (mode == -1) {
    const bool nx = P.has_next != 0;
    double* t1 = pp.tmp;  // L^{-1} g'[:c]: the next snapshot's coordinates in the current Q_U
    // phase 1 (independent products): ell = N^T tvec;  [l1, t1] = L^{-1} [e, g'[:c]]
    cta_gemv_t_cm(src.N, src.ldn, c, r, pp.tvec, ell, false);
    cta_gemv2_cm<8>(Lib, ldl, c, c, pp.fo.e, nx ? pp.fo.gn : nullptr, pp.l1, nx ? t1 : nullptr, part, true);
    double s_ll = 0.0, s_l1 = 0.0, s_lt = 0.0;
    for (int i = threadIdx.x; i < r; i += blockDim.x) s_ll = fma(ell[i], ell[i], s_ll);
    for (int j = threadIdx.x; j < c; j += blockDim.x) {
      s_l1 = fma(pp.l1[j], pp.l1[j], s_l1);
      if (nx) s_lt = fma(pp.l1[j], t1[j], s_lt);
    }
    block_sum3(s_ll, s_l1, s_lt, red);
    p_sq = xx - s_ll;  // the Pythagorean residual (basis.py:136-138)
    p = (p_sq > 0.0) ? sqrt(p_sq) : 0.0;
    dep = (p < P.tol_svd) || (p == 0.0) || ((int64_t)r >= P.n);
    mode = dep ? M_NORMAL_DEP : M_NORMAL_INDEP;
    if (!dep) {
      const double lam2 = rho2 - s_l1;  // out-of-span part of r1 in the G metric
      const bool room = (slot < P.ccap) && ((int64_t)c < P.n);
      const bool app = room && (lam2 > kFoldTau * kFoldTau * rho2) && (rho2 > 0.0);
      if (app) {
        lam = sqrt(lam2);
        // next snapshot in the extended basis: tvec'_c = (g'_c - l1.t1) / lam and
        // gt'[:c] = L^{-T} (t1 - l1 tvec'_c / lam), gt'_c = tvec'_c / lam
        const double tc = nx ? (pp.fo.gn[c] - s_lt) / lam : 0.0;
        if (nx)
          for (int j = threadIdx.x; j < c; j += blockDim.x) pp.h[j] = t1[j] - pp.l1[j] * (tc / lam);
        cta_gemv_cm<8>(src.N, src.ldn, c, r, ell, -1.0, pp.tvec, pp.y, part, false);  // y = tvec - N ell
        // phase 2: [w, u] = L^{-T} [l1, h]  (w for the new row of L^{-1}, u = gt'[:c])
        cta_gemv2_t_cm(Lib, ldl, c, c, pp.l1, nx ? pp.h : pp.l1, pp.w, pp.gt, true);
        for (int j = threadIdx.x; j < c; j += blockDim.x) {
          Lb[(int64_t)j * ldl + c] = pp.l1[j];
          Lib[(int64_t)j * ldl + c] = -pp.w[j] / lam;
        }
        for (int a = threadIdx.x; a <= c; a += blockDim.x) {
          nj[a] = (a < c) ? (pp.y[a] + pp.l1[a]) / p : lam / p;
          if (nx) pp.tvec[a] = (a < c) ? t1[a] : tc;
        }
        if (threadIdx.x == 0) {
          Lb[(int64_t)c * ldl + c] = lam;
          Lib[(int64_t)c * ldl + c] = 1.0 / lam;
          if (nx) pp.gt[c] = tc / lam;
        }
        prepped = nx;
        cn = c + 1;
        action = 1;
      } else if (room) {
        reorth = 1;
        cta_gemv_cm<8>(src.N, src.ldn, c, r, ell, -1.0, pp.tvec, pp.y, part, false);
        cta_gemv_t_cm(Lib, ldl, c, c, pp.l1, pp.h, true);  // h = L^{-T} l1 = G^{-1} e
      } else if (c >= r + 1) {
        cta_gemv_cm<8>(src.N, src.ldn, c, r, ell, -1.0, pp.tvec, pp.y, part, false);
        for (int a = threadIdx.x; a < c; a += blockDim.x) nj[a] = (pp.y[a] + pp.l1[a]) / p;
        action = 2;
      } else {
        dep = 1;
      }
    }
    if ((dep || action == 2) && nx) {  // U unchanged: tvec' = t1, gt' = L^{-T} t1
      __syncthreads();
      for (int j = threadIdx.x; j < c; j += blockDim.x) pp.tvec[j] = t1[j];
      cta_gemv_t_cm(Lib, ldl, c, c, t1, pp.gt, true);
      prepped = true;
    }
    __syncthreads();
  }
  if (mode == M_RESTART_ACCEPT && reorth == 0 && threadIdx.x == 0) {
    P.L[(int64_t)slot * (ldl + 1)] = lam;
    P.Li[(int64_t)slot * (ldl + 1)] = 1.0 / lam;
  }
  if (threadIdx.x == 0) {
    st->mode = mode;
    st->restart = restart;
    st->action = action;
    st->dep = (mode == M_NORMAL_DEP) ? 1 : dep;
    st->c = c;
    st->cn = cn;
    st->base_new = base_new;
    st->slot = slot;
    st->xx = xx;
    st->rho2 = rho2;
    st->p = p;
    st->p_sq = p_sq;
    st->norm = sqrt(xx);
    st->lam = lam;
    pp.ctl->reorth = reorth;
    if (reorth == 0) {
      pp.ctl->c = cn;
      pp.ctl->base = base_new;
    }
  }
  if (reorth == 0 && P.has_next) {
    if (prepped) {
      if (threadIdx.x == 0) pp.ctl->xx = next_xx(P, pp);
    } else {
      prep_next(P, pp, part);
    }
  }
}

__global__ void __launch_bounds__(kDecideThreads) k_decide(StateView src, Pipe pp, IsvdParams P) {
  extern __shared__ double part[];  // 2 * nw * c_cap
  __shared__ double red[96];
  pdl_wait();
  // the core step of the previous snapshot (second stream).  Dependents are
  // released only afterwards: an early-resident next grid must never hold the
  // SM that k_step_b needs while this CTA spins on it.
  wait_counter(&pp.ctl->bdone, P.b_expect);
  pdl_trigger();
  decide_body(src, pp, P, part, red);
}

// ---------------------------------------------------------------------------
// D2: after the second pass.  DGKS: l2 = L^{-1} e2, lambda2^2 = |r2|^2 - |l2|^2;
// append r2 whenever it carries a genuine out-of-span direction (the reference
// appends j = (x - Phi ell)/p even when it is rounding noise, basis.py:155-156),
// else fold it back (U keeps a spare direction) or demote the update to
// dependent.  Restart copy: the new one-column state.
// ---------------------------------------------------------------------------
__device__ inline void decide2_body(const StateView& src, const Pipe& pp, const IsvdParams& P, double* part,
                                    double* red) {
  const int ro = pp.ctl->reorth;
  if (ro == 0) return;
  IsvdStep* st = pp.step[P.parity];
  double* nj = pp.nj[P.parity];
  const int c = st->c, slot = st->slot, r = src.hdr->r, base = src.hdr->base;
  const int ldl = P.ccap;
  double* Lb = P.L + (int64_t)base * (ldl + 1);
  double* Lib = P.Li + (int64_t)base * (ldl + 1);
  __syncthreads();
  int cn = c, action = 0, dep = 0, base_new = base;
  double lam = 0.0;
  if (ro == 1) {
    const double p = st->p;
    // window mode: the row of r2 for the rest of the window, as the second pass
    // measured it (harmless if r2 is not appended: c does not grow)
    if (P.wn > 0) window_row_measured(P, c, pp.ro.gw);
    double* l2 = pp.h;  // h is spent
    cta_gemv_cm<8>(Lib, ldl, c, c, pp.ro.e, 1.0, nullptr, l2, part, true);
    double pq = 0.0;
    for (int j = threadIdx.x; j < c; j += blockDim.x) pq = fma(l2[j], l2[j], pq);
    const double ll2 = block_sum(pq, red);
    const double rho2b = pp.ro.scal[0];
    const double lam2 = rho2b - ll2;
    if ((lam2 > 0.25 * rho2b) && (rho2b > 0.0)) {
      lam = sqrt(lam2);
      append_factor_row(Lb, Lib, ldl, c, l2, lam, pp.tmp);
      for (int a = threadIdx.x; a <= c; a += blockDim.x)
        nj[a] = (a < c) ? (pp.y[a] + pp.l1[a] + l2[a]) / p : lam / p;
      if (P.wn == 0 && threadIdx.x == 0) pp.fo.gn[c] = pp.ro.scal[2];  // r2 . x_next
      cn = c + 1;
      action = 1;
    } else if (c >= r + 1) {
      for (int a = threadIdx.x; a < c; a += blockDim.x) nj[a] = (pp.y[a] + pp.l1[a] + l2[a]) / p;
      action = 2;
    } else {
      dep = 1;
    }
  } else {
    lam = sqrt(pp.ro.scal[0]);
    if (P.wn > 0) window_row(P, 0, 0, nullptr, nullptr);  // U = [x]: row 0 = x . x_j
    if (threadIdx.x == 0) {
      P.L[(int64_t)slot * (ldl + 1)] = lam;
      P.Li[(int64_t)slot * (ldl + 1)] = 1.0 / lam;
      if (P.wn == 0) pp.fo.gn[0] = pp.ro.scal[2];  // x . x_next
      st->rho2 = pp.ro.scal[0];
    }
    cn = 1;
    base_new = slot;
  }
  if (threadIdx.x == 0) {
    if (ro == 1) {
      st->action = action;
      st->dep = dep;
    }
    st->cn = cn;
    st->base_new = base_new;
    st->lam = lam;
    pp.ctl->c = cn;
    pp.ctl->base = base_new;
    pp.ctl->reorth = 0;
  }
  if (P.has_next) prep_next(P, pp, part);
}

__global__ void __launch_bounds__(kDecideThreads) k_decide2(StateView src, Pipe pp, IsvdParams P) {
  extern __shared__ double part[];
  __shared__ double red[96];
  pdl_enter();
  decide2_body(src, pp, P, part, red);
  signal_counter(&pp.ctl->decided);  // the decisions of this snapshot are complete
  trace_stamp(P.trace, 7);
}

// ---------------------------------------------------------------------------
// Window mode: the decisions of update t in two halves around an optional
// residual pass (the projection g_t = U^T x_t came from the window pass).
//   A (k_decide_a): restart / reject, ell = N^T L^{-1} g, the Pythagorean p and
//     the dependent test (basis.py:112-139).  A dependent snapshot needs no pass
//     over U at all: A prepares the next snapshot and the decision is final.
//   B (k_decide_b): after the residual pass (independent snapshots and a first
//     accept): how r enters U, exactly as decide_body's independent branch,
//     plus the new U column's row of the window projections (window_row).
// ---------------------------------------------------------------------------
__device__ inline void decide_a_body(const StateView& src, const Pipe& pp, const IsvdParams& P, double* part,
                                     double* red) {
  const IsvdHdr h = *src.hdr;
  IsvdStep* st = pp.step[P.parity];
  double* ell = pp.ell[P.parity];
  const int c = h.c, base = h.base, r = h.r;
  const double xx = pp.ctl->xx;
  const int slot = base + c;
  int mode = -1, restart = 0, dep = 0, cn = c, base_new = base, reorth = 0, resid = 0;
  double p = 0.0, p_sq = 0.0;
  if (h.status != 0 || !isfinite(xx)) {
    mode = M_ERROR;
  } else {
    const bool at_cap = P.r_max >= 0 && h.r >= P.r_max;
    if (r == 0 || (at_cap && P.cap_mode == 0)) {
      restart = at_cap ? 1 : 0;
      if (sqrt(xx) > P.tol_svd) {
        mode = M_RESTART_ACCEPT;
        if (c == 0) resid = 1;  // the residual pass writes x itself into the slot (B finishes)
        else reorth = 2;        // the second pass copies x into the slot (k_decide2 finishes)
      } else {
        mode = M_REJECT;
        cn = 0;
        base_new = base + c;
      }
    }
  }
  if (mode == -1) {
    cta_gemv_t_cm(src.N, src.ldn, c, r, pp.tvec, ell, false);  // ell = N^T L^{-1} g
    double s_ll = 0.0;
    for (int i = threadIdx.x; i < r; i += blockDim.x) s_ll = fma(ell[i], ell[i], s_ll);
    s_ll = block_sum(s_ll, red);
    p_sq = xx - s_ll;  // the Pythagorean residual (basis.py:136-138)
    p = (p_sq > 0.0) ? sqrt(p_sq) : 0.0;
    dep = (p < P.tol_svd) || (p == 0.0) || ((int64_t)r >= P.n);
    mode = dep ? M_NORMAL_DEP : M_NORMAL_INDEP;
    resid = dep ? 0 : 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st->mode = mode;
    st->restart = restart;
    st->action = 0;
    st->dep = (mode == M_NORMAL_DEP) ? 1 : 0;
    st->c = c;
    st->cn = cn;
    st->base_new = base_new;
    st->slot = slot;
    st->xx = xx;
    st->rho2 = 0.0;
    st->p = p;
    st->p_sq = p_sq;
    st->norm = sqrt(xx);
    st->lam = 0.0;
    pp.ctl->resid = resid;
    pp.ctl->reorth = reorth;
    if (!resid && reorth == 0) {
      pp.ctl->c = cn;
      pp.ctl->base = base_new;
    }
  }
  // a final decision (dependent, reject, error): U is unchanged or emptied,
  // so the next snapshot's coefficients come straight from the window
  if (!resid && reorth == 0 && P.has_next) prep_next(P, pp, part);
}

// `stage` (or null): room for L^{-1}'s live block and N in shared memory.  After a pass over U
// the small state is no longer in L2; the four matrix-vector sweeps below would each pay
// several memory latencies on it, so both are fetched once with every load in flight.
__device__ inline void decide_b_body(const StateView& src, const Pipe& pp, const IsvdParams& P, double* part,
                                     double* red, double* stage = nullptr, size_t stage_doubles = 0) {
  if (!*(volatile const int32_t*)&pp.ctl->resid) return;
  const IsvdHdr h = *src.hdr;
  IsvdStep* st = pp.step[P.parity];
  double* ell = pp.ell[P.parity];
  double* nj = pp.nj[P.parity];
  const int mode = st->mode;
  const int c = st->c, base = h.base, r = h.r, slot = st->slot;
  const int ldl = P.ccap;
  double* Lb = P.L + (int64_t)base * (ldl + 1);
  double* Lib = P.Li + (int64_t)base * (ldl + 1);
  const double* Lir = Lib;  // what the sweeps read
  int ldlr = ldl;
  const double* Nr = src.N;
  int ldnr = src.ldn;
  if (stage && mode != M_RESTART_ACCEPT && (size_t)c * (c + r) <= stage_doubles) {
    cta_stage_block(stage, c, Lib, ldl, c, c, true);
    cta_stage_block(stage + (size_t)c * c, c, src.N, src.ldn, c, r, false);
    Lir = stage;
    ldlr = c;
    Nr = stage + (size_t)c * c;
    ldnr = c;
    __syncthreads();
  }
  const double rho2 = pp.fo.scal[0];
  const double p = st->p;
  int action = 0, dep = 0, cn = c, base_new = base, reorth = 0;
  double lam = 0.0;
  bool prepped = false;
  const bool nx = P.has_next != 0;
  if (mode == M_RESTART_ACCEPT) {  // first accept into an empty U: the slot holds x
    lam = sqrt(rho2);
    cn = 1;
    base_new = slot;
    window_row(P, 0, 0, nullptr, nullptr);
    if (threadIdx.x == 0) {
      P.L[(int64_t)slot * (ldl + 1)] = lam;
      P.Li[(int64_t)slot * (ldl + 1)] = 1.0 / lam;
    }
  } else {
    double* t1 = pp.tmp;  // L^{-1} g'[:c]: the next snapshot's coordinates in the current Q_U
    cta_gemv2_cm<8>(Lir, ldlr, c, c, pp.fo.e, nx ? pp.fo.gn : nullptr, pp.l1, nx ? t1 : nullptr, part, true);
    double s_l1 = 0.0, s_lt = 0.0, s_zero = 0.0;
    for (int j = threadIdx.x; j < c; j += blockDim.x) {
      s_l1 = fma(pp.l1[j], pp.l1[j], s_l1);
      if (nx) s_lt = fma(pp.l1[j], t1[j], s_lt);
    }
    block_sum3(s_l1, s_lt, s_zero, red);
    const double lam2 = rho2 - s_l1;  // out-of-span part of r1 in the G metric
    const bool room = (slot < P.ccap) && ((int64_t)c < P.n);
    const bool app = room && (lam2 > kFoldTau * kFoldTau * rho2) && (rho2 > 0.0);
    if (app) {
      // r1 becomes U column c: its row of the window (and g'_c = r1 . x_next), as
      // the residual pass measured it on the stored r1
      window_row_measured(P, c, pp.fo.gw);
      lam = sqrt(lam2);
      const double tc = nx ? (pp.fo.gn[c] - s_lt) / lam : 0.0;
      if (nx)
        for (int j = threadIdx.x; j < c; j += blockDim.x) pp.h[j] = t1[j] - pp.l1[j] * (tc / lam);
      cta_gemv_cm<8>(Nr, ldnr, c, r, ell, -1.0, pp.tvec, pp.y, part, false);  // y = tvec - N ell
      cta_gemv2_t_cm(Lir, ldlr, c, c, pp.l1, nx ? pp.h : pp.l1, pp.w, pp.gt, true);
      for (int j = threadIdx.x; j < c; j += blockDim.x) {
        Lb[(int64_t)j * ldl + c] = pp.l1[j];
        Lib[(int64_t)j * ldl + c] = -pp.w[j] / lam;
      }
      for (int a = threadIdx.x; a <= c; a += blockDim.x) {
        nj[a] = (a < c) ? (pp.y[a] + pp.l1[a]) / p : lam / p;
        if (nx) pp.tvec[a] = (a < c) ? t1[a] : tc;
      }
      if (threadIdx.x == 0) {
        Lb[(int64_t)c * ldl + c] = lam;
        Lib[(int64_t)c * ldl + c] = 1.0 / lam;
        if (nx) pp.gt[c] = tc / lam;
      }
      prepped = nx;
      cn = c + 1;
      action = 1;
    } else if (room) {
      reorth = 1;
      cta_gemv_cm<8>(Nr, ldnr, c, r, ell, -1.0, pp.tvec, pp.y, part, false);
      cta_gemv_t_cm(Lir, ldlr, c, c, pp.l1, pp.h, true);  // h = L^{-T} l1 = G^{-1} e
    } else if (c >= r + 1) {
      cta_gemv_cm<8>(Nr, ldnr, c, r, ell, -1.0, pp.tvec, pp.y, part, false);
      for (int a = threadIdx.x; a < c; a += blockDim.x) nj[a] = (pp.y[a] + pp.l1[a]) / p;
      action = 2;
    } else {
      dep = 1;
    }
    if ((dep || action == 2) && nx) {  // U unchanged: tvec' = t1, gt' = L^{-T} t1
      __syncthreads();
      for (int j = threadIdx.x; j < c; j += blockDim.x) pp.tvec[j] = t1[j];
      cta_gemv_t_cm(Lir, ldlr, c, c, t1, pp.gt, true);
      prepped = true;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->action = action;
    if (dep) st->dep = 1;
    st->cn = cn;
    st->base_new = base_new;
    st->rho2 = rho2;
    st->lam = lam;
    pp.ctl->reorth = reorth;
    if (reorth == 0) {
      pp.ctl->c = cn;
      pp.ctl->base = base_new;
    }
  }
  if (reorth == 0 && nx) {
    if (prepped) {
      if (threadIdx.x == 0) pp.ctl->xx = next_xx(P, pp);
    } else {
      prep_next(P, pp, part);
    }
  }
}

__global__ void __launch_bounds__(kDecideThreads) k_decide_a(StateView src, Pipe pp, IsvdParams P) {
  extern __shared__ double part[];
  __shared__ double red[96];
  pdl_wait();
  wait_counter(&pp.ctl->bdone, P.b_expect);  // the previous snapshot's core step wrote N, sigma
  pdl_trigger();
  trace_stamp(P.trace, 0);
  if (*(volatile const int32_t*)&pp.ctl->a_inline == P.d_expect) {
    // the previous core step already decided this snapshot's first half
    // (decide_next_inline): only the next snapshot's coefficients remain
    if (!pp.ctl->resid && pp.ctl->reorth == 0 && P.has_next) prep_next(P, pp, part);
  } else {
    decide_a_body(src, pp, P, part, red);
    signal_counter(&pp.ctl->adone);  // the core step of this snapshot may start its SVD
  }
  trace_stamp(P.trace, 1);
}

__global__ void __launch_bounds__(kDecideThreads) k_decide_b(StateView src, Pipe pp, IsvdParams P) {
  extern __shared__ double part[];
  __shared__ double red[96];
  pdl_enter();
  trace_stamp(P.trace, 4);
  const size_t npart = (size_t)2 * (kDecideThreads / 32) * ((P.ccap + 31) / 32 * 32);
  decide_b_body(src, pp, P, part, red, P.stage_doubles > 0 ? part + npart : nullptr, (size_t)P.stage_doubles);
  trace_stamp(P.trace, 5);
}

template <int MAXJ>
__global__ void __launch_bounds__(kPassThreads, 1) k_pass(PassArgs a, int nstages) {
  extern __shared__ __align__(128) double stg[];  // nstages x (kStageRows x cs), column segments
  __shared__ double red_s[96];
  __shared__ __align__(8) uint64_t full[kPassMaxStages];
  __shared__ __align__(8) uint64_t empty[kPassMaxStages];
  __shared__ double gts[kPassConsumers * MAXJ];
  __shared__ __align__(16) double red[2][kPassConsumers][kSubRows];
  __shared__ double wsc[3];
  __shared__ int s_last;
  pdl_enter();
  trace_stamp(a.trace, a.kind == PASS_SECOND ? 6 : 2);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int c = a.ctl->c;
  const int base = a.ctl->base;
  const int slot = base + c;
  const double* x = a.x;
  const double* coef = a.coef;
  bool do_e = false, do_gn = false, x_is_slot = false;
  if (a.kind == PASS_SECOND) {
    const int ro = a.ctl->reorth;
    if (ro == 0) return;
    if (ro == 1) {
      x_is_slot = true;  // r2 = r1 - U h, in place on the slot column
      x = a.U;
      do_e = true;
    } else {
      coef = nullptr;  // slot <- x
      c = 0;
    }
  } else if (a.kind == PASS_FUSED || a.kind == PASS_RESID) {
    if (a.kind == PASS_RESID && *(volatile const int32_t*)&a.ctl->resid == 0) return;
    do_e = true;
    do_gn = a.xn != nullptr;
  } else {
    x = nullptr;
    do_gn = true;
  }
  const int64_t tstride = (int64_t)kUTile * a.ccap;  // one U tile: kUTile rows x ccap columns
  const bool do_r = x != nullptr;
  const bool do_coef = do_r && coef != nullptr && c > 0;
  const bool do_xn = a.xn != nullptr;
  if (a.prof && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(a.prof + (a.kind == PASS_SECOND ? 1 : 0),
              8ull * (unsigned long long)a.n * (unsigned long long)(c + (do_r ? 2 : 0) + (do_xn ? 1 : 0)));
  for (int j = threadIdx.x; j < kPassConsumers * MAXJ; j += blockDim.x) gts[j] = (do_coef && j < c) ? coef[j] : 0.0;
  const int64_t ntiles = a.ldu / kStageRows;
  const int64_t per = ceil_div(ntiles, gridDim.x);
  const int64_t t0 = blockIdx.x * per;
  const int64_t nt = max((int64_t)0, min(ntiles, t0 + per) - t0);
  // stage layout: [U column segments base .. base+cu) [x segment] [xn segment], kStageRows rows each.
  // DGKS reads the slot column as x: it is U column c of the stage.
  const int cu = c + (x_is_slot ? 1 : 0);
  const bool x_stage = x_is_slot || (do_r && a.x_bulk);
  const bool x_own = do_r && !x_is_slot && a.x_bulk;  // x has its own segment
  const bool xn_stage = do_xn && a.xn_bulk;
  const int x_col = x_is_slot ? c : cu;
  const int xn_col = cu + (x_own ? 1 : 0);
  // window mode: the later snapshots' segments ride in the same stage (a.xw_bulk)
  const int nxw_st = (do_r && a.xw_bulk) ? a.nxw : 0;
  const int xw_col = xn_col + (xn_stage ? 1 : 0);
  const int cs = cu + (x_own ? 1 : 0) + (xn_stage ? 1 : 0) + nxw_st;
  const unsigned stage_elems = (unsigned)(kStageRows * cs);  if (threadIdx.x == 0) {
    for (int st = 0; st < nstages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kPassConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wid == 0) {
    // ---------------- producer ----------------
    if (lane == 0 && cs > 0) {
      const uint64_t pol_stream = l2_policy_evict_first();  // U is read once per pass (bulk.cuh)
      const bool x_stream = a.n >= ((int64_t)8 << 20);
      for (int64_t i = 0; i < nt; ++i) {
        const int st = (int)(i % nstages);
        const int64_t use = i / nstages;
        if (use > 0) mbar_wait(&empty[st], (unsigned)((use - 1) & 1));
        const int64_t row0 = (t0 + i) * kStageRows;
        const int valid = (int)max((int64_t)0, min((int64_t)kStageRows, a.n - row0));
        const unsigned bu = (unsigned)(kStageRows * cu) * 8u, bv = (unsigned)valid * 8u;
        mbar_expect_tx(&full[st], bu + (x_own ? bv : 0u) + (xn_stage ? bv : 0u) + bv * (unsigned)nxw_st);
        double* dst = stg + (size_t)st * stage_elems;
        // the live column segments of U tile t0 + i are one contiguous run
        if (bu) bulk_g2s_stream(dst, a.U + (t0 + i) * tstride + (int64_t)base * kUTile, bu, &full[st], pol_stream);
        // snapshot columns: a window's columns are re-read from L2 by its passes while they fit
        // there (8 x 8 MB at n = 2^20); columns of 64 MB and more stream like U
        if (x_stream) {
          if (x_own && bv) bulk_g2s_stream(dst + x_col * kStageRows, x + row0, bv, &full[st], pol_stream);
          if (xn_stage && bv) bulk_g2s_stream(dst + xn_col * kStageRows, a.xn + row0, bv, &full[st], pol_stream);
          if (bv)
            for (int j = 0; j < nxw_st; ++j)
              bulk_g2s_stream(dst + (xw_col + j) * kStageRows, a.xw[j] + row0, bv, &full[st], pol_stream);
        } else {
          if (x_own && bv) bulk_g2s(dst + x_col * kStageRows, x + row0, bv, &full[st]);
          if (xn_stage && bv) bulk_g2s(dst + xn_col * kStageRows, a.xn + row0, bv, &full[st]);
          if (bv)
            for (int j = 0; j < nxw_st; ++j) bulk_g2s(dst + (xw_col + j) * kStageRows, a.xw[j] + row0, bv, &full[st]);
        }
      }
    }
  } else {
    // ---------------- consumers ----------------
    const int cw = wid - 1;
    double ae[MAXJ], ag[MAXJ];
#pragma unroll
    for (int q = 0; q < MAXJ; ++q) { ae[q] = 0.0; ag[q] = 0.0; }
    double rr = 0.0, gs = 0.0, xq = 0.0, gwa = 0.0;
    const double* xwc = (cw < a.nxw) ? a.xw[cw] : nullptr;
    for (int64_t i = 0; i < nt; ++i) {
      const int st = (int)(i % nstages);
      const int64_t use = i / nstages;
      if (cs > 0) mbar_wait(&full[st], (unsigned)(use & 1));
      if (a.dbg & 1) {
        __syncwarp();
        if (lane == 0 && cs > 0) mbar_arrive(&empty[st]);
        continue;
      }
      const double* tile = stg + (size_t)st * stage_elems;
#pragma unroll 1
      for (int hh = 0; hh < kStageRows / kSubRows; ++hh) {
        const int64_t sub = (t0 + i) * (kStageRows / kSubRows) + hh;  // global sub-tile index
        const int64_t row = sub * kSubRows + 2 * lane;
        const bool live0 = row < a.n, live1 = row + 1 < a.n;
        double2 xv = make_double2(0.0, 0.0), xnv = make_double2(0.0, 0.0);
        double* scol = a.U + sub * tstride + (int64_t)slot * kUTile;  // this tile's slot segment
        if (x_stage) {
          xv = reinterpret_cast<const double2*>(tile + x_col * kStageRows + hh * kSubRows)[lane];
        } else if (do_r) {
          xv.x = live0 ? x[row] : 0.0;
          xv.y = live1 ? x[row + 1] : 0.0;
        }
        if (xn_stage) {
          xnv = reinterpret_cast<const double2*>(tile + xn_col * kStageRows + hh * kSubRows)[lane];
        } else if (do_xn) {
          xnv.x = live0 ? __ldg(a.xn + row) : 0.0;
          xnv.y = live1 ? __ldg(a.xn + row + 1) : 0.0;
        }
        if (!live0) { xv.x = 0.0; xnv.x = 0.0; }
        if (!live1) { xv.y = 0.0; xnv.y = 0.0; }
        // this warp's later window snapshot (r . x_j below): read before the stage is released
        double2 wv = make_double2(0.0, 0.0);
        if (do_r && xwc) {
          if (nxw_st) wv = reinterpret_cast<const double2*>(tile + (xw_col + cw) * kStageRows + hh * kSubRows)[lane];
          else wv = make_double2(live0 ? __ldg(xwc + row) : 0.0, live1 ? __ldg(xwc + row + 1) : 0.0);
          if (!live0) wv.x = 0.0;
          if (!live1) wv.y = 0.0;
        }
        double2 u[MAXJ];
#pragma unroll
        for (int q = 0; q < MAXJ; ++q) {
          const int j = cw + kPassConsumers * q;
          u[q] = (j < c) ? reinterpret_cast<const double2*>(tile + j * kStageRows + hh * kSubRows)[lane]
                         : make_double2(0.0, 0.0);
        }
        if (hh == kStageRows / kSubRows - 1 && cs > 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);  // the stage is in registers
        }
        double2 r = xv;
        if (do_coef) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int q = 0; q < MAXJ; ++q) {
            const double gq = gts[cw + kPassConsumers * q];
            s0 = fma(u[q].x, gq, s0);
            s1 = fma(u[q].y, gq, s1);
          }
          reinterpret_cast<double2*>(&red[sub & 1][cw][0])[lane] = make_double2(s0, s1);
          asm volatile("bar.sync 1, %0;" ::"n"(32 * kPassConsumers) : "memory");
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int w = 0; w < kPassConsumers; ++w) {
            const double2 p = reinterpret_cast<const double2*>(&red[sub & 1][w][0])[lane];
            d0 += p.x;
            d1 += p.y;
          }
          r.x = xv.x - d0;
          r.y = xv.y - d1;
        }
        if (!live0) r.x = 0.0;
        if (!live1) r.y = 0.0;
        if (do_r && xwc) gwa = fma(r.y, wv.y, fma(r.x, wv.x, gwa));  // r . x_j on the stored (rounded) r
        if (do_r) {
          if (cw == kPassConsumers - 1) {
            __stcs(reinterpret_cast<double2*>(scol) + lane, r);  // streaming: written once, read by the next pass
            rr = fma(r.y, r.y, fma(r.x, r.x, rr));
            gs = fma(r.y, xnv.y, fma(r.x, xnv.x, gs));
          }
          if (do_e) {
#pragma unroll
            for (int q = 0; q < MAXJ; ++q) ae[q] = fma(u[q].y, r.y, fma(u[q].x, r.x, ae[q]));
          }
        }
        if (do_gn) {
#pragma unroll
          for (int q = 0; q < MAXJ; ++q) ag[q] = fma(u[q].y, xnv.y, fma(u[q].x, xnv.x, ag[q]));
          if (cw == kPassConsumers - 1) xq = fma(xnv.y, xnv.y, fma(xnv.x, xnv.x, xq));
        }
      }
    }
    // per-CTA partials: [0, PG) e | [PG, 2 PG) gn | 2 PG + {0: r.r, 1: xn.xn, 2: r.xn}
    const int PG = (a.pstride - 16) / 2;  // [e | gn | r.r, xn.xn, r.xn, r.x_w (kWB - 1)]
    // output-major: the last CTA's sum over the CTAs then reads contiguous runs (8 sectors
    // per 32 CTAs instead of 32: that reduction is one SM's L2 bandwidth)
    double* mypart = a.part + blockIdx.x;
    const int64_t pl = a.pld;
#pragma unroll
    for (int q = 0; q < MAXJ; ++q) {
      const int j = cw + kPassConsumers * q;
      if (do_e) {
        const double v = warp_sum(ae[q]);
        if (lane == 0 && j < c) mypart[j * pl] = v;
      }
      if (do_gn) {
        const double v = warp_sum(ag[q]);
        if (lane == 0 && j < c) mypart[(PG + j) * pl] = v;
      }
    }
    if (cw == kPassConsumers - 1) {
      rr = warp_sum(rr);
      gs = warp_sum(gs);
      xq = warp_sum(xq);
      if (lane == 0) {
        mypart[(2 * PG) * pl] = rr;
        mypart[(2 * PG + 1) * pl] = xq;
        mypart[(2 * PG + 2) * pl] = gs;
      }
    }
    if (xwc) {
      gwa = warp_sum(gwa);
      if (lane == 0) mypart[(2 * PG + 3 + cw) * pl] = gwa;
    }
  }
  if (!last_cta_arrives(a.counter, &s_last)) return;
  if (a.trace && threadIdx.x == 0 && a.kind != PASS_SECOND) {
    unsigned long long tt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
    a.trace[3] = (long long)tt;
  }
  // one warp per output, lanes stride over the CTA partials, fixed tree: deterministic
  const int PG = (a.pstride - 16) / 2;  // [e | gn | r.r, xn.xn, r.xn, r.x_w (kWB - 1)]
  const int nwarps = blockDim.x >> 5;
  const int ne = do_e ? c : 0, ng = do_gn ? c : 0;
  const int nxw = x ? a.nxw : 0;
  const int nout = ne + ng + 3 + nxw;
  // four outputs per warp at a time (their loads in flight together); each
  // output keeps the same lane / stripe summation order: deterministic
  auto out_col = [&](int o) { return o < ne ? o : (o < ne + ng ? PG + (o - ne) : 2 * PG + (o - ne - ng)); };
  for (int o0 = wid; o0 < nout; o0 += 4 * nwarps) {
    double s[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int o = o0 + q * nwarps;
      s[q][0] = s[q][1] = s[q][2] = s[q][3] = 0.0;
      if (o >= nout) continue;
      const double* pc = a.part + (int64_t)out_col(o) * a.pld;
      const int G = (int)gridDim.x;
      if (G <= 160) {
        // every load of the four outputs in flight at once (the loops below stall on
        // memory once per trip: ~25k cycles for ~100 outputs); the same summation order
        double v[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) v[k] = (lane + 32 * k < G) ? __ldcg(pc + lane + 32 * k) : 0.0;
        if (lane + 96 < G) {
          s[q][0] = v[0]; s[q][1] = v[1]; s[q][2] = v[2]; s[q][3] = v[3];
          if (lane + 128 < G) s[q][0] += v[4];
        } else {
#pragma unroll
          for (int k = 0; k < 5; ++k)
            if (lane + 32 * k < G) s[q][0] += v[k];
        }
        continue;
      }
      int b = lane;
      for (; b + 96 < G; b += 128) {
        s[q][0] += __ldcg(pc + b);
        s[q][1] += __ldcg(pc + b + 32);
        s[q][2] += __ldcg(pc + b + 64);
        s[q][3] += __ldcg(pc + b + 96);
      }
      for (; b < G; b += 32) s[q][0] += __ldcg(pc + b);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int o = o0 + q * nwarps;
      const double sum = warp_sum((s[q][0] + s[q][1]) + (s[q][2] + s[q][3]));
      if (lane == 0 && o < nout) {
        if (o < ne) a.out.e[o] = sum;
        else if (o < ne + ng) a.out.gn[o - ne] = sum;
        else {
          const int k = o - ne - ng;
          if (k < 3) a.out.scal[k] = sum;
          else a.out.gw[k - 3] = sum;
          if (k == 2 && a.kind == PASS_FUSED && do_gn) a.out.gn[c] = sum;  // r . x_next
        }
      }
    }
  }
  if (a.trace && threadIdx.x == 0 && a.kind != PASS_SECOND) {  // the reduction's end
    unsigned long long tt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
    a.trace[13] = (long long)tt;
  }
  if (a.tail) {
    __syncthreads();  // this CTA's outputs are complete
    if (a.tail == 1 && a.b_expect >= 0) {
      // the core step of the previous snapshot (second stream, its own SM) writes
      // the state this decision reads; it signals completion on ctl->bdone
      if (threadIdx.x == 0) {
        const volatile int32_t* bd = &a.dpp.ctl->bdone;
        while (*bd < a.b_expect) __nanosleep(100);
        __threadfence();
      }
      __syncthreads();
    }
    if (a.tail == 1) decide_body(a.dsrc, a.dpp, a.dP, stg, red_s);
    else decide2_body(a.dsrc, a.dpp, a.dP, stg, red_s);
  }
}


// ---------------------------------------------------------------------------
// B (one CTA; second stream): everything of update t that the next snapshot's
// pass does not depend on.
//   * bordered core Q = [[diag(sigma), ell], [0, p]] (basis.py:141-144) and its
//     SVD by the rank-one secular solver, sort + sign rule (linalg.py:31-38, 53)
//   * N' = [N n_j] W_bar (basis.py:150-158 in Q_U coordinates), truncation
//     (basis.py:160-168), drift |phi_0 . phi_last| = |N_0 . N_last| and the QR
//     of basis.py:170-174 on N' (Q_U is orthonormal: QR(Phi') = Q_U QR(N'))
// ---------------------------------------------------------------------------
// mid_ctr (window mode): the core SVD only needs k_decide_a's results; the
// rest (how r entered U: cn, n_j, a demotion to dependent) waits here for
// *mid_ctr >= mid_target (the decision chain's end).
template <bool kSmem>  // the work area in shared memory (LDS/STS instead of generic accesses) or in pp.work
__device__ inline void step_b_body(const StateView& src, const StateView& dst, const Pipe& pp, const IsvdParams& P,
                                   double* smem, double* red, const int32_t* mid_ctr = nullptr,
                                   int32_t mid_target = -1, const double** n_sm = nullptr, int* n_sm_ld = nullptr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const IsvdHdr h = *src.hdr;
  IsvdStep* st = pp.step[P.parity];
  const double* ell = pp.ell[P.parity];
  const double* wj = pp.nj[P.parity];
  const int mode0 = *(volatile const int32_t*)&st->mode;
  if (mid_ctr && mode0 != M_NORMAL_DEP && mode0 != M_NORMAL_INDEP) {
    wait_counter(mid_ctr, mid_target);  // restart / reject / error: cheap, needs the whole chain
    mid_ctr = nullptr;
  }
  const int mode = st->mode;
  IsvdHdr o = h;
  o.flags = 0;
  o.p = 0.0;
  o.drift = 0.0;
  o.xnorm = st->norm;
  if (mode == M_ERROR) {
    if (threadIdx.x == 0) {
      o.status = 1;
      o.flags = F_ERROR;
      *dst.hdr = o;
      st->m = 0;
      st->mkeep = -1;
      *pp.vrec[P.parity] = VRec{mode, 0, -1, 0};
    }
    return;
  }
  if (mode == M_REJECT || mode == M_RESTART_ACCEPT) {
    if (threadIdx.x == 0) {
      if (st->restart) { o.n_restarts += 1; o.flags |= F_RESTART; }
      o.c = st->cn;
      o.base = st->base_new;
      if (mode == M_REJECT) {
        o.r = 0;
        o.n_rejected += 1;
        o.flags |= F_REJECTED;
        st->mkeep = 0;
      } else {
        o.r = 1;
        dst.N[0] = st->lam / st->norm;  // Phi = x / ||x|| = Q_U N with Q_U = x / lam
        dst.sigma[0] = st->norm;
        st->mkeep = 1;
      }
      st->m = 0;
      *dst.hdr = o;
      *pp.vrec[P.parity] = VRec{mode, 0, st->mkeep, 0};
    }
    return;
  }
  STROM_TPROBE(P, 0);
  bool dep = *(volatile const int32_t*)&st->dep != 0;
  const int r = h.r, c = st->c, m = r + 1;
  const double p = st->p;
  o.p = p;
  o.p_sq = st->p_sq;
  STROM_TPROBE(P, 1);
  // ---- shared-memory plan (global fallback when it does not fit) ----------
  //   WS m^2 | Wt m^2 | Vt m^2 | core work 16 ms | WB ccap x m (staged N_b, later QR's M)
  const int64_t ms = P.work_stride;
  double* base = kSmem ? smem : pp.work + 4 * ms;
  double* WS = base;                      // sorted, signed W_bar (m x m)
  double* Wt = WS + (int64_t)m * m;       // vectors by slot, later W^T W
  double* Vt = Wt + (int64_t)m * m;       // vectors by slot, later the polished W_bar
  double* cb = Vt + (int64_t)m * m;
  double* WB = cb + 16 * ms;              // N_b = [[N, n_j]] (cn x m, ld ccap)
  double* NS = Wt;                        // after the SVD: N' (cn x mk, ld cn) over the dead Wt | Vt
  double* svs = cb + 14 * ms;             // m sorted singular values
  CoreSvdWork cw;
  cw.d = cb; cw.z = cb + ms; cw.zh = cb + 2 * ms; cw.mu = cb + 3 * ms; cw.sv = cb + 4 * ms;
  cw.rc = cb + 5 * ms; cw.rs = cb + 6 * ms;
  cw.dk = cb + 11 * ms; cw.zk = cb + 12 * ms; cw.dorg = cb + 13 * ms;
  {
    int* ib = reinterpret_cast<int*>(cb + 7 * ms);
    cw.org = ib; cw.kset = ib + ms; cw.defl = ib + 2 * ms; cw.ra = ib + 3 * ms; cw.rb = ib + 4 * ms;
    cw.perm = ib + 5 * ms; cw.cnt = ib + 6 * ms;
  }
  // stage N (c x r) into N_b now: the L2 loads overlap the solver's set-up; the appended
  // row and the n_j column follow once the decision chain is known (below)
  cta_stage_block(WB, P.ccap, src.N, src.ldn, c, r, false);
  // ---- 2. the bordered core and its SVD (rank-one secular solver) ----------
  for (int attempt = 0; attempt < 2; ++attempt) {  // (one inlined copy of the solver)
    core_svd_secular(src.sigma, ell, dep ? 0.0 : p, r, cw, Wt, Vt, svs, WS, pp.vbar, red,
                     (P.tprobe && attempt == 0) ? P.tprobe + 8 : nullptr,
                     (P.tprobe && attempt == 0) ? P.tprobe + 300 : nullptr);
    if (attempt == 0) trace_stamp(P.trace, 9);
    if (attempt == 1 || !mid_ctr) break;
    wait_counter(mid_ctr, mid_target);
    trace_stamp(P.trace, 10);
    const bool dep2 = *(volatile const int32_t*)&st->dep != 0;
    if (dep2 == dep) break;
    dep = dep2;  // the residual could not enter U: the update is dependent after all
    __syncthreads();
  }
  const int cn = st->cn;
  const int action = st->action;
  const bool appended = (action == 1);
  // rest of N_b: the appended row of columns 0..r-1 is 0, column r = n_j
  for (int idx = threadIdx.x; idx < r * (cn - c); idx += blockDim.x) {
    const int b = idx / (cn - c), a = c + idx - b * (cn - c);
    WB[b * P.ccap + a] = 0.0;
  }
  for (int a = threadIdx.x; a < cn; a += blockDim.x) WB[r * P.ccap + a] = dep ? 0.0 : wj[a];
  __syncthreads();
  STROM_TPROBE(P, 2);
  // (no orthogonality polish needed: the Gu-Eisenstat vectors are orthogonal to
  // working precision, unlike accumulated Jacobi rotations)
  STROM_TPROBE(P, 3);
  // ---- 3. truncation (basis.py:160-168) ------------------------------------
  int mk = dep ? r : m;
  bool trunc = false;
  if (mk > 0 && svs[mk - 1] < P.tol_sv) { mk -= 1; trunc = true; }
  if (P.r_max >= 0 && mk > P.r_max) { mk = P.r_max; trunc = true; }
  // ---- 4. N' = N_b W_bar[:, :mk]  (basis.py:150-158 in Q_U coordinates) ---
  // a second copy of N' stays in the work area (over the dead Wt | Vt) for the drift test,
  // the QR and the next snapshot's inline decision, when it fits there
  const bool ns_ok = (int64_t)cn * mk <= 2 * (int64_t)m * m;
  const double* Nn = ns_ok ? NS : dst.N;
  const int64_t ldnn = ns_ok ? cn : dst.ldn;
  {
    const int kdim = dep ? r : m;
    if (ns_ok)
      cta_gemm_dmma_blk<4, 2>(cn, mk, kdim, WB, 1, P.ccap, WS, 1, m, [&](int a, int k, double v) {
        dst.N[(int64_t)k * dst.ldn + a] = v;
        NS[k * cn + a] = v;
      });
    else
      cta_gemm_dmma_blk<4, 2>(cn, mk, kdim, WB, 1, P.ccap, WS, 1, m,
                              [&](int a, int k, double v) { dst.N[(int64_t)k * dst.ldn + a] = v; });
  }
  for (int k = threadIdx.x; k < mk; k += blockDim.x) dst.sigma[k] = svs[k];
  __syncthreads();
  STROM_TPROBE(P, 4);
  // ---- 5. drift test and small-space QR (basis.py:170-174) -----------------
  bool did_qr = false;
  double drift = 0.0;
  if (mk > 1) {
    // phi_0 . phi_last = N_0 . N_last (Q_U is orthonormal)
    double part = 0.0;
    for (int a = threadIdx.x; a < cn; a += blockDim.x) part = fma(Nn[a], Nn[(mk - 1) * ldnn + a], part);
    drift = fabs(block_sum(part, red));
    const double thr = fmin(P.tol_svd, 2.220446049250313e-16 * (double)P.n);
    STROM_TPROBE(P, 5);
    if (drift > thr) {
      did_qr = true;
      // linalg.qr(phi) (basis.py:174): Phi' = Q_U N' and Q_U is orthonormal, so
      // the positive-diagonal QR of Phi' is Q_U times that of N'.  CholeskyQR2 on
      // the shared-memory N' (two passes: orthonormal to working precision);
      // an ill-conditioned N' (the reference's non-unit j columns can make it so)
      // takes the Householder path.
      double* M = WB;   // cn x mk, ld cn  (N_b is dead)
      double* Bm = Wt;  // mk x mk Gram, then its Cholesky factor (N' has moved to M by then)
      bool chol_ok = true;
      for (int k = wid; k < mk; k += nw)
        for (int a = lane; a < cn; a += 32) M[k * cn + a] = Nn[k * ldnn + a];
      __syncthreads();
      for (int pass = 0; pass < 2 && chol_ok; ++pass) {
        STROM_TPROBE(P, 280 + 6 * pass);
        cta_gemm_dmma(mk, mk, cn, M, cn, 1, M, 1, cn, [&](int i, int k, double v) { Bm[k * mk + i] = v; });
        __syncthreads();
        STROM_TPROBE(P, 281 + 6 * pass);
        const double ratio = cta_cholesky(Bm, mk, mk, nullptr);
        STROM_TPROBE(P, 282 + 6 * pass);
        // CholeskyQR loses ~eps cond^2: only for well-conditioned N' (Householder
        // otherwise, like the reference); one pass suffices when cond <= 2
        if (!(ratio > 1e-2)) { chol_ok = false; break; }
        for (int k = threadIdx.x; k < mk; k += blockDim.x) Vt[k] = 1.0 / Bm[k * mk + k];
        __syncthreads();
        STROM_TPROBE(P, 283 + 6 * pass);
        cta_rows_times_inv_lt(M, cn, cn, Bm, mk, mk, Vt);  // M <- M R^{-1}
        __syncthreads();
        STROM_TPROBE(P, 284 + 6 * pass);
        STROM_TPROBE(P, 285 + 6 * pass);
        if (ratio > 0.5) break;
      }
      if (!chol_ok) {
        for (int k = wid; k < mk; k += nw)
          for (int a = lane; a < cn; a += 32) M[k * cn + a] = dst.N[(int64_t)k * dst.ldn + a];
        __syncthreads();
        cta_householder_qr(M, cn, cn, mk, nullptr, 0, pp.work, pp.work + P.work_stride, red);
      }
      if (P.tprobe && threadIdx.x == 0) P.tprobe[6 + 1] = chol_ok ? 1 : 2;
      for (int k = wid; k < mk; k += nw)
        for (int a = lane; a < cn; a += 32) dst.N[(int64_t)k * dst.ldn + a] = M[k * cn + a];
      __syncthreads();
    }
  }
  if (n_sm) {  // where the caller finds N' in shared memory (the QR result lives in M)
    *n_sm = did_qr ? WB : (ns_ok ? NS : nullptr);
    *n_sm_ld = cn;
  }
  STROM_TPROBE(P, 6);
  if (threadIdx.x == 0) {
    o.r = mk;
    o.c = cn;
    o.drift = drift;
    o.n_dependent += dep ? 1 : 0;
    o.n_truncated += trunc ? 1 : 0;
    o.flags = (dep ? F_DEPENDENT : 0) | (trunc ? F_TRUNCATED : 0) | (did_qr ? F_QR : 0) |
              (appended ? F_APPENDED : 0) | ((mode == M_NORMAL_INDEP && action == 2) ? F_FOLDED : 0);
    *dst.hdr = o;
    st->m = m;
    st->mkeep = mk;
    *pp.vrec[P.parity] = VRec{mode, m, mk, 0};
  }
}

// Window mode: the next snapshot's first-half decision (decide_a_body's normal
// branch, the same arithmetic in the same order, so identical bits) run by the
// core step right after it produced N' -- the next core step can then start
// without waiting for k_decide_a.  Not for restarts, rejects or errors (those
// stay with k_decide_a).  Returns false when it did not run.
__device__ inline bool decide_next_inline(const StateView& dst, const Pipe& pp, const IsvdParams& P, double* red,
                                          const double* n_sm, int n_sm_ld) {
  __syncthreads();
  const IsvdHdr h = *dst.hdr;
  const double xx = *(volatile const double*)&pp.ctl->xx;
  const bool at_cap = P.r_max >= 0 && h.r >= P.r_max;
  if (h.status != 0 || !isfinite(xx) || h.r == 0 || (at_cap && P.cap_mode == 0)) return false;
  const int np = P.parity ^ 1, c = h.c, r = h.r;
  double* ell = pp.ell[np];
  if (n_sm) cta_gemv_t_cm(n_sm, n_sm_ld, c, r, pp.tvec, ell, false);  // N' still in shared memory: same values
  else cta_gemv_t_cm(dst.N, dst.ldn, c, r, pp.tvec, ell, false);
  double s_ll = 0.0;
  for (int i = threadIdx.x; i < r; i += blockDim.x) s_ll = fma(ell[i], ell[i], s_ll);
  s_ll = block_sum(s_ll, red);
  const double p_sq = xx - s_ll;
  const double p = (p_sq > 0.0) ? sqrt(p_sq) : 0.0;
  const int dep = (p < P.tol_svd) || (p == 0.0) || ((int64_t)r >= P.n);
  __syncthreads();
  if (threadIdx.x == 0) {
    IsvdStep* st = pp.step[np];
    st->mode = dep ? M_NORMAL_DEP : M_NORMAL_INDEP;
    st->restart = 0;
    st->action = 0;
    st->dep = dep;
    st->c = c;
    st->cn = c;
    st->base_new = h.base;
    st->slot = h.base + c;
    st->xx = xx;
    st->rho2 = 0.0;
    st->p = p;
    st->p_sq = p_sq;
    st->norm = sqrt(xx);
    st->lam = 0.0;
    pp.ctl->resid = dep ? 0 : 1;
    pp.ctl->reorth = 0;
    pp.ctl->a_inline = P.d_expect + 1;
  }
  return true;
}

template <bool kSmem>
__global__ void __launch_bounds__(kSmallThreads) k_step_b(StateView src, StateView dst, Pipe pp, IsvdParams P) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  if (P.step_try) {
    if (P.wn > 0) wait_counter(&pp.ctl->adone, P.d_expect);
    else wait_counter(&pp.ctl->decided, P.d_expect);
    if (kSmem) {
      const int64_t mm = src.hdr->r + 1;
      if (3 * mm * mm + 16 * (int64_t)P.work_stride + (int64_t)P.ccap * mm > (int64_t)P.step_smem_doubles) {
        if (threadIdx.x == 0) pp.ctl->slow_step = (int32_t)P.k_new;
        return;  // the global-memory kernel behind this one takes the update
      }
    } else if (*(volatile const int32_t*)&pp.ctl->slow_step != (int32_t)P.k_new) {
      return;  // the shared-memory kernel did it
    }
  }
  if (P.wn > 0) {  // window mode: the SVD needs only k_decide_a; the rest waits mid-way
    wait_counter(&pp.ctl->adone, P.d_expect);
    trace_stamp(P.trace, 8);
    const double* n_sm = nullptr;
    int n_sm_ld = 0;
    step_b_body<kSmem>(src, dst, pp, P, smem, red, &pp.ctl->decided, P.d_expect, &n_sm, &n_sm_ld);
    if (P.inline_next && decide_next_inline(dst, pp, P, red, n_sm, n_sm_ld)) {
      signal_counter(&pp.ctl->adone);  // the next core step may start its SVD now
    }
  } else {
    wait_counter(&pp.ctl->decided, P.d_expect);  // this snapshot's decision chain
    trace_stamp(P.trace, 8);
    step_b_body<kSmem>(src, dst, pp, P, smem, red);
  }
  signal_counter(&pp.ctl->bdone);  // the next snapshot's decision may read this state
  trace_stamp(P.trace, 11);
}

// ---------------------------------------------------------------------------
// V' = [[V, 0], [0, 1]] V_bar[:, :mkeep]  (basis.py:147-158); restart/reject
// produce the fresh e_k column (basis.py:83-91).  Thread per row of V'.
// ---------------------------------------------------------------------------
constexpr int kVCols = 16;
constexpr int kVRows = 64;
__global__ void __launch_bounds__(kVRows) k_vupdate(StateView src, StateView dst, Pipe pp, IsvdParams P) {
  extern __shared__ double vbs[];  // (r+1) x kVCols slice of V_bar
  trace_stamp(P.trace, 12);
  const VRec* st = pp.vrec[P.parity];
  const int mode = st->mode;
  const int64_t k = P.k_new;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int col0 = blockIdx.y * kVCols;
  if (mode == M_ERROR || mode == M_REJECT) return;
  if (mode == M_RESTART_ACCEPT) {
    if (col0 == 0 && i < k) dst.V[i] = (i == k - 1) ? 1.0 : 0.0;
    return;
  }
  const int m = st->m, mk = st->mkeep, r = m - 1;
  if (col0 >= mk) return;
  const double* vb = pp.vbar;
  for (int idx = threadIdx.x; idx < m * kVCols; idx += blockDim.x) {
    const int b = idx % m, q = idx / m, col = col0 + q;
    vbs[q * m + b] = (col < mk) ? vb[(int64_t)col * m + b] : 0.0;
  }
  __syncthreads();
  if (i >= k) return;
  double acc[kVCols];
#pragma unroll
  for (int q = 0; q < kVCols; ++q) acc[q] = 0.0;
  if (i < k - 1) {
#pragma unroll 8
    for (int b = 0; b < r; ++b) {  // unrolled: eight V loads in flight (the kernel is load-latency bound)
      const double v = src.V[(int64_t)b * src.ldv + i];
#pragma unroll
      for (int q = 0; q < kVCols; ++q) acc[q] = fma(v, vbs[q * m + b], acc[q]);
    }
  } else {
#pragma unroll
    for (int q = 0; q < kVCols; ++q) acc[q] = vbs[q * m + r];
  }
#pragma unroll
  for (int q = 0; q < kVCols; ++q) {
    const int col = col0 + q;
    if (col < mk) dst.V[(int64_t)col * dst.ldv + i] = acc[q];
  }
}

// ---------------------------------------------------------------------------
// Compaction prep (one CTA): N = Q_c R_c (Householder);  T = L^{-T} Q_c, so
// U_new = U T has orthonormal columns in exact arithmetic and Phi = U_new R_c.
// The new store's L is then MEASURED (Gram of the stored U_new) and
// k_compact_finish sets N_new = L_new^T R_c.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads) k_compact_prep(StateView src, StateView dst, Pipe pp, IsvdParams P,
                                                                int use_smem) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  const IsvdHdr h = *src.hdr;
  const int r = h.r, c = h.c;
  IsvdHdr o = h;
  IsvdStep* st = pp.step[0];
  if (h.status != 0 || r == 0) {
    if (threadIdx.x == 0) {
      if (h.status == 0) { o.c = 0; o.base = 0; }
      *dst.hdr = o;
      st->m = 0;
      st->mkeep = 0;
    }
    return;
  }
  // shared plan (step B's footprint): Bm r^2 | Bi r^2 | spare m^2 | ... | M (c x r, ld c)
  const int m = r + 1;
  double* sbase = use_smem ? smem : pp.work + 4 * (int64_t)P.work_stride;
  double* Bm = sbase;
  double* Bi = Bm + (int64_t)m * m;
  double* M = sbase + 3 * (int64_t)m * m + 16 * (int64_t)P.work_stride;  // c x r
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = wid; k < r; k += nw)
    for (int i = lane; i < c; i += 32) M[k * c + i] = src.N[(int64_t)k * src.ldn + i];
  __syncthreads();
  // N = Q_c R_c by CholeskyQR2 (N has orthonormal columns up to the drift the
  // reference's QR trigger allows); Householder when its Gram is ill-conditioned
  bool chol_ok = true;
  for (int pass = 0; pass < 2 && chol_ok; ++pass) {
    cta_gemm_dmma(r, r, c, M, c, 1, M, 1, c, [&](int i, int k, double v) { Bm[k * r + i] = v; });
    __syncthreads();
    const double ratio = cta_cholesky(Bm, r, r, nullptr);
    if (!(ratio > 1e-2)) { chol_ok = false; break; }
    for (int k = threadIdx.x; k < r; k += blockDim.x) Bi[k] = 1.0 / Bm[k * r + k];
    __syncthreads();
    cta_rows_times_inv_lt(M, c, c, Bm, r, r, Bi);  // M <- M Bm^{-T}
    __syncthreads();
    if (ratio > 0.5) break;  // cond <= 2: one CholeskyQR pass is orthogonal to ~eps cond^2
  }
  if (chol_ok) {
    // R_c = Q_c^T N (upper triangular up to rounding; used in full)
    cta_gemm_dmma(r, r, c, M, c, 1, src.N, 1, src.ldn,
                  [&](int i, int k, double v) { dst.N[(int64_t)k * dst.ldn + i] = v; });
  } else {
    for (int k = wid; k < r; k += nw)
      for (int i = lane; i < c; i += 32) M[k * c + i] = src.N[(int64_t)k * src.ldn + i];
    __syncthreads();
    cta_householder_qr(M, c, c, r, dst.N, dst.ldn, pp.work, pp.work + P.work_stride, red);
  }
  __syncthreads();
  const double* Lib = src.Li + (int64_t)h.base * (src.ldl + 1);
  cta_gemm_dmma(c, r, c, Lib, src.ldl, 1, M, 1, c, [&](int a, int k, double v) { pp.T[(int64_t)k * P.ccap + a] = v; });
  for (int k = threadIdx.x; k < r; k += blockDim.x) dst.sigma[k] = src.sigma[k];
  if (threadIdx.x == 0) {
    o.c = r;
    o.base = 0;
    *dst.hdr = o;
    st->m = c;  // number of source columns for the GEMM
    st->mkeep = r;
  }
}

// After the compaction Gram: N_new = L_new^T R_c (R_c parked in dst.N; base 0;
// R_c is used in full -- CholeskyQR's R_c = Q_c^T N is triangular only up to rounding).
__global__ void __launch_bounds__(256) k_compact_finish(StateView dst, double* tmp, int ldt) {
  const int r = dst.hdr->r;
  if (dst.hdr->status != 0 || r == 0) return;
  for (int idx = threadIdx.x; idx < r * r; idx += blockDim.x) {
    const int i = idx % r, k = idx / r;
    const double* lcol = dst.L + (int64_t)i * dst.ldl;  // column i of L = row i of L^T
    double s = 0.0;
    for (int j = i; j < r; ++j) s = fma(lcol[j], dst.N[(int64_t)k * dst.ldn + j], s);
    tmp[(int64_t)k * ldt + i] = s;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < r * r; idx += blockDim.x) {
    const int i = idx % r, k = idx / r;
    dst.N[(int64_t)k * dst.ldn + i] = tmp[(int64_t)k * ldt + i];
  }
}

// U-coordinates W = L^{-T} N (c x r, ld c) for the export / materialisation.
__global__ void __launch_bounds__(256) k_n_to_w(StateView v, double* w) {
  const int r = v.hdr->r, c = v.hdr->c, base = v.hdr->base;
  const double* Lib = v.Li + (int64_t)base * (v.ldl + 1);
  for (int64_t idx = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; idx < (int64_t)c * r;
       idx += (int64_t)blockDim.x * gridDim.x) {
    const int a = (int)(idx % c), k = (int)(idx / c);
    const double* lcol = Lib + (int64_t)a * v.ldl;
    double s = 0.0;
    for (int i = a; i < c; ++i) s = fma(lcol[i], v.N[(int64_t)k * v.ldn + i], s);
    w[(int64_t)k * c + a] = s;
  }
}

// N = L^T W for a state loaded in U-coordinates (W parked in v.N; base 0).
__global__ void __launch_bounds__(256) k_w_to_n(StateView v, double* tmp) {
  const int r = v.hdr->r, c = v.hdr->c;
  for (int64_t idx = threadIdx.x; idx < (int64_t)c * r; idx += blockDim.x) {
    const int i = (int)(idx % c), k = (int)(idx / c);
    const double* lcol = v.L + (int64_t)i * v.ldl;
    double s = 0.0;
    for (int j = i; j < c; ++j) s = fma(lcol[j], v.N[(int64_t)k * v.ldn + j], s);
    tmp[(int64_t)k * c + i] = s;
  }
  __syncthreads();
  for (int64_t idx = threadIdx.x; idx < (int64_t)c * r; idx += blockDim.x) {
    const int i = (int)(idx % c), k = (int)(idx / c);
    v.N[(int64_t)k * v.ldn + i] = tmp[(int64_t)k * c + i];
  }
}

// ---------------------------------------------------------------------------
// Fused compaction pass on the fp64 tensor cores (DMMA m8n8k4): for every
// 64-row tile of the row-tiled store,
//     U_new tile = U tile (64 x c, columns base..) * T (c x r)      -> new store
//     G         += U_new tile^T U_new tile                          (registers)
// so the Gram of the STORED U_new is measured in the same sweep (one read of
// U, one write of U_new).  c, r are read on the device; r <= 32 * GB * 2 / ...
// Each warp owns 16 x 32 blocks (2 x 4 fragments): of C per tile, and GB
// persistent blocks of G.  Per-CTA Gram partials (QP x QP) go to `part`.
// ---------------------------------------------------------------------------
constexpr int kCompactThreads = 256;
// TR: rows of a store tile handled per step, 64 (the whole tile) or 32 (two half-tiles: the
// U and U_new staging buffers halve, so T (c x r), the U half-tile and the U_new half-tile
// fit shared memory up to r = 128, c ~ 140: 225 KB at cfg5's r = 100 instead of 294 KB).
template <int GB, int TR>
__global__ void __launch_bounds__(kCompactThreads, 1) k_compact_pass(const double* __restrict__ U, int64_t src_ccap,
                                                                     const int32_t* base_dev, const int32_t* c_dev,
                                                                     const int32_t* r_dev, const double* __restrict__ T,
                                                                     int64_t ldt, double* __restrict__ Unew,
                                                                     int64_t dst_ccap, int64_t ntiles,
                                                                     double* __restrict__ part, int QP,
                                                                     unsigned long long* prof) {
  constexpr int tr = TR;
  extern __shared__ __align__(16) double csm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int base = *base_dev, c = *c_dev, r = *r_dev;
  // algorithmic bytes: read c live columns, write r new ones (ntiles * kUTile rows)
  if (prof && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(prof + 6, 8ull * (unsigned long long)(ntiles * kUTile) * (unsigned long long)(c + r));
  const int c4 = (c + 3) & ~3;   // K padded to the DMMA k-step
  const int RP = (r + 31) & ~31;  // C / G columns padded to 32-wide blocks
  // leading dimensions = 4 (mod 16) doubles: the 16 lanes of a half-warp that
  // load one DMMA fragment (lane = 4 g + t, address t ld + g) hit 16 distinct banks
  const int LT = RP + 4, LA = tr + 4, LC = tr + 4;
  double* Ts = csm;                       // c4 x LT, T(k, j) at Ts[k * LT + j]
  double* At = Ts + (size_t)c4 * LT;      // c4 x LA, U(i, k) at At[k * LA + i]
  double* Cs = At + (size_t)c4 * LA;      // RP x LC, C(i, j) at Cs[j * LC + i]
  for (int idx = threadIdx.x; idx < c4 * RP; idx += blockDim.x) {
    const int k = idx / RP, j = idx % RP;
    Ts[k * LT + j] = (k < c && j < r) ? T[(int64_t)j * ldt + k] : 0.0;
  }
  for (int idx = threadIdx.x; idx < (c4 - c) * tr; idx += blockDim.x)
    At[(size_t)(c + idx / tr) * LA + idx % tr] = 0.0;
  const int nbc = (tr / 16) * (RP / 32);          // C blocks per step
  const int nbg = (RP / 16) * (RP / 32);          // G blocks
  const int nsub = kUTile / tr, h2 = tr / 2;
  double gacc[GB][2][4][2];
#pragma unroll
  for (int b = 0; b < GB; ++b)
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) gacc[b][x][y][0] = gacc[b][x][y][1] = 0.0;
  const int64_t per = ceil_div(ntiles, gridDim.x);
  const int64_t tt0 = blockIdx.x * per, tt1 = min(ntiles, tt0 + per);
  for (int64_t step = tt0 * nsub; step < tt1 * nsub; ++step) {
    const int64_t tile = step / nsub;
    const int sub = (int)(step - tile * nsub);
    __syncthreads();  // previous step's At / Cs fully consumed
    {
      const double* src = U + tile * kUTile * src_ccap + (int64_t)base * kUTile + sub * tr;
      for (int idx = threadIdx.x; idx < c * h2; idx += blockDim.x) {
        const int k = idx / h2, i2 = idx - k * h2;
        reinterpret_cast<double2*>(At + (size_t)k * LA)[i2] =
            __ldg(reinterpret_cast<const double2*>(src + (int64_t)k * kUTile) + i2);
      }
    }
    __syncthreads();
    // C(i, j) = sum_k U(i, k) T(k, j)
    for (int blk = wid; blk < nbc; blk += kCompactThreads / 32) {
      const int i0 = (blk % (tr / 16)) * 16, j0 = (blk / (tr / 16)) * 32;
      double acc[2][4][2];
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
      for (int k0 = 0; k0 < c4; k0 += 4) {
        const int k = k0 + t;
        double av[2], bv[4];
#pragma unroll
        for (int x = 0; x < 2; ++x) av[x] = At[k * LA + i0 + 8 * x + g];
#pragma unroll
        for (int y = 0; y < 4; ++y) bv[y] = Ts[k * LT + j0 + 8 * y + g];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) dmma884(acc[x][y][0], acc[x][y][1], av[x], bv[y]);
      }
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int i = i0 + 8 * x + g, j = j0 + 8 * y + 2 * t;
          Cs[(size_t)j * LC + i] = acc[x][y][0];
          Cs[(size_t)(j + 1) * LC + i] = acc[x][y][1];
        }
    }
    __syncthreads();
    {  // the r live column segments of the new tile are one contiguous run
      double* dst = Unew + tile * kUTile * dst_ccap + sub * tr;
      for (int idx = threadIdx.x; idx < r * h2; idx += blockDim.x) {
        const int j = idx / h2, i2 = idx - j * h2;
        reinterpret_cast<double2*>(dst + (int64_t)j * kUTile)[i2] =
            reinterpret_cast<const double2*>(Cs + (size_t)j * LC)[i2];
      }
    }
    // G += C^T C: G(a, b) = sum_i C(i, a) C(i, b)
#pragma unroll
    for (int bb = 0; bb < GB; ++bb) {
      const int blk = wid + bb * (kCompactThreads / 32);
      if (blk >= nbg) break;
      const int a0 = (blk % (RP / 16)) * 16, b0 = (blk / (RP / 16)) * 32;
      for (int k0 = 0; k0 < tr; k0 += 4) {
        const int k = k0 + t;
        double av[2], bv[4];
#pragma unroll
        for (int x = 0; x < 2; ++x) av[x] = Cs[(size_t)(a0 + 8 * x + g) * LC + k];
#pragma unroll
        for (int y = 0; y < 4; ++y) bv[y] = Cs[(size_t)(b0 + 8 * y + g) * LC + k];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) dmma884(gacc[bb][x][y][0], gacc[bb][x][y][1], av[x], bv[y]);
      }
    }
  }
  double* mp = part + (int64_t)blockIdx.x * QP * QP;
#pragma unroll
  for (int bb = 0; bb < GB; ++bb) {
    const int blk = wid + bb * (kCompactThreads / 32);
    if (blk >= nbg) break;
    const int a0 = (blk % (RP / 16)) * 16, b0 = (blk / (RP / 16)) * 32;
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int a = a0 + 8 * x + g, b = b0 + 8 * y + 2 * t;
        if (a < QP && b < QP) mp[a * QP + b] = gacc[bb][x][y][0];
        if (a < QP && b + 1 < QP) mp[a * QP + b + 1] = gacc[bb][x][y][1];
      }
  }
}

// ---------------------------------------------------------------------------
// Tall-skinny GEMM:  out(n x q) = A(n x p) * T(p x q)   (fp64 FMA, register
// blocked 4 rows x 8 cols per thread, T staged through shared memory).
// A and out are Tall views (column-major or row-tiled; first A column a_col0);
// out row-major (row stride out.cs) when out_row_major.  p, q read from device.
// ---------------------------------------------------------------------------
constexpr int kGemmRows = 128;  // rows per CTA tile
constexpr int kGemmKc = 32;     // T chunk (rows of T) per smem stage

__global__ void __launch_bounds__(256) k_tall_gemm(Tall A, const int32_t* a_col0_dev, int a_col0_add,
                                                   const double* __restrict__ T, int64_t ldt,
                                                   const int32_t* p_dev, const int32_t* q_dev,
                                                   int q_max, Tall out, int out_row_major, int64_t n,
                                                   int64_t nrows_pad) {
  extern __shared__ double ts[];  // kGemmKc x q_max
  const int p = *p_dev, q = *q_dev;
  const int col0 = (a_col0_dev ? *a_col0_dev : 0) + a_col0_add;
  if (q <= 0) return;
  const int tx = threadIdx.x & 31;   // row lane: rows tx, tx+32, tx+64, tx+96
  const int ty = threadIdx.x >> 5;   // column group: cols ty*8 .. ty*8+7 (+64 per pass)
  for (int64_t rt = blockIdx.x; rt * kGemmRows < nrows_pad; rt += gridDim.x) {
    const int64_t r0 = rt * kGemmRows;
    for (int cb = 0; cb < q; cb += 64) {
      double acc[4][8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
      for (int k0 = 0; k0 < p; k0 += kGemmKc) {
        const int kc = min(kGemmKc, p - k0);
        __syncthreads();
        for (int idx = threadIdx.x; idx < kGemmKc * 64; idx += blockDim.x) {
          const int kk = idx % kGemmKc, cc = idx / kGemmKc;
          const int col = cb + cc;
          ts[cc * kGemmKc + kk] = (kk < kc && col < q) ? T[(int64_t)col * ldt + k0 + kk] : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
          double av[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) av[a] = __ldg(A.p + A.off(r0 + tx + 32 * a, col0 + k0 + kk));
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            const double t = ts[(ty * 8 + b) * kGemmKc + kk];
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[a][b] = fma(av[a], t, acc[a][b]);
          }
        }
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int col = cb + ty * 8 + b;
        if (col >= q) continue;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int64_t row = r0 + tx + 32 * a;
          if (out_row_major) {
            if (row < n) out.p[row * out.cs + col] = acc[a][b];
          } else if (row < nrows_pad) {
            out.p[out.off(row, col)] = acc[a][b];
          }
        }
      }
    }
  }
}

}  // namespace strom
