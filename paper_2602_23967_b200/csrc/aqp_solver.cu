// aqp_solver.cu -- the device-resident PDHCG-II iteration (reference
// anchorqp/engine.py:207-245,395-428, inner.py:84-134, certify.py:63-164).
//
// One certification window (<= check_every outer iterations) is ONE CUDA
// graph launch:
//
//   WHILE(iterations left && !halted) {                       outer node
//     P1  : A'y SpMV, epilogue lin = c + A'y and x0 = clamp(x)
//           (diagonal Q: + closed-form prox, xbar, Halpern, |z-x|^2, window sum)
//     G0  : Q x0 SpMV, epilogue g0 + 4 reductions -> res0, phi0, alpha0   (BB only)
//     WHILE(bb continue) { S: x_t = clamp(x - alpha g);  G: Q x_t SpMV + gradient
//                          epilogue + 7 reductions -> BB1/BB2 step, best-phi,
//                          stop test on the device }                      (BB only)
//     X   : xbar = 2x+ - x, Halpern, |z-x|^2, window sum, tolerance update (BB only)
//     P2  : A xbar SpMV, epilogue dual step + Halpern(y) + window sum, slot rotation
//   }
//
// All scalars (alpha, best phi, tolerances, counters, slot indices) live in a
// device control block; the host only reads it at certification points.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "aqp_common.cuh"
#include "aqp_internal.h"
#include "aqp_kernels.cuh"

namespace aqp {

constexpr int kFinThreads = 1024;  // fold block: 4x the loads in flight of a 256-thread block

// ---------------------------------------------------------------- control block
enum RedSlot : int {
  // residual ingredients
  R_PV = 0, R_DV, R_QXI, R_ATYI, R_PRP, R_PRN, R_PRB, R_PYP, R_PYN, R_PYB, R_XQX, R_CX, R_PIDX, R_PIDY,
  // y-ray j (base + 9j): norm, viol, aty_inf, var pos/neg/bad, con pos/neg/bad
  R_YR = 16,
  // x-ray j (base + 5j): norm, improvement, viol_x, viol_s, qd_inf
  R_XR = 40,
  // power iteration
  R_PW = 56,
  R_COUNT = 64
};

struct Ctrl {
  aqp_scalars s;         // host-visible part (include/aqp.h)
  double tau, sigma;     // eta/omega, eta*omega (engine.py:148-154), set by the host
  int xcur, xprev, ycur, yprev;
  int bb_cur, bb_best, bb_new, g_cur, g_new, bb_t, bb_xplus, pad0;
  double alpha, alpha0, target, best_phi, best_res, phi, res, move;
  int64_t window_len;
  int pw_stop;
  int bb_cont;     // mirror of the BB WHILE condition (eager mode reads it)
  int pw_src, pad1;  // power iteration: v = xbb[pw_src] / pw_nrm (OpPwA)
  double pw_nrm;
  double red[R_COUNT];
};

struct SV {
  // problem (read-only)
  const double *c, *vlo, *vhi, *qd, *clo, *chi;
  const int8_t *cone_r, *recc_x, *cone_y, *recc_s;
  // iterate slots and companions
  double *xs[3], *ys[3];
  double *anc_x, *anc_y;   // anchor == round start (always equal in engine.py)
  double *xlast, *ylast, *xblk, *yblk, *xavgp, *yavgp;
  double *lin, *xbar, *xbb[3], *gbb[2];
  double *rx, *rtv;        // low-rank temporaries (k and n)
  const double *Rd;        // dense R (k x n row-major) when the problem holds R dense
  double *rxpart;          // dense R x: per-block partials [k][blocks]
  int rk;                  // rows of R
  double *xeval, *qx, *aty, *rs, *dx[2], *dy[2];
  double *tm;              // m-length temporary (power iteration)
  Ctrl *ctrl;
  // constants
  double eps_tol, gamma, tol_scale, tol_floor, diag_bound;
  int adaptive, max_inner, halpern, quad_kind;
  int64_t n, m;
  // row shards: vector pointers above are offset to this rank's slice
  // (x side by xoff, y side by yoff); gathers index the full copies
  int64_t xoff, yoff, nl, ml;
  int pair_ok;  // the BB step's slices are 16-byte aligned: paired (128-bit) step kernel
  Comm cm;
  cudaGraphConditionalHandle bb_cond, outer_cond;
  int in_graph;  // 0 for stand-alone launches (kernel timing): no conditional updates
};


// Gather of a vector the solve itself writes.  AQP_GATHER_NC=1 uses the
// non-coherent read-only path (ld.global.nc, measured 2% slower on C2); the
// default is a plain ld.global.
#ifndef AQP_GATHER_NC
#define AQP_GATHER_NC 0
#endif
__device__ __forceinline__ double gld(const double *p) {
#if AQP_GATHER_NC
  return __ldg(p);
#else
  return *p;
#endif
}

// slot selection without dynamic indexing (keeps the op out of local memory)
template <class T>
__host__ __device__ __forceinline__ T pick3(T const (&a)[3], int i) { return i == 0 ? a[0] : (i == 1 ? a[1] : a[2]); }
template <class T>
__host__ __device__ __forceinline__ T pick2(T const (&a)[2], int i) { return i == 0 ? a[0] : a[1]; }

__device__ __forceinline__ void halpern_coefs(const Ctrl *ct, double &a, double &b, double &c3) {
  // engine.py:239-244: a = (1+theta)*((k+1)/(k+2)), b = (1+theta)*(1/(k+2)), c = -theta
  const double k = (double)ct->s.k, th = ct->s.theta;
  a = (1.0 + th) * ((k + 1.0) / (k + 2.0));
  b = (1.0 + th) * (1.0 / (k + 2.0));
  c3 = -th;
}

// the x-side end of one outer iteration (engine.py:404-419): count, finiteness,
// adaptive tolerance.  Runs in thread 0 of the last block of P1(diag) / X.
__device__ __forceinline__ void x_iteration_end(const SV &v, double move2, int inner_iters) {
  Ctrl *ct = v.ctrl;
  const double move = sqrt(move2);
  ct->move = move;
  ct->s.iters_done += 1;
  ct->s.inner_sum += inner_iters;
  if (!isfinite(move)) {
    ct->s.halted = 1;
    return;
  }
  if (v.adaptive) {
    // inner.py:41-48  min(current, max(scale*omega*move/tau, floor))
    const double cand = py_max(v.tol_scale * ct->s.omega * move / ct->tau, v.tol_floor);
    ct->s.inner_tol = py_min(ct->s.inner_tol, cand);
  }
}

// z = Halpern/plain combination of one coordinate (engine.py:230-245, 400-403)
struct Combine {
  bool plain;
  double a, b, c3;
  bool use_prev;
  __device__ __forceinline__ void init(const SV &v) {
    const Ctrl *ct = v.ctrl;
    plain = ct->s.probing || !v.halpern;
    halpern_coefs(ct, a, b, c3);
    use_prev = ct->s.theta != 0.0;
  }
  // lincomb3 of _core.pyx:160-170: (a*w + b*anchor) + c*prev
  __device__ __forceinline__ double operator()(double w, const double *anc, const double *prev, int i) const {
    if (plain) return w;
    double z = a * w + b * anc[i];
    if (use_prev) z = z + c3 * prev[i];
    return z;
  }
  // the same on preloaded operands
  __device__ __forceinline__ double apply(double w, double anc, double prev) const {
    if (plain) return w;
    double z = a * w + b * anc;
    if (use_prev) z = z + c3 * prev;
    return z;
  }
};

// resident 256-thread blocks per SM the hot passes' register budgets target
// (A/B knobs, scripts/build_variants.sh)
#ifndef AQP_P1_BLOCKS
#define AQP_P1_BLOCKS 6
#endif
#ifndef AQP_GRAD_BLOCKS
#define AQP_GRAD_BLOCKS 6
#endif
#ifndef AQP_P2_BLOCKS
#define AQP_P2_BLOCKS 6
#endif
#ifndef AQP_X_BATCH  // grid-stride iterations whose loads the X pass issues together
#define AQP_X_BATCH 3
#endif

// ================================================================ iteration ops
// P1 (BB path): lin = c + A'y ; x0 = clamp(x)
struct OpP1Bb {
  static constexpr int NS = 0, NM = 0;
  static constexpr bool SYM = false, FINAL = false;
  static constexpr bool ROWIN_LATE = true;
  static constexpr int RING_CLASS = 2;  // AQP_RING_OFF bit 2 (aqp_kernels.cuh RingClassOf)
  static constexpr int UNIFORM_BLOCKS = AQP_P1_BLOCKS;
  SV v;
  const double *y;
  const double *x;
  // no halted test: a halted iteration closes the outer WHILE (OpP2), so no
  // later launch of the window runs; a load + branch here would serialise
  // every block's first memory access behind a round trip
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    y = pick3(v.ys, v.ctrl->ycur) - v.yoff;
    x = pick3(v.xs, v.ctrl->xcur);
  }
  __device__ double gather(int c) const { return gld(y + c); }
  struct RowIn {
    double c, x, lo, hi;
  };
  __device__ RowIn load_row(int r) const { return RowIn{v.c[r], x[r], v.vlo[r], v.vhi[r]}; }
  __device__ void row_in(int r, double s, const RowIn &in, RedVals<0, 0> &) const {
    v.lin[r] = in.c + s;                            // engine.py:214 cost + A'y
    const double x0 = clip(in.x, in.lo, in.hi);       // inner.py:94
    v.xbb[0][r] = x0;
    peer_put_halo(v.cm, 0, v.xbb[0], r, r + v.xoff, x0);                  // G0 gathers x0 on every rank
  }
  __device__ void row(int r, double s, RedVals<0, 0> &acc) const { row_in(r, s, load_row(r), acc); }
  __device__ void finalize(const RedVals<0, 0> &) const {}
};

// P1 (diagonal Q): the whole primal half of the step in one pass
// (engine.py:213-222 with inner.py:69-81, 230-245, 404-428)
struct OpP1Diag {
  static constexpr int NS = 1, NM = 0;
  static constexpr bool SYM = false, FINAL = true, SPLIT = true;
  SV v;
  const double *y, *x, *xprev;
  double *znew;
  double tau;
  Combine cb;
  // no halted test: a halted iteration closes the outer WHILE (OpP2), so no
  // later launch of the window runs; a load + branch here would serialise
  // every block's first memory access behind a round trip
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    y = pick3(v.ys, ct->ycur) - v.yoff;
    x = pick3(v.xs, ct->xcur);
    xprev = pick3(v.xs, ct->xprev);
    znew = pick3(v.xs, 3 - ct->xcur - ct->xprev);
    tau = ct->tau;
    cb.init(v);
  }
  __device__ double gather(int c) const { return gld(y + c); }
  __device__ void row(int r, double s, RedVals<1, 0> &acc) const {
    const double lin = v.c[r] + s;
    const double xk = x[r];
    const double xp = clip((xk - tau * lin) / (1.0 + tau * v.qd[r]), v.vlo[r], v.vhi[r]);  // _core.pyx:127
    const double xb = 2.0 * xp + (-1.0) * xk;                                               // axpby
    v.xbar[r] = xb;
    peer_put_halo(v.cm, 0, v.xbar, r, r + v.xoff, xb);
    const double z = cb(xp, v.anc_x, xprev, r);
    const double d = z - xk;
    acc.s[0] += d * d;
    v.xblk[r] += z;
    znew[r] = z;
  }
  __device__ void finalize(const RedVals<1, 0> &t) const { x_iteration_end(v, t.s[0], 0); }
};

// Q-operator row value: P/Q row sum plus the low-rank correction (linalg.py:251-254)
__device__ __forceinline__ double quad_row(const SV &v, int r, double s) {
  return v.quad_kind == AQP_QUAD_SPARSE_LOW_RANK ? s + v.rtv[r] : s;
}

// G: Q x_t SpMV with the gradient epilogue and the BB reductions (inner.py:61-66,105-124)
template <bool INIT>
struct OpGrad {
  static constexpr int NS = INIT ? 4 : 7, NM = 0;
  static constexpr bool SYM = true, FINAL = true, SPLIT = true;
  static constexpr bool ROWIN_LATE = true;   // see aqp_kernels.cuh RowInLateOf
  static constexpr int RING_CLASS = 1;       // AQP_RING_OFF bit 1 (aqp_kernels.cuh RingClassOf)
  static constexpr int UNIFORM_BLOCKS = AQP_GRAD_BLOCKS;
  SV v;
  const double *xt, *cen, *xo, *go;
  double *gt;
  double tau;
  int cond;  // second half of an unrolled BB body: run only while the loop continues
  // no halted test: a halted iteration closes the outer WHILE (OpP2), so no
  // later launch of the window runs; a load + branch here would serialise
  // every block's first memory access behind a round trip
  __device__ bool skip() const { return cond && !v.ctrl->bb_cont; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    xt = INIT ? pick3(v.xbb, 0) : pick3(v.xbb, ct->bb_new);
    gt = INIT ? pick2(v.gbb, 0) : pick2(v.gbb, ct->g_new);
    xo = pick3(v.xbb, ct->bb_cur);
    go = pick2(v.gbb, ct->g_cur);
    cen = pick3(v.xs, ct->xcur);
    tau = ct->tau;
  }
  __device__ double gather(int c) const { return gld(xt - v.xoff + c); }
  // epilogue operands of row r, loaded ahead of the SpMV tile (THREAD tiles)
  struct RowIn {
    double x, c, l, lo, hi, xo, go, rt;
  };
  __device__ RowIn load_row(int r) const {
    RowIn in;
    in.x = xt[r];
    in.c = cen[r];
    in.l = v.lin[r];
    in.lo = v.vlo[r];
    in.hi = v.vhi[r];
    in.xo = INIT ? 0.0 : xo[r];
    in.go = INIT ? 0.0 : go[r];
    in.rt = v.quad_kind == AQP_QUAD_SPARSE_LOW_RANK ? v.rtv[r] : 0.0;
    return in;
  }
  __device__ void row_in(int r, double s, const RowIn &in, RedVals<NS, 0> &acc) const {
    const double qx = v.quad_kind == AQP_QUAD_SPARSE_LOW_RANK ? s + in.rt : s;
    const double x = in.x, c = in.c, l = in.l;
    const double g = (qx + l) + (x - c) / tau;  // SubproblemSpec.gradient
    gt[r] = g;
    const double nr = x - clip(x - g, in.lo, in.hi);  // natural_res_sq
    acc.s[0] += nr * nr;
    acc.s[1] += x * g;
    acc.s[2] += l * x;
    acc.s[3] += (x - c) * c;
    if constexpr (!INIT) {
      const double sd = x - in.xo, vd = g - in.go;
      acc.s[4] += sd * vd;
      acc.s[5] += sd * sd;
      acc.s[6] += vd * vd;
    }
  }
  __device__ void row(int r, double s, RedVals<NS, 0> &acc) const { row_in(r, s, load_row(r), acc); }
  __device__ void finalize(const RedVals<NS, 0> &t) const {
    Ctrl *ct = v.ctrl;
    const double res = sqrt(t.s[0]);
    const double phi = 0.5 * ((t.s[1] + t.s[2]) - t.s[3] / tau);  // objective_from_gradient
    ct->res = res;
    ct->phi = phi;
    unsigned cont = 0;
    if (INIT) {
      // solve_bb prologue, inner.py:92-104
      ct->s.probing ? ct->target = py_min(ct->s.inner_tol, 1e-12) : ct->target = ct->s.inner_tol;
      ct->best_phi = phi;
      ct->best_res = res;
      ct->bb_cur = 0;
      ct->bb_best = 0;
      ct->g_cur = 0;
      ct->bb_t = 0;
      ct->bb_xplus = 0;
      if (res <= ct->target || v.max_inner <= 0) {
        cont = 0;
      } else {
        ct->alpha0 = tau / (1.0 + tau * v.diag_bound);
        ct->alpha = ct->alpha0;
        ct->bb_new = 1;
        ct->g_new = 1;
        cont = 1;
      }
    } else {
      // one BB iteration's bookkeeping, inner.py:110-124
      const int t_ = ++ct->bb_t;
      const int newslot = ct->bb_new;
      if (phi < ct->best_phi) {
        ct->best_phi = phi;
        ct->bb_best = newslot;
        ct->best_res = res;
      }
      const double sv = t.s[4];
      double alpha;
      if (sv > 0.0) {
        alpha = (t_ % 2 == 1) ? t.s[5] / sv : sv / t.s[6];
        alpha = py_min(py_max(alpha, 1e-10), 1e10);  // BB_STEP_MIN/MAX
      } else {
        alpha = ct->alpha0;
      }
      ct->alpha = alpha;
      ct->bb_cur = newslot;
      ct->g_cur = ct->g_new;
      const bool conv = res <= ct->target;
      if (conv || t_ >= v.max_inner) {
        // return rule, inner.py:129-134
        const double noise = 64.0 * 2.220446049250313e-16 * (1.0 + absd(ct->best_phi));
        if ((conv && phi <= ct->best_phi + noise) || phi <= ct->best_phi)
          ct->bb_xplus = ct->bb_cur;
        else
          ct->bb_xplus = ct->bb_best;
        cont = 0;
      } else {
        int nw = 0;
        while (nw == ct->bb_cur || nw == ct->bb_best) ++nw;
        ct->bb_new = nw;
        ct->g_new = 1 - ct->g_cur;
        cont = 1;
      }
    }
    ct->bb_cont = (int)cont;
    if (v.in_graph) cudaGraphSetConditional(v.bb_cond, cont);
  }
};

// S: x_t = clamp(x - alpha g)  (inner.py:106)
struct OpStep {
  static constexpr int NS = 0, NM = 0;
  static constexpr bool FINAL = false;
  SV v;
  const double *xo, *go;
  double *xn;
  double alpha;
  int cond;  // as OpGrad::cond
  // no halted test: a halted iteration closes the outer WHILE (OpP2), so no
  // later launch of the window runs; a load + branch here would serialise
  // every block's first memory access behind a round trip
  __device__ bool skip() const { return cond && !v.ctrl->bb_cont; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    xo = pick3(v.xbb, ct->bb_cur);
    go = pick2(v.gbb, ct->g_cur);
    xn = pick3(v.xbb, ct->bb_new);
    alpha = ct->alpha;
  }
  __device__ void elem(int64_t i, RedVals<0, 0> &) const {
    const double x = clip(xo[i] - alpha * go[i], v.vlo[i], v.vhi[i]);
    xn[i] = x;
    peer_put_halo(v.cm, 0, xn, i, i + v.xoff, x);  // the next G pass gathers x_t on every rank
  }
  // elements 2j, 2j+1 with 128-bit loads / store (no reduction, so the
  // result is the scalar op's); needs 16-byte aligned slices (even xoff)
  __device__ void elem2(int64_t j) const {
    const int64_t i = 2 * j;
    const double2 a = *reinterpret_cast<const double2 *>(xo + i), g = *reinterpret_cast<const double2 *>(go + i);
    const double2 lo = *reinterpret_cast<const double2 *>(v.vlo + i), hi = *reinterpret_cast<const double2 *>(v.vhi + i);
    double2 x;
    x.x = clip(a.x - alpha * g.x, lo.x, hi.x);
    x.y = clip(a.y - alpha * g.y, lo.y, hi.y);
    *reinterpret_cast<double2 *>(xn + i) = x;
    peer_put_halo(v.cm, 0, xn, i, i + v.xoff, x.x);
    peer_put_halo(v.cm, 0, xn, i + 1, i + 1 + v.xoff, x.y);
  }
  __device__ void finalize(const RedVals<0, 0> &) const {}
};

// the BB step over pairs (OpStep::elem2), scalar tail; grid = elem_grid(n / 2)
__global__ void __launch_bounds__(kThreads) k_step2(int64_t n, OpStep op, GridRed g) {
  pdl_wait();
  trace_mark(g, 1);
  if (op.skip()) return;
  OpStep o = op;
  o.prepare();
  const int64_t half = n >> 1, stride = (int64_t)gridDim.x * kThreads;
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < half; j += stride) o.elem2(j);
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    RedVals<0, 0> none;
    o.elem(n - 1, none);
  }
  pdl_trigger();
}

// X: primal epilogue after the BB solve (engine.py:222, 230-245, 404-428)
struct OpXPost {
  static constexpr int NS = 1, NM = 0;
  static constexpr bool FINAL = true, SPLIT = true;
  SV v;
  const double *xp, *x, *xprev;
  double *znew;
  Combine cb;
  // no halted test: a halted iteration closes the outer WHILE (OpP2), so no
  // later launch of the window runs; a load + branch here would serialise
  // every block's first memory access behind a round trip
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    xp = pick3(v.xbb, ct->bb_xplus);
    x = pick3(v.xs, ct->xcur);
    xprev = pick3(v.xs, ct->xprev);
    znew = pick3(v.xs, 3 - ct->xcur - ct->xprev);
    cb.init(v);
  }
  __device__ void elem(int64_t i, RedVals<1, 0> &acc) const { elem_in(i, load(i), acc); }
  // batched (elem_op BATCH): AQP_X_BATCH iterations' loads in flight per thread,
  // same elements in the same order per thread (C5 X 0.60 -> 0.43 ms; 3 beats 4 and 2
  // on C5-shaped and C2 passes, scripts/variants_ab.sh)
  static constexpr int BATCH = AQP_X_BATCH;
  struct In {
    double p, xk, anc, prev, blk;
  };
  __device__ In load(int64_t i) const {
    In r;
    r.p = xp[i];
    r.xk = x[i];
    r.anc = cb.plain ? 0.0 : v.anc_x[i];
    r.prev = (!cb.plain && cb.use_prev) ? xprev[i] : 0.0;
    r.blk = v.xblk[i];
    return r;
  }
  __device__ void elem_in(int64_t i, const In &in, RedVals<1, 0> &acc) const {
    const double xb = 2.0 * in.p + (-1.0) * in.xk;
    v.xbar[i] = xb;
    peer_put_halo(v.cm, 0, v.xbar, i, i + v.xoff, xb);
    const double z = cb.apply(in.p, in.anc, in.prev);
    const double d = z - in.xk;
    acc.s[0] += d * d;
    v.xblk[i] = in.blk + z;
    znew[i] = z;
  }
  __device__ void finalize(const RedVals<1, 0> &t) const { x_iteration_end(v, t.s[0], v.ctrl->bb_t); }
};

// P2: y+ = dual_step(y, A xbar), Halpern(y), window sum; then slot rotation and
// the outer-loop condition (engine.py:223-226, 420-428)
struct OpP2 {
  static constexpr int NS = 0, NM = 0;
  static constexpr bool SYM = false, FINAL = true, SPLIT = true;
  // measured (scripts/p2_ab.sh): late epilogue loads at 6 blocks/SM take the
  // C5 dual pass from 2.53 to 2.04 ms and cost C2 2 us (once per outer iteration)
  static constexpr bool ROWIN_LATE = true;
  static constexpr int UNIFORM_BLOCKS = AQP_P2_BLOCKS;
  SV v;
  const double *y, *yprev;
  double *ynew;
  double sigma;
  Combine cb;
  bool halted;
  __device__ bool skip() const { return false; }  // must reach finalize to close the loop
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    halted = ct->s.halted != 0;
    y = pick3(v.ys, ct->ycur);
    yprev = pick3(v.ys, ct->yprev);
    ynew = pick3(v.ys, 3 - ct->ycur - ct->yprev);
    sigma = ct->sigma;
    cb.init(v);
  }
  __device__ double gather(int c) const { return halted ? 0.0 : gld(v.xbar - v.xoff + c); }
  struct RowIn {
    double y, lo, hi, anc, blk, prev;
  };
  __device__ RowIn load_row(int r) const {
    RowIn in;
    in.y = y[r];
    in.lo = v.clo[r];
    in.hi = v.chi[r];
    in.anc = cb.plain ? 0.0 : v.anc_y[r];
    in.blk = v.yblk[r];
    in.prev = cb.use_prev ? yprev[r] : 0.0;
    return in;
  }
  __device__ void row_in(int r, double s, const RowIn &in, RedVals<0, 0> &) const {
    if (halted) return;
    const double w = in.y / sigma + s;                           // _core.pyx:155
    const double yp = sigma * (w - clip(w, in.lo, in.hi));       // _core.pyx:156
    double z = yp;                                               // engine.py:230-245
    if (!cb.plain) {
      z = cb.a * yp + cb.b * in.anc;
      if (cb.use_prev) z = z + cb.c3 * in.prev;
    }
    v.yblk[r] = in.blk + z;
    ynew[r] = z;
    peer_put_halo(v.cm, 1, ynew, r, r + v.yoff, z);  // the next P1 gathers y on every rank
  }
  __device__ void row(int r, double s, RedVals<0, 0> &acc) const { row_in(r, s, load_row(r), acc); }
  __device__ void finalize(const RedVals<0, 0> &) const {
    Ctrl *ct = v.ctrl;
    if (ct->s.halted) {
      if (v.in_graph) cudaGraphSetConditional(v.outer_cond, 0u);
      return;
    }
    const int xn = 3 - ct->xcur - ct->xprev, yn = 3 - ct->ycur - ct->yprev;
    ct->xprev = ct->xcur;
    ct->xcur = xn;
    ct->yprev = ct->ycur;
    ct->ycur = yn;
    if (!ct->s.probing) ct->s.k += 1;
    ct->s.block_len += 1;
    if (v.in_graph) cudaGraphSetConditional(v.outer_cond, ct->s.iters_done < ct->window_len ? 1u : 0u);
  }
};

// low-rank: rx = R x (k outputs) and rtv = R' rx (n outputs), linalg.py:251-254
struct OpRx {
  static constexpr int NS = 0, NM = 0;
  static constexpr bool SYM = false, FINAL = false;
  SV v;
  int src;  // 0: BB x0, 1: BB x_new, 2: x_eval, 3/4: x-ray candidate 0/1
  const double *x;
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    x = src == 0 ? pick3(v.xbb, 0) : src == 1 ? pick3(v.xbb, ct->bb_new) : src == 2 ? v.xeval : pick2(v.dx, src - 3);
    x -= v.xoff;
  }
  __device__ double gather(int c) const { return gld(x + c); }
  __device__ void row(int r, double s, RedVals<0, 0> &) const { v.rx[r] = s; }
  __device__ void finalize(const RedVals<0, 0> &) const {}
};

struct OpRtv {
  static constexpr int NS = 0, NM = 0;
  static constexpr bool SYM = false, FINAL = false;
  SV v;
  int src;
  __device__ bool skip() const { return false; }
  __device__ void prepare() {}
  __device__ double gather(int c) const { return gld(v.rx + c); }
  __device__ void row(int r, double s, RedVals<0, 0> &) const { v.rtv[r] = s; }
  __device__ void finalize(const RedVals<0, 0> &) const {}
};

// ---------------------------------------------------------------- dense low-rank factor
// Factor-model Q = P + R'R with R dense (k x n row-major, aqp_problem_desc.r_dense):
// R x is k streaming dot products over n (each block folds a column chunk of
// every row into per-block partials, a k-block kernel folds those in block
// order), R'(Rx) is a streaming pass whose entry i sums k products in row
// order -- bitwise the order of the reference's csr_matvec_t over R
// (_core.pyx:45-59).  Both read R once: 8 k n bytes per pass.
// R x, every warp on every row: a block owns kRxCols columns; warp w owns the
// column slice [w*S, (w+1)*S) (S = kRxCols / kWarps) of the chunk and walks
// all k rows over it (coalesced 128-bit loads of R, x from shared memory),
// folds each row with a fixed xor tree into smem[row][warp], and the block
// sums the kWarps slice values of a row in warp order.  Every warp does the
// same work for any k (no row imbalance), and 2048-column chunks keep 8
// blocks resident per SM (2.06 waves at C3 instead of 1.18).
constexpr int kRxCols = 2048;
constexpr int kRxMaxRows = 128;  // rows handled per pass over the chunk (smem [kRxMaxRows][kWarps])
inline int64_t dense_rx_blocks(int64_t n) { return std::max<int64_t>((n + kRxCols - 1) / kRxCols, 1); }
__device__ __forceinline__ bool cand_valid(const Ctrl *ct, int j, double norm);
__device__ __forceinline__ const double *lowrank_src(const SV &v, int src) {
  const Ctrl *ct = v.ctrl;
  return src == 0 ? pick3(v.xbb, 0) : src == 1 ? pick3(v.xbb, ct->bb_new) : src == 2 ? v.xeval : pick2(v.dx, src - 3);
}
// x-ray candidates only when the cheap test passed (certify.py:148-157)
__device__ __forceinline__ bool lowrank_skip(const SV &v, int src) {
  if (src < 3) return false;
  const Ctrl *ct = v.ctrl;
  const int j = src - 3;
  const double *xr = ct->red + R_XR + 5 * j;
  return !(cand_valid(ct, j, xr[0]) && xr[1] < -v.eps_tol);
}

__global__ void __launch_bounds__(kThreads) k_dense_rx(SV v, int src) {
  constexpr int S = kRxCols / kWarps;  // columns per warp slice (256)
  __shared__ __align__(16) double xs[kRxCols];
  __shared__ double red[kRxMaxRows][kWarps + 1];
  pdl_wait();
  if (lowrank_skip(v, src)) return;
  const double *x = lowrank_src(v, src);
  const int64_t n = v.nl;  // this rank's columns of R (all of them unsharded)
  const int64_t j0 = (int64_t)blockIdx.x * kRxCols;
  const int len = (int)min((int64_t)kRxCols, n - j0);
  for (int t = threadIdx.x; t < kRxCols; t += kThreads) xs[t] = t < len ? x[j0 + t] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = warp * S;                        // this warp's slice of the chunk
  const int clen = max(0, min(S, len - c0));
  const bool vec = (n & 1) == 0 && clen == S;     // full slice, 16-byte aligned rows
  for (int kb = 0; kb < v.rk; kb += kRxMaxRows) {
    const int kend = min(v.rk, kb + kRxMaxRows);
    for (int kk = kb; kk < kend; ++kk) {
      const double *row = v.Rd + (int64_t)kk * n + j0 + c0;
      double a0 = 0.0, a1 = 0.0;
      if (vec) {
        const double2 *r2 = reinterpret_cast<const double2 *>(row);
        const double2 *x2 = reinterpret_cast<const double2 *>(xs + c0);
#pragma unroll
        for (int u = 0; u < S / 64; ++u) {
          const double2 r = __ldcs(r2 + lane + 32 * u);  // streamed once per pass
          const double2 q = x2[lane + 32 * u];
          a0 += r.x * q.x;
          a1 += r.y * q.y;
        }
      } else {
        for (int u = lane; u < clen; u += 32) a0 += __ldcs(row + u) * xs[c0 + u];
      }
      double a = a0 + a1;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      if (lane == 0) red[kk - kb][warp] = a;
    }
    __syncthreads();
    for (int kk = kb + threadIdx.x; kk < kend; kk += kThreads) {
      double a = red[kk - kb][0];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) a += red[kk - kb][w];
      v.rxpart[(size_t)kk * gridDim.x + blockIdx.x] = a;
    }
    __syncthreads();
  }
  pdl_trigger();
}


// rx[k] = fold of the k-th row's block partials (block order, fixed tree)
__global__ void __launch_bounds__(kThreads) k_dense_rx_fold(SV v, int src, int nb) {
  __shared__ double sred[kWarps * kMaxRed];
  pdl_wait();
  pdl_trigger();
  if (lowrank_skip(v, src)) return;
  const int kk = blockIdx.x;
  RedVals<1, 0> a;
  a.zero();
  for (int b = threadIdx.x; b < nb; b += kThreads) a.s[0] += v.rxpart[(size_t)kk * nb + b];
  block_reduce<1, 0>(a, sred);
  if (threadIdx.x == 0) v.rx[kk] = a.s[0];
}

// Row shards: R x over this rank's columns is a partial sum; all-reduce the
// k values over the ranks (rank order, bitwise-identical on every rank)
// before R'(R x).  One block.
__global__ void __launch_bounds__(kThreads) k_rx_allreduce(SV v, int src) {
  __shared__ double buf[kMaxVec];
  pdl_wait();
  if (lowrank_skip(v, src)) {  // identical decision on every rank (all-reduced scalars)
    pdl_trigger();
    return;
  }
  for (int i = threadIdx.x; i < v.rk; i += blockDim.x) buf[i] = v.rx[i];
  __syncthreads();
  comm_allreduce_vec(buf, v.rk, v.cm);
  for (int i = threadIdx.x; i < v.rk; i += blockDim.x) v.rx[i] = buf[i];
  pdl_trigger();  // after the wait: see the scheduling rule in DESIGN.md §6
}

// rtv[i] = sum_k R[k, i] rx[k], k ascending
__global__ void __launch_bounds__(kThreads) k_dense_rtv(SV v, int src) {
  __shared__ double rxs[1024];
  pdl_wait();
  if (lowrank_skip(v, src)) return;
  const int k = v.rk;
  for (int t = threadIdx.x; t < k && t < 1024; t += kThreads) rxs[t] = v.rx[t];
  __syncthreads();
  const int64_t n = v.nl;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    double s = 0.0;
#pragma unroll 8
    for (int kk = 0; kk < k; ++kk) s += __ldcs(v.Rd + (int64_t)kk * n + i) * (kk < 1024 ? rxs[kk] : v.rx[kk]);
    v.rtv[i] = s;
  }
  pdl_trigger();
}

// ================================================================ certification ops
__device__ __forceinline__ bool cand_valid(const Ctrl *ct, int j, double norm) {
  return (j == 1 || ct->s.have_avg_prev) && norm != 0.0 && isfinite(norm);
}

// x side: x_eval, window average, candidate differences, PID norm (engine.py:436-453, 267)
struct OpChkX {
  static constexpr int NS = 1, NM = 2;
  static constexpr bool FINAL = true;
  SV v;
  int rays;
  const double *x;
  double inv_len;
  double len;
  int have_prev;
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    x = pick3(v.xs, ct->xcur);
    len = (double)ct->s.block_len;
    have_prev = ct->s.have_avg_prev;
  }
  __device__ void elem(int64_t i, RedVals<1, 2> &acc) const {
    const double xi = x[i];
    v.xeval[i] = clip(xi, v.vlo[i], v.vhi[i]);
    const double dr = xi - v.anc_x[i];
    acc.s[0] += dr * dr;
    if (rays) {
      const double avg = v.xblk[i] / len;
      if (have_prev) {
        const double d0 = avg - v.xavgp[i];
        pick2(v.dx, 0)[i] = d0;
        acc.m[0] = nanmax(acc.m[0], absd(d0));
      }
      v.xavgp[i] = avg;
      v.xblk[i] = 0.0;
      const double d1 = xi - v.xlast[i];
      pick2(v.dx, 1)[i] = d1;
      acc.m[1] = nanmax(acc.m[1], absd(d1));
    }
  }
  __device__ void finalize(const RedVals<1, 2> &t) const {
    double *red = v.ctrl->red;
    red[R_PIDX] = t.s[0];
    red[R_XR + 0] = t.m[0];
    red[R_XR + 5] = t.m[1];
  }
};

// y side: PID norm, p(proj_Y y), window average, projected candidates
struct OpChkY {
  static constexpr int NS = 4, NM = 2;
  static constexpr bool FINAL = true;
  SV v;
  int rays;
  const double *y;
  double len;
  int have_prev;
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    y = pick3(v.ys, ct->ycur);
    len = (double)ct->s.block_len;
    have_prev = ct->s.have_avg_prev;
  }
  __device__ void elem(int64_t i, RedVals<4, 2> &acc) const {
    const double yi = y[i];
    const int8_t cy = v.cone_y[i];
    const double dr = yi - v.anc_y[i];
    acc.s[0] += dr * dr;
    double bad = acc.s[3];
    support_add(cone_proj(yi, cy), v.clo[i], v.chi[i], acc.s[1], acc.s[2], bad);
    acc.s[3] = bad;
    if (rays) {
      const double avg = v.yblk[i] / len;
      if (have_prev) {
        const double p0 = cone_proj(avg - v.yavgp[i], cy);
        pick2(v.dy, 0)[i] = p0;
        acc.m[0] = nanmax(acc.m[0], absd(p0));
      }
      v.yavgp[i] = avg;
      v.yblk[i] = 0.0;
      const double p1 = cone_proj(yi - v.ylast[i], cy);
      pick2(v.dy, 1)[i] = p1;
      acc.m[1] = nanmax(acc.m[1], absd(p1));
    }
  }
  __device__ void finalize(const RedVals<4, 2> &t) const {
    double *red = v.ctrl->red;
    red[R_PIDY] = t.s[0];
    red[R_PYP] = t.s[1];
    red[R_PYN] = t.s[2];
    red[R_PYB] = t.s[3] > 0.0 ? 1.0 : 0.0;
    red[R_YR + 0] = t.m[0];
    red[R_YR + 9] = t.m[1];
  }
};

// A x_eval: primal violation; with rays also normalise the y candidates and
// take p(ray; l_c, u_c) (certify.py:66,75-77,120,131)
struct OpChkA {
  static constexpr int NS = 6, NM = 1;
  static constexpr bool SYM = false, FINAL = true;
  SV v;
  int rays;
  double nrm[2];
  bool ok[2];
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    for (int j = 0; j < 2; ++j) {
      nrm[j] = ct->red[R_YR + 9 * j];
      ok[j] = rays && cand_valid(ct, j, nrm[j]);
    }
  }
  __device__ double gather(int c) const { return gld(v.xeval - v.xoff + c); }
  __device__ void row(int r, double s, RedVals<6, 1> &acc) const {
    acc.m[0] = nanmax(acc.m[0], absd(s - clip(s, v.clo[r], v.chi[r])));
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (!ok[j]) continue;
      const double ray = pick2(v.dy, j)[r] / nrm[j];
      pick2(v.dy, j)[r] = ray;
      double bad = acc.s[3 * j + 2];
      support_add(ray, v.clo[r], v.chi[r], acc.s[3 * j], acc.s[3 * j + 1], bad);
      acc.s[3 * j + 2] = bad;
    }
  }
  __device__ void finalize(const RedVals<6, 1> &t) const {
    double *red = v.ctrl->red;
    red[R_PV] = t.m[0];
    for (int j = 0; j < 2; ++j) {
      red[R_YR + 9 * j + 6] = t.s[3 * j];
      red[R_YR + 9 * j + 7] = t.s[3 * j + 1];
      red[R_YR + 9 * j + 8] = t.s[3 * j + 2] > 0.0 ? 1.0 : 0.0;
    }
  }
};

// plain stores of an SpMV result: Q x_eval -> qx, A'y -> aty, A v -> tm, ...
struct OpStore {
  static constexpr int NS = 1, NM = 0;
  static constexpr bool SYM_ = false;
  static constexpr bool FINAL = true;
  SV v;
  int src;   // gather source: 0 x_eval, 1 y (current), 2 power-iteration v (xbb[1]), 3 tm
  int dst;   // 0 qx (adds low-rank part), 1 aty, 2 tm, 3 xbb[2]
  int red;   // reduction slot for sum of squares of the output (or -1)
  const double *x;
  double *out;
  __device__ bool skip() const { return src >= 2 && v.ctrl->pw_stop; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    x = src == 0 ? v.xeval - v.xoff : src == 1 ? pick3(v.ys, ct->ycur) - v.yoff
        : src == 2 ? pick3(v.xbb, 1) - v.xoff : v.tm - v.yoff;
    out = dst == 0 ? v.qx : dst == 1 ? v.aty : dst == 2 ? v.tm : pick3(v.xbb, 2);
  }
  __device__ double gather(int c) const { return gld(x + c); }
  __device__ void row(int r, double s, RedVals<1, 0> &acc) const {
    const double o = dst == 0 ? quad_row(v, r, s) : s;
    out[r] = o;
    acc.s[0] += o * o;
  }
  __device__ void finalize(const RedVals<1, 0> &t) const {
    if (red >= 0) v.ctrl->red[red] = t.s[0];
  }
};
template <bool S>
struct OpStoreT : OpStore {
  static constexpr bool SYM = S;
};

// dual residual, gap ingredients, dual slack; x-ray normalisation (certify.py:67-95,148-157)
struct OpChkR {
  static constexpr int NS = 7, NM = 5;
  static constexpr bool FINAL = true;
  SV v;
  int rays;
  double nrm[2];
  bool ok[2];
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    for (int j = 0; j < 2; ++j) {
      nrm[j] = ct->red[R_XR + 5 * j];
      ok[j] = rays && cand_valid(ct, j, nrm[j]);
    }
  }
  __device__ void elem(int64_t i, RedVals<7, 5> &acc) const {
    const double x = v.xeval[i];
    double q;
    if (v.quad_kind == AQP_QUAD_DIAGONAL) {
      q = v.qd[i] * x;
      v.qx[i] = q;
    } else {
      q = v.qx[i];
    }
    const double at = v.aty[i], c = v.c[i];
    const double r = (q + c) + at;
    v.rs[i] = r;
    const double rp = cone_proj(r, v.cone_r[i]);
    acc.m[0] = nanmax(acc.m[0], absd(r - rp));
    acc.m[1] = nanmax(acc.m[1], absd(q));
    acc.m[2] = nanmax(acc.m[2], absd(at));
    double bad = acc.s[2];
    support_add(-rp, v.vlo[i], v.vhi[i], acc.s[0], acc.s[1], bad);
    acc.s[2] = bad;
    acc.s[3] += x * q;
    acc.s[4] += c * x;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (!ok[j]) continue;
      const double d = pick2(v.dx, j)[i] / nrm[j];
      pick2(v.dx, j)[i] = d;
      acc.s[5 + j] += c * d;
      acc.m[3 + j] = nanmax(acc.m[3 + j], absd(d - cone_proj(d, v.recc_x[i])));
    }
  }
  __device__ void finalize(const RedVals<7, 5> &t) const {
    double *red = v.ctrl->red;
    red[R_PRP] = t.s[0];
    red[R_PRN] = t.s[1];
    red[R_PRB] = t.s[2] > 0.0 ? 1.0 : 0.0;
    red[R_XQX] = t.s[3];
    red[R_CX] = t.s[4];
    red[R_DV] = t.m[0];
    red[R_QXI] = t.m[1];
    red[R_ATYI] = t.m[2];
    for (int j = 0; j < 2; ++j) {
      red[R_XR + 5 * j + 1] = t.s[5 + j];
      red[R_XR + 5 * j + 2] = t.m[3 + j];
    }
  }
};

// y-ray test body: A' ray (certify.py:121-127)
struct OpChkYRay {
  static constexpr int NS = 3, NM = 2;
  static constexpr bool SYM = false, FINAL = true;
  SV v;
  int j;
  const double *ray;
  __device__ bool skip() const {
    const Ctrl *ct = v.ctrl;
    return !cand_valid(ct, j, ct->red[R_YR + 9 * j]);
  }
  __device__ void prepare() { ray = pick2(v.dy, j) - v.yoff; }
  __device__ double gather(int c) const { return gld(ray + c); }
  __device__ void row(int r, double s, RedVals<3, 2> &acc) const {
    const double p = cone_proj(s, v.cone_r[r]);
    acc.m[0] = nanmax(acc.m[0], absd(s - p));
    acc.m[1] = nanmax(acc.m[1], absd(s));
    double bad = acc.s[2];
    support_add(-p, v.vlo[r], v.vhi[r], acc.s[0], acc.s[1], bad);
    acc.s[2] = bad;
  }
  __device__ void finalize(const RedVals<3, 2> &t) const {
    double *red = v.ctrl->red + R_YR + 9 * j;
    red[1] = t.m[0];
    red[2] = t.m[1];
    red[3] = t.s[0];
    red[4] = t.s[1];
    red[5] = t.s[2] > 0.0 ? 1.0 : 0.0;
  }
};

// x-ray test body: A d and Q d (certify.py:158-160); skipped unless c'd < -eps_tol
struct OpChkXRay {
  static constexpr int NS = 0, NM = 1;
  static constexpr bool FINAL = true;
  SV v;
  int j;
  int which;  // 0: A d (recession of S), 1: Q d
  const double *d;
  __device__ bool skip() const {
    const Ctrl *ct = v.ctrl;
    const double *xr = ct->red + R_XR + 5 * j;
    return !(cand_valid(ct, j, xr[0]) && xr[1] < -v.eps_tol);
  }
  __device__ void prepare() { d = pick2(v.dx, j); }
  __device__ double gather(int c) const { return gld(d - v.xoff + c); }
  __device__ void row(int r, double s, RedVals<0, 1> &acc) const {
    if (which == 0) {
      acc.m[0] = nanmax(acc.m[0], absd(s - cone_proj(s, v.recc_s[r])));
    } else {
      acc.m[0] = nanmax(acc.m[0], absd(quad_row(v, r, s)));
    }
  }
  __device__ void elem(int64_t i, RedVals<0, 1> &acc) const {  // diagonal Q: |q_i d_i|
    acc.m[0] = nanmax(acc.m[0], absd(v.qd[i] * d[i]));
  }
  __device__ void finalize(const RedVals<0, 1> &t) const {
    v.ctrl->red[R_XR + 5 * j + 3 + which] = t.m[0];
  }
};
template <bool S>
struct OpChkXRayT : OpChkXRay {
  static constexpr bool SYM = S;
};

struct OpXRayRx : OpRx {
  int j;
  __device__ bool skip() const {
    const Ctrl *ct = v.ctrl;
    const double *xr = ct->red + R_XR + 5 * j;
    return !(cand_valid(ct, j, xr[0]) && xr[1] < -v.eps_tol);
  }
};
struct OpXRayRtv : OpRtv {
  int j;
  __device__ bool skip() const {
    const Ctrl *ct = v.ctrl;
    const double *xr = ct->red + R_XR + 5 * j;
    return !(cand_valid(ct, j, xr[0]) && xr[1] < -v.eps_tol);
  }
};

// ---------------------------------------------------------------- state transitions
struct OpState {
  static constexpr int NS = 0, NM = 0;
  static constexpr bool FINAL = false;
  SV v;
  int side;  // 0: n side, 1: m side
  int mode;  // 0 init, 1 mark cert, 2 restart/reanchor, 3 rollback
  double *cur, *prev, *anc, *last, *blk, *avgp, *spare;
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    if (side == 0) {
      cur = pick3(v.xs, ct->xcur); prev = pick3(v.xs, ct->xprev); spare = pick3(v.xs, 3 - ct->xcur - ct->xprev);
      anc = v.anc_x; last = v.xlast; blk = v.xblk; avgp = v.xavgp;
    } else {
      cur = pick3(v.ys, ct->ycur); prev = pick3(v.ys, ct->yprev); spare = pick3(v.ys, 3 - ct->ycur - ct->yprev);
      anc = v.anc_y; last = v.ylast; blk = v.yblk; avgp = v.yavgp;
    }
  }
  __device__ void elem(int64_t i, RedVals<0, 0> &) const {
    switch (mode) {
      case 0: {  // engine.py:174-204: x0 = clamp(0), y0 = 0
        const double z = side == 0 ? clip(0.0, v.vlo[i], v.vhi[i]) : 0.0;
        cur[i] = z; prev[i] = z; spare[i] = z; anc[i] = z; last[i] = z; blk[i] = 0.0; avgp[i] = 0.0;
        break;
      }
      case 1: last[i] = cur[i]; break;
      case 2: { const double z = cur[i]; anc[i] = z; prev[i] = z; break; }
      case 3: { const double z = anc[i]; cur[i] = z; prev[i] = z; break; }
      default: blk[i] = 0.0; break;
    }
  }
  __device__ void finalize(const RedVals<0, 0> &) const {}
};

// row shards: replicate this rank's slice of a gathered vector into every
// peer's copy (cold paths; the hot producers store to the peers directly)
struct OpPush {
  static constexpr int NS = 0, NM = 0;
  static constexpr bool FINAL = false;
  SV v;
  int which;  // PushBuf
  double *p;
  __device__ bool skip() const { return false; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    switch (which) {
      case 0: p = pick3(v.ys, ct->ycur); break;
      case 1: p = v.xeval; break;
      case 2: p = v.dy[0]; break;
      case 3: p = v.dy[1]; break;
      case 4: p = v.dx[0]; break;
      case 5: p = v.dx[1]; break;
      case 6: p = pick3(v.xbb, 1); break;
      case 8: p = pick3(v.xbb, 2); break;
      default: p = v.tm; break;
    }
  }
  int side;  // 0: x side, 1: y side
  __device__ void elem(int64_t i, RedVals<0, 0> &) const {
    peer_put_halo(v.cm, side, p, i, i + (side ? v.yoff : v.xoff), p[i]);
  }
  __device__ void finalize(const RedVals<0, 0> &) const {}
};
// gathered (windowed) buffers only: a push stores this rank's slice into the peers' windows
enum PushBuf : int { PB_Y = 0, PB_XEVAL, PB_DY0, PB_DY1, PB_DX0, PB_DX1, PB_PW, PB_TM, PB_PW2 };

// ---------------------------------------------------------------- scaled solves
// Certification of a scaled solve (aqp_problem_scale) on the ORIGINAL
// problem: copy the scaled solver's current iterate, anchor and window sums
// into an unscaled solver as x = D x~, y = E y~ (averages commute with the
// diagonal map), which then runs the reference's checks unchanged.
__global__ void __launch_bounds__(kThreads) k_import_scaled(SV dst, SV src, const double *__restrict__ D,
                                                            const double *__restrict__ E, int64_t n, int64_t m) {
  const Ctrl *sc = src.ctrl;
  const double *sx = pick3(src.xs, sc->xcur), *sy = pick3(src.ys, sc->ycur);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = D[i];
    dst.xs[0][i] = d * sx[i];
    dst.anc_x[i] = d * src.anc_x[i];
    dst.xblk[i] = d * src.xblk[i];
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double e = E[i];
    dst.ys[0][i] = e * sy[i];
    dst.anc_y[i] = e * src.anc_y[i];
    dst.yblk[i] = e * src.yblk[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctrl *dc = dst.ctrl;
    dc->xcur = 0; dc->xprev = 1; dc->ycur = 0; dc->yprev = 1;
    dc->s.block_len = sc->s.block_len;
  }
}

// ---------------------------------------------------------------- power iteration ops
struct OpPwNorm {  // sum of squares of xbb[idx] -> red[slot]
  static constexpr int NS = 1, NM = 0;
  static constexpr bool FINAL = true;
  SV v;
  int idx, slot;
  const double *x;
  __device__ bool skip() const { return v.ctrl->pw_stop != 0; }
  __device__ void prepare() { x = pick3(v.xbb, idx); }
  __device__ void elem(int64_t i, RedVals<1, 0> &acc) const { acc.s[0] += x[i] * x[i]; }
  __device__ void finalize(const RedVals<1, 0> &t) const { v.ctrl->red[slot] = t.s[0]; }
};

// The power iteration keeps v implicit: v = xbb[pw_src] / pw_nrm, divided at
// the gather of the A pass -- the reference's `v = w / nw` (linalg.py:302-308)
// is the same IEEE quotient, so no pass stores v.  w alternates between xbb[1]
// and xbb[2] (the start vector stays in xbb[0]), so a stopping iteration
// (`nw == 0`) leaves the last v intact for the final |A v|.
template <bool RED>
struct OpPwA {  // tm = A v  (|A v|^2 -> red[slot] when RED)
  static constexpr int NS = RED ? 1 : 0, NM = 0;
  static constexpr bool SYM = false, FINAL = RED;
  static constexpr int RING_CLASS = 4;  // AQP_RING_OFF bit 4
  SV v;
  int slot;
  const double *x;
  double nrm;
  __device__ bool skip() const { return v.ctrl->pw_stop != 0; }
  __device__ void prepare() {
    const Ctrl *ct = v.ctrl;
    x = pick3(v.xbb, ct->pw_src) - v.xoff;
    nrm = ct->pw_nrm;
  }
  __device__ double gather(int c) const { return gld(x + c) / nrm; }
  __device__ void row(int r, double s, RedVals<NS, 0> &acc) const {
    v.tm[r] = s;
    if constexpr (RED) acc.s[0] += s * s;
  }
  __device__ void finalize(const RedVals<NS, 0> &t) const {
    if constexpr (RED) v.ctrl->red[slot] = t.s[0];
  }
};

struct OpPwAt {  // w = A' tm -> xbb[dst], |w|^2; the fold sets the next v (or stops)
  static constexpr int NS = 1, NM = 0;
  static constexpr bool SYM = false, FINAL = true, SPLIT = true;
  static constexpr int RING_CLASS = 3;  // AQP_RING_OFF bit 3
  SV v;
  int dst;
  double *w;
  __device__ bool skip() const { return v.ctrl->pw_stop != 0; }
  __device__ void prepare() { w = pick3(v.xbb, dst); }
  __device__ double gather(int c) const { return gld(v.tm - v.yoff + c); }
  __device__ void row(int r, double s, RedVals<1, 0> &acc) const {
    w[r] = s;
    acc.s[0] += s * s;
  }
  __device__ void finalize(const RedVals<1, 0> &t) const {
    Ctrl *ct = v.ctrl;
    ct->red[R_PW + 2] = t.s[0];
    if (t.s[0] == 0.0) {
      ct->pw_stop = 1;  // linalg.py:307 `if nw == 0.0: break`
    } else {
      ct->pw_src = dst;
      ct->pw_nrm = sqrt(t.s[0]);  // np.linalg.norm(w)
    }
  }
};

__global__ void k_pw_start(Ctrl *ct, int slot) {  // v = xbb[0] / |xbb[0]|
  ct->pw_src = 0;
  ct->pw_nrm = sqrt(ct->red[slot]);
}

// Fold + finalize for the solver's SPLIT ops.  The finalize code (BB step
// rule, tolerance update, slot rotation) is a chain of dependent reads and
// writes of the control block; run on global memory that chain cost ~19 us
// per BB iteration (device trace).  Here the block stages the whole control
// block in shared memory with one coalesced copy (overlapping the fold),
// thread 0 finalizes against the staged copy, and the block writes it back.
template <class Op>
__global__ void __launch_bounds__(kFinThreads) fin_ctrl_op(Op op, GridRed g, unsigned nb) {
  constexpr int NS = Op::NS, NM = Op::NM;
  static_assert(sizeof(Ctrl) % 8 == 0, "Ctrl must be a whole number of words");
  constexpr int W = (int)(sizeof(Ctrl) / 8);
  __shared__ unsigned long long cbuf[W];
  __shared__ double sred[(kFinThreads / 32) * kMaxRed];
  pdl_wait();
  // row shards: this block waits on its peers, so its dependents must not be
  // made resident (and occupy SMs other ranks' kernels need) before that
  const bool shard = g.comm.nranks > 1;
  if (!shard) pdl_trigger();
  trace_mark(g, 2);
  if (op.skip()) {
    pdl_trigger();
    return;
  }
  Ctrl *gctrl = op.v.ctrl;
  const unsigned long long *src = reinterpret_cast<const unsigned long long *>(gctrl);
  for (int i = threadIdx.x; i < W; i += blockDim.x) cbuf[i] = __ldcg(src + i);
  RedVals<NS, NM> a;
  fold_partials<NS, NM>(a, g.partials, nb, sred);  // ends with __syncthreads
  comm_allreduce<NS, NM>(a, g.comm);               // all ranks: identical totals
  if (shard) pdl_trigger();
  trace_mark(g, 4);
  Op o = op;
  o.v.ctrl = reinterpret_cast<Ctrl *>(cbuf);
  o.prepare();
  if (threadIdx.x == 0) o.finalize(a);
  trace_mark(g, 5);
  __syncthreads();
  unsigned long long *dst = reinterpret_cast<unsigned long long *>(gctrl);
  for (int i = threadIdx.x; i < W; i += blockDim.x) dst[i] = cbuf[i];
  trace_mark(g, 3);
}


// The same fold + finalize on a cluster of 8 CTAs x 128 threads.  Measured
// on C2 the one-block fold spends ~4.2 us loading the 3907 x 7 partials
// (219 KB): one SM's share of L2 bandwidth.  Here CTA c is virtual threads
// [128 c, 128 c + 128) of that 1024-thread block -- same per-thread sums,
// whole virtual warps, same xor trees -- and the warp totals go to CTA 0
// through distributed shared memory, which adds them in warp order: bitwise
// the one-block fold, with 8 SMs pulling the partials.
// The cluster fold is a virtual VT-thread fold: virtual thread v sums
// partials v, v + VT, ... (batched 4 at a time), then the warp trees and the
// warp totals in virtual-warp order.  VT = 1024 (8 CTAs x 128) for up to
// kWideFoldMin partials, else 8192 (8 x 1024): C5's gradient pass leaves
// 195,313 partials per sum, which 1024 virtual threads summed in dependent
// chains of 190 (61 us per fold in the device trace; 8192: 19 us), while on
// C2 (3,906 partials) the wide fold is slower (9 -> 15 us).  For nb <= 1024
// both widths fold in the same order (the extra virtual warps add exact zeros).
constexpr int kFoldCtas = 8;
constexpr int kFoldVT = 1024;
constexpr int kFoldVTWide = 8192;
constexpr unsigned kWideFoldMin = 32768;

template <class Op, int VT>
__global__ void __cluster_dims__(kFoldCtas, 1, 1) __launch_bounds__(VT / kFoldCtas)
    fin_ctrl_cl(Op op, GridRed g, unsigned nb) {
  namespace cg = cooperative_groups;
  constexpr int NS = Op::NS, NM = Op::NM, NT = NS + NM;
  constexpr int W = (int)(sizeof(Ctrl) / 8);
  constexpr int kFoldThreads = VT / kFoldCtas;
  constexpr int NW = VT / 32;
  __shared__ unsigned long long cbuf[W];
  __shared__ double swarp[NW * (NT > 0 ? NT : 1)];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned crank = cl.block_rank();
  // DSMEM stores into CTA 0 need it to have started: arrive now, wait just
  // before the remote stores (the partials loads overlap the barrier)
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  pdl_wait();
  const bool shard = g.comm.nranks > 1;
  if (!shard) pdl_trigger();
  trace_mark(g, 2);
  if (op.skip()) {  // the same control block for every CTA: all skip or none
    pdl_trigger();
    return;
  }
  Ctrl *gctrl = op.v.ctrl;
  if (crank == 0) {
    const unsigned long long *src = reinterpret_cast<const unsigned long long *>(gctrl);
    for (int i = threadIdx.x; i < W; i += blockDim.x) cbuf[i] = __ldcg(src + i);
  }
  RedVals<NS, NM> a;
  a.zero();
  if constexpr (NT > 0) {
    constexpr int U = 4;
    const unsigned vt = crank * kFoldThreads + threadIdx.x;  // virtual thread of the VT-thread fold
    for (unsigned b0 = vt; b0 < nb; b0 += U * VT) {
      double t[U][NT];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned b = b0 + u * VT;
#pragma unroll
        for (int i = 0; i < NT; ++i) t[u][i] = b < nb ? g.partials[(size_t)i * nb + b] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int i = 0; i < NS; ++i) a.s[i] += t[u][i];
#pragma unroll
        for (int i = 0; i < NM; ++i) a.m[i] = nanmax(a.m[i], t[u][NS + i]);
      }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int i = 0; i < NS; ++i) a.s[i] += __shfl_xor_sync(0xffffffffu, a.s[i], off);
#pragma unroll
      for (int i = 0; i < NM; ++i) a.m[i] = nanmax(a.m[i], __shfl_xor_sync(0xffffffffu, a.m[i], off));
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (lane == 0) {
      double *dst = cl.map_shared_rank(swarp, 0);
      const int vw = (int)crank * (kFoldThreads / 32) + warp;
#pragma unroll
      for (int i = 0; i < NS; ++i) dst[vw * NT + i] = a.s[i];
#pragma unroll
      for (int i = 0; i < NM; ++i) dst[vw * NT + NS + i] = a.m[i];
    }
  } else {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  cl.sync();  // every CTA's warp totals are in CTA 0
  if (crank != 0) return;
  if constexpr (NT > 0) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int i = 0; i < NS; ++i) a.s[i] = swarp[i];
#pragma unroll
      for (int i = 0; i < NM; ++i) a.m[i] = swarp[NS + i];
      for (int w = 1; w < NW; ++w) {
#pragma unroll
        for (int i = 0; i < NS; ++i) a.s[i] += swarp[w * NT + i];
#pragma unroll
        for (int i = 0; i < NM; ++i) a.m[i] = nanmax(a.m[i], swarp[w * NT + NS + i]);
      }
    }
  }
  __syncthreads();
  comm_allreduce<NS, NM>(a, g.comm);
  if (shard) pdl_trigger();
  trace_mark(g, 4);
  Op o = op;
  o.v.ctrl = reinterpret_cast<Ctrl *>(cbuf);
  o.prepare();
  if (threadIdx.x == 0) o.finalize(a);
  trace_mark(g, 5);
  __syncthreads();
  unsigned long long *dstc = reinterpret_cast<unsigned long long *>(gctrl);
  for (int i = threadIdx.x; i < W; i += blockDim.x) dstc[i] = cbuf[i];
  trace_mark(g, 3);
}

#ifndef AQP_FOLD_CLUSTER
#define AQP_FOLD_CLUSTER 1
#endif

}  // namespace aqp

using namespace aqp;

// ====================================================================== solver object
struct aqp_solver {
  aqp_problem *p = nullptr;
  aqp_solver_params prm{};
  SV v{};
  Ctrl *d_ctrl = nullptr;
  Ctrl h{};  // host mirror (valid after sync points)
  GridRed gr{};
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t launches_per_iter_fixed = 0;
  int64_t kernel_launches = 0;
  bool eager = false;
  bool pdl = false;
  void *ws_base = nullptr;  // workspace (its front is the peer-visible exchange region)
  // pinned host staging: every host<->device copy of the solver is a true
  // async copy (pageable copies serialise on the driver's staging buffer,
  // which can stall one rank's launches behind another rank's pending read)
  struct Pinned {
    Ctrl pull;                    // control-block reads
    Ctrl ring[32];                // host -> device scalar pushes (reused after a sync)
    unsigned long long err;       // exchange error word
    int flag;                     // eager-mode flag reads
  } *pin = nullptr;               // the context's (aqp_ctx::pinned)
  double *bounce = nullptr;       // vector reads / start-vector upload (aqp_ctx::bounce)
  static constexpr size_t kBounce = 1 << 21;  // doubles (16 MB)
  bool shard = false;       // problem is row-sharded (nranks > 1): graph built at connect
};

namespace {

void layout_solver(Bump &b, aqp_problem *p, SV &v, Ctrl **ctrl, GridRed &gr) {
  // gathered vectors: one gather window each (the whole vector unsharded);
  // the others: this rank's rows.  Sizes are max-over-ranks capacities, so
  // every offset below is the same on every rank.
  const int64_t xw = std::max<int64_t>(p->xw_cap, 1), yw = std::max<int64_t>(p->yw_cap, 1);
  const int64_t n = std::max<int64_t>(p->nl_cap, 1), m = std::max<int64_t>(p->ml_cap, 1);
  auto vxw = [&]() { return (double *)b.take(xw * 8); };
  auto vyw = [&]() { return (double *)b.take(yw * 8); };
  auto vn = [&]() { return (double *)b.take(n * 8); };
  auto vm = [&]() { return (double *)b.take(m * 8); };
  for (int i = 0; i < 3; ++i) v.xs[i] = vn();
  for (int i = 0; i < 3; ++i) v.ys[i] = vyw();
  v.anc_x = vn(); v.anc_y = vm();
  v.xlast = vn(); v.ylast = vm();
  v.xblk = vn(); v.yblk = vm();
  v.xavgp = vn(); v.yavgp = vm();
  v.lin = vn(); v.xbar = vxw();
  for (int i = 0; i < 3; ++i) v.xbb[i] = vxw();
  for (int i = 0; i < 2; ++i) v.gbb[i] = vn();
  v.rx = (double *)b.take(std::max<int64_t>(p->R.rows, 1) * 8);
  v.rtv = vn();
  v.xeval = vxw(); v.qx = vn(); v.aty = vn(); v.rs = vn();
  v.dx[0] = vxw(); v.dx[1] = vxw();
  v.dy[0] = vyw(); v.dy[1] = vyw();
  v.tm = vyw();
  *ctrl = (Ctrl *)b.take(sizeof(Ctrl));
  // everything above (and the comm block) has the same offsets on every
  // rank: the peer-visible exchange region.  Partials below are sized by this
  // rank's plan.
  gr.comm.cb = (CommBlock *)b.take(sizeof(CommBlock));
  int64_t maxg = kElemGridMax;
  for (const DevCsr *M : {&p->A, &p->At, &p->Q, &p->R, &p->Rt}) maxg = std::max<int64_t>(maxg, M->nitems);
  gr.partials = (double *)b.take(maxg * kMaxRed * 8);
  gr.ticket = (unsigned *)b.take(64);  // [0] grid_end ticket
  if (p->r_dense) v.rxpart = (double *)b.take(std::max<int64_t>(p->R.rows, 1) * dense_rx_blocks(p->R.cols) * 8);
}

// explicit graph construction helpers
static bool g_use_pdl = true;
// a graph cursor: the last node added and whether it is a kernel node
// (cudaGraphNodeGetType fails on conditional nodes with this runtime)
struct GNode {
  cudaGraphNode_t n = nullptr;
  bool kernel = false;
};

template <class K, class... A>
cudaError_t add_node_cfg(cudaGraph_t g, GNode &last, unsigned grid, unsigned block, unsigned smem, K fn,
                         A... args) {
  void *params[] = {(void *)&args...};
  cudaKernelNodeParams kp = {};
  kp.func = (void *)fn;
  kp.gridDim = dim3(grid);
  kp.blockDim = dim3(block);
  kp.sharedMemBytes = smem;
  kp.kernelParams = params;
  kp.extra = nullptr;
  cudaGraphNode_t node;
  cudaError_t e;
  if (last.n && last.kernel && g_use_pdl) {
    // kernel -> kernel edge: programmatic (PDL)
    e = cudaGraphAddKernelNode(&node, g, nullptr, 0, &kp);
    if (e != cudaSuccess) return e;
    cudaGraphEdgeData ed = {};
    ed.from_port = cudaGraphKernelNodePortProgrammatic;
    ed.type = cudaGraphDependencyTypeProgrammatic;
    e = cudaGraphAddDependencies_v2(g, &last.n, &node, &ed, 1);
  } else {
    e = cudaGraphAddKernelNode(&node, g, last.n ? &last.n : nullptr, last.n ? 1 : 0, &kp);
  }
  if (e == cudaSuccess) {
    last.n = node;
    last.kernel = true;
  }
  return e;
}
template <class K, class... A>
cudaError_t add_node_smem(cudaGraph_t g, GNode &last, unsigned grid, unsigned smem, K fn, A... args) {
  return add_node_cfg(g, last, grid, (unsigned)kThreads, smem, fn, args...);
}
template <class K, class... A>
cudaError_t add_node(cudaGraph_t g, GNode &last, unsigned grid, K fn, A... args) {
  return add_node_smem(g, last, grid, 0u, fn, args...);
}

// banded ring path (spmv_ring_op): M.win is set when M's band fits the ring;
// AQP_RING_OFF (bit c: ops of RingClassOf c -- 1 gradient, 2 P1, 3 / 4 the
// power iteration's A'w / A v, 0 every other op) keeps op classes on the
// tile kernels -- default 0b110, the gradient and P1 (measured slower on the ring)
static int ring_off_mask() {
  const char *e = getenv("AQP_RING_OFF");  // read per graph build / eager launch (tests toggle it)
  return e ? atoi(e) : 0b110;
}
template <class Op>
bool use_ring(const DevCsr &M) {
  if constexpr (!kRingable<Op>) return false;
  return M.win && !((ring_off_mask() >> RingClassOf<Op>::value) & 1);
}
template <class Op, int RT>
cudaError_t ring_attr() {
  const int smem = ring_cols(RT) * 8;
  cudaError_t e = cudaFuncSetAttribute(spmv_ring_op<Op, false, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if constexpr (!Op::SYM)
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(spmv_ring_op<Op, true, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return e;
}
template <class Op, int RT>
cudaError_t node_ring_rt(cudaGraph_t g, GNode &last, const DevCsr &M, const Op &op, GridRed gr) {
  cudaError_t e = ring_attr<Op, RT>();
  if (e != cudaSuccess) return e;
  const unsigned smem = (unsigned)(ring_cols(RT) * 8);
  if constexpr (!Op::SYM)
    if (M.sell_perm)
      return add_node_cfg(g, last, (unsigned)M.win_grid, (unsigned)RT, smem, spmv_ring_op<Op, true, RT>, M, op, gr);
  return add_node_cfg(g, last, (unsigned)M.win_grid, (unsigned)RT, smem, spmv_ring_op<Op, false, RT>, M, op, gr);
}
template <class Op>
cudaError_t node_ring(cudaGraph_t g, GNode &last, const DevCsr &M, const Op &op, GridRed gr) {
  return M.win_rt == kRingRT2 ? node_ring_rt<Op, kRingRT2>(g, last, M, op, gr)
                              : node_ring_rt<Op, kRingRT>(g, last, M, op, gr);
}
template <class Op, int RT>
cudaError_t run_ring_rt(cudaStream_t st, const DevCsr &M, const Op &op, GridRed gr) {
  cudaError_t e = ring_attr<Op, RT>();
  if (e != cudaSuccess) return e;
  const int smem = ring_cols(RT) * 8;
  if constexpr (!Op::SYM)
    if (M.sell_perm) {
      spmv_ring_op<Op, true, RT><<<M.win_grid, RT, smem, st>>>(M, op, gr);
      return cudaGetLastError();
    }
  spmv_ring_op<Op, false, RT><<<M.win_grid, RT, smem, st>>>(M, op, gr);
  return cudaGetLastError();
}
template <class Op>
cudaError_t run_ring(cudaStream_t st, const DevCsr &M, const Op &op, GridRed gr) {
  return M.win_rt == kRingRT2 ? run_ring_rt<Op, kRingRT2>(st, M, op, gr) : run_ring_rt<Op, kRingRT>(st, M, op, gr);
}

template <class Op>
cudaError_t node_spmv(cudaGraph_t g, GNode &last, const DevCsr &M, const Op &op, GridRed gr) {
  if constexpr (kRingable<Op>)
    if (use_ring<Op>(M)) return node_ring(g, last, M, op, gr);
  if (M.sell_perm) return add_node_smem(g, last, (unsigned)M.nitems, 0u, spmv_sellp_op<Op>, M, op, gr);
  if (M.uniform) return add_node_smem(g, last, (unsigned)M.nitems, 0u, spmv_op<Op, true>, M, op, gr);
  return add_node_smem(g, last, (unsigned)M.nitems, (unsigned)M.smem_bytes, spmv_op<Op>, M, op, gr);
}
template <class Op>
cudaError_t node_elem(cudaGraph_t g, GNode &last, int64_t n, const Op &op, GridRed gr) {
  return add_node(g, last, (unsigned)elem_grid(n), elem_op<Op>, n, op, gr);
}

// the cluster fold of `nb` partials, its width chosen by nb (fin_ctrl_cl)
template <class Op>
cudaError_t node_fold(cudaGraph_t g, GNode &last, const Op &op, GridRed gr, unsigned nb) {
  if (nb >= kWideFoldMin)
    return add_node_cfg(g, last, (unsigned)kFoldCtas, (unsigned)(kFoldVTWide / kFoldCtas), 0u,
                        fin_ctrl_cl<Op, kFoldVTWide>, op, gr, nb);
  return add_node_cfg(g, last, (unsigned)kFoldCtas, (unsigned)(kFoldVT / kFoldCtas), 0u, fin_ctrl_cl<Op, kFoldVT>,
                      op, gr, nb);
}
template <class Op>
void run_fold(cudaStream_t st, const Op &op, GridRed gr, unsigned nb) {
  if (nb >= kWideFoldMin)
    fin_ctrl_cl<Op, kFoldVTWide><<<kFoldCtas, kFoldVTWide / kFoldCtas, 0, st>>>(op, gr, nb);
  else
    fin_ctrl_cl<Op, kFoldVT><<<kFoldCtas, kFoldVT / kFoldCtas, 0, st>>>(op, gr, nb);
}

// SPLIT ops: the main launch followed by its one-block fold/finalize
template <class Op>
cudaError_t node_spmv_fin(cudaGraph_t g, GNode &last, const DevCsr &M, const Op &op, GridRed gr) {
  cudaError_t e = use_ring<Op>(M) ? node_ring(g, last, M, op, gr)
                  : M.sell_perm ? add_node_smem(g, last, (unsigned)M.nitems, 0u, spmv_sellp_op<Op>, M, op, gr)
                   : M.uniform  ? add_node_smem(g, last, (unsigned)M.nitems, 0u, spmv_op<Op, true>, M, op, gr)
                                : add_node_smem(g, last, (unsigned)M.nitems, (unsigned)M.smem_bytes, spmv_op<Op>, M,
                                                op, gr);
  if (e != cudaSuccess) return e;
#if AQP_FOLD_CLUSTER
  return node_fold(g, last, op, gr, (unsigned)M.nitems);
#else
  return add_node_cfg(g, last, 1u, (unsigned)kFinThreads, 0u, fin_ctrl_op<Op>, op, gr, (unsigned)M.nitems);
#endif
}
template <class Op>
cudaError_t node_elem_fin(cudaGraph_t g, GNode &last, int64_t n, const Op &op, GridRed gr) {
  cudaError_t e = add_node(g, last, (unsigned)elem_grid(n), elem_op<Op>, n, op, gr);
  if (e != cudaSuccess) return e;
#if AQP_FOLD_CLUSTER
  return node_fold(g, last, op, gr, (unsigned)elem_grid(n));
#else
  return add_node_cfg(g, last, 1u, (unsigned)kFinThreads, 0u, fin_ctrl_op<Op>, op, gr, (unsigned)elem_grid(n));
#endif
}

// row shards: a one-block exchange after a producer whose output the next
// node gathers (the peers' stores must have landed)
cudaError_t node_barrier(cudaGraph_t g, GNode &last, GridRed gr) {
  return add_node_cfg(g, last, 1u, 32u, 0u, k_comm_barrier, gr);
}

template <class Op>
cudaError_t run_spmv(cudaStream_t st, const DevCsr &M, const Op &op, GridRed gr) {
  if constexpr (kRingable<Op>)
    if (use_ring<Op>(M)) return run_ring(st, M, op, gr);
  if (M.sell_perm)
    spmv_sellp_op<Op><<<M.nitems, kThreads, 0, st>>>(M, op, gr);
  else if (M.uniform)
    spmv_op<Op, true><<<M.nitems, kThreads, 0, st>>>(M, op, gr);
  else
    spmv_op<Op><<<M.nitems, kThreads, M.smem_bytes, st>>>(M, op, gr);
  return cudaGetLastError();
}
template <class Op>
cudaError_t run_elem(cudaStream_t st, int64_t n, const Op &op, GridRed gr) {
  elem_op<Op><<<elem_grid(n), kThreads, 0, st>>>(n, op, gr);
  return cudaGetLastError();
}
template <class Op>
cudaError_t run_spmv_fin(cudaStream_t st, const DevCsr &M, const Op &op, GridRed gr) {
  if (use_ring<Op>(M)) {
    cudaError_t e = run_ring(st, M, op, gr);
    if (e != cudaSuccess) return e;
  } else if (M.sell_perm)
    spmv_sellp_op<Op><<<M.nitems, kThreads, 0, st>>>(M, op, gr);
  else if (M.uniform)
    spmv_op<Op, true><<<M.nitems, kThreads, 0, st>>>(M, op, gr);
  else
    spmv_op<Op><<<M.nitems, kThreads, M.smem_bytes, st>>>(M, op, gr);
#if AQP_FOLD_CLUSTER
  run_fold(st, op, gr, (unsigned)M.nitems);
#else
  fin_ctrl_op<Op><<<1, kFinThreads, 0, st>>>(op, gr, (unsigned)M.nitems);
#endif
  return cudaGetLastError();
}
template <class Op>
cudaError_t run_elem_fin(cudaStream_t st, int64_t n, const Op &op, GridRed gr) {
  elem_op<Op><<<elem_grid(n), kThreads, 0, st>>>(n, op, gr);
#if AQP_FOLD_CLUSTER
  run_fold(st, op, gr, (unsigned)elem_grid(n));
#else
  fin_ctrl_op<Op><<<1, kFinThreads, 0, st>>>(op, gr, (unsigned)elem_grid(n));
#endif
  return cudaGetLastError();
}

// stream launch of the dense R x / R'(R x) passes (eager windows, checks)
// stream launch of Q's low-rank part R'(R x) for source `src` (lowrank_src);
// row shards all-reduce the partial R x between the two passes
int run_lowrank(aqp_solver *s, int src) {
  aqp_problem *p = s->p;
  cudaStream_t st = p->ctx->stream;
  SV v = s->v;
  v.in_graph = 0;
  if (p->r_dense) {
    const int nb = (int)dense_rx_blocks(p->R.cols);
    k_dense_rx<<<nb, kThreads, 0, st>>>(v, src);
    k_dense_rx_fold<<<p->R.rows, kThreads, 0, st>>>(v, src, nb);
  } else if (src >= 3) {
    OpXRayRx rx{}; rx.v = v; rx.src = src; rx.j = src - 3;
    AQP_CUDA(run_spmv(st, p->R, rx, s->gr));
  } else {
    OpRx rx{}; rx.v = v; rx.src = src;
    AQP_CUDA(run_spmv(st, p->R, rx, s->gr));
  }
  if (s->shard) k_rx_allreduce<<<1, kThreads, 0, st>>>(v, src);
  if (p->r_dense) {
    k_dense_rtv<<<elem_grid(p->R.cols), kThreads, 0, st>>>(v, src);
  } else if (src >= 3) {
    OpXRayRtv rt{}; rt.v = v; rt.src = src; rt.j = src - 3;
    AQP_CUDA(run_spmv(st, p->Rt, rt, s->gr));
  } else {
    OpRtv rt{}; rt.v = v; rt.src = src;
    AQP_CUDA(run_spmv(st, p->Rt, rt, s->gr));
  }
  AQP_CUDA(cudaGetLastError());
  return AQP_OK;
}

// grid of the paired BB step: no reduction, so any grid gives the same
// result; AQP_STEP_BLOCKS_PER_SM caps it (A/B knob: 64 vs the reductions' 8
// blocks per SM -- C5-shaped step 0.066 -> 0.062 ms, C2 unchanged)
#ifndef AQP_STEP_BLOCKS_PER_SM
#define AQP_STEP_BLOCKS_PER_SM 64
#endif
inline unsigned step_grid(int64_t n) {
  const int64_t pairs = std::max<int64_t>(n / 2, 1), b = (pairs + kThreads - 1) / kThreads;
  return (unsigned)std::min<int64_t>(b, 148 * AQP_STEP_BLOCKS_PER_SM);
}

// stream launch of the BB step (paired 128-bit kernel when the slice is aligned)
int run_step(cudaStream_t st, const SV &v, const OpStep &o, GridRed gr) {
  if (v.pair_ok)
    k_step2<<<step_grid(v.nl), kThreads, 0, st>>>(v.nl, o, gr);
  else
    elem_op<OpStep><<<elem_grid(v.nl), kThreads, 0, st>>>(v.nl, o, gr);
  AQP_CUDA(cudaGetLastError());
  return AQP_OK;
}

int add_lowrank(aqp_solver *s, cudaGraph_t g, GNode &last, int src) {
  aqp_problem *p = s->p;
  SV v = s->v;
  v.in_graph = 1;
  if (p->r_dense) {
    const int nb = (int)dense_rx_blocks(p->R.cols);
    AQP_CUDA(add_node(g, last, (unsigned)nb, k_dense_rx, v, src));
    AQP_CUDA(add_node(g, last, (unsigned)p->R.rows, k_dense_rx_fold, v, src, nb));
    if (s->shard) AQP_CUDA(add_node(g, last, 1u, k_rx_allreduce, v, src));
    AQP_CUDA(add_node(g, last, (unsigned)elem_grid(p->R.cols), k_dense_rtv, v, src));
    return AQP_OK;
  }
  OpRx rx{};
  rx.v = v;
  rx.src = src;
  OpRtv rt{};
  rt.v = v;
  rt.src = src;
  AQP_CUDA(node_spmv(g, last, p->R, rx, s->gr));
  if (s->shard) AQP_CUDA(add_node(g, last, 1u, k_rx_allreduce, v, src));
  AQP_CUDA(node_spmv(g, last, p->Rt, rt, s->gr));
  return AQP_OK;
}

// Build the window graph: WHILE(outer) { one outer iteration }
int build_graph(aqp_solver *s) {
  aqp_problem *p = s->p;
  cudaGraph_t g;
  AQP_CUDA(cudaGraphCreate(&g, 0));
  s->graph = g;
  cudaGraphConditionalHandle hout, hbb;
  AQP_CUDA(cudaGraphConditionalHandleCreate(&hout, g, 1u, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hout;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t outer;
  AQP_CUDA(cudaGraphAddNode(&outer, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  s->v.outer_cond = hout;
  const bool diag = p->quad_kind == AQP_QUAD_DIAGONAL;
  const bool lowrank = p->quad_kind == AQP_QUAD_SPARSE_LOW_RANK;
  if (!diag) {
    AQP_CUDA(cudaGraphConditionalHandleCreate(&hbb, body, 0u, cudaGraphCondAssignDefault));
    s->v.bb_cond = hbb;
  }
  SV v = s->v;
  v.in_graph = 1;
  GridRed gr = s->gr;
  GNode last;
  int64_t fixed = 0;
  if (diag) {
    OpP1Diag o{};
    o.v = v;
    AQP_CUDA(node_spmv_fin(body, last, p->At, o, gr));
    fixed += 2;
  } else {
    OpP1Bb o{};
    o.v = v;
    AQP_CUDA(node_spmv(body, last, p->At, o, gr));
    if (s->shard) {
      AQP_CUDA(node_barrier(body, last, gr));
      fixed += 1;
    }
    if (lowrank) AQP_TRY(add_lowrank(s, body, last, 0));
    OpGrad<true> g0{};
    g0.v = v;
    AQP_CUDA(node_spmv_fin(body, last, p->Q, g0, gr));
    fixed += 3 + (lowrank ? (p->r_dense ? 3 : 2) : 0);
    // inner WHILE
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hbb;
    ip.conditional.type = cudaGraphCondTypeWhile;
    ip.conditional.size = 1;
    cudaGraphNode_t inner;
    AQP_CUDA(cudaGraphAddNode(&inner, body, &last.n, 1, &ip));
    last.n = inner;
    last.kernel = false;
    cudaGraph_t ib = ip.conditional.phGraph_out[0];
    GNode il;
    // The body holds `unroll` BB iterations; copies after the first run only
    // while the loop continues (their kernels exit at once otherwise).  A
    // WHILE-node iteration boundary costs ~6.5 us (device trace: fold end ->
    // next step start) against ~1 us for a programmatic edge inside the body.
    // Measured (scripts/c2_unroll.py, c1_time.py): 4 vs 2 -- C2 solve 52.9 ->
    // 51.7 s, C1 0.137 -> 0.130 s, C5 window unchanged; 8 gains C2 little more.
    int unroll = 4;
    if (const char *e = getenv("AQP_BB_UNROLL")) unroll = std::max(1, atoi(e));
    if (lowrank) unroll = 1;  // the low-rank passes have no conditional exit
    for (int u = 0; u < unroll; ++u) {
      OpStep st{};
      st.v = v;
      st.cond = u > 0;
      if (v.pair_ok)  // 16-byte aligned slices: the paired (128-bit) step
        AQP_CUDA(add_node(ib, il, step_grid(v.nl), k_step2, v.nl, st, gr));
      else
        AQP_CUDA(node_elem(ib, il, v.nl, st, gr));
      if (s->shard) AQP_CUDA(node_barrier(ib, il, gr));
      if (lowrank) AQP_TRY(add_lowrank(s, ib, il, 1));
      OpGrad<false> gg{};
      gg.v = v;
      gg.cond = u > 0;
      AQP_CUDA(node_spmv_fin(ib, il, p->Q, gg, gr));
    }
    OpXPost xp{};
    xp.v = v;
    AQP_CUDA(node_elem_fin(body, last, v.nl, xp, gr));
    fixed += 2;
  }
  OpP2 p2{};
  p2.v = v;
  AQP_CUDA(node_spmv_fin(body, last, p->A, p2, gr));
  fixed += 2;
  s->launches_per_iter_fixed = fixed;
  AQP_CUDA(cudaGraphInstantiate(&s->exec, g, 0));
  return AQP_OK;
}

int build_graph_any(aqp_solver *s) {
  const char *env = getenv("AQP_NO_PDL");
  g_use_pdl = !(env && env[0] == '1');
  int rc = build_graph(s);
  if (rc != AQP_OK && g_use_pdl) {
    // programmatic edges rejected (e.g. inside conditional bodies): plain edges
    const std::string first = aqp_last_error();
    if (s->graph) cudaGraphDestroy(s->graph);
    s->graph = nullptr;
    cudaGetLastError();
    g_use_pdl = false;
    rc = build_graph(s);
    if (rc != AQP_OK) set_error(first + " | without PDL: " + aqp_last_error());
  }
  s->pdl = g_use_pdl;
  return rc;
}

// Push only the host-owned prefix of the control block (aqp_scalars + tau,
// sigma); device-owned fields (slots, BB state, reductions) are never
// overwritten from a possibly stale host mirror.
int push_scalars(aqp_solver *s) {
  s->h.tau = s->h.s.eta / s->h.s.omega;    // engine.py:148-150
  s->h.sigma = s->h.s.eta * s->h.s.omega;  // engine.py:152-154
  Ctrl *slot = &s->pin->ring[s->p->ctx->ring_i++ % 32];
  std::memcpy(slot, &s->h, offsetof(Ctrl, xcur));
  AQP_CUDA(cudaMemcpyAsync(s->d_ctrl, slot, offsetof(Ctrl, xcur), cudaMemcpyHostToDevice, s->p->ctx->stream));
  return AQP_OK;
}

template <class T>
int poke(aqp_solver *s, T Ctrl::*field, T value) {
  s->h.*field = value;
  Ctrl *slot = &s->pin->ring[s->p->ctx->ring_i++ % 32];
  slot->*field = value;
  AQP_CUDA(cudaMemcpyAsync(&(s->d_ctrl->*field), &(slot->*field), sizeof(T), cudaMemcpyHostToDevice,
                           s->p->ctx->stream));
  return AQP_OK;
}

// full push (only at init, when the host mirror is authoritative)
int push_all(aqp_solver *s) {
  s->h.tau = s->h.s.eta / s->h.s.omega;
  s->h.sigma = s->h.s.eta * s->h.s.omega;
  Ctrl *slot = &s->pin->ring[s->p->ctx->ring_i++ % 32];
  *slot = s->h;
  AQP_CUDA(cudaMemcpyAsync(s->d_ctrl, slot, sizeof(Ctrl), cudaMemcpyHostToDevice, s->p->ctx->stream));
  AQP_CUDA(cudaStreamSynchronize(s->p->ctx->stream));
  return AQP_OK;
}

int pull_ctrl(aqp_solver *s) {
  cudaStream_t st = s->p->ctx->stream;
  AQP_CUDA(cudaMemcpyAsync(&s->pin->pull, s->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  s->pin->err = 0;
  if (s->shard) AQP_CUDA(cudaMemcpyAsync(&s->pin->err, &s->gr.comm.cb->err, 8, cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  s->h = s->pin->pull;
  const unsigned long long err = s->pin->err;
  if (err)
    return fail(AQP_ECUDA, "row-shard exchange " + std::to_string(err) + " timed out on rank " +
                               std::to_string(s->p->rank) + " (a peer stopped arriving)");
  return AQP_OK;
}

// row shards: replicate this rank's slice of buffer `which` (PushBuf) into
// the peers' copies and wait until every rank has done the same
int push_buf(aqp_solver *s, int which) {
  if (!s->shard) return AQP_OK;
  cudaStream_t st = s->p->ctx->stream;
  const bool yside = which == PB_Y || which == PB_DY0 || which == PB_DY1 || which == PB_TM;
  OpPush o{};
  o.v = s->v;
  o.which = which;
  o.side = yside ? 1 : 0;
  AQP_CUDA(run_elem(st, yside ? s->v.ml : s->v.nl, o, s->gr));
  k_comm_barrier<<<1, 32, 0, st>>>(s->gr);
  AQP_CUDA(cudaGetLastError());
  return AQP_OK;
}

int state_op(aqp_solver *s, int mode) {
  cudaStream_t st = s->p->ctx->stream;
  for (int side = 0; side < 2; ++side) {
    OpState o{};
    o.v = s->v;
    o.side = side;
    o.mode = mode;
    AQP_CUDA(run_elem(st, side == 0 ? s->v.nl : s->v.ml, o, s->gr));
  }
  // init / rollback rewrite the current y, which the next P1 gathers
  if (mode == 0 || mode == 3) AQP_TRY(push_buf(s, PB_Y));
  return AQP_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

static int run_eager(aqp_solver *s, int64_t n_iters);

int aqp_solver_sizes(const aqp_problem *p, size_t *workspace_bytes) {
  if (!p || !workspace_bytes) return fail(AQP_EINVAL, "NULL argument");
  // the workspace is sized by the plans: a deferred A' plan is made now (the
  // lazily computed part of the problem's state)
  AQP_TRY(plan_deferred_at(const_cast<aqp_problem *>(p)));
  Bump b;
  SV v{};
  Ctrl *c = nullptr;
  GridRed gr{};
  layout_solver(b, const_cast<aqp_problem *>(p), v, &c, gr);
  *workspace_bytes = b.used + 256;
  return AQP_OK;
}

int aqp_solver_create(aqp_problem *p, const aqp_solver_params *prm, void *ws, size_t ws_bytes, aqp_solver **out) {
  if (!p || !prm || !ws || !out) return fail(AQP_EINVAL, "NULL argument");
  AQP_TRY(plan_deferred_at(p));  // A' without its SELL-P copy attached: the CSR plan now
  aqp_solver *s = new aqp_solver();
  s->p = p;
  s->prm = *prm;
  Bump b;
  b.base = ws;
  b.cap = ws_bytes;
  layout_solver(b, p, s->v, &s->d_ctrl, s->gr);
  if (b.overflow) {
    delete s;
    return fail(AQP_ENOMEM, "solver workspace too small");
  }
  SV &v = s->v;
  v.c = p->c; v.vlo = p->vlo; v.vhi = p->vhi; v.qd = p->qd; v.clo = p->clo; v.chi = p->chi;
  v.cone_r = p->cone_r; v.recc_x = p->recc_x; v.cone_y = p->cone_y; v.recc_s = p->recc_s;
  v.ctrl = s->d_ctrl;
  v.eps_tol = prm->eps_tol;
  v.gamma = prm->gamma_sys;
  v.tol_scale = prm->tol_scale;
  v.tol_floor = prm->tol_floor;
  v.diag_bound = prm->diag_bound;
  v.adaptive = prm->adaptive;
  v.max_inner = prm->max_inner;
  v.halpern = prm->halpern;
  v.quad_kind = p->quad_kind;
  v.Rd = p->r_dense ? p->R.val : nullptr;
  v.rk = p->R.rows;
  v.n = p->n;
  v.m = p->m;
  // row shards (aqp_shard_desc): vectors of this rank's rows start at its
  // row 0; gathered vectors (windows starting at global xw0 / yw0) point at
  // the rank's own slice inside the window, so `ptr - xoff + global column`
  // addresses the window and every local row r is `ptr[r]`
  v.xoff = p->n0;
  v.yoff = p->m0;
  v.nl = p->n1 - p->n0;
  v.ml = p->m1 - p->m0;
  s->ws_base = ws;
  s->shard = p->nranks > 1;
  {
    std::lock_guard<std::recursive_mutex> lk(p->ctx->mu);
    if (!p->ctx->pinned) {
      AQP_CUDA(cudaMallocHost(&p->ctx->pinned, sizeof(aqp_solver::Pinned)));
      AQP_CUDA(cudaMallocHost(&p->ctx->bounce, aqp_solver::kBounce * 8));
    }
  }
  s->pin = static_cast<aqp_solver::Pinned *>(p->ctx->pinned);
  s->bounce = static_cast<double *>(p->ctx->bounce);
  {
    const int64_t gx = p->n0 - p->xw0(), gy = p->m0 - p->yw0();
    for (int i = 0; i < 3; ++i) { v.ys[i] += gy; v.xbb[i] += gx; }
    for (int i = 0; i < 2; ++i) { v.dx[i] += gx; v.dy[i] += gy; }
    v.xbar += gx;
    v.xeval += gx;
    v.tm += gy;
    v.pair_ok = (gx & 1) == 0;  // x_t / x slots sit gx entries into 256-byte aligned windows
  }
  s->gr.comm.rank = p->rank;
  s->gr.comm.nranks = 1;  // until aqp_solver_connect
  for (int k = 0; k < kMaxRanks; ++k) {  // default halos: the gather windows
    s->gr.comm.xlo[k] = p->xwin[2 * k];
    s->gr.comm.xhi[k] = p->xwin[2 * k + 1];
    s->gr.comm.ylo[k] = p->ywin[2 * k];
    s->gr.comm.yhi[k] = p->ywin[2 * k + 1];
  }
  v.cm = s->gr.comm;
  std::memset(&s->h, 0, sizeof(Ctrl));
  s->h.xcur = 0; s->h.xprev = 1; s->h.ycur = 0; s->h.yprev = 1;
  const char *eager = getenv("AQP_EAGER");
  s->eager = eager && eager[0] == '1';
  const char *trace = getenv("AQP_TRACE");
  if (trace && trace[0] == '1') {
    // debug facility: a device ring of (tag, ns) stamps, outside the workspace
    s->gr.trace_cap = 1u << 20;
    AQP_CUDA(cudaMalloc(&s->gr.trace, sizeof(unsigned long long) * 2 * s->gr.trace_cap));
    AQP_CUDA(cudaMalloc(&s->gr.trace_n, sizeof(unsigned)));
    AQP_CUDA(cudaMemset(s->gr.trace_n, 0, sizeof(unsigned)));
  }
  cudaStream_t st = p->ctx->stream;
  AQP_CUDA(cudaMemsetAsync(s->gr.ticket, 0, 64, st));
  AQP_CUDA(cudaMemsetAsync(s->gr.comm.cb, 0, sizeof(CommBlock), st));
  // the mailbox must be zero before any peer can write to it (the caller
  // holds a host barrier between every rank's create and the first exchange)
  AQP_CUDA(cudaStreamSynchronize(st));
  if (!s->shard) {  // sharded solvers build their graph once the peers are connected
    int rc = build_graph_any(s);
    if (rc) {
      aqp_solver_destroy(s);
      return rc;
    }
  }
  *out = s;
  return AQP_OK;
}

int aqp_solver_import_scaled(aqp_solver *dst, aqp_solver *src, const double *D, const double *E) {
  if (!dst || !src || !D || !E) return fail(AQP_EINVAL, "NULL argument");
  if (dst->p->n != src->p->n || dst->p->m != src->p->m || dst->shard || src->shard)
    return fail(AQP_EINVAL, "import needs two unsharded solvers of the same shape");
  std::lock_guard<std::recursive_mutex> ctx_lock_(dst->p->ctx->mu);
  cudaStream_t st = dst->p->ctx->stream;
  if (src->p->ctx->stream != st) AQP_CUDA(cudaStreamSynchronize(src->p->ctx->stream));
  const int64_t big = std::max(dst->p->n, dst->p->m);
  k_import_scaled<<<elem_grid(big), kThreads, 0, st>>>(dst->v, src->v, D, E, dst->p->n, dst->p->m);
  AQP_CUDA(cudaGetLastError());
  dst->h.xcur = 0; dst->h.xprev = 1; dst->h.ycur = 0; dst->h.yprev = 1;
  return AQP_OK;
}

int aqp_solver_exchange_region(aqp_solver *s, void **base, size_t *bytes) {
  if (!s || !base || !bytes) return fail(AQP_EINVAL, "NULL argument");
  *base = s->ws_base;
  *bytes = (size_t)((char *)s->gr.comm.cb - (char *)s->ws_base) + sizeof(CommBlock);
  return AQP_OK;
}

int aqp_solver_set_halos(aqp_solver *s, const int64_t *x_lohi, const int64_t *y_lohi, int nranks) {
  if (!s || !x_lohi || !y_lohi) return fail(AQP_EINVAL, "NULL argument");
  if (nranks != s->p->nranks || nranks > kMaxRanks) return fail(AQP_EINVAL, "nranks differs from the problem's shard");
  if (s->exec) return fail(AQP_ESTATE, "set the halos before aqp_solver_connect");
  const aqp_problem *p = s->p;
  for (int k = 0; k < nranks; ++k) {
    const bool xe = x_lohi[2 * k] >= x_lohi[2 * k + 1], ye = y_lohi[2 * k] >= y_lohi[2 * k + 1];
    if ((!xe && (x_lohi[2 * k] < p->xwin[2 * k] || x_lohi[2 * k + 1] > p->xwin[2 * k + 1])) ||
        (!ye && (y_lohi[2 * k] < p->ywin[2 * k] || y_lohi[2 * k + 1] > p->ywin[2 * k + 1])))
      return fail(AQP_EINVAL, "halo range outside the rank's gather window");
    s->gr.comm.xlo[k] = x_lohi[2 * k];
    s->gr.comm.xhi[k] = x_lohi[2 * k + 1];
    s->gr.comm.ylo[k] = y_lohi[2 * k];
    s->gr.comm.yhi[k] = y_lohi[2 * k + 1];
  }
  s->v.cm = s->gr.comm;
  return AQP_OK;
}

int aqp_solver_connect(aqp_solver *s, void *const *peer_bases, int nranks) {
  if (!s || !peer_bases) return fail(AQP_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  aqp_problem *p = s->p;
  if (nranks != p->nranks) return fail(AQP_EINVAL, "nranks differs from the problem's shard");
  if (nranks == 1) return peer_bases[0] == s->ws_base ? AQP_OK : fail(AQP_EINVAL, "peer_bases[0] is not this workspace");
  if (s->exec) return fail(AQP_ESTATE, "solver already connected");
  Comm c = s->gr.comm;
  c.nranks = nranks;
  if (const char *t = getenv("AQP_COMM_TIMEOUT_S")) c.timeout_ns = (unsigned long long)(atof(t) * 1e9);
  for (int k = 0; k < kMaxRanks; ++k) c.delta[k] = c.xdelta[k] = c.ydelta[k] = 0;
  for (int k = 0; k < nranks; ++k) {
    if (!peer_bases[k]) return fail(AQP_EINVAL, "NULL peer base");
    c.delta[k] = (long long)((const char *)peer_bases[k] - (const char *)s->ws_base);
    // entry g sits at window offset g - w0 on every rank
    c.xdelta[k] = c.delta[k] + 8 * (long long)(p->xw0() - p->xwin[2 * k]);
    c.ydelta[k] = c.delta[k] + 8 * (long long)(p->yw0() - p->ywin[2 * k]);
  }
  if (c.delta[p->rank] != 0) return fail(AQP_EINVAL, "peer_bases[rank] must be this solver's workspace");
  AQP_CUDA(cudaSetDevice(p->ctx->device));
  // Load every kernel of the solve now, while this rank still runs alone
  // (comm not yet enabled: no exchange waits).  With lazy module loading the
  // first launch of a kernel loads it under a context-wide synchronisation;
  // ranks that share a device would otherwise deadlock (until the exchange
  // timeout) when one rank loads a kernel while another spins in an exchange.
  {
    std::vector<double> ones((size_t)p->n, 1.0);
    double est = 0.0;
    int ann = 0;
    AQP_TRY(aqp_solver_estimate_norm(s, ones.data(), 1, &est, &ann));
    aqp_scalars sc{};
    sc.eta = 1.0;
    sc.omega = 1.0;
    sc.inner_tol = 1e-2;
    AQP_TRY(aqp_solver_init(s, &sc));
    AQP_TRY(run_eager(s, 1));
    aqp_check_result cr;
    AQP_TRY(aqp_solver_check(s, 1, &cr));
    AQP_TRY(state_op(s, 1));
    AQP_TRY(state_op(s, 2));
    AQP_TRY(state_op(s, 3));
    AQP_TRY(state_op(s, 4));
    AQP_TRY(pull_ctrl(s));
  }
  s->gr.comm = c;
  s->v.cm = c;
  return build_graph_any(s);
}

int aqp_solver_destroy(aqp_solver *s) {
  if (!s) return AQP_OK;
  if (s->gr.trace) cudaFree(s->gr.trace);
  if (s->gr.trace_n) cudaFree(s->gr.trace_n);
  if (s->exec) cudaGraphExecDestroy(s->exec);
  if (s->graph) cudaGraphDestroy(s->graph);
  delete s;
  return AQP_OK;
}

int aqp_solver_init(aqp_solver *s, const aqp_scalars *sc) {
  if (!s || !sc) return fail(AQP_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  s->h.s = *sc;
  s->h.xcur = 0; s->h.xprev = 1; s->h.ycur = 0; s->h.yprev = 1;
  s->h.pw_stop = 0;
  AQP_TRY(push_all(s));
  AQP_TRY(state_op(s, 0));
  return AQP_OK;
}

int aqp_solver_set_scalars(aqp_solver *s, const aqp_scalars *sc) {
  if (!s || !sc) return fail(AQP_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  s->h.s = *sc;
  return push_scalars(s);
}

int aqp_solver_get_scalars(aqp_solver *s, aqp_scalars *sc) {
  if (!s || !sc) return fail(AQP_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  AQP_TRY(pull_ctrl(s));
  *sc = s->h.s;
  return AQP_OK;
}

// Eager (non-graph) execution of a window: the same kernels launched one by
// one from the host, which reads the BB continuation flag after every inner
// iteration.  Used for profiling (ncu cannot profile kernel nodes of graphs
// with conditional nodes) and debugging; enabled by AQP_EAGER=1.
static int run_eager(aqp_solver *s, int64_t n_iters) {
  aqp_problem *p = s->p;
  cudaStream_t st = p->ctx->stream;
  SV v = s->v;
  v.in_graph = 0;
  GridRed gr = s->gr;
  const bool diag = p->quad_kind == AQP_QUAD_DIAGONAL;
  const bool lowrank = p->quad_kind == AQP_QUAD_SPARSE_LOW_RANK;
  auto lowrank_pass = [&](int src) -> int { return run_lowrank(s, src); };
  for (int64_t it = 0; it < n_iters; ++it) {
    if (diag) {
      OpP1Diag o{};
      o.v = v;
      AQP_CUDA(run_spmv_fin(st, p->At, o, gr));
    } else {
      OpP1Bb o{};
      o.v = v;
      AQP_CUDA(run_spmv(st, p->At, o, gr));
      if (s->shard) {
        k_comm_barrier<<<1, 32, 0, st>>>(gr);
        AQP_CUDA(cudaGetLastError());
      }
      if (lowrank) AQP_TRY(lowrank_pass(0));
      OpGrad<true> g0{};
      g0.v = v;
      AQP_CUDA(run_spmv_fin(st, p->Q, g0, gr));
      for (;;) {
        AQP_CUDA(cudaMemcpyAsync(&s->pin->flag, &s->d_ctrl->bb_cont, sizeof(int), cudaMemcpyDeviceToHost, st));
        AQP_CUDA(cudaStreamSynchronize(st));
        const int cont = s->pin->flag;
        if (!cont) break;
        OpStep sp{};
        sp.v = v;
        AQP_TRY(run_step(st, v, sp, gr));
        if (s->shard) {
          k_comm_barrier<<<1, 32, 0, st>>>(gr);
          AQP_CUDA(cudaGetLastError());
        }
        if (lowrank) AQP_TRY(lowrank_pass(1));
        OpGrad<false> gg{};
        gg.v = v;
        AQP_CUDA(run_spmv_fin(st, p->Q, gg, gr));
      }
      OpXPost xp{};
      xp.v = v;
      AQP_CUDA(run_elem_fin(st, v.nl, xp, gr));
    }
    OpP2 p2{};
    p2.v = v;
    AQP_CUDA(run_spmv_fin(st, p->A, p2, gr));
    AQP_CUDA(cudaMemcpyAsync(&s->pin->flag, &s->d_ctrl->s.halted, sizeof(int), cudaMemcpyDeviceToHost, st));
    AQP_CUDA(cudaStreamSynchronize(st));
    const int halted = s->pin->flag;
    if (halted) break;
  }
  return AQP_OK;
}

int aqp_solver_run(aqp_solver *s, int64_t n_iters) {
  if (!s) return fail(AQP_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  if (!s->exec && !s->eager) return fail(AQP_ESTATE, "sharded solver is not connected (aqp_solver_connect)");
  if (n_iters <= 0) return AQP_OK;
  // host mirror is current (the host only changes scalars between windows)
  s->h.s.iters_done = 0;
  s->h.s.inner_sum = 0;
  AQP_TRY(push_scalars(s));
  AQP_TRY(poke(s, &Ctrl::window_len, (int64_t)n_iters));
  if (s->eager) return run_eager(s, n_iters);
  AQP_CUDA(cudaGraphLaunch(s->exec, s->p->ctx->stream));
  return AQP_OK;
}

int aqp_solver_check(aqp_solver *s, int with_rays, aqp_check_result *out) {
  if (!s || !out) return fail(AQP_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  aqp_problem *p = s->p;
  cudaStream_t st = p->ctx->stream;
  const SV &v = s->v;
  GridRed gr = s->gr;
  const int rays = with_rays ? 1 : 0;
  AQP_CUDA(cudaMemsetAsync(&s->d_ctrl->red[0], 0, sizeof(double) * R_PW, st));
  { OpChkX o{}; o.v = v; o.rays = rays; AQP_CUDA(run_elem(st, v.nl, o, gr)); }
  AQP_TRY(push_buf(s, PB_XEVAL));
  { OpChkY o{}; o.v = v; o.rays = rays; AQP_CUDA(run_elem(st, v.ml, o, gr)); }
  { OpChkA o{}; o.v = v; o.rays = rays; AQP_CUDA(run_spmv(st, p->A, o, gr)); }
  if (rays) {  // normalised y-ray candidates: gathered by the A' ray passes
    AQP_TRY(push_buf(s, PB_DY0));
    AQP_TRY(push_buf(s, PB_DY1));
  }
  if (p->quad_kind != AQP_QUAD_DIAGONAL) {
    if (p->quad_kind == AQP_QUAD_SPARSE_LOW_RANK) AQP_TRY(run_lowrank(s, 2));
    OpStoreT<true> q{}; q.v = v; q.src = 0; q.dst = 0; q.red = -1;
    AQP_CUDA(run_spmv(st, p->Q, q, gr));
  }
  { OpStoreT<false> a{}; a.v = v; a.src = 1; a.dst = 1; a.red = -1; AQP_CUDA(run_spmv(st, p->At, a, gr)); }
  { OpChkR o{}; o.v = v; o.rays = rays; AQP_CUDA(run_elem(st, v.nl, o, gr)); }
  if (rays) {
    AQP_TRY(push_buf(s, PB_DX0));
    AQP_TRY(push_buf(s, PB_DX1));
    for (int j = 0; j < 2; ++j) {
      OpChkYRay o{}; o.v = v; o.j = j;
      AQP_CUDA(run_spmv(st, p->At, o, gr));
    }
    for (int j = 0; j < 2; ++j) {
      OpChkXRayT<false> a{}; a.v = v; a.j = j; a.which = 0;
      AQP_CUDA(run_spmv(st, p->A, a, gr));
      if (p->quad_kind == AQP_QUAD_DIAGONAL) {
        OpChkXRayT<false> q{}; q.v = v; q.j = j; q.which = 1;
        AQP_CUDA(run_elem(st, v.nl, q, gr));
      } else {
        if (p->quad_kind == AQP_QUAD_SPARSE_LOW_RANK) AQP_TRY(run_lowrank(s, 3 + j));
        OpChkXRayT<true> q{}; q.v = v; q.j = j; q.which = 1;
        AQP_CUDA(run_spmv(st, p->Q, q, gr));
      }
    }
  }
  AQP_TRY(pull_ctrl(s));
  const double *r = s->h.red;
  aqp_check_result &o = *out;
  std::memset(&o, 0, sizeof(o));
  o.primal_viol = r[R_PV];
  o.dual_viol = r[R_DV];
  o.qx_inf = r[R_QXI];
  o.aty_inf = r[R_ATYI];
  o.pr_pos = r[R_PRP]; o.pr_neg = r[R_PRN]; o.pr_bad = (int32_t)r[R_PRB];
  o.py_pos = r[R_PYP]; o.py_neg = r[R_PYN]; o.py_bad = (int32_t)r[R_PYB];
  o.xqx = r[R_XQX];
  o.cx = r[R_CX];
  o.pid_dx2 = r[R_PIDX];
  o.pid_dy2 = r[R_PIDY];
  o.have_avg_prev = s->h.s.have_avg_prev;
  for (int j = 0; j < 2; ++j) {
    const double *y = r + R_YR + 9 * j;
    o.yr_norm[j] = y[0]; o.yr_viol[j] = y[1]; o.yr_aty_inf[j] = y[2];
    o.yr_var_pos[j] = y[3]; o.yr_var_neg[j] = y[4]; o.yr_var_bad[j] = (int32_t)y[5];
    o.yr_con_pos[j] = y[6]; o.yr_con_neg[j] = y[7]; o.yr_con_bad[j] = (int32_t)y[8];
    const double *x = r + R_XR + 5 * j;
    o.xr_norm[j] = x[0]; o.xr_improvement[j] = x[1]; o.xr_viol_x[j] = x[2];
    o.xr_viol_s[j] = x[3]; o.xr_qd_inf[j] = x[4];
  }
  if (rays) {
    // engine.py:443-453: the window restarts and the averages become "previous"
    s->h.s.block_len = 0;
    s->h.s.have_avg_prev = 1;
    AQP_TRY(push_scalars(s));
  }
  return AQP_OK;
}

static int locked_state_op(aqp_solver *s, int mode) {
  if (!s) return fail(AQP_EINVAL, "NULL");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  return state_op(s, mode);
}
int aqp_solver_mark_cert(aqp_solver *s) { return locked_state_op(s, 1); }
int aqp_solver_restart(aqp_solver *s) { return locked_state_op(s, 2); }
int aqp_solver_rollback(aqp_solver *s) { return locked_state_op(s, 3); }

int aqp_solver_reset_window(aqp_solver *s) {
  if (!s) return fail(AQP_EINVAL, "NULL");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  AQP_TRY(state_op(s, 4));
  return AQP_OK;
}

int aqp_solver_read(aqp_solver *s, int which, double *host_out, int64_t len) {
  if (!s || !host_out) return fail(AQP_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  const SV &v = s->v;
  const double *src = nullptr;
  const int64_t nx = v.nl, ny = v.ml;  // a row shard copies its own slice
  int64_t need = 0;
  switch (which) {
    case 0: src = v.xeval; need = nx; break;
    case 1: src = pick3(v.ys, s->h.ycur); need = ny; break;
    case 2: src = v.rs; need = nx; break;
    case 3: src = pick2(v.dy, 0); need = ny; break;
    case 4: src = pick2(v.dy, 1); need = ny; break;
    case 5: src = pick2(v.dx, 0); need = nx; break;
    case 6: src = pick2(v.dx, 1); need = nx; break;
    case 7: src = pick3(v.xs, s->h.xcur); need = nx; break;
    default: return fail(AQP_EINVAL, "unknown buffer id");
  }
  if (len != need) return fail(AQP_EINVAL, "length mismatch");
  if (which == 1 || which == 7) {
    AQP_TRY(pull_ctrl(s));
    src = which == 1 ? pick3(v.ys, s->h.ycur) : pick3(v.xs, s->h.xcur);
  }
  cudaStream_t st = s->p->ctx->stream;
  if (need > (int64_t)aqp_solver::kBounce) {  // bulk: the multi-threaded pinned pipeline (aqp_xfer.cu)
    AQP_CUDA(cudaStreamSynchronize(st));
    AQP_TRY(bulk_copy(s->p->ctx->device, const_cast<double *>(src), host_out, (size_t)need * 8, false));
  }
  for (int64_t off = 0; off < need && need <= (int64_t)aqp_solver::kBounce; off += (int64_t)aqp_solver::kBounce) {
    const int64_t len = std::min<int64_t>(need - off, (int64_t)aqp_solver::kBounce);
    AQP_CUDA(cudaMemcpyAsync(s->bounce, src + off, len * 8, cudaMemcpyDeviceToHost, st));
    AQP_CUDA(cudaStreamSynchronize(st));
    std::memcpy(host_out + off, s->bounce, len * 8);
  }
  AQP_CUDA(cudaStreamSynchronize(st));
  if (s->shard) AQP_TRY(pull_ctrl(s));  // surfaces an exchange timeout
  return AQP_OK;
}

int aqp_solver_counters(aqp_solver *s, int64_t *out) {
  if (!s || !out) return fail(AQP_EINVAL, "NULL argument");
  out[0] = s->launches_per_iter_fixed;
  out[2] = s->pdl ? 1 : 0;
  out[1] = s->p->quad_kind == AQP_QUAD_DIAGONAL ? 0
           : (s->p->quad_kind == AQP_QUAD_SPARSE_LOW_RANK ? (s->p->r_dense ? 6 : 5) : 3);
  return AQP_OK;
}

// power iteration for the step size (linalg.py:287-312); runs before init
int aqp_solver_estimate_norm(aqp_solver *s, const double *host_v0, int iters, double *out, int *annihilated) {
  if (!s || !host_v0 || !out || !annihilated) return fail(AQP_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  aqp_problem *p = s->p;
  cudaStream_t st = p->ctx->stream;
  const SV &v = s->v;
  GridRed gr = s->gr;
  const int64_t n = v.nl;
  *annihilated = 0;
  AQP_TRY(poke(s, &Ctrl::pw_stop, 0));
  // every rank holds the whole start vector (drawn on the host): copy its
  // gather window (the whole vector unsharded)
  const int64_t w0 = p->xwin[2 * p->rank], w1 = p->xwin[2 * p->rank + 1];
  double *win = pick3(v.xbb, 0) - v.xoff + w0;
  if (w1 - w0 > (int64_t)aqp_solver::kBounce) {  // bulk: the multi-threaded pinned pipeline (aqp_xfer.cu)
    AQP_CUDA(cudaStreamSynchronize(st));
    AQP_TRY(bulk_copy(p->ctx->device, win, const_cast<double *>(host_v0 + w0), (size_t)(w1 - w0) * 8, true));
  }
  for (int64_t off = 0; off < w1 - w0 && w1 - w0 <= (int64_t)aqp_solver::kBounce; off += (int64_t)aqp_solver::kBounce) {
    const int64_t len = std::min<int64_t>(w1 - w0 - off, (int64_t)aqp_solver::kBounce);
    AQP_CUDA(cudaStreamSynchronize(st));  // the bounce buffer is free again
    std::memcpy(s->bounce, host_v0 + w0 + off, len * 8);
    AQP_CUDA(cudaMemcpyAsync(win + off, s->bounce, len * 8, cudaMemcpyHostToDevice, st));
  }
  // nv = |v|; u = v / nv; |A u| > 0 ?
  { OpPwNorm o{}; o.v = v; o.idx = 0; o.slot = R_PW; AQP_CUDA(run_elem(st, n, o, gr)); }
  k_pw_start<<<1, 1, 0, st>>>(s->d_ctrl, R_PW);
  AQP_CUDA(cudaGetLastError());
  { OpPwA<true> a{}; a.v = v; a.slot = R_PW + 1; AQP_CUDA(run_spmv(st, p->A, a, gr)); }
  AQP_TRY(pull_ctrl(s));
  if (!(s->h.red[R_PW] > 0.0) || !(s->h.red[R_PW + 1] > 0.0)) {
    *annihilated = 1;
    return AQP_OK;
  }
  for (int it = 0; it < iters; ++it) {
    OpPwA<false> a{}; a.v = v;                                   // t = A v
    AQP_CUDA(run_spmv(st, p->A, a, gr));
    AQP_TRY(push_buf(s, PB_TM));
    OpPwAt b{}; b.v = v; b.dst = 1 + (it & 1);                   // w = A't, |w|, next v
    AQP_CUDA(run_spmv_fin(st, p->At, b, gr));
    AQP_TRY(push_buf(s, b.dst == 1 ? PB_PW : PB_PW2));
  }
  // final |A v| (the stop flag must not suppress it)
  AQP_TRY(poke(s, &Ctrl::pw_stop, 0));
  { OpPwA<true> a{}; a.v = v; a.slot = R_PW + 3; AQP_CUDA(run_spmv(st, p->A, a, gr)); }
  AQP_TRY(pull_ctrl(s));
  *out = sqrt(s->h.red[R_PW + 3]);
  return AQP_OK;
}

// L2 eviction by a streaming READ of a large buffer: a memset would leave
// the L2 full of dirty lines whose write-back the timed kernel then pays.
__global__ void k_flush_read(const double2 *p, int64_t n2, double *sink) {
  double a = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 q = __ldcs(p + i);
    a += q.x + q.y;
  }
  if (a == 1.2345e-300) *sink = a;
}

// Stand-alone timing of one hot kernel (for the roofline in bench.py): `reps`
// launches on the solver stream, each preceded by an L2 flush (a write of
// `flush_bytes` to `flush`), timed with events around the kernel only.
// kernel: 0 = BB gradient pass (Q SpMV + epilogue + 7 partial sums),
//         1 = BB step (x_t = clamp(x - alpha g)), 2 = P1 (A'y + epilogue),
//         3 = P2 (A xbar + dual epilogue + fold), 4 = X (primal epilogue +
//         fold), 5 = the fold/finalize kernel of pass 0.
// Run after aqp_solver_init; it overwrites BB scratch and the control block's
// BB fields, so re-init before solving.
int aqp_solver_time_kernel(aqp_solver *s, int kernel, int reps, void *flush, size_t flush_bytes, double *avg_ms) {
  if (!s || !avg_ms || reps <= 0) return fail(AQP_EINVAL, "bad argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  aqp_problem *p = s->p;
  cudaStream_t st = p->ctx->stream;
  SV v = s->v;
  v.in_graph = 0;
  GridRed gr = s->gr;
  cudaEvent_t e0, e1;
  AQP_CUDA(cudaEventCreate(&e0));
  AQP_CUDA(cudaEventCreate(&e1));
  // a valid BB state: slots 0/1/2 distinct, alpha finite
  AQP_TRY(poke(s, &Ctrl::bb_cur, 0));
  AQP_TRY(poke(s, &Ctrl::bb_best, 0));
  AQP_TRY(poke(s, &Ctrl::bb_new, 1));
  AQP_TRY(poke(s, &Ctrl::g_cur, 0));
  AQP_TRY(poke(s, &Ctrl::g_new, 1));
  AQP_TRY(poke(s, &Ctrl::alpha, 1e-3));
  double total = 0.0;
  for (int r = 0; r < reps; ++r) {
    if (flush && flush_bytes) {
      k_flush_read<<<148 * 8, 256, 0, st>>>((const double2 *)flush, (int64_t)(flush_bytes / 16), s->gr.partials);
      AQP_CUDA(cudaGetLastError());
    }
    AQP_CUDA(cudaEventRecord(e0, st));
    switch (kernel) {
      case 0: {  // the SpMV pass alone (its partials fold is kernel 5)
        OpGrad<false> o{};
        o.v = v;
        AQP_CUDA(run_spmv(st, p->Q, o, gr));
        break;
      }
      case 5: {
        OpGrad<false> o{};
        o.v = v;
#if AQP_FOLD_CLUSTER
        run_fold(st, o, gr, (unsigned)p->Q.nitems);
#else
        fin_ctrl_op<OpGrad<false>><<<1, kFinThreads, 0, st>>>(o, gr, (unsigned)p->Q.nitems);
#endif
        AQP_CUDA(cudaGetLastError());
        break;
      }
      case 1: {
        OpStep o{};
        o.v = v;
        AQP_TRY(run_step(st, v, o, gr));
        break;
      }
      case 2: {
        OpP1Bb o{};
        o.v = v;
        AQP_CUDA(run_spmv(st, p->At, o, gr));
        break;
      }
      case 3: {
        OpP2 o{};
        o.v = v;
        AQP_CUDA(run_spmv_fin(st, p->A, o, gr));
        break;
      }
      case 4: {
        OpXPost o{};
        o.v = v;
        AQP_CUDA(run_elem_fin(st, v.nl, o, gr));
        break;
      }
      case 6: {  // dense R x (block partials + fold), source x_t
        if (!p->r_dense) return fail(AQP_EINVAL, "kernel 6 needs a dense low-rank R");
        const int nb = (int)dense_rx_blocks(p->R.cols);
        k_dense_rx<<<nb, kThreads, 0, st>>>(v, 1);
        k_dense_rx_fold<<<p->R.rows, kThreads, 0, st>>>(v, 1, nb);
        AQP_CUDA(cudaGetLastError());
        break;
      }
      case 7: {  // dense R'(R x)
        if (!p->r_dense) return fail(AQP_EINVAL, "kernel 7 needs a dense low-rank R");
        k_dense_rtv<<<elem_grid(p->R.cols), kThreads, 0, st>>>(v, 1);
        AQP_CUDA(cudaGetLastError());
        break;
      }
      default: return fail(AQP_EINVAL, "unknown kernel id");
    }
    AQP_CUDA(cudaEventRecord(e1, st));
    AQP_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    AQP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    total += ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *avg_ms = total / reps;
  return AQP_OK;
}

// ---------------------------------------------------------------- CUDA IPC (peer workspaces)
typedef int (*PFN_addr_range)(unsigned long long *, size_t *, unsigned long long);

int aqp_ipc_get_handle(const void *dev_ptr, void *handle64, size_t *offset) {
  if (!dev_ptr || !handle64 || !offset) return fail(AQP_EINVAL, "NULL argument");
  static PFN_addr_range fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *f = nullptr;
    AQP_CUDA(cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) return fail(AQP_ECUDA, "cuMemGetAddressRange unavailable");
    fn = (PFN_addr_range)f;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (fn(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0) return fail(AQP_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  AQP_CUDA(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base));
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (size_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  return AQP_OK;
}

int aqp_ipc_open(const void *handle64, size_t offset, void **dev_ptr) {
  if (!handle64 || !dev_ptr) return fail(AQP_EINVAL, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void *base = nullptr;
  AQP_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr = (char *)base + offset;
  return AQP_OK;
}

int aqp_ipc_close(void *dev_ptr, size_t offset) {
  if (!dev_ptr) return fail(AQP_EINVAL, "NULL argument");
  AQP_CUDA(cudaIpcCloseMemHandle((char *)dev_ptr - offset));
  return AQP_OK;
}

// Device trace (AQP_TRACE=1): copies up to `cap` (tag, ns) pairs, oldest
// first, and resets the ring; *count = pairs copied (0 when tracing is off).
int aqp_solver_trace(aqp_solver *s, unsigned long long *host_out, int64_t cap, int64_t *count) {
  if (!s || !count) return fail(AQP_EINVAL, "NULL argument");
  std::lock_guard<std::recursive_mutex> ctx_lock_(s->p->ctx->mu);
  *count = 0;
  if (!s->gr.trace) return AQP_OK;
  cudaStream_t st = s->p->ctx->stream;
  unsigned n = 0;
  AQP_CUDA(cudaMemcpyAsync(&n, s->gr.trace_n, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  const int64_t m = std::min<int64_t>({(int64_t)n, (int64_t)s->gr.trace_cap, cap});
  if (m > 0 && host_out) {
    AQP_CUDA(cudaMemcpyAsync(host_out, s->gr.trace, sizeof(unsigned long long) * 2 * m, cudaMemcpyDeviceToHost, st));
  }
  AQP_CUDA(cudaMemsetAsync(s->gr.trace_n, 0, sizeof(unsigned), st));
  AQP_CUDA(cudaStreamSynchronize(st));
  *count = m;
  return AQP_OK;
}

}  // extern "C"
