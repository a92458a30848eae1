/*
 * claw_oracle.c -- CPU ORACLE (test infrastructure only; see claw_oracle.h).
 *
 * A plain, slow, literal implementation of one AMR-level step of the
 * wave-propagation method of arXiv 1808.02638 for 2D linear acoustics.
 * The per-patch step follows Clawpack's classic structure (P:50, P:433-440
 * name Clawpack's rpn2/rpt2 "normal" and "transverse" Riemann solvers):
 *
 *   step2  : x-sweeps over rows j = 0..my+1, then y-sweeps over columns
 *            i = 0..mx+1, accumulating fm/fp/gm/gp, then the flux-difference
 *            update, which is eq. (W);
 *   flux2  : Riemann solves at every interface 0..n+2 of the 1D slice
 *            (rpn2), wave limiting (limiter), second-order correction
 *            cqxx = sum |s|(1-|s|dt/dx) W~ (the F~ terms of eq. (W)),
 *            transverse splitting of A-dq, A+dq (rpt2; "corner transport",
 *            P:500) into the transverse fluxes gadd;
 *   rpn2   : eigen-decomposition of A (or B) for acoustics;
 *   rpt2   : eigen-decomposition of B (or A) applied to A-dq / A+dq.
 *
 * Ghost fill follows the three cases of P:125-132 with the composite reading
 * of DESIGN.md ("Readings" R1, R8-R10): per-axis clamp (extrapolation) or
 * wrap (periodic) of the global index, then a copy from the same-level patch
 * holding the mapped cell, else (level > 1) space-time interpolation from the
 * coarser level.
 *
 * Index convention (Clawpack, 1-based): interior cells i = 1..mx,
 * j = 1..my; ghost cells -1, 0 and mx+1, mx+2.  Interface i is the left edge
 * of cell i (x_{i-1/2}).  Padded storage index = i + 1.
 */
#include "claw_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#define NTHREADS(c) ((c)->cfg.nthreads > 0 ? (c)->cfg.nthreads : omp_get_max_threads())
#else
#define NTHREADS(c) 1
#endif

#define MAXLEVEL 8
#define MEQN 3
#define MWAVES 2
#define BUCKET 16

typedef struct {
  int npatch;
  oracle_patch_desc* desc;
  int64_t* i0; /* global 0-based index of interior cell (1,1) */
  int64_t* j0;
  double** qpad;  /* current time level, padded [3][my+4][mx+4] */
  double** qold;  /* previous time level, interior [3][my][mx] */
  double* pcfl;   /* per-patch max Courant number of the last step */
  double** auxpad; /* variable media (oracle_set_aux), padded [2][my+4][mx+4] rho, K; NULL: per-patch constants */
  double dx, dy;
  int64_t nx, ny; /* level index extent of the domain */
  int ratio_to_coarser; /* R_{L-1}; 0 for level 1 */
  double t_old, t_new;
  /* bucket grid for "which patch holds cell (I,J)" */
  int64_t nbx, nby;
  int64_t* bstart; /* CSR offsets, nbx*nby+1 */
  int* blist;
  /* conservation-fix registers of this (fine) level against level-1: one per
   * coarse-fine edge E, i.e. a level-1 cell C not covered by this level whose
   * edge neighbour (through periodic wrap) is covered.  E's fine side is the
   * R cells of this level adjacent to E, starting at (rfi, rfj) in patch rfp
   * and running along E. */
  int nreg;
  int *rcp, *rli, *rlj;   /* coarse patch, local cell of C */
  int *rdir, *rside;      /* 0: x-edge, 1: y-edge; side 0: C left/below E, 1: C right/above */
  int *rfp, *rfi, *rfj;   /* fine patch and local index of the first fine cell */
  double* racc;           /* [nreg][3] accumulated modification of C */
} olevel;

struct oracle_ctx {
  oracle_config cfg;
  int reflux;             /* conservation fix on (oracle_set_reflux) */
  olevel lev[MAXLEVEL + 1];
  olevel stash[MAXLEVEL + 1]; /* levels discarded by a regrid: copy sources for
                                 the regrid that re-creates them (R18) */
  char err[512];
};

static int fail(oracle_ctx* c, int code, const char* msg) {
  if (c) snprintf(c->err, sizeof c->err, "%s", msg);
  return code;
}

const char* oracle_last_error(const oracle_ctx* c) { return c ? c->err : "null ctx"; }

/* ------------------------------------------------------------------------ */
/* Riemann solvers: linear acoustics, A = [[0,K,0],[1/rho,0,0],[0,0,0]],    */
/* B = [[0,0,K],[0,0,0],[1/rho,0,0]].  c = sqrt(K/rho),          */
/* Z = rho c.  Eigenvalues -c, 0, +c; the zero-speed wave carries nothing     */
/* into the flux and is omitted (mwaves = 2), as in Clawpack's acoustics.     */
/* ------------------------------------------------------------------------ */

void oracle_rpn2(int ixy, const double* ql, const double* qr, double rho,
                 double K, double* wave, double* s, double* amdq, double* apdq) {
  /* ql = state of cell i-1 (left of the interface), qr = state of cell i. */
  const double cc = sqrt(K / rho);
  const double zz = rho * cc;
  const int mu = (ixy == 1) ? 1 : 2; /* normal velocity component */
  const int mv = (ixy == 1) ? 2 : 1; /* tangential velocity component */
  const double delta1 = qr[0] - ql[0];
  const double delta2 = qr[mu] - ql[mu];
  const double a1 = (-delta1 + zz * delta2) / (2.0 * zz);
  const double a2 = (delta1 + zz * delta2) / (2.0 * zz);
  /* wave 1: left-going, speed -c, eigenvector (-Z, 1, 0) */
  wave[0 * MEQN + 0] = -a1 * zz;
  wave[0 * MEQN + mu] = a1;
  wave[0 * MEQN + mv] = 0.0;
  s[0] = -cc;
  /* wave 2: right-going, speed +c, eigenvector (Z, 1, 0) */
  wave[1 * MEQN + 0] = a2 * zz;
  wave[1 * MEQN + mu] = a2;
  wave[1 * MEQN + mv] = 0.0;
  s[1] = cc;
  for (int m = 0; m < MEQN; ++m) {
    amdq[m] = s[0] * wave[0 * MEQN + m];
    apdq[m] = s[1] * wave[1 * MEQN + m];
  }
}

void oracle_rpt2(int ixy, const double* asdq, double rho, double K,
                 double* bmasdq, double* bpasdq) {
  /* Split asdq into down-going (B^-) and up-going (B^+) parts with the
   * eigenvectors of the matrix for the transverse direction. */
  const double cc = sqrt(K / rho);
  const double zz = rho * cc;
  const int mu = (ixy == 1) ? 1 : 2;
  const int mv = (ixy == 1) ? 2 : 1;
  const double a1 = (-asdq[0] + zz * asdq[mv]) / (2.0 * zz);
  const double a2 = (asdq[0] + zz * asdq[mv]) / (2.0 * zz);
  bmasdq[0] = cc * a1 * zz;
  bmasdq[mu] = 0.0;
  bmasdq[mv] = -cc * a1;
  bpasdq[0] = cc * a2 * zz;
  bpasdq[mu] = 0.0;
  bpasdq[mv] = cc * a2;
}

/* ------------------------------------------------------------------------ */
/* Variable-coefficient acoustics (NEXT-4; heterogeneous media P:66;   */
/* per-system normal/transverse solvers P:433-436; R20).  Each cell */
/* has its own rho, K (an aux array), so A and B of P:457-466 differ between  */
/* the two sides of an interface.  The interface Riemann problem is solved   */
/* with the eigenvectors of each side's own matrix: the left-going wave lives */
/* in the left medium (speed -c_l, eigenvector (-Z_l, 1, 0)), the right-going */
/* one in the right medium (+c_r, (Z_r, 1, 0)), and qr - ql = W1 + W2.         */
/* ------------------------------------------------------------------------ */

void oracle_rpn2_vc(int ixy, const double* ql, const double* qr, double rhol, double Kl,
                    double rhor, double Kr, double* wave, double* s, double* amdq, double* apdq) {
  const double cl = sqrt(Kl / rhol), zl = rhol * cl;
  const double cr = sqrt(Kr / rhor), zr = rhor * cr;
  const int mu = (ixy == 1) ? 1 : 2;
  const int mv = (ixy == 1) ? 2 : 1;
  const double delta1 = qr[0] - ql[0];
  const double delta2 = qr[mu] - ql[mu];
  /* solve  -a1 zl + a2 zr = delta1,  a1 + a2 = delta2 */
  const double a1 = (-delta1 + zr * delta2) / (zl + zr);
  const double a2 = (delta1 + zl * delta2) / (zl + zr);
  wave[0 * MEQN + 0] = -a1 * zl;
  wave[0 * MEQN + mu] = a1;
  wave[0 * MEQN + mv] = 0.0;
  s[0] = -cl;
  wave[1 * MEQN + 0] = a2 * zr;
  wave[1 * MEQN + mu] = a2;
  wave[1 * MEQN + mv] = 0.0;
  s[1] = cr;
  for (int m = 0; m < MEQN; ++m) {
    amdq[m] = s[0] * wave[0 * MEQN + m];
    apdq[m] = s[1] * wave[1 * MEQN + m];
  }
}

/* Transverse split of asdq, which enters a cell with medium (rho, K), into a
 * part going to the cell below it in the transverse direction (rho_m, K_m) and
 * a part going to the cell above (rho_p, K_p).  Each part is the transmitted
 * wave of the Riemann problem across that transverse edge with jump asdq:
 * below:  asdq = a1 (-Z_m, 0, 1) + b (Z, 0, 1)    -> B-asdq = -c_m a1 (-Z_m, 0, 1)
 * above:  asdq = b (-Z, 0, 1) + a2 (Z_p, 0, 1)    -> B+asdq = +c_p a2 (Z_p, 0, 1)
 * (components written for ixy = 1, i.e. the transverse velocity is v). */
void oracle_rpt2_vc(int ixy, const double* asdq, double rho_m, double K_m, double rho, double K,
                    double rho_p, double K_p, double* bmasdq, double* bpasdq) {
  const int mu = (ixy == 1) ? 1 : 2;
  const int mv = (ixy == 1) ? 2 : 1;
  const double cm = sqrt(K_m / rho_m), zm = rho_m * cm;
  const double cc = sqrt(K / rho), zz = rho * cc;
  const double cp = sqrt(K_p / rho_p), zp = rho_p * cp;
  const double a1 = (-asdq[0] + zz * asdq[mv]) / (zm + zz);
  const double a2 = (asdq[0] + zz * asdq[mv]) / (zz + zp);
  bmasdq[0] = cm * a1 * zm;
  bmasdq[mu] = 0.0;
  bmasdq[mv] = -cm * a1;
  bpasdq[0] = cp * a2 * zp;
  bpasdq[mu] = 0.0;
  bpasdq[mv] = cp * a2;
}

/* Wave limiter function phi(theta) (P:501 names van Leer; BASELINE configs use
 * MC and minmod).  Clawpack numbering. */
double oracle_philim(int limiter, double r) {
  double c;
  switch (limiter) {
    case 1: /* minmod */
      return fmax(0.0, fmin(1.0, r));
    case 2: /* superbee */
      return fmax(0.0, fmax(fmin(1.0, 2.0 * r), fmin(2.0, r)));
    case 3: /* van Leer */
      return (r + fabs(r)) / (1.0 + fabs(r));
    case 4: /* monotonized centered */
      c = (1.0 + r) / 2.0;
      return fmax(0.0, fmin(c, fmin(2.0, 2.0 * r)));
    default: /* 0: no limiting (Lax-Wendroff) */
      return 1.0;
  }
}

/* ------------------------------------------------------------------------ */
/* flux2: one 1D slice of n cells with ghosts -1..n+2.                       */
/* q1d[m][i+1], i=-1..n+2.  Outputs (index = i+1):                           */
/*   faddm[m][i], faddp[m][i]   i = 1..n+1   (fluxes at interface i)         */
/*   gadd[k][m][i]              i = 0..n+1   (k=0: B^- part -> edge of cell  */
/*                              i at the "low" transverse side, k=1: high)   */
/* ------------------------------------------------------------------------ */
/* aux1d (variable media, else NULL): [r][k][i+1], r = 0 the slice below in the
 * transverse direction, 1 this slice, 2 the slice above; k = 0 rho, 1 K. */
static void flux2(int ixy, int n, const double* q1d, const double* aux1d, double dtdx, double rho,
                  double K, int limiter, int order_trans, double* faddm,
                  double* faddp, double* gadd, double* cfl1d) {
  const int W = n + 4; /* stride of every per-slice array */
#define Q1(m, i) q1d[(m) * W + (i) + 1]
#define FM(m, i) faddm[(m) * W + (i) + 1]
#define FP(m, i) faddp[(m) * W + (i) + 1]
#define GADD(k, m, i) gadd[((k) * MEQN + (m)) * W + (i) + 1]
  double* wave = (double*)calloc((size_t)MWAVES * MEQN * W, sizeof(double));
  double* s = (double*)calloc((size_t)MWAVES * W, sizeof(double));
  double* amdq = (double*)calloc((size_t)MEQN * W, sizeof(double));
  double* apdq = (double*)calloc((size_t)MEQN * W, sizeof(double));
  double* cqxx = (double*)calloc((size_t)MEQN * W, sizeof(double));
#define WAVE(mw, m, i) wave[((mw) * MEQN + (m)) * W + (i) + 1]
#define S(mw, i) s[(mw) * W + (i) + 1]
#define AM(m, i) amdq[(m) * W + (i) + 1]
#define AP(m, i) apdq[(m) * W + (i) + 1]
#define CQ(m, i) cqxx[(m) * W + (i) + 1]
#define AUX(r, k, i) aux1d[((r) * 2 + (k)) * W + (i) + 1]

  for (int m = 0; m < MEQN; ++m)
    for (int i = -1; i <= n + 2; ++i) {
      FM(m, i) = 0.0;
      FP(m, i) = 0.0;
      GADD(0, m, i) = 0.0;
      GADD(1, m, i) = 0.0;
    }

  /* Normal Riemann problems at interfaces i = 0..n+2 (between i-1 and i). */
  for (int i = 0; i <= n + 2; ++i) {
    double ql[MEQN], qr[MEQN], wv[MWAVES * MEQN], sp[MWAVES], am[MEQN], ap[MEQN];
    for (int m = 0; m < MEQN; ++m) {
      ql[m] = Q1(m, i - 1);
      qr[m] = Q1(m, i);
    }
    if (aux1d)
      oracle_rpn2_vc(ixy, ql, qr, AUX(1, 0, i - 1), AUX(1, 1, i - 1), AUX(1, 0, i), AUX(1, 1, i),
                     wv, sp, am, ap);
    else
      oracle_rpn2(ixy, ql, qr, rho, K, wv, sp, am, ap);
    for (int mw = 0; mw < MWAVES; ++mw) {
      S(mw, i) = sp[mw];
      for (int m = 0; m < MEQN; ++m) WAVE(mw, m, i) = wv[mw * MEQN + m];
    }
    for (int m = 0; m < MEQN; ++m) {
      AM(m, i) = am[m];
      AP(m, i) = ap[m];
    }
  }

  /* First-order fluctuations enter the fluxes (eq. (W) terms A+-dq). */
  for (int i = 1; i <= n + 1; ++i)
    for (int m = 0; m < MEQN; ++m) {
      FP(m, i) = FP(m, i) - AP(m, i);
      FM(m, i) = FM(m, i) + AM(m, i);
    }

  /* CFL number nu = |s dt/dx|, max over the slice. */
  double cfl = 0.0;
  for (int mw = 0; mw < MWAVES; ++mw)
    for (int i = 1; i <= n + 1; ++i) {
      cfl = fmax(cfl, dtdx * S(mw, i));
      cfl = fmax(cfl, -dtdx * S(mw, i));
    }
  *cfl1d = cfl;

  /* Wave limiter (Clawpack limiter.f): theta = <W_up, W> / <W, W>, upwind
   * side chosen by the sign of the speed; waves with <W,W> = 0 skipped. */
  if (limiter != 0) {
    for (int mw = 0; mw < MWAVES; ++mw) {
      double dotr = 0.0;
      for (int i = 0; i <= n + 1; ++i) {
        double wnorm2 = 0.0, dotl = dotr;
        dotr = 0.0;
        for (int m = 0; m < MEQN; ++m) {
          wnorm2 = wnorm2 + WAVE(mw, m, i) * WAVE(mw, m, i);
          dotr = dotr + WAVE(mw, m, i) * WAVE(mw, m, i + 1);
        }
        if (i == 0) continue;
        if (wnorm2 == 0.0) continue;
        double r = (S(mw, i) > 0.0) ? dotl / wnorm2 : dotr / wnorm2;
        double wlimitr = oracle_philim(limiter, r);
        for (int m = 0; m < MEQN; ++m) WAVE(mw, m, i) = wlimitr * WAVE(mw, m, i);
      }
    }
  }

  /* Second-order corrections cqxx = sum_p |s_p| (1 - |s_p| dt/dx) W~_p. */
  for (int i = 1; i <= n + 1; ++i) {
    const double dtdxave = 0.5 * (dtdx + dtdx);
    for (int m = 0; m < MEQN; ++m) {
      CQ(m, i) = 0.0;
      for (int mw = 0; mw < MWAVES; ++mw)
        CQ(m, i) = CQ(m, i) + fabs(S(mw, i)) * (1.0 - fabs(S(mw, i)) * dtdxave) * WAVE(mw, m, i);
      FM(m, i) = FM(m, i) + 0.5 * CQ(m, i);
      FP(m, i) = FP(m, i) + 0.5 * CQ(m, i);
    }
  }

  if (order_trans != 0) {
    if (order_trans == 2)
      for (int i = 1; i <= n + 1; ++i)
        for (int m = 0; m < MEQN; ++m) {
          AM(m, i) = AM(m, i) + CQ(m, i);
          AP(m, i) = AP(m, i) - CQ(m, i);
        }
    /* Transverse propagation: A-dq at interface i enters cell i-1, A+dq cell i;
     * each is split into B^- (to that cell's low transverse edge) and B^+
     * (high edge). */
    for (int i = 1; i <= n + 1; ++i) {
      double asdq[MEQN], bm[MEQN], bp[MEQN];
      for (int m = 0; m < MEQN; ++m) asdq[m] = AM(m, i);
      if (aux1d) /* A-dq enters cell i-1 */
        oracle_rpt2_vc(ixy, asdq, AUX(0, 0, i - 1), AUX(0, 1, i - 1), AUX(1, 0, i - 1),
                       AUX(1, 1, i - 1), AUX(2, 0, i - 1), AUX(2, 1, i - 1), bm, bp);
      else
        oracle_rpt2(ixy, asdq, rho, K, bm, bp);
      for (int m = 0; m < MEQN; ++m) {
        GADD(0, m, i - 1) = GADD(0, m, i - 1) - 0.5 * dtdx * bm[m];
        GADD(1, m, i - 1) = GADD(1, m, i - 1) - 0.5 * dtdx * bp[m];
      }
      for (int m = 0; m < MEQN; ++m) asdq[m] = AP(m, i);
      if (aux1d) /* A+dq enters cell i */
        oracle_rpt2_vc(ixy, asdq, AUX(0, 0, i), AUX(0, 1, i), AUX(1, 0, i), AUX(1, 1, i),
                       AUX(2, 0, i), AUX(2, 1, i), bm, bp);
      else
        oracle_rpt2(ixy, asdq, rho, K, bm, bp);
      for (int m = 0; m < MEQN; ++m) {
        GADD(0, m, i) = GADD(0, m, i) - 0.5 * dtdx * bm[m];
        GADD(1, m, i) = GADD(1, m, i) - 0.5 * dtdx * bp[m];
      }
    }
  }
  free(wave);
  free(s);
  free(amdq);
  free(apdq);
  free(cqxx);
#undef Q1
#undef FM
#undef FP
#undef GADD
#undef WAVE
#undef S
#undef AM
#undef AP
#undef CQ
#undef AUX
}

/* ------------------------------------------------------------------------ */
/* step2: one step of eq. (W) on one padded patch.                           */
/* ------------------------------------------------------------------------ */
/* step2 proper.  If flux_out is not NULL it receives the four accumulated
 * edge arrays fm, fp, gm, gp (each [3][my+4][mx+4], padded index = Clawpack
 * index + 1; the caller frees them) -- the conservation fix reads the ones on
 * coarse-fine interfaces ("can be saved ... for later use"). */
/* auxpad (variable media, else NULL): [2][my+4][mx+4] rho, K with the ghost
 * frame filled (oracle_set_aux); then rho and K are not used. */
static int step2(int mx, int my, const double* qpad, const double* auxpad, double dx, double dy,
                 double dt, double rho, double K, int limiter, int order_trans,
                 double* qout_pad, double* cfl_out, double** flux_out) {
  if (mx < 1 || my < 1 || !(dx > 0.0) || !(dy > 0.0) || (!auxpad && (!(rho > 0.0) || !(K > 0.0))))
    return -1;
  const int PX = mx + 4, PY = my + 4;
  const size_t plane = (size_t)PX * PY;
#define QP(m, i, j) qpad[(m) * plane + (size_t)((j) + 1) * PX + (i) + 1]
#define QN(m, i, j) qout_pad[(m) * plane + (size_t)((j) + 1) * PX + (i) + 1]
  double* fm = (double*)calloc(MEQN * plane, sizeof(double));
  double* fp = (double*)calloc(MEQN * plane, sizeof(double));
  double* gm = (double*)calloc(MEQN * plane, sizeof(double));
  double* gp = (double*)calloc(MEQN * plane, sizeof(double));
#define FMA_(m, i, j) fm[(m) * plane + (size_t)((j) + 1) * PX + (i) + 1]
#define FPA_(m, i, j) fp[(m) * plane + (size_t)((j) + 1) * PX + (i) + 1]
#define GMA_(m, i, j) gm[(m) * plane + (size_t)((j) + 1) * PX + (i) + 1]
#define GPA_(m, i, j) gp[(m) * plane + (size_t)((j) + 1) * PX + (i) + 1]
  const int NMAX = (mx > my ? mx : my) + 4;
  double* q1d = (double*)calloc((size_t)MEQN * NMAX, sizeof(double));
  double* faddm = (double*)calloc((size_t)MEQN * NMAX, sizeof(double));
  double* faddp = (double*)calloc((size_t)MEQN * NMAX, sizeof(double));
  double* gadd = (double*)calloc((size_t)2 * MEQN * NMAX, sizeof(double));
  double* aux1d = auxpad ? (double*)calloc((size_t)3 * 2 * NMAX, sizeof(double)) : NULL;
#define AP_(k, i, j) auxpad[(k) * plane + (size_t)((j) + 1) * PX + (i) + 1]
  double cfl = 0.0, cfl1d;

  /* x-sweeps: rows j = 0..my+1 */
  const double dtdx = dt / dx;
  const int WX = mx + 4;
  for (int j = 0; j <= my + 1; ++j) {
    for (int m = 0; m < MEQN; ++m)
      for (int i = -1; i <= mx + 2; ++i) q1d[m * WX + i + 1] = QP(m, i, j);
    if (aux1d) /* media of rows j-1, j, j+1 */
      for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 2; ++k)
          for (int i = -1; i <= mx + 2; ++i) aux1d[(r * 2 + k) * WX + i + 1] = AP_(k, i, j - 1 + r);
    flux2(1, mx, q1d, aux1d, dtdx, rho, K, limiter, order_trans, faddm, faddp, gadd, &cfl1d);
    cfl = fmax(cfl, cfl1d);
    for (int i = 1; i <= mx + 1; ++i)
      for (int m = 0; m < MEQN; ++m) {
        FMA_(m, i, j) = FMA_(m, i, j) + faddm[m * WX + i + 1];
        FPA_(m, i, j) = FPA_(m, i, j) + faddp[m * WX + i + 1];
        GMA_(m, i, j) = GMA_(m, i, j) + gadd[(0 * MEQN + m) * WX + i + 1];
        GPA_(m, i, j) = GPA_(m, i, j) + gadd[(0 * MEQN + m) * WX + i + 1];
        GMA_(m, i, j + 1) = GMA_(m, i, j + 1) + gadd[(1 * MEQN + m) * WX + i + 1];
        GPA_(m, i, j + 1) = GPA_(m, i, j + 1) + gadd[(1 * MEQN + m) * WX + i + 1];
      }
  }

  /* y-sweeps: columns i = 0..mx+1 */
  const double dtdy = dt / dy;
  const int WY = my + 4;
  for (int i = 0; i <= mx + 1; ++i) {
    for (int m = 0; m < MEQN; ++m)
      for (int j = -1; j <= my + 2; ++j) q1d[m * WY + j + 1] = QP(m, i, j);
    if (aux1d) /* media of columns i-1, i, i+1 */
      for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 2; ++k)
          for (int j = -1; j <= my + 2; ++j) aux1d[(r * 2 + k) * WY + j + 1] = AP_(k, i - 1 + r, j);
    flux2(2, my, q1d, aux1d, dtdy, rho, K, limiter, order_trans, faddm, faddp, gadd, &cfl1d);
    cfl = fmax(cfl, cfl1d);
    for (int j = 1; j <= my + 1; ++j)
      for (int m = 0; m < MEQN; ++m) {
        GMA_(m, i, j) = GMA_(m, i, j) + faddm[m * WY + j + 1];
        GPA_(m, i, j) = GPA_(m, i, j) + faddp[m * WY + j + 1];
        FMA_(m, i, j) = FMA_(m, i, j) + gadd[(0 * MEQN + m) * WY + j + 1];
        FPA_(m, i, j) = FPA_(m, i, j) + gadd[(0 * MEQN + m) * WY + j + 1];
        FMA_(m, i + 1, j) = FMA_(m, i + 1, j) + gadd[(1 * MEQN + m) * WY + j + 1];
        FPA_(m, i + 1, j) = FPA_(m, i + 1, j) + gadd[(1 * MEQN + m) * WY + j + 1];
      }
  }

  /* Flux-difference update, eq. (W). */
  memcpy(qout_pad, qpad, MEQN * plane * sizeof(double));
  for (int m = 0; m < MEQN; ++m)
    for (int j = 1; j <= my; ++j)
      for (int i = 1; i <= mx; ++i)
        QN(m, i, j) = QP(m, i, j) - dtdx * (FMA_(m, i + 1, j) - FPA_(m, i, j))
                      - dtdy * (GMA_(m, i, j + 1) - GPA_(m, i, j));

  *cfl_out = cfl;
  if (flux_out) {
    flux_out[0] = fm; flux_out[1] = fp; flux_out[2] = gm; flux_out[3] = gp;
  } else {
    free(fm); free(fp); free(gm); free(gp);
  }
  free(q1d); free(faddm); free(faddp); free(gadd); free(aux1d);
  return 0;
#undef AP_
#undef QP
#undef QN
#undef FMA_
#undef FPA_
#undef GMA_
#undef GPA_
}

int oracle_step_patch(int mx, int my, const double* qpad, double dx, double dy,
                      double dt, double rho, double K, int limiter,
                      int order_trans, double* qout_pad, double* cfl_out) {
  return step2(mx, my, qpad, NULL, dx, dy, dt, rho, K, limiter, order_trans, qout_pad, cfl_out, NULL);
}

int oracle_step_patch_vc(int mx, int my, const double* qpad, const double* auxpad, double dx,
                         double dy, double dt, int limiter, int order_trans, double* qout_pad,
                         double* cfl_out) {
  if (!auxpad) return -1;
  return step2(mx, my, qpad, auxpad, dx, dy, dt, 0.0, 0.0, limiter, order_trans, qout_pad, cfl_out, NULL);
}

/* ------------------------------------------------------------------------ */
/* Level bookkeeping                                                          */
/* ------------------------------------------------------------------------ */

static void free_level(olevel* L) {
  if (L->qpad)
    for (int p = 0; p < L->npatch; ++p) free(L->qpad[p]);
  if (L->qold)
    for (int p = 0; p < L->npatch; ++p) free(L->qold[p]);
  if (L->auxpad)
    for (int p = 0; p < L->npatch; ++p) free(L->auxpad[p]);
  free(L->auxpad);
  free(L->qpad); free(L->qold); free(L->desc); free(L->i0); free(L->j0);
  free(L->pcfl); free(L->bstart); free(L->blist);
  free(L->rcp); free(L->rli); free(L->rlj); free(L->rdir); free(L->rside);
  free(L->rfp); free(L->rfi); free(L->rfj); free(L->racc);
  memset(L, 0, sizeof *L);
}

int oracle_create(const oracle_config* cfg, oracle_ctx** out) {
  if (!cfg || !out) return -1;
  oracle_ctx* c = (oracle_ctx*)calloc(1, sizeof *c);
  c->cfg = *cfg;
  if (!(cfg->xhi > cfg->xlo) || !(cfg->yhi > cfg->ylo)) { free(c); return -1; }
  for (int k = 0; k < 4; ++k)
    if (cfg->bc[k] != 1 && cfg->bc[k] != 2) { free(c); return -1; }
  if ((cfg->bc[0] == 2) != (cfg->bc[1] == 2) || (cfg->bc[2] == 2) != (cfg->bc[3] == 2)) {
    free(c);
    return -1;
  }
  if (cfg->limiter < 0 || cfg->limiter > 4 || cfg->order_trans < 0 || cfg->order_trans > 2) {
    free(c);
    return -1;
  }
  *out = c;
  return 0;
}

int oracle_destroy(oracle_ctx* c) {
  if (!c) return -1;
  for (int l = 0; l <= MAXLEVEL; ++l) {
    free_level(&c->lev[l]);
    free_level(&c->stash[l]);
  }
  free(c);
  return 0;
}

static int find_patch(const olevel* L, int64_t I, int64_t J) {
  if (I < 0 || J < 0 || I >= L->nx || J >= L->ny) return -1;
  const int64_t b = (J / BUCKET) * L->nbx + (I / BUCKET);
  for (int64_t k = L->bstart[b]; k < L->bstart[b + 1]; ++k) {
    const int p = L->blist[k];
    const oracle_patch_desc* d = &L->desc[p];
    if (I >= L->i0[p] && I < L->i0[p] + d->mx && J >= L->j0[p] && J < L->j0[p] + d->my)
      return p;
  }
  return -1;
}

/* Is level-(F-1) cell (Ic,Jc) covered, i.e. are all R x R children interior
 * cells of level F?  (The updating rule of P:120-121.) */
static int covered(const olevel* F, int R, int64_t Ic, int64_t Jc) {
  for (int b = 0; b < R; ++b)
    for (int a = 0; a < R; ++a)
      if (find_patch(F, Ic * R + a, Jc * R + b) < 0) return 0;
  return 1;
}

int oracle_set_reflux(oracle_ctx* c, int on) {
  if (!c) return -1;
  for (int l = 1; l <= MAXLEVEL; ++l)
    if (c->lev[l].npatch) return fail(c, -2, "oracle_set_reflux must precede oracle_set_level");
  c->reflux = on ? 1 : 0;
  return 0;
}

/* Registers of fine level `level` (R17).  Needs the fine patches
 * aligned to the coarse cells (so a coarse cell is covered entirely or not at
 * all and every coarse-fine edge is a fine patch boundary). */
static int build_registers(oracle_ctx* c, int level) {
  olevel* F = &c->lev[level];
  const olevel* C = &c->lev[level - 1];
  const int R = F->ratio_to_coarser;
  const int* bc = c->cfg.bc;
  for (int p = 0; p < F->npatch; ++p)
    if (F->i0[p] % R || F->j0[p] % R || F->desc[p].mx % R || F->desc[p].my % R)
      return fail(c, -1, "conservation fix needs fine patches aligned to the coarse cells");
  for (int pass = 0; pass < 2; ++pass) {
    int n = 0;
    for (int cp = 0; cp < C->npatch; ++cp) {
      const oracle_patch_desc* cd = &C->desc[cp];
      for (int lj = 0; lj < cd->my; ++lj)
        for (int li = 0; li < cd->mx; ++li) {
          const int64_t Ic = C->i0[cp] + li, Jc = C->j0[cp] + lj;
          if (covered(F, R, Ic, Jc)) continue;
          /* neighbours in the order x-, x+, y-, y+ */
          for (int e = 0; e < 4; ++e) {
            const int dir = e / 2, side = (e % 2 == 0) ? 1 : 0;  /* neighbour below/left: C is on the high side */
            int64_t In = Ic + (dir == 0 ? (e % 2 ? 1 : -1) : 0);
            int64_t Jn = Jc + (dir == 1 ? (e % 2 ? 1 : -1) : 0);
            const int64_t n_ax = dir == 0 ? C->nx : C->ny;
            const int64_t v = dir == 0 ? In : Jn;
            if (v < 0 || v >= n_ax) {
              if (bc[2 * dir] != 2) continue; /* physical boundary: no neighbour */
              if (dir == 0) In = (In + C->nx) % C->nx; else Jn = (Jn + C->ny) % C->ny;
            }
            if (!covered(F, R, In, Jn)) continue;
            if (pass == 1) {
              /* first fine cell adjacent to E on the neighbour's side */
              int64_t I, J;
              if (dir == 0) { I = In * R + (side == 0 ? 0 : R - 1); J = Jc * R; }
              else          { I = Ic * R; J = Jn * R + (side == 0 ? 0 : R - 1); }
              const int fp = find_patch(F, I, J);
              F->rcp[n] = cp; F->rli[n] = li; F->rlj[n] = lj;
              F->rdir[n] = dir; F->rside[n] = side;
              F->rfp[n] = fp;
              F->rfi[n] = (int)(I - F->i0[fp]);
              F->rfj[n] = (int)(J - F->j0[fp]);
            }
            ++n;
          }
        }
    }
    if (pass == 0) {
      F->nreg = n;
      const size_t k = (size_t)(n > 0 ? n : 1);
      F->rcp = (int*)malloc(k * sizeof(int)); F->rli = (int*)malloc(k * sizeof(int));
      F->rlj = (int*)malloc(k * sizeof(int)); F->rdir = (int*)malloc(k * sizeof(int));
      F->rside = (int*)malloc(k * sizeof(int)); F->rfp = (int*)malloc(k * sizeof(int));
      F->rfi = (int*)malloc(k * sizeof(int)); F->rfj = (int*)malloc(k * sizeof(int));
      F->racc = (double*)calloc(k * MEQN, sizeof(double));
    }
  }
  return 0;
}

static int set_level_impl(oracle_ctx* c, int level, int npatch, const oracle_patch_desc* descs,
                          const double* q0, int keep_stash);

int oracle_set_level(oracle_ctx* c, int level, int npatch,
                     const oracle_patch_desc* descs, const double* q0) {
  return set_level_impl(c, level, npatch, descs, q0, 0);
}

static int set_level_impl(oracle_ctx* c, int level, int npatch, const oracle_patch_desc* descs,
                          const double* q0, int keep_stash) {
  if (!c || level < 1 || level > MAXLEVEL || npatch < 1 || !descs)
    return fail(c, -1, "bad arguments");
  if (level > 1 && c->lev[level - 1].npatch == 0)
    return fail(c, -2, "coarser level not set");
  if (level > 1 && c->lev[1].auxpad)
    return fail(c, -1, "variable media (oracle_set_aux) are single-level (DESIGN.md R20)");
  olevel* L = &c->lev[level];
  free_level(L);
  L->npatch = npatch;
  L->desc = (oracle_patch_desc*)malloc(sizeof(oracle_patch_desc) * npatch);
  memcpy(L->desc, descs, sizeof(oracle_patch_desc) * npatch);
  L->dx = descs[0].dx;
  L->dy = descs[0].dy;
  L->nx = llround((c->cfg.xhi - c->cfg.xlo) / L->dx);
  L->ny = llround((c->cfg.yhi - c->cfg.ylo) / L->dy);
  if (level > 1) {
    L->ratio_to_coarser = (int)llround(c->lev[level - 1].dx / L->dx);
    if (L->ratio_to_coarser < 1) return fail(c, -1, "bad refinement ratio");
  }
  L->i0 = (int64_t*)malloc(sizeof(int64_t) * npatch);
  L->j0 = (int64_t*)malloc(sizeof(int64_t) * npatch);
  for (int p = 0; p < npatch; ++p) {
    const oracle_patch_desc* d = &descs[p];
    if (d->mx < 1 || d->my < 1 || d->mbc != 2 || !(d->rho > 0) || !(d->K > 0) ||
        d->dx != L->dx || d->dy != L->dy)
      return fail(c, -1, "bad patch descriptor");
    const double fi = (d->xlower - c->cfg.xlo) / L->dx, fj = (d->ylower - c->cfg.ylo) / L->dy;
    L->i0[p] = llround(fi);
    L->j0[p] = llround(fj);
    if (fabs(fi - (double)L->i0[p]) > 1e-6 || fabs(fj - (double)L->j0[p]) > 1e-6)
      return fail(c, -1, "patch not aligned to the level grid");
    if (L->i0[p] < 0 || L->j0[p] < 0 || L->i0[p] + d->mx > L->nx || L->j0[p] + d->my > L->ny)
      return fail(c, -1, "patch outside the domain");
  }
  /* bucket grid */
  L->nbx = (L->nx + BUCKET - 1) / BUCKET;
  L->nby = (L->ny + BUCKET - 1) / BUCKET;
  const int64_t nb = L->nbx * L->nby;
  L->bstart = (int64_t*)calloc((size_t)nb + 1, sizeof(int64_t));
  for (int pass = 0; pass < 2; ++pass) {
    int64_t* fillp = NULL;
    if (pass == 1) {
      for (int64_t b = 0; b < nb; ++b) L->bstart[b + 1] += L->bstart[b];
      L->blist = (int*)malloc(sizeof(int) * (size_t)(L->bstart[nb] + 1));
      fillp = (int64_t*)malloc(sizeof(int64_t) * (size_t)nb);
      memcpy(fillp, L->bstart, sizeof(int64_t) * (size_t)nb);
    }
    for (int p = 0; p < npatch; ++p) {
      const int64_t bx0 = L->i0[p] / BUCKET, bx1 = (L->i0[p] + descs[p].mx - 1) / BUCKET;
      const int64_t by0 = L->j0[p] / BUCKET, by1 = (L->j0[p] + descs[p].my - 1) / BUCKET;
      for (int64_t by = by0; by <= by1; ++by)
        for (int64_t bx = bx0; bx <= bx1; ++bx) {
          const int64_t b = by * L->nbx + bx;
          if (pass == 0) L->bstart[b + 1] += 1;
          else L->blist[fillp[b]++] = p;
        }
    }
    free(fillp);
  }
  /* same-level overlap check */
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t k = L->bstart[b]; k < L->bstart[b + 1]; ++k)
      for (int64_t k2 = k + 1; k2 < L->bstart[b + 1]; ++k2) {
        const int p = L->blist[k], q = L->blist[k2];
        if (L->i0[p] < L->i0[q] + descs[q].mx && L->i0[q] < L->i0[p] + descs[p].mx &&
            L->j0[p] < L->j0[q] + descs[q].my && L->j0[q] < L->j0[p] + descs[p].my)
          return fail(c, -1, "same-level patches overlap");
      }
  if (level == 1) {
    int64_t cells = 0;
    for (int p = 0; p < npatch; ++p) cells += (int64_t)descs[p].mx * descs[p].my;
    if (cells != L->nx * L->ny) return fail(c, -1, "level 1 does not tile the domain");
  }
  L->qpad = (double**)calloc(npatch, sizeof(double*));
  L->qold = (double**)calloc(npatch, sizeof(double*));
  L->pcfl = (double*)calloc(npatch, sizeof(double));
  size_t off = 0;
  for (int p = 0; p < npatch; ++p) {
    const int mx = descs[p].mx, my = descs[p].my;
    const size_t plane = (size_t)(mx + 4) * (my + 4);
    L->qpad[p] = (double*)calloc(MEQN * plane, sizeof(double));
    L->qold[p] = (double*)calloc((size_t)MEQN * mx * my, sizeof(double));
    if (q0) {
      for (int m = 0; m < MEQN; ++m)
        for (int j = 0; j < my; ++j)
          for (int i = 0; i < mx; ++i)
            L->qpad[p][m * plane + (size_t)(j + 2) * (mx + 4) + i + 2] =
                q0[off + ((size_t)m * my + j) * mx + i];
      memcpy(L->qold[p], q0 + off, sizeof(double) * MEQN * mx * my);
    }
    off += (size_t)MEQN * mx * my;
  }
  L->t_old = L->t_new = (level > 1) ? c->lev[level - 1].t_old : 0.0;
  for (int l = level + 1; l <= MAXLEVEL; ++l) free_level(&c->lev[l]);
  if (!keep_stash)
    for (int l = level; l <= MAXLEVEL; ++l) free_level(&c->stash[l]);
  if (level > 1 && c->reflux) return build_registers(c, level);
  return 0;
}

/* Value of component m of coarse level cell (I,J) (already inside the domain)
 * at the time-interpolation weight alpha.  Returns 0 if no patch holds it. */
static int coarse_value(const olevel* C, int64_t I, int64_t J, double alpha, double* v) {
  const int p = find_patch(C, I, J);
  if (p < 0) return 0;
  const oracle_patch_desc* d = &C->desc[p];
  const int li = (int)(I - C->i0[p]), lj = (int)(J - C->j0[p]);
  const size_t plane = (size_t)(d->mx + 4) * (d->my + 4);
  for (int m = 0; m < MEQN; ++m) {
    const double qn = C->qpad[p][m * plane + (size_t)(lj + 2) * (d->mx + 4) + li + 2];
    const double qo = C->qold[p][((size_t)m * d->my + lj) * d->mx + li];
    v[m] = (1.0 - alpha) * qo + alpha * qn;
  }
  return 1;
}

static int64_t map_axis(int64_t I, int64_t n, int bc_lo, int bc_hi) {
  if (I < 0) return (bc_lo == 2) ? ((I % n) + n) % n : 0;
  if (I >= n) return (bc_hi == 2) ? I % n : n - 1;
  return I;
}

int oracle_fill_ghost(oracle_ctx* c, int level, double t) {
  if (!c || level < 1 || level > MAXLEVEL || c->lev[level].npatch == 0)
    return fail(c, -2, "level not set");
  olevel* L = &c->lev[level];
  const olevel* C = (level > 1) ? &c->lev[level - 1] : NULL;
  double alpha = 0.0;
  if (C && C->t_new > C->t_old) alpha = (t - C->t_old) / (C->t_new - C->t_old);
  const int* bc = c->cfg.bc;
  int status = 0;
#pragma omp parallel for schedule(dynamic, 4) num_threads(NTHREADS(c))
  for (int p = 0; p < L->npatch; ++p) {
    const oracle_patch_desc* d = &L->desc[p];
    const int mx = d->mx, my = d->my, PX = mx + 4;
    const size_t plane = (size_t)PX * (my + 4);
    double* q = L->qpad[p];
    for (int j = -1; j <= my + 2; ++j)
      for (int i = -1; i <= mx + 2; ++i) {
        if (i >= 1 && i <= mx && j >= 1 && j <= my) continue; /* interior */
        const int64_t I = map_axis(L->i0[p] + i - 1, L->nx, bc[0], bc[1]);
        const int64_t J = map_axis(L->j0[p] + j - 1, L->ny, bc[2], bc[3]);
        double v[MEQN];
        const int src = find_patch(L, I, J);
        if (src >= 0) { /* case 1+2: physical BC mapping, then same-level copy */
          const oracle_patch_desc* sd = &L->desc[src];
          const size_t splane = (size_t)(sd->mx + 4) * (sd->my + 4);
          const int li = (int)(I - L->i0[src]), lj = (int)(J - L->j0[src]);
          for (int m = 0; m < MEQN; ++m)
            v[m] = L->qpad[src][m * splane + (size_t)(lj + 2) * (sd->mx + 4) + li + 2];
        } else if (C) { /* case 3: interpolate from the coarser level */
          const int R = L->ratio_to_coarser;
          const int64_t Ic = I / R, Jc = J / R;
          double vc[MEQN], vxm[MEQN], vxp[MEQN], vym[MEQN], vyp[MEQN];
          int ok = coarse_value(C, Ic, Jc, alpha, vc);
          ok &= coarse_value(C, map_axis(Ic - 1, C->nx, bc[0], bc[1]), Jc, alpha, vxm);
          ok &= coarse_value(C, map_axis(Ic + 1, C->nx, bc[0], bc[1]), Jc, alpha, vxp);
          ok &= coarse_value(C, Ic, map_axis(Jc - 1, C->ny, bc[2], bc[3]), alpha, vym);
          ok &= coarse_value(C, Ic, map_axis(Jc + 1, C->ny, bc[2], bc[3]), alpha, vyp);
          if (!ok) {
#pragma omp atomic write
            status = -6;
            continue;
          }
          const double xi = ((double)(I % R) + 0.5) / (double)R - 0.5;
          const double eta = ((double)(J % R) + 0.5) / (double)R - 0.5;
          for (int m = 0; m < MEQN; ++m) {
            double sx = 0.0, sy = 0.0;
            const double dxp = vxp[m] - vc[m], dxm = vc[m] - vxm[m];
            const double dyp = vyp[m] - vc[m], dym = vc[m] - vym[m];
            if (dxp * dxm > 0.0) sx = (dxp > 0.0 ? 1.0 : -1.0) * fmin(fabs(dxp), fabs(dxm));
            if (dyp * dym > 0.0) sy = (dyp > 0.0 ? 1.0 : -1.0) * fmin(fabs(dyp), fabs(dym));
            v[m] = vc[m] + sx * xi + sy * eta;
          }
        } else {
#pragma omp atomic write
          status = -6;
          continue;
        }
        for (int m = 0; m < MEQN; ++m) q[m * plane + (size_t)(j + 1) * PX + i + 1] = v[m];
      }
  }
  if (status) return fail(c, status, "ghost cell with no same-level or coarse donor");
  return 0;
}

/* Variable media (NEXT-4, R20): aux = [patch][2][my][mx] (rho, K per
 * interior cell) for every patch of the single level 1.  The ghost frame of
 * each patch's padded aux is filled once here by the same composite rule as q
 * (BC map per axis, then the same-level cell); the medium does not
 * change in time. */
int oracle_set_aux(oracle_ctx* c, int level, const double* aux) {
  if (!c || level != 1 || c->lev[1].npatch == 0 || !aux)
    return fail(c, -1, "variable media need level 1 set and no finer level (DESIGN.md R20)");
  if (c->lev[2].npatch != 0) return fail(c, -1, "variable media are single-level (DESIGN.md R20)");
  olevel* L = &c->lev[1];
  size_t off = 0;
  for (int p = 0; p < L->npatch; ++p) {
    const size_t n = (size_t)L->desc[p].mx * L->desc[p].my;
    for (size_t k = 0; k < 2 * n; ++k)
      if (!(aux[off + k] > 0.0) || !isfinite(aux[off + k])) return fail(c, -1, "rho, K must be finite and > 0");
    off += 2 * n;
  }
  if (!L->auxpad) L->auxpad = (double**)calloc((size_t)(unsigned)L->npatch, sizeof(double*));
  off = 0;
  for (int p = 0; p < L->npatch; ++p) {
    const int mx = L->desc[p].mx, my = L->desc[p].my;
    const size_t plane = (size_t)(mx + 4) * (my + 4);
    free(L->auxpad[p]);
    L->auxpad[p] = (double*)calloc(2 * plane, sizeof(double));
    for (int k = 0; k < 2; ++k)
      for (int j = 0; j < my; ++j)
        for (int i = 0; i < mx; ++i)
          L->auxpad[p][k * plane + (size_t)(j + 2) * (mx + 4) + i + 2] = aux[off + ((size_t)k * my + j) * mx + i];
    off += (size_t)2 * mx * my;
  }
  const int* bc = c->cfg.bc;
  for (int p = 0; p < L->npatch; ++p) {
    const int mx = L->desc[p].mx, my = L->desc[p].my;
    const size_t plane = (size_t)(mx + 4) * (my + 4);
    for (int j = -1; j <= my + 2; ++j)
      for (int i = -1; i <= mx + 2; ++i) {
        if (i >= 1 && i <= mx && j >= 1 && j <= my) continue;
        const int64_t I = map_axis(L->i0[p] + i - 1, L->nx, bc[0], bc[1]);
        const int64_t J = map_axis(L->j0[p] + j - 1, L->ny, bc[2], bc[3]);
        const int src = find_patch(L, I, J);
        if (src < 0) return fail(c, -6, "aux ghost cell with no same-level donor");
        const oracle_patch_desc* sd = &L->desc[src];
        const size_t splane = (size_t)(sd->mx + 4) * (sd->my + 4);
        const int li = (int)(I - L->i0[src]), lj = (int)(J - L->j0[src]);
        for (int k = 0; k < 2; ++k)
          L->auxpad[p][k * plane + (size_t)(j + 1) * (mx + 4) + i + 1] =
              L->auxpad[src][k * splane + (size_t)(lj + 2) * (sd->mx + 4) + li + 2];
      }
  }
  return 0;
}

/* Edge-array entry (component m, Clawpack index i, j) of a patch's flux arrays. */
static double edge(double* const* fl, int k, const oracle_patch_desc* d, int m, int i, int j) {
  const size_t plane = (size_t)(d->mx + 4) * (d->my + 4);
  return fl[k][m * plane + (size_t)(j + 1) * (d->mx + 4) + i + 1];
}

/* Coarse part of the registers of fine level `level` after level-1 advanced
 * by dt with edge arrays cfl_[p] (Step A; terms eq:c2_3 and eq:c3_3).
 * C left/below E: C's update used -dt/dx fm(E)  -> acc += dt/dx fm(E);
 * C right/above E: C's update used +dt/dx fp(E) -> acc -= dt/dx fp(E). */
static void reflux_coarse_part(oracle_ctx* c, int level, double dt, double** const* cfl_) {
  olevel* F = &c->lev[level];
  const olevel* C = &c->lev[level - 1];
  for (int e = 0; e < F->nreg; ++e) {
    const int cp = F->rcp[e], i = F->rli[e] + 1, j = F->rlj[e] + 1; /* Clawpack index of C */
    const oracle_patch_desc* d = &C->desc[cp];
    const double r = (F->rdir[e] == 0) ? dt / C->dx : dt / C->dy;
    for (int m = 0; m < MEQN; ++m) {
      double v;
      if (F->rdir[e] == 0)
        v = (F->rside[e] == 0) ? edge(cfl_[cp], 0, d, m, i + 1, j) : -edge(cfl_[cp], 1, d, m, i, j);
      else
        v = (F->rside[e] == 0) ? edge(cfl_[cp], 2, d, m, i, j + 1) : -edge(cfl_[cp], 3, d, m, i, j);
      F->racc[e * MEQN + m] = F->racc[e * MEQN + m] + r * v;
    }
  }
}

/* Fine part after level `level` advanced by dt_f with edge arrays ffl[p]
 * (Step B; terms eq:c1_1/c1_2, eq:c2_1/c2_2, eq:c3_1/c3_2).  For each
 * of the R fine cells F along E, with fine state Qf at the start of this fine
 * step and the coarse state Qc = Q_C^n at the start of the coarse step:
 *   jump = A-dq + A+dq of the Riemann problem between Qc and Qf,
 *          = f(right state) - f(left state);
 *   C left/below E (F on the right): F's update used +dt_f/dx_f fp(e), so
 *          acc -= (dt_f/dx_c)(1/R) (fp(e) + f(Qf) - f(Qc));
 *   C right/above E (F on the left): acc += (dt_f/dx_c)(1/R) (fm(e) + f(Qf) - f(Qc)).
 * (R17 derives these from "the coarse flux through E is replaced by
 * the space-time average of the fine fluxes".) */
static void reflux_fine_part(oracle_ctx* c, int level, double dt, double** const* ffl) {
  olevel* F = &c->lev[level];
  const olevel* C = &c->lev[level - 1];
  const int R = F->ratio_to_coarser;
  for (int e = 0; e < F->nreg; ++e) {
    const int dir = F->rdir[e], side = F->rside[e];
    const oracle_patch_desc* cd = &C->desc[F->rcp[e]];
    const oracle_patch_desc* fd = &F->desc[F->rfp[e]];
    const double w = ((dir == 0) ? dt / C->dx : dt / C->dy) / (double)R;
    double qc[MEQN];
    for (int m = 0; m < MEQN; ++m)
      qc[m] = C->qold[F->rcp[e]][((size_t)m * cd->my + F->rlj[e]) * cd->mx + F->rli[e]];
    for (int b = 0; b < R; ++b) {
      const int fi = F->rfi[e] + (dir == 1 ? b : 0), fj = F->rfj[e] + (dir == 0 ? b : 0);
      double qf[MEQN], wv[MWAVES * MEQN], sp[MWAVES], am[MEQN], ap[MEQN];
      for (int m = 0; m < MEQN; ++m)
        qf[m] = F->qold[F->rfp[e]][((size_t)m * fd->my + fj) * fd->mx + fi];
      if (side == 0) oracle_rpn2(dir + 1, qc, qf, fd->rho, fd->K, wv, sp, am, ap);
      else           oracle_rpn2(dir + 1, qf, qc, fd->rho, fd->K, wv, sp, am, ap);
      const int i = fi + 1, j = fj + 1; /* Clawpack index of F */
      for (int m = 0; m < MEQN; ++m) {
        const double jump = am[m] + ap[m];
        double v;
        if (side == 0) {
          const double fl = (dir == 0) ? edge(ffl[F->rfp[e]], 1, fd, m, i, j) : edge(ffl[F->rfp[e]], 3, fd, m, i, j);
          v = -(fl + jump);
        } else {
          const double fl = (dir == 0) ? edge(ffl[F->rfp[e]], 0, fd, m, i + 1, j) : edge(ffl[F->rfp[e]], 2, fd, m, i, j + 1);
          v = fl - jump;
        }
        F->racc[e * MEQN + m] = F->racc[e * MEQN + m] + w * v;
      }
    }
  }
}

int oracle_advance_level(oracle_ctx* c, int level, double dt, double* cfl_max) {
  if (!c || level < 1 || level > MAXLEVEL || c->lev[level].npatch == 0)
    return fail(c, -2, "level not set");
  for (int l = 1; l <= MAXLEVEL; ++l) free_level(&c->stash[l]);  /* stale once time moves */
  olevel* L = &c->lev[level];
  const int fine_part = c->reflux && level > 1 && L->nreg > 0;
  const int coarse_part = c->reflux && level < MAXLEVEL && c->lev[level + 1].nreg > 0;
  double*** fl = (fine_part || coarse_part) ? (double***)calloc(L->npatch, sizeof(double**)) : NULL;
  int status = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(NTHREADS(c))
  for (int p = 0; p < L->npatch; ++p) {
    const oracle_patch_desc* d = &L->desc[p];
    const int mx = d->mx, my = d->my;
    const size_t plane = (size_t)(mx + 4) * (my + 4);
    double* qn = (double*)malloc(MEQN * plane * sizeof(double));
    double cfl = 0.0;
    if (fl) fl[p] = (double**)calloc(4, sizeof(double*));
    if (step2(mx, my, L->qpad[p], L->auxpad ? L->auxpad[p] : NULL, d->dx, d->dy, dt, d->rho, d->K,
              c->cfg.limiter, c->cfg.order_trans, qn, &cfl, fl ? fl[p] : NULL) != 0) {
#pragma omp atomic write
      status = -1;
    }
    for (int m = 0; m < MEQN; ++m)
      for (int j = 0; j < my; ++j)
        for (int i = 0; i < mx; ++i)
          L->qold[p][((size_t)m * my + j) * mx + i] =
              L->qpad[p][m * plane + (size_t)(j + 2) * (mx + 4) + i + 2];
    memcpy(L->qpad[p], qn, MEQN * plane * sizeof(double));
    free(qn);
    L->pcfl[p] = cfl;
  }
  if (fl) {
    if (!status && fine_part) reflux_fine_part(c, level, dt, (double** const*)fl);
    if (!status && coarse_part) reflux_coarse_part(c, level + 1, dt, (double** const*)fl);
    for (int p = 0; p < L->npatch; ++p) {
      for (int k = 0; k < 4 && fl[p]; ++k) free(fl[p][k]);
      free(fl[p]);
    }
    free(fl);
  }
  if (status) return fail(c, status, "step failed");
  double cmax = 0.0;
  for (int p = 0; p < L->npatch; ++p) cmax = fmax(cmax, L->pcfl[p]);
  L->t_old = L->t_new;
  L->t_new = L->t_new + dt;
  *cfl_max = cmax;
  return 0;
}

int oracle_update_level(oracle_ctx* c, int level) {
  if (!c || level < 2 || level > MAXLEVEL || c->lev[level].npatch == 0 || c->lev[level - 1].npatch == 0)
    return fail(c, -2, "update needs a fine level >= 2 and its coarser level");
  olevel* F = &c->lev[level];
  olevel* C = &c->lev[level - 1];
  if (fabs(F->t_new - C->t_new) > 1e-12 * fmax(1.0, fabs(C->t_new)))
    return fail(c, -2, "update: fine and coarse levels are not at the same time");
  const int R = F->ratio_to_coarser;
  /* For every coarse cell of every coarse patch: if all R x R children are
   * interior cells of the fine level, replace the coarse value by their mean. */
  for (int cp = 0; cp < C->npatch; ++cp) {
    const oracle_patch_desc* cd = &C->desc[cp];
    const size_t cplane = (size_t)(cd->mx + 4) * (cd->my + 4);
    for (int lj = 0; lj < cd->my; ++lj)
      for (int li = 0; li < cd->mx; ++li) {
        const int64_t Ic = C->i0[cp] + li, Jc = C->j0[cp] + lj;
        double v[MEQN] = {0.0, 0.0, 0.0};
        int all = 1;
        for (int b = 0; b < R && all; ++b)
          for (int a = 0; a < R && all; ++a) {
            const int64_t I = Ic * R + a, J = Jc * R + b;
            const int fp = find_patch(F, I, J);
            if (fp < 0) { all = 0; break; }
            const oracle_patch_desc* fd = &F->desc[fp];
            const size_t fplane = (size_t)(fd->mx + 4) * (fd->my + 4);
            const int fi = (int)(I - F->i0[fp]), fj = (int)(J - F->j0[fp]);
            for (int m = 0; m < MEQN; ++m)
              v[m] = v[m] + F->qpad[fp][m * fplane + (size_t)(fj + 2) * (fd->mx + 4) + fi + 2];
          }
        if (!all) continue;
        for (int m = 0; m < MEQN; ++m)
          C->qpad[cp][m * cplane + (size_t)(lj + 2) * (cd->mx + 4) + li + 2] = v[m] / (double)(R * R);
      }
  }
  /* Conservation fix (Step 7 of the paper's flow chart): add each
   * register to its coarse cell, then clear it for the next coarse step. */
  if (c->reflux)
    for (int e = 0; e < F->nreg; ++e) {
      const int cp = F->rcp[e];
      const oracle_patch_desc* cd = &C->desc[cp];
      const size_t cplane = (size_t)(cd->mx + 4) * (cd->my + 4);
      for (int m = 0; m < MEQN; ++m) {
        double* q = &C->qpad[cp][m * cplane + (size_t)(F->rlj[e] + 2) * (cd->mx + 4) + F->rli[e] + 2];
        *q = *q + F->racc[e * MEQN + m];
        F->racc[e * MEQN + m] = 0.0;
      }
    }
  return 0;
}

int oracle_reflux_count(const oracle_ctx* c, int level) {
  if (!c || level < 2 || level > MAXLEVEL) return -1;
  return c->lev[level].nreg;
}

int oracle_reflux_read(const oracle_ctx* c, int level, int32_t* edges, double* acc) {
  if (!c || level < 2 || level > MAXLEVEL) return -1;
  const olevel* F = &c->lev[level];
  for (int e = 0; e < F->nreg; ++e) {
    if (edges) {
      int32_t* r = edges + 8 * e;
      r[0] = F->rcp[e]; r[1] = F->rli[e]; r[2] = F->rlj[e]; r[3] = F->rdir[e];
      r[4] = F->rside[e]; r[5] = F->rfp[e]; r[6] = F->rfi[e]; r[7] = F->rfj[e];
    }
    if (acc)
      for (int m = 0; m < MEQN; ++m) acc[e * MEQN + m] = F->racc[e * MEQN + m];
  }
  return 0;
}

int oracle_read(const oracle_ctx* c, int level, int patch, double* q_out) {
  if (!c || level < 1 || level > MAXLEVEL || patch < 0 || patch >= c->lev[level].npatch) return -1;
  const olevel* L = &c->lev[level];
  const int mx = L->desc[patch].mx, my = L->desc[patch].my;
  const size_t plane = (size_t)(mx + 4) * (my + 4);
  for (int m = 0; m < MEQN; ++m)
    for (int j = 0; j < my; ++j)
      for (int i = 0; i < mx; ++i)
        q_out[((size_t)m * my + j) * mx + i] = L->qpad[patch][m * plane + (size_t)(j + 2) * (mx + 4) + i + 2];
  return 0;
}

int oracle_write(oracle_ctx* c, int level, int patch, const double* q_in) {
  if (!c || level < 1 || level > MAXLEVEL || patch < 0 || patch >= c->lev[level].npatch) return -1;
  olevel* L = &c->lev[level];
  const int mx = L->desc[patch].mx, my = L->desc[patch].my;
  const size_t plane = (size_t)(mx + 4) * (my + 4);
  for (int m = 0; m < MEQN; ++m)
    for (int j = 0; j < my; ++j)
      for (int i = 0; i < mx; ++i)
        L->qpad[patch][m * plane + (size_t)(j + 2) * (mx + 4) + i + 2] = q_in[((size_t)m * my + j) * mx + i];
  return 0;
}

int oracle_read_padded(const oracle_ctx* c, int level, int patch, double* q_out) {
  if (!c || level < 1 || level > MAXLEVEL || patch < 0 || patch >= c->lev[level].npatch) return -1;
  const olevel* L = &c->lev[level];
  const size_t n = (size_t)MEQN * (L->desc[patch].mx + 4) * (L->desc[patch].my + 4);
  memcpy(q_out, L->qpad[patch], n * sizeof(double));
  return 0;
}

int oracle_patch_cfl(const oracle_ctx* c, int level, int patch, double* cfl) {
  if (!c || level < 1 || level > MAXLEVEL || patch < 0 || patch >= c->lev[level].npatch) return -1;
  *cfl = c->lev[level].pcfl[patch];
  return 0;
}

int oracle_level_time(const oracle_ctx* c, int level, double* t_old, double* t_new) {
  if (!c || level < 1 || level > MAXLEVEL || c->lev[level].npatch == 0) return -1;
  *t_old = c->lev[level].t_old;
  *t_new = c->lev[level].t_new;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Regridding (NEXT-3; R18)                  */
/* ------------------------------------------------------------------------ */

/* Flag every interior cell of `level` whose pressure differs from one of its
 * four edge neighbours (composite values: the ghost frames as filled) by more
 * than tol (undivided gradient of the first component; the paper
 * allows "the gradient").  flags[J*nx + I] over the level's index
 * space; cells outside the level's patches stay 0. */
int oracle_flag(oracle_ctx* c, int level, double tol, uint8_t* flags) {
  if (!c || level < 1 || level > MAXLEVEL || c->lev[level].npatch == 0 || !flags)
    return fail(c, -2, "level not set");
  const olevel* L = &c->lev[level];
  memset(flags, 0, (size_t)(L->nx * L->ny));
  for (int p = 0; p < L->npatch; ++p) {
    const oracle_patch_desc* d = &L->desc[p];
    const int PX = d->mx + 4;
    const double* q = L->qpad[p];
    for (int j = 1; j <= d->my; ++j)
      for (int i = 1; i <= d->mx; ++i) {
        const double pc = q[(size_t)(j + 1) * PX + i + 1];
        const double pn[4] = {q[(size_t)(j + 1) * PX + i], q[(size_t)(j + 1) * PX + i + 2],
                              q[(size_t)j * PX + i + 1], q[(size_t)(j + 2) * PX + i + 1]};
        double g = 0.0;
        for (int k = 0; k < 4; ++k) g = fmax(g, fabs(pn[k] - pc));
        if (g > tol) flags[(L->j0[p] + j - 1) * L->nx + (L->i0[p] + i - 1)] = 1;
      }
  }
  return 0;
}

/* Chebyshev dilation by b cells, clipped to [0,nx) x [0,ny) and,
 * if mask is not NULL, to cells with mask != 0. */
void oracle_buffer_flags(const uint8_t* in, int64_t nx, int64_t ny, int b, const uint8_t* mask,
                         uint8_t* out) {
  for (int64_t J = 0; J < ny; ++J)
    for (int64_t I = 0; I < nx; ++I) {
      uint8_t v = 0;
      for (int64_t dj = -b; dj <= b && !v; ++dj)
        for (int64_t di = -b; di <= b && !v; ++di) {
          const int64_t a = I + di, bb = J + dj;
          if (a >= 0 && a < nx && bb >= 0 && bb < ny && in[bb * nx + a]) v = 1;
        }
      if (mask && !mask[J * nx + I]) v = 0;
      out[J * nx + I] = v;
    }
}

/* Berger-Rigoutsos clustering (reading R18), recursive:
 *   1. shrink the box to the bounding box of its flags (none: no box);
 *   2. accept if efficiency = flags/area >= cutoff and both sides <= max_dim;
 *   3. otherwise cut, trying in order
 *        a. a zero of the column / row flag signature (a hole),
 *        b. the strongest inflection of the signature's second difference
 *           (largest |D2[k] - D2[k-1]| where D2 changes sign),
 *        c. the middle of the longer side;
 *      a cut at k splits [lo, k) | [k, hi) and must leave both parts at least
 *      min_dim wide; for a and b the longer side is tried first, candidates
 *      closest to the box centre win, ties to the lower index; if no cut is
 *      allowed the box is accepted;
 *   4. recurse on the low part, then the high part. */
typedef struct { int32_t* out; int cap, n; const uint8_t* f; int64_t nx; double cutoff; int maxd, mind; } br_ctx;

static void br_rec(br_ctx* B, int64_t x0, int64_t y0, int64_t x1, int64_t y1) {
  /* 1. shrink */
  int64_t a0 = x1, a1 = x0 - 1, b0 = y1, b1 = y0 - 1, nf = 0;
  for (int64_t J = y0; J < y1; ++J)
    for (int64_t I = x0; I < x1; ++I)
      if (B->f[J * B->nx + I]) {
        if (I < a0) a0 = I;
        if (I > a1) a1 = I;
        if (J < b0) b0 = J;
        if (J > b1) b1 = J;
        ++nf;
      }
  if (nf == 0) return;
  x0 = a0; x1 = a1 + 1; y0 = b0; y1 = b1 + 1;
  const int64_t w = x1 - x0, h = y1 - y0;
  /* 2. accept */
  if ((double)nf / (double)(w * h) >= B->cutoff && w <= B->maxd && h <= B->maxd) {
    if (B->n < B->cap) {
      B->out[4 * B->n + 0] = (int32_t)x0; B->out[4 * B->n + 1] = (int32_t)y0;
      B->out[4 * B->n + 2] = (int32_t)w;  B->out[4 * B->n + 3] = (int32_t)h;
    }
    B->n++;
    return;
  }
  /* signatures */
  int64_t* sx = (int64_t*)calloc((size_t)w, sizeof(int64_t));
  int64_t* sy = (int64_t*)calloc((size_t)h, sizeof(int64_t));
  for (int64_t J = y0; J < y1; ++J)
    for (int64_t I = x0; I < x1; ++I)
      if (B->f[J * B->nx + I]) { sx[I - x0]++; sy[J - y0]++; }
  int dirs[2];
  if (w >= h) { dirs[0] = 0; dirs[1] = 1; } else { dirs[0] = 1; dirs[1] = 0; }
  int cut_dir = -1;
  int64_t cut = -1;
  /* a. holes */
  for (int t = 0; t < 2 && cut_dir < 0; ++t) {
    const int d = dirs[t];
    const int64_t n = d == 0 ? w : h;
    const int64_t* sg = d == 0 ? sx : sy;
    int64_t best = -1, bestdist = 0;
    for (int64_t k = 1; k < n; ++k) {
      if (sg[k] != 0) continue;
      if (k < B->mind || n - k < B->mind) continue;
      const int64_t dist = llabs(2 * k - n);  /* twice the distance of the cut from the centre */
      if (best < 0 || dist < bestdist) { best = k; bestdist = dist; }
    }
    if (best >= 0) { cut_dir = d; cut = best; }
  }
  /* b. inflections: D2[k] = s[k-1] - 2 s[k] + s[k+1], k = 1..n-2; a sign
   * change between D2[k-1] and D2[k] gives a cut at k (between cells k-1, k) */
  if (cut_dir < 0) {
    int64_t bestv = -1, bestdist = 0;
    for (int t = 0; t < 2; ++t) {
      const int d = dirs[t];
      const int64_t n = d == 0 ? w : h;
      const int64_t* sg = d == 0 ? sx : sy;
      for (int64_t k = 2; k <= n - 2; ++k) {
        const int64_t dp = sg[k - 2] - 2 * sg[k - 1] + sg[k];
        const int64_t dc = sg[k - 1] - 2 * sg[k] + sg[k + 1];
        if (!((dp < 0 && dc > 0) || (dp > 0 && dc < 0))) continue;
        if (k < B->mind || n - k < B->mind) continue;
        const int64_t v = llabs(dc - dp);
        const int64_t dist = llabs(2 * k - n);
        if (v > bestv || (v == bestv && dist < bestdist)) { bestv = v; bestdist = dist; cut_dir = d; cut = k; }
      }
    }
  }
  /* c. bisect the longer side */
  if (cut_dir < 0) {
    const int d = dirs[0];
    const int64_t n = d == 0 ? w : h;
    const int64_t k = n / 2;
    if (k >= B->mind && n - k >= B->mind) { cut_dir = d; cut = k; }
  }
  free(sx);
  free(sy);
  if (cut_dir < 0) { /* no admissible cut: accept */
    if (B->n < B->cap) {
      B->out[4 * B->n + 0] = (int32_t)x0; B->out[4 * B->n + 1] = (int32_t)y0;
      B->out[4 * B->n + 2] = (int32_t)w;  B->out[4 * B->n + 3] = (int32_t)h;
    }
    B->n++;
    return;
  }
  if (cut_dir == 0) {
    br_rec(B, x0, y0, x0 + cut, y1);
    br_rec(B, x0 + cut, y0, x1, y1);
  } else {
    br_rec(B, x0, y0, x1, y0 + cut);
    br_rec(B, x0, y0 + cut, x1, y1);
  }
}

int oracle_cluster(const uint8_t* flags, int64_t nx, int64_t ny, double cutoff, int max_dim,
                   int min_dim, int32_t* boxes, int cap, int* nbox) {
  if (!flags || nx < 1 || ny < 1 || !(cutoff > 0.0) || cutoff > 1.0 || max_dim < 1 || min_dim < 1 ||
      2 * min_dim > max_dim || !nbox)
    return -1;
  br_ctx B = {boxes, boxes ? cap : 0, 0, flags, nx, cutoff, max_dim, min_dim};
  br_rec(&B, 0, 0, nx, ny);
  *nbox = B.n;
  return (boxes && B.n > cap) ? -3 : 0;
}

/* Replace level+1 by patches = boxes (in level-`level` index space) refined by
 * R.  New fine cells take the value of the old level+1 cell at the same place
 * if there is one ("copy from overlapping old same-level patches"), else
 * the R10 interpolation from `level` at its current time (the ghost-fill
 * formula with alpha = 1).  Levels finer than level+1 are discarded. */
int oracle_regrid(oracle_ctx* c, int level, int nbox, const int32_t* boxes, int R) {
  if (!c || level < 1 || level >= MAXLEVEL || c->lev[level].npatch == 0 || nbox < 0 || R < 1)
    return fail(c, -1, "bad regrid arguments");
  olevel* C = &c->lev[level];
  /* the old fine level: the current level+1, else the one a regrid of a
   * coarser level discarded just before (R18: a regrid of levels 1, 2, ...
   * in turn copies every level's old data) */
  olevel old;
  if (c->lev[level + 1].npatch) {
    old = c->lev[level + 1];
    memset(&c->lev[level + 1], 0, sizeof(olevel));
    free_level(&c->stash[level + 1]);
  } else {
    old = c->stash[level + 1];
    memset(&c->stash[level + 1], 0, sizeof(olevel));
  }
  if (old.npatch && nbox > 0 && (int)(C->dx / old.dx + 0.5) != R) {
    free_level(&old);
    return fail(c, -1, "regrid: R differs from the old fine level's ratio");
  }
  for (int l = level + 2; l <= MAXLEVEL; ++l) { /* discarded levels become copy sources */
    if (c->lev[l].npatch) {
      free_level(&c->stash[l]);
      c->stash[l] = c->lev[l];
      memset(&c->lev[l], 0, sizeof(olevel));
    }
  }
  int rc = 0;
  if (nbox > 0) {
    const double dxf = C->dx / R, dyf = C->dy / R;
    oracle_patch_desc* d = (oracle_patch_desc*)calloc((size_t)nbox, sizeof(oracle_patch_desc));
    int64_t ncell = 0;
    for (int b = 0; b < nbox; ++b) {
      d[b].mx = boxes[4 * b + 2] * R;
      d[b].my = boxes[4 * b + 3] * R;
      d[b].dx = dxf;
      d[b].dy = dyf;
      d[b].xlower = c->cfg.xlo + (double)(boxes[4 * b + 0] * R) * dxf;
      d[b].ylower = c->cfg.ylo + (double)(boxes[4 * b + 1] * R) * dyf;
      d[b].mbc = 2;
      d[b].rho = C->desc[0].rho;
      d[b].K = C->desc[0].K;
      ncell += (int64_t)d[b].mx * d[b].my;
    }
    double* q0 = (double*)calloc((size_t)(3 * ncell), sizeof(double));
    const int* bc = c->cfg.bc;
    int64_t off = 0;
    for (int b = 0; b < nbox && !rc; ++b) {
      const int64_t I0 = (int64_t)boxes[4 * b + 0] * R, J0 = (int64_t)boxes[4 * b + 1] * R;
      for (int j = 0; j < d[b].my && !rc; ++j)
        for (int i = 0; i < d[b].mx; ++i) {
          const int64_t I = I0 + i, J = J0 + j;
          double v[MEQN];
          const int op = old.npatch ? find_patch(&old, I, J) : -1;
          if (op >= 0) {
            const oracle_patch_desc* od = &old.desc[op];
            const size_t plane = (size_t)(od->mx + 4) * (od->my + 4);
            for (int m = 0; m < MEQN; ++m)
              v[m] = old.qpad[op][m * plane + (size_t)(J - old.j0[op] + 2) * (od->mx + 4) + (I - old.i0[op]) + 2];
          } else {
            const int64_t Ic = I / R, Jc = J / R;
            double vc[MEQN], vxm[MEQN], vxp[MEQN], vym[MEQN], vyp[MEQN];
            int ok = coarse_value(C, Ic, Jc, 1.0, vc);
            ok &= coarse_value(C, map_axis(Ic - 1, C->nx, bc[0], bc[1]), Jc, 1.0, vxm);
            ok &= coarse_value(C, map_axis(Ic + 1, C->nx, bc[0], bc[1]), Jc, 1.0, vxp);
            ok &= coarse_value(C, Ic, map_axis(Jc - 1, C->ny, bc[2], bc[3]), 1.0, vym);
            ok &= coarse_value(C, Ic, map_axis(Jc + 1, C->ny, bc[2], bc[3]), 1.0, vyp);
            if (!ok) { rc = fail(c, -6, "regrid: new fine cell not nested in level"); break; }
            const double xi = ((double)(I % R) + 0.5) / (double)R - 0.5;
            const double eta = ((double)(J % R) + 0.5) / (double)R - 0.5;
            for (int m = 0; m < MEQN; ++m) {
              double sx = 0.0, sy = 0.0;
              const double dxp = vxp[m] - vc[m], dxm = vc[m] - vxm[m];
              const double dyp = vyp[m] - vc[m], dym = vc[m] - vym[m];
              if (dxp * dxm > 0.0) sx = (dxp > 0.0 ? 1.0 : -1.0) * fmin(fabs(dxp), fabs(dxm));
              if (dyp * dym > 0.0) sy = (dyp > 0.0 ? 1.0 : -1.0) * fmin(fabs(dyp), fabs(dym));
              v[m] = vc[m] + sx * xi + sy * eta;
            }
          }
          for (int m = 0; m < MEQN; ++m) q0[off + ((int64_t)m * d[b].my + j) * d[b].mx + i] = v[m];
        }
      off += 3 * (int64_t)d[b].mx * d[b].my;
    }
    if (!rc) rc = set_level_impl(c, level + 1, nbox, d, q0, 1);
    free(q0);
    free(d);
  }
  free_level(&old);
  if (!rc && nbox > 0) {
    c->lev[level + 1].t_old = c->lev[level + 1].t_new = C->t_new;
  }
  return rc;
}

int oracle_level_count(const oracle_ctx* c, int level) {
  if (!c || level < 1 || level > MAXLEVEL) return -1;
  return c->lev[level].npatch;
}

int oracle_level_desc(const oracle_ctx* c, int level, oracle_patch_desc* out) {
  if (!c || level < 1 || level > MAXLEVEL || !out) return -1;
  memcpy(out, c->lev[level].desc, sizeof(oracle_patch_desc) * (size_t)c->lev[level].npatch);
  return 0;
}
