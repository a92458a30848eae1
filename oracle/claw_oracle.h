/*
 * claw_oracle.h -- CPU ORACLE for the batched AMR-level advance of
 * arXiv 1808.02638 (Qin, LeVeque & Motley), 2D linear acoustics.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1808_02638_b200/, libclaw.so) never links, loads
 * or calls it, and this oracle shares no code, header, table or constant
 * generator with the CUDA path.
 *
 * What it computes (citations: P:a-b = /root/reference/PAPER.md lines a-b,
 * S:a-b = SPEC.md lines a-b; "Clawpack convention" = readings listed in
 * DESIGN.md section "Readings"):
 *   - eq. (W) (sec. 2.1): unsplit wave-propagation update with
 *     second-order corrections and transverse waves, written in Clawpack's
 *     classic step2 / flux2 / rpn2 / rpt2 / limiter structure;
 *   - the acoustics system q_t + A q_x + B q_y = 0 (sec. 4.1)
 *     solved exactly by rpn2 (normal) and rpt2 (transverse) eigen-splits;
 *   - ghost-cell fill, three cases (sec. 2.2): physical BC,
 *     same-level copy, coarse-level interpolation;
 *   - the CFL number nu = |s dt/dx| (sec. 2.4), maximised over
 *     every swept interface of a patch, then over the level.
 *
 * Arithmetic: IEEE binary64, built with -O2 -ffp-contract=off (no FMA
 * contraction, no fast-math) so every operation is a single rounding in the
 * order written.  OpenMP is used only across patches; each patch is computed
 * sequentially, so results do not depend on the thread count.
 *
 * Storage conventions of this API: a patch's interior is exchanged as
 * [3][my][mx] (component p,u,v; x fastest).  A "padded" patch is
 * [3][my+4][mx+4] including the two-deep ghost frame (mbc = 2).
 *
 * Parity pins for every function here live in tests/test_oracle_*.py.
 */
#ifndef CLAW_ORACLE_H
#define CLAW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Per-patch description, the north_star's descriptor fields. */
typedef struct {
  int32_t mx, my;          /* interior cells */
  double dx, dy;           /* cell sizes (identical for all patches of a level) */
  double xlower, ylower;   /* physical lower-left corner of the interior */
  int32_t mbc;             /* ghost width, must be 2 */
  double rho, K;           /* density, bulk modulus */
} oracle_patch_desc;

typedef struct {
  double xlo, xhi, ylo, yhi; /* physical domain */
  int32_t bc[4];             /* left,right,bottom,top: 1 extrapolation, 2 periodic */
  int32_t limiter;           /* 0 none, 1 minmod, 2 superbee, 3 van Leer, 4 MC */
  int32_t order_trans;       /* 0 none, 1 fluctuations only, 2 incl. corrections */
  int32_t nthreads;          /* OpenMP threads over patches (<=0: runtime default) */
} oracle_config;

typedef struct oracle_ctx oracle_ctx;

/* All calls return 0 on success, <0 on error (message via oracle_last_error). */
int oracle_create(const oracle_config* cfg, oracle_ctx** out);
int oracle_destroy(oracle_ctx* ctx);
const char* oracle_last_error(const oracle_ctx* ctx);

/* Level L = 1..8.  q0 may be NULL (zeros); else [patch][3][my][mx]. */
int oracle_set_level(oracle_ctx* ctx, int level, int npatch,
                     const oracle_patch_desc* descs, const double* q0);

/* Fill every ghost cell (corners included) of every patch of `level` at time t
 * by the composite rule.  t only matters for level > 1 (time
 * interpolation of the coarser level). */
int oracle_fill_ghost(oracle_ctx* ctx, int level, double t);

/* One step of eq. (W) on every patch of `level` with the ghost frames as they
 * stand; returns the level's max Courant number. */
int oracle_advance_level(oracle_ctx* ctx, int level, double dt, double* cfl_max);

/* Updating: every level-(level-1) cell whose R x R
 * children are all interior cells of level `level` is overwritten by their
 * mean (sum over children, rows then columns, divided by R*R; R16).
 * Requires equal times (t_new) on both levels (else -2).  With the
 * conservation fix on, the registers of `level` are then applied (below).
 * Setting a level discards every finer level. */
int oracle_update_level(oracle_ctx* ctx, int level);

/* Conservation fix (R17).  When on
 * (call before the first oracle_set_level), every level L >= 2 keeps one
 * register per coarse-fine edge E (a level L-1 cell C not covered by level L,
 * sharing an edge -- through periodic wrap -- with a covered cell; fine
 * patches must be aligned to the coarse cells, else set_level fails with -1):
 *   - advancing level L-1 by dt adds the coarse flux through E that C's update
 *     used (+dt/dx fm if C lies left/below E, -dt/dx fp otherwise);
 *   - each advance of level L by dt_f subtracts (adds) the fine fluxes through
 *     the R fine edges of E, (dt_f/dx_c)(1/R)(fp + A-dq + A+dq) with the
 *     Riemann problem between Q_C^n and the fine cell (the paper's C1 + C2 +
 *     C3 terms, eq:c123-eq:c3_3);
 *   - oracle_update_level(L) then adds each register to its cell C and clears
 *     it, so the level L-1 total equals the composite total.
 * Protocol: Berger-Oliger order (level L-1 step, then its R level-L steps,
 * then oracle_update_level(L)). */
int oracle_set_reflux(oracle_ctx* ctx, int on);
/* Number of registers of level L (>= 2), or -1. */
int oracle_reflux_count(const oracle_ctx* ctx, int level);
/* Registers of level L: edges[8e..8e+7] = coarse patch, C's local i, j,
 * dir (0 x, 1 y), side (0: C left/below E), fine patch, first fine cell
 * local i, j; acc[3e..3e+2] the accumulated values (either may be NULL). */
int oracle_reflux_read(const oracle_ctx* ctx, int level, int32_t* edges, double* acc);

int oracle_read(const oracle_ctx* ctx, int level, int patch, double* q_out);
int oracle_write(oracle_ctx* ctx, int level, int patch, const double* q_in);
int oracle_read_padded(const oracle_ctx* ctx, int level, int patch, double* q_out);
int oracle_patch_cfl(const oracle_ctx* ctx, int level, int patch, double* cfl);
int oracle_level_time(const oracle_ctx* ctx, int level, double* t_old, double* t_new);

/* The single-patch step itself, exposed for the pins: qpad is [3][my+4][mx+4]
 * with ghosts already set; qout_pad receives the same shape with the interior
 * replaced by q^{n+1} (ghost entries copied through). */
int oracle_step_patch(int mx, int my, const double* qpad, double dx, double dy,
                      double dt, double rho, double K, int limiter,
                      int order_trans, double* qout_pad, double* cfl);

/* Regridding (NEXT-3; "every K time steps ... regenerated", "cells
 * are flagged ... clustered into new rectangular grid patches"; S:219-290;
 * DESIGN.md R18).
 * oracle_flag: flags[J*nx + I] = 1 iff interior cell (I,J) of `level` has a
 *   pressure jump > tol to one of its 4 edge neighbours (ghost frames as
 *   filled by oracle_fill_ghost).
 * oracle_buffer_flags: Chebyshev dilation by b, clipped to the index space
 *   and (mask != NULL) to mask.
 * oracle_cluster: Berger-Rigoutsos boxes (i0, j0, w, h) covering every flag
 *   exactly once; -3 if more than cap boxes (nbox still set).
 * oracle_regrid: replace level+1 by the boxes refined by R; data copied from
 *   the old level+1 where it overlaps, else interpolated from `level` (R10
 *   at alpha = 1); finer levels are discarded but kept as the copy sources of
 *   the regrid that re-creates them next (until any level advances), so a
 *   regrid of levels 1, 2, ... in turn keeps every level's old data; -6 if a
 *   box is not on `level`. */
int oracle_flag(oracle_ctx* ctx, int level, double tol, uint8_t* flags);
void oracle_buffer_flags(const uint8_t* in, int64_t nx, int64_t ny, int b, const uint8_t* mask,
                         uint8_t* out);
int oracle_cluster(const uint8_t* flags, int64_t nx, int64_t ny, double cutoff, int max_dim,
                   int min_dim, int32_t* boxes, int cap, int* nbox);
int oracle_regrid(oracle_ctx* ctx, int level, int nbox, const int32_t* boxes, int R);
int oracle_level_count(const oracle_ctx* ctx, int level);
int oracle_level_desc(const oracle_ctx* ctx, int level, oracle_patch_desc* out);

/* Riemann solvers and limiter function exposed for the pins.
 * ixy = 1 (x) or 2 (y).  ql, qr: 3-vectors.  wave: [2][3], s: [2]. */
void oracle_rpn2(int ixy, const double* ql, const double* qr, double rho,
                 double K, double* wave, double* s, double* amdq, double* apdq);
void oracle_rpt2(int ixy, const double* asdq, double rho, double K,
                 double* bmasdq, double* bpasdq);
double oracle_philim(int limiter, double r);

/* Variable-coefficient acoustics (NEXT-4; heterogeneous media P:66, P:640;
 * normal / transverse solvers per system P:433-436; R20).
 * oracle_set_aux: per-cell media of the single level 1, aux =
 *   [patch][2][my][mx] (rho, K), all > 0; ghost media by the composite rule
 *   (BC map, same-level copy).  A finer level is then refused (-1).
 * oracle_rpn2_vc: interface between a left cell (rhol, Kl) and a right cell
 *   (rhor, Kr): W1 = a1 (-Z_l, 1, 0) at -c_l, W2 = a2 (Z_r, 1, 0) at +c_r
 *   with qr - ql = W1 + W2.
 * oracle_rpt2_vc: asdq entering a cell (rho, K) split into the transmitted
 *   waves across its low (rho_m, K_m) and high (rho_p, K_p) transverse edges.
 * oracle_step_patch_vc: one step with a padded aux [2][my+4][mx+4]. */
int oracle_set_aux(oracle_ctx* ctx, int level, const double* aux);
void oracle_rpn2_vc(int ixy, const double* ql, const double* qr, double rhol, double Kl,
                    double rhor, double Kr, double* wave, double* s, double* amdq, double* apdq);
void oracle_rpt2_vc(int ixy, const double* asdq, double rho_m, double K_m, double rho, double K,
                    double rho_p, double K_p, double* bmasdq, double* bpasdq);
int oracle_step_patch_vc(int mx, int my, const double* qpad, const double* auxpad, double dx,
                         double dy, double dt, int limiter, int order_trans, double* qout_pad,
                         double* cfl);

#ifdef __cplusplus
}
#endif
#endif
