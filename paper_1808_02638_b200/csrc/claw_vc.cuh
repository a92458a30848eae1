// claw_vc.cuh -- fused step kernel for variable-coefficient acoustics
// (NEXT-4; heterogeneous media P:66; the per-system normal and
// transverse Riemann solvers of P:433-436 with the matrices A, B of
// P:457-466 varying per cell; R20).  Included by claw_kernels.cu
// inside its anonymous namespace (shares the march helpers).
//
// Same march as step_grid_kernel (a warp owns a 30-column strip of a uniform
// grid, lane = column, lanes 0 / 31 halo columns, rows through a cp.async
// ring), but every cell carries its medium (Z = rho c, c) from the aux
// buffer ([patch][2][my][mx], same patch layout as q), so
//   * a face's waves are W1 = a1 (-Z_l, 1) at -c_l and W2 = a2 (Z_r, 1) at
//     +c_r with a1 = (-dp + Z_r dn) / (Z_l + Z_r), a2 = (dp + Z_l dn) / (Z_l + Z_r);
//   * theta = <W_up, W> / <W, W> = a_up (Z_up Z_w + 1) / (a (Z_w^2 + 1)), Z_w the
//     impedance in W's eigenvector; phi(theta) a is the constant-coefficient
//     min/max expression of (a, a_up m nu) with m = Z_l Z_r + 1 and
//     nu = 1 / (Z_w^2 + 1) (exact in real arithmetic; the oracle divides);
//   * second-order corrections 1/2 cq = sum_p |s_p| (1 - |s_p| dt/dx) W~_p / 2;
//   * the transverse sum T entering a cell (its A-dq + A+dq, corrections
//     included) is split across its low / high transverse edges with the
//     media of the cells there (the oracle's rpt2_vc), and the two cells
//     sharing an edge combine into one edge flux:
//       G(j+1/2) = sigma (K_{j+1} T_j - K_j T_{j+1},  0,  c_{j+1} T_j + c_j T_{j+1}),
//     sigma = 1 / (Z_j + Z_{j+1}), K = c Z (y-sweep edges likewise along x);
//   * the Courant number is the max over every swept face of max(c_l, c_r)
//     times dt/dx (dt/dy): every cell is a left or right cell of a swept
//     face, so each lane keeps the max c of its column's cells, then warp max
//     and atomicMax.
// Rounding differs from the oracle (FMA, reciprocals, division-free
// limiters, combined transverse splits): parity is by tolerance.

#ifndef CLAW_VC_RES_WARPS
#define CLAW_VC_RES_WARPS 12   // resident warps per SM (168 registers per thread)
#endif
#ifndef CLAW_VC_KW
#define CLAW_VC_KW 1           // warps (consecutive strips of a row block) per CTA (2-4 measured slower:
                               // this kernel is fp64-bound, profiles/r02_vc_rowcopy.txt)
#endif
static_assert(CLAW_VC_RES_WARPS % CLAW_VC_KW == 0, "CLAW_VC_KW must divide CLAW_VC_RES_WARPS");

// q and aux pointers of (level column C, band row Jl = J - Y0) of this rank's
// band (a whole level on one rank)
__device__ __forceinline__ void vc_ptrs(const StepParams& P, int C, int J, const double*& q, const double*& a) {
  const int pc = C / P.mx, li = C - pc * P.mx;
  const int pr = J / P.my, lj = J - pr * P.my;
  const int64_t pid = static_cast<int64_t>(pr) * P.npx + pc;
  const int64_t in = static_cast<int64_t>(lj) * P.mx + li;
  const int64_t plane = static_cast<int64_t>(P.mx) * P.my;
  q = P.q + pid * 3 * plane + in;
  a = P.aux + pid * 2 * plane + in;
}

// 1/x for the positive, normal x of this kernel (impedance sums, Z^2 + 1):
// the SFU's reciprocal estimate (~2^-20 measured) and one cubic step (error ~2^-60,
// i.e. the last bit of the double), no special-case branch; the rounding may
// differ from the correctly rounded __drcp_rn by one ulp (parity is by
// tolerance, R20)
// sources of (column C, level row J) for any row the march reads: the band
// (after the BC map), or -- multi-rank band mode -- one of the four halo
// rows: q from the frame the NCCL receives land in (grid_src's rule), the
// medium from the rank's static copy of those rows (claw_set_aux)
__device__ __forceinline__ void vc_src(const StepParams& P, int C, int J, const double*& q, const double*& a,
                                       int64_t& cq, int64_t& ca) {
  const int Jm = map_idx(J, P.NY, P.per_y);
  if (Jm >= P.Y0 && Jm < P.Y1) {
    vc_ptrs(P, C, Jm - P.Y0, q, a);
    cq = ca = static_cast<int64_t>(P.mx) * P.my;
    return;
  }
  const int kk = (J < P.Y0) ? (J - (P.Y0 - 2)) : (2 + J - P.Y1);
  q = P.frame + P.hoff[kk] + C;
  cq = P.hcs[kk];
  a = P.aux_halo + static_cast<int64_t>(kk) * 2 * P.NX + C;
  ca = P.NX;
}

#ifndef CLAW_VC_RCP3
#define CLAW_VC_RCP3 1
#endif
__device__ __forceinline__ double vc_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = __fma_rn(-x, y, 1.0);
#if CLAW_VC_RCP3
  // one cubic step instead of two Newton steps: with e = 1 - x y0 (exact up
  // to one rounding of a ~2^-22 quantity), 1/x = y0 (1 + e + e^2 + ...), so
  // y0 + y0 (e + e^2) leaves ~e^3 ~ 2^-66 relative before its final rounding
  // -- the accuracy of two Newton steps in three dependent FMAs, not four
  return __fma_rn(y, __fma_rn(e, e, e), y);
#else
  y = __fma_rn(y, e, y);
  e = __fma_rn(-x, y, 1.0);
  return __fma_rn(y, e, y);
#endif
}

// Row copies as in the grid kernel's RC 1: the rows inside the tile of an
// interior strip (all 34 ring columns in the level; wide = the level's rows
// and planes are 16-byte aligned) arrive as 85 16-byte chunks (5 components
// x 17 column pairs, 3 LDGSTS.128 per row instead of 9 8-byte copies),
// allocated in L1 (a CTA may run CLAW_VC_KW consecutive strips so the
// columns neighbouring strips share are re-read from L1; one is fastest).
template <int LIM, int OT>
__global__ void __launch_bounds__(32 * CLAW_VC_KW, CLAW_VC_RES_WARPS / CLAW_VC_KW) step_vc_kernel(const StepParams P) {
  // ring row x = lane + 1 holds lane `lane`'s column; x = 0 / 33 the aux
  // columns (p, u, Z, c) left of lane 0 / right of the last halo lane
  constexpr int KW = CLAW_VC_KW;
  __shared__ __align__(16) double sqr[KW][kGRD][5][34];
  // sources of the two halo rows above the tile (rtop, rtop + 1), resolved
  // once in the prologue (the grid kernel's branch-free tail): q and aux of
  // the lane's column and of its aux column, component strides
  struct HaloSrcVC {
    const double *g, *ga, *x, *xa;
    int32_t cq, ca, xcq, xca;
  };
  __shared__ HaloSrcVC shalo[KW][2][32];
  constexpr int XP = 0, XU = 1, XV = 2, XZ = 3, XC = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * KW + warp;
  const int nstrip = (P.NX + kStrip - 1) / kStrip;
  const int myv = P.my, mx = P.mx;
  const bool span = P.span != 0;
  griddep_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0 && P.level_cfl_reset) *P.level_cfl_reset = 0ull;
  if (t >= P.ntiles) return;
  const int s = t % nstrip;
  const int b = P.blk_first + (t / nstrip) * P.blk_stride;
  int j0, th;
  if (span) {
    j0 = P.R0 + b * P.th;
    th = min(P.th, P.R1 - j0);
  } else {
    const int nbr = (myv + P.th - 1) / P.th;
    const int prow = b / nbr, r0 = (b - prow * nbr) * P.th;
    th = min(P.th, myv - r0);
    j0 = P.Y0 + prow * myv + r0;
  }
  const int c0 = s * kStrip;
  const int tw = min(kStrip, P.NX - c0);
  const int64_t cs = static_cast<int64_t>(mx) * myv;  // component stride (q and aux)
  const double r = P.k.r, sy = P.k.s;
  constexpr double inv2ls = 0.5 / Limiter<LIM>::LS;    // 1/2 cq from the limiter's LS-scaled waves
  const double hrs = 0.5 * r * sy;                     // the transverse terms' 1/2 dt/dx dt/dy

  const int lcol = min(lane, tw + 2);
  const int C = map_idx(c0 - 1 + lcol, P.NX, P.per_x);
  const int Ca = map_idx(lane == 0 ? c0 - 2 : c0 - 1 + min(32, tw + 2), P.NX, P.per_x);
  const bool edge = lane == 0 || lane == 31;
  const int ax = lane == 0 ? 0 : 33;
  const int rtop = j0 + th;
  const double *gq0, *ga0, *xq0, *xa0;   // main / aux column at row j0
  vc_ptrs(P, C, j0 - P.Y0, gq0, ga0);
  vc_ptrs(P, Ca, j0 - P.Y0, xq0, xa0);
  double (*ring)[5][34] = sqr[warp];
  // wide strip (see above): chunk ch < 85 is component ch / 17 (p, u, v from
  // q; Z, c from aux), columns cb + 2 (ch % 17) + {0, 1} (pairs start on even
  // columns like the patches: no pair straddles two patches).  Lane l copies
  // chunks l (q), l + 32 (q for l < 19, else aux) and l + 64 (aux, l < 21):
  // running sources wq (chunk l) and wa (the lane's first aux chunk)
  const bool wstrip = P.wide && c0 >= 2 && c0 + 32 <= P.NX;
  const int cb = c0 - 2;
  auto chunk_src = [&](int ch, int J) {
    const int comp = ch / 17, pr2 = ch - 17 * comp;
    const double *q, *a;
    vc_ptrs(P, cb + 2 * pr2, J - P.Y0, q, a);
    return comp < 3 ? q + comp * cs : a + (comp - 3) * cs;
  };
  auto chunk_dst = [&](int ch) {
    const int comp = ch / 17, pr2 = ch - 17 * comp;
    return smem_u32(&ring[0][comp][2 * pr2]);
  };
  const bool c2q = lane < 19, c3on = lane < 21;
  const double *wq0 = nullptr, *wa0 = nullptr;
  int32_t woff2 = 0;
  unsigned wd1 = 0, wd2 = 0, wd3 = 0;
  if (wstrip) {
    wq0 = chunk_src(lane, j0);
    wa0 = chunk_src(c3on ? lane + 64 : lane + 32, j0);
    woff2 = static_cast<int32_t>(chunk_src(lane + 32, j0) - (c2q ? wq0 : wa0));
    wd1 = chunk_dst(lane);
    wd2 = chunk_dst(lane + 32);
    wd3 = c3on ? chunk_dst(lane + 64) : 0u;
  }
  constexpr unsigned kSlotB = 5 * 34 * 8;   // bytes per ring slot
  auto issue_wide = [&](int sl, const double* wq, const double* wa) {
    const unsigned so = static_cast<unsigned>(sl) * kSlotB;
    cp16s(wd1 + so, wq);
    cp16s(wd2 + so, (c2q ? wq : wa) + woff2);
    cp16s_pred(wd3 + so, wa, c3on);
    cp_commit();
  };
  // (no commit: the per-lane copies that follow it commit the row's group)
  auto issue_wide_pred = [&](int sl, const double* wq, const double* wa, bool p) {
    const unsigned so = static_cast<unsigned>(sl) * kSlotB;
    cp16s_pred(wd1 + so, wq, p);
    cp16s_pred(wd2 + so, (c2q ? wq : wa) + woff2, p);
    cp16s_pred(wd3 + so, wa, c3on && p);
  };

  // (component strides: cq / ca of the main column, xcq / xca of the aux
  // column; the band's plane size except on halo rows)
  auto issue_ptr = [&](int sl, const double* g, const double* ga, const double* x, const double* xa, bool on,
                       int64_t cq, int64_t ca, int64_t xcq, int64_t xca) {
    cp8_pred(&ring[sl][XP][lane + 1], g, on);
    cp8_pred(&ring[sl][XU][lane + 1], g + cq, on);
    cp8_pred(&ring[sl][XV][lane + 1], g + 2 * cq, on);
    cp8_pred(&ring[sl][XZ][lane + 1], ga, on);
    cp8_pred(&ring[sl][XC][lane + 1], ga + ca, on);
    cp8_pred(&ring[sl][XP][ax], x, edge && on);
    cp8_pred(&ring[sl][XU][ax], x + xcq, edge && on);
    cp8_pred(&ring[sl][XZ][ax], xa, edge && on);
    cp8_pred(&ring[sl][XC][ax], xa + xca, edge && on);
    cp_commit();
  };
  // general issue of row R (halo rows mapped by the BCs; rows past rtop + 1,
  // never read for a stored cell, commit an empty group)
  auto issue = [&](int R) {
    const bool on = R <= rtop + 1;
    if (wstrip && R >= j0 && R < rtop) {
      const int sl = (R - j0 + 2) & (kGRD - 1);
      if (span) {
        const double* wq = chunk_src(lane, R);
        const double* wa = chunk_src(c3on ? lane + 64 : lane + 32, R);
        issue_wide(sl, wq, wa);
      } else {
        issue_wide(sl, wq0 + static_cast<int64_t>(R - j0) * mx, wa0 + static_cast<int64_t>(R - j0) * mx);
      }
      return;
    }
    R = min(R, rtop + 1);
    const int sl = (R - j0 + 2) & (kGRD - 1);
    const double *g, *ga, *x, *xa;
    int64_t cq = cs, ca = cs, xcq = cs, xca = cs;
    if (R >= j0 && R < rtop) {
      g = gq0 + static_cast<int64_t>(R - j0) * mx;   // tile rows: inside one patch row unless span
      ga = ga0 + static_cast<int64_t>(R - j0) * mx;
      x = xq0 + static_cast<int64_t>(R - j0) * mx;
      xa = xa0 + static_cast<int64_t>(R - j0) * mx;
      if (span) {
        vc_ptrs(P, C, R - P.Y0, g, ga);
        vc_ptrs(P, Ca, R - P.Y0, x, xa);
      }
    } else {
      vc_src(P, C, R, g, ga, cq, ca);
      vc_src(P, Ca, R, x, xa, xcq, xca);
    }
    issue_ptr(sl, g, ga, x, xa, on, cq, ca, xcq, xca);
  };
  auto slot = [&](int R) { return (R - j0 + 2) & (kGRD - 1); };

  // per-row state, rings of 4 indexed by (row - j0) & 3; face F(k) (between
  // rows k-1 and k) by (k - j0) & 3.  Compile-time slots: registers are
  // renamed across the 4 unrolled phases, not moved.
  double cZ[4], cc[4], cnu[4], cK[4], cey[4], ceyZ[4], cp_[4], cv[4];  // cells
  double fa1[4], fa2[4], fm[4], fsg[4], fqp[4], fqv[4];               // y-faces
  double xP[4], xU[4], xT[4], xsR[4], pk[4], uk[4];                   // x-swept rows
  double Gp[4], Gv[4];                                                // x-transverse edge fluxes
  double cm = 0.0;   // max sound speed over the cells of this lane's column the march reads (CFL)

  // derived medium values of a freshly loaded row (own column); live: the
  // row belongs to the tile's stencil (the unrolled march runs past the last
  // row on ring slots holding stale rows, whose speeds must not count)
  auto cell = [&](int S, int sl, bool live) {
    const double Z = ring[sl][XZ][lane + 1], c = ring[sl][XC][lane + 1];
    if (live) cm = dmax(cm, c);
    cZ[S] = Z;
    cc[S] = c;
    cnu[S] = vc_rcp(__fma_rn(Z, Z, 1.0));
    cK[S] = __dmul_rn(c, Z);
    cey[S] = __dmul_rn(__dmul_rn(c, __fma_rn(-c, sy, 1.0)), inv2ls);
    ceyZ[S] = __dmul_rn(cey[S], Z);
    cp_[S] = ring[sl][XP][lane + 1];
    cv[S] = ring[sl][XV][lane + 1];
  };
  // y-face F(k) between the cells in slots Sl (row k-1) and Su (row k)
  auto yface = [&](int Sf, int Sl, int Su) {
    const double sg = vc_rcp(__dadd_rn(cZ[Sl], cZ[Su]));
    const double dp = __dsub_rn(cp_[Su], cp_[Sl]), dv = __dsub_rn(cv[Su], cv[Sl]);
    fa1[Sf] = __dmul_rn(sg, __fma_rn(cZ[Su], dv, -dp));
    fa2[Sf] = __dmul_rn(sg, __fma_rn(cZ[Sl], dv, dp));
    fm[Sf] = __fma_rn(cZ[Sl], cZ[Su], 1.0);
    fsg[Sf] = sg;
  };
  // limit y-face F(k): Sf its slot, Sl / Su its cells, Sd / Sup the faces
  // below / above (upwind of wave 2 / wave 1)
  auto ylimit = [&](int Sf, int Sl, int Su, int Sd, int Sup) {
    const double t1 = Limiter<LIM>::apply(fa1[Sf], __dmul_rn(fa1[Sup], __dmul_rn(fm[Sf], cnu[Sl])));
    const double t2 = Limiter<LIM>::apply(fa2[Sf], __dmul_rn(fa2[Sd], __dmul_rn(fm[Sf], cnu[Su])));
    fqp[Sf] = __fma_rn(ceyZ[Su], t2, -__dmul_rn(ceyZ[Sl], t1));
    fqv[Sf] = __fma_rn(cey[Su], t2, __dmul_rn(cey[Sl], t1));
  };
  // x-sweep of the row in ring slot sl whose cell values sit in slot S
  auto xsweep = [&](int S, int sl) {
    const double p = ring[sl][XP][lane + 1], u = ring[sl][XU][lane + 1];
    const double pl = ring[sl][XP][lane], ul = ring[sl][XU][lane], Zl = ring[sl][XZ][lane];
    const double pr = ring[sl][XP][lane + 2], ur = ring[sl][XU][lane + 2], Zr = ring[sl][XZ][lane + 2];
    const double Z = cZ[S], c = cc[S], K = cK[S];
    pk[S] = p;
    uk[S] = u;
    const double sL = vc_rcp(__dadd_rn(Zl, Z)), sR = vc_rcp(__dadd_rn(Z, Zr));
    const double dpl = __dsub_rn(p, pl), dul = __dsub_rn(u, ul);
    const double a1 = __dmul_rn(sL, __fma_rn(Z, dul, -dpl));
    const double a2 = __dmul_rn(sL, __fma_rn(Zl, dul, dpl));
    const double a1r = __dmul_rn(sR, __fma_rn(Zr, __dsub_rn(ur, u), -__dsub_rn(pr, p)));
    const double mL = __fma_rn(Zl, Z, 1.0);
    const double nul = shfl_up(cnu[S]), a2u = shfl_up(a2);
    const double t1 = Limiter<LIM>::apply(a1, __dmul_rn(a1r, __dmul_rn(mL, nul)));
    const double t2 = Limiter<LIM>::apply(a2, __dmul_rn(a2u, __dmul_rn(mL, cnu[S])));
    const double ex = __dmul_rn(__dmul_rn(c, __fma_rn(-c, r, 1.0)), inv2ls);
    const double exZ = __dmul_rn(ex, Z);
    const double exl = shfl_up(ex), exZl = shfl_up(exZ);   // the left cell's (lane 0: unused)
    const double qp = __fma_rn(exZ, t2, -__dmul_rn(exZl, t1));   // 1/2 cq of the left face
    const double qu = __fma_rn(ex, t2, __dmul_rn(exl, t1));
    const double dqp = __dsub_rn(shfl_dn(qp), qp), dqu = __dsub_rn(shfl_dn(qu), qu);
    const double as = __dadd_rn(a1r, a2);
    xP[S] = __fma_rn(K, as, dqp);
    xU[S] = __fma_rn(c, __dsub_rn(a2, a1r), dqu);
    xT[S] = (OT == 2) ? __fma_rn(2.0, dqp, __dmul_rn(K, as)) : __dmul_rn(K, as);
    xsR[S] = sR;
  };
  // x-transverse edge flux G of face F(k) (slot Sf) from rows k-1 (Sl), k (Su)
  auto gedge = [&](int Sf, int Sl, int Su) {
    Gp[Sf] = __dmul_rn(fsg[Sf], __fma_rn(cK[Su], xT[Sl], -__dmul_rn(cK[Sl], xT[Su])));
    Gv[Sf] = __dmul_rn(fsg[Sf], __fma_rn(cc[Su], xT[Sl], __dmul_rn(cc[Sl], xT[Su])));
  };

  // ---- prologue: rows j0-2 .. j0+1 (slots 2, 3, 0, 1)
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {
    HaloSrcVC h;
    int64_t cq, ca, xcq, xca;
    vc_src(P, C, rtop + k2, h.g, h.ga, cq, ca);
    vc_src(P, Ca, rtop + k2, h.x, h.xa, xcq, xca);
    h.cq = static_cast<int32_t>(cq);
    h.ca = static_cast<int32_t>(ca);
    h.xcq = static_cast<int32_t>(xcq);
    h.xca = static_cast<int32_t>(xca);
    shalo[warp][k2][lane] = h;
  }
#pragma unroll 1
  for (int R = j0 - 2; R <= j0 + kGRD - 3; ++R) issue(R);
  cp_wait<kGRD - 4>();
  __syncwarp();
  cell(2, slot(j0 - 2), true);
  cell(3, slot(j0 - 1), true);
  cell(0, slot(j0), true);
  cell(1, slot(j0 + 1), true);
  yface(3, 2, 3);   // F(j0-1)
  yface(0, 3, 0);   // F(j0)
  yface(1, 0, 1);   // F(j0+1)
  ylimit(0, 3, 0, 3, 1);
  xsweep(3, slot(j0 - 1));
  xsweep(0, slot(j0));
  if (OT != 0) gedge(0, 3, 0);
  __syncwarp();
  issue(j0 + kGPD + 1);
  const bool act = lane >= 1 && lane <= tw;
  double* o = P.qn + (gq0 - P.q);
  const int64_t jump_q = static_cast<int64_t>(P.npx) * 3 * mx * myv - static_cast<int64_t>(myv) * mx;
  const int64_t jump_a = static_cast<int64_t>(P.npx) * 2 * mx * myv - static_cast<int64_t>(myv) * mx;
  // (wide strips: gq / ga run the lane's chunk sources wq / wa instead)
  // (a tile that starts kGPD+2 or fewer rows before its patch row ends --
  // band split with tile heights that are not multiples of my -- already
  // crossed into the next patch row at the first row the march prefetches)
  const bool x0 = span && (j0 % myv) + kGPD + 2 >= myv;
  const double* gq = (wstrip ? wq0 : gq0) + static_cast<int64_t>(kGPD + 2) * mx + (x0 ? jump_q : 0);
  const double* ga = (wstrip ? wa0 : ga0) + static_cast<int64_t>(kGPD + 2) * mx + (x0 ? jump_a : 0);
  const double* xq = xq0 + static_cast<int64_t>(kGPD + 2) * mx + (x0 ? jump_q : 0);
  const double* xa = xa0 + static_cast<int64_t>(kGPD + 2) * mx + (x0 ? jump_a : 0);

  auto step = [&](auto phc, int jb, auto fastc) {
    constexpr int PH = decltype(phc)::value;
    constexpr int S0 = PH & 3, S1 = (PH + 1) & 3, S2 = (PH + 2) & 3, S3 = (PH + 3) & 3;
    const int j = jb + PH;
    static_assert((kGPD + 2 + 1) % 4 == 0, "the prefetched row crosses patch rows in phase 1");
    if (PH == 1 && span && (jb + kGPD + 3 - P.Y0) % myv == 0) {  // row j+2+kGPD starts a patch row
      gq += jump_q;
      xq += jump_q;
      ga += jump_a;
      xa += jump_a;
    }
    if (PH == 0 && span && jb != j0 && (jb - P.Y0) % myv == 0) o += jump_q;
    // row j+2 landed (rows up to j+1+kGPD are in flight); the warp barrier
    // also orders every read of the slot the next issue overwrites (row j-1:
    // its finalisation read neighbours' media, one step ago) before the copy
    cp_wait<kGPD - 1>();
    __syncwarp();
    if (decltype(fastc)::value) {
      if (wstrip)
        issue_wide((j + 2 + kGPD - j0 + 2) & (kGRD - 1), gq, ga);
      else
        issue_ptr((j + 2 + kGPD - j0 + 2) & (kGRD - 1), gq, ga, xq, xa, true, cs, cs, cs, cs);
    } else {
      // general issue, branch-free (see HaloSrcVC): rows inside the tile from
      // the running pointers (wide strips: 16-byte chunks), rows rtop, rtop + 1
      // from the table, rows past rtop + 1 nothing (empty group)
      const int R = j + 2 + kGPD;
      const bool in = R < rtop, on = R <= rtop + 1, wide = wstrip && in;
      const int sl = (min(R, rtop + 1) - j0 + 2) & (kGRD - 1);
      const HaloSrcVC& h = shalo[warp][min(max(R - rtop, 0), 1)][lane];
      issue_wide_pred(sl, gq, ga, wide);
      issue_ptr(sl, in ? gq : h.g, in ? ga : h.ga, in ? xq : h.x, in ? xa : h.xa, on && !wide,
                in ? cs : h.cq, in ? cs : h.ca, in ? cs : h.xcq, in ? cs : h.xca);
    }
    gq += mx;
    ga += mx;
    xq += mx;
    xa += mx;
    const int rs0 = slot(j), rs1 = slot(j + 1), rs2 = slot(j + 2);
    const bool live = j < rtop;
    cell(S2, rs2, live);              // row j+2
    yface(S2, S1, S2);                // F(j+2)
    ylimit(S1, S0, S1, S0, S2);       // F(j+1)
    xsweep(S1, rs1);                  // row j+1
    if (OT != 0) gedge(S1, S0, S1);   // G of F(j+1)
    // finalise row j
    const double K0 = cK[S0], c0v = cc[S0];
    const double asy = __dadd_rn(fa1[S1], fa2[S0]);
    const double dqy = __dsub_rn(fqp[S1], fqp[S0]);
    const double Py = __fma_rn(K0, asy, dqy);
    const double Vy = __fma_rn(c0v, __dsub_rn(fa2[S0], fa1[S1]), __dsub_rn(fqv[S1], fqv[S0]));
    const double q0v = ring[rs0][XV][lane + 1];
    double pn = __fma_rn(-r, xP[S0], pk[S0]);
    pn = __fma_rn(-sy, Py, pn);
    double un = __fma_rn(-r, xU[S0], uk[S0]);
    double vn = __fma_rn(-sy, Vy, q0v);
    if (OT != 0) {
      const double Ty = (OT == 2) ? __fma_rn(2.0, dqy, __dmul_rn(K0, asy)) : __dmul_rn(K0, asy);
      const double TyR = shfl_dn(Ty);
      const double cR = ring[rs0][XC][lane + 2], KR = __dmul_rn(cR, ring[rs0][XZ][lane + 2]);
      const double FpR = __dmul_rn(xsR[S0], __fma_rn(KR, Ty, -__dmul_rn(K0, TyR)));
      const double FuR = __dmul_rn(xsR[S0], __fma_rn(cR, Ty, __dmul_rn(c0v, TyR)));
      const double FpL = shfl_up(FpR), FuL = shfl_up(FuR);
      pn = __fma_rn(hrs, __dadd_rn(__dsub_rn(Gp[S1], Gp[S0]), __dsub_rn(FpR, FpL)), pn);
      un = __fma_rn(hrs, __dsub_rn(FuR, FuL), un);
      vn = __fma_rn(hrs, __dsub_rn(Gv[S1], Gv[S0]), vn);
    }
    (void)S3;
    const bool st = act && j < rtop;
    st_pred(o, pn, st);
    st_pred(o + cs, un, st);
    st_pred(o + 2 * cs, vn, st);
    o += mx;
  };

  using Fast = std::integral_constant<bool, true>;
  using Slow = std::integral_constant<bool, false>;
  int jb = j0;
  for (; jb + 3 + 2 + kGPD < rtop; jb += 4) {
    step(std::integral_constant<int, 0>{}, jb, Fast{});
    step(std::integral_constant<int, 1>{}, jb, Fast{});
    step(std::integral_constant<int, 2>{}, jb, Fast{});
    step(std::integral_constant<int, 3>{}, jb, Fast{});
  }
  for (; jb < rtop; jb += 4) {
    step(std::integral_constant<int, 0>{}, jb, Slow{});
    step(std::integral_constant<int, 1>{}, jb, Slow{});
    step(std::integral_constant<int, 2>{}, jb, Slow{});
    step(std::integral_constant<int, 3>{}, jb, Slow{});
  }
  cp_wait<0>();
  // Courant number: max over this warp's swept faces of max(c_l, c_r) dt/dx
  // (dt/dy) -- every face's cells are cells of the domain (BC images are
  // copies), so the level max is exact
  // every swept x- (y-) face's speed is max(c_l, c_r) of two cells of the
  // domain, and every cell is a left or right cell of such a face, so the max
  // over the faces of max(c_l, c_r) dt/dx is dt/dx times the max over the
  // cells; each cell is in some lane's column (BC images are copies)
  double cf = fmax(__dmul_rn(r, cm), __dmul_rn(sy, cm));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) cf = fmax(cf, __shfl_xor_sync(kFull, cf, off));
  if (lane == 0 && cf > 0.0) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(cf));
    atomicMax(P.level_cfl, bits);
    if (P.hier_cfl) atomicMax(P.hier_cfl, bits);
  }
}

template <int LIM>
cudaError_t launch_vc(const StepParams& p, cudaStream_t st) {
  const dim3 grid((p.ntiles + CLAW_VC_KW - 1) / CLAW_VC_KW), block(32 * CLAW_VC_KW);
  StepParams w = p;   // 16-byte row copies: even patch width, 16-byte aligned q and aux
  w.wide = g_rowcopy != 0 && p.mx % 2 == 0 && ((reinterpret_cast<uintptr_t>(p.q) | reinterpret_cast<uintptr_t>(p.aux)) & 15) == 0;
  switch (p.order_trans) {
    case 0: return launch_k(step_vc_kernel<LIM, 0>, grid, block, st, w);
    case 1: return launch_k(step_vc_kernel<LIM, 1>, grid, block, st, w);
    default: return launch_k(step_vc_kernel<LIM, 2>, grid, block, st, w);
  }
}
