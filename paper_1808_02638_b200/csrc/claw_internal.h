// claw_internal.h -- device-table layouts shared by the host planner
// (claw_host.cpp) and the sm_100a kernels (claw_kernels.cu).  Not part of the
// public ABI (include/claw.h).
#pragma once
#include <cstdint>

namespace claw {

// One owned patch of a level.  The level buffer stores owned patches back to
// back as [3][my][mx] fp64 (components p, u, v; x fastest), each patch's
// component planes starting on a 256-byte boundary when mx*my allows.
struct DevPatch {
  int64_t off;        // element offset of (m=0, j=0, i=0) in the level buffer
  int64_t cs;         // component stride (elements)
  int32_t mx, my;
  int32_t rect_begin; // ghost-source rectangles [rect_begin, rect_end)
  int32_t rect_end;
  int32_t region[8];  // rectangle covering the whole W, E, S, N ghost strip or
                      // SW, SE, NW, NE 2x2 corner block, or -1 (search the list)
  double dx, dy;
  double c, Z;        // sound speed sqrt(K/rho), impedance rho*c
  int64_t crect;      // offset of this patch's ghost-frame rectangle map in the level's
                      // cell-rect table (one int32 rectangle index per ghost cell, frame
                      // ring order), or -1
};
static_assert(sizeof(DevPatch) == 104, "DevPatch layout");

// Ghost-source rectangle: patch-local cells (i, j) with i0 <= i < i0+w,
// j0 <= j < j0+h (0-based, ghosts are -2..-1 and mx..mx+1) take their value
// from  buffer[base + (i-i0)*sx + (j-j0)*sy + m*cs].
//   kind 0: the level's current ping-pong buffer (same-level donor interior,
//           physical BC mapped onto an interior cell);
//   kind 1: the level's frame buffer (coarse-interpolated or remote cells).
struct DevRect {
  int32_t i0, j0, w, h;
  int32_t kind, pad;
  int64_t base, sx, sy, cs;
};
static_assert(sizeof(DevRect) == 56, "DevRect layout");

// Work unit of the fused step kernel: a strip of <= 32 columns of one patch
// (tile columns [i0, i0+tw), rows [j0, j0+th)); packed as int4 {patch, i0, j0,
// tw | th << 16}.

// Coarse-interpolation spec for one frame slot (P:131 case 3; R10):
// 5 coarse donors (centre, x-, x+, y-, y+) given as element offsets of their
// p component in the coarse level buffer and component strides.
struct DevInterp {
  int64_t off[5];
  int64_t cs[5];
  double xi, eta;     // fine-cell offset inside the coarse cell, in coarse cells
  int64_t dst;        // frame slot (p component); components at dst + m*fcs
};

// Per-patch step constants (dt, dx, dy, c, Z and the limiter scale LS folded
// in).  For a level whose patches share one medium they are computed once on
// the host and passed as kernel parameters (no registers); otherwise every
// tile derives them on the device with the same operation order.
struct StepConsts {
  double Z, h, hz;        // Z, c/2, c/(2Z)
  double r, s;            // dt/dx, dt/dy
  double kx4, kx2, kx4z;  // kx/(4 LS), kx/(2 LS) (order_trans 2 else 0), kx/(4 LS Z); kx = c(1 - c r)
  double ky4, ky2, ky4z;
  double T, TZ;           // r s c / 4, r s c / (4 Z)   (0 when order_trans = 0)
  double cfl;             // max(c dt/dx, c dt/dy)
  double mr, ms, mT;      // -r, -s, -T (negation is exact)
};

struct StepParams {
  const double* q;        // current buffer (read)
  double* qn;             // next buffer (write)
  const double* frame;    // frame buffer
  const DevPatch* patches;
  const DevRect* rects;
  const int32_t* cellrect;        // generic levels: per ghost cell its rectangle (DevPatch::crect)
  const int4* tiles;
  int32_t ntiles;
  int32_t limiter, order_trans;
  double dt;
  unsigned long long* patch_cfl;  // per owned patch, bits of a non-negative double (plain stores)
  unsigned long long* level_cfl;  // level slot of this step (atomicMax)
  unsigned long long* level_cfl_reset;  // the other generation's slot, zeroed by the kernel
  unsigned long long* hier_cfl;   // coarse-step slot of claw_advance_hierarchy, or null
  int32_t uniform;                // 1: every patch uses `k` below
  int32_t lane_tiles;             // generic tiles are 30-column strips for step_lane_kernel
  StepConsts k;
  // grid mode (uniform tiling of the whole domain by equal patches in
  // row-major order, gapless buffer): level-index strips, no tables
  int32_t grid;
  int32_t NX, NY, mx, my, npx;    // level extent, patch size, patches per row
  int32_t th;                     // rows per tile (tiles stay in one patch row unless span)
  int32_t span;                   // 1: row block b is rows [R0 + b th, min(R0 + (b+1) th, R1))
                                  // and tiles may span patch rows (th > my, or a band-split
                                  // launch); 0: blocks of th rows inside each patch row
  int32_t R0, R1;                 // span: the launch's row range (whole band: Y0, Y1)
  int32_t per_x, per_y;           // periodic in x / y
  int32_t Y0, Y1;                 // this rank's band of level rows (whole level: 0, NY)
  int32_t blk_first, blk_stride;  // grid tiles: row block = blk_first + k*blk_stride,
                                  // k < ntiles / nstrip (interior / edge launches)
  int32_t tile_offset;            // generic tiles: first tile index of this launch
  int64_t hoff[4];                // band halo rows Y0-2, Y0-1, Y1, Y1+1: frame offset of
  int64_t hcs[4];                 // column 0 (-1: the row is local) and component stride
  const int32_t* slots;           // grid kernel on a sparse lattice of equal patches: per
                                  // lattice slot (row-major, npx per row) the patch index
                                  // (>= 0) or -1-v for virtual slot v of the frame (coarse
                                  // ghost values); P.tiles then lists (strip, row block)
  const double* aux;              // variable media (grid mode): [owned patch][2][my][mx] (Z, c) in
                                  // q's patch order; null: constant media (R20)
  const double* aux_halo;         // band mode: (Z, c) of the 4 halo rows, [4][2][NX]
  int32_t wide;                   // step_vc_kernel: 16-byte row copies allowed (set by its launcher)
  double* side;                   // generic kernel: per-tile side records (side_stride()
                                  // doubles per tile), filled by a side_kernel launched
                                  // ahead of the step kernel; null: computed in the kernel
};

// Launchers (claw_kernels.cu).  All return cudaError_t as int.
int launch_step(const StepParams& p, void* stream);
// alpha_dev (may be null): read alpha from device memory instead (graph replay)
// nal time levels (alphas, or alpha_dev[k] when non-null) into frame slices
// k * slice apart (the R substeps of a fine level at once; nal = 1 otherwise)
constexpr int kMaxInterpAlphas = 8;
struct InterpAlphas {
  double a[kMaxInterpAlphas];
};
int launch_interp(const double* q_old, const double* q_new, const double* alphas, int nal, const double* alpha_dev,
                  const DevInterp* spec, int64_t n, double* frame, int64_t fcs, int64_t slice, void* stream);
// debug check (claw_config.check_finite): atomicMax(flag, level) if any of
// q[0..n) is NaN or +-Inf
int launch_nonfinite(const double* q, int64_t n, int level, int32_t* flag, void* stream);
// scatter [3][n] values into q at offset off[s] (+ m cs[s]) (update exchange)
int launch_scatter(const double* buf, const int64_t* off, const int64_t* cs, int64_t n, double* q, void* stream);
// the ghost-cell rectangle map of a generic level (DevPatch::crect; one CTA
// per patch, every cell of every rectangle of the patch)
int launch_cellrect(const DevPatch* patches, int32_t npatch, const DevRect* rects, int32_t* map, void* stream);
int launch_pack(const double* q, const int64_t* off, const int64_t* cs, int64_t n,
                double* out, void* stream);
int launch_gather_padded(const double* q, const double* frame, const DevPatch* patches,
                         const DevRect* rects, int32_t patch, double* out, void* stream);
// Updating entry (one covered coarse cell).  Usual case: its R x R children
// lie in one fine patch, child (a, b) at src + b*fmx + a.  Otherwise (slow),
// src indexes R*R (offset, cs) pairs in the slow lists.
struct DevUpdate {
  int64_t dst;      // coarse offset (p component)
  int64_t src;
  int32_t dcs, fcs; // component strides (coarse, fine)
  int32_t fmx, slow;
};
static_assert(sizeof(DevUpdate) == 32, "DevUpdate layout");
// Updating rectangle: w x h coarse cells (row pitch cmx) whose R x R children
// all lie in one fine patch (row pitch fmx); dst / src: offsets of the first
// coarse cell and of its first child (p components).
struct DevUpdateRect {
  int64_t dst, src;
  int64_t dcs, fcs;
  int32_t cmx, fmx, w, h;
  int32_t chunk0, pad;  // first work chunk (kUpdChunk coarse cells each) of this rectangle
};
constexpr int kUpdChunk = 128;
// nchunk work chunks; chunk_rect[k] = the rectangle chunk k belongs to
int launch_update_rects(double* q_coarse, const double* q_fine, const DevUpdateRect* rects,
                        const int32_t* chunk_rect, int32_t nchunk, int R, void* stream);
int launch_update(double* q_coarse, const double* q_fine, const DevUpdate* tab, int64_t n, int R,
                  const int64_t* slow_off, const int64_t* slow_cs, void* stream);
// Conservation-fix register of a fine level (NEXT-2, R17): coarse
// cell C = (ci, cj) of owned coarse patch cp, not covered by the fine level,
// sharing edge E (dir 0: x-edge, 1: y-edge) with a covered cell; side 0: C
// lies left of / below E.  The R fine cells on the other side of E start at
// (fi, fj) of owned fine patch fp and run along E.  Registers of one C are
// consecutive (heads list).
struct DevReflux {
  int32_t cp, ci, cj;
  int32_t ds;         // dir | side << 1
  int32_t fp, fi, fj;
  int32_t pad;
};
static_assert(sizeof(DevReflux) == 32, "DevReflux layout");
// which 0: coarse part (p = the coarse level's step params with q = q^n);
// which 1: fine part (p = the fine level's step params, qc = coarse q^n,
// cpatches = coarse patch records).  acc: [n][3].
int launch_reflux(int which, const StepParams& p, const double* qc, const DevPatch* cpatches,
                  const DevReflux* tab, int64_t n, int R, double* acc, void* stream);
int launch_reflux_apply(double* qc, const DevPatch* cpatches, const DevReflux* tab, const int32_t* heads,
                        int64_t nheads, double* acc, void* stream);
// Regridding (NEXT-3; R18).
// Flagging: every interior cell of owned patch lp (origin orig[lp] in the
// level index space) sets raw[J*nx+I] = (max over its 4 edge neighbours of
// |p_n - p| > tol) and on[J*nx+I] = 1; neighbours resolved like the step
// kernel's (p.q, p.frame, p.patches, p.rects).
int launch_flag(const StepParams& p, const int2* orig, int32_t nown, int64_t nx, double tol, uint8_t* raw,
                uint8_t* on, int64_t max_cells, void* stream);
// Chebyshev dilation by b, clipped to [0,nx) x [0,ny) and (mask != null) to
// mask != 0; *count (device, zeroed by the caller) receives the set cells.
int launch_dilate(const uint8_t* in, uint8_t* tmp, uint8_t* out, const uint8_t* mask, int64_t nx, int64_t ny, int b,
                  unsigned long long* count, void* stream);
int launch_not(const uint8_t* in, uint8_t* out, int64_t n, void* stream);
// summed-area table (ny+1) x (nx+1) int32 of a uint8 flag map (clustering)
int launch_sat(const uint8_t* f, int64_t nx, int64_t ny, int32_t* sat, void* stream);
// Patch-id map of a level's index space: map[J*nx + I] = owned patch index
// or -1 (map memset to 0xff first); one CTA per patch paints its rectangle.
int launch_paint(int32_t* map, int64_t nx, const int2* orig, const DevPatch* patches, int32_t npatch, void* stream);
// New fine level (regrid): one CTA per new patch, one thread per cell.  A cell
// takes the old fine level's value where oldmap (fine index space, may be
// null) names a patch, else the R10 interpolation at alpha = 1 from the
// coarse level (donors through cmap and the BCs); a missing donor sets *err.
struct RegridParams {
  const double* qc_old;
  const double* qc_new;
  const int32_t* cmap;
  const DevPatch* cpatch;
  const int2* corig;
  int64_t cnx, cny;
  const double* qf_old;
  const int32_t* oldmap;
  const DevPatch* opatch;
  const int2* oorig;
  int64_t fnx;
  double* qf;
  const DevPatch* npatch;
  const int2* norig;
  int32_t R;
  int32_t per_x, per_y;
  int32_t* err;
};
int launch_regrid(const RegridParams& p, int32_t nnew, void* stream);
// programmatic dependent launches of the step-sequence kernels (default on)
extern int g_pdl;
void set_pdl(int on);
// row copies of the grid kernel where the layout allows (step_grid_kernel RC:
// 0 per-lane 8 B; 1 per-lane 16 B, 4-warp CTAs; 2 per-lane 16 B, one-warp
// CTAs; 3 = auto: 1 for dense launches of a wave or more, else 2)
extern int g_rowcopy;
void set_rowcopy(int rc);
// warps of one full wave of the grid kernel (SMs x resident warps): smaller
// launches take one-warp CTAs
extern int g_grid_wave;
void set_grid_wave(int warps);
int max_tile_rows();
int grid_resident_warps();   // resident warps per SM the grid kernel is compiled for
int side_stride();
int grid_strip();
// grid-mode strips: count over nx level columns, output columns of strip s
int64_t grid_nstrip(int64_t nx);
void grid_strip_cols(int64_t s, int64_t nx, int64_t& c0, int64_t& c1);

}  // namespace claw
