/*
 * claw.h -- C ABI of libclaw.so, the B200 (sm_100a) batched AMR-level advance
 * for 2D linear acoustics with Clawpack's wave-propagation method
 * (arXiv 1808.02638, Qin, LeVeque & Motley).
 *
 * Citations: P:a-b = /root/reference/PAPER.md lines a-b (section / equation
 * named), S:a-b = SPEC.md lines (interfaces only).  DESIGN.md lists every
 * reading of the paper these calls implement.
 *
 * Conventions for every entry point
 *   - Return value: CLAW_OK (0) or a negative CLAW_E* code; nothing aborts or
 *     throws.  claw_last_error() names the offending field / patch.
 *   - Host arrays passed in are copied during the call; the library keeps no
 *     caller pointer.  Device memory, tables, events and the NCCL communicator
 *     are owned by the context (a caller-supplied stream is borrowed).
 *   - One context per device and process; a context is not thread-safe.
 *   - CLAW_ECUDA / CLAW_ENCCL are sticky: the context is unusable afterwards.
 *   - Patch data on the host is [3][my][mx] per patch: components (p, u, v),
 *     x fastest, fp64.  "Level arrays" concatenate the patches a rank OWNS in
 *     ascending global patch index (claw_owner tells which rank owns what).
 *
 * Call order: claw_create; claw_set_level(1), then 2.. (each nested in the
 * previous); per level step claw_fill_ghost(L, t) then claw_advance_level(L,
 * dt); claw_read* at any time.
 */
#ifndef CLAW_H
#define CLAW_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CLAW_OK 0
#define CLAW_EINVAL (-1)     /* bad argument / descriptor field */
#define CLAW_ESTATE (-2)     /* call order violated */
#define CLAW_ENOMEM (-3)     /* device or host allocation failed */
#define CLAW_ECUDA (-4)      /* CUDA error (sticky) */
#define CLAW_ENCCL (-5)      /* NCCL error or NCCL unavailable (sticky) */
#define CLAW_ENEST (-6)      /* ghost cell with no same-level or coarse donor */
#define CLAW_ENONFINITE (-7) /* claw_config.check_finite: a step produced NaN / Inf;
                                not sticky (the state is left as computed) */
#define CLAW_ENODEV (-8)     /* compute requested from a host-only (device = -1) context */

#define CLAW_BC_EXTRAP 1     /* zero-order extrapolation, the paper's outflow BC */
#define CLAW_BC_PERIODIC 2

/* One grid patch (uniform rectangular patch of a level; P:125-126:
 * mbc ghost cells around it).  Same field list as north_star's descriptor. */
typedef struct {
  int32_t mx, my;          /* interior cells, >= 1 */
  double dx, dy;           /* > 0, identical for every patch of a level */
  double xlower, ylower;   /* physical lower-left corner of the interior; must
                              sit on the level's index grid */
  int32_t mbc;             /* ghost width; must be 2 (the stencil is 5x5 minus corners) */
  double rho, K;           /* density rho_0 and bulk modulus K_0 of P:457-466, > 0;
                              c = sqrt(K/rho), Z = rho c */
} claw_patch_desc;

typedef struct {
  double xlo, xhi, ylo, yhi;   /* physical domain; level-1 patches must tile it */
  int32_t bc[4];               /* left, right, bottom, top: CLAW_BC_*; periodic pairs */
  int32_t limiter;             /* wave limiter phi: 0 none (Lax-Wendroff), 1 minmod,
                                  2 superbee, 3 van Leer, 4 MC */
  int32_t order_trans;         /* transverse propagation ("corner transport"):
                                  0 none, 1 fluctuations, 2 fluctuations + corrections */
  int32_t device;              /* CUDA device ordinal; -1 = host-only context that
                                  builds every table but never touches CUDA (tests) */
  int32_t rank, world;         /* this process's rank among `world` (1 = no NCCL) */
  const void* nccl_unique_id;  /* world > 1: 128-byte ncclUniqueId, identical on
                                  every rank (distributed by the caller) */
  void* stream;                /* cudaStream_t to launch on, or NULL: the library
                                  creates a non-blocking stream */
  int32_t tile_rows;           /* rows per tile of the fused step kernel (0 = default
                                  64); results are bitwise independent of it */
  int32_t path;                /* 0 auto: a level that is one uniform grid of equal
                                  patches (row-major, whole domain, one medium, one
                                  rank) uses the table-free grid kernel; 1 always the
                                  generic ghost-table kernel.  Bitwise identical. */
  int32_t exchange;            /* world > 1 only.  0: NCCL (send/recv halo, max
                                  all-reduce of the CFL).  1: external -- the caller
                                  moves remote ghost cells with claw_halo_pack /
                                  claw_halo_unpack between claw_fill_ghost and
                                  claw_advance_level and reduces the CFL itself
                                  (tests and custom transports; no NCCL needed) */
  int32_t reflux;              /* 1: conservation fix at coarse-fine interfaces (P:122-123,
                                  P:151-225; R17).  Fine patches
                                  must be aligned to the coarser cells; single rank
                                  (EINVAL with world > 1).
                                  See claw_update_level. */
  int32_t check_finite;        /* 1: debug check -- after every level step a
                                  reduction over the new state; claw_advance_level /
                                  claw_wait_cfl / claw_advance_hierarchy then return
                                  CLAW_ENONFINITE naming the level if any value is NaN or
                                  Inf (costs one extra read of the level per step) */
  void* arena;                 /* device memory of `device` the caller owns (e.g. a torch
                                  tensor's storage), or NULL.  Given: EVERY device buffer of
                                  this context (levels, tables, frames, scratch) is carved
                                  from it by the library's pool rules (one big
                                  allocation carved per patch/level instead of cudaMalloc
                                  per patch); no cudaMalloc happens for the context and a
                                  request that does not fit fails with CLAW_ENOMEM.  The
                                  arena is borrowed: it must outlive claw_destroy and is
                                  never freed by the library.  NULL: the library's own
                                  process-wide cudaMalloc'ed pool (claw_pool_stats). */
  uint64_t arena_bytes;        /* size of the arena in bytes */
  int32_t dist_level;          /* world > 1: the level partitioned across the ranks.
                                  0: level 1 (single-level runs: band or Morton partition,
                                  levels > 1 refused).  K >= 2: levels 1 .. K-1 are
                                  replicated -- every rank holds and steps all their
                                  patches, identically -- and level K (the finest; setting
                                  a level above K fails) is Morton-partitioned: its coarse
                                  interpolation donors are local, its same-level halo is
                                  exchanged as for level 1, and claw_update_level(K)
                                  averages each rank's patches locally, then exchanges the
                                  averaged level-(K-1) cells so the replicas stay equal
                                  (NCCL, or claw_update_pack / claw_update_unpack with
                                  exchange = 1).  The finest level must be aligned to the
                                  coarse cells (every coarse cell's children in one fine
                                  patch).  Conservation fix and regridding stay single-rank. */
  int32_t reserved[3];
} claw_config;

/* Kernel-level statistics, accumulated while profiling is on. */
typedef struct {
  int64_t step_launches;        /* fused step kernel launches */
  double step_ms;               /* summed CUDA-event time of those launches */
  int64_t ghost_launches;       /* ghost-fill (coarse interp / pack) launches */
  double ghost_ms;
  int64_t cells_advanced;       /* interior cell-updates performed */
  int64_t halo_bytes_sent;      /* NCCL halo bytes sent by this rank */
} claw_stats;

typedef struct claw_ctx claw_ctx;

/* Create a context for one AMR hierarchy on one device (the paper's GPU
 * advance, P:316-352 / P:410-440, with its memory pool P:422-426): validates
 * cfg (EINVAL, message via claw_last_error even on failure: *out is then a
 * dead context to destroy), selects the device, creates or adopts the stream,
 * adopts cfg->arena if given, and for world > 1 joins the NCCL communicator
 * (ENCCL).  *out receives the context (owned by the caller until
 * claw_destroy). */
int claw_create(const claw_config* cfg, claw_ctx** out);
/* Synchronise the context's stream and release everything it owns: device
 * buffers go back to the pool (or the caller's arena), the stream (if the
 * library created it), events and the NCCL communicator.  EINVAL for NULL. */
int claw_destroy(claw_ctx* ctx);
/* The message of the last failing call on ctx (a field / patch / level is
 * named); valid until the next call on ctx.  Never NULL. */
const char* claw_last_error(const claw_ctx* ctx);

/* Deterministic owner map used by claw_set_level for the partitioned level
 * (claw_config.dist_level) on `world` ranks: a uniform grid of equal patches
 * covering the domain in bands of whole patch rows, otherwise patches in
 * Morton order of their lower-left index (relative to the level's minimum
 * corner), split contiguously into chunks of ~equal cell count.
 * owner[npatch] receives ranks.  Host-only. */
int claw_partition(int32_t npatch, const claw_patch_desc* descs, int32_t world,
                   int32_t* owner);

/* Define level `level` (1..8) from the FULL descriptor list (identical on every
 * rank).  Validates (EINVAL: mx,my < 1, mbc != 2, rho/K <= 0, dx/dy differing
 * within the level, patch off the level grid or outside the domain, same-level
 * overlap, level 1 not tiling the domain; ENEST: a ghost cell without donor),
 * builds the ghost-source, tile and exchange tables, allocates the level's
 * device pool (two ping-pong buffers) and uploads q0 (NULL = zeros): the
 * owned patches' level array.  Replaces any previous definition of the level;
 * finer levels must be set again afterwards.  world > 1: the level named by
 * claw_config.dist_level (default level 1) is partitioned (q0: the owned
 * patches, in global patch order); every other level is replicated (q0: all
 * patches) and levels above dist_level fail (EINVAL). */
int claw_set_level(claw_ctx* ctx, int32_t level, int32_t npatch,
                   const claw_patch_desc* descs, const double* q0);

/* Variable-coefficient acoustics (NEXT-4: heterogeneous media, P:66 and P:640;
 * the per-system normal / transverse Riemann solvers of P:433-436 with the
 * matrices A, B of P:457-466 varying from cell to cell; R20).
 * aux = [patch][2][my][mx] fp64 (rho, K per interior cell, every value finite
 * and > 0) for ALL npatch patches of the level, in global patch order, on
 * every rank (the medium is part of the problem description, like the
 * descriptors); copied during the call.  The library stores (Z = rho c,
 * c = sqrt(K/rho)) per cell in device memory, 16 B per cell, next to q; ghost
 * cells take their medium by the composite rule (BC map, same-level copy),
 * exactly as q.  From then on claw_advance_level solves every face's Riemann
 * problem with the two cells' own media (W1 at -c_l in the left medium, W2 at
 * +c_r in the right one), splits transverse fluctuations with the media of
 * the cells across each transverse edge, and returns the Courant number as the
 * max over every swept face of max(c_l, c_r) dt/dx (dt/dy); the descriptors'
 * rho, K are then ignored.  claw_patch_cfl gives each patch's max over its own
 * faces.  Requirements (EINVAL otherwise): level 1 set as one uniform grid of
 * equal patches covering the domain (claw_level_mode 1; with world > 1 its
 * band partition -- each rank then keeps its band's medium and the medium of
 * its four halo rows, which is static, so nothing is exchanged), no finer
 * level; a later claw_set_level(2..) or claw_regrid is refused while the
 * medium is set, and claw_set_level(1) discards it. */
int claw_set_aux(claw_ctx* ctx, int32_t level, const double* aux);

/* Ghost fill at time t: same-level and physical-BC ghosts are read
 * by the step kernel straight from their donors' interiors; this call fills
 * the ghost cells that need work: space-time interpolation from level-1's two
 * time levels (t must lie in level-1's [t_old, t_new], else ESTATE), and for
 * world > 1 the NCCL halo exchange with neighbouring ranks. */
int claw_fill_ghost(claw_ctx* ctx, int32_t level, double t);

/* One step of eq. (W) on every owned patch of `level` with time step
 * dt (>= 0): x/y Riemann solves, wave limiter, second-order corrections,
 * transverse propagation and flux-difference update in ONE fused kernel
 * launch, plus the per-patch max Courant number nu = |s| dt/dx (P:230-232,
 * P:417-420) reduced on the device to the level max (and across ranks with an
 * NCCL max all-reduce).  *cfl_max receives it (8-byte device-to-host copy;
 * the only per-step host synchronisation).  cfl_max > 1 is returned, not
 * rejected.  dt = 0 leaves q unchanged and gives cfl_max = 0. */
int claw_advance_level(claw_ctx* ctx, int32_t level, double dt, double* cfl_max);

/* Same as claw_advance_level without the host synchronisation; the result is
 * fetched later with claw_wait_cfl (for CUDA-graph / pipelined drivers). */
int claw_advance_level_async(claw_ctx* ctx, int32_t level, double dt);
int claw_wait_cfl(claw_ctx* ctx, int32_t level, double* cfl_max);

/* The current time level q^n of one owned patch's interior (the
 * patch's state; eq. (W)'s Q_ij), [3][my][mx] fp64 host array of
 * 3*mx*my doubles the caller owns; synchronous (device->host copy, stream
 * synchronised).  EINVAL: patch out of range or not owned here, NULL
 * pointer; ESTATE: level not set.  claw_write is the inverse (host->device;
 * the values become q^n of the next step; a test/helper entry). */
int claw_read(claw_ctx* ctx, int32_t level, int32_t patch, double* q_out);
int claw_write(claw_ctx* ctx, int32_t level, int32_t patch, const double* q_in);
/* The owned patches' level array (see conventions above): the same for all
 * owned patches of the level in one copy (the bench's e2e path). */
int claw_read_level(claw_ctx* ctx, int32_t level, double* q_out);
int claw_write_level(claw_ctx* ctx, int32_t level, const double* q_in);
/* [3][my+4][mx+4]: the patch with its ghost frame exactly as the step kernel
 * sees it after claw_fill_ghost (ghost-fill parity checks). */
int claw_read_padded(claw_ctx* ctx, int32_t level, int32_t patch, double* q_out);
/* Per-patch max Courant number of the last step (owned patches). */
int claw_patch_cfl(claw_ctx* ctx, int32_t level, int32_t patch, double* cfl);

/* Which rank owns (advances, stores) patch `patch` of `level` under the
 * claw_partition map (patches partitioned by cell-count balance, BASELINE
 * north_star; the paper is single-GPU and cites multi-GPU AMR codes).
 * Host-only lookup; EINVAL for a bad level / patch / NULL. */
int claw_owner(const claw_ctx* ctx, int32_t level, int32_t patch, int32_t* rank);
/* Kernel path chosen for a level: 0 generic ghost-table kernel, 1 grid kernel
 * (see claw_config.path), 2 grid kernel on a sparse lattice (a finer level of
 * equal, lattice-aligned patches: one rank, one medium; coarse ghost values are
 * kept in the lattice's empty slots). */
int claw_level_mode(const claw_ctx* ctx, int32_t level, int32_t* mode);

/* Updating: every level-(level-1) cell whose R x R
 * children are all interior cells of `level` is overwritten by their mean
 * (children summed row by row, divided by R*R).  Both levels must be at the
 * same time (else ESTATE).  Single rank. */
int claw_update_level(claw_ctx* ctx, int32_t level);
/* With claw_config.reflux = 1 the update is followed by the conservation fix
 * (Step 7 of the paper's flow chart): every level-(level-1) cell C
 * not covered by `level` that shares an edge E with a covered cell receives
 * the register of E, which the steps have filled with
 *   + dt/dx (fm or -fp through E as C's own update used it)   [coarse step]
 *   - sum over the R fine edges of E and the fine sub-steps of
 *     (dt_f/dx)/R (fp + f(Q_fine) - f(Q_C^n))  (mirror for C right/above E)
 * -- the paper's C1 + C2 + C3 terms (eq:c123) with the coarse flux replaced
 * by the space-time average of the fine fluxes -- and the register is
 * cleared.  Call order: Berger-Oliger (level-1 step, its R level steps, then
 * this call), as claw_advance_hierarchy does.
 *
 * Registers of fine level `level` (tests): *n = count; edges[8e..8e+7] =
 * coarse patch, C's local i, j, dir (0 x, 1 y), side (0: C left/below E),
 * fine patch, local i, j of the first fine cell along E (may be NULL);
 * acc[3e..3e+2] = the accumulated values (device copy; may be NULL). */
int claw_reflux_registers(claw_ctx* ctx, int32_t level, int64_t* n, int32_t* edges, double* acc);

#define CLAW_HIER_UPDATE 1   /* claw_advance_hierarchy: average each finer level onto
                                its coarser one when it has caught up */

/* One coarse step of the whole hierarchy, level by level with subcycling
 * (P:113-118): level 1 advances by dt, then every finer level L+1 R_L times
 * with dt / prod(R), each level step preceded by its ghost fill at its own
 * time; with CLAW_HIER_UPDATE in flags, level L+1 is averaged onto level L
 * after its R_L steps.  Runs entirely on the library's stream with one host
 * synchronisation at the end; *cfl_max receives the max Courant number over
 * all level steps.  Ratios are taken from the levels' dx.  With world > 1
 * that value is reduced across ranks once per call (one 8-byte NCCL max
 * all-reduce per call, not per level step); the levels' own CFL slots
 * (claw_wait_cfl) then hold rank-local maxima.  With exchange = 1
 * (external) the hierarchy drivers move no halo or update data and reduce
 * nothing across ranks: drive the levels with the level calls and
 * claw_halo_* / claw_update_* instead (timing tools use it to run one rank's
 * launches alone). */
int claw_advance_hierarchy(claw_ctx* ctx, double t, double dt, int32_t flags, double* cfl_max);
/* nsteps consecutive coarse steps at the fixed dt (times t + k dt), each
 * exactly as claw_advance_hierarchy would run it, with ONE host
 * synchronisation at the end instead of one per coarse step: the launches of
 * all steps are queued back to back, the per-step Courant numbers land in
 * device slots (one memset for the batch) and cfl_out[k] (host array of
 * nsteps doubles) receives the max Courant number of coarse step k.  The
 * caller checks them afterwards (dt_next = dt nu / cfl; a step
 * with cfl > 1 is to be retaken from saved data, as for the single-step
 * call).  With world > 1 the nsteps values are reduced across ranks by one
 * all-reduce at the end.  A single level (level 1 only) is a valid
 * hierarchy: K level steps per host synchronisation.  EINVAL: nsteps < 1 or
 * cfl_out NULL. */
int claw_advance_hierarchy_n(claw_ctx* ctx, double t, double dt, int32_t nsteps, int32_t flags, double* cfl_out);
int claw_level_owned(const claw_ctx* ctx, int32_t level, int32_t* npatch_owned,
                     int64_t* cells_owned, int64_t* device_bytes);

/* ---- Regridding ("every K time steps ... cells are flagged for
 * refinement ... clustered into new rectangular grid patches"; S:219-290;
 * DESIGN.md R18).  Single rank.  Levels are described on their own index
 * space [0,nx) x [0,ny) (nx = domain width / dx); maps are [ny][nx] uint8,
 * x fastest. ---- */

/* Index-space extent of a set level. */
int claw_level_extent(const claw_ctx* ctx, int32_t level, int64_t* nx, int64_t* ny);
/* Number of patches of `level` (0 if unset) and their descriptors (the
 * level's current patch list, e.g. after claw_regrid). */
int claw_level_count(const claw_ctx* ctx, int32_t level, int32_t* npatch);
int claw_level_descs(const claw_ctx* ctx, int32_t level, claw_patch_desc* out);

/* Flag cells of `level` on the device.  A cell is flagged when its pressure
 * differs from one of its four edge neighbours by more than tol (undivided
 * gradient; neighbours are the composite values the step kernel reads
 * -- call claw_fill_ghost(level, t) first for coarse-interpolated ghosts).
 * The flags are then dilated by `buffer` cells in the Chebyshev metric
 * (S:243-250), clipped to the index space and to
 *   clip 0: nothing more; clip 1: the level's own cells; clip 2: the nesting
 *   mask -- level cells whose in-domain neighbours within Chebyshev distance 2
 *   all belong to the level (a fine box inside it has coarse donors for its
 *   interpolation and its ghost frame).
 * flags_out: host [ny][nx] (may be NULL); *nflag: set cells (may be NULL). */
int claw_flag(claw_ctx* ctx, int32_t level, double tol, int32_t buffer, int32_t clip,
              uint8_t* flags_out, int64_t* nflag);

/* Berger-Rigoutsos clustering of a host flag map (host-only, no context):
 * boxes[4k..4k+3] = (i0, j0, w, h) cover every flag exactly once.  Rules
 * (R18): shrink to the flags' bounding box; accept when the
 * efficiency flags/area >= cutoff and w, h <= max_dim; else cut at a hole of
 * the row/column signature, else at the strongest inflection of its second
 * difference, else at the middle of the longer side, each cut leaving >=
 * min_dim cells on both sides (none possible: accept).  EINVAL unless
 * 0 < cutoff <= 1, max_dim >= 2 min_dim >= 2.  *nbox is always set; ENOMEM
 * (boxes untouched past cap) if more than cap boxes. */
int claw_cluster(const uint8_t* flags, int64_t nx, int64_t ny, double cutoff, int32_t max_dim,
                 int32_t min_dim, int32_t* boxes, int32_t cap, int32_t* nbox);

/* Replace level+1 by the boxes (in level's index space) refined by R
 * (P:110-111).  A new fine cell takes the value of the old level+1 cell at
 * the same place if there is one, else the R10 coarse interpolation
 * from `level` at its current time (the ghost-fill formula with alpha = 1).
 * Levels finer than level+1 are discarded -- but kept as the copy sources of
 * the regrid that re-creates them next, until any level advances, so a regrid
 * of levels 1, 2, ... in turn keeps every level's old data (R18);
 * nbox = 0 just removes them.  The
 * new level's time is level's t_new.  EINVAL: box outside the index space or
 * overlapping another; ENEST: a cell to interpolate has no coarse donor, or a
 * ghost cell of the new level none.  Device memory comes from the library's
 * caching pool (no cudaMalloc when a similar level was freed before). */
int claw_regrid(claw_ctx* ctx, int32_t level, int32_t nbox, const int32_t* boxes, int32_t R);

/* The whole regrid of level+1 in one call: claw_flag(level, tol, buffer,
 * clip 2) on the device, the flag map to the host, claw_cluster, each box
 * split into the row-run rectangles of the nesting mask (identical runs of
 * consecutive rows merged; pieces without flags dropped), then claw_regrid.
 * *nbox receives the number of new patches (may be NULL). */
int claw_regrid_auto(claw_ctx* ctx, int32_t level, double tol, int32_t buffer, double cutoff,
                     int32_t max_dim, int32_t min_dim, int32_t R, int32_t* nbox);

/* Host-only introspection of the ghost-source tables (works with device=-1):
 * for every cell of the padded frame of `patch`, out[(j+2)*(mx+4)+(i+2)]
 * receives the global patch index whose interior supplies the value
 * (patch*2^32 + local_j*2^16 + local_i), or -1 for coarse-interpolated cells,
 * or -2 for cells received from another rank (their donor is then in
 * out2, may be NULL). */
int claw_debug_ghost_sources(const claw_ctx* ctx, int32_t level, int32_t patch,
                             int64_t* out, int64_t* out2);
/* External halo exchange (claw_config.exchange = 1): pack the cells this rank
 * sends to `peer` into host_out ([3][nsend], component-major, in the plan's
 * order), or place the cells received from `peer` (host_in, [3][nrecv]) into
 * this rank's ghost frames.  Synchronous. */
int claw_halo_pack(claw_ctx* ctx, int32_t level, int32_t peer, double* host_out);
int claw_halo_unpack(claw_ctx* ctx, int32_t level, int32_t peer, const double* host_in);

/* Halo exchange plan: number of cells this rank sends to / receives from
 * `peer` for `level`. */
int claw_debug_halo_counts(const claw_ctx* ctx, int32_t level, int32_t peer,
                           int64_t* nsend, int64_t* nrecv);
/* The k-th cell sent to `peer`: global donor patch and local (i, j). */
int claw_debug_halo_send(const claw_ctx* ctx, int32_t level, int32_t peer,
                         int64_t k, int32_t* patch, int32_t* i, int32_t* j);

/* Update exchange of the partitioned level `level` (claw_config.dist_level
 * >= 2) with exchange = 1 (the coarse level takes the average of
 * its children; it is replicated on every rank, so each rank's averages must
 * reach every replica).  After claw_update_level(level) on every rank:
 * claw_update_pack writes the level-(level-1) cells this rank's patches
 * averaged into host_out ([3][n], component-major, in patch / rectangle /
 * row-major order); claw_update_unpack writes rank `peer`'s pack into this
 * rank's replica.  Synchronous.  EINVAL: `level` not the partitioned level,
 * peer out of range or this rank, NULL buffer.  With exchange = 0
 * claw_update_level does the same through NCCL itself. */
int claw_update_pack(claw_ctx* ctx, int32_t level, double* host_out);
int claw_update_unpack(claw_ctx* ctx, int32_t level, int32_t peer, const double* host_in);
/* Update exchange plan: the number of cells this rank sends (to every peer)
 * and the number it receives from `peer` (0 for peer = this rank, and 0 and 0
 * for a level that is not partitioned). */
int claw_debug_update_counts(const claw_ctx* ctx, int32_t level, int32_t peer,
                             int64_t* nsend, int64_t* nrecv);

/* The process-wide device memory pool every context allocates from (the
 * paper's GPU memory pool): per device, chunks from cudaMalloc (the
 * first 1 GiB, each new one at least the size of all chunks so far, up to
 * 2 GiB, or the request if larger) carved best-fit with coalescing frees.  hits = requests served
 * from free ranges, misses = requests that needed a new chunk, cached_bytes =
 * free bytes held.  Wholly free chunks beyond CLAW_POOL_LIMIT_MB (environment,
 * default 16384) of free memory are returned to the driver; claw_pool_trim
 * returns every wholly free chunk (call with no kernel of the library in
 * flight). */
int claw_pool_stats(int64_t* hits, int64_t* misses, int64_t* cached_bytes);
int claw_pool_trim(void);

int claw_set_profiling(claw_ctx* ctx, int32_t on);
int claw_get_stats(claw_ctx* ctx, claw_stats* out);   /* synchronises */
int claw_reset_stats(claw_ctx* ctx);
int claw_synchronize(claw_ctx* ctx);

/* Create an NCCL unique id (128 bytes) on one rank, to be broadcast to all
 * ranks by the caller (e.g. torch.distributed) before claw_create.  ENCCL if
 * NCCL cannot be loaded. */
int claw_nccl_unique_id(void* out128);

/* The context's NCCL communicator as NCCL itself reports it (ncclCommCount,
 * ncclCommUserRank, ncclCommCuDevice): multi-GPU runs log it so the rank
 * count and device mapping are checked, not assumed.  ESTATE if the context
 * has no NCCL communicator (world = 1 or exchange = 1) or the loaded NCCL
 * lacks these calls; ENCCL if NCCL fails. */
int claw_comm_info(const claw_ctx* ctx, int32_t* nranks, int32_t* rank, int32_t* cuda_device);

/* Library version / build string (host-only). */
const char* claw_version(void);

#ifdef __cplusplus
}
#endif
#endif
