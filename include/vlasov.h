/*
 * vlasov.h -- C ABI of libvlasov, the B200 (sm_100a, fp64) hot path of the block-structured
 * AMR Vlasov-Poisson method of Hittinger & Banks, arXiv:1204.3853.
 *
 * Citations "P:n" are lines of the paper's text; "reading #k" refers to the list of
 * interpretations of garbled / silent passages in DESIGN.md.
 *
 * ---- Conventions -----------------------------------------------------------------------------
 * Status:     every int-returning call returns VLASOV_OK (0) or a negative VLASOV_E* code; the
 *             message of the last failure on the calling host thread is vlasov_last_error().
 *             Kernel faults are asynchronous: they surface as VLASOV_ECUDA at a later call.
 * Ownership:  every phase-space or configuration-space FIELD array (f, k, u, E, rho, flux
 *             registers, tags) is a caller-owned DEVICE buffer of the length reported by
 *             vlasov_level_get_info(), passed as a raw pointer.  The library owns only level
 *             metadata (box lists, tiles, ghost/transfer task lists, Green's functions) and small
 *             scratch (moment partial sums) on host and device, freed by the matching *_destroy.
 *             No call other than *_create allocates device memory.
 * Streams:    a level (and a Poisson plan) is bound to the cudaStream_t given at creation (passed
 *             as void*; NULL = legacy default stream).  Every compute call is enqueued on that
 *             stream and returns without synchronising, so the calls can be captured in a CUDA
 *             graph.  Only *_create and the host queries block.  One host thread per level.
 * Indexing:   phase space has D = 2*C dims, configuration dims first then velocity dims
 *             (P:1056-1059); C = 1 (1D+1V) or C = 2 (2D+2V).  Boxes are inclusive [lo, hi]
 *              in the level's own global index space; level l is refined by
 *             ratio_to_level0 with respect to level 0.  Configuration dims are
 *             periodic, velocity dims are truncated with the characteristic boundary condition
 *             (P:222-231).  The velocity dim is the fastest-varying (contiguous) one.
 * Layout:     a level stores its cells in one device array of fp64 with a ghost frame of G = 2
 *             cells on every side of every storage block; vlasov_level_layout() reports, per
 *             patch, the offset of the patch's interior cell `lo` and the strides (in doubles).
 *             A level whose boxes exactly tile their bounding box is stored as ONE block (the
 *             patches are then views into it); otherwise each patch is its own block.
 * Precision:  all arithmetic is IEEE fp64.  No CPU fallback exists: without a CUDA device of
 *             compute capability 10.0 every compute call returns VLASOV_ECUDA.
 */
#ifndef VLASOV_H
#define VLASOV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------------------------------- */
#define VLASOV_OK            0
#define VLASOV_EINVAL       -1  /* bad argument or shape (empty box, nboxes < 1, n < 5 for Poisson) */
#define VLASOV_ENOMEM       -2  /* host or device allocation failed                                 */
#define VLASOV_ECUDA        -3  /* CUDA runtime / launch error, or no usable sm_100 device          */
#define VLASOV_ENEST        -4  /* boxes overlap, leave the domain, or are not properly nested      */
#define VLASOV_ESTALE       -5  /* a transfer between levels whose metadata no longer match         */
#define VLASOV_ESTENCIL     -6  /* a coarse-fine stencil needs coarse data outside the coarse level */
#define VLASOV_EUNSUPPORTED -7  /* valid request that this build does not implement                 */

/* ---- options ----------------------------------------------------------------------------------- */
enum { VLASOV_CENTERED4 = 0,   /* ideal weights 1/2, 1/2: centered 4th order face average */
       VLASOV_UPWIND = 1 };    /* WENO provisional weights, larger weight upwind; #4-#5   */
enum { VLASOV_LINEAR5 = 0,     /* unlimited quintic-stencil interpolation b_j(s); #12     */
       VLASOV_WENO5 = 1 };     /* limited WENO5 conservative interpolation; #8-#10        */
enum { VLASOV_GHOST_INTERIOR = 0, VLASOV_GHOST_SIBLING = 1, VLASOV_GHOST_COARSE = 2,
       VLASOV_GHOST_PHYS = 3 };

/* ---- plain data --------------------------------------------------------------------------------- */
typedef struct { int32_t lo[4], hi[4]; } vlasov_box;   /* inclusive; entries >= ndim unused */

typedef struct {
    int32_t    ndim;        /* 2 (1D+1V) or 4 (2D+2V)                                         */
    vlasov_box domain;      /* level-0 index domain, lo = 0                                  */
    double     lower[4];    /* physical coordinate of the domain's lower corner              */
    double     dx0[4];      /* level-0 mesh spacings                                          */
} vlasov_geom;

typedef struct {
    int64_t field_doubles;    /* length of every phase-space field array of this level          */
    int64_t e_doubles;        /* length of this level's E array: C * prod(ncfg_d + 4)             */
    int64_t cfg_cells;        /* configuration cells of this level (prod ncfg_d)                 */
    int64_t fluxreg_doubles;  /* flux-register length of this level w.r.t. its coarser level      */
    int64_t tag_bytes;        /* length of the tag array of vlasov_tag_cells (level domain)      */
    int32_t nblocks, npatches, ntiles, ndim;
    int32_t ratio[4];         /* ratio to level 0                                               */
    int32_t ncfg[2];          /* configuration cells per config dim at this level               */
    int32_t domain_cells[4];  /* level domain cells per dim                                      */
} vlasov_level_info;

typedef struct vlasov_level vlasov_level;
typedef struct vlasov_poisson vlasov_poisson;

/* ---- levels ------------------------------------------------------------------------------------- *
 * Create the metadata of one refinement level from its box list (patch id = index
 * in `boxes`).  Boxes must be disjoint and inside the level domain (refined level-0 domain);
 * `coarser` (NULL for level 0) must be the next coarser level, and the level must be properly
 * nested in it (Fig.1 caption): else VLASOV_ENEST / VLASOV_ESTENCIL.  Level 0 must
 * tile the whole domain.  Builds the ghost-fill, coarse-fine, flux-register and average-down
 * task lists and the stage-kernel tile table, uploads them to the device (on `stream`).       */
int vlasov_level_create(const vlasov_geom* geom, const int32_t ratio_to_level0[4],
                        const vlasov_box* boxes, int32_t nboxes, const vlasov_level* coarser,
                        void* cuda_stream, vlasov_level** out);
int vlasov_level_destroy(vlasov_level* level);
int vlasov_level_get_info(const vlasov_level* level, vlasov_level_info* info);

/* Offset (doubles) of patch `patch`'s interior cell `lo` in the level field array, and the
 * strides (doubles) of that array per dim (entries >= ndim are 0).                             */
int vlasov_level_layout(const vlasov_level* level, int32_t patch, int64_t* offset,
                        int64_t strides[4]);

/* Dense ghost map of patch `patch` over grow(box, 2), row-major (last dim fastest).  Host
 * arrays of prod(size+4) entries.  kind[]: VLASOV_GHOST_*.  src_patch/src_cell:
 *   INTERIOR: patch, row-major index in the patch box;
 *   SIBLING : same-level patch holding the cell after the periodic wrap of the configuration
 *             indices (may be `patch` itself), index of the wrapped cell in it;
 *   COARSE  : coarser-level patch holding the coarse parent of the wrapped cell, index of that
 *             parent in it;
 *   PHYS    : -1, 2*(velocity dim number) + (0 low | 1 high) for the first velocity dim outside
 *             the domain.
 * Precedence (reading #15): PHYS, then SIBLING, then COARSE.                                   */
int vlasov_level_ghost_map(const vlasov_level* level, int32_t patch, int32_t* kind,
                           int32_t* src_patch, int64_t* src_cell);

/* Alg.7 ComputeSubPatches of patch `patch` of levels[level_index] against all
 * finer levels of the hierarchy `levels[0..nlev-1]`; boxes in the patch's index space, sorted
 * lexicographically by (lo, hi).  *n receives the count; at most `cap` are written.          */
int vlasov_subpatches(const vlasov_level* const* levels, int32_t nlev, int32_t level_index,
                      int32_t patch, vlasov_box* out, int32_t cap, int32_t* n);

/* ---- ghost fill (Alg.2) --------------------------- *
 * Fill the ghost frame of every block of `level` in `f`: same-level and periodic copies, then
 * coarse-fine interpolation from `f_coarse` on `coarser` (whose ghosts must be current;
 * `interp` = VLASOV_LINEAR5 | VLASOV_WENO5, dimension by dimension, x first), then the
 * characteristic velocity boundary condition: per configuration column the speed a_d = -E_d
 * (E_bc: this level's E array, reading #6b) decides outgoing (cubic extrapolation, reading #6)
 * or incoming / zero (the cell averages `f0v` of the unperturbed profile on the level's ghosted
 * velocity range: (nv+4) doubles for 1V, (nvx+4)*(nvy+4) for 2V).                              */
int vlasov_fill_ghosts(vlasov_level* level, double* f, const vlasov_level* coarser,
                       const double* f_coarse, const double* E_bc, const double* f0v,
                       int32_t interp);

/* ---- right-hand side and RK4 stage ------------------------------------------------- *
 * vlasov_rhs: k = L(f) on every interior cell (face averages P:322-368, fluxes P:263-282 with
 * the +1/48 reading #3, divergence P:246-250); `f` ghosts must be filled; `E` is this level's
 * E array.  k has the level layout (ghost cells of k untouched); k must not alias f.  2D+2V: one
 * block covering the periodic (x, y) domain (x, y wrapped in-kernel; the velocity ghost frame of f
 * filled, e.g. by vlasov_fill_ghosts with E_bc and f0v); CENTERED4 in the telescoped form.
 *
 * vlasov_rk4_stage: one stage of classic RK4 in the minimum-traffic rearrangement
 * (identical to the flux-accumulation form P:399-410 in exact arithmetic):
 *   stage 1: f_next = f_n + dt/2 k(f_n)                         (f_s == f_n)
 *   stage 2: u = (f_n + f_s)/3 + dt/3 k(f_s);  f_next = f_n + dt/2 k(f_s)
 *   stage 3: f_next = f_n + dt k(f_s)
 *   stage 4: f_next = u + f_s/3 + dt/6 k(f_s)      (f_n is not read; f_next may alias f_n)
 * (u = (f_2 + 2 f_3 - f_n)/3 is everything of the RK4 sum f_{n+1} = (f_2 + 2 f_3 + f_4 - f_n)/3 +
 * dt/6 k(f_4) that stage 4 cannot form from f_s = f_4, so stage 4 reads two fields only:
 * 16 + 32 + 24 + 24 = 96 B per cell per step.)
 * Ghosts of f_s: if f0v is non-NULL the level must be ONE block covering the (periodic) domain
 * with a number of velocity cells divisible by 4; x is wrapped periodically in-kernel (the ghost
 * rows are never read), and the velocity ghosts of f_s follow the characteristic v-boundary
 * condition (reading #6) either derived in-kernel from E_bc (E_bc non-NULL, exactly as
 * vlasov_fill_ghosts(E_bc, f0v) would) or, with E_bc == NULL ("carried ghosts"), read from f_s's
 * velocity ghost columns.  Stage 1 decides the direction with its own field E, which is E(f_n),
 * the end-of-step constraint evaluation of Alg.5 (reading #6b); E_bc is ignored at
 * stage 1 (with E_bc == NULL the carried ghost columns of f_n must hold the outgoing candidate,
 * the cubic extrapolation, wherever E(f_n) is outgoing -- stage 4 writes it there, and so does
 * vlasov_fill_ghosts with E(f_n)).  With f0v non-NULL the stage also writes f_next's velocity
 * ghost columns (interior rows) for the field E of this stage -- the E_bc of the next stage
 * (reading #6b); stage 4 writes the cubic extrapolation -- so a chain of steps with E_bc == NULL
 * needs one vlasov_fill_ghosts of the initial state only.  Only the velocity faces the
 * level marks physical (vlasov_level_set_velocity_faces; default both) get the boundary
 * condition in-kernel; a non-physical face keeps the ghost columns stored in f_s.
 * With f0v == NULL (E_bc must be NULL too) the ghost frame of f_s must have been filled by
 * vlasov_fill_ghosts.
 * rho_next (nullable; single block covering the domain only): receives the velocity moment of
 * f_next, rho = 1 - dv sum_v f_next, fused into the stage: per-(row, v-tile) partial
 * sums combined in a fixed order by the last CTA of each row strip (deterministic).
 * 2D+2V levels (ndim 4): one block covering the periodic (x, y) domain, n_vx % 4 == 0, n_vy even;
 * f0v ([(n_vx + 4)(n_vy + 4)], the unperturbed profile on the ghosted velocity range) and E_bc
 * (the level's ghosted E array) required; the velocity ghosts of f_s follow the characteristic
 * condition with E_bc (reading #6), derived into f_s's velocity ghost frame by a pass before the
 * stage kernel (f_s's ghost frame is written; its interior is not).  rho_next receives
 * 1 - dvx dvy sum_v f_next per (x, y) cell ([nx][ny]), from per-(vx line, vy tile) partials summed
 * in a fixed order (deterministic).                                                             */
int vlasov_rhs(vlasov_level* level, const double* f, const double* E, double* k, int32_t recon);

/* vlasov_rk4_stage_vp: the constraint evaluation of Alg.5 fused into the stage for a
 * uniform 1D+1V level: E_s = -D4 phi(rho_s) (readings #1-#2; the same operator as
 * vlasov_poisson_solve with `plan`) is computed inside the stage kernel from rho_s, the moment of
 * f_s, and written to E_s (the level's ghosted E array), then the stage runs as vlasov_rk4_stage
 * with E = E_s.  Requirements: f0v non-NULL (one periodic block, nv % 4 == 0; E_bc non-NULL or
 * carried ghosts as in vlasov_rk4_stage), plan->n == the level's x cells <= 4096, even,
 * rho_next != rho_s (ping-pong buffers).  One launch per stage instead of two.                  */
int vlasov_rk4_stage_vp(vlasov_level* level, const vlasov_poisson* plan, int32_t stage, double dt,
                        double* f_n, const double* f_s, double* u, double* f_next, const double* rho_s,
                        double* E_s, const double* E_bc, const double* f0v, int32_t recon,
                        double* rho_next);
int vlasov_rk4_stage(vlasov_level* level, int32_t stage, double dt, double* f_n, const double* f_s,
                     double* u, double* f_next, const double* E, const double* E_bc,
                     const double* f0v, int32_t recon, double* rho_next);

/* ---- reduction ------------------------------------------------------ *
 * rho on the finest configuration mesh: rho = 1 - sum_levels dv_l sum_v f (reading #13), from the
 * (host array of) device field pointers f[l] of the hierarchy levels[0..nlev-1].  One level
 * covering the domain: direct velocity sums.  Otherwise Alg.8 Sub-Patch Reduction: x-ghosts of
 * every level must be current; per sub-patch, v-sums including 2 ghost columns in x (reading
 * #16), linear5 refinement to the finest x resolution, deposit; fixed summation order (level,
 * patch, sub-patch).  The sub-patch plan is rebuilt lazily when any level changed.*/
int vlasov_reduce_moment(const vlasov_level* const* levels, int32_t nlev, const double* const* f,
                         double* rho_finest);
/* Several species (one hierarchy each): rho[x] = (accumulate ? rho[x] : base)
 * + q * n[x], n = sum_l dv_l sum_v f the same moment (direct or Alg.8); vlasov_reduce_moment is
 * (q, base, accumulate) = (-1, 1, 0).  Call once per species, the first with accumulate = 0 and
 * base = the background charge.                                                              */
int vlasov_reduce_charge(const vlasov_level* const* levels, int32_t nlev, const double* const* f, double q,
                         double base, int32_t accumulate, double* rho_finest);

/* Current moment toward Vlasov-Maxwell (N4, reading #31) on the finest configuration
 * mesh of a 1D+1V hierarchy: j[x] = (accumulate ? j[x] : 0) + q sum_l dv_l sum_v <v f>, with the
 * fourth-order cell average of the product <v f>_j = vbar_j f_j + (dv/24)(f_{j+1} - f_{j-1}) (the
 * product rule of the fluxes, reading #3).  One block covering the domain: direct v-sums (the
 * velocity ghost columns of f must be current).  Otherwise Alg.8 with the first moment per
 * sub-patch column (the telescoped correction (dv/24)(f_{j1+1} + f_{j1} - f_{j0} - f_{j0-1}) over
 * its v range; x- and v-ghosts current), the same plan and order as vlasov_reduce_moment.  Call
 * once per species (accumulate = 0 for the first).  Deterministic (fixed order).               */
int vlasov_reduce_current(const vlasov_level* const* levels, int32_t nlev, const double* const* f, double q,
                          int32_t accumulate, double* j);

/* Alg.6 Mask Reduction: the same rho by refining every patch in x (linear5 with 2
 * ghost columns), masking the cells covered by the next finer level and summing over v -- the
 * paper's comparator of Alg.8 (sub-patch reduction = 64% of mask-reduction time).
 * Same arguments and plan caching as vlasov_reduce_moment; equal to it up to rounding.          */
int vlasov_reduce_moment_mask(const vlasov_level* const* levels, int32_t nlev, const double* const* f,
                              double* rho_finest);

/* ---- periodic Poisson + E -------------------------------------------------------- *
 * Plan for n >= 5 periodic cells of width dx (1D configuration space).  solve: projects rho to
 * mean zero, solves 30 phi_i - 16(phi_{i+1}+phi_{i-1}) + (phi_{i+2}+phi_{i-2}) = 12 dx^2 rho_i
 * (reading #2) with mean-zero phi, and E_i = -[8(phi_{i+1}-phi_{i-1}) - phi_{i+2} + phi_{i-2}]
 * /(12 dx) (reading #1).  Implemented as circulant convolutions with the exact discrete
 * Green's functions (computed on the host at plan creation).  phi or E may be NULL.  Both are
 * written with `ghost` periodic ghost cells on each side (length n + 2*ghost), so that with
 * ghost = 2 the E of a level at the finest x resolution is produced directly.                  */
int vlasov_poisson_create(int32_t n, double dx, void* cuda_stream, vlasov_poisson** out);
int vlasov_poisson_solve(vlasov_poisson* plan, const double* rho, double* phi, double* E,
                         int32_t ghost);
int vlasov_poisson_destroy(vlasov_poisson* plan);

/* ---- injection ----------------------------------------------------------------- *
 * E_lvl (this level's ghosted E array, 1D) from the finest configuration field E_finest of
 * n_finest cells: mean of the R finest values per level cell, periodic ghosts.
 * For 2D configuration space (prescribed field), E_finest holds C components of n_finest[0] x
 * n_finest[1] cells.                                                                          */
int vlasov_inject_field(vlasov_level* level, const double* E_finest, const int32_t n_finest[2],
                        double* E_lvl);
/* As vlasov_inject_field (1D+1V) times `scale`: for species s the field entering its update is
 * A_s = -(q_s/m_s) E (electrons: scale 1).                                         */
int vlasov_inject_field_scaled(vlasov_level* level, const double* E_finest, const int32_t n_finest[2],
                               double scale, double* E_lvl);

/* ---- AMR transfers -------------------------------------------------------------- *
 * Flux registers of `fine` with respect to its coarser level: for every coarse face on the
 * coarse-fine interface, regs += b_s * (F_coarse - mean of the overlying fine F) evaluated on
 * the stage states (ghosts filled) with the stage field.  Zero them (cudaMemsetAsync) at the
 * start of a step.  vlasov_average_down then applies the Alg.4 flux substitution to the coarse
 * cells next to the interface (f_coarse += +-dt * regs / h) and replaces every coarse cell
 * covered by `fine` by the mean of its fine cells (reading #14).  regs may be NULL
 * in vlasov_average_down (plain average-down).                                                 */
int vlasov_flux_register_accumulate(vlasov_level* fine, const double* f_fine, const double* E_fine,
                                    const double* f_coarse, const double* E_coarse, double b_s,
                                    double* regs, int32_t recon);
int vlasov_average_down(vlasov_level* fine, const double* f_fine, double* f_coarse,
                        const double* regs, double dt);

/* ---- tagging and regrid -------------------------------------------- *
 * tags[cell of the level domain] = (delta1 f + delta2 f > tol) on the level's patches (0 off
 * them), dilated by `buffer` cells (Chebyshev, periodic in configuration dims, clipped in
 * velocity); f ghosts must be filled.  Evaluated without FMA contraction in the fixed order stated in
 * DESIGN.md so that tags are bit-identical to the oracle's.                                      */
int vlasov_tag_cells(vlasov_level* level, const double* f, double tol, int32_t buffer,
                     uint8_t* tags);
/* Host: fixed-tile rule of the C3 workload (reading #18): boxes of `tile` fine cells (fine =
 * level domain refined by `ratio`) whose coarse footprint holds a tag; sorted lexicographically. */
int vlasov_tags_to_boxes(const uint8_t* tags_host, const int32_t domain_cells[4], int32_t ndim,
                         const int32_t ratio[4], int32_t tile, vlasov_box* out, int32_t cap,
                         int32_t* n);
/* Host: tag clustering into rectangular patches ("grouped and expanded minimally";
 * reading #28 in DESIGN.md): signature-based recursive bisection (cut at a hole of the tag
 * signature closest to the centre, else at the strongest inflection of its Laplacian, else at the
 * midpoint of the longest side) until the fill efficiency |tags|/|box| >= `efficiency` and every
 * side is <= largest (P:1495-1515 largest_patch_size); cuts keep >= smallest cells per side
 * (smallest_patch_size).  tags: row-major [shape[0]][shape[1]] (velocity fastest), index (0,0) =
 * level cell `lo`.  Boxes in level index space, disjoint, sorted lexicographically; *n receives
 * the count, at most `cap` are written.  1D+1V only.                                            */
int vlasov_cluster_tags(const uint8_t* tags, const int32_t shape[2], const int32_t lo[2],
                        const int32_t smallest[2], const int32_t largest[2], double efficiency,
                        vlasov_box* out, int32_t cap, int32_t* n);
/* Host: boxes of the next finer level (level index space of the finer level, sorted) from the
 * dilated tags of `level` (row-major over the level domain): tags restricted to the nesting region
 * of `level` (cells whose Chebyshev `nest`-neighbourhood lies in its patches, configuration dims
 * periodic, cells beyond the velocity domain count as covered; Fig.1 caption proper nesting),
 * clustered as vlasov_cluster_tags with smallest / largest given in FINER-level cells (converted
 * by `ratio`, ceil / floor), each cluster intersected with the nesting region (row-run
 * decomposition), refined by `ratio` (reading #28).                                           */
int vlasov_regrid_boxes(const vlasov_level* level, const uint8_t* tags, const int32_t ratio[2],
                        const int32_t smallest[2], const int32_t largest[2], double efficiency,
                        int32_t nest, vlasov_box* out, int32_t cap, int32_t* n);
/* Regrid data motion: interior of every patch of `level` (new) from `old` (same resolution,
 * may be NULL) where the old patches overlap, else by conservative interpolation from
 * `coarser` (ghosts of f_coarse current).                                                         */
int vlasov_level_fill_from(vlasov_level* level, double* f, const vlasov_level* old,
                           const double* f_old, const vlasov_level* coarser,
                           const double* f_coarse, int32_t interp);

/* ---- adaptive time step ("50% of the stability limit"; reading #17) -------------- *
 * out[0] (device) = max_i |x_i| over n doubles, on `cuda_stream`; deterministic.  The drivers form
 * dt = min(cfl / max_l(max|vbar|/dx_l + max|E_l|/dv_l), growth * dt_prev) from it.              */
int vlasov_absmax(const double* x, int64_t n, double* out, void* cuda_stream);
/* vlasov_next_dt: the adaptive step of Alg.1/5 "Compute next dt" ("50% of
 * the local stability condition", growth <= 10%, any decrease; reading #29) for a 1D+1V hierarchy
 * levels[0..nlev-1] (coarse first) with E[l] the ghosted E array of level l (device, dom_x + 4
 * doubles) from the last constraint evaluation:
 *   dt = min(cfl / max_l(vmax / dx_l + max|E_l| / dv_l), growth * dt_prev),
 * vmax = max |cell-centre velocity| over the finest level's velocity domain.  Host call: launches
 * one reduction per level on its stream and synchronises them; *dt_out is written on the host.
 * Errors: EINVAL (null pointers, nlev < 1, non-positive cfl / growth / dt_prev, 2D+2V level).     */
int vlasov_next_dt(const vlasov_level* const* levels, int32_t nlev, const double* const* E, double dt_prev,
                   double cfl, double growth, double* dt_out);

/* ---- 2D periodic field of a 2D+2V problem (NEXT row N3; reading #32) ----------------------- *
 * The paper's 1D fourth-order Poisson discretisation generalised dimension by
 * dimension (as its fluxes and interpolation are):
 *   [30 phi - 16 (phi_{i+-1,k}) + (phi_{i+-2,k})] / dx^2 + [same along k] / dy^2 = 12 rho,
 *   rho projected to mean zero, phi of mean zero, E = -(D4_x phi, D4_y phi).
 * vlasov_poisson2d_create: exact discrete Green's functions of E_x and E_y (host, long double,
 *   uploaded once; nx, ny >= 5, nx ny <= 26000).  Synchronises `cuda_stream`.
 * vlasov_poisson2d_solve: rho (device, nx ny row-major [x][y]) -> E (device, the 2D level field
 *   layout [2][(nx + 4)(ny + 4)]: component, then ghosted x, ghosted y; the 2 periodic ghost
 *   layers are written too); one launch on the plan's stream; deterministic.               */
/* ---- 2D+2V hierarchies in the paper's F* form (NEXT row N3; Alg.3-4) ---- *
 * vlasov_level_face_doubles: doubles of a 2D+2V level's F* buffer (caller-owned device array):
 *   per patch, per dim d, the face array of the patch's cells with n_d + 1 along d (row-major
 *   x, y, v_x, v_y).
 * vlasov_rk4_stage_fstar: stage s of Alg.3 on every patch from the ghosted predictor f_s (ghosts
 *   filled by vlasov_fill_ghosts): the face fluxes (P:263-282 dimension by dimension, +1/48 of
 *   reading #3), F* = b_1 F (s = 1) or F* += b_s F, and f_next = f_n + alpha_{s+1} dt k(f_s)
 *   (interior; stages 1-3; NULL at stage 4).  E: the level's ghosted E array.  f_next must not
 *   alias f_s.
 * vlasov_fstar_coarsen: Alg.4 "coarsen fluxes down to level l-1": every coarse F* face lying
 *   under a face of a patch of `fine` := the mean of the fine F* over it (reading #14; x, y
 *   periodic images).  Call finest -> coarsest before the coarser level's update.
 * vlasov_fstar_update: f_new = f_n + dt div(F*) on the interiors (ComputeUpdate);
 *   f_new may alias f_n.  vlasov_average_down(fine, f_fine, f_coarse, NULL, dt) then sets the
 *   covered coarse cells to the mean of their fine cells.                        */
int vlasov_level_face_doubles(const vlasov_level* level, int64_t* n);
int vlasov_rk4_stage_fstar(vlasov_level* level, int32_t stage, double dt, const double* f_n,
                           const double* f_s, double* f_next, const double* E, int32_t recon,
                           double* Fstar);
int vlasov_fstar_coarsen(const vlasov_level* fine, const double* F_fine, const vlasov_level* coarse,
                         double* F_coarse);
int vlasov_fstar_update(vlasov_level* level, double dt, const double* f_n, const double* Fstar,
                        double* f_new);

/* vlasov_inject_field_ghosted: as vlasov_inject_field for a 2D+2V level, from a finest field in the
 * ghosted level layout [2][(n_finest[0] + 4)(n_finest[1] + 4)] (the output of
 * vlasov_poisson2d_solve): E_lvl (ghosted, periodic ghosts written) = mean over the R_x x R_y
 * finest cells of each level cell.                                 */
int vlasov_inject_field_ghosted(vlasov_level* level, const double* E_finest, const int32_t n_finest[2],
                                double* E_lvl);
typedef struct vlasov_poisson2d vlasov_poisson2d;
int vlasov_poisson2d_create(int32_t nx, int32_t ny, double dx, double dy, void* cuda_stream,
                            vlasov_poisson2d** out);
int vlasov_poisson2d_solve(const vlasov_poisson2d* plan, const double* rho, double* E);
int vlasov_poisson2d_destroy(vlasov_poisson2d* plan);

/* ---- velocity-slab decomposition of a uniform 1D+1V level -------- *
 * Each GPU (rank) owns all x and a contiguous velocity slab, created as its own level (one block,
 * lower[1] = the slab's lower velocity).  Per stage: the fused moment of every slab is reduced
 * over the ranks (sum), and the two velocity ghost columns on each interior slab face are the
 * neighbour's boundary columns (halo exchange).
 * vlasov_level_set_moment_base: the fused stage moment writes rho = base - dv sum_v f_next
 *   (default base 1; a slab decomposition uses 1 on one rank and 0 on the others, so that the
 *   sum over ranks is rho = 1 - dv sum_v f).  One periodic block only.
 * vlasov_vslab_pack: lo[2x + c] = f(x, c), hi[2x + c] = f(x, nv - 2 + c) for c = 0, 1 and every
 *   interior row x (device arrays of 2 nx doubles; either may be NULL).
 * vlasov_vslab_unpack: the inverse into the velocity ghost columns: f(x, -2 + c) = lo[2x + c],
 *   f(x, nv + c) = hi[2x + c] (NULL leaves that side -- a physical boundary -- untouched).      */
int vlasov_level_set_moment_base(vlasov_level* level, double base);
/* vlasov_level_set_velocity_faces: which velocity faces of a one-block periodic level are physical
 * boundaries (1) -- the stage kernels apply the characteristic condition there -- and which are
 * interior slab faces (0) whose ghost columns the caller provides (vlasov_vslab_unpack).  Default
 * (1, 1).                                                                                         */
int vlasov_level_set_velocity_faces(vlasov_level* level, int32_t phys_lo, int32_t phys_hi);
int vlasov_vslab_pack(const vlasov_level* level, const double* f, double* lo, double* hi);
int vlasov_vslab_unpack(const vlasov_level* level, double* f, const double* lo, const double* hi);

/* ---- misc ------------------------------------------------------------------------------------ */
const char* vlasov_last_error(void);
int vlasov_device_ok(void);         /* 1 if a compute-capability 10.x device is current, else 0 */
int vlasov_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VLASOV_H */
