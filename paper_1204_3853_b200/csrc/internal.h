// Internal declarations of libvlasov (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <utility>
#include <memory>
#include <string>
#include <vector>

#include "vlasov.h"

namespace vk {

constexpr int G = 2;              // ghost width (reading #7)
constexpr int GX_PAD = 16;        // padding of the periodically extended Green's function gX
constexpr int GX_TAIL = 176;      // gX continues periodically past 2n + GX_PAD for unwrapped rows
constexpr int MAXR = 16;          // largest refinement ratio per dim supported by the transfers

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_check(cudaError_t e, const char* what);
#define VK_CUDA(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) return ::vk::cuda_check(_e, #call); } while (0)
// Level / plan metadata is allocated stream-ordered (cudaMallocAsync on the owner's stream, pooled):
// a regrid's level create / destroy then neither blocks on cudaMalloc nor synchronises the device.
inline void dfree(void* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}
#define VK_LAUNCH(what) do { cudaError_t _e = cudaGetLastError(); if (_e != cudaSuccess) return ::vk::cuda_check(_e, what); } while (0)

// Launch with programmatic dependent launch allowed: the kernel may start while the previous
// kernel on the stream retires, so it must execute griddep_wait() (ptx.cuh) before it reads
// anything earlier kernels wrote.  The small AMR / field kernels call griddep_wait() and
// griddep_launch_dependents() first thing, so their launch latencies overlap along the stream.
#ifndef VK_PDL
#define VK_PDL 1
#endif
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = VK_PDL;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ boxes
struct Box {
    int lo[4] = {0, 0, 0, 0}, hi[4] = {-1, -1, -1, -1};
};
int box_ncells_dim(const Box& b, int d);
int64_t box_ncells(const Box& b, int nd);
bool box_empty(const Box& b, int nd);
Box box_intersect(const Box& a, const Box& b, int nd);
bool box_contains(const Box& b, const int* c, int nd);
Box box_refine(const Box& b, const int* r, int nd);
Box box_coarsen(const Box& b, const int* r, int nd);
Box box_grow(const Box& b, int g, int nd);
std::vector<Box> box_subtract(const Box& a, const Box& b, int nd);
bool box_less(const Box& a, const Box& b, int nd);
int64_t box_index(const Box& b, const int* c, int nd);   // row-major, last dim fastest
inline int floordiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

// ------------------------------------------------------------------ device task structs
struct Block1 {               // one storage block of a 1D+1V level
    int64_t off;              // index of the ghosted origin (x = lo-2, v = lo-2)
    int32_t pitch;            // doubles per ghosted x-row
    int32_t lo_x, lo_v, nx, nv;
};
struct Tile1 {                // one CTA of the 1D+1V stage kernel
    int32_t block, x0, nrows, j0, ncols;
    int32_t pvt, strip;       // v-tile index and row-strip index (moment partials; single block)
};
struct CFTask {               // one coarse-fine ghost value
    int64_t dst;              // fine index in the level array
    int64_t csrc;             // coarse index of the parent cell in the coarse level array
    int32_t cstride[4];       // coarse strides (doubles) per dim
    int8_t sub[4];            // sub-cell offsets per dim
};
struct PhysTask {             // characteristic v-BC of one column side (1D+1V)
    int64_t cell0;            // index of the boundary cell (j = 0 for low, j = n-1 for high)
    int32_t e_idx;            // index into the level E array (wrapped x + 2)
    int32_t side;             // 0 low, 1 high
};
struct RedCol {               // one grown x-column of one Alg.8 sub-patch
    int64_t addr;             // index of the column's first velocity cell in its level array
    int32_t nv;               // velocity cells summed (the sub-patch's v extent)
    int32_t level;            // index of the level in the hierarchy
    int32_t j0;               // level velocity index of the column's first cell (first moment)
};
struct RedContrib {           // one refined partial sum landing on one finest x cell
    int64_t cs;               // index of the first of the 5 stencil column sums (columns c-2..c+2)
    double dv;                // velocity spacing of the sub-patch's level (reading #13)
    double b[5];              // linear5 weights b_j(s), j = -2..2 (reading #12)
};
struct FaceRef {              // a face flux stencil in a level array
    int64_t s0;               // first of the 4 cells along the face normal
    int32_t pitch;            // x stride of the block holding the stencil
    int32_t g;                // x-faces: global v index j (vbar_j); v-faces: E index of the column
};
struct RefluxTask {           // one coarse face on the coarse-fine interface
    int64_t ccell;            // uncovered coarse cell whose face is corrected
    int32_t dir;              // 0: x-face, 1: v-face
    int32_t sign;             // +1: the face is the cell's high face, -1: its low face
    int32_t nfine;            // fine faces under the coarse face (transverse ratio)
    int32_t pad;
    FaceRef cf;               // coarse face stencil
    FaceRef ff[MAXR];         // fine face stencils
};
struct AvgTask {              // one covered coarse cell (reading #14)
    int64_t ccell;
    int64_t fcell0;           // first fine cell
    int32_t fpitch;           // fine x stride
    int32_t pad;
};

// ---- 2D+2V hierarchies (NEXT row N3) ----
struct PhysTask4 {            // characteristic velocity BC of one 2D+2V column side (reading #6)
    int64_t cell0;            // boundary cell (velocity index 0 or n-1 along vd) in the level array
    int32_t stride;           // level-array stride along vd (doubles)
    int32_t e_idx;            // level E array index: component vd-2, wrapped (x, y) + 2 ghosts
    int32_t p_idx;            // f0v index of the first ghost layer (vd index -1 or n)
    int16_t side;             // 0 low, 1 high
    int16_t pstep;            // f0v stride along vd
};
struct Red4Col {              // one grown (x, y) column of one 4D Alg.8 sub-patch
    int64_t addr;             // index of the column's first velocity cell (lo_vx, lo_vy)
    int32_t nvx, nvy;         // the sub-patch's velocity extent
    int32_t s2;               // vx stride of the patch's block
    int32_t level;
};
struct Red4Contrib {          // one refined 2D partial sum landing on one finest (x, y) cell
    int64_t cs;               // column (x_c - 2, y_c - 2) of the sub-patch's grown grid
    int32_t ystride;          // columns per grown x row (n_y of the sub-patch + 4)
    int32_t pad;
    double dvv;               // dvx dvy of the sub-patch's level (reading #13)
    double bx[5], by[5];      // linear5 weights of the finest cell's sub-offsets (reading #12)
};
struct Mask4Item {            // Alg.6 4D: one finest (x, y) cell of one patch's refined footprint
    int64_t addr;             // cell (x_c - 2, y_c - 2, lo_vx, lo_vy) of the patch
    int64_t mask;             // patch-mask offset of (x_c, y_c, 0, 0)
    int32_t s0, s1, s2;       // block strides of x, y, vx
    int32_t nvx, nvy, level;
    int32_t mstride0, mstride1;   // mask strides of x, y (nvx nvy ny, nvx nvy)
    int32_t wx, wy;           // offsets of the 5 linear5 weights (x, y) in the weight table
};

struct Patch4 {               // one patch of a 2D+2V level (N3 stepping in the F* form)
    int64_t org;              // index of its interior cell lo in the level array
    int64_t s[3];             // strides of x, y, v_x (v_y: 1)
    int32_t lo[4], n[4];      // box lo and cells per dim (level index space)
    int64_t foff[4];          // offsets of its 4 face arrays in the level's F* buffer
};
struct FaceAvgTask {          // Alg.4: one coarse F* face := mean of the R^3 fine faces over it
    int64_t coarse, fine;     // coarse face index; first fine face
    int64_t st[3];            // fine face strides of the 3 transverse dims
    int32_t r[3], pad;
};
struct AvgTask4 {             // average-down: one covered coarse cell := mean of R^4 fine cells
    int64_t coarse, fine;
    int64_t st[3];            // fine strides of x, y, v_x (v_y: 1)
    int32_t r[4];
};

constexpr int MAXLEV = 8;     // levels of one hierarchy handled by the reduction
struct RedPlan {              // Alg.8 sub-patch reduction plan (built on the host, level.cpp)
    std::vector<uint64_t> uids;   // the hierarchy it was built for
    cudaStream_t st = nullptr;    // stream its device arrays were allocated on (stream-ordered)
    int nxf = 0;                  // finest configuration cells
    int64_t ncols = 0, ncontrib = 0;
    RedCol* d_cols = nullptr;
    double* d_colsum = nullptr;
    RedContrib* d_contrib = nullptr;
    int32_t* d_xoff = nullptr;    // CSR over finest x [nxf + 1]
};
void free_red_plan(RedPlan* p);

struct MaskCol {              // Alg.6: one coarse x column of one patch, refined by R in x
    int64_t addr;             // index of cell (x_c - 2, lo_v) of the patch in its level array
    int64_t mask;             // index of (x_c, lo_v) in the hierarchy mask buffer
    int32_t pitch, nv, level, R;
    int32_t out;              // first of the R partial sums of this column
    int32_t woff;             // offset of the R x 5 linear5 weights in the weight table
};
struct MaskPlan {             // Alg.6 Mask Reduction plan (comparator of Alg.8)
    std::vector<uint64_t> uids;
    cudaStream_t st = nullptr;
    int nxf = 0;
    int64_t ncols = 0, npart = 0;
    MaskCol* d_cols = nullptr;
    uint8_t* d_mask = nullptr;    // mu per level (1: not covered by the next finer level)
    double* d_w = nullptr;        // linear5 weights per distinct R
    double* d_part = nullptr;     // partial sums
    int32_t* d_xoff = nullptr;    // CSR over finest x
    int32_t* d_idx = nullptr;     // partial index per contribution
    double* d_dv = nullptr;       // dv of the contribution's level
};
void free_mask_plan(MaskPlan* p);
struct RedPlan4 {             // 4D -> 2D Alg.8 plan (N3)
    std::vector<uint64_t> uids;
    cudaStream_t st = nullptr;
    int nxf = 0, nyf = 0;
    int64_t ncols = 0, ncontrib = 0;
    Red4Col* d_cols = nullptr;
    double* d_colsum = nullptr;
    Red4Contrib* d_contrib = nullptr;
    int32_t* d_off = nullptr;     // CSR over finest (x, y) [nxf nyf + 1]
};
struct MaskPlan4 {            // 4D -> 2D Alg.6 plan (N3 comparator)
    std::vector<uint64_t> uids;
    cudaStream_t st = nullptr;
    int nxf = 0, nyf = 0;
    int64_t nitems = 0;
    Mask4Item* d_items = nullptr;
    uint8_t* d_mask = nullptr;    // mu per patch cell (1: not covered by the next finer level)
    double* d_w = nullptr;        // linear5 weight table
    double* d_part = nullptr;     // per-item partial sums
    double* d_dvv = nullptr;      // dvx dvy per item
    int32_t* d_off = nullptr;     // CSR over finest (x, y)
    int32_t* d_idx = nullptr;     // item index per contribution
};
void free_red_plan4(RedPlan4* p);
void free_mask_plan4(MaskPlan4* p);
int launch_reduce_subpatch4(const RedPlan4* P, const double* const* f, int nlev, double* rho, cudaStream_t st);
int launch_reduce_mask4(const MaskPlan4* P, const double* const* f, int nlev, double* rho, cudaStream_t st);
int launch_fill4(vlasov_level* L, double* f, const double* f_coarse, const double* E_bc, const double* f0v, int interp);
int launch_stage4_fstar(const vlasov_level* L, int stage, double dt, const double* f_n, const double* f_s,
                        double* f_next, const double* E, int recon, double* Fstar);
int launch_fstar_update(const vlasov_level* L, double dt, const double* f_n, const double* Fstar, double* f_new);
int launch_fstar_coarsen(const vlasov_level* L, const double* F_fine, double* F_coarse);
int launch_average_down4(const vlasov_level* L, const double* f_fine, double* f_coarse);
int launch_reduce_mask(const MaskPlan* P, const double* const* f, int nlev, double* rho, cudaStream_t st);
}  // namespace vk

// ------------------------------------------------------------------ opaque structs
struct vlasov_level {
    int ndim = 2, ncfg = 1;
    double moment_base = 1.0;             // fused stage moment: rho = moment_base - dv sum_v f
    int vphys[2] = {1, 1};                // velocity faces that are physical boundaries (lo, hi)
    double lower[4] = {0, 0, 0, 0}, h[4] = {0, 0, 0, 0};
    int ratio[4] = {1, 1, 1, 1};
    int dom[4] = {0, 0, 0, 0};            // level domain cells per dim
    std::vector<vk::Box> boxes;           // logical patches
    std::vector<int> patch_block;         // patch -> block
    std::vector<vk::Box> blocks;          // storage blocks (interior boxes)
    std::vector<int64_t> block_off;       // ghosted-origin offset per block
    std::vector<std::array<int64_t, 4>> block_str;  // strides per block
    int64_t field_doubles = 0;
    const vlasov_level* coarser = nullptr;
    uint64_t uid = 0, coarser_uid = 0;
    cudaStream_t stream = nullptr;
    bool single_block = false;            // one block covering the whole domain
    // 1D+1V stage tables
    std::vector<vk::Block1> h_blocks1;
    vk::Block1* d_blocks1 = nullptr;
    std::vector<vk::Tile1> h_tiles_wide, h_tiles_narrow;
    vk::Tile1* d_tiles_wide = nullptr;
    vk::Tile1* d_tiles_narrow = nullptr;
    int tile_rows = 0;
    int n_vtiles = 0;                     // partial v-tiles (single-block only)
    int n_strips = 0;
    int cluster_size = 1;                 // v-tiles per cluster of the fused-field stage launch
    double* d_partials = nullptr;         // moment scratch [n_vtiles][dom_x]
    uint8_t* d_rawtags = nullptr;         // raw tags of a multi-patch level (level domain)
    unsigned* d_tickets = nullptr;        // per-strip arrival tickets
    double* d_scalar = nullptr;           // one device double (max|E| of vlasov_next_dt)
    bool self_ghost_ok = false;           // single periodic block, nv % 4 == 0: in-kernel ghosts
    // ghost fill
    int64_t n_copy = 0, n_cf = 0, n_phys = 0;
    int64_t* d_copy = nullptr;            // pairs (dst, src)
    vk::CFTask* d_cf = nullptr;
    vk::PhysTask* d_phys = nullptr;
    int coarse_ratio[4] = {1, 1, 1, 1};   // ratio to the coarser level
    // AMR transfers w.r.t. the coarser level
    int64_t n_reflux = 0, n_avg = 0;
    vk::RefluxTask* d_reflux = nullptr;
    int64_t* d_reflux_cells = nullptr;    // CSR: distinct corrected coarse cells [n_reflux_cells]
    int32_t* d_reflux_off = nullptr;      //      task range per cell [n_reflux_cells + 1]
    int64_t n_reflux_cells = 0;
    vk::AvgTask* d_avg = nullptr;
    int avg_count = 1;                    // fine cells per coarse cell
    // Alg.8 plan cached on the finest level of the hierarchy it was built for
    mutable vk::RedPlan* red_plan = nullptr;
    mutable vk::MaskPlan* mask_plan = nullptr;
    mutable vk::RedPlan4* red_plan4 = nullptr;
    mutable vk::MaskPlan4* mask_plan4 = nullptr;
    // 2D+2V multi-patch levels (N3): velocity BC tasks, v_x pass first
    vk::PhysTask4* d_phys4 = nullptr;
    int64_t n_phys4[2] = {0, 0};
    bool ghost4_built = false;            // task lists of a 2D+2V level (built lazily for a single block)
    vk::Patch4* d_patch4 = nullptr;       // F*-form stepping of 2D+2V levels
    int64_t face_doubles = 0;             // size of the level's F* buffer
    int64_t max_patch_cells = 0;
    vk::FaceAvgTask* d_fcoarsen4 = nullptr;   // Alg.4 flux coarsening into the coarser level
    int64_t n_fcoarsen4 = 0;
    vk::AvgTask4* d_avg4 = nullptr;       // average-down into the coarser level
    int64_t n_avg4 = 0;
    // 2D+2V
    int64_t e_doubles = 0;
    int strips2 = 1;                      // x strips of the 2D+2V stage kernel
    int tel_ns = 0;                       // strips of the telescoped 2D+2V kernel (0: not chosen yet)
    int tel_xb[33] = {0};                 // their boundaries (stage2d_tel.cu)
    int acc_ns = 0;                       // the same for the accumulator-form kernel (stage2d_acc.cu)
    int acc_xb[33] = {0};
    // scratch (device): interpolation tables
    double* d_b5 = nullptr;               // linear5 weights for coarse_ratio, [dim][s][5]
};

struct vlasov_poisson {
    int n = 0;
    double dx = 0;
    cudaStream_t stream = nullptr;
    double* d_gE = nullptr;
    double* d_gphi = nullptr;
    double* d_gX = nullptr;               // gX[m] = gE[(m - GX_PAD) mod n], m < 2n + GX_PAD + GX_TAIL
    double* d_hs = nullptr;               // split field: h(m), m = -16 .. 16 (null: Toeplitz field)
    double K2 = 0.0, Kn = 0.0;            // split field: dx / 2, dx / n
};

struct vlasov_poisson2d {
    int nx = 0, ny = 0;
    double dx = 0, dy = 0;
    cudaStream_t stream = nullptr;
    double* d_gx = nullptr;               // [nx][ny] Green's function of E_x (row-major, (m, n))
    double* d_gy = nullptr;               // [nx][ny] Green's function of E_y
};

namespace vk {
int launch_poisson2d(const vlasov_poisson2d* P, const double* rho, double* E);
// ------------------------------------------------------------------ kernels (launchers)
int launch_stage_1d1v(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s,
                      double* u, double* f_next, const double* E, const double* E_bc,
                      const double* f0v, int recon, double* rho, const double* rho_in = nullptr,
                      const double* gE = nullptr, double* E_out = nullptr, const double* gX = nullptr,
                      const double* hs = nullptr, double K2 = 0.0, double Kn = 0.0);
int launch_stage_2d2v(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s, double* u,
                      double* f_next, const double* E, const double* E_bc, const double* f0v, int recon,
                      double* rho);
bool stage_2d2v_tel_ok(const vlasov_level* L);
int stage_2d2v_choose_strips(int64_t tiles, int nx, int rmax, int smax, const char* env, int* xb);
bool stage_2d2v_acc_ok(const vlasov_level* L);
int launch_stage_2d2v_acc(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s, double* u,
                          double* f_next, const double* E, double* rho_partials);
int launch_stage_2d2v_tel(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s, double* u,
                          double* f_next, const double* E, double* rho_partials);
int launch_moment_2d2v(const vlasov_level* L, const double* f, double* rho);
int stage_1d1v_ctas_per_sm(bool wide, int tile_rows);
int stage_1d1v_tile_width(bool wide);   // cells per v-tile of the stage kernel
int stage_1d1v_max_clusters(bool wide, int tile_rows, int cs, int n);
int launch_fill(vlasov_level* L, double* f, const double* f_coarse, const double* E_bc,
                const double* f0v, int interp);
int launch_moment_direct(const vlasov_level* L, const double* f, double* rho, double q = -1.0, double base = 1.0,
                         int accumulate = 0);
int launch_poisson(vlasov_poisson* P, const double* rho, double* phi, double* E, int ghost);
int launch_inject_1d(const vlasov_level* L, const double* E_finest, int n_finest, double* E_lvl, double scale = 1.0);
int launch_inject_2d(const vlasov_level* L, const double* E_finest, const int32_t* n_finest, double* E_lvl, int gin = 0);
int linear5_weights(int R, double* out /* R*5 */);
int launch_absmax(const double* x, int64_t n, double* out, cudaStream_t st);
int launch_vslab(const vlasov_level* L, double* f, double* lo, double* hi, bool pack);
int launch_current(const vlasov_level* L, const double* f, double q, int accumulate, double* j);
int launch_reduce_first_subpatch(const RedPlan* P, const double* const* f, int nlev, const double* vlo,
                                 const double* dv, double* j, cudaStream_t st, double q, int accumulate);
int launch_reduce_subpatch(const RedPlan* P, const double* const* f, int nlev, double* rho, cudaStream_t st,
                           double q = -1.0, double base = 1.0, int accumulate = 0);
int launch_flux_registers(const vlasov_level* L, const double* f_fine, const double* E_fine, const double* f_coarse,
                          const double* E_coarse, double b_s, double* regs, int recon);
int launch_average_down(const vlasov_level* L, const double* f_fine, double* f_coarse, const double* regs, double dt);
int launch_tags(const vlasov_level* L, const double* f, double tol, int buffer, uint8_t* tags);
struct RectCopy {              // fill_from: one old-patch / new-patch overlap rectangle (1D+1V)
    int64_t dst, src;         // level-array index of the rectangle's first cell (new / old)
    int32_t dpitch, spitch;   // x strides (doubles) of the new / old block
    int32_t nx, nv;
};
int launch_fill_from(const vlasov_level* L, double* f, const double* f_old, const std::vector<RectCopy>& rects,
                     const double* f_coarse, const std::vector<CFTask>& cfs, int interp);
}  // namespace vk
