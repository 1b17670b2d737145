// libvlasov host side: errors, box calculus, level metadata (layout, tiles, ghost / transfer task
// lists), Poisson plans, C ABI entry points.  See include/vlasov.h for the contract.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>

#include <nvtx3/nvToolsExt.h>
#include <vector>

#include "internal.h"

using vk::Box;

// ====================================================================== errors
namespace vk {
static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
int fail(int code, const std::string& m) {
    g_err = m;
    return code;
}
int cuda_check(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return VLASOV_ECUDA;
}

// ====================================================================== boxes
int box_ncells_dim(const Box& b, int d) { return b.hi[d] - b.lo[d] + 1; }
bool box_empty(const Box& b, int nd) {
    for (int d = 0; d < nd; ++d)
        if (b.lo[d] > b.hi[d]) return true;
    return false;
}
int64_t box_ncells(const Box& b, int nd) {
    if (box_empty(b, nd)) return 0;
    int64_t n = 1;
    for (int d = 0; d < nd; ++d) n *= box_ncells_dim(b, d);
    return n;
}
Box box_intersect(const Box& a, const Box& b, int nd) {
    Box r;
    for (int d = 0; d < nd; ++d) {
        r.lo[d] = std::max(a.lo[d], b.lo[d]);
        r.hi[d] = std::min(a.hi[d], b.hi[d]);
    }
    return r;
}
bool box_contains(const Box& b, const int* c, int nd) {
    for (int d = 0; d < nd; ++d)
        if (c[d] < b.lo[d] || c[d] > b.hi[d]) return false;
    return true;
}
Box box_refine(const Box& b, const int* r, int nd) {
    Box o;
    for (int d = 0; d < nd; ++d) {
        o.lo[d] = b.lo[d] * r[d];
        o.hi[d] = (b.hi[d] + 1) * r[d] - 1;
    }
    return o;
}
Box box_coarsen(const Box& b, const int* r, int nd) {
    Box o;
    for (int d = 0; d < nd; ++d) {
        o.lo[d] = floordiv(b.lo[d], r[d]);
        o.hi[d] = floordiv(b.hi[d], r[d]);
    }
    return o;
}
Box box_grow(const Box& b, int g, int nd) {
    Box o = b;
    for (int d = 0; d < nd; ++d) {
        o.lo[d] -= g;
        o.hi[d] += g;
    }
    return o;
}
// a \ b: split dim 0 first, low fragment before high (deterministic, same rule as the oracle)
std::vector<Box> box_subtract(const Box& a, const Box& b, int nd) {
    std::vector<Box> out;
    if (box_empty(box_intersect(a, b, nd), nd)) {
        out.push_back(a);
        return out;
    }
    Box rem = a;
    for (int d = 0; d < nd; ++d) {
        if (rem.lo[d] < b.lo[d]) {
            Box f = rem;
            f.hi[d] = b.lo[d] - 1;
            out.push_back(f);
            rem.lo[d] = b.lo[d];
        }
        if (rem.hi[d] > b.hi[d]) {
            Box f = rem;
            f.lo[d] = b.hi[d] + 1;
            out.push_back(f);
            rem.hi[d] = b.hi[d];
        }
    }
    return out;
}
bool box_less(const Box& a, const Box& b, int nd) {
    for (int d = 0; d < nd; ++d)
        if (a.lo[d] != b.lo[d]) return a.lo[d] < b.lo[d];
    for (int d = 0; d < nd; ++d)
        if (a.hi[d] != b.hi[d]) return a.hi[d] < b.hi[d];
    return false;
}
int64_t box_index(const Box& b, const int* c, int nd) {
    int64_t idx = 0;
    for (int d = 0; d < nd; ++d) idx = idx * box_ncells_dim(b, d) + (c[d] - b.lo[d]);
    return idx;
}

// linear5 weights b_j(s), j=-2..2 with p_k(s) = ((s+1)^{k+1} - s^{k+1}) / R^k
// (reading #12).  For R = 2^m the values are dyadic and exact in fp64.
int linear5_weights(int R, double* out) {
    for (int s = 0; s < R; ++s) {
        double p[5];
        for (int k = 0; k <= 4; ++k) {
            const double a = std::pow((double)(s + 1), k + 1) - std::pow((double)s, k + 1);
            p[k] = a / std::pow((double)R, k);
        }
        out[5 * s + 0] = (p[4] - 5 * p[3] + 5 * p[2] + 5 * p[1] - 6) / 120.0;
        out[5 * s + 1] = (-4 * p[4] + 15 * p[3] + 10 * p[2] - 75 * p[1] + 54) / 120.0;
        out[5 * s + 2] = (6 * p[4] - 15 * p[3] - 40 * p[2] + 75 * p[1] + 94) / 120.0;
        out[5 * s + 3] = (-4 * p[4] + 5 * p[3] + 30 * p[2] - 5 * p[1] - 26) / 120.0;
        out[5 * s + 4] = (p[4] - 5 * p[2] + 4) / 120.0;
    }
    return 0;
}
void free_mask_plan(MaskPlan* p) {
    if (!p) return;
    dfree(p->d_cols, p->st);
    dfree(p->d_mask, p->st);
    dfree(p->d_w, p->st);
    dfree(p->d_part, p->st);
    dfree(p->d_xoff, p->st);
    dfree(p->d_idx, p->st);
    dfree(p->d_dv, p->st);
    delete p;
}

void free_red_plan(RedPlan* p) {
    if (!p) return;
    dfree(p->d_cols, p->st);
    dfree(p->d_colsum, p->st);
    dfree(p->d_contrib, p->st);
    dfree(p->d_xoff, p->st);
    delete p;
}
}  // namespace vk

// NVTX range per C-ABI call (one named range per entry point, visible in nsys / ncu
// --nvtx; near-zero cost without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define VK_NVTX() NvtxRange vk_nvtx_range_(__func__)

// ====================================================================== device helpers
namespace {
std::atomic<uint64_t> g_uid{1};

template <class T>
int upload(T** dptr, const std::vector<T>& h, cudaStream_t st) {
    *dptr = nullptr;
    if (h.empty()) return VLASOV_OK;
    VK_CUDA(cudaMallocAsync((void**)dptr, h.size() * sizeof(T), st));
    VK_CUDA(cudaMemcpyAsync(*dptr, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return VLASOV_OK;
}

void free_level(vlasov_level* L) {
    if (!L) return;
    vk::dfree(L->d_blocks1, L->stream);
    vk::dfree(L->d_tiles_wide, L->stream);
    vk::dfree(L->d_tiles_narrow, L->stream);
    vk::dfree(L->d_copy, L->stream);
    vk::dfree(L->d_cf, L->stream);
    vk::dfree(L->d_phys, L->stream);
    vk::dfree(L->d_reflux, L->stream);
    vk::dfree(L->d_reflux_cells, L->stream);
    vk::dfree(L->d_reflux_off, L->stream);
    vk::dfree(L->d_avg, L->stream);
    vk::free_red_plan(L->red_plan);
    vk::free_mask_plan(L->mask_plan);
    vk::dfree(L->d_b5, L->stream);
    vk::dfree(L->d_partials, L->stream);
    vk::dfree(L->d_tickets, L->stream);
    vk::dfree(L->d_rawtags, L->stream);
    vk::dfree(L->d_scalar, L->stream);
    vk::dfree(L->d_phys4, L->stream);
    vk::dfree(L->d_patch4, L->stream);
    vk::dfree(L->d_fcoarsen4, L->stream);
    vk::dfree(L->d_avg4, L->stream);
    vk::free_red_plan4(L->red_plan4);
    vk::free_mask_plan4(L->mask_plan4);
    delete L;
}

inline int wrap(int x, int n) { return ((x % n) + n) % n; }

// fused field of the 1D+1V stage: the O(n) split of the Green's function, each CTA for its own rows
// (default for n >= 64; C4 on B200: 151 us per step), or the Toeplitz rows split over the strip's
// cluster (VLASOV_FIELD=toeplitz: 160 us)
bool split_field() {
    static const bool s = [] { const char* e = std::getenv("VLASOV_FIELD"); return !(e && std::string(e) == "toeplitz"); }();
    return s;
}

int device_ok_uncached() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return p.major == 10 ? 1 : 0;
}

// cached per current device (cudaGetDeviceProperties costs milliseconds)
int device_ok_impl() {
    static int cache[64];
    static bool init[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (dev < 0 || dev >= 64) return device_ok_uncached();
    if (!init[dev]) {
        cache[dev] = device_ok_uncached();
        init[dev] = true;
    }
    return cache[dev];
}

// owner lookup over the level domain: which block (or patch) holds a cell (-1: none)
struct Owner {
    // cell -> index of the box holding it (-1: none).  1D+1V: per x row, the boxes' v intervals
    // sorted by their start (binary search; no dense map of the level domain to build and clear);
    // 2D+2V: a dense map (those levels are single blocks).
    int nd = 2;
    int dom[4] = {0, 0, 0, 0};
    std::vector<int32_t> id;
    std::vector<std::vector<std::array<int32_t, 3>>> rows;   // [x] -> {v_lo, v_hi, box}
    int64_t lin(const int* c) const {
        int64_t i = 0;
        for (int d = 0; d < nd; ++d) i = i * dom[d] + c[d];
        return i;
    }
    int find(const int* c) const {
        for (int d = 0; d < nd; ++d)
            if (c[d] < 0 || c[d] >= dom[d]) return -1;
        if (nd == 2) {
            const auto& r = rows[c[0]];
            int lo = 0, hi = (int)r.size() - 1;
            while (lo <= hi) {                   // last interval starting at or below c[1]
                const int mid = (lo + hi) >> 1;
                if (r[mid][0] <= c[1]) lo = mid + 1; else hi = mid - 1;
            }
            return (hi >= 0 && c[1] <= r[hi][1]) ? r[hi][2] : -1;
        }
        return id[lin(c)];
    }
};

Owner make_owner(const vlasov_level* L, const std::vector<Box>& bs) {
    Owner o;
    o.nd = L->ndim;
    int64_t tot = 1;
    for (int d = 0; d < L->ndim; ++d) {
        o.dom[d] = L->dom[d];
        tot *= L->dom[d];
    }
    if (L->ndim == 2) {
        o.rows.assign(L->dom[0], {});
        for (size_t p = 0; p < bs.size(); ++p)
            for (int x = bs[p].lo[0]; x <= bs[p].hi[0]; ++x)
                o.rows[x].push_back({bs[p].lo[1], bs[p].hi[1], (int32_t)p});
        for (auto& r : o.rows) std::sort(r.begin(), r.end());
        return o;
    }
    o.id.assign(tot, -1);
    for (size_t p = 0; p < bs.size(); ++p) {
        const Box& b = bs[p];
        int c[4];
        for (c[0] = b.lo[0]; c[0] <= b.hi[0]; ++c[0])
            for (c[1] = b.lo[1]; c[1] <= b.hi[1]; ++c[1])
                for (c[2] = b.lo[2]; c[2] <= b.hi[2]; ++c[2])
                    for (c[3] = b.lo[3]; c[3] <= b.hi[3]; ++c[3]) o.id[o.lin(c)] = (int32_t)p;
    }
    return o;
}

// index of a (block-local interior) cell c of block b in the level array
inline int64_t cell_addr(const vlasov_level* L, int b, const int* c) {
    const Box& B = L->blocks[b];
    int64_t a = L->block_off[b];
    for (int d = 0; d < L->ndim; ++d) a += (int64_t)(c[d] - B.lo[d] + vk::G) * L->block_str[b][d];
    return a;
}

// wrap configuration dims into the domain
inline void wrap_cfg(const vlasov_level* L, const int* c, int* w) {
    for (int d = 0; d < L->ndim; ++d) w[d] = (d < L->ncfg) ? wrap(c[d], L->dom[d]) : c[d];
}

int phys_code(const vlasov_level* L, const int* c) {
    for (int d = L->ncfg; d < L->ndim; ++d) {
        if (c[d] < 0) return 2 * (d - L->ncfg);
        if (c[d] >= L->dom[d]) return 2 * (d - L->ncfg) + 1;
    }
    return -1;
}

void for_each_cell(const Box& b, int nd, const std::function<void(const int*)>& fn) {
    int c[4] = {0, 0, 0, 0};
    if (vk::box_empty(b, nd)) return;
    for (int d = 0; d < nd; ++d) c[d] = b.lo[d];
    while (true) {
        fn(c);
        int d = nd - 1;
        while (d >= 0) {
            if (++c[d] <= b.hi[d]) break;
            c[d] = b.lo[d];
            --d;
        }
        if (d < 0) break;
    }
}

// ------------------------------------------------------------------ task-list construction
int build_tiles_1d(vlasov_level* L, bool have_device) {
    const bool wide = [&] {
        int mx = 0;
        for (const Box& b : L->blocks) mx = std::max(mx, vk::box_ncells_dim(b, 1));
        return mx >= 512;
    }();
    const int TV = vk::stage_1d1v_tile_width(wide);
    int64_t strips_total = 0;
    for (const Box& b : L->blocks) {
        const int nvt = (vk::box_ncells_dim(b, 1) + TV - 1) / TV;
        strips_total += (int64_t)vk::box_ncells_dim(b, 0) * nvt;
    }
    // one-wave tiling: as many row strips as resident CTAs allow (occupancy of the stage-4
    // instance, the one with the largest shared-memory ring)
    int nsm = 148, per_sm = 3;
    if (have_device) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int occ = vk::stage_1d1v_ctas_per_sm(wide, 128);
        if (occ > 0) per_sm = occ;
    }
    const int64_t slots = (int64_t)nsm * per_sm;
    int rows = (int)((strips_total + slots - 1) / slots);
    if (L->blocks.size() == 1) {              // exact one-wave tiling of a single block
        const int nx = vk::box_ncells_dim(L->blocks[0], 0);
        const int nvt = (vk::box_ncells_dim(L->blocks[0], 1) + TV - 1) / TV;
        int64_t max_strips = std::max<int64_t>(1, slots / nvt);
        // the fused-field launch groups the v-tiles of a strip into one cluster: one wave of
        // clusters (the unfused launch uses the same tiles)
        L->cluster_size = 1;
        if (have_device && L->single_block && nvt >= 2 && L->dom[0] <= 4096 &&
            (!split_field() || std::getenv("VLASOV_SPLIT_CLUSTER"))) {
            // cluster size: the divisor of nvt (<= 8) that keeps the most strips in one wave
            int64_t best = 0;
            for (int cs = std::min(8, nvt); cs >= 2; --cs) {
                if (nvt % cs) continue;
                const int mc = vk::stage_1d1v_max_clusters(wide, 128, cs, L->dom[0]);
                const int64_t strips = std::min<int64_t>(max_strips, (int64_t)mc * cs / nvt);
                if (strips > best) { best = strips; L->cluster_size = cs; }
            }
            if (const char* e = std::getenv("VLASOV_CLUSTER")) {   // experiments: force the cluster size
                const int cs = atoi(e);
                if (cs >= 1 && cs <= 8 && nvt % cs == 0) {
                    L->cluster_size = cs;
                    best = cs > 1 ? std::min<int64_t>(max_strips, (int64_t)vk::stage_1d1v_max_clusters(wide, 128, cs, L->dom[0]) * cs / nvt) : max_strips;
                }
            }
            if (best > 0) max_strips = best;
        }
        rows = (int)((nx + max_strips - 1) / max_strips);
    }
    rows = std::max(8, std::min(128, rows));
    if (const char* e = std::getenv("VLASOV_TILE_ROWS")) rows = std::max(4, std::min(128, atoi(e)));
    L->tile_rows = rows;
    std::vector<vk::Tile1>& tiles = wide ? L->h_tiles_wide : L->h_tiles_narrow;
    tiles.clear();
    L->n_vtiles = 0;
    L->n_strips = 0;
    for (size_t b = 0; b < L->blocks.size(); ++b) {
        const int nx = vk::box_ncells_dim(L->blocks[b], 0), nv = vk::box_ncells_dim(L->blocks[b], 1);
        const int nvt = (nv + TV - 1) / TV;
        // balance the strips: equal row counts (+-1) instead of a short last strip
        const int nstrip = (nx + rows - 1) / rows;
        if (L->single_block) L->n_vtiles = nvt;
        for (int s = 0; s < nstrip; ++s) {
            const int x0 = (int)((int64_t)nx * s / nstrip), x1 = (int)((int64_t)nx * (s + 1) / nstrip);
            for (int vt = 0; vt < nvt; ++vt) {
                vk::Tile1 t;
                t.block = (int)b;
                t.x0 = x0;
                t.nrows = x1 - x0;
                t.j0 = vt * TV;
                t.ncols = std::min(TV, nv - vt * TV);
                t.pvt = L->single_block ? vt : -1;
                t.strip = L->n_strips;
                tiles.push_back(t);
            }
            ++L->n_strips;
        }
    }
    L->h_blocks1.clear();
    for (size_t b = 0; b < L->blocks.size(); ++b) {
        vk::Block1 B;
        B.off = L->block_off[b];
        B.pitch = (int32_t)L->block_str[b][0];
        B.lo_x = L->blocks[b].lo[0];
        B.lo_v = L->blocks[b].lo[1];
        B.nx = vk::box_ncells_dim(L->blocks[b], 0);
        B.nv = vk::box_ncells_dim(L->blocks[b], 1);
        L->h_blocks1.push_back(B);
    }
    L->self_ghost_ok = L->single_block && (L->dom[1] % 4 == 0) && L->dom[1] >= 4;
    return VLASOV_OK;
}

// ghost-fill tasks of every block: copies (siblings / periodic), CF interpolation, PHYS columns
int build_ghost_tasks(vlasov_level* L, const vlasov_level* C, std::vector<int64_t>& copies,
                      std::vector<vk::CFTask>& cfs, std::vector<vk::PhysTask>& phys) {
    const int nd = L->ndim;
    Owner own;
    if (!L->single_block) own = make_owner(L, L->blocks);
    Owner cown;
    if (C) cown = make_owner(C, C->blocks);
    int rr[4] = {1, 1, 1, 1};
    if (C)
        for (int d = 0; d < nd; ++d) rr[d] = L->ratio[d] / C->ratio[d];
    int err = VLASOV_OK;
    {   // capacity: the ghost frames of all blocks (avoids reallocating the task lists)
        int64_t fr = 0;
        for (const Box& B : L->blocks) fr += vk::box_ncells(vk::box_grow(B, vk::G, nd), nd) - vk::box_ncells(B, nd);
        copies.reserve((size_t)(2 * fr));
    }
    for (size_t b = 0; b < L->blocks.size(); ++b) {
        const Box& B = L->blocks[b];
        const Box GB = vk::box_grow(B, vk::G, nd);
        auto ghost_cell = [&](const int* c) {
            if (err) return;
            if (vk::box_contains(B, c, nd)) return;
            if (phys_code(L, c) >= 0) return;                     // PHYS: handled per column
            int w[4];
            wrap_cfg(L, c, w);
            const int q = L->single_block ? (vk::box_contains(L->blocks[0], w, nd) ? 0 : -1) : own.find(w);
            const int64_t dst = cell_addr(L, (int)b, c);
            if (q >= 0) {
                copies.push_back(dst);
                copies.push_back(cell_addr(L, q, w));
                return;
            }
            if (!C) {
                err = vk::fail(VLASOV_ENEST, "ghost cell without a source on a level without a coarser level");
                return;
            }
            int cc[4];
            for (int d = 0; d < nd; ++d) cc[d] = vk::floordiv(w[d], rr[d]);
            const int cq = cown.find(cc);
            if (cq < 0) {
                err = vk::fail(VLASOV_ESTENCIL, "coarse-fine ghost: coarse parent not on the coarser level");
                return;
            }
            vk::CFTask t;
            t.dst = dst;
            t.csrc = cell_addr(C, cq, cc);
            for (int d = 0; d < 4; ++d) {
                t.cstride[d] = d < nd ? (int32_t)C->block_str[cq][d] : 0;
                t.sub[d] = d < nd ? (int8_t)(w[d] - cc[d] * rr[d]) : 0;
            }
            cfs.push_back(t);
        };
        if (nd == 2) {
            // the ghost frame only, row by row (x major, v fastest: the same task order as a
            // sweep of the grown block), without visiting the interior; runs of sibling copies
            // from one source box take one owner lookup (the copy addresses are consecutive)
            for (int x = GB.lo[0]; x <= GB.hi[0] && !err; ++x) {
                const bool xin = x >= B.lo[0] && x <= B.hi[0];
                for (int v = GB.lo[1]; v <= GB.hi[1] && !err; ++v) {
                    if (xin && v == B.lo[1]) v = B.hi[1] + 1;
                    const int c[4] = {x, v, 0, 0};
                    if (phys_code(L, c) < 0 && !L->single_block) {
                        int w[4];
                        wrap_cfg(L, c, w);
                        const int q = own.find(w);
                        if (q >= 0) {
                            // the run: up to the end of box q in v, of this row's ghost range
                            const int vend = std::min(L->blocks[q].hi[1], (xin && v < B.lo[1]) ? B.lo[1] - 1 : GB.hi[1]);
                            const int64_t d0 = cell_addr(L, (int)b, c), s0 = cell_addr(L, q, w);
                            for (int k = 0; k <= vend - v; ++k) {
                                copies.push_back(d0 + k);
                                copies.push_back(s0 + k);
                            }
                            v = vend;
                            continue;
                        }
                    }
                    ghost_cell(c);
                }
            }
        } else {
            for_each_cell(GB, nd, ghost_cell);
        }
        if (err) return err;
        if (nd == 2) {
            const int nv = L->dom[1];
            for (int side = 0; side < 2; ++side) {
                if (side == 0 && B.lo[1] != 0) continue;
                if (side == 1 && B.hi[1] != nv - 1) continue;
                if (vk::box_ncells_dim(B, 1) < 4)
                    return vk::fail(VLASOV_EINVAL, "blocks touching the v-boundary need >= 4 v-cells");
                for (int x = B.lo[0] - vk::G; x <= B.hi[0] + vk::G; ++x) {
                    int c[4] = {x, side == 0 ? 0 : nv - 1, 0, 0};
                    vk::PhysTask t;
                    t.cell0 = cell_addr(L, (int)b, c);
                    t.e_idx = wrap(x, L->dom[0]) + vk::G;
                    t.side = side;
                    phys.push_back(t);
                }
            }
        }
    }
    return VLASOV_OK;
}

std::vector<Box> subpatches_of(const vlasov_level* const* levels, int nlev, int li, int patch);

// F*-form stepping of a 2D+2V level (N3): per-patch face layout (dim d: the patch's cells with
// n_d + 1 along d, row-major), and w.r.t. the coarser level the Alg.4 flux-coarsening tasks
// (every coarse face of every coarse patch that coincides with a fine patch face, periodic images
// in x and y) and the average-down tasks
int build_fstar4(vlasov_level* L, const vlasov_level* C, std::vector<vk::Patch4>& pt,
                 std::vector<vk::FaceAvgTask>& fc, std::vector<vk::AvgTask4>& av) {
    int64_t foff = 0;
    std::vector<std::array<int64_t, 4>> offs;
    for (size_t p = 0; p < L->boxes.size(); ++p) {
        const Box& b = L->boxes[p];
        const int blk = L->patch_block[p];
        vk::Patch4 P;
        int lo[4];
        for (int d = 0; d < 4; ++d) { lo[d] = b.lo[d]; P.lo[d] = b.lo[d]; P.n[d] = vk::box_ncells_dim(b, d); }
        P.org = cell_addr(L, blk, lo);
        for (int d = 0; d < 3; ++d) P.s[d] = L->block_str[blk][d];
        int64_t ncell = 1;
        for (int d = 0; d < 4; ++d) ncell *= P.n[d];
        L->max_patch_cells = std::max(L->max_patch_cells, ncell);
        std::array<int64_t, 4> o;
        for (int d = 0; d < 4; ++d) {
            P.foff[d] = o[d] = foff;
            foff += ncell / P.n[d] * (P.n[d] + 1);
        }
        offs.push_back(o);
        pt.push_back(P);
    }
    L->face_doubles = foff;
    if (!C) return VLASOV_OK;
    const int* rr = L->coarse_ratio;
    for (const Box& fb : L->boxes)
        for (int d = 0; d < 4; ++d)
            if (fb.lo[d] % rr[d] || (fb.hi[d] + 1) % rr[d])
                return vk::fail(VLASOV_EINVAL, "fine boxes must be unions of refined coarse cells");
    // coarse patch face layout (the same rule as for L)
    std::vector<std::array<int64_t, 4>> coffs;
    {
        int64_t o = 0;
        for (const Box& cb : C->boxes) {
            int64_t ncell = 1;
            for (int d = 0; d < 4; ++d) ncell *= vk::box_ncells_dim(cb, d);
            std::array<int64_t, 4> a;
            for (int d = 0; d < 4; ++d) { a[d] = o; o += ncell / vk::box_ncells_dim(cb, d) * (vk::box_ncells_dim(cb, d) + 1); }
            coffs.push_back(a);
        }
    }
    auto face_index = [](const int* n, int d, const int* q) {   // q: face coords (q[d] in 0..n_d)
        int64_t idx = 0;
        for (int e = 0; e < 4; ++e) idx = idx * (n[e] + (e == d ? 1 : 0)) + q[e];
        return idx;
    };
    for (size_t p = 0; p < L->boxes.size(); ++p) {
        const Box& fb = L->boxes[p];
        int nf[4];
        for (int d = 0; d < 4; ++d) nf[d] = vk::box_ncells_dim(fb, d);
        const Box cbx = vk::box_coarsen(fb, rr, 4);
        for (int d = 0; d < 4; ++d) {
            int fst[4];                                          // fine face-array strides
            {
                int64_t s = 1;
                for (int e = 3; e >= 0; --e) { fst[e] = (int)s; s *= nf[e] + (e == d ? 1 : 0); }
            }
            for (int side = 0; side < 2; ++side) {
                const int cface = side == 0 ? cbx.lo[d] : cbx.hi[d] + 1;      // coarse face = low face of cell cface
                const int ff = side == 0 ? 0 : nf[d];                        // fine face index along d
                const int nimg = d < 2 ? 3 : 1;
                for (int im = 0; im < nimg; ++im) {
                    const int shift = im == 0 ? 0 : (im == 1 ? -C->dom[d] : C->dom[d]);
                    const int cf = cface + shift;
                    for (size_t cp = 0; cp < C->boxes.size(); ++cp) {
                        const Box& cb = C->boxes[cp];
                        if (cf < cb.lo[d] || cf > cb.hi[d] + 1) continue;
                        int lo[4], hi[4];
                        bool ok = true;
                        for (int e = 0; e < 4 && ok; ++e) {
                            if (e == d) continue;
                            lo[e] = std::max(cbx.lo[e], cb.lo[e]);
                            hi[e] = std::min(cbx.hi[e], cb.hi[e]);
                            ok = lo[e] <= hi[e];
                        }
                        if (!ok) continue;
                        int cn[4];
                        for (int e = 0; e < 4; ++e) cn[e] = vk::box_ncells_dim(cb, e);
                        int c[4];
                        c[d] = cf;
                        const int e0 = d == 0 ? 1 : 0, e1 = (d <= 1) ? 2 : 1, e2 = d == 3 ? 2 : 3;
                        for (c[e0] = lo[e0]; c[e0] <= hi[e0]; ++c[e0])
                            for (c[e1] = lo[e1]; c[e1] <= hi[e1]; ++c[e1])
                                for (c[e2] = lo[e2]; c[e2] <= hi[e2]; ++c[e2]) {
                                    int qc[4], qf[4];
                                    for (int e = 0; e < 4; ++e) {
                                        qc[e] = c[e] - cb.lo[e];
                                        qf[e] = e == d ? ff : c[e] * rr[e] - fb.lo[e];
                                    }
                                    vk::FaceAvgTask t;
                                    t.coarse = coffs[cp][d] + face_index(cn, d, qc);
                                    t.fine = offs[p][d] + face_index(nf, d, qf);
                                    const int es[3] = {e0, e1, e2};
                                    for (int k = 0; k < 3; ++k) { t.st[k] = fst[es[k]]; t.r[k] = rr[es[k]]; }
                                    t.pad = 0;
                                    fc.push_back(t);
                                }
                    }
                }
            }
        }
        // average-down tasks
        const int fblk = L->patch_block[p];
        for (size_t cp = 0; cp < C->boxes.size(); ++cp) {
            const Box ov = vk::box_intersect(C->boxes[cp], cbx, 4);
            if (vk::box_empty(ov, 4)) continue;
            const int cblk = C->patch_block[cp];
            for_each_cell(ov, 4, [&](const int* c) {
                vk::AvgTask4 t;
                int fc0[4];
                for (int e = 0; e < 4; ++e) fc0[e] = c[e] * rr[e];
                t.coarse = cell_addr(C, cblk, c);
                t.fine = cell_addr(L, fblk, fc0);
                for (int e = 0; e < 3; ++e) t.st[e] = L->block_str[fblk][e];
                for (int e = 0; e < 4; ++e) t.r[e] = rr[e];
                av.push_back(t);
            });
        }
    }
    return VLASOV_OK;
}

// Characteristic velocity condition of a 2D+2V multi-patch level (reading #6): for each patch
// touching a velocity boundary, one task per column side, v_x pass first (columns over the whole
// ghosted extent of x, y, v_y), then v_y (over the ghosted x, y, v_x), as the oracle (amr4).
int build_phys4_tasks(const vlasov_level* L, std::vector<vk::PhysTask4>& tasks, int64_t counts[2]) {
    counts[0] = counts[1] = 0;
    const int nyg = L->dom[1] + 4, nvyg = L->dom[3] + 4;
    for (int pass = 0; pass < 2; ++pass) {
        const int vd = 2 + pass, od = 5 - vd;                    // the other velocity dim
        for (size_t b = 0; b < L->blocks.size(); ++b) {
            const Box& B = L->blocks[b];
            const int n = vk::box_ncells_dim(B, vd);
            const int dlo = B.lo[vd], dhi = L->dom[vd] - 1 - B.hi[vd];
            if ((dlo > 0 && dlo < vk::G) || (dhi > 0 && dhi < vk::G))
                return vk::fail(VLASOV_EINVAL, "2D+2V: a patch must touch the velocity boundary or stay >= 2 cells from it");
            for (int side = 0; side < 2; ++side) {
                if (side == 0 ? dlo != 0 : dhi != 0) continue;
                if (n < 4) return vk::fail(VLASOV_EINVAL, "blocks touching a velocity boundary need >= 4 cells along it");
                for (int x = B.lo[0] - vk::G; x <= B.hi[0] + vk::G; ++x)
                    for (int y = B.lo[1] - vk::G; y <= B.hi[1] + vk::G; ++y)
                        for (int o = B.lo[od] - vk::G; o <= B.hi[od] + vk::G; ++o) {
                            int c[4] = {x, y, 0, 0};
                            c[vd] = side == 0 ? 0 : L->dom[vd] - 1;
                            c[od] = o;
                            vk::PhysTask4 t;
                            t.cell0 = cell_addr(L, (int)b, c);
                            t.stride = (int32_t)L->block_str[b][vd];
                            t.e_idx = (int32_t)((int64_t)pass * (L->dom[0] + 4) * nyg +
                                                (int64_t)(wrap(x, L->dom[0]) + 2) * nyg + (wrap(y, L->dom[1]) + 2));
                            int pv[2];                            // f0v coordinates (vx, vy) of the first ghost layer
                            pv[vd - 2] = side == 0 ? -1 : L->dom[vd];
                            pv[od - 2] = o;
                            t.p_idx = (pv[0] + 2) * nvyg + (pv[1] + 2);
                            t.pstep = (int16_t)(vd == 2 ? nvyg : 1);
                            t.side = (int16_t)side;
                            tasks.push_back(t);
                        }
            }
        }
        counts[pass] = (int64_t)tasks.size() - (pass ? counts[0] : 0);
    }
    return VLASOV_OK;
}

// Alg.8 Sub-Patch Reduction plan of a 2D+2V hierarchy (N3): grown (x, y) columns of every
// sub-patch (Alg.7) and, per finest (x, y) cell, its refined contributions in (level, patch,
// sub-patch) order with the linear5 weights of its sub-offsets
int build_red_plan4(const vlasov_level* const* levels, int nlev, vk::RedPlan4** out) {
    *out = nullptr;
    const vlasov_level* Lf = levels[nlev - 1];
    const int nxf = Lf->dom[0], nyf = Lf->dom[1];
    std::vector<vk::Red4Col> cols;
    std::vector<std::vector<vk::Red4Contrib>> per((size_t)nxf * nyf);
    for (int l = 0; l < nlev; ++l) {
        const vlasov_level* L = levels[l];
        if (L->ndim != 4) return vk::fail(VLASOV_EINVAL, "reduce_moment: mixed 1D+1V / 2D+2V levels");
        if (nxf % L->dom[0] || nyf % L->dom[1]) return vk::fail(VLASOV_EINVAL, "finest (x, y) resolution not a multiple of a level's");
        if (l > 0 && (L->coarser != levels[l - 1] || L->coarser_uid != levels[l - 1]->uid))
            return vk::fail(VLASOV_ESTALE, "reduce_moment: levels are not a hierarchy (coarser mismatch)");
        const int Rx = nxf / L->dom[0], Ry = nyf / L->dom[1];
        if (Rx > vk::MAXR * vk::MAXR || Ry > vk::MAXR * vk::MAXR) return vk::fail(VLASOV_EUNSUPPORTED, "ratio to the finest level too large");
        std::vector<double> wx((size_t)Rx * 5), wy((size_t)Ry * 5);
        vk::linear5_weights(Rx, wx.data());
        vk::linear5_weights(Ry, wy.data());
        for (size_t p = 0; p < L->boxes.size(); ++p) {
            const int blk = L->patch_block[p];
            for (const Box& sp : subpatches_of(levels, nlev, l, (int)p)) {
                const int64_t base = (int64_t)cols.size();
                const int nxs = vk::box_ncells_dim(sp, 0), nys = vk::box_ncells_dim(sp, 1);
                for (int a = 0; a < nxs + 2 * vk::G; ++a)
                    for (int c = 0; c < nys + 2 * vk::G; ++c) {
                        int cc[4] = {sp.lo[0] - vk::G + a, sp.lo[1] - vk::G + c, sp.lo[2], sp.lo[3]};
                        vk::Red4Col rc;
                        rc.addr = cell_addr(L, blk, cc);
                        rc.nvx = vk::box_ncells_dim(sp, 2);
                        rc.nvy = vk::box_ncells_dim(sp, 3);
                        rc.s2 = (int32_t)L->block_str[blk][2];
                        rc.level = l;
                        cols.push_back(rc);
                    }
                for (int xc = sp.lo[0]; xc <= sp.hi[0]; ++xc)
                    for (int yc = sp.lo[1]; yc <= sp.hi[1]; ++yc)
                        for (int sx = 0; sx < Rx; ++sx)
                            for (int sy = 0; sy < Ry; ++sy) {
                                vk::Red4Contrib k;
                                k.cs = base + (int64_t)(xc - sp.lo[0]) * (nys + 2 * vk::G) + (yc - sp.lo[1]);
                                k.ystride = nys + 2 * vk::G;
                                k.pad = 0;
                                k.dvv = L->h[2] * L->h[3];
                                for (int j = 0; j < 5; ++j) {
                                    k.bx[j] = wx[(size_t)sx * 5 + j];
                                    k.by[j] = wy[(size_t)sy * 5 + j];
                                }
                                per[(size_t)(xc * Rx + sx) * nyf + (yc * Ry + sy)].push_back(k);
                            }
            }
        }
    }
    std::vector<vk::Red4Contrib> con;
    std::vector<int32_t> off((size_t)nxf * nyf + 1, 0);
    for (size_t c = 0; c < per.size(); ++c) {
        off[c] = (int32_t)con.size();
        con.insert(con.end(), per[c].begin(), per[c].end());
    }
    off[per.size()] = (int32_t)con.size();
    vk::RedPlan4* P = new vk::RedPlan4();
    P->st = Lf->stream;
    for (int l = 0; l < nlev; ++l) P->uids.push_back(levels[l]->uid);
    P->nxf = nxf;
    P->nyf = nyf;
    P->ncols = (int64_t)cols.size();
    P->ncontrib = (int64_t)con.size();
    int rc;
    if ((rc = upload(&P->d_cols, cols, P->st)) || (rc = upload(&P->d_contrib, con, P->st)) ||
        (rc = upload(&P->d_off, off, P->st))) {
        vk::free_red_plan4(P);
        return rc;
    }
    if (!cols.empty()) VK_CUDA(cudaMallocAsync((void**)&P->d_colsum, sizeof(double) * cols.size(), P->st));
    cudaError_t e = cudaStreamSynchronize(P->st);
    if (e != cudaSuccess) { vk::free_red_plan4(P); return vk::cuda_check(e, "reduction plan upload"); }
    *out = P;
    return VLASOV_OK;
}

// Alg.6 Mask Reduction plan of a 2D+2V hierarchy (N3 comparator): one item per (patch, finest
// (x, y) cell of its refined footprint); mask per patch cell (0 where the next finer level covers)
int build_mask_plan4(const vlasov_level* const* levels, int nlev, vk::MaskPlan4** out) {
    *out = nullptr;
    const vlasov_level* Lf = levels[nlev - 1];
    const int nxf = Lf->dom[0], nyf = Lf->dom[1];
    std::vector<vk::Mask4Item> items;
    std::vector<uint8_t> mask;
    std::vector<double> w;
    std::map<int, int> woff;
    std::vector<std::vector<std::pair<int32_t, double>>> per((size_t)nxf * nyf);
    auto weights = [&](int R) {
        if (!woff.count(R)) {
            woff[R] = (int)w.size();
            std::vector<double> b((size_t)R * 5);
            vk::linear5_weights(R, b.data());
            w.insert(w.end(), b.begin(), b.end());
        }
        return woff[R];
    };
    for (int l = 0; l < nlev; ++l) {
        const vlasov_level* L = levels[l];
        if (L->ndim != 4) return vk::fail(VLASOV_EINVAL, "reduce_moment_mask: mixed 1D+1V / 2D+2V levels");
        if (nxf % L->dom[0] || nyf % L->dom[1]) return vk::fail(VLASOV_EINVAL, "finest (x, y) resolution not a multiple of a level's");
        if (l > 0 && (L->coarser != levels[l - 1] || L->coarser_uid != levels[l - 1]->uid))
            return vk::fail(VLASOV_ESTALE, "reduce_moment_mask: levels are not a hierarchy (coarser mismatch)");
        const int Rx = nxf / L->dom[0], Ry = nyf / L->dom[1];
        if (Rx > vk::MAXR || Ry > vk::MAXR) return vk::fail(VLASOV_EUNSUPPORTED, "mask reduction: ratio to the finest level > 16");
        const int wx0 = weights(Rx), wy0 = weights(Ry);
        int rr[4] = {1, 1, 1, 1};
        if (l + 1 < nlev)
            for (int d = 0; d < 4; ++d) rr[d] = levels[l + 1]->ratio[d] / L->ratio[d];
        for (size_t p = 0; p < L->boxes.size(); ++p) {
            const Box& b = L->boxes[p];
            const int blk = L->patch_block[p];
            int n[4];
            for (int d = 0; d < 4; ++d) n[d] = vk::box_ncells_dim(b, d);
            const int64_t moff = (int64_t)mask.size();
            std::vector<uint8_t> mu((size_t)n[0] * n[1] * n[2] * n[3], 1);
            if (l + 1 < nlev)
                for (const Box& fb : levels[l + 1]->boxes) {
                    const Box cb = vk::box_intersect(vk::box_coarsen(fb, rr, 4), b, 4);
                    if (vk::box_empty(cb, 4)) continue;
                    for_each_cell(cb, 4, [&](const int* c) {
                        mu[(((size_t)(c[0] - b.lo[0]) * n[1] + (c[1] - b.lo[1])) * n[2] + (c[2] - b.lo[2])) * n[3] +
                           (c[3] - b.lo[3])] = 0;
                    });
                }
            mask.insert(mask.end(), mu.begin(), mu.end());
            for (int xc = b.lo[0]; xc <= b.hi[0]; ++xc)
                for (int yc = b.lo[1]; yc <= b.hi[1]; ++yc)
                    for (int sx = 0; sx < Rx; ++sx)
                        for (int sy = 0; sy < Ry; ++sy) {
                            vk::Mask4Item it;
                            int cc[4] = {xc - 2, yc - 2, b.lo[2], b.lo[3]};
                            it.addr = cell_addr(L, blk, cc);
                            it.mask = moff + ((int64_t)(xc - b.lo[0]) * n[1] + (yc - b.lo[1])) * n[2] * n[3];
                            it.s0 = (int32_t)L->block_str[blk][0];
                            it.s1 = (int32_t)L->block_str[blk][1];
                            it.s2 = (int32_t)L->block_str[blk][2];
                            it.nvx = n[2];
                            it.nvy = n[3];
                            it.level = l;
                            it.mstride0 = n[1] * n[2] * n[3];
                            it.mstride1 = n[2] * n[3];
                            it.wx = wx0 + 5 * sx;
                            it.wy = wy0 + 5 * sy;
                            per[(size_t)(xc * Rx + sx) * nyf + (yc * Ry + sy)].push_back(
                                {(int32_t)items.size(), L->h[2] * L->h[3]});
                            items.push_back(it);
                        }
        }
    }
    std::vector<int32_t> off(per.size() + 1, 0), idx;
    std::vector<double> dvv;
    for (size_t c = 0; c < per.size(); ++c) {
        off[c] = (int32_t)idx.size();
        for (auto& pr : per[c]) { idx.push_back(pr.first); dvv.push_back(pr.second); }
    }
    off[per.size()] = (int32_t)idx.size();
    vk::MaskPlan4* P = new vk::MaskPlan4();
    P->st = Lf->stream;
    for (int l = 0; l < nlev; ++l) P->uids.push_back(levels[l]->uid);
    P->nxf = nxf;
    P->nyf = nyf;
    P->nitems = (int64_t)items.size();
    int rc;
    if ((rc = upload(&P->d_items, items, P->st)) || (rc = upload(&P->d_mask, mask, P->st)) ||
        (rc = upload(&P->d_w, w, P->st)) || (rc = upload(&P->d_dvv, dvv, P->st)) ||
        (rc = upload(&P->d_off, off, P->st)) || (rc = upload(&P->d_idx, idx, P->st))) {
        vk::free_mask_plan4(P);
        return rc;
    }
    if (!items.empty()) VK_CUDA(cudaMallocAsync((void**)&P->d_part, sizeof(double) * items.size(), P->st));
    cudaError_t e = cudaStreamSynchronize(P->st);
    if (e != cudaSuccess) { vk::free_mask_plan4(P); return vk::cuda_check(e, "mask plan upload"); }
    *out = P;
    return VLASOV_OK;
}

// Alg.7 ComputeSubPatches, same set operations as the oracle, sorted output
std::vector<Box> subpatches_of(const vlasov_level* const* levels, int nlev, int li, int patch) {
    const vlasov_level* L = levels[li];
    const int nd = L->ndim;
    const Box pin = L->boxes[patch];
    std::vector<Box> S{pin};
    for (int fl = li + 1; fl < nlev; ++fl) {
        const vlasov_level* F = levels[fl];
        int rr[4];
        for (int d = 0; d < nd; ++d) rr[d] = F->ratio[d] / L->ratio[d];
        for (const Box& fb : F->boxes) {
            const Box P = vk::box_coarsen(fb, rr, nd);
            if (vk::box_empty(vk::box_intersect(P, pin, nd), nd)) continue;
            Box Pext = P;                                           // extend in reduction dims
            for (int d = L->ncfg; d < nd; ++d) { Pext.lo[d] = pin.lo[d]; Pext.hi[d] = pin.hi[d]; }
            std::vector<Box> S2;
            for (const Box& Ps : S) {
                const Box I = vk::box_intersect(Ps, Pext, nd);
                if (vk::box_empty(I, nd)) { S2.push_back(Ps); continue; }
                S2.push_back(I);
                for (const Box& r : vk::box_subtract(Ps, I, nd)) S2.push_back(r);
            }
            S.clear();
            for (const Box& Ps : S2)
                for (const Box& r : vk::box_subtract(Ps, P, nd)) S.push_back(r);
        }
    }
    std::vector<Box> T;
    for (const Box& b : S)
        if (!vk::box_empty(b, nd)) T.push_back(b);
    std::sort(T.begin(), T.end(), [&](const Box& a, const Box& b) { return vk::box_less(a, b, nd); });
    return T;
}

// Flux-register tasks (Alg.4 flux substitution as refluxing) and average-down tasks
// of a 1D+1V fine level L with respect to its coarser level C.
int build_amr_tasks(const vlasov_level* L, const vlasov_level* C, std::vector<vk::RefluxTask>& tasks,
                    std::vector<int64_t>& cells, std::vector<int32_t>& offs, std::vector<vk::AvgTask>& avg) {
    const int nd = 2;
    const int* rr = L->coarse_ratio;
    for (const Box& fb : L->boxes)
        for (int d = 0; d < nd; ++d)
            if (fb.lo[d] % rr[d] || (fb.hi[d] + 1) % rr[d])
                return vk::fail(VLASOV_EINVAL, "fine boxes must be unions of refined coarse cells");
    Owner cown = make_owner(C, C->blocks);
    std::vector<uint8_t> covered((size_t)C->dom[0] * C->dom[1], 0);
    for (const Box& fb : L->boxes) {
        const Box cb = vk::box_coarsen(fb, rr, nd);
        for (int x = cb.lo[0]; x <= cb.hi[0]; ++x)
            for (int v = cb.lo[1]; v <= cb.hi[1]; ++v) covered[(size_t)x * C->dom[1] + v] = 1;
    }
    auto is_cov = [&](int x, int v) { return covered[(size_t)x * C->dom[1] + v] != 0; };
    std::vector<vk::RefluxTask> T;
    for (size_t q = 0; q < L->boxes.size(); ++q) {
        const Box& fb = L->boxes[q];
        const int fblk = L->patch_block[q];
        const int64_t fpitch = L->block_str[fblk][0];
        const Box cb = vk::box_coarsen(fb, rr, nd);
        for (int side = 0; side < 2; ++side) {                   // x-faces
            const int ux = wrap(side == 0 ? cb.lo[0] - 1 : cb.hi[0] + 1, C->dom[0]);
            for (int jc = cb.lo[1]; jc <= cb.hi[1]; ++jc) {
                if (is_cov(ux, jc)) continue;
                int uc[4] = {ux, jc, 0, 0};
                const int cq = cown.find(uc);
                if (cq < 0) return vk::fail(VLASOV_ESTENCIL, "coarse cell next to a fine patch not on the coarser level");
                vk::RefluxTask t;
                std::memset(&t, 0, sizeof(t));
                t.ccell = cell_addr(C, cq, uc);
                t.dir = 0;
                t.sign = side == 0 ? +1 : -1;
                int cs[4] = {side == 0 ? ux - 1 : ux - 2, jc, 0, 0};
                t.cf.s0 = cell_addr(C, cq, cs);
                t.cf.pitch = (int32_t)C->block_str[cq][0];
                t.cf.g = jc;
                t.nfine = rr[1];
                for (int s = 0; s < rr[1]; ++s) {
                    const int jf = jc * rr[1] + s;
                    int fs[4] = {side == 0 ? fb.lo[0] - 2 : fb.hi[0] - 1, jf, 0, 0};
                    t.ff[s].s0 = cell_addr(L, fblk, fs);
                    t.ff[s].pitch = (int32_t)fpitch;
                    t.ff[s].g = jf;
                }
                T.push_back(t);
            }
        }
        for (int side = 0; side < 2; ++side) {                   // v-faces
            const int uv = side == 0 ? cb.lo[1] - 1 : cb.hi[1] + 1;
            if (uv < 0 || uv >= C->dom[1]) continue;             // physical v boundary
            for (int xc = cb.lo[0]; xc <= cb.hi[0]; ++xc) {
                if (is_cov(xc, uv)) continue;
                int uc[4] = {xc, uv, 0, 0};
                const int cq = cown.find(uc);
                if (cq < 0) return vk::fail(VLASOV_ESTENCIL, "coarse cell next to a fine patch not on the coarser level");
                vk::RefluxTask t;
                std::memset(&t, 0, sizeof(t));
                t.ccell = cell_addr(C, cq, uc);
                t.dir = 1;
                t.sign = side == 0 ? +1 : -1;
                int cs[4] = {xc, side == 0 ? uv - 1 : uv - 2, 0, 0};
                t.cf.s0 = cell_addr(C, cq, cs);
                t.cf.pitch = (int32_t)C->block_str[cq][0];
                t.cf.g = xc + vk::G;
                t.nfine = rr[0];
                for (int s = 0; s < rr[0]; ++s) {
                    const int xf = xc * rr[0] + s;
                    int fs[4] = {xf, side == 0 ? fb.lo[1] - 2 : fb.hi[1] - 1, 0, 0};
                    t.ff[s].s0 = cell_addr(L, fblk, fs);
                    t.ff[s].pitch = (int32_t)fpitch;
                    t.ff[s].g = xf + vk::G;
                }
                T.push_back(t);
            }
        }
        for (int xc = cb.lo[0]; xc <= cb.hi[0]; ++xc)            // average-down
            for (int jc = cb.lo[1]; jc <= cb.hi[1]; ++jc) {
                int uc[4] = {xc, jc, 0, 0};
                const int cq = cown.find(uc);
                if (cq < 0) return vk::fail(VLASOV_ENEST, "fine patch not covered by the coarser level");
                int fc[4] = {xc * rr[0], jc * rr[1], 0, 0};
                vk::AvgTask a;
                a.ccell = cell_addr(C, cq, uc);
                a.fcell0 = cell_addr(L, fblk, fc);
                a.fpitch = (int32_t)fpitch;
                a.pad = 0;
                avg.push_back(a);
            }
    }
    // group by corrected coarse cell (stable: the face order above within a cell)
    std::vector<size_t> idx(T.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return T[a].ccell < T[b].ccell; });
    tasks.clear();
    cells.clear();
    offs.clear();
    for (size_t k = 0; k < idx.size(); ++k) {
        const vk::RefluxTask& t = T[idx[k]];
        if (cells.empty() || cells.back() != t.ccell) {
            cells.push_back(t.ccell);
            offs.push_back((int32_t)tasks.size());
        }
        tasks.push_back(t);
    }
    offs.push_back((int32_t)tasks.size());
    return VLASOV_OK;
}

// Alg.8 plan: grown columns of every sub-patch (level-major, patch-minor, Alg.7 order) and, per
// finest x cell, its linear5-refined contributions in that order (readings #13, #16).
int build_red_plan(const vlasov_level* const* levels, int nlev, vk::RedPlan** out) {
    *out = nullptr;
    const vlasov_level* Lf = levels[nlev - 1];
    const int nxf = Lf->dom[0];
    std::vector<vk::RedCol> cols;
    std::vector<std::vector<vk::RedContrib>> per_x(nxf);
    for (int l = 0; l < nlev; ++l) {
        const vlasov_level* L = levels[l];
        if (L->ndim != 2) return vk::fail(VLASOV_EUNSUPPORTED, "sub-patch reduction: 1D+1V levels only");
        if (nxf % L->dom[0]) return vk::fail(VLASOV_EINVAL, "finest x resolution not a multiple of a level's");
        if (l > 0 && (L->coarser != levels[l - 1] || L->coarser_uid != levels[l - 1]->uid))
            return vk::fail(VLASOV_ESTALE, "reduce_moment: levels are not a hierarchy (coarser mismatch)");
        const int R = nxf / L->dom[0];
        if (R > vk::MAXR * vk::MAXR) return vk::fail(VLASOV_EUNSUPPORTED, "x ratio to the finest level too large");
        std::vector<double> b5((size_t)R * 5);
        vk::linear5_weights(R, b5.data());
        for (size_t p = 0; p < L->boxes.size(); ++p) {
            const int blk = L->patch_block[p];
            for (const Box& sp : subpatches_of(levels, nlev, l, (int)p)) {
                const int64_t base = (int64_t)cols.size();
                const int nxs = vk::box_ncells_dim(sp, 0);
                for (int c = 0; c < nxs + 2 * vk::G; ++c) {
                    int cc[4] = {sp.lo[0] - vk::G + c, sp.lo[1], 0, 0};
                    vk::RedCol rc;
                    rc.addr = cell_addr(L, blk, cc);
                    rc.nv = vk::box_ncells_dim(sp, 1);
                    rc.level = l;
                    rc.j0 = sp.lo[1];
                    cols.push_back(rc);
                }
                for (int xc = sp.lo[0]; xc <= sp.hi[0]; ++xc)
                    for (int s = 0; s < R; ++s) {
                        vk::RedContrib k;
                        k.cs = base + (xc - sp.lo[0]);            // grown column xc - 2
                        k.dv = L->h[1];
                        for (int j = 0; j < 5; ++j) k.b[j] = b5[(size_t)s * 5 + j];
                        per_x[(size_t)xc * R + s].push_back(k);
                    }
            }
        }
    }
    std::vector<vk::RedContrib> con;
    std::vector<int32_t> xoff(nxf + 1, 0);
    for (int x = 0; x < nxf; ++x) {
        xoff[x] = (int32_t)con.size();
        con.insert(con.end(), per_x[x].begin(), per_x[x].end());
    }
    xoff[nxf] = (int32_t)con.size();
    vk::RedPlan* P = new vk::RedPlan();
    P->st = Lf->stream;
    for (int l = 0; l < nlev; ++l) P->uids.push_back(levels[l]->uid);
    P->nxf = nxf;
    P->ncols = (int64_t)cols.size();
    P->ncontrib = (int64_t)con.size();
    cudaStream_t st = Lf->stream;
    int rc;
    if ((rc = upload(&P->d_cols, cols, st)) || (rc = upload(&P->d_contrib, con, st)) ||
        (rc = upload(&P->d_xoff, xoff, st))) {
        vk::free_red_plan(P);
        return rc;
    }
    if (!cols.empty()) VK_CUDA(cudaMallocAsync((void**)&P->d_colsum, sizeof(double) * cols.size(), st));
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { vk::free_red_plan(P); return vk::cuda_check(e, "reduction plan upload"); }
    *out = P;
    return VLASOV_OK;
}
}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* vlasov_last_error(void) { return vk::g_err.c_str(); }
int vlasov_version(void) { return 1; }
int vlasov_device_ok(void) { return device_ok_impl(); }

int vlasov_level_create(const vlasov_geom* geom, const int32_t ratio_to_level0[4], const vlasov_box* boxes,
                        int32_t nboxes, const vlasov_level* coarser, void* cuda_stream, vlasov_level** out) {
    VK_NVTX();
    if (!geom || !ratio_to_level0 || !boxes || !out) return vk::fail(VLASOV_EINVAL, "null argument");
    *out = nullptr;
    const int nd = geom->ndim;
    if (nd != 2 && nd != 4) return vk::fail(VLASOV_EINVAL, "ndim must be 2 or 4");
    if (nboxes < 1) return vk::fail(VLASOV_EINVAL, "nboxes < 1");
    vlasov_level* L = new vlasov_level();
    L->ndim = nd;
    L->ncfg = nd / 2;
    L->stream = (cudaStream_t)cuda_stream;
    L->uid = g_uid++;
    L->coarser = coarser;
    L->coarser_uid = coarser ? coarser->uid : 0;
    for (int d = 0; d < nd; ++d) {
        if (ratio_to_level0[d] < 1) { free_level(L); return vk::fail(VLASOV_EINVAL, "ratio < 1"); }
        if (geom->domain.lo[d] != 0 || geom->domain.hi[d] < 0) {
            free_level(L);
            return vk::fail(VLASOV_EINVAL, "level-0 domain must start at 0 and be non-empty");
        }
        L->ratio[d] = ratio_to_level0[d];
        L->dom[d] = (geom->domain.hi[d] + 1) * L->ratio[d];
        L->lower[d] = geom->lower[d];
        L->h[d] = geom->dx0[d] / L->ratio[d];
    }
    if (coarser) {
        if (coarser->ndim != nd) { free_level(L); return vk::fail(VLASOV_EINVAL, "coarser level ndim mismatch"); }
        for (int d = 0; d < nd; ++d) {
            if (L->ratio[d] % coarser->ratio[d]) {
                free_level(L);
                return vk::fail(VLASOV_EINVAL, "ratio not a multiple of the coarser level's ratio");
            }
            L->coarse_ratio[d] = L->ratio[d] / coarser->ratio[d];
            if (L->coarse_ratio[d] > vk::MAXR) { free_level(L); return vk::fail(VLASOV_EUNSUPPORTED, "ratio > 16"); }
        }
    }
    // boxes: inside the domain, non-empty, disjoint
    Box bbox;
    int64_t total = 0;
    for (int p = 0; p < nboxes; ++p) {
        Box b;
        for (int d = 0; d < nd; ++d) {
            b.lo[d] = boxes[p].lo[d];
            b.hi[d] = boxes[p].hi[d];
            if (b.lo[d] > b.hi[d]) { free_level(L); return vk::fail(VLASOV_EINVAL, "empty box"); }
            if (b.lo[d] < 0 || b.hi[d] >= L->dom[d]) { free_level(L); return vk::fail(VLASOV_ENEST, "box outside the level domain"); }
            bbox.lo[d] = p ? std::min(bbox.lo[d], b.lo[d]) : b.lo[d];
            bbox.hi[d] = p ? std::max(bbox.hi[d], b.hi[d]) : b.hi[d];
        }
        total += vk::box_ncells(b, nd);
        L->boxes.push_back(b);
    }
    {   // disjointness
        int64_t tot = 1;
        for (int d = 0; d < nd; ++d) tot *= L->dom[d];
        bool overlap = false;
        if (nd == 2) {                           // per row: sorted v intervals must not overlap
            const Owner o = make_owner(L, L->boxes);
            for (const auto& r : o.rows)
                for (size_t k = 1; k < r.size(); ++k)
                    if (r[k][0] <= r[k - 1][1]) overlap = true;
        } else {
            Owner o;
            o.nd = nd;
            for (int d = 0; d < nd; ++d) o.dom[d] = L->dom[d];
            std::vector<uint8_t> cnt(tot, 0);
            for (const Box& b : L->boxes)
                for_each_cell(b, nd, [&](const int* c) { if (cnt[o.lin(c)]++) overlap = true; });
        }
        if (overlap) { free_level(L); return vk::fail(VLASOV_ENEST, "boxes overlap"); }
        if (!coarser && total != tot) { free_level(L); return vk::fail(VLASOV_ENEST, "level 0 must tile the domain"); }
        if (coarser) {   // proper nesting: coarse parents of every fine cell on the coarser level
            Owner co = make_owner(coarser, coarser->boxes);
            bool bad = false;
            for (const Box& b : L->boxes) {
                Box cb = vk::box_coarsen(b, L->coarse_ratio, nd);
                for_each_cell(cb, nd, [&](const int* c) { if (co.find(c) < 0) bad = true; });
            }
            if (bad) { free_level(L); return vk::fail(VLASOV_ENEST, "level not nested in the coarser level"); }
        }
    }
    // storage blocks
    L->single_block = (total == vk::box_ncells(bbox, nd));
    if (L->single_block) {
        L->blocks.push_back(bbox);
        L->patch_block.assign(nboxes, 0);
    } else {
        L->blocks = L->boxes;
        for (int p = 0; p < nboxes; ++p) L->patch_block.push_back(p);
    }
    bool covers_domain = L->single_block;
    for (int d = 0; d < nd && covers_domain; ++d) covers_domain = (bbox.lo[d] == 0 && bbox.hi[d] == L->dom[d] - 1);
    L->single_block = covers_domain && L->single_block;
    if (!covers_domain && L->blocks.size() == 1 && nboxes > 1) {
        // a single rectangle not covering the domain still stores as one block
    }
    int64_t off = 0;
    for (const Box& b : L->blocks) {
        std::array<int64_t, 4> st = {0, 0, 0, 0};
        int64_t ext[4];
        for (int d = 0; d < nd; ++d) ext[d] = vk::box_ncells_dim(b, d) + 2 * vk::G;
        ext[nd - 1] = (ext[nd - 1] + 1) & ~int64_t(1);                // even pitch (16-B rows)
        st[nd - 1] = 1;
        for (int d = nd - 2; d >= 0; --d) st[d] = st[d + 1] * ext[d + 1];
        L->block_off.push_back(off);
        L->block_str.push_back(st);
        off += ((st[0] * ext[0] + 31) / 32) * 32;                        // 256-B aligned blocks
    }
    L->field_doubles = off;
    L->e_doubles = (nd == 2) ? (int64_t)(L->dom[0] + 4) : (int64_t)2 * (L->dom[0] + 4) * (L->dom[1] + 4);

    int rc = VLASOV_OK;
    std::vector<int64_t> copies;
    std::vector<vk::CFTask> cfs;
    std::vector<vk::PhysTask> phys;
    std::vector<vk::RefluxTask> reflux;
    std::vector<int64_t> reflux_cells;
    std::vector<int32_t> reflux_off;
    std::vector<vk::AvgTask> avg;
    std::vector<vk::PhysTask4> phys4;
    static const bool prof = std::getenv("VLASOV_PROFILE_CREATE") != nullptr;
    auto tnow = [] { return std::chrono::steady_clock::now(); };
    auto us = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::micro>(b - a).count();
    };
    const auto t0 = tnow();
    auto t1 = t0, t2 = t0, t3 = t0;
    if (nd == 2) {
        rc = build_tiles_1d(L, device_ok_impl() != 0);
        t1 = tnow();
        if (!rc) rc = build_ghost_tasks(L, coarser, copies, cfs, phys);
        t2 = tnow();
        if (!rc && coarser) rc = build_amr_tasks(L, coarser, reflux, reflux_cells, reflux_off, avg);
        t3 = tnow();
        if (prof)
            fprintf(stderr, "level_create build: tiles %.1f ghost %.1f amr %.1f us (copies %zu cf %zu phys %zu reflux %zu avg %zu)\n",
                    us(t0, t1), us(t1, t2), us(t2, t3), copies.size() / 2, cfs.size(), phys.size(), reflux.size(), avg.size());
    } else if (!L->single_block) {
        // 2D+2V hierarchy level (N3): one block per patch, ghost tasks (siblings / periodic
        // images, coarse-fine) and the characteristic velocity tasks (v_x pass, then v_y pass)
        rc = build_ghost_tasks(L, coarser, copies, cfs, phys);
        if (!rc) rc = build_phys4_tasks(L, phys4, L->n_phys4);
        L->ghost4_built = true;
    } else {
        // 2D+2V: uniform levels stored as one block covering the periodic domain (in-kernel
        // ghosts); the stage kernel marches along x in strips sized for about one wave
        if (L->field_doubles >= ((int64_t)1 << 31))
            rc = vk::fail(VLASOV_EUNSUPPORTED, "2D+2V: level block larger than 2^31 doubles");
        else if (L->dom[3] % 2 || L->dom[2] % 4 || L->dom[2] < 4 || L->dom[3] < 4)
            rc = vk::fail(VLASOV_EINVAL, "2D+2V: need nvx % 4 == 0, nvy even and >= 4 cells per velocity dim");
        else {
            const int nmt = (L->dom[3] + 63) / 64, nlg = L->dom[2] / 4;   // CTA tile: 4 vx lines x 64 vy
            const int64_t per = (int64_t)nmt * nlg * L->dom[1];
            // about one wave of 2 CTAs per SM, strips of at least 8 rows
            L->strips2 = (int)std::max<int64_t>(1, std::min<int64_t>(L->dom[0] / 8, (148 * 2 + per - 1) / per));
            if (const char* e = std::getenv("VLASOV_STRIPS2")) L->strips2 = std::max(1, std::min(L->dom[0] / 4, atoi(e)));
            L->self_ghost_ok = true;
            L->n_vtiles = L->dom[2] * nmt;                 // moment partial planes
        }
    }
    std::vector<vk::Patch4> patch4;
    std::vector<vk::FaceAvgTask> fcoarsen4;
    std::vector<vk::AvgTask4> avg4;
    if (!rc && nd == 4) rc = build_fstar4(L, coarser, patch4, fcoarsen4, avg4);
    if (rc) { free_level(L); return rc; }
    L->n_fcoarsen4 = (int64_t)fcoarsen4.size();
    L->n_avg4 = (int64_t)avg4.size();
    L->n_copy = (int64_t)copies.size() / 2;
    L->n_cf = (int64_t)cfs.size();
    L->n_phys = (int64_t)phys.size();
    L->n_reflux = (int64_t)reflux.size();
    L->n_reflux_cells = (int64_t)reflux_cells.size();
    L->n_avg = (int64_t)avg.size();
    L->avg_count = L->coarse_ratio[0] * L->coarse_ratio[1];
    std::vector<double> b5(4 * vk::MAXR * 5, 0.0);
    for (int d = 0; d < nd; ++d) vk::linear5_weights(L->coarse_ratio[d], b5.data() + (size_t)d * 5 * vk::MAXR);
    if (!device_ok_impl()) {            // host metadata only (queries work, compute calls fail)
        *out = L;
        return VLASOV_OK;
    }
    VK_CUDA(cudaMallocAsync((void**)&L->d_scalar, sizeof(double), L->stream));
    if (!L->single_block && L->ndim == 2) {      // tag scratch of multi-patch levels (regrid)
        int64_t tb = (int64_t)L->dom[0] * L->dom[1];
        VK_CUDA(cudaMallocAsync((void**)&L->d_rawtags, (size_t)tb, L->stream));
    }
    if (L->single_block && L->ndim == 4)
        VK_CUDA(cudaMallocAsync((void**)&L->d_partials, sizeof(double) * (size_t)L->n_vtiles * L->dom[0] * L->dom[1], L->stream));
    if (L->single_block && L->ndim == 2) {
        VK_CUDA(cudaMallocAsync((void**)&L->d_partials, sizeof(double) * (size_t)L->n_vtiles * L->dom[0], L->stream));
        VK_CUDA(cudaMallocAsync((void**)&L->d_tickets, sizeof(unsigned) * (size_t)std::max(1, L->n_strips), L->stream));
        VK_CUDA(cudaMemsetAsync(L->d_tickets, 0, sizeof(unsigned) * (size_t)std::max(1, L->n_strips), L->stream));
    }
    if ((rc = upload(&L->d_blocks1, L->h_blocks1, L->stream)) ||
        (rc = upload(&L->d_tiles_wide, L->h_tiles_wide, L->stream)) ||
        (rc = upload(&L->d_tiles_narrow, L->h_tiles_narrow, L->stream)) ||
        (rc = upload(&L->d_copy, copies, L->stream)) || (rc = upload(&L->d_cf, cfs, L->stream)) ||
        (rc = upload(&L->d_phys, phys, L->stream)) || (rc = upload(&L->d_b5, b5, L->stream)) ||
        (rc = upload(&L->d_phys4, phys4, L->stream)) || (rc = upload(&L->d_patch4, patch4, L->stream)) ||
        (rc = upload(&L->d_fcoarsen4, fcoarsen4, L->stream)) || (rc = upload(&L->d_avg4, avg4, L->stream)) ||
        (rc = upload(&L->d_reflux, reflux, L->stream)) || (rc = upload(&L->d_reflux_cells, reflux_cells, L->stream)) ||
        (rc = upload(&L->d_reflux_off, reflux_off, L->stream)) || (rc = upload(&L->d_avg, avg, L->stream))) {
        free_level(L);
        return rc;
    }
    const auto t4 = tnow();
    cudaError_t e = cudaStreamSynchronize(L->stream);
    if (e != cudaSuccess) { free_level(L); return vk::cuda_check(e, "level_create upload"); }
    if (prof)
        fprintf(stderr, "level_create device: alloc+upload %.1f sync %.1f us\n", us(t3, t4), us(t4, tnow()));
    *out = L;
    return VLASOV_OK;
}

int vlasov_level_destroy(vlasov_level* level) {
    VK_NVTX();
    if (level) {
        cudaStreamSynchronize(level->stream);
        free_level(level);
    }
    return VLASOV_OK;
}

int vlasov_level_get_info(const vlasov_level* L, vlasov_level_info* info) {
    VK_NVTX();
    if (!L || !info) return vk::fail(VLASOV_EINVAL, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->field_doubles = L->field_doubles;
    info->e_doubles = L->e_doubles;
    info->cfg_cells = (L->ndim == 2) ? L->dom[0] : (int64_t)L->dom[0] * L->dom[1];
    info->fluxreg_doubles = L->n_reflux;
    info->tag_bytes = 1;
    for (int d = 0; d < L->ndim; ++d) info->tag_bytes *= L->dom[d];
    info->nblocks = (int32_t)L->blocks.size();
    info->npatches = (int32_t)L->boxes.size();
    info->ntiles = (int32_t)(L->h_tiles_wide.size() + L->h_tiles_narrow.size());
    info->ndim = L->ndim;
    for (int d = 0; d < 4; ++d) {
        info->ratio[d] = L->ratio[d];
        info->domain_cells[d] = d < L->ndim ? L->dom[d] : 0;
    }
    info->ncfg[0] = L->dom[0];
    info->ncfg[1] = L->ndim == 4 ? L->dom[1] : 1;
    return VLASOV_OK;
}

int vlasov_level_layout(const vlasov_level* L, int32_t patch, int64_t* offset, int64_t strides[4]) {
    VK_NVTX();
    if (!L || !offset || !strides) return vk::fail(VLASOV_EINVAL, "null argument");
    if (patch < 0 || patch >= (int)L->boxes.size()) return vk::fail(VLASOV_EINVAL, "patch out of range");
    const int b = L->patch_block[patch];
    *offset = cell_addr(L, b, L->boxes[patch].lo);
    for (int d = 0; d < 4; ++d) strides[d] = d < L->ndim ? L->block_str[b][d] : 0;
    return VLASOV_OK;
}

int vlasov_level_ghost_map(const vlasov_level* L, int32_t patch, int32_t* kind, int32_t* src_patch,
                           int64_t* src_cell) {
    VK_NVTX();
    if (!L || !kind || !src_patch || !src_cell) return vk::fail(VLASOV_EINVAL, "null argument");
    if (patch < 0 || patch >= (int)L->boxes.size()) return vk::fail(VLASOV_EINVAL, "patch out of range");
    const int nd = L->ndim;
    const Box& B = L->boxes[patch];
    Owner own = make_owner(L, L->boxes);
    Owner cown;
    const vlasov_level* C = L->coarser;
    if (C) cown = make_owner(C, C->boxes);
    int64_t t = 0;
    int err = VLASOV_OK;
    for_each_cell(vk::box_grow(B, vk::G, nd), nd, [&](const int* c) {
        if (err) return;
        if (vk::box_contains(B, c, nd)) {
            kind[t] = VLASOV_GHOST_INTERIOR; src_patch[t] = patch; src_cell[t] = vk::box_index(B, c, nd);
        } else if (int pc = phys_code(L, c); pc >= 0) {
            kind[t] = VLASOV_GHOST_PHYS; src_patch[t] = -1; src_cell[t] = pc;
        } else {
            int w[4];
            wrap_cfg(L, c, w);
            const int q = own.find(w);
            if (q >= 0) {
                kind[t] = VLASOV_GHOST_SIBLING; src_patch[t] = q; src_cell[t] = vk::box_index(L->boxes[q], w, nd);
            } else if (C) {
                int cc[4];
                for (int d = 0; d < nd; ++d) cc[d] = vk::floordiv(w[d], L->coarse_ratio[d]);
                const int cq = cown.find(cc);
                if (cq < 0) { err = vk::fail(VLASOV_ESTENCIL, "no coarse parent"); return; }
                kind[t] = VLASOV_GHOST_COARSE; src_patch[t] = cq; src_cell[t] = vk::box_index(C->boxes[cq], cc, nd);
            } else {
                err = vk::fail(VLASOV_ENEST, "ghost cell without source");
                return;
            }
        }
        ++t;
    });
    return err;
}

// Alg.7 ComputeSubPatches
int vlasov_subpatches(const vlasov_level* const* levels, int32_t nlev, int32_t li, int32_t patch,
                      vlasov_box* out, int32_t cap, int32_t* n) {
    VK_NVTX();
    if (!levels || !n || li < 0 || li >= nlev) return vk::fail(VLASOV_EINVAL, "bad arguments");
    const vlasov_level* L = levels[li];
    if (patch < 0 || patch >= (int)L->boxes.size()) return vk::fail(VLASOV_EINVAL, "patch out of range");
    const int nd = L->ndim;
    const std::vector<Box> T = subpatches_of(levels, nlev, li, patch);
    *n = (int32_t)T.size();
    for (int i = 0; i < (int)T.size() && i < cap; ++i) {
        for (int d = 0; d < 4; ++d) {
            out[i].lo[d] = d < nd ? T[i].lo[d] : 0;
            out[i].hi[d] = d < nd ? T[i].hi[d] : 0;
        }
    }
    return VLASOV_OK;
}

int vlasov_tags_to_boxes(const uint8_t* tags, const int32_t domain_cells[4], int32_t ndim, const int32_t ratio[4],
                         int32_t tile, vlasov_box* out, int32_t cap, int32_t* n) {
    VK_NVTX();
    if (!tags || !domain_cells || !ratio || !n || ndim != 2) return vk::fail(VLASOV_EINVAL, "bad arguments");
    int foot[2];
    for (int d = 0; d < 2; ++d) {
        if (ratio[d] < 1 || tile % ratio[d]) return vk::fail(VLASOV_EINVAL, "tile must be a multiple of the ratio");
        foot[d] = tile / ratio[d];
    }
    const int nx = domain_cells[0], nv = domain_cells[1];
    int cnt = 0;
    for (int tx = 0; tx < nx / foot[0]; ++tx)
        for (int tv = 0; tv < nv / foot[1]; ++tv) {
            bool any = false;
            for (int i = tx * foot[0]; i < (tx + 1) * foot[0] && !any; ++i)
                for (int j = tv * foot[1]; j < (tv + 1) * foot[1]; ++j)
                    if (tags[(int64_t)i * nv + j]) { any = true; break; }
            if (!any) continue;
            if (cnt < cap) {
                std::memset(&out[cnt], 0, sizeof(vlasov_box));
                out[cnt].lo[0] = tx * tile; out[cnt].hi[0] = (tx + 1) * tile - 1;
                out[cnt].lo[1] = tv * tile; out[cnt].hi[1] = (tv + 1) * tile - 1;
            }
            ++cnt;
        }
    *n = cnt;
    return VLASOV_OK;
}

// Tag clustering into rectangular patches (reading #28, same rules and tie-breaks as the
// oracle): signature-based recursive bisection -- holes, then Laplacian inflection, then midpoint --
// until the fill efficiency is reached and every side is <= largest; cuts keep >= smallest cells.
namespace {
struct Clusterer {
    const uint8_t* t;
    int nx, nv, lo0, lo1;
    int smallest[2], largest[2];
    double eff;
    std::vector<Box> out;
    bool tag(int i, int j) const { return t[(int64_t)i * nv + j] != 0; }
    void tile_large(const Box& b) {
        std::vector<std::pair<int, int>> r[2];
        for (int d = 0; d < 2; ++d) {
            const int n = b.hi[d] - b.lo[d] + 1, k = (n + largest[d] - 1) / largest[d];
            for (int j = 0; j < k; ++j)
                r[d].push_back({b.lo[d] + (int)((int64_t)n * j / k), b.lo[d] + (int)((int64_t)n * (j + 1) / k) - 1});
        }
        for (auto& a : r[0])
            for (auto& c : r[1]) {
                Box o;
                o.lo[0] = a.first; o.hi[0] = a.second; o.lo[1] = c.first; o.hi[1] = c.second;
                out.push_back(o);
            }
    }
    // region in local tag indices [a0, b0] x [a1, b1]
    void rec(int a0, int b0, int a1, int b1) {
        int lo[2] = {INT32_MAX, INT32_MAX}, hi[2] = {-1, -1};
        for (int i = a0; i <= b0; ++i)
            for (int j = a1; j <= b1; ++j)
                if (tag(i, j)) {
                    lo[0] = std::min(lo[0], i); hi[0] = std::max(hi[0], i);
                    lo[1] = std::min(lo[1], j); hi[1] = std::max(hi[1], j);
                }
        if (hi[0] < 0) return;
        const int n[2] = {hi[0] - lo[0] + 1, hi[1] - lo[1] + 1};
        std::vector<int64_t> sig[2] = {std::vector<int64_t>(n[0], 0), std::vector<int64_t>(n[1], 0)};
        int64_t cnt = 0;
        for (int i = lo[0]; i <= hi[0]; ++i)
            for (int j = lo[1]; j <= hi[1]; ++j)
                if (tag(i, j)) { ++sig[0][i - lo[0]]; ++sig[1][j - lo[1]]; ++cnt; }
        const bool too_big = n[0] > largest[0] || n[1] > largest[1];
        const double e = (double)cnt / (double)((int64_t)n[0] * n[1]);
        Box B;
        B.lo[0] = lo[0] + lo0; B.hi[0] = hi[0] + lo0; B.lo[1] = lo[1] + lo1; B.hi[1] = hi[1] + lo1;
        if (e >= eff && !too_big) { out.push_back(B); return; }
        int order[2] = {0, 1};
        if (n[1] > n[0]) { order[0] = 1; order[1] = 0; }
        auto adm = [&](int d, int c) { return c >= smallest[d] && n[d] - c >= smallest[d]; };
        int cd = -1, cc = -1;
        for (int oi = 0; oi < 2 && cd < 0; ++oi) {                     // a. holes
            const int d = order[oi];
            int64_t best = -1;
            for (int c = 1; c < n[d]; ++c)
                if ((sig[d][c - 1] == 0 || sig[d][c] == 0) && adm(d, c)) {
                    const int64_t key = std::llabs(2LL * c - n[d]);
                    if (best < 0 || key < best) { best = key; cc = c; cd = d; }
                }
        }
        for (int oi = 0; oi < 2 && cd < 0; ++oi) {                     // b. inflection
            const int d = order[oi];
            if (n[d] < 3) continue;
            std::vector<int64_t> lap(n[d] - 2);
            for (int j = 0; j + 2 < n[d]; ++j) lap[j] = sig[d][j] - 2 * sig[d][j + 1] + sig[d][j + 2];
            int64_t bj = 0, bcent = 0;
            int bc = -1;
            for (int j = 1; j < (int)lap.size(); ++j)
                if ((lap[j - 1] < 0 && lap[j] > 0) || (lap[j - 1] > 0 && lap[j] < 0)) {
                    const int c = j + 1;
                    if (!adm(d, c)) continue;
                    const int64_t jump = std::llabs(lap[j] - lap[j - 1]), cent = std::llabs(2LL * c - n[d]);
                    if (bc < 0 || jump > bj || (jump == bj && (cent < bcent || (cent == bcent && c < bc)))) {
                        bj = jump; bcent = cent; bc = c;
                    }
                }
            if (bc >= 0) { cd = d; cc = bc; }
        }
        for (int oi = 0; oi < 2 && cd < 0; ++oi) {                     // c. bisection
            const int d = order[oi], c = n[d] / 2;
            if (adm(d, c)) { cd = d; cc = c; }
        }
        if (cd < 0) {
            if (too_big) tile_large(B);
            else out.push_back(B);
            return;
        }
        if (cd == 0) {
            rec(lo[0], lo[0] + cc - 1, lo[1], hi[1]);
            rec(lo[0] + cc, hi[0], lo[1], hi[1]);
        } else {
            rec(lo[0], hi[0], lo[1], lo[1] + cc - 1);
            rec(lo[0], hi[0], lo[1] + cc, hi[1]);
        }
    }
};
}  // namespace

int vlasov_cluster_tags(const uint8_t* tags, const int32_t shape[2], const int32_t lo[2],
                        const int32_t smallest[2], const int32_t largest[2], double efficiency,
                        vlasov_box* out, int32_t cap, int32_t* n) {
    VK_NVTX();
    if (!tags || !shape || !lo || !smallest || !largest || !n) return vk::fail(VLASOV_EINVAL, "null argument");
    if (shape[0] < 0 || shape[1] < 0 || !(efficiency > 0.0) || efficiency > 1.0)
        return vk::fail(VLASOV_EINVAL, "cluster_tags: bad shape or efficiency");
    for (int d = 0; d < 2; ++d)
        if (smallest[d] < 1 || largest[d] < smallest[d])
            return vk::fail(VLASOV_EINVAL, "cluster_tags: need 1 <= smallest <= largest");
    Clusterer C;
    C.t = tags; C.nx = shape[0]; C.nv = shape[1]; C.lo0 = lo[0]; C.lo1 = lo[1];
    for (int d = 0; d < 2; ++d) { C.smallest[d] = smallest[d]; C.largest[d] = largest[d]; }
    C.eff = efficiency;
    if (shape[0] > 0 && shape[1] > 0) C.rec(0, shape[0] - 1, 0, shape[1] - 1);
    std::sort(C.out.begin(), C.out.end(), [](const Box& a, const Box& b) { return vk::box_less(a, b, 2); });
    *n = (int32_t)C.out.size();
    for (int i = 0; i < (int)C.out.size() && i < cap; ++i) {
        std::memset(&out[i], 0, sizeof(vlasov_box));
        for (int d = 0; d < 2; ++d) { out[i].lo[d] = C.out[i].lo[d]; out[i].hi[d] = C.out[i].hi[d]; }
    }
    return VLASOV_OK;
}

// Boxes of the next finer level from the dilated tags of `level` (reading #28): tags restricted to
// the nesting region (cells whose Chebyshev `nest`-neighbourhood lies in the level's patches; x
// periodic, beyond the velocity domain counts as covered), clustered, each cluster intersected with
// the nesting region (row-run decomposition), refined by `ratio`.  Same rules as the oracle.
int vlasov_regrid_boxes(const vlasov_level* L, const uint8_t* tags, const int32_t ratio[2],
                        const int32_t smallest[2], const int32_t largest[2], double efficiency, int32_t nest,
                        vlasov_box* out, int32_t cap, int32_t* n) {
    VK_NVTX();
    if (!L || !tags || !ratio || !smallest || !largest || !n) return vk::fail(VLASOV_EINVAL, "null argument");
    if (L->ndim != 2) return vk::fail(VLASOV_EUNSUPPORTED, "regrid_boxes: 1D+1V levels only");
    if (nest < 0 || ratio[0] < 1 || ratio[1] < 1) return vk::fail(VLASOV_EINVAL, "regrid_boxes: bad nest or ratio");
    const int nx = L->dom[0], nv = L->dom[1];
    std::vector<uint8_t> cov((size_t)nx * nv, 0), nm((size_t)nx * nv, 0);
    for (const Box& b : L->boxes)
        for (int x = b.lo[0]; x <= b.hi[0]; ++x)
            for (int v = b.lo[1]; v <= b.hi[1]; ++v) cov[(size_t)x * nv + v] = 1;
    for (int x = 0; x < nx; ++x)
        for (int v = 0; v < nv; ++v) {
            bool ok = true;
            for (int a = -nest; a <= nest && ok; ++a)
                for (int c = -nest; c <= nest && ok; ++c) {
                    const int vv = v + c;
                    if (vv < 0 || vv >= nv) continue;
                    ok = cov[(size_t)wrap(x + a, nx) * nv + vv] != 0;
                }
            nm[(size_t)x * nv + v] = ok ? 1 : 0;
        }
    std::vector<uint8_t> t((size_t)nx * nv);
    for (size_t i = 0; i < t.size(); ++i) t[i] = (tags[i] && nm[i]) ? 1 : 0;
    int sm[2], lg[2];
    for (int d = 0; d < 2; ++d) {
        sm[d] = (smallest[d] + ratio[d] - 1) / ratio[d];
        lg[d] = std::max(sm[d], largest[d] / ratio[d]);
    }
    Clusterer C;
    C.t = t.data(); C.nx = nx; C.nv = nv; C.lo0 = 0; C.lo1 = 0;
    for (int d = 0; d < 2; ++d) { C.smallest[d] = sm[d]; C.largest[d] = lg[d]; }
    C.eff = efficiency;
    if (nx > 0 && nv > 0) C.rec(0, nx - 1, 0, nv - 1);
    std::vector<Box> res;
    for (const Box& b : C.out) {               // cluster box  x  nesting region, row runs
        std::map<std::pair<int, int>, int> active;
        for (int x = b.lo[0]; x <= b.hi[0] + 1; ++x) {
            std::vector<std::pair<int, int>> cur;
            if (x <= b.hi[0]) {
                int j = b.lo[1];
                while (j <= b.hi[1]) {
                    if (nm[(size_t)x * nv + j]) {
                        int k = j;
                        while (k + 1 <= b.hi[1] && nm[(size_t)x * nv + k + 1]) ++k;
                        cur.push_back({j, k});
                        j = k + 1;
                    } else {
                        ++j;
                    }
                }
            }
            for (auto it = active.begin(); it != active.end();) {
                if (std::find(cur.begin(), cur.end(), it->first) == cur.end()) {
                    Box o;
                    o.lo[0] = it->second; o.hi[0] = x - 1; o.lo[1] = it->first.first; o.hi[1] = it->first.second;
                    res.push_back(o);
                    it = active.erase(it);
                } else {
                    ++it;
                }
            }
            for (auto& r : cur)
                if (!active.count(r)) active[r] = x;
        }
    }
    std::vector<Box> fine;
    for (const Box& b : res) fine.push_back(vk::box_refine(b, ratio, 2));
    std::sort(fine.begin(), fine.end(), [](const Box& a, const Box& b) { return vk::box_less(a, b, 2); });
    *n = (int32_t)fine.size();
    for (int i = 0; i < (int)fine.size() && i < cap; ++i) {
        std::memset(&out[i], 0, sizeof(vlasov_box));
        for (int d = 0; d < 2; ++d) { out[i].lo[d] = fine[i].lo[d]; out[i].hi[d] = fine[i].hi[d]; }
    }
    return VLASOV_OK;
}

// ---------------------------------------------------------------- compute entry points
int vlasov_fill_ghosts(vlasov_level* L, double* f, const vlasov_level* coarser, const double* f_coarse,
                       const double* E_bc, const double* f0v, int32_t interp) {
    VK_NVTX();
    if (!L || !f) return vk::fail(VLASOV_EINVAL, "null argument");
    if (L->ndim == 4 && !L->ghost4_built) {
        // a 2D+2V level stored as one block (the stage kernel derives its ghosts itself): the task
        // lists of the ghost frame (periodic images, velocity condition) are built on first use
        std::vector<int64_t> copies;
        std::vector<vk::CFTask> cfs;
        std::vector<vk::PhysTask> phys;
        std::vector<vk::PhysTask4> phys4;
        int rc = build_ghost_tasks(L, L->coarser, copies, cfs, phys);
        if (!rc) rc = build_phys4_tasks(L, phys4, L->n_phys4);
        if (!rc && device_ok_impl()) {
            vk::dfree(L->d_copy, L->stream);
            vk::dfree(L->d_cf, L->stream);
            if ((rc = upload(&L->d_copy, copies, L->stream)) || (rc = upload(&L->d_cf, cfs, L->stream)) ||
                (rc = upload(&L->d_phys4, phys4, L->stream)))
                return rc;
            L->n_copy = (int64_t)copies.size() / 2;
            L->n_cf = (int64_t)cfs.size();
        }
        if (rc) return rc;
        L->ghost4_built = true;
    }
    if (L->n_cf > 0 && (coarser != L->coarser || !coarser || coarser->uid != L->coarser_uid))
        return vk::fail(VLASOV_ESTALE, "fill_ghosts: coarser level does not match the one of level_create");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    if (L->ndim == 4) return vk::launch_fill4(L, f, f_coarse, E_bc, f0v, interp);
    return vk::launch_fill(L, f, f_coarse, E_bc, f0v, interp);
}

int vlasov_rhs(vlasov_level* L, const double* f, const double* E, double* k, int32_t recon) {
    VK_NVTX();
    if (!L || !f || !E || !k) return vk::fail(VLASOV_EINVAL, "null argument");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    if (recon != VLASOV_CENTERED4 && recon != VLASOV_UPWIND) return vk::fail(VLASOV_EINVAL, "bad recon");
    if (k == f) return vk::fail(VLASOV_EINVAL, "k must not alias f");
    if (L->ndim == 4) {
        // 2D+2V: one periodic block (x, y wrapped in-kernel), velocity ghost frame of f current
        if (!L->self_ghost_ok) return vk::fail(VLASOV_EUNSUPPORTED, "rhs: 2D+2V needs one periodic block");
        return vk::launch_stage_2d2v(L, 0, 0.0, const_cast<double*>(f), f, nullptr, k, E, nullptr, nullptr, recon,
                                     nullptr);
    }
    return vk::launch_stage_1d1v(L, 0, 0.0, nullptr, f, nullptr, k, E, nullptr, nullptr, recon, nullptr);
}

int vlasov_rk4_stage(vlasov_level* L, int32_t stage, double dt, double* f_n, const double* f_s, double* u,
                     double* f_next, const double* E, const double* E_bc, const double* f0v, int32_t recon,
                     double* rho_next) {
    VK_NVTX();
    if (!L || !f_s || !f_next || !E) return vk::fail(VLASOV_EINVAL, "null argument");
    if (stage < 1 || stage > 4) return vk::fail(VLASOV_EINVAL, "stage must be 1..4");
    if (stage >= 2 && !f_n) return vk::fail(VLASOV_EINVAL, "f_n required");
    if ((stage == 2 || stage == 4) && !u) return vk::fail(VLASOV_EINVAL, "u required");
    if (recon != VLASOV_CENTERED4 && recon != VLASOV_UPWIND) return vk::fail(VLASOV_EINVAL, "bad recon");
    if (rho_next && !L->single_block) return vk::fail(VLASOV_EUNSUPPORTED, "fused moment needs a single-block level");
    if (E_bc && !f0v) return vk::fail(VLASOV_EINVAL, "E_bc needs f0v");
    // neighbouring CTAs read halo rows of f_s while others write f_next rows
    if (f_next == f_s) return vk::fail(VLASOV_EINVAL, "f_next must not alias f_s");
    if (f0v && !L->self_ghost_ok)
        return vk::fail(VLASOV_EUNSUPPORTED, "in-kernel ghosts need one periodic block with nv a multiple of 4");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    if (L->ndim == 4) {
        if (!E_bc) return vk::fail(VLASOV_EUNSUPPORTED, "2D+2V stage: in-kernel ghosts (E_bc, f0v) required");
        return vk::launch_stage_2d2v(L, stage, dt, stage == 1 ? const_cast<double*>(f_s) : f_n, f_s, u, f_next, E,
                                     E_bc, f0v, recon, rho_next);
    }
    return vk::launch_stage_1d1v(L, stage, dt, stage == 1 ? const_cast<double*>(f_s) : f_n, f_s, u, f_next, E,
                                 E_bc, f0v, recon, rho_next);
}

int vlasov_rk4_stage_vp(vlasov_level* L, const vlasov_poisson* plan, int32_t stage, double dt, double* f_n,
                        const double* f_s, double* u, double* f_next, const double* rho_s, double* E_s,
                        const double* E_bc, const double* f0v, int32_t recon, double* rho_next) {
    VK_NVTX();
    if (!L || !plan || !f_s || !f_next || !rho_s || !E_s || !f0v)
        return vk::fail(VLASOV_EINVAL, "null argument");
    if (stage < 1 || stage > 4) return vk::fail(VLASOV_EINVAL, "stage must be 1..4");
    if (stage >= 2 && !f_n) return vk::fail(VLASOV_EINVAL, "f_n required");
    if ((stage == 2 || stage == 4) && !u) return vk::fail(VLASOV_EINVAL, "u required");
    if (recon != VLASOV_CENTERED4 && recon != VLASOV_UPWIND) return vk::fail(VLASOV_EINVAL, "bad recon");
    if (L->ndim != 2 || !L->self_ghost_ok)
        return vk::fail(VLASOV_EUNSUPPORTED, "rk4_stage_vp: one periodic 1D+1V block with nv % 4 == 0");
    if (plan->n != L->dom[0] || std::fabs(plan->dx - L->h[0]) > 1e-12 * L->h[0])
        return vk::fail(VLASOV_EINVAL, "rk4_stage_vp: Poisson plan does not match the level's x mesh");
    if (plan->n > 4096 || plan->n % 2)
        return vk::fail(VLASOV_EUNSUPPORTED, "rk4_stage_vp: needs an even n <= 4096 (else use poisson_solve)");
    if (rho_next == rho_s) return vk::fail(VLASOV_EINVAL, "rk4_stage_vp: rho_next must not alias rho_s");
    // CTAs write rows of E_s while others read E_bc
    if (E_bc && E_bc == E_s) return vk::fail(VLASOV_EINVAL, "rk4_stage_vp: E_bc must not alias E_s");
    if (f_next == f_s) return vk::fail(VLASOV_EINVAL, "f_next must not alias f_s");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_stage_1d1v(L, stage, dt, stage == 1 ? const_cast<double*>(f_s) : f_n, f_s, u, f_next, E_s,
                                 E_bc, f0v, recon, rho_next, rho_s, plan->d_gE, E_s, plan->d_gX,
                                 split_field() ? plan->d_hs : nullptr, plan->K2, plan->Kn);
}

int vlasov_reduce_charge(const vlasov_level* const* levels, int32_t nlev, const double* const* f, double q,
                         double base, int32_t accumulate, double* rho_finest) {
    VK_NVTX();
    if (!levels || nlev < 1 || !rho_finest || !f) return vk::fail(VLASOV_EINVAL, "null argument");
    if (nlev > vk::MAXLEV) return vk::fail(VLASOV_EUNSUPPORTED, "more than 8 levels");
    for (int l = 0; l < nlev; ++l)
        if (!levels[l] || !f[l]) return vk::fail(VLASOV_EINVAL, "reduce_moment: level / field pointer required");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    if (nlev == 1 && levels[0]->single_block && levels[0]->ndim == 2)
        return vk::launch_moment_direct(levels[0], f[0], rho_finest, q, base, accumulate);
    if (nlev == 1 && levels[0]->single_block && levels[0]->ndim == 4) {
        if (q != -1.0 || base != 1.0 || accumulate)
            return vk::fail(VLASOV_EUNSUPPORTED, "reduce_charge: 2D+2V levels compute the electron density 1 - n only");
        return vk::launch_moment_2d2v(levels[0], f[0], rho_finest);
    }
    const vlasov_level* Lf = levels[nlev - 1];
    if (Lf->ndim == 4) {                            // 2D+2V hierarchy: Alg.8 4D -> 2D (N3)
        if (q != -1.0 || base != 1.0 || accumulate)
            return vk::fail(VLASOV_EUNSUPPORTED, "reduce_charge: 2D+2V levels compute the electron density 1 - n only");
        bool fresh4 = Lf->red_plan4 != nullptr && (int)Lf->red_plan4->uids.size() == nlev;
        for (int l = 0; fresh4 && l < nlev; ++l) fresh4 = Lf->red_plan4->uids[l] == levels[l]->uid;
        if (!fresh4) {
            vk::free_red_plan4(Lf->red_plan4);
            Lf->red_plan4 = nullptr;
            vk::RedPlan4* P = nullptr;
            if (int rc = build_red_plan4(levels, nlev, &P)) return rc;
            Lf->red_plan4 = P;
        }
        return vk::launch_reduce_subpatch4(Lf->red_plan4, f, nlev, rho_finest, Lf->stream);
    }
    bool fresh = Lf->red_plan != nullptr && (int)Lf->red_plan->uids.size() == nlev;
    for (int l = 0; fresh && l < nlev; ++l) fresh = Lf->red_plan->uids[l] == levels[l]->uid;
    if (!fresh) {                                   // observer: rebuild after a regrid
        vk::free_red_plan(Lf->red_plan);
        Lf->red_plan = nullptr;
        vk::RedPlan* P = nullptr;
        if (int rc = build_red_plan(levels, nlev, &P)) return rc;
        Lf->red_plan = P;
    }
    return vk::launch_reduce_subpatch(Lf->red_plan, f, nlev, rho_finest, Lf->stream, q, base, accumulate);
}

int vlasov_reduce_moment(const vlasov_level* const* levels, int32_t nlev, const double* const* f,
                         double* rho_finest) {
    VK_NVTX();
    return vlasov_reduce_charge(levels, nlev, f, -1.0, 1.0, 0, rho_finest);
}

int vlasov_reduce_current(const vlasov_level* const* levels, int32_t nlev, const double* const* f, double q,
                          int32_t accumulate, double* j) {
    VK_NVTX();
    if (!levels || nlev < 1 || !f || !j) return vk::fail(VLASOV_EINVAL, "null argument");
    if (nlev > vk::MAXLEV) return vk::fail(VLASOV_EUNSUPPORTED, "more than 8 levels");
    for (int l = 0; l < nlev; ++l) {
        if (!levels[l] || !f[l]) return vk::fail(VLASOV_EINVAL, "reduce_current: level / field pointer required");
        if (levels[l]->ndim != 2) return vk::fail(VLASOV_EUNSUPPORTED, "current moment: 1D+1V levels");
    }
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    if (nlev == 1 && levels[0]->single_block) return vk::launch_current(levels[0], f[0], q, accumulate, j);
    const vlasov_level* Lf = levels[nlev - 1];
    bool fresh = Lf->red_plan != nullptr && (int)Lf->red_plan->uids.size() == nlev;
    for (int l = 0; fresh && l < nlev; ++l) fresh = Lf->red_plan->uids[l] == levels[l]->uid;
    if (!fresh) {
        vk::free_red_plan(Lf->red_plan);
        Lf->red_plan = nullptr;
        vk::RedPlan* P = nullptr;
        if (int rc = build_red_plan(levels, nlev, &P)) return rc;
        Lf->red_plan = P;
    }
    double vlo[vk::MAXLEV], dv[vk::MAXLEV];
    for (int l = 0; l < nlev; ++l) { vlo[l] = levels[l]->lower[1]; dv[l] = levels[l]->h[1]; }
    return vk::launch_reduce_first_subpatch(Lf->red_plan, f, nlev, vlo, dv, j, Lf->stream, q, accumulate);
}

int vlasov_level_set_moment_base(vlasov_level* L, double base) {
    VK_NVTX();
    if (!L) return vk::fail(VLASOV_EINVAL, "null argument");
    if (!L->single_block) return vk::fail(VLASOV_EUNSUPPORTED, "moment base: one periodic block only");
    L->moment_base = base;
    return VLASOV_OK;
}

int vlasov_level_set_velocity_faces(vlasov_level* L, int32_t phys_lo, int32_t phys_hi) {
    VK_NVTX();
    if (!L) return vk::fail(VLASOV_EINVAL, "null argument");
    if (!L->single_block || L->ndim != 2) return vk::fail(VLASOV_EUNSUPPORTED, "velocity faces: one periodic 1D+1V block only");
    L->vphys[0] = phys_lo ? 1 : 0;
    L->vphys[1] = phys_hi ? 1 : 0;
    return VLASOV_OK;
}

int vlasov_vslab_pack(const vlasov_level* L, const double* f, double* lo, double* hi) {
    VK_NVTX();
    if (!L || !f) return vk::fail(VLASOV_EINVAL, "null argument");
    if (L->ndim != 2 || !L->single_block || L->dom[1] < 2)
        return vk::fail(VLASOV_EUNSUPPORTED, "vslab: one 1D+1V block with >= 2 velocity cells");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_vslab(L, const_cast<double*>(f), lo, hi, true);
}

int vlasov_vslab_unpack(const vlasov_level* L, double* f, const double* lo, const double* hi) {
    VK_NVTX();
    if (!L || !f) return vk::fail(VLASOV_EINVAL, "null argument");
    if (L->ndim != 2 || !L->single_block || L->dom[1] < 2)
        return vk::fail(VLASOV_EUNSUPPORTED, "vslab: one 1D+1V block with >= 2 velocity cells");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_vslab(L, f, const_cast<double*>(lo), const_cast<double*>(hi), false);
}

int vlasov_absmax(const double* x, int64_t n, double* out, void* cuda_stream) {
    VK_NVTX();
    if (!x || !out || n < 0) return vk::fail(VLASOV_EINVAL, "null argument or n < 0");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_absmax(x, n, out, (cudaStream_t)cuda_stream);
}

// Adaptive time step (reading #29): dt = min(cfl / rate, growth * dt_prev),
// rate = max_l (vmax / dx_l + max|E_l| / dv_l), vmax = the largest |cell-centre velocity| of the
// finest level's velocity domain; max|E_l| on the device (k_absmax), one 8-byte read per level.
int vlasov_next_dt(const vlasov_level* const* levels, int32_t nlev, const double* const* E, double dt_prev,
                   double cfl, double growth, double* dt_out) {
    VK_NVTX();
    if (!levels || !E || !dt_out || nlev < 1) return vk::fail(VLASOV_EINVAL, "null argument or nlev < 1");
    if (!(cfl > 0.0) || !(growth > 0.0) || !(dt_prev > 0.0)) return vk::fail(VLASOV_EINVAL, "next_dt: cfl, growth, dt_prev > 0");
    for (int l = 0; l < nlev; ++l)
        if (!levels[l] || !E[l] || levels[l]->ndim != 2) return vk::fail(VLASOV_EINVAL, "next_dt: 1D+1V level and E per level");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    const vlasov_level* Lf = levels[nlev - 1];
    const double dvf = Lf->h[1];
    const double vlo = Lf->lower[1] + 0.5 * dvf, vhi = Lf->lower[1] + ((double)Lf->dom[1] - 0.5) * dvf;
    const double vmax = std::max(std::fabs(vlo), std::fabs(vhi));
    std::vector<double> em(nlev, 0.0);
    for (int l = 0; l < nlev; ++l) {
        const vlasov_level* L = levels[l];
        if (int rc = vk::launch_absmax(E[l], (int64_t)L->dom[0] + 2 * vk::G, L->d_scalar, L->stream)) return rc;
        VK_CUDA(cudaMemcpyAsync(&em[l], L->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, L->stream));
    }
    for (int l = 0; l < nlev; ++l) VK_CUDA(cudaStreamSynchronize(levels[l]->stream));
    double rate = 0.0;
    for (int l = 0; l < nlev; ++l) rate = std::max(rate, vmax / levels[l]->h[0] + em[l] / levels[l]->h[1]);
    *dt_out = std::min(cfl / rate, growth * dt_prev);
    return VLASOV_OK;
}

// Alg.6 Mask Reduction: every patch refined in x (linear5, ghost columns current),
// covered cells masked, summed over v; the comparator of Alg.8.
static int build_mask_plan(const vlasov_level* const* levels, int nlev, vk::MaskPlan** out) {
    *out = nullptr;
    const vlasov_level* Lf = levels[nlev - 1];
    const int nxf = Lf->dom[0];
    std::vector<vk::MaskCol> cols;
    std::vector<uint8_t> mask;
    std::vector<double> w;
    std::map<int, int> woff;
    std::vector<std::vector<std::pair<int32_t, double>>> per_x(nxf);
    int32_t npart = 0;
    for (int l = 0; l < nlev; ++l) {
        const vlasov_level* L = levels[l];
        if (L->ndim != 2) return vk::fail(VLASOV_EUNSUPPORTED, "mask reduction: 1D+1V levels only");
        if (nxf % L->dom[0]) return vk::fail(VLASOV_EINVAL, "finest x resolution not a multiple of a level's");
        if (l > 0 && (L->coarser != levels[l - 1] || L->coarser_uid != levels[l - 1]->uid))
            return vk::fail(VLASOV_ESTALE, "reduce_moment_mask: levels are not a hierarchy (coarser mismatch)");
        const int R = nxf / L->dom[0];
        if (R > vk::MAXR) return vk::fail(VLASOV_EUNSUPPORTED, "mask reduction: x ratio to the finest level > 16");
        if (!woff.count(R)) {
            woff[R] = (int)w.size();
            std::vector<double> b((size_t)R * 5);
            vk::linear5_weights(R, b.data());
            w.insert(w.end(), b.begin(), b.end());
        }
        const int64_t moff = (int64_t)mask.size();
        std::vector<uint8_t> mu((size_t)L->dom[0] * L->dom[1], 1);
        if (l + 1 < nlev) {
            const vlasov_level* F = levels[l + 1];
            int rr[4];
            for (int d = 0; d < 2; ++d) rr[d] = F->ratio[d] / L->ratio[d];
            for (const Box& fb : F->boxes) {
                const Box cb = vk::box_coarsen(fb, rr, 2);
                for (int x = cb.lo[0]; x <= cb.hi[0]; ++x)
                    for (int v = cb.lo[1]; v <= cb.hi[1]; ++v) mu[(size_t)x * L->dom[1] + v] = 0;
            }
        }
        mask.insert(mask.end(), mu.begin(), mu.end());
        for (size_t p = 0; p < L->boxes.size(); ++p) {
            const Box& b = L->boxes[p];
            const int blk = L->patch_block[p];
            for (int xc = b.lo[0]; xc <= b.hi[0]; ++xc) {
                vk::MaskCol c;
                int cc[4] = {xc - 2, b.lo[1], 0, 0};
                c.addr = cell_addr(L, blk, cc);
                c.mask = moff + (int64_t)xc * L->dom[1] + b.lo[1];
                c.pitch = (int32_t)L->block_str[blk][0];
                c.nv = vk::box_ncells_dim(b, 1);
                c.level = l;
                c.R = R;
                c.out = npart;
                c.woff = woff[R];
                cols.push_back(c);
                for (int s = 0; s < R; ++s) per_x[(size_t)xc * R + s].push_back({npart + s, L->h[1]});
                npart += R;
            }
        }
    }
    std::vector<int32_t> xoff(nxf + 1, 0), idx;
    std::vector<double> dv;
    for (int x = 0; x < nxf; ++x) {
        xoff[x] = (int32_t)idx.size();
        for (auto& e : per_x[x]) { idx.push_back(e.first); dv.push_back(e.second); }
    }
    xoff[nxf] = (int32_t)idx.size();
    vk::MaskPlan* P = new vk::MaskPlan();
    P->st = Lf->stream;
    for (int l = 0; l < nlev; ++l) P->uids.push_back(levels[l]->uid);
    P->nxf = nxf;
    P->ncols = (int64_t)cols.size();
    P->npart = npart;
    cudaStream_t st = Lf->stream;
    int rc;
    if ((rc = upload(&P->d_cols, cols, st)) || (rc = upload(&P->d_mask, mask, st)) || (rc = upload(&P->d_w, w, st)) ||
        (rc = upload(&P->d_xoff, xoff, st)) || (rc = upload(&P->d_idx, idx, st)) || (rc = upload(&P->d_dv, dv, st))) {
        vk::free_mask_plan(P);
        return rc;
    }
    if (npart) VK_CUDA(cudaMallocAsync((void**)&P->d_part, sizeof(double) * (size_t)npart, st));
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { vk::free_mask_plan(P); return vk::cuda_check(e, "mask plan upload"); }
    *out = P;
    return VLASOV_OK;
}

int vlasov_reduce_moment_mask(const vlasov_level* const* levels, int32_t nlev, const double* const* f,
                              double* rho_finest) {
    VK_NVTX();
    if (!levels || nlev < 1 || !rho_finest || !f) return vk::fail(VLASOV_EINVAL, "null argument");
    if (nlev > vk::MAXLEV) return vk::fail(VLASOV_EUNSUPPORTED, "more than 8 levels");
    for (int l = 0; l < nlev; ++l)
        if (!levels[l] || !f[l]) return vk::fail(VLASOV_EINVAL, "reduce_moment_mask: level / field pointer required");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    const vlasov_level* Lf = levels[nlev - 1];
    if (Lf->ndim == 4) {                            // 2D+2V hierarchy: Alg.6 4D -> 2D (N3)
        bool fresh4 = Lf->mask_plan4 != nullptr && (int)Lf->mask_plan4->uids.size() == nlev;
        for (int l = 0; fresh4 && l < nlev; ++l) fresh4 = Lf->mask_plan4->uids[l] == levels[l]->uid;
        if (!fresh4) {
            vk::free_mask_plan4(Lf->mask_plan4);
            Lf->mask_plan4 = nullptr;
            vk::MaskPlan4* P = nullptr;
            if (int rc = build_mask_plan4(levels, nlev, &P)) return rc;
            Lf->mask_plan4 = P;
        }
        return vk::launch_reduce_mask4(Lf->mask_plan4, f, nlev, rho_finest, Lf->stream);
    }
    bool fresh = Lf->mask_plan != nullptr && (int)Lf->mask_plan->uids.size() == nlev;
    for (int l = 0; fresh && l < nlev; ++l) fresh = Lf->mask_plan->uids[l] == levels[l]->uid;
    if (!fresh) {
        vk::free_mask_plan(Lf->mask_plan);
        Lf->mask_plan = nullptr;
        vk::MaskPlan* P = nullptr;
        if (int rc = build_mask_plan(levels, nlev, &P)) return rc;
        Lf->mask_plan = P;
    }
    return vk::launch_reduce_mask(Lf->mask_plan, f, nlev, rho_finest, Lf->stream);
}

// 2D periodic field (N3, reading #32): exact discrete Green's functions of
//   Lambda(p, q) phi^ = 12 rho^,  Lambda = lambda(th_p) / dx^2 + lambda(th_q) / dy^2,
//   lambda(th) = 30 - 32 cos th + 2 cos 2th,  E = -(D4_x, D4_y) phi,
// in long double on the host (separable sums, O(nx ny (nx + ny))):
//   g_x(m, n) = (1/N) sum_{(p,q) != 0} S_x(p) / Lambda sin(th_p m) cos(th_q n),  S_x = (16 sin th - 2 sin 2th)/dx
//   g_y(m, n) = (1/N) sum_{(p,q) != 0} S_y(q) / Lambda cos(th_p m) sin(th_q n)
int vlasov_poisson2d_create(int32_t nx, int32_t ny, double dx, double dy, void* cuda_stream, vlasov_poisson2d** out) {
    VK_NVTX();
    if (!out) return vk::fail(VLASOV_EINVAL, "null argument");
    *out = nullptr;
    if (nx < 5 || ny < 5 || !(dx > 0) || !(dy > 0)) return vk::fail(VLASOV_EINVAL, "poisson2d: need nx, ny >= 5 and dx, dy > 0");
    if ((int64_t)nx * ny > 26000) return vk::fail(VLASOV_EUNSUPPORTED, "poisson2d: nx * ny > 26000");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    const long double PI = 3.141592653589793238462643383279502884L;
    auto lam = [](long double th) { return 30.0L - 32.0L * cosl(th) + 2.0L * cosl(2.0L * th); };
    std::vector<long double> lx(nx), ly(ny), Sx(nx), Sy(ny);
    for (int p = 0; p < nx; ++p) {
        const long double th = 2.0L * PI * p / nx;
        lx[p] = lam(th) / ((long double)dx * dx);
        Sx[p] = (16.0L * sinl(th) - 2.0L * sinl(2.0L * th)) / dx;
    }
    for (int q = 0; q < ny; ++q) {
        const long double th = 2.0L * PI * q / ny;
        ly[q] = lam(th) / ((long double)dy * dy);
        Sy[q] = (16.0L * sinl(th) - 2.0L * sinl(2.0L * th)) / dy;
    }
    auto cs = [&](int k, int n, bool s) { const long double th = 2.0L * PI * (long double)k / n; return s ? sinl(th) : cosl(th); };
    // T(p, n) = sum_q cos(th_q n) / Lambda,  U(p, n) = sum_q S_y(q) sin(th_q n) / Lambda
    std::vector<long double> T((size_t)nx * ny, 0.0L), U((size_t)nx * ny, 0.0L);
    for (int p = 0; p < nx; ++p)
        for (int q = 0; q < ny; ++q) {
            if (p == 0 && q == 0) continue;
            const long double il = 1.0L / (lx[p] + ly[q]);
            for (int n = 0; n < ny; ++n) {
                const int kq = (int)(((int64_t)q * n) % ny);
                T[(size_t)p * ny + n] += il * cs(kq, ny, false);
                U[(size_t)p * ny + n] += il * Sy[q] * cs(kq, ny, true);
            }
        }
    std::vector<double> gx((size_t)nx * ny), gy((size_t)nx * ny);
    const long double N = (long double)nx * ny;
    for (int m = 0; m < nx; ++m)
        for (int n = 0; n < ny; ++n) {
            long double ax = 0.0L, ay = 0.0L;
            for (int p = 0; p < nx; ++p) {
                const int kp = (int)(((int64_t)p * m) % nx);
                ax += Sx[p] * cs(kp, nx, true) * T[(size_t)p * ny + n];
                ay += cs(kp, nx, false) * U[(size_t)p * ny + n];
            }
            gx[(size_t)m * ny + n] = (double)(ax / N);
            gy[(size_t)m * ny + n] = (double)(ay / N);
        }
    vlasov_poisson2d* P = new vlasov_poisson2d();
    P->nx = nx; P->ny = ny; P->dx = dx; P->dy = dy;
    P->stream = (cudaStream_t)cuda_stream;
    int rc;
    if ((rc = upload(&P->d_gx, gx, P->stream)) || (rc = upload(&P->d_gy, gy, P->stream))) {
        vk::dfree(P->d_gx, P->stream);
        vk::dfree(P->d_gy, P->stream);
        delete P;
        return rc;
    }
    cudaError_t e = cudaStreamSynchronize(P->stream);
    if (e != cudaSuccess) {
        vk::dfree(P->d_gx, P->stream); vk::dfree(P->d_gy, P->stream);
        delete P;
        return vk::cuda_check(e, "poisson2d upload");
    }
    *out = P;
    return VLASOV_OK;
}

int vlasov_poisson2d_solve(const vlasov_poisson2d* P, const double* rho, double* E) {
    VK_NVTX();
    if (!P || !rho || !E) return vk::fail(VLASOV_EINVAL, "null argument");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_poisson2d(P, rho, E);
}

int vlasov_poisson2d_destroy(vlasov_poisson2d* P) {
    VK_NVTX();
    if (!P) return VLASOV_OK;
    vk::dfree(P->d_gx, P->stream);
    vk::dfree(P->d_gy, P->stream);
    delete P;
    return VLASOV_OK;
}

int vlasov_poisson_create(int32_t n, double dx, void* cuda_stream, vlasov_poisson** out) {
    VK_NVTX();
    if (!out) return vk::fail(VLASOV_EINVAL, "null argument");
    *out = nullptr;
    if (n < 5 || !(dx > 0)) return vk::fail(VLASOV_EINVAL, "poisson: need n >= 5 and dx > 0");
    if (n > 16384) return vk::fail(VLASOV_EUNSUPPORTED, "poisson: n > 16384");
    // exact discrete Green's functions of the circulant system (long double on the host):
    //   gE[d]   = (1/n) sum_m S_m sin(theta_m d),  S_m = dx (16 sin th - 2 sin 2th) / lambda_m
    //   gphi[d] = (1/n) sum_{m != 0} 12 dx^2 / lambda_m cos(theta_m d)
    //   lambda_m = 30 - 32 cos th + 2 cos 2th,  th = 2 pi m / n
    std::vector<long double> lam(n), S(n);
    const long double PI = 3.141592653589793238462643383279502884L;
    for (int m = 0; m < n; ++m) {
        const long double th = 2.0L * PI * m / n;
        lam[m] = 30.0L - 32.0L * cosl(th) + 2.0L * cosl(2.0L * th);
        S[m] = (m == 0) ? 0.0L : (long double)dx * (16.0L * sinl(th) - 2.0L * sinl(2.0L * th)) / lam[m];
    }
    std::vector<double> gE(n), gphi(n);
    std::vector<long double> c(n), s(n);
    for (int k = 0; k < n; ++k) {
        const long double th = 2.0L * PI * k / n;
        c[k] = cosl(th);
        s[k] = sinl(th);
    }
    for (int d = 0; d < n; ++d) {
        long double aE = 0.0L, aP = 0.0L;
        for (int m = 1; m < n; ++m) {
            const int k = (int)(((int64_t)m * d) % n);   // theta_m d mod 2 pi
            aE += S[m] * s[k];
            aP += (12.0L * dx * dx / lam[m]) * c[k];
        }
        gE[d] = (double)(aE / n);
        gphi[d] = (double)(aP / n);
    }
    // gE is stored periodically extended (2n + 4 values, gE[j] = g[j mod n]); gX (fused stage
    // kernel) is the same with GX_PAD / GX_TAIL values of padding, gX[m] = g[(m - GX_PAD) mod n],
    // so that the prologue reads g[(i - k) mod n] = gX[GX_PAD + n + i - k] without a modulo
    // split of gE: S_m = dx [cot(th/2)/2 + sin th / (2 (7 - cos th))], and
    // (1/n) sum_m cot(th_m/2) sin(th_m d) = 1 - 2d/n (0 < d < n), so gE(d) = (dx/2)(1 - 2d/n)[d != 0]
    // + h(d) with h(d) = (dx/n) sum_m sin th_m sin(th_m d) / (2 (7 - cos th_m)), which decays like
    // (7 - sqrt 48)^|d| = 0.0718^|d| (|h(16)| < 1e-18 max|gE|): only h(-16 .. 16) is kept
    std::vector<double> hs(33, 0.0);
    for (int m = -16; m <= 16; ++m) {
        const int d = ((m % n) + n) % n;
        long double a = 0.0L;
        for (int q = 1; q < n; ++q) {
            const int k = (int)(((int64_t)q * d) % n);
            a += s[q] * s[k] / (2.0L * (7.0L - c[q]));
        }
        hs[m + 16] = (double)((long double)dx * a / n);
    }
    std::vector<double> gX(2 * (size_t)n + vk::GX_PAD + vk::GX_TAIL);
    for (size_t m = 0; m < gX.size(); ++m) gX[m] = gE[((int64_t)m - vk::GX_PAD + 4 * (int64_t)n) % n];
    gE.resize(2 * (size_t)n + 4);
    for (size_t j = n; j < gE.size(); ++j) gE[j] = gE[j % n];
    vlasov_poisson* P = new vlasov_poisson();
    P->n = n;
    P->dx = dx;
    P->stream = (cudaStream_t)cuda_stream;
    int rc;
    P->K2 = 0.5 * dx;
    P->Kn = dx / n;
    if ((rc = upload(&P->d_gE, gE, P->stream)) || (rc = upload(&P->d_gphi, gphi, P->stream)) ||
        (rc = upload(&P->d_gX, gX, P->stream)) || (n >= 64 && (rc = upload(&P->d_hs, hs, P->stream)))) {
        vk::dfree(P->d_gE, P->stream);
        vk::dfree(P->d_gphi, P->stream);
        vk::dfree(P->d_gX, P->stream);
        delete P;
        return rc;
    }
    cudaError_t e = cudaStreamSynchronize(P->stream);
    if (e != cudaSuccess) {
        vk::dfree(P->d_gE, P->stream); vk::dfree(P->d_gphi, P->stream); vk::dfree(P->d_gX, P->stream);
        vk::dfree(P->d_hs, P->stream);
        delete P;
        return vk::cuda_check(e, "poisson upload");
    }
    *out = P;
    return VLASOV_OK;
}

int vlasov_poisson_solve(vlasov_poisson* P, const double* rho, double* phi, double* E, int32_t ghost) {
    VK_NVTX();
    if (!P || !rho) return vk::fail(VLASOV_EINVAL, "null argument");
    if (ghost < 0 || ghost > P->n) return vk::fail(VLASOV_EINVAL, "bad ghost width");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_poisson(P, rho, phi, E, ghost);
}

int vlasov_poisson_destroy(vlasov_poisson* P) {
    VK_NVTX();
    if (P) {
        vk::dfree(P->d_gE, P->stream);
        vk::dfree(P->d_gphi, P->stream);
        vk::dfree(P->d_gX, P->stream);
        vk::dfree(P->d_hs, P->stream);
        cudaStreamSynchronize(P->stream);
        delete P;
    }
    return VLASOV_OK;
}

int vlasov_inject_field(vlasov_level* L, const double* E_finest, const int32_t n_finest[2], double* E_lvl) {
    VK_NVTX();
    if (!L || !E_finest || !n_finest || !E_lvl) return vk::fail(VLASOV_EINVAL, "null argument");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    if (L->ndim == 2) return vk::launch_inject_1d(L, E_finest, n_finest[0], E_lvl);
    return vk::launch_inject_2d(L, E_finest, n_finest, E_lvl);
}

int vlasov_level_face_doubles(const vlasov_level* L, int64_t* n) {
    VK_NVTX();
    if (!L || !n) return vk::fail(VLASOV_EINVAL, "null argument");
    if (L->ndim != 4) return vk::fail(VLASOV_EUNSUPPORTED, "face_doubles: 2D+2V levels (F* form)");
    *n = L->face_doubles;
    return VLASOV_OK;
}

int vlasov_rk4_stage_fstar(vlasov_level* L, int32_t stage, double dt, const double* f_n, const double* f_s,
                           double* f_next, const double* E, int32_t recon, double* Fstar) {
    VK_NVTX();
    if (!L || !f_n || !f_s || !E || !Fstar) return vk::fail(VLASOV_EINVAL, "null argument");
    if (L->ndim != 4) return vk::fail(VLASOV_EUNSUPPORTED, "rk4_stage_fstar: 2D+2V levels");
    if (stage < 1 || stage > 4) return vk::fail(VLASOV_EINVAL, "stage must be 1..4");
    if (stage < 4 && !f_next) return vk::fail(VLASOV_EINVAL, "f_next required for stages 1..3");
    if (f_next && f_next == f_s) return vk::fail(VLASOV_EINVAL, "f_next must not alias f_s");
    if (recon != VLASOV_CENTERED4 && recon != VLASOV_UPWIND) return vk::fail(VLASOV_EINVAL, "bad recon");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_stage4_fstar(L, stage, dt, f_n, f_s, f_next, E, recon, Fstar);
}

int vlasov_fstar_coarsen(const vlasov_level* fine, const double* F_fine, const vlasov_level* coarse, double* F_coarse) {
    VK_NVTX();
    if (!fine || !F_fine || !coarse || !F_coarse) return vk::fail(VLASOV_EINVAL, "null argument");
    if (fine->ndim != 4) return vk::fail(VLASOV_EUNSUPPORTED, "fstar_coarsen: 2D+2V levels");
    if (fine->coarser != coarse || coarse->uid != fine->coarser_uid)
        return vk::fail(VLASOV_ESTALE, "fstar_coarsen: coarse level does not match the one of level_create");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_fstar_coarsen(fine, F_fine, F_coarse);
}

int vlasov_fstar_update(vlasov_level* L, double dt, const double* f_n, const double* Fstar, double* f_new) {
    VK_NVTX();
    if (!L || !f_n || !Fstar || !f_new) return vk::fail(VLASOV_EINVAL, "null argument");
    if (L->ndim != 4) return vk::fail(VLASOV_EUNSUPPORTED, "fstar_update: 2D+2V levels");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_fstar_update(L, dt, f_n, Fstar, f_new);
}

int vlasov_inject_field_ghosted(vlasov_level* L, const double* E_finest, const int32_t n_finest[2], double* E_lvl) {
    VK_NVTX();
    if (!L || !E_finest || !n_finest || !E_lvl) return vk::fail(VLASOV_EINVAL, "null argument");
    if (L->ndim != 4) return vk::fail(VLASOV_EUNSUPPORTED, "inject_field_ghosted: 2D+2V levels");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_inject_2d(L, E_finest, n_finest, E_lvl, vk::G);
}

int vlasov_inject_field_scaled(vlasov_level* L, const double* E_finest, const int32_t n_finest[2], double scale,
                               double* E_lvl) {
    VK_NVTX();
    if (!L || !E_finest || !n_finest || !E_lvl) return vk::fail(VLASOV_EINVAL, "null argument");
    if (L->ndim != 2) return vk::fail(VLASOV_EUNSUPPORTED, "inject_field_scaled: 1D+1V levels only");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_inject_1d(L, E_finest, n_finest[0], E_lvl, scale);
}

int vlasov_flux_register_accumulate(vlasov_level* fine, const double* f_fine, const double* E_fine,
                                    const double* f_coarse, const double* E_coarse, double b_s, double* regs,
                                    int32_t recon) {
    VK_NVTX();
    if (!fine || !f_fine || !E_fine || !f_coarse || !E_coarse) return vk::fail(VLASOV_EINVAL, "null argument");
    if (!fine->coarser) return vk::fail(VLASOV_EINVAL, "flux registers: level has no coarser level");
    if (fine->n_reflux > 0 && !regs) return vk::fail(VLASOV_EINVAL, "flux registers: regs required");
    if (recon != VLASOV_CENTERED4 && recon != VLASOV_UPWIND) return vk::fail(VLASOV_EINVAL, "bad recon");
    if (fine->ndim != 2) return vk::fail(VLASOV_EUNSUPPORTED, "flux registers: 1D+1V only");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_flux_registers(fine, f_fine, E_fine, f_coarse, E_coarse, b_s, regs, recon);
}

int vlasov_average_down(vlasov_level* fine, const double* f_fine, double* f_coarse, const double* regs, double dt) {
    VK_NVTX();
    if (!fine || !f_fine || !f_coarse) return vk::fail(VLASOV_EINVAL, "null argument");
    if (!fine->coarser) return vk::fail(VLASOV_EINVAL, "average_down: level has no coarser level");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    if (fine->ndim == 4) {                        // F* form: refluxing is the flux coarsening (Alg.4)
        if (regs) return vk::fail(VLASOV_EINVAL, "average_down: 2D+2V levels take no flux registers");
        return vk::launch_average_down4(fine, f_fine, f_coarse);
    }
    return vk::launch_average_down(fine, f_fine, f_coarse, regs, dt);
}

int vlasov_tag_cells(vlasov_level* L, const double* f, double tol, int32_t buffer, uint8_t* tags) {
    VK_NVTX();
    if (!L || !f || !tags) return vk::fail(VLASOV_EINVAL, "null argument");
    if (buffer < 0) return vk::fail(VLASOV_EINVAL, "tag buffer < 0");
    if (L->ndim != 2) return vk::fail(VLASOV_EUNSUPPORTED, "tag_cells: 1D+1V levels only");
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_tags(L, f, tol, buffer, tags);
}

int vlasov_level_fill_from(vlasov_level* L, double* f, const vlasov_level* old, const double* f_old,
                           const vlasov_level* coarser, const double* f_coarse, int32_t interp) {
    VK_NVTX();
    if (!L || !f) return vk::fail(VLASOV_EINVAL, "null argument");
    if (old && !f_old) return vk::fail(VLASOV_EINVAL, "fill_from: f_old required with old");
    if (L->ndim != 2) return vk::fail(VLASOV_EUNSUPPORTED, "fill_from: 1D+1V only");
    if (coarser && (coarser != L->coarser || coarser->uid != L->coarser_uid))
        return vk::fail(VLASOV_ESTALE, "fill_from: coarser level does not match the one of level_create");
    if (old) {
        if (old->ndim != L->ndim) return vk::fail(VLASOV_EINVAL, "fill_from: old level ndim mismatch");
        for (int d = 0; d < L->ndim; ++d)
            if (old->ratio[d] != L->ratio[d]) return vk::fail(VLASOV_EINVAL, "fill_from: old level resolution differs");
    }
    // copy where an old patch holds the cell (same-level data wins): one rectangle per
    // (new patch, old patch) overlap; the cells of a new patch no old patch covers interpolate
    Owner cown;
    const vlasov_level* C = L->coarser;
    if (C) cown = make_owner(C, C->blocks);
    std::vector<vk::RectCopy> rects;
    std::vector<vk::CFTask> cfs;
    std::vector<char> cover;
    int err = VLASOV_OK;
    for (size_t p = 0; p < L->boxes.size(); ++p) {
        const vk::Box& P = L->boxes[p];
        const int blk = L->patch_block[p];
        const int nx = vk::box_ncells_dim(P, 0), nv = vk::box_ncells_dim(P, 1);
        cover.assign((size_t)nx * nv, 0);
        if (old) {
            for (size_t q = 0; q < old->boxes.size(); ++q) {
                const vk::Box I = vk::box_intersect(P, old->boxes[q], L->ndim);
                if (vk::box_empty(I, L->ndim)) continue;
                const int ob = old->patch_block[q];
                vk::RectCopy r;
                r.dst = cell_addr(L, blk, I.lo);
                r.src = cell_addr(old, ob, I.lo);
                r.dpitch = (int32_t)L->block_str[blk][0];
                r.spitch = (int32_t)old->block_str[ob][0];
                r.nx = vk::box_ncells_dim(I, 0);
                r.nv = vk::box_ncells_dim(I, 1);
                rects.push_back(r);
                for (int x = I.lo[0]; x <= I.hi[0]; ++x)
                    std::fill(cover.begin() + (size_t)(x - P.lo[0]) * nv + (I.lo[1] - P.lo[1]),
                              cover.begin() + (size_t)(x - P.lo[0]) * nv + (I.hi[1] - P.lo[1]) + 1, (char)1);
            }
        }
        for (int x = 0; x < nx && !err; ++x)
            for (int v = 0; v < nv; ++v) {
                if (cover[(size_t)x * nv + v]) continue;
                const int c[4] = {P.lo[0] + x, P.lo[1] + v, 0, 0};
                if (!C || !coarser || !f_coarse) {
                    err = vk::fail(VLASOV_EINVAL, "fill_from: cell without old data needs the coarser level");
                    break;
                }
                int cc[4] = {0, 0, 0, 0};
                for (int d = 0; d < L->ndim; ++d) cc[d] = vk::floordiv(c[d], L->coarse_ratio[d]);
                const int cq = cown.find(cc);
                if (cq < 0) { err = vk::fail(VLASOV_ESTENCIL, "fill_from: coarse parent missing"); break; }
                vk::CFTask t;
                t.dst = cell_addr(L, blk, c);
                t.csrc = cell_addr(C, cq, cc);
                for (int d = 0; d < 4; ++d) {
                    t.cstride[d] = d < L->ndim ? (int32_t)C->block_str[cq][d] : 0;
                    t.sub[d] = d < L->ndim ? (int8_t)(c[d] - cc[d] * L->coarse_ratio[d]) : 0;
                }
                cfs.push_back(t);
            }
        if (err) return err;
    }
    if (!device_ok_impl()) return vk::fail(VLASOV_ECUDA, "no sm_100 CUDA device");
    return vk::launch_fill_from(L, f, f_old, rects, f_coarse, cfs, interp);
}

}  // extern "C"
