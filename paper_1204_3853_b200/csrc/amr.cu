// AMR transfers of 1D+1V levels: Alg.8 sub-patch reduction, interface flux
// registers + refluxing (Alg.4 flux substitution), average-down, tags
// (P:1423-1437).  Task lists are built on the host at level creation (level.cpp).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"
#include "scheme.cuh"

namespace vk {

// ------------------------------------------------------------------ Alg.8 sub-patch reduction
struct LevelPtrs {
    const double* f[MAXLEV];
};

// colsum[c] = sum over the sub-patch's velocity range of column c (one warp per grown column)
__global__ void k_red_cols(const LevelPtrs P, const RedCol* __restrict__ cols, int64_t ncols,
                           double* __restrict__ colsum) {
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= ncols) return;
    const RedCol C = cols[c];
    const double* p = P.f[C.level] + C.addr;
    double s = 0.0;
    for (int j = lane; j < C.nv; j += 32) s += p[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) colsum[c] = s;
}

// rho[x] = 1 - sum over the contributions of x (level, patch, sub-patch order) of
//          dv_l * sum_j b_j(s) colsum[c + j]          (linear5 refinement of the partial sums)
// One warp per finest cell x: lane l takes the contributions l, l + 32, ... of x (the loads of
// different contributions are independent, so they overlap), then a fixed butterfly
// (deterministic; the order differs from the oracle's sequential sum only by rounding).
__global__ void k_red_finest(const double* __restrict__ colsum, const RedContrib* __restrict__ con,
                             const int32_t* __restrict__ xoff, int nxf, double q, double base, int accumulate,
                             double* __restrict__ rho) {
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int x = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (x >= nxf) return;
    double acc = 0.0;
    for (int k = xoff[x] + lane; k < xoff[x + 1]; k += 32) {
        const RedContrib& C = con[k];
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < 5; ++j) t += C.b[j] * colsum[C.cs + j];
        acc += C.dv * t;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) rho[x] = (accumulate ? rho[x] : base) + q * acc;
}

// first moment of each grown sub-patch column (N4 current, reading #31): sum_j vbar_j f_j +
// (dv/24)(f_{nv} + f_{nv-1} - f_0 - f_{-1}); one warp per column, fixed butterfly
struct LevelV {
    double vlo[MAXLEV], dv[MAXLEV];
};
__global__ void k_red_cols_first(const LevelPtrs P, const LevelV V, const RedCol* __restrict__ cols, int64_t ncols,
                                 double* __restrict__ colsum) {
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= ncols) return;
    const RedCol C = cols[c];
    const double* p = P.f[C.level] + C.addr;
    const double vlo = V.vlo[C.level], dv = V.dv[C.level];
    double s = 0.0;
    for (int j = lane; j < C.nv; j += 32) s += (vlo + ((double)(C.j0 + j) + 0.5) * dv) * p[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) colsum[c] = s + (dv * (1.0 / 24.0)) * ((p[C.nv] + p[C.nv - 1]) - (p[0] + p[-1]));
}

int launch_reduce_first_subpatch(const RedPlan* P, const double* const* f, int nlev, const double* vlo,
                                 const double* dv, double* j, cudaStream_t st, double q, int accumulate) {
    LevelPtrs lp;
    LevelV lv;
    for (int l = 0; l < MAXLEV; ++l) {
        lp.f[l] = l < nlev ? f[l] : nullptr;
        lv.vlo[l] = l < nlev ? vlo[l] : 0.0;
        lv.dv[l] = l < nlev ? dv[l] : 0.0;
    }
    if (P->ncols > 0)
        VK_CUDA(launch_pdl(k_red_cols_first, dim3((unsigned)((P->ncols + 7) / 8)), dim3(256), 0, st, lp, lv,
                           (const RedCol*)P->d_cols, (int64_t)P->ncols, P->d_colsum));
    VK_CUDA(launch_pdl(k_red_finest, dim3((P->nxf + 3) / 4), dim3(128), 0, st, (const double*)P->d_colsum,
                       (const RedContrib*)P->d_contrib, (const int32_t*)P->d_xoff, P->nxf, q, 0.0, accumulate, j));
    return VLASOV_OK;
}

int launch_reduce_subpatch(const RedPlan* P, const double* const* f, int nlev, double* rho, cudaStream_t st,
                           double q, double base, int accumulate) {
    LevelPtrs lp;
    for (int l = 0; l < MAXLEV; ++l) lp.f[l] = l < nlev ? f[l] : nullptr;
    if (P->ncols > 0) {
        VK_CUDA(launch_pdl(k_red_cols, dim3((unsigned)((P->ncols + 7) / 8)), dim3(256), 0, st, lp,
                           (const RedCol*)P->d_cols, (int64_t)P->ncols, P->d_colsum));
    }
    VK_CUDA(launch_pdl(k_red_finest, dim3((P->nxf + 3) / 4), dim3(128), 0, st, (const double*)P->d_colsum,
                       (const RedContrib*)P->d_contrib, (const int32_t*)P->d_xoff, P->nxf, q, base, accumulate, rho));
    return VLASOV_OK;
}

// ------------------------------------------------------------------ Alg.6 Mask Reduction
// one warp per (patch, coarse x column): over the patch's v range, the R linear5-refined values
// of the column (from columns x_c-2 .. x_c+2), masked by mu(x_c, v), summed
__global__ void k_red_mask(const LevelPtrs P, const MaskCol* __restrict__ cols, int64_t ncols,
                           const uint8_t* __restrict__ mask, const double* __restrict__ w, double* __restrict__ part) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= ncols) return;
    const MaskCol C = cols[c];
    const double* f = P.f[C.level] + C.addr;
    const double* b = w + C.woff;
    double acc[MAXR];
#pragma unroll
    for (int s = 0; s < MAXR; ++s) acc[s] = 0.0;
    for (int j = lane; j < C.nv; j += 32) {
        if (!mask[C.mask + j]) continue;
        double u[5];
#pragma unroll
        for (int a = 0; a < 5; ++a) u[a] = f[(int64_t)a * C.pitch + j];
#pragma unroll
        for (int s = 0; s < MAXR; ++s) {
            if (s >= C.R) break;
            double v = 0.0;
#pragma unroll
            for (int a = 0; a < 5; ++a) v += b[5 * s + a] * u[a];
            acc[s] += v;
        }
    }
#pragma unroll
    for (int s = 0; s < MAXR; ++s) {
        if (s >= C.R) break;
        double v = acc[s];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) part[C.out + s] = v;
    }
}

__global__ void k_red_mask_finest(const double* __restrict__ part, const int32_t* __restrict__ xoff,
                                  const int32_t* __restrict__ idx, const double* __restrict__ dv, int nxf,
                                  double* __restrict__ rho) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= nxf) return;
    double acc = 0.0;
    for (int k = xoff[x]; k < xoff[x + 1]; ++k) acc += dv[k] * part[idx[k]];
    rho[x] = 1.0 - acc;
}

int launch_reduce_mask(const MaskPlan* P, const double* const* f, int nlev, double* rho, cudaStream_t st) {
    LevelPtrs lp;
    for (int l = 0; l < MAXLEV; ++l) lp.f[l] = l < nlev ? f[l] : nullptr;
    if (P->ncols > 0) {
        k_red_mask<<<(unsigned)((P->ncols + 7) / 8), 256, 0, st>>>(lp, P->d_cols, P->ncols, P->d_mask, P->d_w,
                                                                   P->d_part);
        VK_LAUNCH("k_red_mask");
    }
    k_red_mask_finest<<<(P->nxf + 127) / 128, 128, 0, st>>>(P->d_part, P->d_xoff, P->d_idx, P->d_dv, P->nxf, rho);
    VK_LAUNCH("k_red_mask_finest");
    return VLASOV_OK;
}

// ------------------------------------------------------------------ face fluxes at one face
// x-face flux F^x_{i+1/2,j} = vbar_j <f> + (dv/24)(<f>_{j+1} - <f>_{j-1})
template <int RECON>
__device__ double xface_flux(const double* f, const FaceRef& r, double v_lo, double dv) {
    double fa[3];
#pragma unroll
    for (int t = -1; t <= 1; ++t) {
        const double* p = f + r.s0 + t;
        const double vb = v_lo + ((double)(r.g + t) + 0.5) * dv;
        fa[t + 1] = face_avg<RECON>(p[0], p[r.pitch], p[2 * (int64_t)r.pitch], p[3 * (int64_t)r.pitch], vb);
    }
    const double vb0 = v_lo + ((double)r.g + 0.5) * dv;
    return vb0 * fa[1] + (dv * (1.0 / 24.0)) * (fa[2] - fa[0]);
}

// v-face flux F^E_{i,j+1/2} = E_i <f> + (1/48)(E_{i+1} - E_{i-1})(<f>_{i+1} - <f>_{i-1})
// (+1/48 reading #3); speed on each face a = -E of its column
template <int RECON>
__device__ double vface_flux(const double* f, const FaceRef& r, const double* E) {
    double fa[3];
#pragma unroll
    for (int t = -1; t <= 1; ++t) {
        const double* p = f + r.s0 + (int64_t)t * r.pitch;
        fa[t + 1] = face_avg<RECON>(p[0], p[1], p[2], p[3], -E[r.g + t]);
    }
    const double c48 = (E[r.g + 1] - E[r.g - 1]) * (1.0 / 48.0);
    return E[r.g] * fa[1] + c48 * (fa[2] - fa[0]);
}

// regs[t] += b_s (F_coarse - mean of the fine F) on every coarse face of the interface.
// FR_G = 8 lanes per task: lane g computes the fine faces g, g + 8, ... (their loads overlap),
// lane 0 also the coarse face; a fixed butterfly sums the fine fluxes (deterministic).
constexpr int FR_G = 8;
template <int RECON>
__global__ void k_flux_registers(const RefluxTask* __restrict__ tasks, int64_t n, const double* __restrict__ ff,
                                 const double* __restrict__ Ef, const double* __restrict__ fc,
                                 const double* __restrict__ Ec, double vlo, double dvf, double dvc, double b_s,
                                 double* __restrict__ regs) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t t = gt / FR_G;
    const int g = (int)(gt % FR_G);
    const bool valid = t < n;
    const RefluxTask& T = tasks[valid ? t : 0];
    double Fs = 0.0, Fc = 0.0;
    if (valid) {
        for (int s = g; s < T.nfine; s += FR_G)
            Fs += (T.dir == 0) ? xface_flux<RECON>(ff, T.ff[s], vlo, dvf) : vface_flux<RECON>(ff, T.ff[s], Ef);
        if (g == 0) Fc = (T.dir == 0) ? xface_flux<RECON>(fc, T.cf, vlo, dvc) : vface_flux<RECON>(fc, T.cf, Ec);
    }
#pragma unroll
    for (int o = FR_G / 2; o > 0; o >>= 1) Fs += __shfl_xor_sync(0xffffffffu, Fs, o);
    if (valid && g == 0) regs[t] += b_s * (Fc - Fs / (double)T.nfine);
}

int launch_flux_registers(const vlasov_level* L, const double* f_fine, const double* E_fine, const double* f_coarse,
                          const double* E_coarse, double b_s, double* regs, int recon) {
    if (L->n_reflux == 0) return VLASOV_OK;
    const vlasov_level* C = L->coarser;
    const unsigned blocks = (unsigned)((L->n_reflux * FR_G + 127) / 128);
    auto kern = recon == VLASOV_UPWIND ? k_flux_registers<VLASOV_UPWIND> : k_flux_registers<VLASOV_CENTERED4>;
    VK_CUDA(launch_pdl(kern, dim3(blocks), dim3(128), 0, L->stream, (const RefluxTask*)L->d_reflux, (int64_t)L->n_reflux,
                       f_fine, E_fine, f_coarse, E_coarse, L->lower[1], L->h[1], C->h[1], b_s, regs));
    return VLASOV_OK;
}

// ------------------------------------------------------------------ refluxing + average-down
// Coarse cell next to the interface: f += dt * dk, where dk replaces the coarse face flux by the
// mean fine one in k = -(Fx_hi - Fx_lo)/dx + (Fv_hi - Fv_lo)/dv and regs = F*_c - <F*_f>:
//   x high face: +dt reg/dx, x low face: -dt reg/dx, v high face: -dt reg/dv, v low: +dt reg/dv.
__global__ void k_reflux(const RefluxTask* __restrict__ tasks, const int64_t* __restrict__ cells,
                         const int32_t* __restrict__ off, int64_t ncells, const double* __restrict__ regs,
                         double dt, double dxc, double dvc, double* __restrict__ fc) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    double d = 0.0;
    for (int k = off[c]; k < off[c + 1]; ++k) {
        const RefluxTask& T = tasks[k];
        const double r = regs[k];
        if (T.dir == 0) d += (T.sign > 0 ? r : -r) / dxc;
        else d += (T.sign > 0 ? -r : r) / dvc;
    }
    fc[cells[c]] += dt * d;
}

__global__ void k_average_down(const AvgTask* __restrict__ tasks, int64_t n, int Rx, int Rv,
                               const double* __restrict__ ff, double* __restrict__ fc) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const AvgTask T = tasks[t];
    double s = 0.0;
    for (int a = 0; a < Rx; ++a)
        for (int b = 0; b < Rv; ++b) s += ff[T.fcell0 + (int64_t)a * T.fpitch + b];
    fc[T.ccell] = s / (double)(Rx * Rv);
}

int launch_average_down(const vlasov_level* L, const double* f_fine, double* f_coarse, const double* regs, double dt) {
    const vlasov_level* C = L->coarser;
    if (regs && L->n_reflux_cells > 0) {
        VK_CUDA(launch_pdl(k_reflux, dim3((unsigned)((L->n_reflux_cells + 127) / 128)), dim3(128), 0, L->stream,
                           (const RefluxTask*)L->d_reflux, (const int64_t*)L->d_reflux_cells,
                           (const int32_t*)L->d_reflux_off, (int64_t)L->n_reflux_cells, regs, dt, C->h[0], C->h[1],
                           f_coarse));
    }
    if (L->n_avg > 0) {
        VK_CUDA(launch_pdl(k_average_down, dim3((unsigned)((L->n_avg + 127) / 128)), dim3(128), 0, L->stream,
                           (const AvgTask*)L->d_avg, (int64_t)L->n_avg, L->coarse_ratio[0], L->coarse_ratio[1], f_fine,
                           f_coarse));
    }
    return VLASOV_OK;
}

// ------------------------------------------------------------------ tags (reading #18)
// crit = sqrt(0.5 (hx (f_{i+1}-f_{i-1})^2 + hv (f_{j+1}-f_{j-1})^2))
//      + 0.5 (hx^2 |f_{i+1} - 2f + f_{i-1}| + hv^2 |f_{j+1} - 2f + f_{j-1}|),  evaluated in this
// order with round-to-nearest intrinsics (no FMA contraction), as the oracle does.
__device__ __forceinline__ bool crit_exceeds(const double* f, int64_t c, int64_t pitch, double hx, double hv,
                                             double tol) {
    const double f0 = f[c], xp = f[c + pitch], xm = f[c - pitch], vp = f[c + 1], vm = f[c - 1];
    const double dx1 = __dsub_rn(xp, xm), dv1 = __dsub_rn(vp, vm);
    const double d1 = __dsqrt_rn(__dmul_rn(0.5, __dadd_rn(__dmul_rn(hx, __dmul_rn(dx1, dx1)),
                                                          __dmul_rn(hv, __dmul_rn(dv1, dv1)))));
    const double sx = __dadd_rn(__dsub_rn(xp, __dmul_rn(2.0, f0)), xm);
    const double sv = __dadd_rn(__dsub_rn(vp, __dmul_rn(2.0, f0)), vm);
    const double d2 = __dmul_rn(0.5, __dadd_rn(__dmul_rn(__dmul_rn(hx, hx), fabs(sx)),
                                               __dmul_rn(__dmul_rn(hv, hv), fabs(sv))));
    return __dadd_rn(d1, d2) > tol;
}

// tags[x * nv + j] = any crit > tol within the Chebyshev `buffer` (periodic in x, clipped in v)
__global__ void k_tags(const double* __restrict__ f, int64_t off, int64_t pitch, int nx, int nv, double hx,
                       double hv, double tol, int buffer, uint8_t* __restrict__ tags) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)nx * nv) return;
    const int x = (int)(t / nv), j = (int)(t % nv);
    uint8_t hit = 0;
    for (int a = -buffer; a <= buffer && !hit; ++a) {
        int xx = x + a;
        xx = (xx % nx + nx) % nx;
        for (int b = -buffer; b <= buffer; ++b) {
            const int jj = j + b;
            if (jj < 0 || jj >= nv) continue;
            if (crit_exceeds(f, off + (int64_t)(xx + G) * pitch + (jj + G), pitch, hx, hv, tol)) { hit = 1; break; }
        }
    }
    tags[t] = hit;
}

// Multi-patch levels: raw tags per block interior (the crit of a cell uses its block's ghost
// frame), into a level-domain scratch that is zero off the patches; then the dilation.
__global__ void k_tags_raw(const double* __restrict__ f, const Block1* __restrict__ blocks, int maxcells, int nv,
                           double hx, double hv, double tol, uint8_t* __restrict__ raw) {
    const Block1 B = blocks[blockIdx.y];
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= B.nx * B.nv || t >= maxcells) return;
    const int i = t / B.nv, j = t % B.nv;
    const int64_t c = B.off + (int64_t)(i + G) * B.pitch + (j + G);
    raw[(int64_t)(B.lo_x + i) * nv + (B.lo_v + j)] = crit_exceeds(f, c, B.pitch, hx, hv, tol) ? 1 : 0;
}

__global__ void k_tags_dilate(const uint8_t* __restrict__ raw, int nx, int nv, int buffer, uint8_t* __restrict__ tags) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)nx * nv) return;
    const int x = (int)(t / nv), j = (int)(t % nv);
    uint8_t hit = 0;
    for (int a = -buffer; a <= buffer && !hit; ++a) {
        const int xx = ((x + a) % nx + nx) % nx;
        for (int b = -buffer; b <= buffer; ++b) {
            const int jj = j + b;
            if (jj < 0 || jj >= nv) continue;
            if (raw[(int64_t)xx * nv + jj]) { hit = 1; break; }
        }
    }
    tags[t] = hit;
}

int launch_tags(const vlasov_level* L, const double* f, double tol, int buffer, uint8_t* tags) {
    const int nx = L->dom[0], nv = L->dom[1];
    const int64_t n = (int64_t)nx * nv;
    if (L->single_block) {                               // fused: crit + dilation in one pass
        k_tags<<<(unsigned)((n + 255) / 256), 256, 0, L->stream>>>(f, L->block_off[0], L->block_str[0][0], nx, nv,
                                                                   L->h[0], L->h[1], tol, buffer, tags);
        VK_LAUNCH("k_tags");
        return VLASOV_OK;
    }
    VK_CUDA(cudaMemsetAsync(L->d_rawtags, 0, (size_t)n, L->stream));
    int maxcells = 0;
    for (const Block1& B : L->h_blocks1) maxcells = std::max(maxcells, B.nx * B.nv);
    const dim3 grid((unsigned)((maxcells + 255) / 256), (unsigned)L->h_blocks1.size());
    k_tags_raw<<<grid, 256, 0, L->stream>>>(f, L->d_blocks1, maxcells, nv, L->h[0], L->h[1], tol, L->d_rawtags);
    VK_LAUNCH("k_tags_raw");
    k_tags_dilate<<<(unsigned)((n + 255) / 256), 256, 0, L->stream>>>(L->d_rawtags, nx, nv, buffer, tags);
    VK_LAUNCH("k_tags_dilate");
    return VLASOV_OK;
}

}  // namespace vk
