// 2D+2V hierarchies (NEXT row N3): ghost fill of multi-patch 4D levels and the two 4D -> 2D
// reductions of the paper's Section 4.
//
// PAPER.md: ghost fill Alg.2 (reading #15: siblings / periodic images, then CF, then
// the physical velocity condition), conservative interpolation dimension by dimension x, y, v_x,
// v_y with linear5 (reading #12) or WENO5 (readings #8-#10),
// characteristic condition along v_x over the whole ghosted extent, then along v_y (P:227-231,
// reading #6); Alg.8 Sub-Patch Reduction and Alg.6 Mask Reduction
// with N = M = 2, each level weighted by its own dvx dvy (reading #13).
// Task lists and plans are built on the host (level.cpp) from the same box calculus as the
// oracle; the kernels are flat one-thread-per-value / one-warp-per-sum loops (these levels are
// a few MiB: latency-bound, L2-resident).
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace vk {

// 1D conservative interpolation (u[0..4] = u_{i-2..i+2}); same formulas as transfer.cu
__device__ __forceinline__ double lin5(const double* u, const double* b) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 5; ++j) acc += b[j] * u[j];
    return acc;
}

__device__ double weno5_sub(const double* u, int R, int s) {
    const double um2 = u[0], um1 = u[1], u0 = u[2], up1 = u[3], up2 = u[4];
    const double Dm2 = um1 - um2, Dm1 = u0 - um1, D0 = up1 - u0, Dp1 = up2 - up1;
    const double Lm1 = Dm1 - Dm2, L0 = D0 - Dm1, Lp1 = Dp1 - D0;
    const double b0 = (13.0 / 12.0) * Lp1 * Lp1 + 0.25 * (Dp1 - 3.0 * D0) * (Dp1 - 3.0 * D0);
    const double b1 = (13.0 / 12.0) * L0 * L0 + 0.25 * (D0 + Dm1) * (D0 + Dm1);
    const double b2 = (13.0 / 12.0) * Lm1 * Lm1 + 0.25 * (3.0 * Dm1 - Dm2) * (3.0 * Dm1 - Dm2);
    const double a0 = 0.3 / ((1e-6 + b0) * (1e-6 + b0));
    const double a1 = 0.6 / ((1e-6 + b1) * (1e-6 + b1));
    const double a2 = 0.1 / ((1e-6 + b2) * (1e-6 + b2));
    const double asum = a0 + a1 + a2;
    const double w0 = a0 / asum, w1 = a1 / asum, w2 = a2 / asum;
    const double A0 = u0 + (2.0 * Dp1 - 5.0 * D0) / 6.0;
    const double A1 = u0 - (D0 + 2.0 * Dm1) / 6.0;
    const double A2 = u0 - (4.0 * Dm1 - Dm2) / 6.0;
    const double B0 = 2.0 * D0 - Dp1, B1 = Dm1, B2 = Dm1;                              // reading #8
    const double C0 = Lp1, C1 = L0, C2 = Lm1;
    double mine = 0.0, sum = 0.0;
    for (int q = 0; q < R; ++q) {
        const double bs = (2.0 * q + 1.0) / (2.0 * R);
        const double cs = (3.0 * q * q + 3.0 * q + 1.0) / (6.0 * R * R);
        const double v = w0 * (A0 + B0 * bs + C0 * cs) + w1 * (A1 + B1 * bs + C1 * cs) + w2 * (A2 + B2 * bs + C2 * cs);
        sum += v;
        if (q == s) mine = v;
    }
    return mine + (u0 - sum / R);                                                      // reading #10
}

template <int INTERP>
__device__ __forceinline__ double interp1d(const double* u, const double* b5, int R, int s) {
    return INTERP == VLASOV_WENO5 ? weno5_sub(u, R, s) : lin5(u, b5 + 5 * s);
}

// siblings / periodic images (copy pairs) and coarse-fine values: the fine value of sub-cell
// (s_x, s_y, s_vx, s_vy) of the coarse parent from its 5^4 coarse block, one dimension at a time
// (x on the 125 columns, then y on 25, v_x on 5, v_y) -- the oracle's refine_patch_4d per cell
template <int INTERP>
__global__ void k_fill_copy_cf4(double* __restrict__ f, const int64_t* __restrict__ copies, int64_t ncopy,
                                const double* __restrict__ fc, const CFTask* __restrict__ cf, int64_t ncf,
                                const double* __restrict__ b5, int4 R) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < ncopy) {
        f[copies[2 * t]] = f[copies[2 * t + 1]];
        return;
    }
    const int64_t c = t - ncopy;
    if (c >= ncf) return;
    const CFTask T = cf[c];
    const double* bx = b5;
    const double* by = b5 + 5 * MAXR;
    const double* bvx = b5 + 10 * MAXR;
    const double* bvy = b5 + 15 * MAXR;
    double p3[5];
    for (int d = 0; d < 5; ++d) {                 // v_y column d
        double p2[5];
        for (int cc = 0; cc < 5; ++cc) {          // v_x column cc
            double p1[5];
            for (int b = 0; b < 5; ++b) {         // y column b
                double col[5];
#pragma unroll
                for (int a = 0; a < 5; ++a)
                    col[a] = fc[T.csrc + (int64_t)(a - 2) * T.cstride[0] + (int64_t)(b - 2) * T.cstride[1] +
                                (int64_t)(cc - 2) * T.cstride[2] + (d - 2)];
                p1[b] = interp1d<INTERP>(col, bx, R.x, T.sub[0]);
            }
            p2[cc] = interp1d<INTERP>(p1, by, R.y, T.sub[1]);
        }
        p3[d] = interp1d<INTERP>(p2, bvx, R.z, T.sub[2]);
    }
    f[T.dst] = interp1d<INTERP>(p3, bvy, R.w, T.sub[3]);
}

// characteristic velocity condition of one column side: outgoing (a = -E_d points out) ->
// cubic extrapolation of the 4 boundary cells, else the unperturbed profile (reading #6)
__global__ void k_fill_phys4(double* __restrict__ f, const PhysTask4* __restrict__ tasks, int64_t n,
                             const double* __restrict__ E_bc, const double* __restrict__ f0v) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const PhysTask4 T = tasks[t];
    const double a = -E_bc[T.e_idx];
    const int64_t st = T.side == 0 ? T.stride : -(int64_t)T.stride;        // inward step
    const double f0 = f[T.cell0], f1 = f[T.cell0 + st], f2 = f[T.cell0 + 2 * st], f3 = f[T.cell0 + 3 * st];
    const bool out = T.side == 0 ? (a < 0.0) : (a > 0.0);
    double g1, g2;
    if (out) {
        g1 = 4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3;
        g2 = 10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3;
    } else {
        g1 = f0v[T.p_idx];
        g2 = f0v[T.p_idx + (T.side == 0 ? -T.pstep : T.pstep)];
    }
    f[T.cell0 - st] = g1;
    f[T.cell0 - 2 * st] = g2;
}

int launch_fill4(vlasov_level* L, double* f, const double* f_coarse, const double* E_bc, const double* f0v,
                 int interp) {
    const int64_t n1 = L->n_copy + L->n_cf;
    if (L->n_cf > 0 && f_coarse == nullptr) return fail(VLASOV_EINVAL, "fill_ghosts: coarse data required");
    if (n1 > 0) {
        const int4 R = make_int4(L->coarse_ratio[0], L->coarse_ratio[1], L->coarse_ratio[2], L->coarse_ratio[3]);
        auto kern = interp == VLASOV_WENO5 ? k_fill_copy_cf4<VLASOV_WENO5> : k_fill_copy_cf4<VLASOV_LINEAR5>;
        VK_CUDA(launch_pdl(kern, dim3((unsigned)((n1 + 127) / 128)), dim3(128), 0, L->stream, f,
                           (const int64_t*)L->d_copy, (int64_t)L->n_copy, f_coarse, (const CFTask*)L->d_cf,
                           (int64_t)L->n_cf, (const double*)L->d_b5, R));
    }
    if (L->n_phys4[0] + L->n_phys4[1] > 0) {
        if (E_bc == nullptr || f0v == nullptr) return fail(VLASOV_EINVAL, "fill_ghosts: E_bc and f0v required");
        for (int pass = 0; pass < 2; ++pass) {                              // v_x, then v_y
            const int64_t n = L->n_phys4[pass], first = pass ? L->n_phys4[0] : 0;
            if (n == 0) continue;
            VK_CUDA(launch_pdl(k_fill_phys4, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, L->stream, f,
                               (const PhysTask4*)(L->d_phys4 + first), n, E_bc, f0v));
        }
    }
    return VLASOV_OK;
}

// ------------------------------------------------------------------ Alg.8, 4D -> 2D
struct LevelPtrs4 {
    const double* f[MAXLEV];
};

// colsum[c] = sum over the sub-patch's (v_x, v_y) rectangle of grown column c (one warp each)
__global__ void k_red4_cols(const LevelPtrs4 P, const Red4Col* __restrict__ cols, int64_t ncols,
                            double* __restrict__ colsum) {
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= ncols) return;
    const Red4Col C = cols[c];
    const double* p = P.f[C.level] + C.addr;
    double s = 0.0;
    for (int j = 0; j < C.nvx; ++j)
        for (int m = lane; m < C.nvy; m += 32) s += p[(int64_t)j * C.s2 + m];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) colsum[c] = s;
}

// rho(x, y) = base + q sum_contributions dvv sum_b by[b] sum_a bx[a] colsum[cs + a ystride + b]
// (x pass first, then y, as the oracle); one warp per finest cell, lanes over contributions
__global__ void k_red4_finest(const double* __restrict__ colsum, const Red4Contrib* __restrict__ con,
                              const int32_t* __restrict__ off, int ncell, double q, double base,
                              double* __restrict__ rho) {
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int x = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (x >= ncell) return;
    double acc = 0.0;
    for (int k = off[x] + lane; k < off[x + 1]; k += 32) {
        const Red4Contrib& C = con[k];
        double t = 0.0;
#pragma unroll
        for (int b = 0; b < 5; ++b) {
            double tx = 0.0;
#pragma unroll
            for (int a = 0; a < 5; ++a) tx += C.bx[a] * colsum[C.cs + (int64_t)a * C.ystride + b];
            t += C.by[b] * tx;
        }
        acc += C.dvv * t;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) rho[x] = base + q * acc;
}

int launch_reduce_subpatch4(const RedPlan4* P, const double* const* f, int nlev, double* rho, cudaStream_t st) {
    LevelPtrs4 lp;
    for (int l = 0; l < MAXLEV; ++l) lp.f[l] = l < nlev ? f[l] : nullptr;
    if (P->ncols > 0)
        VK_CUDA(launch_pdl(k_red4_cols, dim3((unsigned)((P->ncols + 7) / 8)), dim3(256), 0, st, lp,
                           (const Red4Col*)P->d_cols, (int64_t)P->ncols, P->d_colsum));
    const int ncell = P->nxf * P->nyf;
    VK_CUDA(launch_pdl(k_red4_finest, dim3((ncell + 3) / 4), dim3(128), 0, st, (const double*)P->d_colsum,
                       (const Red4Contrib*)P->d_contrib, (const int32_t*)P->d_off, ncell, -1.0, 1.0, rho));
    return VLASOV_OK;
}

// ------------------------------------------------------------------ Alg.6, 4D -> 2D
// one warp per item (patch, finest (x, y)): over the patch's (v_x, v_y) cells the linear5-refined
// value of the 5x5 (x, y) block (x pass first), masked by mu of the coarse cell, summed
__global__ void k_red4_mask(const LevelPtrs4 P, const Mask4Item* __restrict__ items, int64_t n,
                            const uint8_t* __restrict__ mask, const double* __restrict__ w,
                            double* __restrict__ part) {
    griddep_wait();
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t it = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (it >= n) return;
    const Mask4Item I = items[it];
    const double* p = P.f[I.level] + I.addr;
    const double* bx = w + I.wx;
    const double* by = w + I.wy;
    double s = 0.0;
    const int nv = I.nvx * I.nvy;
    for (int t = lane; t < nv; t += 32) {
        const int j = t / I.nvy, m = t - j * I.nvy;
        if (!mask[I.mask + t]) continue;
        const double* q = p + (int64_t)j * I.s2 + m;
        double v = 0.0;
#pragma unroll
        for (int b = 0; b < 5; ++b) {
            double tx = 0.0;
#pragma unroll
            for (int a = 0; a < 5; ++a) tx += bx[a] * q[(int64_t)a * I.s0 + (int64_t)b * I.s1];
            v += by[b] * tx;
        }
        s += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) part[it] = s;
}

__global__ void k_red4_mask_finest(const double* __restrict__ part, const double* __restrict__ dvv,
                                   const int32_t* __restrict__ off, const int32_t* __restrict__ idx, int ncell,
                                   double* __restrict__ rho) {
    griddep_wait();
    griddep_launch_dependents();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    double acc = 0.0;
    for (int k = off[c]; k < off[c + 1]; ++k) acc += dvv[k] * part[idx[k]];
    rho[c] = 1.0 - acc;
}

int launch_reduce_mask4(const MaskPlan4* P, const double* const* f, int nlev, double* rho, cudaStream_t st) {
    LevelPtrs4 lp;
    for (int l = 0; l < MAXLEV; ++l) lp.f[l] = l < nlev ? f[l] : nullptr;
    if (P->nitems > 0)
        VK_CUDA(launch_pdl(k_red4_mask, dim3((unsigned)((P->nitems + 7) / 8)), dim3(256), 0, st, lp,
                           (const Mask4Item*)P->d_items, (int64_t)P->nitems, (const uint8_t*)P->d_mask,
                           (const double*)P->d_w, P->d_part));
    const int ncell = P->nxf * P->nyf;
    VK_CUDA(launch_pdl(k_red4_mask_finest, dim3((ncell + 127) / 128), dim3(128), 0, st, (const double*)P->d_part,
                       (const double*)P->d_dvv, (const int32_t*)P->d_off, (const int32_t*)P->d_idx, ncell, rho));
    return VLASOV_OK;
}

void free_red_plan4(RedPlan4* p) {
    if (!p) return;
    dfree(p->d_cols, p->st);
    dfree(p->d_colsum, p->st);
    dfree(p->d_contrib, p->st);
    dfree(p->d_off, p->st);
    delete p;
}

void free_mask_plan4(MaskPlan4* p) {
    if (!p) return;
    dfree(p->d_items, p->st);
    dfree(p->d_mask, p->st);
    dfree(p->d_w, p->st);
    dfree(p->d_part, p->st);
    dfree(p->d_dvv, p->st);
    dfree(p->d_off, p->st);
    dfree(p->d_idx, p->st);
    delete p;
}

}  // namespace vk
