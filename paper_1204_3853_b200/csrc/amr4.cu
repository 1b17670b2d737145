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
#include "scheme.cuh"

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

namespace vk {

// ------------------------------------------------------------------ RK4 in the F* form (4D AMR)
// One stage of Alg.3 on every patch of a 2D+2V level from the ghosted predictor state
// f_s: the face fluxes of P:263-282 generalised dimension by dimension (one transverse term on
// configuration faces, one (1/48) product term per configuration dim on velocity faces, +1/48 by
// reading #3), F* += b_s F on every face (the paper's flux accumulation), and the next
// predictor f_{s+1} = f_n + alpha_{s+1} dt k(f_s) (Alg.2).  One thread per cell; every
// cell computes its low and high faces (a face is computed by both neighbours; these levels are
// small and latency-bound).  The level update (vlasov_fstar_update), Alg.4's flux coarsening
// (vlasov_fstar_coarsen) and average-down complete the step.

template <int RECON>
__device__ __forceinline__ double fval(const double* __restrict__ f, int64_t c, int64_t st, double upw) {
    // face between c and c + st from the cells c - st .. c + 2 st
    return face_avg<RECON>(f[c - st], f[c], f[c + st], f[c + 2 * st], upw);
}

struct Stage4Args {
    const Patch4* patches;
    int npatch;
    const double* f_s;
    const double* f_n;
    double* f_next;            // nullable (stage 4)
    const double* E;           // [2][(nx+4)(ny+4)] ghosted level field
    double* Fstar;
    double dt, b_s, alpha_next;
    double h[4];
    double vlo[2];             // lower velocity corner of the level domain
    int nx, ny;                // level (x, y) domain, for the E array
};

template <int STAGE, int RECON>
__global__ void k_stage4_fstar(const Stage4Args A) {
    griddep_wait();
    griddep_launch_dependents();
    const Patch4 P = A.patches[blockIdx.y];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ncell = (int64_t)P.n[0] * P.n[1] * P.n[2] * P.n[3];
    if (t >= ncell) return;
    int q[4];
    int64_t r = t;
    q[3] = (int)(r % P.n[3]); r /= P.n[3];
    q[2] = (int)(r % P.n[2]); r /= P.n[2];
    q[1] = (int)(r % P.n[1]); r /= P.n[1];
    q[0] = (int)r;
    const int64_t s[4] = {P.s[0], P.s[1], P.s[2], 1};
    const int64_t c = P.org + q[0] * s[0] + q[1] * s[1] + q[2] * s[2] + q[3];
    const double* f = A.f_s;
    const int gx = P.lo[0] + q[0], gy = P.lo[1] + q[1], gl = P.lo[2] + q[2], gm = P.lo[3] + q[3];
    const int nyg = A.ny + 4;
    const int64_t ec = (int64_t)(A.nx + 4) * nyg;
    auto Eat = [&](int comp, int di, int dk) { return A.E[comp * ec + (int64_t)(gx + di + 2) * nyg + (gy + dk + 2)]; };
    auto vb = [&](int d, int j) { return A.vlo[d] + ((double)j + 0.5) * A.h[2 + d]; };
    double F[4][2];
    // configuration faces: x (d = 0, transverse along v_x), y (d = 1, transverse along v_y)
    for (int d = 0; d < 2; ++d) {
        const int vd = 2 + d;
        const double v = vb(d, d == 0 ? gl : gm);
        for (int side = 0; side < 2; ++side) {
            const int64_t cf = c + (side == 0 ? -s[d] : 0);                 // face between cf and cf + s[d]
            const double fm = fval<RECON>(f, cf, s[d], v);
            const double fl = fval<RECON>(f, cf - s[vd], s[d], v - A.h[vd]);
            const double fh = fval<RECON>(f, cf + s[vd], s[d], v + A.h[vd]);
            F[d][side] = v * fm + (A.h[vd] / 24.0) * (fh - fl);
        }
    }
    // velocity faces: v_x (d = 2, field E_x), v_y (d = 3, field E_y); product terms along x and y
    for (int d = 2; d < 4; ++d) {
        const int comp = d - 2;
        const double e = Eat(comp, 0, 0);
        const double cx = (1.0 / 48.0) * (Eat(comp, 1, 0) - Eat(comp, -1, 0));
        const double cy = (1.0 / 48.0) * (Eat(comp, 0, 1) - Eat(comp, 0, -1));
        for (int side = 0; side < 2; ++side) {
            const int64_t cf = c + (side == 0 ? -s[d] : 0);
            const double fm = fval<RECON>(f, cf, s[d], -e);
            const double fxm = fval<RECON>(f, cf - s[0], s[d], -Eat(comp, -1, 0));
            const double fxp = fval<RECON>(f, cf + s[0], s[d], -Eat(comp, 1, 0));
            const double fym = fval<RECON>(f, cf - s[1], s[d], -Eat(comp, 0, -1));
            const double fyp = fval<RECON>(f, cf + s[1], s[d], -Eat(comp, 0, 1));
            F[d][side] = e * fm + cx * (fxp - fxm) + cy * (fyp - fym);
        }
    }
    double k = -(F[0][1] - F[0][0]) / A.h[0];
    k = k + (-(F[1][1] - F[1][0]) / A.h[1]);
    k = k + (F[2][1] - F[2][0]) / A.h[2];
    k = k + (F[3][1] - F[3][0]) / A.h[3];
    // F* on the faces this cell owns: its low faces, and its high faces at the patch top
    for (int d = 0; d < 4; ++d) {
        int nf[4] = {P.n[0], P.n[1], P.n[2], P.n[3]};
        nf[d] += 1;
        int64_t idx = 0;
        for (int e = 0; e < 4; ++e) idx = idx * nf[e] + q[e];              // low face of the cell
        double* Fd = A.Fstar + P.foff[d];
        int64_t sd = 1;
        for (int e = 3; e > d; --e) sd *= nf[e];                           // stride of dim d in the face array
        if (STAGE == 1) Fd[idx] = A.b_s * F[d][0];
        else Fd[idx] += A.b_s * F[d][0];
        if (q[d] == P.n[d] - 1) {
            if (STAGE == 1) Fd[idx + sd] = A.b_s * F[d][1];
            else Fd[idx + sd] += A.b_s * F[d][1];
        }
    }
    if (STAGE < 4) A.f_next[c] = A.f_n[c] + A.alpha_next * A.dt * k;
}

// f_new = f_n + dt div(F*) on every cell of the level (Alg.4 ComputeUpdate)
__global__ void k_fstar_update(const Patch4* __restrict__ patches, const double* __restrict__ f_n,
                               const double* __restrict__ Fstar, double4 h, double dt, double* __restrict__ f_new) {
    griddep_wait();
    griddep_launch_dependents();
    const Patch4 P = patches[blockIdx.y];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ncell = (int64_t)P.n[0] * P.n[1] * P.n[2] * P.n[3];
    if (t >= ncell) return;
    int q[4];
    int64_t r = t;
    q[3] = (int)(r % P.n[3]); r /= P.n[3];
    q[2] = (int)(r % P.n[2]); r /= P.n[2];
    q[1] = (int)(r % P.n[1]); r /= P.n[1];
    q[0] = (int)r;
    const double hh[4] = {h.x, h.y, h.z, h.w};
    double k = 0.0;
    for (int d = 0; d < 4; ++d) {
        int nf[4] = {P.n[0], P.n[1], P.n[2], P.n[3]};
        nf[d] += 1;
        int64_t idx = 0;
        for (int e = 0; e < 4; ++e) idx = idx * nf[e] + q[e];
        int64_t sd = 1;
        for (int e = 3; e > d; --e) sd *= nf[e];
        const double* Fd = Fstar + P.foff[d];
        const double term = (Fd[idx + sd] - Fd[idx]) / hh[d];
        k = d == 0 ? -term : (d < 2 ? k - term : k + term);
    }
    const int64_t c = P.org + q[0] * P.s[0] + q[1] * P.s[1] + q[2] * P.s[2] + q[3];
    f_new[c] = f_n[c] + dt * k;
}

// Alg.4 "coarsen fluxes down to level l-1": every coarse F* face under a fine patch face := the
// mean of the R^3 fine F* faces over it (reading #14)
__global__ void k_fstar_coarsen(const FaceAvgTask* __restrict__ tasks, int64_t n, const double* __restrict__ Ff,
                                double* __restrict__ Fc) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const FaceAvgTask T = tasks[t];
    double s = 0.0;
    for (int a = 0; a < T.r[0]; ++a)
        for (int b = 0; b < T.r[1]; ++b)
            for (int c = 0; c < T.r[2]; ++c) s += Ff[T.fine + a * T.st[0] + b * T.st[1] + c * T.st[2]];
    Fc[T.coarse] = s / (double)(T.r[0] * T.r[1] * T.r[2]);
}

// average-down in 4D: covered coarse cell := mean of its R^4 fine cells
__global__ void k_average_down4(const AvgTask4* __restrict__ tasks, int64_t n, const double* __restrict__ ff,
                                double* __restrict__ fc) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const AvgTask4 T = tasks[t];
    double s = 0.0;
    for (int a = 0; a < T.r[0]; ++a)
        for (int b = 0; b < T.r[1]; ++b)
            for (int c = 0; c < T.r[2]; ++c)
                for (int d = 0; d < T.r[3]; ++d)
                    s += ff[T.fine + a * T.st[0] + b * T.st[1] + c * T.st[2] + d];
    fc[T.coarse] = s / (double)(T.r[0] * T.r[1] * T.r[2] * T.r[3]);
}

template <int STAGE, int RECON>
static int launch_s4(const Stage4Args& A, int maxcells, cudaStream_t st) {
    VK_CUDA(launch_pdl(k_stage4_fstar<STAGE, RECON>, dim3((unsigned)((maxcells + 127) / 128), (unsigned)A.npatch),
                       dim3(128), 0, st, A));
    return VLASOV_OK;
}

int launch_stage4_fstar(const vlasov_level* L, int stage, double dt, const double* f_n, const double* f_s,
                        double* f_next, const double* E, int recon, double* Fstar) {
    static const double B[4] = {1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0};
    static const double ALPHA[4] = {0.0, 0.5, 0.5, 1.0};
    Stage4Args A;
    A.patches = L->d_patch4;
    A.npatch = (int)L->boxes.size();
    A.f_s = f_s;
    A.f_n = f_n;
    A.f_next = f_next;
    A.E = E;
    A.Fstar = Fstar;
    A.dt = dt;
    A.b_s = B[stage - 1];
    A.alpha_next = stage < 4 ? ALPHA[stage] : 0.0;
    for (int d = 0; d < 4; ++d) A.h[d] = L->h[d];
    A.vlo[0] = L->lower[2];
    A.vlo[1] = L->lower[3];
    A.nx = L->dom[0];
    A.ny = L->dom[1];
    const int mc = L->max_patch_cells;
    const bool up = recon == VLASOV_UPWIND;
    switch (stage) {
        case 1: return up ? launch_s4<1, VLASOV_UPWIND>(A, mc, L->stream) : launch_s4<1, VLASOV_CENTERED4>(A, mc, L->stream);
        case 2: return up ? launch_s4<2, VLASOV_UPWIND>(A, mc, L->stream) : launch_s4<2, VLASOV_CENTERED4>(A, mc, L->stream);
        case 3: return up ? launch_s4<3, VLASOV_UPWIND>(A, mc, L->stream) : launch_s4<3, VLASOV_CENTERED4>(A, mc, L->stream);
        default: return up ? launch_s4<4, VLASOV_UPWIND>(A, mc, L->stream) : launch_s4<4, VLASOV_CENTERED4>(A, mc, L->stream);
    }
}

int launch_fstar_update(const vlasov_level* L, double dt, const double* f_n, const double* Fstar, double* f_new) {
    VK_CUDA(launch_pdl(k_fstar_update, dim3((unsigned)((L->max_patch_cells + 127) / 128), (unsigned)L->boxes.size()),
                       dim3(128), 0, L->stream, (const Patch4*)L->d_patch4, f_n, Fstar,
                       make_double4(L->h[0], L->h[1], L->h[2], L->h[3]), dt, f_new));
    return VLASOV_OK;
}

int launch_fstar_coarsen(const vlasov_level* L, const double* F_fine, double* F_coarse) {
    if (L->n_fcoarsen4 == 0) return VLASOV_OK;
    VK_CUDA(launch_pdl(k_fstar_coarsen, dim3((unsigned)((L->n_fcoarsen4 + 127) / 128)), dim3(128), 0, L->stream,
                       (const FaceAvgTask*)L->d_fcoarsen4, (int64_t)L->n_fcoarsen4, F_fine, F_coarse));
    return VLASOV_OK;
}

int launch_average_down4(const vlasov_level* L, const double* f_fine, double* f_coarse) {
    if (L->n_avg4 == 0) return VLASOV_OK;
    VK_CUDA(launch_pdl(k_average_down4, dim3((unsigned)((L->n_avg4 + 127) / 128)), dim3(128), 0, L->stream,
                       (const AvgTask4*)L->d_avg4, (int64_t)L->n_avg4, f_fine, f_coarse));
    return VLASOV_OK;
}

}  // namespace vk
