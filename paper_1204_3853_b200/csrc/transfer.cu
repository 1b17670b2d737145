// Same-level and coarse-fine ghost fill, characteristic velocity BC (1D+1V task lists).
//
// PAPER.md: ghost exchange P:482-483; Alg.2 order interpolate / exchange / BC P:605-609
// (reading #15: siblings + CF, then PHYS); conservative interpolation P:695-876 (linear5
// P:959-996 with reading #12, WENO5 P:741-831 with readings #8-#10, dimension by dimension,
// x first P:864-876); characteristic BC P:227-231 (reading #6).
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace vk {

// ------------------------------------------------------------------ 1D conservative interpolation
// u[0..4] = coarse u_{i-2..i+2}; returns fine average of sub-cell s of R.
__device__ __forceinline__ double interp_linear5(const double* u, const double* b5 /* [R][5] */, int s) {
    const double* b = b5 + 5 * s;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 5; ++j) acc += b[j] * u[j];
    return acc;
}

__device__ double interp_weno5(const double* u, int R, int s) {
    const double um2 = u[0], um1 = u[1], u0 = u[2], up1 = u[3], up2 = u[4];
    const double Dm2 = um1 - um2, Dm1 = u0 - um1, D0 = up1 - u0, Dp1 = up2 - up1;   // (aux1)
    const double Lm1 = Dm1 - Dm2, L0 = D0 - Dm1, Lp1 = Dp1 - D0;
    const double b0 = (13.0 / 12.0) * Lp1 * Lp1 + 0.25 * (Dp1 - 3.0 * D0) * (Dp1 - 3.0 * D0);
    const double b1 = (13.0 / 12.0) * L0 * L0 + 0.25 * (D0 + Dm1) * (D0 + Dm1);
    const double b2 = (13.0 / 12.0) * Lm1 * Lm1 + 0.25 * (3.0 * Dm1 - Dm2) * (3.0 * Dm1 - Dm2);
    const double a0 = 0.3 / ((1e-6 + b0) * (1e-6 + b0));
    const double a1 = 0.6 / ((1e-6 + b1) * (1e-6 + b1));
    const double a2 = 0.1 / ((1e-6 + b2) * (1e-6 + b2));
    const double asum = a0 + a1 + a2;
    const double w0 = a0 / asum, w1 = a1 / asum, w2 = a2 / asum;
    const double A0 = u0 + (2.0 * Dp1 - 5.0 * D0) / 6.0;                             // (aux2)
    const double A1 = u0 - (D0 + 2.0 * Dm1) / 6.0;
    const double A2 = u0 - (4.0 * Dm1 - Dm2) / 6.0;
    const double B0 = 2.0 * D0 - Dp1, B1 = Dm1, B2 = Dm1;                              // reading #8
    const double C0 = Lp1, C1 = L0, C2 = Lm1;
    double mine = 0.0, sum = 0.0;
    for (int q = 0; q < R; ++q) {
        const double bs = (2.0 * q + 1.0) / (2.0 * R);
        const double cs = (3.0 * q * q + 3.0 * q + 1.0) / (6.0 * R * R);
        const double v = w0 * (A0 + B0 * bs + C0 * cs) + w1 * (A1 + B1 * bs + C1 * cs) +
                         w2 * (A2 + B2 * bs + C2 * cs);
        sum += v;
        if (q == s) mine = v;
    }
    return mine + (u0 - sum / R);                                                      // reading #10
}

template <int INTERP>
__device__ __forceinline__ double interp1(const double* u, const double* b5, int R, int s) {
    return INTERP == VLASOV_WENO5 ? interp_weno5(u, R, s) : interp_linear5(u, b5, s);
}

// ------------------------------------------------------------------ ghost fill kernels
template <int INTERP>
__global__ void k_fill_copy_cf(double* __restrict__ f, const double* __restrict__ fsrc,
                               const int64_t* __restrict__ copies, int64_t ncopy, const double* __restrict__ fc, const CFTask* __restrict__ cf, int64_t ncf,
                               const double* __restrict__ b5, int Rx, int Rv) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < ncopy) {
        f[copies[2 * t]] = fsrc[copies[2 * t + 1]];
        return;
    }
    const int64_t c = t - ncopy;
    if (c >= ncf) return;
    const CFTask T = cf[c];
    double part[5];
#pragma unroll
    for (int b = 0; b < 5; ++b) {                 // x pass on the 5 coarse v-columns
        double col[5];
#pragma unroll
        for (int a = 0; a < 5; ++a) col[a] = fc[T.csrc + (int64_t)(a - 2) * T.cstride[0] + (b - 2)];
        part[b] = interp1<INTERP>(col, b5, Rx, T.sub[0]);
    }
    f[T.dst] = interp1<INTERP>(part, b5 + 5 * MAXR, Rv, T.sub[1]);   // v pass
}

__global__ void k_fill_phys(double* __restrict__ f, const PhysTask* __restrict__ tasks, int64_t n,
                            const double* __restrict__ E_bc, const double* __restrict__ f0v, int nv) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const PhysTask T = tasks[t];
    const double a = -E_bc[T.e_idx];
    const int64_t dir = T.side == 0 ? 1 : -1;     // inward step along v
    const double f0 = f[T.cell0], f1 = f[T.cell0 + dir], f2 = f[T.cell0 + 2 * dir], f3 = f[T.cell0 + 3 * dir];
    const bool out = T.side == 0 ? (a < 0.0) : (a > 0.0);
    double g1, g2;
    if (out) {                                    // cubic extrapolation (reading #6)
        g1 = 4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3;
        g2 = 10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3;
    } else if (T.side == 0) {                     // unperturbed profile
        g1 = f0v[1]; g2 = f0v[0];
    } else {
        g1 = f0v[nv + 2]; g2 = f0v[nv + 3];
    }
    f[T.cell0 - dir] = g1;
    f[T.cell0 - 2 * dir] = g2;
}

int launch_fill(vlasov_level* L, double* f, const double* f_coarse, const double* E_bc,
                const double* f0v, int interp) {
    const int64_t n1 = L->n_copy + L->n_cf;
    if (L->n_cf > 0 && f_coarse == nullptr) return fail(VLASOV_EINVAL, "fill_ghosts: coarse data required");
    if (n1 > 0) {
        const int64_t blocks = (n1 + 255) / 256;
        auto kern = interp == VLASOV_WENO5 ? k_fill_copy_cf<VLASOV_WENO5> : k_fill_copy_cf<VLASOV_LINEAR5>;
        VK_CUDA(launch_pdl(kern, dim3((unsigned)blocks), dim3(256), 0, L->stream, f, (const double*)f,
                           (const int64_t*)L->d_copy, (int64_t)L->n_copy, f_coarse, (const CFTask*)L->d_cf,
                           (int64_t)L->n_cf, (const double*)L->d_b5, L->coarse_ratio[0], L->coarse_ratio[1]));
    }
    if (L->n_phys > 0) {
        if (E_bc == nullptr || f0v == nullptr) return fail(VLASOV_EINVAL, "fill_ghosts: E_bc and f0v required");
        VK_CUDA(launch_pdl(k_fill_phys, dim3((unsigned)((L->n_phys + 255) / 256)), dim3(256), 0, L->stream, f,
                           (const PhysTask*)L->d_phys, (int64_t)L->n_phys, E_bc, f0v, L->dom[1]));
    }
    return VLASOV_OK;
}

// Regrid data motion (vlasov_level_fill_from): the task lists depend on the old level, so they
// are built per call and staged through stream-ordered scratch; the call synchronises its stream
// (a regrid is a host decision point anyway).
// fill_from: one block per overlap rectangle, threads strided over its cells (v fastest)
__global__ void k_copy_rects(double* __restrict__ f, const double* __restrict__ fo, const RectCopy* __restrict__ R) {
    const RectCopy r = R[blockIdx.x];
    const int64_t n = (int64_t)r.nx * r.nv;
    for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
        const int x = (int)(t / r.nv), v = (int)(t - (int64_t)x * r.nv);
        f[r.dst + (int64_t)x * r.dpitch + v] = fo[r.src + (int64_t)x * r.spitch + v];
    }
}

int launch_fill_from(const vlasov_level* L, double* f, const double* f_old, const std::vector<RectCopy>& rects,
                     const double* f_coarse, const std::vector<CFTask>& cfs, int interp) {
    const int64_t nrect = (int64_t)rects.size(), ncf = (int64_t)cfs.size();
    if (nrect + ncf == 0) return VLASOV_OK;
    RectCopy* d_rect = nullptr;
    CFTask* d_cf = nullptr;
    if (nrect) {
        VK_CUDA(cudaMallocAsync((void**)&d_rect, rects.size() * sizeof(RectCopy), L->stream));
        VK_CUDA(cudaMemcpyAsync(d_rect, rects.data(), rects.size() * sizeof(RectCopy), cudaMemcpyHostToDevice, L->stream));
        k_copy_rects<<<(unsigned)nrect, 256, 0, L->stream>>>(f, f_old, d_rect);
        VK_LAUNCH("k_copy_rects");
    }
    if (ncf) {
        VK_CUDA(cudaMallocAsync((void**)&d_cf, cfs.size() * sizeof(CFTask), L->stream));
        VK_CUDA(cudaMemcpyAsync(d_cf, cfs.data(), cfs.size() * sizeof(CFTask), cudaMemcpyHostToDevice, L->stream));
        const unsigned blocks = (unsigned)((ncf + 255) / 256);
        if (interp == VLASOV_WENO5)
            k_fill_copy_cf<VLASOV_WENO5><<<blocks, 256, 0, L->stream>>>(f, f, nullptr, 0, f_coarse, d_cf, ncf, L->d_b5,
                                                                          L->coarse_ratio[0], L->coarse_ratio[1]);
        else
            k_fill_copy_cf<VLASOV_LINEAR5><<<blocks, 256, 0, L->stream>>>(f, f, nullptr, 0, f_coarse, d_cf, ncf,
                                                                            L->d_b5, L->coarse_ratio[0], L->coarse_ratio[1]);
        VK_LAUNCH("k_fill_copy_cf(fill_from)");
    }
    if (d_rect) cudaFreeAsync(d_rect, L->stream);
    if (d_cf) cudaFreeAsync(d_cf, L->stream);
    VK_CUDA(cudaStreamSynchronize(L->stream));
    return VLASOV_OK;
}

}  // namespace vk
