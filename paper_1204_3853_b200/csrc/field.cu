// Configuration-space kernels: fused-partial moment sum, periodic Poisson + E as
// circulant convolutions with exact discrete Green's functions (readings #1, #2),
// injection to a level.
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace vk {

// rho[x] = 1 - dv * sum_v f[x][v] on a single block covering the domain (one warp per x row;
// lane-strided sums combined by a fixed butterfly: deterministic)
__global__ void k_moment_direct(const double* __restrict__ f, int64_t off, int pitch, int nx, int nv, double dv,
                                double q, double base, int accumulate, double* __restrict__ rho) {
    const int lane = threadIdx.x & 31;
    const int x = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (x >= nx) return;
    const double* row = f + off + (int64_t)(x + G) * pitch + G;
    double s = 0.0;
    for (int j = lane; j < nv; j += 32) s += row[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) rho[x] = (accumulate ? rho[x] : base) + q * (dv * s);
}

int launch_moment_direct(const vlasov_level* L, const double* f, double* rho, double q, double base, int accumulate) {
    const int nx = L->dom[0], nv = L->dom[1];
    k_moment_direct<<<(nx + 7) / 8, 256, 0, L->stream>>>(f, L->block_off[0], (int)L->block_str[0][0], nx, nv,
                                                          L->h[1], q, base, accumulate, rho);
    VK_LAUNCH("k_moment_direct");
    return VLASOV_OK;
}

// out[i + ghost] = sum_k g[(i - k) mod n] (rho[k] - mean(rho)), plus periodic ghost copies.
// CTA = 16 x 16 threads for CIRC_OUT = 64 consecutive outputs: thread (tx, ty) accumulates outputs
// o0 = 4 tx .. o0 + 3 over the k-chunk ty with a sliding 4-value window of the (periodically
// extended) Green's function in shared memory; the 16 chunk partials are summed in chunk order.
// Every CTA stages the whole projected rho and reduces the mean itself in a fixed order, so the
// result is deterministic.  n <= CIRC_SMEM_MAX keeps g in shared memory (else read through L2).
constexpr int CIRC_TX = 16, CIRC_TY = 16, CIRC_OUT = 4 * CIRC_TX, CIRC_SMEM_MAX = 4096;

template <bool G_SMEM>
__global__ void __launch_bounds__(CIRC_TX * CIRC_TY) k_circulant(const double* __restrict__ rho,
                                                                  const double* __restrict__ g, int n, int ghost,
                                                                  double* __restrict__ out) {
    griddep_wait();
    griddep_launch_dependents();
    extern __shared__ double sm[];
    double* s_rho = sm;                                  // [n]
    double* s_part = sm + n;                             // [CIRC_TY][CIRC_OUT]
    double* s_g = s_part + CIRC_TY * CIRC_OUT;           // [2n + 4]: g[j mod n]
    __shared__ double s_red[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    double acc = 0.0;
    for (int k = tid; k < n; k += blockDim.x) {
        const double v = rho[k];
        s_rho[k] = v;
        acc += v;
    }
    if (G_SMEM)
        for (int j = tid; j < 2 * n + 4; j += blockDim.x) s_g[j] = __ldg(g + (j % n));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) s_red[warp] = acc;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += s_red[w];
        s_red[0] = s / (double)n;
    }
    __syncthreads();
    const double mean = s_red[0];
    for (int k = tid; k < n; k += blockDim.x) s_rho[k] -= mean;      // projection
    __syncthreads();

    const int tx = tid % CIRC_TX, ty = tid / CIRC_TX;
    const int o0 = blockIdx.x * CIRC_OUT + 4 * tx;
    const int kb = (int)((int64_t)n * ty / CIRC_TY), ke = (int)((int64_t)n * (ty + 1) / CIRC_TY);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (o0 < n && kb < ke) {
        auto gv = [&](int j) -> double { return G_SMEM ? s_g[j] : __ldg(g + (j % n)); };
        int j = n + o0 - kb;                             // g index of output o0 at k = kb
        double w0 = gv(j), w1 = gv(j + 1), w2 = gv(j + 2), w3 = gv(j + 3);
        for (int k = kb; k < ke; ++k) {
            const double r = s_rho[k];
            a0 = fma(w0, r, a0);
            a1 = fma(w1, r, a1);
            a2 = fma(w2, r, a2);
            a3 = fma(w3, r, a3);
            w3 = w2; w2 = w1; w1 = w0;
            w0 = gv(--j);
        }
    }
    double* pp = s_part + ty * CIRC_OUT + 4 * tx;
    pp[0] = a0; pp[1] = a1; pp[2] = a2; pp[3] = a3;
    __syncthreads();
    if (tid < CIRC_OUT) {
        const int i = blockIdx.x * CIRC_OUT + tid;
        if (i < n) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < CIRC_TY; ++c) s += s_part[c * CIRC_OUT + tid];
            out[i + ghost] = s;
            if (i < ghost) out[i + ghost + n] = s;
            if (i >= n - ghost) out[i + ghost - n] = s;
        }
    }
}

int launch_poisson(vlasov_poisson* P, const double* rho, double* phi, double* E, int ghost) {
    const int n = P->n;
    const int blocks = (n + CIRC_OUT - 1) / CIRC_OUT;
    const bool gs = n <= CIRC_SMEM_MAX;
    const size_t smem = (size_t)(n + CIRC_TY * CIRC_OUT + (gs ? 2 * n + 4 : 0)) * sizeof(double);
    static bool conf = false;
    if (!conf) {
        VK_CUDA(cudaFuncSetAttribute(k_circulant<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        VK_CUDA(cudaFuncSetAttribute(k_circulant<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        conf = true;
    }
    auto kern = gs ? k_circulant<true> : k_circulant<false>;
    if (E) {
        VK_CUDA(launch_pdl(kern, dim3(blocks), dim3(CIRC_TX * CIRC_TY), smem, P->stream, rho, (const double*)P->d_gE, n,
                           ghost, E));
    }
    if (phi) {
        VK_CUDA(launch_pdl(kern, dim3(blocks), dim3(CIRC_TX * CIRC_TY), smem, P->stream, rho, (const double*)P->d_gphi,
                           n, ghost, phi));
    }
    return VLASOV_OK;
}

// E_lvl[i + 2] = scale * mean_{s<R} E_f[R i + s]; periodic ghosts i = -2, -1, n, n+1.
__global__ void k_inject_1d(const double* __restrict__ Ef, int nf, int R, int n, double scale, double* __restrict__ El) {
    griddep_wait();
    griddep_launch_dependents();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n + 4) return;
    int i = t - 2;
    i = (i < 0) ? i + n : (i >= n ? i - n : i);
    double s = 0.0;
    for (int q = 0; q < R; ++q) s += Ef[(int64_t)i * R + q];
    El[t] = scale * ((R == 1) ? s : s / (double)R);
}

int launch_inject_1d(const vlasov_level* L, const double* E_finest, int n_finest, double* E_lvl, double scale) {
    const int n = L->dom[0];
    if (n_finest % n) return fail(VLASOV_EINVAL, "inject: finest size not a multiple of the level size");
    const int R = n_finest / n;
    VK_CUDA(launch_pdl(k_inject_1d, dim3((n + 4 + 127) / 128), dim3(128), 0, L->stream, E_finest, n_finest, R, n, scale,
                       E_lvl));
    VK_LAUNCH("k_inject_1d");
    return VLASOV_OK;
}

// 2D configuration space, C = 2 components: El[c][(i+2)*(ny+4) + (k+2)] = mean over Rx x Ry.
__global__ void k_inject_2d(const double* __restrict__ Ef, int nfx, int nfy, int Rx, int Ry, int nx,
                            int ny, double* __restrict__ El, int gin) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int nxg = nx + 4, nyg = ny + 4;
    if (t >= 2 * nxg * nyg) return;
    const int c = t / (nxg * nyg), rem = t % (nxg * nyg);
    int i = rem / nyg - 2, k = rem % nyg - 2;
    i = (i < 0) ? i + nx : (i >= nx ? i - nx : i);
    k = (k < 0) ? k + ny : (k >= ny ? k - ny : k);
    double s = 0.0;
    for (int a = 0; a < Rx; ++a)
        for (int b = 0; b < Ry; ++b)
            s += Ef[(int64_t)c * (nfx + 2 * gin) * (nfy + 2 * gin) + (int64_t)(i * Rx + a + gin) * (nfy + 2 * gin) +
                    (k * Ry + b + gin)];
    El[t] = (Rx * Ry == 1) ? s : s / (double)(Rx * Ry);
}

int launch_inject_2d(const vlasov_level* L, const double* E_finest, const int32_t* n_finest, double* E_lvl, int gin) {
    const int nx = L->dom[0], ny = L->dom[1];
    if (n_finest[0] % nx || n_finest[1] % ny) return fail(VLASOV_EINVAL, "inject: size mismatch");
    const int tot = 2 * (nx + 4) * (ny + 4);
    k_inject_2d<<<(tot + 255) / 256, 256, 0, L->stream>>>(E_finest, n_finest[0], n_finest[1],
                                                            n_finest[0] / nx, n_finest[1] / ny, nx, ny, E_lvl, gin);
    VK_LAUNCH("k_inject_2d");
    return VLASOV_OK;
}

// out[0] = max_i |x_i| (one CTA, fixed-order tree: deterministic); used by the adaptive time step
__global__ void k_absmax(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
    __shared__ double s[32];
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = (threadIdx.x < (blockDim.x >> 5)) ? s[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) out[0] = m;
    }
}

// velocity-slab halo: pack the two lowest / highest interior velocity columns of every interior
// row into [nx][2] arrays, or unpack arrays into the two low / high ghost columns.  One thread per
// (side, row, column pair); rows of a single block.
__global__ void k_vslab(double* __restrict__ f, int64_t org, int64_t pitch, int nx, int nv, double* __restrict__ lo,
                        double* __restrict__ hi, int pack) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * nx) return;
    const int side = t / nx, x = t - side * nx;
    double* buf = side ? hi : lo;
    if (!buf) return;
    double* row = f + org + (int64_t)x * pitch;                   // interior column 0 of row x
    double* col = pack ? (side ? row + nv - 2 : row) : (side ? row + nv : row - 2);
    double2* b2 = reinterpret_cast<double2*>(buf + 2 * x);
    if (pack) {
        *b2 = make_double2(col[0], col[1]);
    } else {
        const double2 v = *b2;
        col[0] = v.x;
        col[1] = v.y;
    }
}

int launch_vslab(const vlasov_level* L, double* f, double* lo, double* hi, bool pack) {
    const int nx = L->dom[0], nv = L->dom[1];
    const int64_t pitch = L->block_str[0][0];
    const int64_t org = L->block_off[0] + (int64_t)G * pitch + G;
    k_vslab<<<(2 * nx + 127) / 128, 128, 0, L->stream>>>(f, org, pitch, nx, nv, lo, hi, pack ? 1 : 0);
    VK_LAUNCH("k_vslab");
    return VLASOV_OK;
}

// j[x] = (acc ? j[x] : 0) + q dv sum_v (vbar_v f_v + dv/24 (f_{v+1} - f_{v-1})): one warp per row x,
// lanes strided over v, fixed butterfly (deterministic)
__global__ void k_current_1d(const double* __restrict__ f, int64_t org, int64_t pitch, int nx, int nv, double vlo,
                             double dv, double q, int accumulate, double* __restrict__ j) {
    const int lane = threadIdx.x & 31;
    const int x = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (x >= nx) return;
    const double* row = f + org + (int64_t)x * pitch;            // interior column 0 of row x
    double s = 0.0, d = 0.0;
    for (int v = lane; v < nv; v += 32) {
        s += (vlo + ((double)v + 0.5) * dv) * row[v];
        d += row[v + 1] - row[v - 1];
    }
    double t = s + (dv * (1.0 / 24.0)) * d;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) j[x] = (accumulate ? j[x] : 0.0) + q * dv * t;
}

int launch_current(const vlasov_level* L, const double* f, double q, int accumulate, double* j) {
    const int nx = L->dom[0], nv = L->dom[1];
    const int64_t pitch = L->block_str[0][0];
    const int64_t org = L->block_off[0] + (int64_t)G * pitch + G;
    k_current_1d<<<(nx + 3) / 4, 128, 0, L->stream>>>(f, org, pitch, nx, nv, L->lower[1], L->h[1], q, accumulate, j);
    VK_LAUNCH("k_current_1d");
    return VLASOV_OK;
}

int launch_absmax(const double* x, int64_t n, double* out, cudaStream_t st) {
    k_absmax<<<1, 1024, 0, st>>>(x, n, out);
    VK_LAUNCH("k_absmax");
    return VLASOV_OK;
}

}  // namespace vk

namespace vk {

// 2D periodic field (N3, reading #32): E_c(i, k) = sum_{i', k'} g_c((i - i') mod nx, (k - k') mod ny)
// (rho(i', k') - mean rho), c = x, y, with the exact discrete Green's functions of the 2D fourth-
// order operator composed with -D4 (host, long double).  CTA = one output row i (all k): the
// projected rho and both Green's functions staged in shared memory (nx ny <= P2_SMEM_MAX), thread
// group t sums a fixed i' range for its outputs, the partials are added in group order
// (deterministic); the CTA writes its row of the ghosted E arrays and the periodic ghost copies.
constexpr int P2_THREADS = 256, P2_SMEM_MAX = 8192;

template <bool G_SMEM>
__global__ void __launch_bounds__(P2_THREADS) k_poisson2d(const double* __restrict__ rho, const double* __restrict__ gx,
                                                           const double* __restrict__ gy, int nx, int ny,
                                                           double* __restrict__ E) {
    griddep_wait();
    griddep_launch_dependents();
    extern __shared__ double sm[];
    const int n = nx * ny;
    double* s_rho = sm;                                   // [n]
    double* s_gx = sm + n;                                // [n] (G_SMEM)
    double* s_gy = s_gx + n;                              // [n] (G_SMEM)
    double* s_part = G_SMEM ? s_gy + n : s_gx;            // [2][P2_THREADS]
    __shared__ double s_red[P2_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double acc = 0.0;
    for (int t = tid; t < n; t += P2_THREADS) {
        const double v = rho[t];
        s_rho[t] = v;
        acc += v;
        if (G_SMEM) { s_gx[t] = gx[t]; s_gy[t] = gy[t]; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) s_red[warp] = acc;
    __syncthreads();
    double mean = 0.0;
#pragma unroll
    for (int w = 0; w < P2_THREADS / 32; ++w) mean += s_red[w];
    mean /= (double)n;
    const double* Gx = G_SMEM ? s_gx : gx;
    const double* Gy = G_SMEM ? s_gy : gy;
    const int i = blockIdx.x;
    const int ngrp = P2_THREADS / ny > 0 ? P2_THREADS / ny : 1;      // thread groups per output
    const int nyg = ny + 4;
    for (int k0 = 0; k0 < ny; k0 += P2_THREADS / ngrp) {
        const int kk = k0 + tid % (P2_THREADS / ngrp), grp = tid / (P2_THREADS / ngrp);
        double ax = 0.0, ay = 0.0;
        if (kk < ny && grp < ngrp) {
            const int ib = (int)((int64_t)nx * grp / ngrp), ie = (int)((int64_t)nx * (grp + 1) / ngrp);
            for (int ip = ib; ip < ie; ++ip) {
                const int di = i - ip < 0 ? i - ip + nx : i - ip;
                const double* rr = s_rho + ip * ny;
                const double* gxr = Gx + di * ny;
                const double* gyr = Gy + di * ny;
                for (int kp = 0; kp < ny; ++kp) {
                    const int dk = kk - kp < 0 ? kk - kp + ny : kk - kp;
                    const double r = rr[kp] - mean;
                    ax = fma(gxr[dk], r, ax);
                    ay = fma(gyr[dk], r, ay);
                }
            }
        }
        __syncthreads();
        s_part[tid] = ax;
        s_part[P2_THREADS + tid] = ay;
        __syncthreads();
        if (grp == 0 && kk < ny) {
            const int per = P2_THREADS / ngrp;
            double ex = 0.0, ey = 0.0;
            for (int g = 0; g < ngrp; ++g) { ex += s_part[g * per + tid % per]; ey += s_part[P2_THREADS + g * per + tid % per]; }
            // own row and the periodic ghost rows / columns (x ghosts: rows i -+ nx)
            for (int c = 0; c < 2; ++c) {
                const double e = c ? ey : ex;
                double* Ec = E + (int64_t)c * (nx + 4) * nyg;
                const int rows[3] = {i + 2, i + 2 + nx, i + 2 - nx};
                for (int r = 0; r < 3; ++r) {
                    const int gr = rows[r];
                    if (gr < 0 || gr >= nx + 4) continue;
                    double* row = Ec + (int64_t)gr * nyg;
                    row[kk + 2] = e;
                    if (kk < 2) row[kk + 2 + ny] = e;
                    if (kk >= ny - 2) row[kk + 2 - ny] = e;
                }
            }
        }
    }
}

// Toeplitz-blocked variant (ny in {8, 16, ..., 256}): thread (subset s, output block b) sums, for the
// i' of its subset (i' = s, s + S, ...), the 8 outputs k = 8b .. 8b+7 of row i with a sliding
// register window of the Green's functions (one new g value per component and k', one broadcast
// rho value, 16 FMAs); the S subset partials are added in subset order (deterministic).
constexpr int P2T_K = 8;
// Launched as clusters of P2T_SPLIT CTAs per output row: CTA rank c of the cluster takes the i'
// of every P2T_SPLIT-th subset; rank 0 adds the ranks' partials (DSMEM) in rank order.
constexpr int P2T_SPLIT = 2;
__global__ void __launch_bounds__(P2_THREADS) k_poisson2d_tb(const double* __restrict__ rho, const double* __restrict__ gx,
                                                              const double* __restrict__ gy, int nx, int ny,
                                                              double* __restrict__ E) {
    griddep_wait();
    griddep_launch_dependents();
    extern __shared__ double sm[];
    const int n = nx * ny;
    double* s_rho = sm;                                   // [n]
    double* s_gx = sm + n;                                // [n]
    double* s_gy = s_gx + n;                              // [n]
    double* s_part = s_gy + n;                            // [2][P2_THREADS][8]
    __shared__ double s_red[P2_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double acc = 0.0;
    // 16-byte loads, 4 in flight per thread per array (n = nx ny is a multiple of 8: ny % 8 == 0)
    const int n2 = n / 2;
    for (int t0 = tid; t0 < n2; t0 += 4 * P2_THREADS) {
        double2 r[4], a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = t0 + u * P2_THREADS;
            if (t < n2) {
                r[u] = __ldg(reinterpret_cast<const double2*>(rho) + t);
                a[u] = __ldg(reinterpret_cast<const double2*>(gx) + t);
                b[u] = __ldg(reinterpret_cast<const double2*>(gy) + t);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = t0 + u * P2_THREADS;
            if (t < n2) {
                reinterpret_cast<double2*>(s_rho)[t] = r[u];
                reinterpret_cast<double2*>(s_gx)[t] = a[u];
                reinterpret_cast<double2*>(s_gy)[t] = b[u];
                acc += r[u].x + r[u].y;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) s_red[warp] = acc;
    __syncthreads();
    double mean = 0.0;
#pragma unroll
    for (int w = 0; w < P2_THREADS / 32; ++w) mean += s_red[w];
    mean /= (double)n;
    for (int t = tid; t < n; t += P2_THREADS) s_rho[t] -= mean;
    __syncthreads();
    const int i = blockIdx.x / P2T_SPLIT, crank = (int)cluster_ctarank();
    const int nb = ny / P2T_K, S = P2_THREADS / nb;
    const int b = tid % nb, sub = tid / nb;
    double ax[P2T_K], ay[P2T_K];
#pragma unroll
    for (int j = 0; j < P2T_K; ++j) ax[j] = ay[j] = 0.0;
    for (int ip = sub * P2T_SPLIT + crank; ip < nx; ip += S * P2T_SPLIT) {
        const int di = i - ip < 0 ? i - ip + nx : i - ip;
        const double* rr = s_rho + ip * ny;
        const double* gxr = s_gx + di * ny;
        const double* gyr = s_gy + di * ny;
        // window w[j] = g[(8b + j - kp) mod ny]
        double wx[P2T_K], wy[P2T_K];
#pragma unroll
        for (int j = 0; j < P2T_K; ++j) { wx[j] = gxr[P2T_K * b + j]; wy[j] = gyr[P2T_K * b + j]; }
        for (int kp0 = 0; kp0 < ny; kp0 += P2T_K) {
#pragma unroll
            for (int u = 0; u < P2T_K; ++u) {
                const int kp = kp0 + u;
                const double r = rr[kp];
#pragma unroll
                for (int j = 0; j < P2T_K; ++j) {
                    // slot of output j in the rotating window after u shifts
                    const int sl = (j - u + P2T_K * 8) % P2T_K;
                    ax[j] = fma(wx[sl], r, ax[j]);
                    ay[j] = fma(wy[sl], r, ay[j]);
                }
                // shift: the slot of output 7 becomes the slot of output 0 with g[(8b - kp - 1) mod ny]
                const int sl7 = (P2T_K - 1 - u + P2T_K * 8) % P2T_K;
                int q = P2T_K * b - kp - 1;
                q += (q < 0) ? ny : 0;
                wx[sl7] = gxr[q];
                wy[sl7] = gyr[q];
            }
        }
    }
    double* px = s_part + (size_t)tid * P2T_K;
    double* py = s_part + (size_t)(P2_THREADS + tid) * P2T_K;
#pragma unroll
    for (int j = 0; j < P2T_K; ++j) { px[j] = ax[j]; py[j] = ay[j]; }
    __syncthreads();
    // per-rank sums over the S subsets (fixed order), into the dead rho area: s_sum[c][k]
    double* s_sum = s_rho;
    for (int t = tid; t < 2 * ny; t += P2_THREADS) {
        const int c = t / ny, kk = t - c * ny, bb = kk / P2T_K, jj = kk % P2T_K;
        const double* pp = s_part + (size_t)c * P2_THREADS * P2T_K;
        double e = 0.0;
        for (int g = 0; g < S; ++g) e += pp[(size_t)(g * nb + bb) * P2T_K + jj];
        s_sum[t] = e;
    }
    cluster_sync_all();                                   // every rank's sums visible
    const int nyg = ny + 4;
    for (int t = tid; t < 2 * ny && crank == 0; t += P2_THREADS) {
        const int c = t / ny, kk = t - c * ny;
        double e = s_sum[t];
        for (int r = 1; r < P2T_SPLIT; ++r) {             // ranks in order (deterministic)
            double v;
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(map_shared_rank(s_sum + t, (uint32_t)r)) : "memory");
            e += v;
        }
        double* Ec = E + (int64_t)c * (nx + 4) * nyg;
        const int rows[3] = {i + 2, i + 2 + nx, i + 2 - nx};
        for (int r = 0; r < 3; ++r) {
            const int gr = rows[r];
            if (gr < 0 || gr >= nx + 4) continue;
            double* row = Ec + (int64_t)gr * nyg;
            row[kk + 2] = e;
            if (kk < 2) row[kk + 2 + ny] = e;
            if (kk >= ny - 2) row[kk + 2 - ny] = e;
        }
    }
    cluster_sync_all();                                   // rank 0 done reading the other ranks
}

int launch_poisson2d(const vlasov_poisson2d* P, const double* rho, double* E) {
    const int n = P->nx * P->ny;
    const int ny = P->ny;
    static const bool plain = std::getenv("VLASOV_POISSON2D_PLAIN") != nullptr;   // experiment switch
    if (!plain && ny % P2T_K == 0 && ny / P2T_K <= 32 && (32 % (ny / P2T_K)) == 0 && n <= P2_SMEM_MAX &&
        ((uintptr_t)rho & 15) == 0) {
        const size_t smem = (size_t)(3 * n + 2 * P2_THREADS * P2T_K) * sizeof(double);
        static bool cfg = false;
        if (!cfg) {
            VK_CUDA(cudaFuncSetAttribute(k_poisson2d_tb, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            cfg = true;
        }
        cudaLaunchConfig_t cfgl = {};
        cfgl.gridDim = dim3(P->nx * P2T_SPLIT);
        cfgl.blockDim = dim3(P2_THREADS);
        cfgl.dynamicSmemBytes = smem;
        cfgl.stream = P->stream;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = VK_PDL;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = P2T_SPLIT;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfgl.attrs = at;
        cfgl.numAttrs = 2;
        VK_CUDA(cudaLaunchKernelEx(&cfgl, k_poisson2d_tb, rho, (const double*)P->d_gx, (const double*)P->d_gy,
                                   P->nx, P->ny, E));
        return VLASOV_OK;
    }
    if (n <= P2_SMEM_MAX) {
        const size_t smem = (size_t)(3 * n + 2 * P2_THREADS) * sizeof(double);
        static bool cfg = false;
        if (!cfg) {
            VK_CUDA(cudaFuncSetAttribute(k_poisson2d<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            cfg = true;
        }
        VK_CUDA(launch_pdl(k_poisson2d<true>, dim3(P->nx), dim3(P2_THREADS), smem, P->stream, rho,
                           (const double*)P->d_gx, (const double*)P->d_gy, P->nx, P->ny, E));
    } else {
        const size_t smem = (size_t)(n + 2 * P2_THREADS) * sizeof(double);
        if (smem > 220 * 1024) return fail(VLASOV_EUNSUPPORTED, "poisson2d: nx * ny too large");
        static bool cfg = false;
        if (!cfg) {
            VK_CUDA(cudaFuncSetAttribute(k_poisson2d<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            cfg = true;
        }
        VK_CUDA(launch_pdl(k_poisson2d<false>, dim3(P->nx), dim3(P2_THREADS), smem, P->stream, rho,
                           (const double*)P->d_gx, (const double*)P->d_gy, P->nx, P->ny, E));
    }
    return VLASOV_OK;
}

}  // namespace vk
