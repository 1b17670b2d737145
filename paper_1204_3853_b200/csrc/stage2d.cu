// 2D+2V fused RK4 stage kernel (BASELINE.json C5): face averages -> fluxes -> divergence -> RK4
// stage combine -> per-(vx line, vy tile) partials of the velocity moment.
//
// PAPER.md: the 1D+1V discretisation generalised dimension by dimension, as the oracle
// (oracle/scheme.py) does: a configuration face along x_d carries one transverse term along v_d
// (dv_d/24); a velocity face along v_d carries one (1/48) product term per configuration dim.
// Divergence of  f_t + div_x(v f) - div_v(E f) = 0  (reading #1).  Periodic x, y; the
// characteristic condition on vx, vy (reading #6) is evaluated in the kernel, so the
// level must be ONE block covering the periodic domain (SELF mode).
//
// Layout: [x][y][vx][vy], vy contiguous, ghost frame 2 (never read).  Thread = (y = k, vx = l,
// vy pair m0, m0+1); the CTA is 32 vy-pairs x 4 vx lines; every thread marches along x over a strip
// of rows with register windows of the x-direction data (x-faces computed once per row) and of
// the velocity-face averages of rows i-1, i, i+1 (x-transverse terms).  y-direction and vx +-2
// neighbours are read through L1/L2 as 16-byte pairs.
#include <cuda_runtime.h>

#include "internal.h"
#include "scheme.cuh"

namespace vk {
#ifndef STAGE2D_MINB
#define STAGE2D_MINB 2
#endif

struct StageArgs2 {
    const double* f_s;
    const double* f_n;
    const double* u_in;
    double* u_out;
    double* f_next;
    const double* E;           // [2][(nx+4)(ny+4)] ghosted level field
    const double* E_bc;        // same layout: decides the characteristic direction
    const double* f0v;         // [(nvx+4)(nvy+4)] unperturbed profile on the ghosted v range
    double* partials;          // [nvx * n_mtiles][nx][ny] moment partials (nullable)
    int64_t s0, s1, s2;        // strides of x, y, vx (vy stride 1)
    int64_t org;               // index of interior cell (0,0,0,0)
    int nx, ny, nvx, nvy, nrows, nstrips;
    double dt, hx, hy, hvx, hvy, vx_lo, vy_lo;
};

// f at (i, k, l, m) with periodic x, y and the characteristic v-boundary condition
__device__ __forceinline__ double f_at(const StageArgs2& A, int i, int k, int l, int m) {
    i = (i < 0) ? i + A.nx : (i >= A.nx ? i - A.nx : i);
    k = (k < 0) ? k + A.ny : (k >= A.ny ? k - A.ny : k);
    const int64_t base = A.org + (int64_t)i * A.s0 + (int64_t)k * A.s1;
    const int nyg = A.ny + 4;
    if (l < 0 || l >= A.nvx) {               // vx ghost: a = -E_x(i, k)
        const double a = -__ldg(A.E_bc + (int64_t)(i + 2) * nyg + (k + 2));
        const bool lo = l < 0;
        if (lo ? (a < 0.0) : (a > 0.0)) {
            const int j0 = lo ? 0 : A.nvx - 1, dj = lo ? 1 : -1;
            const double* p = A.f_s + base + m;
            const double f0 = p[(int64_t)j0 * A.s2], f1 = p[(int64_t)(j0 + dj) * A.s2];
            const double f2 = p[(int64_t)(j0 + 2 * dj) * A.s2], f3 = p[(int64_t)(j0 + 3 * dj) * A.s2];
            const bool first = lo ? (l == -1) : (l == A.nvx);
            return first ? 4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3 : 10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3;
        }
        return __ldg(A.f0v + (int64_t)(l + 2) * (A.nvy + 4) + (m + 2));
    }
    if (m < 0 || m >= A.nvy) {               // vy ghost: a = -E_y(i, k)
        const double a = -__ldg(A.E_bc + (int64_t)(A.nx + 4) * nyg + (int64_t)(i + 2) * nyg + (k + 2));
        const bool lo = m < 0;
        if (lo ? (a < 0.0) : (a > 0.0)) {
            const int j0 = lo ? 0 : A.nvy - 1, dj = lo ? 1 : -1;
            const double* p = A.f_s + base + (int64_t)l * A.s2;
            const double f0 = p[j0], f1 = p[j0 + dj], f2 = p[j0 + 2 * dj], f3 = p[j0 + 3 * dj];
            const bool first = lo ? (m == -1) : (m == A.nvy);
            return first ? 4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3 : 10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3;
        }
        return __ldg(A.f0v + (int64_t)(l + 2) * (A.nvy + 4) + (m + 2));
    }
    return __ldg(A.f_s + base + (int64_t)l * A.s2 + m);
}

// pair (m, m+1), m even
__device__ __forceinline__ double2 f2_at(const StageArgs2& A, int i, int k, int l, int m) {
    if (l >= 0 && l < A.nvx && m >= 0 && m + 1 < A.nvy) {
        i = (i < 0) ? i + A.nx : (i >= A.nx ? i - A.nx : i);
        k = (k < 0) ? k + A.ny : (k >= A.ny ? k - A.ny : k);
        return __ldg(reinterpret_cast<const double2*>(A.f_s + A.org + (int64_t)i * A.s0 + (int64_t)k * A.s1 +
                                                      (int64_t)l * A.s2 + m));
    }
    return make_double2(f_at(A, i, k, l, m), f_at(A, i, k, l, m + 1));
}

// Unconditional 16-byte load of the pair (m, m+1) at clamped velocity indices (always a valid
// interior address, so the loads of a row step issue back to back); `fix` tells whether the pair
// holds ghost values that must be recomputed with f_at (rare: velocity-boundary threads only).
__device__ __forceinline__ double2 ld2(const StageArgs2& A, int i, int k, int l, int m, bool& fix) {
    fix = (l < 0) | (l >= A.nvx);            // vx ghosts: warp-uniform (whole vx line)
    i += (i < 0) ? A.nx : 0;
    i -= (i >= A.nx) ? A.nx : 0;
    k += (k < 0) ? A.ny : 0;
    k -= (k >= A.ny) ? A.ny : 0;
    const int lc = min(max(l, 0), A.nvx - 1), mc = min(max(m, 0), A.nvy - 2);
    return __ldg(reinterpret_cast<const double2*>(A.f_s + A.org + (int64_t)i * A.s0 + (int64_t)k * A.s1 +
                                                  (int64_t)lc * A.s2 + mc));
}

// vx-ghost pair through the characteristic boundary condition: out of line (rare, warp-uniform
// path) so that the unrolled row steps stay small enough for the instruction cache
__device__ __noinline__ double2 fix_pair(const StageArgs2& A, int i, int k, int l, int m) {
    return make_double2(f_at(A, i, k, l, m), f_at(A, i, k, l, m + 1));
}

// a batch of N pair loads (i, k[n], l[n], m[n]) followed by the ghost fix-up
template <int N>
__device__ __forceinline__ void ld2_batch(const StageArgs2& A, int i, const int (&k)[N], const int (&l)[N],
                                          const int (&m)[N], double2 (&out)[N]) {
    bool fix[N];
#pragma unroll
    for (int n = 0; n < N; ++n) out[n] = ld2(A, i, k[n], l[n], m[n], fix[n]);
#pragma unroll
    for (int n = 0; n < N; ++n)
        if (fix[n]) out[n] = fix_pair(A, i, k[n], l[n], m[n]);
}

// vy ghosts of a line triple (pl, pc, ph) = pairs at (m0-2, m0), (m0, m0+1), (m0+2, m0+3) of line
// (i, k, l): the edge lanes replace pl (m0 == 0) or ph (m0 + 2 == nvy) by the characteristic
// condition with a = -E_y(i, k) (warp-uniform), from the interior values they hold already.
__device__ __forceinline__ void vy_fix(const StageArgs2& A, int i, int k, int l, int m0, double2& pl, const double2& pc,
                                       double2& ph) {
    const bool lo = (m0 == 0), hi = (m0 + 2 == A.nvy);
    if (!(lo || hi)) return;
    i += (i < 0) ? A.nx : 0;
    i -= (i >= A.nx) ? A.nx : 0;
    k += (k < 0) ? A.ny : 0;
    k -= (k >= A.ny) ? A.ny : 0;
    const int nyg = A.ny + 4;
    const double a = -__ldg(A.E_bc + (int64_t)(A.nx + 4) * nyg + (int64_t)(i + 2) * nyg + (k + 2));
    const double* prof = A.f0v + (int64_t)(l + 2) * (A.nvy + 4);
    if (lo) {
        if (a < 0.0) {
            const double f0 = pc.x, f1 = pc.y, f2 = ph.x, f3 = ph.y;
            pl = make_double2(10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3, 4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3);
        } else {
            pl = make_double2(__ldg(prof + 0), __ldg(prof + 1));
        }
    }
    if (hi) {
        if (a > 0.0) {
            const double f0 = pc.y, f1 = pc.x, f2 = pl.y, f3 = pl.x;
            ph = make_double2(4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3, 10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3);
        } else {
            ph = make_double2(__ldg(prof + A.nvy + 2), __ldg(prof + A.nvy + 3));
        }
    }
}

template <int STAGE, int RECON>
__global__ void __launch_bounds__(128, STAGE2D_MINB) k_stage_2d2v(const StageArgs2 A) {
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int m0 = 2 * (blockIdx.x * 32 + tx);
    const int l = blockIdx.y * 4 + ty;
    const int k = blockIdx.z % A.ny;
    const int strip = blockIdx.z / A.ny;
    const int x0 = (int)((int64_t)A.nx * strip / A.nstrips);
    const int x1 = (int)((int64_t)A.nx * (strip + 1) / A.nstrips);
    const bool act = (m0 < A.nvy) && (l < A.nvx);
    const int mc = act ? m0 : 0, lc = (l < A.nvx) ? l : 0;     // clamped for inactive threads
    const int nyg = A.ny + 4;
    const int64_t ecomp = (int64_t)(A.nx + 4) * nyg;
    auto Ex = [&](int i, int kk) { return __ldg(A.E + (int64_t)(i + 2) * nyg + (kk + 2)); };
    auto Ey = [&](int i, int kk) { return __ldg(A.E + ecomp + (int64_t)(i + 2) * nyg + (kk + 2)); };
    // per-thread constant load offsets (doubles): y lines k-2..k+2 (periodic), vx lines l-2..l+2
    // (clamped: out-of-range lines are recomputed by the boundary condition), vy pairs
    int ko[5];                       // 32-bit offsets: one block of a C5-sized level is < 2^31 doubles
    int lo5[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        int kk = k - 2 + d;
        kk += (kk < 0) ? A.ny : 0;
        kk -= (kk >= A.ny) ? A.ny : 0;
        ko[d] = kk * (int)A.s1;
        lo5[d] = min(max(lc - 2 + d, 0), A.nvx - 1) * (int)A.s2;
    }
    const int mlo = max(mc - 2, 0), mhi = min(mc + 2, A.nvy - 2);
    const bool l_edge = (lc < 2) || (lc + 2 >= A.nvx);            // warp-uniform
    const bool m_edge = (mc == 0) || (mc + 2 == A.nvy);            // lanes at the vy boundary
    const double* fbase = A.f_s + A.org;
    auto P = [&](const double* rowp, int d, int e, int m) {
        return __ldg(reinterpret_cast<const double2*>(rowp + (ko[d] + lo5[e] + m)));
    };
    auto rowptr = [&](int r) {
        r += (r < 0) ? A.nx : 0;
        r -= (r >= A.nx) ? A.nx : 0;
        return fbase + (int64_t)r * A.s0;
    };
    const double vbx = A.vx_lo + ((double)lc + 0.5) * A.hvx;
    const double vbxm = vbx - A.hvx, vbxp = vbx + A.hvx;
    double vby[4];                                     // m0-1 .. m0+2
#pragma unroll
    for (int a = 0; a < 4; ++a) vby[a] = A.vy_lo + ((double)(mc + a - 1) + 0.5) * A.hvy;
    const double rdx = 1.0 / A.hx, rdy = 1.0 / A.hy, rdvx = 1.0 / A.hvx, rdvy = 1.0 / A.hvy;
    const double dvx24 = A.hvx * (1.0 / 24.0), dvy24 = A.hvy * (1.0 / 24.0);

    double W[4][3][2];        // f rows (mod 4) at vx lines l-1, l, l+1, vy m0, m0+1
    double VX[4][2][2];       // vx-face averages (rows mod 4) at l-1/2, l+1/2
    double VY[4][3];          // vy-face averages (rows mod 4) at m0-1/2, m0+1/2, m0+3/2
    double Fxp[2] = {0.0, 0.0};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int b = 0; b < 3; ++b) { W[a][b][0] = W[a][b][1] = 0.0; VY[a][b] = 0.0; }
        VX[a][0][0] = VX[a][0][1] = VX[a][1][0] = VX[a][1][1] = 0.0;
    }
    const int Q = (x1 - x0) + 4;
    for (int q0 = 0; q0 < Q; q0 += 4) {
#pragma unroll
        for (int K = 0; K < 4; ++K) {
            const int q = q0 + K;
            if (q < Q) {
                const int r = x0 - 2 + q;
                // ---- row r: x-window, vx-faces, vy-faces
                const double* rp = rowptr(r);
                double2 c01 = P(rp, 2, 2, mlo), c23 = P(rp, 2, 2, mc), c45 = P(rp, 2, 2, mhi);
                double2 am1 = P(rp, 2, 1, mc), ap1 = P(rp, 2, 3, mc), am2 = P(rp, 2, 0, mc), ap2 = P(rp, 2, 4, mc);
                if (l_edge) {
                    if (lc - 2 < 0) am2 = fix_pair(A, r, k, lc - 2, mc);
                    if (lc - 1 < 0) am1 = fix_pair(A, r, k, lc - 1, mc);
                    if (lc + 1 >= A.nvx) ap1 = fix_pair(A, r, k, lc + 1, mc);
                    if (lc + 2 >= A.nvx) ap2 = fix_pair(A, r, k, lc + 2, mc);
                }
                if (m_edge) vy_fix(A, r, k, lc, mc, c01, c23, c45);
                W[K][0][0] = am1.x; W[K][0][1] = am1.y;
                W[K][1][0] = c23.x; W[K][1][1] = c23.y;
                W[K][2][0] = ap1.x; W[K][2][1] = ap1.y;
                {
                    const double ax = -Ex(r, k);
                    VX[K][0][0] = face_avg<RECON>(am2.x, am1.x, c23.x, ap1.x, ax);
                    VX[K][0][1] = face_avg<RECON>(am2.y, am1.y, c23.y, ap1.y, ax);
                    VX[K][1][0] = face_avg<RECON>(am1.x, c23.x, ap1.x, ap2.x, ax);
                    VX[K][1][1] = face_avg<RECON>(am1.y, c23.y, ap1.y, ap2.y, ax);
                    const double ay = -Ey(r, k);
                    VY[K][0] = face_avg<RECON>(c01.x, c01.y, c23.x, c23.y, ay);
                    VY[K][1] = face_avg<RECON>(c01.y, c23.x, c23.y, c45.x, ay);
                    VY[K][2] = face_avg<RECON>(c23.x, c23.y, c45.x, c45.y, ay);
                }
                const int R0 = (K + 1) & 3, R1 = (K + 2) & 3, R2 = (K + 3) & 3;   // rows r-3, r-2, r-1
                if (q >= 3) {
                    // x-faces at (r-2)+1/2 from rows r-3..r, lines l-1, l, l+1
                    double XF[3][2];
#pragma unroll
                    for (int b = 0; b < 3; ++b)
#pragma unroll
                        for (int mm = 0; mm < 2; ++mm)
                            XF[b][mm] = face_avg<RECON>(W[R0][b][mm], W[R1][b][mm], W[R2][b][mm], W[K][b][mm],
                                                        b == 0 ? vbxm : (b == 1 ? vbx : vbxp));
                    double Fxn[2];
#pragma unroll
                    for (int mm = 0; mm < 2; ++mm) Fxn[mm] = vbx * XF[1][mm] + dvx24 * (XF[2][mm] - XF[0][mm]);
                    if (q >= 4) {
                        const int i = r - 2;
                        // ---- y-faces at (i, k -+ 1/2) for vy m0-1 .. m0+2
                        // loads of row i: lines k-2..k+2 at (l, m0-2..m0+3), lines k-+1 at l-+1, l-+2
                        const double* ip = rowptr(i);
                        double2 yy[23];
#pragma unroll
                        for (int d = 0; d < 5; ++d) {
                            yy[3 * d] = P(ip, d, 2, mlo);
                            yy[3 * d + 1] = P(ip, d, 2, mc);
                            yy[3 * d + 2] = P(ip, d, 2, mhi);
                        }
#pragma unroll
                        for (int sg = 0; sg < 2; ++sg) {          // lines k-1 (sg 0), k+1 (sg 1) at l-1, l+1, l-2, l+2
                            const int d = sg ? 3 : 1;
                            yy[15 + 4 * sg] = P(ip, d, 1, mc);
                            yy[16 + 4 * sg] = P(ip, d, 3, mc);
                            yy[17 + 4 * sg] = P(ip, d, 0, mc);
                            yy[18 + 4 * sg] = P(ip, d, 4, mc);
                        }
                        if (l_edge) {
#pragma unroll
                            for (int sg = 0; sg < 2; ++sg) {
                                const int kk = k + (sg ? 1 : -1);
                                if (lc - 1 < 0) yy[15 + 4 * sg] = fix_pair(A, i, kk, lc - 1, mc);
                                if (lc + 1 >= A.nvx) yy[16 + 4 * sg] = fix_pair(A, i, kk, lc + 1, mc);
                                if (lc - 2 < 0) yy[17 + 4 * sg] = fix_pair(A, i, kk, lc - 2, mc);
                                if (lc + 2 >= A.nvx) yy[18 + 4 * sg] = fix_pair(A, i, kk, lc + 2, mc);
                            }
                        }
                        if (m_edge) {
#pragma unroll
                            for (int d = 0; d < 5; ++d) vy_fix(A, i, k - 2 + d, lc, mc, yy[3 * d], yy[3 * d + 1], yy[3 * d + 2]);
                        }
                        double y[5][4];
#pragma unroll
                        for (int d = 0; d < 5; ++d) {
                            const double2 pl = yy[3 * d], pc = yy[3 * d + 1], ph = yy[3 * d + 2];
                            y[d][0] = pl.y; y[d][1] = pc.x; y[d][2] = pc.y; y[d][3] = ph.x;
                        }
                        double YL[4], YH[4];
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            YL[a] = face_avg<RECON>(y[0][a], y[1][a], y[2][a], y[3][a], vby[a]);
                            YH[a] = face_avg<RECON>(y[1][a], y[2][a], y[3][a], y[4][a], vby[a]);
                        }
                        // ---- y-transverse velocity-face averages at (i, k -+ 1)
                        double VXk[2][2][2], VYk[2][3];
#pragma unroll
                        for (int sgn = 0; sgn < 2; ++sgn) {
                            const int kk = k + (sgn ? 1 : -1);
                            const int yb = sgn ? 9 : 3, nb = sgn ? 19 : 15;
                            const double2 b01 = yy[yb], b23 = yy[yb + 1], b45 = yy[yb + 2];
                            const double2 bm1 = yy[nb], bp1 = yy[nb + 1], bm2 = yy[nb + 2], bp2 = yy[nb + 3];
                            const double ax = -Ex(i, kk), ay = -Ey(i, kk);
                            VXk[sgn][0][0] = face_avg<RECON>(bm2.x, bm1.x, b23.x, bp1.x, ax);
                            VXk[sgn][0][1] = face_avg<RECON>(bm2.y, bm1.y, b23.y, bp1.y, ax);
                            VXk[sgn][1][0] = face_avg<RECON>(bm1.x, b23.x, bp1.x, bp2.x, ax);
                            VXk[sgn][1][1] = face_avg<RECON>(bm1.y, b23.y, bp1.y, bp2.y, ax);
                            VYk[sgn][0] = face_avg<RECON>(b01.x, b01.y, b23.x, b23.y, ay);
                            VYk[sgn][1] = face_avg<RECON>(b01.y, b23.x, b23.y, b45.x, ay);
                            VYk[sgn][2] = face_avg<RECON>(b23.x, b23.y, b45.x, b45.y, ay);
                        }
                        const double exi = Ex(i, k), eyi = Ey(i, k);
                        const double cxi = (Ex(i + 1, k) - Ex(i - 1, k)) * (1.0 / 48.0);
                        const double cxk = (Ex(i, k + 1) - Ex(i, k - 1)) * (1.0 / 48.0);
                        const double cyi = (Ey(i + 1, k) - Ey(i - 1, k)) * (1.0 / 48.0);
                        const double cyk = (Ey(i, k + 1) - Ey(i, k - 1)) * (1.0 / 48.0);
                        double Fvy[3];
#pragma unroll
                        for (int fc = 0; fc < 3; ++fc)
                            Fvy[fc] = eyi * VY[R1][fc] + cyi * (VY[R2][fc] - VY[R0][fc]) +
                                      cyk * (VYk[1][fc] - VYk[0][fc]);
                        double o[2];
                        const double* fnp = A.f_n + A.org + (int64_t)i * A.s0 + (int64_t)k * A.s1 + (int64_t)lc * A.s2 + mc;
                        double2 fn = make_double2(0.0, 0.0), uu = make_double2(0.0, 0.0);
                        if (STAGE >= 2 && act) fn = *reinterpret_cast<const double2*>(fnp);
                        if (STAGE == 4 && act)
                            uu = *reinterpret_cast<const double2*>(A.u_in + (fnp - A.f_n));
                        double un[2];
#pragma unroll
                        for (int mm = 0; mm < 2; ++mm) {
                            const double Fvxl = exi * VX[R1][0][mm] + cxi * (VX[R2][0][mm] - VX[R0][0][mm]) +
                                                cxk * (VXk[1][0][mm] - VXk[0][0][mm]);
                            const double Fvxh = exi * VX[R1][1][mm] + cxi * (VX[R2][1][mm] - VX[R0][1][mm]) +
                                                cxk * (VXk[1][1][mm] - VXk[0][1][mm]);
                            const double Fyl = vby[mm + 1] * YL[mm + 1] + dvy24 * (YL[mm + 2] - YL[mm]);
                            const double Fyh = vby[mm + 1] * YH[mm + 1] + dvy24 * (YH[mm + 2] - YH[mm]);
                            double kk = -(Fxn[mm] - Fxp[mm]) * rdx;
                            kk = kk - (Fyh - Fyl) * rdy;
                            kk = kk + (Fvxh - Fvxl) * rdvx;
                            kk = kk + (Fvy[mm + 1] - Fvy[mm]) * rdvy;
                            const double fs = W[R1][1][mm];
                            const double fnm = mm ? fn.y : fn.x, um = mm ? uu.y : uu.x;
                            if (STAGE == 0) {
                                o[mm] = kk;
                            } else if (STAGE == 1) {
                                o[mm] = fs + (0.5 * A.dt) * kk;
                            } else if (STAGE == 2) {
                                un[mm] = fnm + (fs - fnm) * (1.0 / 3.0) + (A.dt * (1.0 / 3.0)) * kk;
                                o[mm] = fnm + (0.5 * A.dt) * kk;
                            } else if (STAGE == 3) {
                                o[mm] = fnm + A.dt * kk;
                            } else {
                                o[mm] = um + (fs - fnm) * (1.0 / 3.0) + (A.dt * (1.0 / 6.0)) * kk;
                            }
                        }
                        if (act) {
                            const int64_t off = fnp - A.f_n;
                            *reinterpret_cast<double2*>(A.f_next + off) = make_double2(o[0], o[1]);
                            if (STAGE == 2) *reinterpret_cast<double2*>(A.u_out + off) = make_double2(un[0], un[1]);
                        }
                        if (A.partials != nullptr) {
                            double s = act ? (o[0] + o[1]) : 0.0;
#pragma unroll
                            for (int of = 16; of > 0; of >>= 1) s += __shfl_xor_sync(0xffffffffu, s, of);
                            if (tx == 0 && l < A.nvx) {
                                const int nmt = gridDim.x;
                                A.partials[((int64_t)l * nmt + blockIdx.x) * A.nx * A.ny + (int64_t)i * A.ny + k] = s;
                            }
                        }
                    }
                    Fxp[0] = Fxn[0];
                    Fxp[1] = Fxn[1];
                }
            }
        }
    }
}

// rho[i][k] = 1 - dvx dvy sum_p partials[p][i][k]  (fixed order: deterministic)
__global__ void k_moment_2d2v_finish(const double* __restrict__ partials, int np, int ncfg, double dvv,
                                     double* __restrict__ rho) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncfg) return;
    double s = 0.0;
    for (int p = 0; p < np; ++p) s += partials[(int64_t)p * ncfg + t];
    rho[t] = 1.0 - dvv * s;
}

// rho from a stored state (one warp per configuration cell)
__global__ void k_moment_2d2v_direct(const double* __restrict__ f, int64_t org, int64_t s0, int64_t s1, int64_t s2,
                                     int nx, int ny, int nvx, int nvy, double dvv, double* __restrict__ rho) {
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= nx * ny) return;
    const int i = c / ny, k = c % ny;
    const double* p = f + org + (int64_t)i * s0 + (int64_t)k * s1;
    double s = 0.0;
    for (int l = 0; l < nvx; ++l)
        for (int m = lane; m < nvy; m += 32) s += p[(int64_t)l * s2 + m];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) rho[c] = 1.0 - dvv * s;
}

template <int RECON>
static int dispatch2(int stage, const StageArgs2& A, dim3 grid, cudaStream_t st) {
    const dim3 block(32, 4);
    switch (stage) {
        case 0: k_stage_2d2v<0, RECON><<<grid, block, 0, st>>>(A); break;
        case 1: k_stage_2d2v<1, RECON><<<grid, block, 0, st>>>(A); break;
        case 2: k_stage_2d2v<2, RECON><<<grid, block, 0, st>>>(A); break;
        case 3: k_stage_2d2v<3, RECON><<<grid, block, 0, st>>>(A); break;
        case 4: k_stage_2d2v<4, RECON><<<grid, block, 0, st>>>(A); break;
        default: return fail(VLASOV_EINVAL, "stage must be 0..4");
    }
    VK_LAUNCH("k_stage_2d2v");
    return VLASOV_OK;
}

int launch_stage_2d2v(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s, double* u,
                      double* f_next, const double* E, const double* E_bc, const double* f0v, int recon,
                      double* rho) {
    StageArgs2 A;
    A.f_s = f_s;
    A.f_n = f_n;
    A.u_in = u;
    A.u_out = u;
    A.f_next = f_next;
    A.E = E;
    A.E_bc = E_bc;
    A.f0v = f0v;
    A.s0 = L->block_str[0][0];
    A.s1 = L->block_str[0][1];
    A.s2 = L->block_str[0][2];
    A.org = L->block_off[0] + vk::G * (A.s0 + A.s1 + A.s2 + 1);
    A.nx = L->dom[0];
    A.ny = L->dom[1];
    A.nvx = L->dom[2];
    A.nvy = L->dom[3];
    A.dt = dt;
    A.hx = L->h[0];
    A.hy = L->h[1];
    A.hvx = L->h[2];
    A.hvy = L->h[3];
    A.vx_lo = L->lower[2];
    A.vy_lo = L->lower[3];
    const int nmt = (A.nvy / 2 + 31) / 32, nlg = (A.nvx + 3) / 4;
    A.nstrips = L->strips2;
    A.nrows = (A.nx + A.nstrips - 1) / A.nstrips;
    A.partials = rho ? L->d_partials : nullptr;
    const dim3 grid(nmt, nlg, A.ny * A.nstrips);
    int rc = recon == VLASOV_UPWIND ? dispatch2<VLASOV_UPWIND>(stage, A, grid, L->stream)
                                    : dispatch2<VLASOV_CENTERED4>(stage, A, grid, L->stream);
    if (rc || !rho) return rc;
    const int ncfg = A.nx * A.ny;
    k_moment_2d2v_finish<<<(ncfg + 127) / 128, 128, 0, L->stream>>>(L->d_partials, A.nvx * nmt, ncfg,
                                                                     A.hvx * A.hvy, rho);
    VK_LAUNCH("k_moment_2d2v_finish");
    return VLASOV_OK;
}

int launch_moment_2d2v(const vlasov_level* L, const double* f, double* rho) {
    const int64_t s0 = L->block_str[0][0], s1 = L->block_str[0][1], s2 = L->block_str[0][2];
    const int64_t org = L->block_off[0] + vk::G * (s0 + s1 + s2 + 1);
    const int ncfg = L->dom[0] * L->dom[1];
    k_moment_2d2v_direct<<<(ncfg + 7) / 8, 256, 0, L->stream>>>(f, org, s0, s1, s2, L->dom[0], L->dom[1], L->dom[2],
                                                                L->dom[3], L->h[2] * L->h[3], rho);
    VK_LAUNCH("k_moment_2d2v_direct");
    return VLASOV_OK;
}

}  // namespace vk
