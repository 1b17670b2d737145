// 2D+2V fused RK4 stage for CENTERED4 in telescoped form (BASELINE.json C5): the flux divergence
// of P:246-250 with the face averages of P:344-345 and the fluxes of P:263-282 (generalised
// dimension by dimension as in oracle/scheme.py), evaluated through the identity
//
//   12 (<g>_{d+1/2} - <g>_{d-1/2}) = D_d g := g_{-2} - 8 g_{-1} + 8 g_{+1} - g_{+2}
//
// (CENTERED4 face average 12<g>_{d+1/2} = 7(g_0 + g_1) - (g_{-1} + g_2)).  Since each flux is a
// face average of f times coefficients that are constant along the face's normal direction, the
// divergence of every flux is D_d of a cell-centred "pre-field":
//
//   x  : -(1/12hx)  [vx D_x f + (hvx/24) D_x d_vx f]     = bx D_x P,  P = rx f + d_vx f
//   y  : -(1/12hy)  [vy D_y f + (hvy/24) D_y d_vy f]     = by D_y Q,  Q = ry f + d_vy f
//   vx : +(1/12hvx) [Ex D_vx f + (dEx^x/48) d_x D_vx f + (dEx^y/48) d_y D_vx f]
//   vy : +(1/12hvy) [Ey D_vy f + (dEy^x/48) d_x D_vy f + (dEy^y/48) d_y D_vy f]
//
// with d_d g = g_{+1} - g_{-1}, rx = 24 vx/hvx, bx = -hvx/(288 hx) (same for y), and the velocity
// coefficients (E and its centred differences, reading #3's +1/48) taken at the cell's (x, y).
// This is the same linear map as faces -> fluxes -> divergence, equal in exact arithmetic; it
// needs ~37 fp64 operations per cell instead of ~105 and, with two y lines per thread, about half
// the shared-memory traffic of the face form (k_stage_2d2v, kept for UPWIND).  A constant f gives
// k == 0 bitwise (every D_d and d_d of equal values is an exact zero).
//
// Layout: [x][y][vx][vy], vy contiguous, ghost frame 2; the velocity ghost frame of f_s is derived
// before the stage by k_vghost_2d2v (characteristic condition, reading #6); x, y periodic by
// coordinates.  CTA = two y lines k0, k0+1 (in every thread), 4 vx lines l0..l0+3 (one consumer
// warp each), a vy tile of 64 cells (2 per lane), marching along x over a strip; a producer
// warpgroup (one lane issues) streams per row step into a shared-memory ring with TMA tensor
// copies (cp.async.bulk.tensor.4d):
//   A   row r,     y = k0, k0+1,   vx l0-2 .. l0+5   (P, D_vx f, D_vy f, Q, f of the own lines)
//   B   row i,     y = k0-1, k0+2, vx l0-2 .. l0+5   (D_vx f, D_vy f, Q of the y neighbours)
//   C   row i,     y = k0-2, k0+3, vx l0 .. l0+3     (Q for D_y)
//   F   row i,     y = k0, k0+1,   vx l0 .. l0+3     (f_n in stages 2-3, u in stage 4: RK4 combine)
// with output row i = r - 2.  Own-line quantities are kept in register windows along x (the
// x-differences come from the window).  Per-(x, y) velocity coefficients are tabulated in shared
// memory at kernel start.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <type_traits>

#include "internal.h"
#include "ptx.cuh"

namespace vk {

constexpr int T2_LT = 4;                    // vx lines (consumer warps) per CTA
constexpr int T2_TM = 64;                   // vy cells per tile (2 per lane)
constexpr int T2_LW = T2_TM + 4;            // doubles per line segment
constexpr int T2_THREADS = 256;             // 4 consumer warps + producer warpgroup
constexpr int T2_RMAX = 64;                 // rows per strip (coefficient table capacity)
constexpr int T2_SMAX = 16;                 // strips along x
// slot layout (doubles); every part offset is a multiple of 16 doubles (128-B TMA destinations)
constexpr int T2_A = 0;                     // [2 y][8 vx][68]
constexpr int T2_B0 = 16 * T2_LW;           // [8][68]
constexpr int T2_B1 = 24 * T2_LW;           // [8][68]
constexpr int T2_C0 = 32 * T2_LW;           // [4][68]
constexpr int T2_C1 = 36 * T2_LW;           // [4][68]
constexpr int T2_F = 40 * T2_LW;            // [2][4][64]
constexpr int T2_FU = 2 * T2_LT * T2_TM;    // doubles of one F or U part

template <int STAGE>
struct SlotT {
    static constexpr int NFU = STAGE >= 2 ? 1 : 0;                             // f_n (stages 2, 3) or u (stage 4)
    static constexpr int SIZE = T2_F + NFU * T2_FU;                           // doubles
    static constexpr int NSLOT = STAGE == 4 ? 3 : 4;                          // 2 CTAs per SM
    static constexpr size_t smem_bytes() { return ((size_t)NSLOT * SIZE + 16 * T2_RMAX) * sizeof(double); }
};

struct TMapsT {
    CUtensorMap a;      // f_s, box (68 vy, 8 vx, 2 y)
    CUtensorMap b;      // f_s, box (68, 8, 1)
    CUtensorMap c;      // f_s, box (68, 4, 1)
    CUtensorMap fn;     // f_n, box (64, 4, 2)
    CUtensorMap u;      // u,   box (64, 4, 2)
};

struct StageArgsT {
    double* u_out;
    double* f_next;
    const double* E;           // [2][(nx+4)(ny+4)] ghosted level field
    double* partials;          // [nvx * nmt][nx][ny] moment partials (nullable)
    int64_t s0, s1, s2, org;
    int nx, ny, nvx, nvy, nmt, nstrips;
    int xb[T2_SMAX + 1];       // strip s covers rows xb[s] .. xb[s+1]-1 (strip lengths may differ)
    double hx, hy, hvx, hvy, vx_lo, vy_lo;
    double sc;                 // stage factor of k (0.5 dt, 0.5 dt, dt, dt/6; 1 for STAGE 0)
};

__device__ __forceinline__ int wrapt(int i, int n) {
    i += (i < 0) ? n : 0;
    i -= (i >= n) ? n : 0;
    return i;
}

// D g = g_{-2} - 8 g_{-1} + 8 g_{+1} - g_{+2}, given t = g_{+1} - g_{-1}
__device__ __forceinline__ double dtel(double gm2, double gp2, double t) { return fma(8.0, t, gm2 - gp2); }

template <int STAGE>
__global__ void __launch_bounds__(T2_THREADS, 2) k_stage_2d2v_tel(const StageArgsT A, const __grid_constant__ TMapsT M) {
    using SL = SlotT<STAGE>;
    constexpr int SIZE = SL::SIZE, NSLOT = SL::NSLOT;
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full_bar[NSLOT];
    __shared__ __align__(8) uint64_t empty_bar[NSLOT];
    __shared__ uint32_t s_dep[32 * T2_LT];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int b = blockIdx.x;
    const int mt = b % A.nmt;
    b /= A.nmt;
    const int nlt = A.nvx / T2_LT;
    const int l0 = (b % nlt) * T2_LT;
    b /= nlt;
    const int k0 = 2 * (b % (A.ny / 2));
    const int strip = b / (A.ny / 2);
    const int x0 = A.nstrips <= T2_SMAX ? A.xb[strip] : (int)((int64_t)A.nx * strip / A.nstrips);
    const int x1 = A.nstrips <= T2_SMAX ? A.xb[strip + 1] : (int)((int64_t)A.nx * (strip + 1) / A.nstrips);
    const int rows = x1 - x0, Q = rows + 4;
    const int ncols = min(T2_TM, A.nvy - mt * T2_TM);
    const int nyg = A.ny + 4;
    const int64_t ecomp = (int64_t)(A.nx + 4) * nyg;

    if (tid == 0) {
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], T2_LT);
        }
        fence_mbar_init();
    }
    griddep_wait();
    // velocity coefficients per (output row j, y): {gx, hx, px, gy, hy, py} (x stage factor)
    double* cE = smem + NSLOT * SIZE;                                     // [rows][2][8]
    {
        const double cg = A.sc / 12.0, cdx = A.sc / (576.0 * A.hvx), cdy = A.sc / (576.0 * A.hvy);
        for (int t = tid; t < 2 * rows; t += blockDim.x) {
            const int j = t >> 1, y = t & 1;
            const int i = wrapt(x0 + j, A.nx), k = k0 + y;
            const int im = wrapt(i - 1, A.nx), ip = wrapt(i + 1, A.nx);
            const int km = wrapt(k - 1, A.ny), kp = wrapt(k + 1, A.ny);
            auto ex = [&](int c, int ii, int kk) { return __ldg(A.E + c * ecomp + (int64_t)(ii + 2) * nyg + (kk + 2)); };
            double* o = cE + 8 * t;
            o[0] = ex(0, i, k) * (cg / A.hvx);
            o[1] = (ex(0, ip, k) - ex(0, im, k)) * cdx;
            o[2] = (ex(0, i, kp) - ex(0, i, km)) * cdx;
            o[3] = ex(1, i, k) * (cg / A.hvy);
            o[4] = (ex(1, ip, k) - ex(1, im, k)) * cdy;
            o[5] = (ex(1, i, kp) - ex(1, i, km)) * cdy;
        }
    }
    __syncthreads();

    if (warp >= T2_LT) {                                                   // ---------------- producer
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(24));
        if (warp == T2_LT && lane == 0) {
            constexpr uint32_t BA = 16 * T2_LW * 8, BB = 8 * T2_LW * 8, BC = 4 * T2_LW * 8, BF = T2_FU * 8;
            const int cm = mt * T2_TM;                                     // ghosted vy coord of m = mt*TM - 2
            const int ym1 = wrapt(k0 - 1, A.ny) + 2, yp2 = wrapt(k0 + 2, A.ny) + 2;
            const int ym2 = wrapt(k0 - 2, A.ny) + 2, yp3 = wrapt(k0 + 3, A.ny) + 2;
            int slot = 0;
            uint32_t phase = 0;
            for (int q = 0; q < Q; ++q) {
                if (q >= NSLOT) mbar_wait(&empty_bar[slot], phase ^ 1u);
                const bool out_row = q >= 4;
                const int r = wrapt(x0 - 2 + q, A.nx) + 2, i = wrapt(x0 - 4 + q, A.nx) + 2;
                double* dst = smem + slot * SIZE;
                uint64_t* fb = &full_bar[slot];
                mbar_arrive_expect_tx(fb, out_row ? BA + 2 * BB + 2 * BC + SL::NFU * BF : BA);
                tma_load_4d(dst + T2_A, &M.a, cm, l0, k0 + 2, r, fb);
                if (out_row) {
                    tma_load_4d(dst + T2_B0, &M.b, cm, l0, ym1, i, fb);
                    tma_load_4d(dst + T2_B1, &M.b, cm, l0, yp2, i, fb);
                    tma_load_4d(dst + T2_C0, &M.c, cm, l0 + 2, ym2, i, fb);
                    tma_load_4d(dst + T2_C1, &M.c, cm, l0 + 2, yp3, i, fb);
                    if (STAGE == 2 || STAGE == 3) tma_load_4d(dst + T2_F, &M.fn, cm + 2, l0 + 2, k0 + 2, i, fb);
                    if (STAGE == 4) tma_load_4d(dst + T2_F, &M.u, cm + 2, l0 + 2, k0 + 2, i, fb);
                }
                if (++slot == NSLOT) { slot = 0; phase ^= 1u; }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(232));
    const int w = warp, l = l0 + w;
    const int cl = 2 * lane + 2;                                          // slot column of my first cell
    const int m0 = mt * T2_TM + 2 * lane;
    const bool act = 2 * lane < ncols;
    const double rx = 24.0 * (A.vx_lo + ((double)l + 0.5) * A.hvx) / A.hvx;
    const double ry0 = 24.0 * (A.vy_lo + ((double)m0 + 0.5) * A.hvy) / A.hvy;
    const double ry1 = 24.0 * (A.vy_lo + ((double)m0 + 1.5) * A.hvy) / A.hvy;
    const double bx = -A.sc * A.hvx / (288.0 * A.hx), by = -A.sc * A.hvy / (288.0 * A.hy);

    // register windows along x (row slot = row mod 4), per own y line and vy cell
    double PW[4][2][2];       // P = rx f + d_vx f
    double DL[4][2][2];       // D_vx f
    double DM[4][2][2];       // D_vy f
    double QW[4][2][2];       // Q = ry f + d_vy f
    double FW[4][2][2];       // f
    int slot = 0;
    uint32_t phase = 0;

    // pre-fields of one line segment at column cl: D_vx f, D_vy f, Q (and P, f for own lines)
    auto line_fields = [&](const double* Ln, double& dl0, double& dl1, double& dm0, double& dm1, double& q0,
                           double& q1, double* p, double2* f, uint32_t& dep) {
        const double2 c01 = lds2(Ln + cl - 2), c23 = lds2(Ln + cl), c45 = lds2(Ln + cl + 2);
        const double2 lm1 = lds2(Ln - T2_LW + cl), lp1 = lds2(Ln + T2_LW + cl);
        const double2 lm2 = lds2(Ln - 2 * T2_LW + cl), lp2 = lds2(Ln + 2 * T2_LW + cl);
        const double t0 = lp1.x - lm1.x, t1 = lp1.y - lm1.y;
        dl0 = dtel(lm2.x, lp2.x, t0);
        dl1 = dtel(lm2.y, lp2.y, t1);
        const double d0 = c23.y - c01.y, d1 = c45.x - c23.x;               // d_vy f at m0, m0+1
        dm0 = fma(8.0, d0, c01.x - c45.x);
        dm1 = fma(8.0, d1, c01.y - c45.y);
        q0 = fma(ry0, c23.x, d0);
        q1 = fma(ry1, c23.y, d1);
        if (p) {
            p[0] = fma(rx, c23.x, t0);
            p[1] = fma(rx, c23.y, t1);
            *f = c23;
        }
        dep ^= __double2hiint(dl0) ^ __double2hiint(dm0);                 // depends on every load above
    };

    auto row = [&](auto Kc, auto OUTc, int q, bool live, double (&rs)[2]) {
        constexpr int K = decltype(Kc)::value;
        constexpr bool OUT = decltype(OUTc)::value;
        constexpr int RM = (K + 1) & 3, RI = (K + 2) & 3, RP = (K + 3) & 3;   // rows i-1, i, i+1 (i = r-2)
        if (live) mbar_wait(&full_bar[slot], phase);
        const double* S = smem + slot * SIZE;
        uint32_t dep = 0;
        // ---- own lines at row r
        double Pn[2][2];
#pragma unroll
        for (int y = 0; y < 2; ++y) {
            double2 fv;
            line_fields(S + T2_A + (y * 8 + w + 2) * T2_LW, DL[K][y][0], DL[K][y][1], DM[K][y][0], DM[K][y][1],
                        QW[K][y][0], QW[K][y][1], Pn[y], &fv, dep);
            FW[K][y][0] = fv.x;
            FW[K][y][1] = fv.y;
        }
        if (OUT) {
            const int j = q - 4;
            const int i = wrapt(x0 + j, A.nx);
            // ---- y neighbours at row i
            double bl[2][2], bm[2][2], bq[2][2], cq[2][2];
            line_fields(S + T2_B0 + (w + 2) * T2_LW, bl[0][0], bl[0][1], bm[0][0], bm[0][1], bq[0][0], bq[0][1],
                        nullptr, nullptr, dep);
            line_fields(S + T2_B1 + (w + 2) * T2_LW, bl[1][0], bl[1][1], bm[1][0], bm[1][1], bq[1][0], bq[1][1],
                        nullptr, nullptr, dep);
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const double* Ln = S + (c ? T2_C1 : T2_C0) + w * T2_LW;
                const double2 c01 = lds2(Ln + cl - 2), c23 = lds2(Ln + cl), c45 = lds2(Ln + cl + 2);
                cq[c][0] = fma(ry0, c23.x, c23.y - c01.y);
                cq[c][1] = fma(ry1, c23.y, c45.x - c23.x);
                dep ^= __double2hiint(cq[c][0]) ^ __double2hiint(cq[c][1]);
            }
            double2 fn[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
            double2 uu[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
            for (int y = 0; y < 2; ++y) {
                if (STAGE == 2 || STAGE == 3) fn[y] = lds2(S + T2_F + (y * T2_LT + w) * T2_TM + 2 * lane);
                if (STAGE == 4) uu[y] = lds2(S + T2_F + (y * T2_LT + w) * T2_TM + 2 * lane);
            }
            const double* ce = cE + 16 * j;
            double o[2][2], un[2][2];
#pragma unroll
            for (int y = 0; y < 2; ++y) {
                const double2 g01 = lds2(ce + 8 * y), g23 = lds2(ce + 8 * y + 2), g45 = lds2(ce + 8 * y + 4);
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    // x: P at rows i-2, i-1, i+1, i+2 = window slot K (row r-4), RM, RP, and Pn (row r)
                    const double dxp = dtel(PW[K][y][mm], Pn[y][mm], PW[RP][y][mm] - PW[RM][y][mm]);
                    // y: Q at k-2, k-1, k+1, k+2
                    const double qm2 = y ? bq[0][mm] : cq[0][mm];
                    const double qm1 = y ? QW[RI][0][mm] : bq[0][mm];
                    const double qp1 = y ? bq[1][mm] : QW[RI][1][mm];
                    const double qp2 = y ? cq[1][mm] : bq[1][mm];
                    const double dyq = dtel(qm2, qp2, qp1 - qm1);
                    // velocity terms: D f at (i, k), its x difference (window) and y difference
                    const double dlk = (y ? bl[1][mm] : DL[RI][1][mm]) - (y ? DL[RI][0][mm] : bl[0][mm]);
                    const double dmk = (y ? bm[1][mm] : DM[RI][1][mm]) - (y ? DM[RI][0][mm] : bm[0][mm]);
                    double kk = bx * dxp;
                    kk = fma(by, dyq, kk);
                    kk = fma(g01.x, DL[RI][y][mm], kk);
                    kk = fma(g01.y, DL[RP][y][mm] - DL[RM][y][mm], kk);
                    kk = fma(g23.x, dlk, kk);
                    kk = fma(g23.y, DM[RI][y][mm], kk);
                    kk = fma(g45.x, DM[RP][y][mm] - DM[RM][y][mm], kk);
                    kk = fma(g45.y, dmk, kk);
                    // kk = sc * k; RK4 stage combine (minimum-traffic form, DESIGN 6.1)
                    const double fs = FW[RI][y][mm];
                    const double fnm = mm ? fn[y].y : fn[y].x, um = mm ? uu[y].y : uu[y].x;
                    if (STAGE == 0 || STAGE == 1) {
                        o[y][mm] = STAGE == 0 ? kk : fs + kk;
                    } else if (STAGE == 2) {
                        un[y][mm] = fma(2.0 / 3.0, kk, (fnm + fs) * (1.0 / 3.0));
                        o[y][mm] = fnm + kk;
                    } else if (STAGE == 3) {
                        o[y][mm] = fnm + kk;
                    } else {
                        o[y][mm] = fma(fs, 1.0 / 3.0, um) + kk;
                    }
                }
                dep ^= __double2hiint(o[y][0]);
            }
            if (live && act) {
#pragma unroll
                for (int y = 0; y < 2; ++y) {
                    const int64_t off = A.org + (int64_t)i * A.s0 + (int64_t)(k0 + y) * A.s1 + (int64_t)l * A.s2 + m0;
                    *reinterpret_cast<double2*>(A.f_next + off) = make_double2(o[y][0], o[y][1]);
                    if (STAGE == 2) *reinterpret_cast<double2*>(A.u_out + off) = make_double2(un[y][0], un[y][1]);
                }
            }
            rs[0] = (live && act) ? o[0][0] + o[0][1] : 0.0;
            rs[1] = (live && act) ? o[1][0] + o[1][1] : 0.0;
        }
#pragma unroll
        for (int y = 0; y < 2; ++y) {
            PW[K][y][0] = Pn[y][0];
            PW[K][y][1] = Pn[y][1];
        }
        if (live) {
            // release the slot behind a store that depends on every load of the row (shared loads
            // complete asynchronously; in-order issue holds the arrive until they have landed)
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(&s_dep[tid])), "r"(dep) : "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[slot]);
            if (++slot == NSLOT) { slot = 0; phase ^= 1u; }
        }
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    {
        double dummy[2];
        row(I0{}, std::false_type{}, 0, true, dummy);
        row(I1{}, std::false_type{}, 1, true, dummy);
        row(I2{}, std::false_type{}, 2, true, dummy);
        row(I3{}, std::false_type{}, 3, true, dummy);
    }
    for (int q0 = 4; q0 < Q; q0 += 4) {
        double rs[4][2];
        row(I0{}, std::true_type{}, q0, true, rs[0]);
        row(I1{}, std::true_type{}, q0 + 1, q0 + 1 < Q, rs[1]);
        row(I2{}, std::true_type{}, q0 + 2, q0 + 2 < Q, rs[2]);
        row(I3{}, std::true_type{}, q0 + 3, q0 + 3 < Q, rs[3]);
        if (A.partials != nullptr) {
            // warp sums of the group's 8 (row, y) values with one transposed butterfly: after the
            // xor-16/8/4 stages lane L holds value v = 4 bit4 + 2 bit3 + bit2 (row = v >> 1, y = v & 1)
            double v[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) v[t] = rs[t >> 1][t & 1];
            const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
            double h4[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const double keep = b16 ? v[t + 4] : v[t], give = b16 ? v[t] : v[t + 4];
                h4[t] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
            }
            double h2[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const double keep = b8 ? h4[t + 2] : h4[t], give = b8 ? h4[t] : h4[t + 2];
                h2[t] = keep + __shfl_xor_sync(0xffffffffu, give, 8);
            }
            double s = (b4 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, b4 ? h2[0] : h2[1], 4);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            const int vv = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
            const int qq = q0 + (vv >> 1), y = vv & 1;
            if ((lane & 3) == 0 && qq < Q) {
                const int i = wrapt(x0 - 4 + qq, A.nx);
                A.partials[((int64_t)l * A.nmt + mt) * A.nx * A.ny + (int64_t)i * A.ny + (k0 + y)] = s;
            }
        }
    }
    griddep_launch_dependents();
}

// tensor map of one field over the ghosted block of a single-block 2D+2V level, box (vy, vx, y, 1)
static int encode_map_t(const vlasov_level* L, const double* f, unsigned bvy, unsigned bvx, unsigned by,
                        CUtensorMap* out) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult qr;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn) {
            cudaGetLastError();
            return fail(VLASOV_ECUDA, "cuTensorMapEncodeTiled not available");
        }
        enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const cuuint64_t dims[4] = {(cuuint64_t)L->block_str[0][2], (cuuint64_t)(L->dom[2] + 2 * G),
                                (cuuint64_t)(L->dom[1] + 2 * G), (cuuint64_t)(L->dom[0] + 2 * G)};
    const cuuint64_t strides[3] = {(cuuint64_t)L->block_str[0][2] * 8, (cuuint64_t)L->block_str[0][1] * 8,
                                   (cuuint64_t)L->block_str[0][0] * 8};
    const cuuint32_t box[4] = {bvy, bvx, by, 1}, estr[4] = {1, 1, 1, 1};
    CUresult rc = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)(f + L->block_off[0]), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) return fail(VLASOV_ECUDA, "cuTensorMapEncodeTiled failed");
    return VLASOV_OK;
}

template <int STAGE>
static int launch_tel_t(const StageArgsT& A, const TMapsT& M, unsigned grid, cudaStream_t st) {
    auto kern = k_stage_2d2v_tel<STAGE>;
    static bool configured = false;
    if (!configured) {
        VK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SlotT<STAGE>::smem_bytes()));
        configured = true;
    }
    VK_CUDA(launch_pdl(kern, dim3(grid), dim3(T2_THREADS), SlotT<STAGE>::smem_bytes(), st, A, M));
    return VLASOV_OK;
}

bool stage_2d2v_tel_ok(const vlasov_level* L) {
    return L->dom[1] % 2 == 0 && L->dom[2] % T2_LT == 0 && L->dom[3] % 2 == 0;
}

// Strip boundaries along x.  All CTAs of a strip take the same time (rows + warm-up), and the block
// scheduler hands CTAs out in blockIdx order (strip-major) to 2 slots per SM, so the stage time is
// the makespan of that list schedule.  Equal strips quantise badly when tiles / slots is far from an
// integer (C5: 512 tiles on 296 slots = 1.73 waves); two strips of unequal length (long first) fill
// the last wave.  Candidates: ns equal strips (ns from the T2_RMAX minimum up), and for a level that
// fits one strip every split (a, nx - a); cost of a CTA = its row steps (rows + 4, rounded up to the
// unroll group of 4: the dead steps of a ragged group still execute) - 2 (the 4 warm-up rows load
// the A part only).  Measured on C5 (B200, 3 interleaved runs each, +-0.1): one strip 29.55 G
// cell-updates/s, (52,12) 31.24, (56,8) 31.46, (60,4) 30.95, (54,10) 30.0, (49,15) 29.6.  CTAs of one strip march in lockstep, so neighbouring tiles still share halo lines
// through the L2.
static double strips_makespan(const int* len, int ns, int64_t tiles, int slots) {
    std::vector<double> heap((size_t)slots, 0.0);                          // min-heap of slot end times
    auto cmp = [](double a, double b) { return a > b; };
    double end = 0.0;
    for (int s = 0; s < ns; ++s)
        for (int64_t t = 0; t < tiles; ++t) {
            std::pop_heap(heap.begin(), heap.end(), cmp);
            const double e = heap.back() + (len[s] + 4 + 3) / 4 * 4 - 2.0;   // row steps run in groups of 4
            heap.back() = e;
            std::push_heap(heap.begin(), heap.end(), cmp);
            end = std::max(end, e);
        }
    return end;
}

int stage_2d2v_choose_strips(int64_t tiles, int nx, int rmax, int smax, const char* env, int* xb) {
    static int slots = 0;
    if (!slots) {
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
            cudaGetLastError();
            sms = 148;
        }
        slots = 2 * sms;
    }
    const int nsmin = (nx + rmax - 1) / rmax;
    if (nsmin > smax) return nsmin;                                        // equal strips, bounds computed in the kernel
    std::vector<int> best_len((size_t)smax), len((size_t)smax);
    int best_ns = 0;
    double best = 0.0;
    auto consider = [&](int ns) {
        const double m = strips_makespan(len.data(), ns, tiles, slots);
        if (best_ns == 0 || m < (best_ns == nsmin ? best * 0.97 : best)) { // the default must be beaten by 3 %
            best = m;
            best_ns = ns;
            std::copy(len.begin(), len.begin() + ns, best_len.begin());
        }
    };
    auto equal = [&](int ns) {
        for (int s = 0; s < ns; ++s) len[s] = (int)((int64_t)nx * (s + 1) / ns - (int64_t)nx * s / ns);
    };
    const char* e = env ? std::getenv(env) : nullptr;                      // experiments: "ns" or "a,b,..."
    if (e && std::strchr(e, ',')) {
        int ns = 0, sum = 0;
        for (const char* p = e; ns < smax; ++p) {
            len[ns] = atoi(p);
            sum += len[ns++];
            p = std::strchr(p, ',');
            if (!p) break;
        }
        bool ok = sum == nx;
        for (int s = 0; s < ns; ++s) ok = ok && len[s] >= 1 && len[s] <= rmax;
        if (ok) consider(ns);
    } else if (e) {
        const int ns = std::min(std::max(nsmin, std::min(atoi(e), nx)), smax);
        equal(ns);
        consider(ns);
    }
    if (best_ns == 0 && tiles * nsmin <= 65536) {                          // bound the host-side search
        for (int ns = nsmin; ns <= std::min({nsmin + 3, nx, smax}); ++ns) {
            equal(ns);
            consider(ns);
        }
        if (nsmin == 1 && nx <= 256)
            for (int a = nx - 1; 2 * a >= nx; --a) {                       // long strip first
                len[0] = a;
                len[1] = nx - a;
                consider(2);
            }
    }
    if (best_ns == 0) {
        best_ns = nsmin;
        equal(best_ns);
        std::copy(len.begin(), len.begin() + best_ns, best_len.begin());
    }
    xb[0] = 0;
    for (int s = 0; s < best_ns; ++s) xb[s + 1] = xb[s] + best_len[s];
    return best_ns;
}

int stage_2d2v_tel_strips(const vlasov_level* L, int* xb) {
    const int64_t tiles = (int64_t)((L->dom[3] + T2_TM - 1) / T2_TM) * (L->dom[2] / T2_LT) * (L->dom[1] / 2);
    return stage_2d2v_choose_strips(tiles, L->dom[0], T2_RMAX, T2_SMAX, "VLASOV_STRIPS2T", xb);
}

int launch_stage_2d2v_tel(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s, double* u,
                          double* f_next, const double* E, double* rho_partials) {
    StageArgsT A;
    A.u_out = u;
    A.f_next = f_next;
    A.E = E;
    A.s0 = L->block_str[0][0];
    A.s1 = L->block_str[0][1];
    A.s2 = L->block_str[0][2];
    A.org = L->block_off[0] + vk::G * (A.s0 + A.s1 + A.s2 + 1);
    A.nx = L->dom[0];
    A.ny = L->dom[1];
    A.nvx = L->dom[2];
    A.nvy = L->dom[3];
    A.nmt = (A.nvy + T2_TM - 1) / T2_TM;
    if (L->tel_ns == 0) L->tel_ns = stage_2d2v_tel_strips(L, L->tel_xb);
    A.nstrips = L->tel_ns;
    std::copy(L->tel_xb, L->tel_xb + T2_SMAX + 1, A.xb);
    A.hx = L->h[0];
    A.hy = L->h[1];
    A.hvx = L->h[2];
    A.hvy = L->h[3];
    A.vx_lo = L->lower[2];
    A.vy_lo = L->lower[3];
    A.sc = stage == 1 || stage == 2 ? 0.5 * dt : stage == 3 ? dt : stage == 4 ? dt / 6.0 : 1.0;
    A.partials = rho_partials;
    TMapsT M;
    int rc;
    if ((rc = encode_map_t(L, f_s, T2_LW, 8, 2, &M.a)) || (rc = encode_map_t(L, f_s, T2_LW, 8, 1, &M.b)) ||
        (rc = encode_map_t(L, f_s, T2_LW, 4, 1, &M.c)) ||
        (rc = encode_map_t(L, f_n ? f_n : f_s, T2_TM, T2_LT, 2, &M.fn)) ||
        (rc = encode_map_t(L, u ? u : f_s, T2_TM, T2_LT, 2, &M.u)))
        return rc;
    const unsigned grid = (unsigned)A.nmt * (A.nvx / T2_LT) * (A.ny / 2) * A.nstrips;
    switch (stage) {
        case 0: return launch_tel_t<0>(A, M, grid, L->stream);
        case 1: return launch_tel_t<1>(A, M, grid, L->stream);
        case 2: return launch_tel_t<2>(A, M, grid, L->stream);
        case 3: return launch_tel_t<3>(A, M, grid, L->stream);
        case 4: return launch_tel_t<4>(A, M, grid, L->stream);
    }
    return fail(VLASOV_EINVAL, "stage must be 0..4");
}

}  // namespace vk
