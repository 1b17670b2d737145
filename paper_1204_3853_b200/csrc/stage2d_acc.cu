// 2D+2V fused RK4 stage for CENTERED4, telescoped form with per-output accumulators (BASELINE.json
// C5).  Same linear map as stage2d_tel.cu (the flux divergence of P:246-250 with the face averages
// of P:344-345 and the fluxes of P:263-282, written as D_d of cell-centred pre-fields):
//
//   sc k = bx D_x P + by D_y Q + g0 D_vx f + g1 d_x D_vx f + g2 d_y D_vx f
//                               + g3 D_vy f + g4 d_x D_vy f + g5 d_y D_vy f
//
//   D g = g_{-2} - 8 g_{-1} + 8 g_{+1} - g_{+2},  d g = g_{+1} - g_{-1},
//   P = rx f + d_vx f,  Q = ry f + d_vy f,  g0..g5 from E and its centred differences at the
//   cell's (x, y) (reading #3's +1/48).
//
// stage2d_tel.cu keeps register windows of the *inputs* along the march direction x (P, D_vx f,
// D_vy f, Q, f at 4 rows: 20 doubles per cell), which limits a thread to 4 cells and makes the
// kernel shared-memory bound (every thread re-derives the pre-fields of its y neighbours from raw
// f).  Here the x stencils are applied in scatter form: row r adds its contribution to the
// accumulators of the output rows r-2 .. r+1 and the accumulator of row r-2 is then complete.
// With the row differences e(r) = P(r) - P(r-1),
//
//   D_x P (i) = -e(i-1) + 7 e(i) + 7 e(i+1) - e(i+2)
//
// so a cell needs 3 live accumulators and the previous row's P (4 doubles instead of 20), and a
// thread owns 4 y lines x 2 vy cells.  Per cell this takes ~30 % fewer shared-memory loads (2 y
// neighbour lines per 4 own lines instead of per 2) and ~30 % fewer TMA bytes (56 line segments per
// 16 output lines instead of 40 per 8).  A constant f still gives k == 0 exactly (every e, D and d
// of equal values is an exact zero).  The stage's f_s enters the RK4 combine through the
// accumulator (stages 1, 4) or a two-row register window (stage 2).
//
// Measured on B200: parity-green but not faster than stage2d_tel.cu in any variant
// tried, so it is opt-in (VLASOV_C5_ACC=1): at 8 warps per SM the row step is a latency chain, and
// fewer shared-memory wavefronts do not shorten it.
//
// Layout: [x][y][vx][vy], vy contiguous, ghost frame 2; the velocity ghost frame of f_s is derived
// before the stage by k_vghost_2d2v (reading #6); x, y periodic by coordinates.  CTA = 4 y lines
// k0..k0+3 (in every thread), 4 vx lines l0..l0+3 (one consumer warp each), a vy tile of 64 cells
// (2 per lane), marching along x over a strip; a producer warpgroup (one lane issues) streams per
// row r into a shared-memory ring with TMA tensor copies:
//   A   y = k0 .. k0+3,   vx l0-2 .. l0+5   (P, D_vx f, D_vy f, Q, f of the own lines)
//   B   y = k0-1, k0+4,   vx l0-2 .. l0+5   (D_vx f, D_vy f, Q of the y neighbours)
//   C   y = k0-2, k0+5,   vx l0 .. l0+3     (Q for D_y)
// B and C only for rows inside the strip (the 2+2 rows around it contribute through x only).
// f_n (stages 2, 3) or u (stage 4) of the completing row arrives in a single-buffered part of its
// own (issued when the previous row's has been consumed, prefetched into the L2 earlier).
// The per-(x, y) velocity coefficients are produced row by row by a helper warp of the producer
// warpgroup into an 8-row ring (they ride on the slot's full barrier), so a strip may have any
// number of rows.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "internal.h"
#include "ptx.cuh"

namespace vk {

constexpr int A2_LT = 4;                    // vx lines (consumer warps) per CTA
constexpr int A2_NY = 4;                    // y lines per CTA (all in every thread)
constexpr int A2_TM = 64;                   // vy cells per tile (2 per lane)
constexpr int A2_LW = A2_TM + 4;            // doubles per line segment
constexpr int A2_THREADS = 256;             // 4 consumer warps + producer warpgroup
constexpr int A2_RMAX = 1 << 20;            // rows per strip (no table: any length)
constexpr int A2_CR = 8;                    // rows of the coefficient ring
constexpr int A2_SMAX = 16;                 // strips along x with explicit bounds
// slot layout (doubles); every part offset is a multiple of 16 doubles (128-B TMA destinations)
constexpr int A2_A = 0;                     // [4 y][8 vx][68]
constexpr int A2_B0 = 32 * A2_LW;           // [8][68]
constexpr int A2_B1 = 40 * A2_LW;           // [8][68]
constexpr int A2_C0 = 48 * A2_LW;           // [4][68]
constexpr int A2_C1 = 52 * A2_LW;           // [4][68]
constexpr int A2_SIZE = 56 * A2_LW;         // doubles per slot
constexpr int A2_CE = A2_CR * A2_NY * 8;    // coefficient ring (doubles)
constexpr int A2_FU = A2_NY * A2_LT * A2_TM;   // doubles of one f_n / u / f_s part [4 y][4 vx][64]
template <int STAGE>
struct SlotA {
    static constexpr int NFU = STAGE >= 2 ? 1 : 0;              // f_n (stages 2, 3) or u (stage 4)
#ifndef A2_MINB3
#define A2_MINB3 0
#endif
    // stages 0-3: 3 CTAs per SM (2 slots, 144 registers per consumer thread); stage 4 (two f_n / u
    // parts): 2 CTAs per SM (3 slots, 232 registers)
    static constexpr int MINB = (A2_MINB3 && STAGE != 4) ? 3 : 2;
    static constexpr int NSLOT = MINB == 3 ? 2 : 3;
    static constexpr int CREGS = MINB == 3 ? 136 : 232;      // 128 (C + 24) <= launch registers x 256
    static constexpr size_t smem_bytes() { return ((size_t)NSLOT * A2_SIZE + A2_CE + NFU * A2_FU) * sizeof(double); }
};

struct TMapsA {
    CUtensorMap a;      // f_s, box (68 vy, 8 vx, 4 y)
    CUtensorMap b;      // f_s, box (68, 8, 1)
    CUtensorMap c;      // f_s, box (68, 4, 1)
    CUtensorMap fn;     // f_n, box (64, 4, 4)
    CUtensorMap fu;     // stage 4: u, box (64, 4, 4)
};

struct StageArgsA {
    double* u_out;
    double* f_next;
    const double* E;           // [2][(nx+4)(ny+4)] ghosted level field
    double* partials;          // [nvx * nmt][nx][ny] moment partials (nullable)
    int64_t s0, s1, s2, org;
    int nx, ny, nvx, nvy, nmt, nstrips;
    int xb[A2_SMAX + 1];       // strip s covers rows xb[s] .. xb[s+1]-1
    double hx, hy, hvx, hvy, vx_lo, vy_lo;
    double sc;                 // stage factor of k (0.5 dt, 0.5 dt, dt, dt/6; 1 for STAGE 0)
};

__device__ __forceinline__ int wrapa(int i, int n) {
    i += (i < 0) ? n : 0;
    i -= (i >= n) ? n : 0;
    return i;
}

// D g = g_{-2} - 8 g_{-1} + 8 g_{+1} - g_{+2}, given t = g_{+1} - g_{-1}
__device__ __forceinline__ double dtela(double gm2, double gp2, double t) { return fma(8.0, t, gm2 - gp2); }

template <int STAGE>
__global__ void __launch_bounds__(A2_THREADS, SlotA<STAGE>::MINB) k_stage_2d2v_acc(const StageArgsA A, const __grid_constant__ TMapsA M) {
    constexpr int SIZE = A2_SIZE, NSLOT = SlotA<STAGE>::NSLOT, NY = A2_NY;
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full_bar[NSLOT];
    __shared__ __align__(8) uint64_t empty_bar[NSLOT];
    __shared__ __align__(8) uint64_t fu_bar;
    __shared__ uint32_t s_dep[32 * A2_LT];
    constexpr int NFU = SlotA<STAGE>::NFU;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int b = blockIdx.x;
    const int mt = b % A.nmt;
    b /= A.nmt;
    const int nlt = A.nvx / A2_LT;
    const int l0 = (b % nlt) * A2_LT;
    b /= nlt;
    const int k0 = NY * (b % (A.ny / NY));
    const int strip = b / (A.ny / NY);
    const int x0 = A.nstrips <= A2_SMAX ? A.xb[strip] : (int)((int64_t)A.nx * strip / A.nstrips);
    const int x1 = A.nstrips <= A2_SMAX ? A.xb[strip + 1] : (int)((int64_t)A.nx * (strip + 1) / A.nstrips);
    const int rows = x1 - x0, Q = rows + 4;
    const int ncols = min(A2_TM, A.nvy - mt * A2_TM);
    const int nyg = A.ny + 4;
    const int64_t ecomp = (int64_t)(A.nx + 4) * nyg;

    if (tid == 0) {
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(&full_bar[s], 2);                               // TMA issuer + coefficient warp
            mbar_init(&empty_bar[s], A2_LT);
        }
        mbar_init(&fu_bar, 1);
        fence_mbar_init();
    }
    griddep_wait();
    double* cE = smem + NSLOT * SIZE;                                     // [A2_CR][NY][8] coefficient ring
    double* FU = cE + A2_CE;                                              // [NFU][NY][LT][64]
    __syncthreads();

    if (warp >= A2_LT) {                                                   // ---------------- producer
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(24));
        if (warp == A2_LT && lane == 0) {
            constexpr uint32_t BA = 32 * A2_LW * 8, BB = 8 * A2_LW * 8, BC = 4 * A2_LW * 8, BF = A2_FU * 8;
            const int cm = mt * A2_TM;                                     // ghosted vy coord of m = mt*TM - 2
            const int ym1 = wrapa(k0 - 1, A.ny) + 2, yp4 = wrapa(k0 + 4, A.ny) + 2;
            const int ym2 = wrapa(k0 - 2, A.ny) + 2, yp5 = wrapa(k0 + 5, A.ny) + 2;
            int slot = 0;
            uint32_t phase = 0;
            // iteration q: main parts of step q; f_n / u part of step q - NSLOT + 1 (the consumers
            // have finished step q - NSLOT, so the single buffer is free); L2 prefetch of that part
            // for step q
            for (int q = 0; q < Q + NSLOT - 1; ++q) {
                if (q >= NSLOT) mbar_wait(&empty_bar[slot], phase ^ 1u);
                if (q < Q) {
                    const bool centre = q >= 2 && q < rows + 2;
                    const int r = wrapa(x0 - 2 + q, A.nx) + 2;
                    double* dst = smem + slot * SIZE;
                    uint64_t* fb = &full_bar[slot];
                    mbar_arrive_expect_tx(fb, centre ? BA + 2 * BB + 2 * BC : BA);
                    tma_load_4d(dst + A2_A, &M.a, cm, l0, k0 + 2, r, fb);
                    if (centre) {
                        tma_load_4d(dst + A2_B0, &M.b, cm, l0, ym1, r, fb);
                        tma_load_4d(dst + A2_B1, &M.b, cm, l0, yp4, r, fb);
                        tma_load_4d(dst + A2_C0, &M.c, cm, l0 + 2, ym2, r, fb);
                        tma_load_4d(dst + A2_C1, &M.c, cm, l0 + 2, yp5, r, fb);
                    }
                    if (NFU >= 1 && q >= 4) {
                        const int ip = x0 - 4 + q + 2;                     // output row of step q (no wrap: in the strip)
                        tma_prefetch_4d(STAGE == 4 ? &M.fu : &M.fn, cm + 2, l0 + 2, k0 + 2, ip);
                    }
                }
                if (NFU >= 1 && q >= 4 + NSLOT - 1) {
                    const int i = x0 - 4 + (q - NSLOT + 1) + 2;            // output row of step q - NSLOT + 1
                    mbar_arrive_expect_tx(&fu_bar, NFU * BF);
                    tma_load_4d(FU, STAGE == 4 ? &M.fu : &M.fn, cm + 2, l0 + 2, k0 + 2, i, &fu_bar);
                }
                if (++slot == NSLOT) { slot = 0; phase ^= 1u; }
            }
        } else if (warp == A2_LT + 1) {
            // coefficient warp: ring entry t (position t mod 8) holds row x0-1+t, times the stage
            // factor: {g0, g3 | g2, g5 | g1, g4 | -, -} per y line (values, d_y, d_x of E_x, E_y);
            // lane = 8 y + entry.  Step q reads the entries q-2 .. q; the warp arrives on the slot's
            // full barrier as soon as the slot is free (entries <= q+1 are written by then) and
            // produces entry q+2 afterwards, so its loads are never on the consumers' path.
            const int y = lane >> 3, c = lane & 7, k = k0 + y;
            const int comp = c & 1, kind = c >> 1;                         // E_x / E_y; value, d_y, d_x
            const double h = comp ? A.hvy : A.hvx;
            const double coef = kind == 0 ? A.sc / (12.0 * h) : A.sc / (576.0 * h);
            const double* Ec = A.E + comp * ecomp;
            const int km = wrapa(k - 1, A.ny), kp = wrapa(k + 1, A.ny);
            auto entry = [&](int t) {
                const int i = wrapa(wrapa(x0 - 1 + t, A.nx), A.nx);
                const int im = wrapa(i - 1, A.nx), ip = wrapa(i + 1, A.nx);
                const int ia = kind == 2 ? ip : i, ib = kind == 2 ? im : i;
                const int ka = kind == 1 ? kp : k, kb = kind == 1 ? km : k;
                const double ea = __ldg(Ec + (int64_t)(ia + 2) * nyg + (ka + 2));
                const double eb = __ldg(Ec + (int64_t)(ib + 2) * nyg + (kb + 2));
                const double v = (kind == 0 ? ea : ea - eb) * coef;
                if (c < 6) cE[((t & (A2_CR - 1)) * NY + y) * 8 + c] = v;
            };
            entry(0);
            entry(1);
            int slot = 0;
            uint32_t phase = 0;
            for (int q = 0; q < Q; ++q) {
                if (q >= NSLOT) mbar_wait(&empty_bar[slot], phase ^ 1u);
                __syncwarp();
                if (lane == 0) mbar_arrive(&full_bar[slot]);
                entry(q + 2);
                if (++slot == NSLOT) { slot = 0; phase ^= 1u; }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(SlotA<STAGE>::CREGS));
    const int w = warp, l = l0 + w;
    const int cl = 2 * lane + 2;                                          // slot column of my first cell
    const int m0 = mt * A2_TM + 2 * lane;
    const bool act = 2 * lane < ncols;
    const double rx = 24.0 * (A.vx_lo + ((double)l + 0.5) * A.hvx) / A.hvx;
    const double ry0 = 24.0 * (A.vy_lo + ((double)m0 + 0.5) * A.hvy) / A.hvy;
    const double ry1 = 24.0 * (A.vy_lo + ((double)m0 + 1.5) * A.hvy) / A.hvy;
    const double bx = -A.sc * A.hvx / (288.0 * A.hx), by = -A.sc * A.hvy / (288.0 * A.hy);
    const double bx7 = 7.0 * bx, by7 = 7.0 * by;
    const int64_t cell0 = A.org + (int64_t)k0 * A.s1 + (int64_t)l * A.s2 + m0;   // (x = 0, y = k0) of my cells

    double acc[4][NY][2];     // accumulators of the output rows (slot = row step mod 4)
    double PP[NY][2];         // P of the previous row
    double FW[4][NY][2];      // stage 2: f_s of the rows r-2 .. r (slot = row step mod 4)
#pragma unroll
    for (int y = 0; y < NY; ++y) {
        PP[y][0] = PP[y][1] = 0.0;
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[s][y][0] = acc[s][y][1] = FW[s][y][0] = FW[s][y][1] = 0.0;
    }
    int slot = 0;
    uint32_t phase = 0, fu_phase = 0;

    // pre-fields of one line segment: D_vx f, D_vy f, Q (and P, f for own lines)
    auto line_fields = [&](const double* Ln, double (&dl)[2], double (&dm)[2], double (&qq)[2], double* p, double* f,
                           uint32_t& dep) {
        const double2 c01 = lds2(Ln + cl - 2), c23 = lds2(Ln + cl), c45 = lds2(Ln + cl + 2);
        const double2 lm1 = lds2(Ln - A2_LW + cl), lp1 = lds2(Ln + A2_LW + cl);
        const double2 lm2 = lds2(Ln - 2 * A2_LW + cl), lp2 = lds2(Ln + 2 * A2_LW + cl);
        const double t0 = lp1.x - lm1.x, t1 = lp1.y - lm1.y;
        dl[0] = dtela(lm2.x, lp2.x, t0);
        dl[1] = dtela(lm2.y, lp2.y, t1);
        const double d0 = c23.y - c01.y, d1 = c45.x - c23.x;               // d_vy f at m0, m0+1
        dm[0] = fma(8.0, d0, c01.x - c45.x);
        dm[1] = fma(8.0, d1, c01.y - c45.y);
        qq[0] = fma(ry0, c23.x, d0);
        qq[1] = fma(ry1, c23.y, d1);
        if (p) {
            p[0] = fma(rx, c23.x, t0);
            p[1] = fma(rx, c23.y, t1);
            f[0] = c23.x;
            f[1] = c23.y;
        }
        dep ^= __double2hiint(dl[0]) ^ __double2hiint(dm[0]) ^ __double2hiint(dl[1]) ^ __double2hiint(dm[1]);
    };

    // One row step.  K = q mod 4 is the accumulator slot of row r; rows r-2, r-1, r+1 are slots
    // K+2, K+3, K+1 (mod 4).  centre: r lies in the strip (B, C parts loaded, centre-row terms due).
    // The y stencils are applied in scatter form too (lines j = -2 .. 5 in order, each line's
    // pre-fields go straight into the accumulators of the lines they reach; D_y Q through the line
    // differences eq(j) = Q(j) - Q(j-1): D_y Q (y) = -eq(y-1) + 7 eq(y) + 7 eq(y+1) - eq(y+2)), so
    // only one line's pre-fields are live at a time.
    auto row = [&](auto Kc, auto OUTc, int q, bool live, bool centre, double (&rs)[NY]) {
        constexpr int K = decltype(Kc)::value;
        constexpr bool OUT = decltype(OUTc)::value;
        constexpr int S2 = (K + 2) & 3, S1 = (K + 3) & 3, SP = (K + 1) & 3;     // rows r-2, r-1, r+1
        if (live) mbar_wait(&full_bar[slot], phase);
        const double* S = smem + slot * SIZE;
        uint32_t dep = 0;
        const int i = wrapa(x0 - 4 + q, A.nx);
        const int jr = q + 7;                                             // ring row of r (+8: non-negative)
        const double* ce0 = cE + ((jr & (A2_CR - 1)) * NY) * 8;           // row r:   {g0, g3 | g2, g5 | g1, g4}
        const double* cm1 = cE + (((jr - 1) & (A2_CR - 1)) * NY) * 8 + 4; // row r-1: {g1, g4}
        const double* cp1 = cE + (((jr + 1) & (A2_CR - 1)) * NY) * 8 + 4; // row r+1: {g1, g4}
        double pq[2] = {0.0, 0.0};                                         // Q of the previous line
        if (centre) {
            // j = -2: Q only
            {
                const double* Ln = S + A2_C0 + w * A2_LW;
                const double2 c01 = lds2(Ln + cl - 2), c23 = lds2(Ln + cl), c45 = lds2(Ln + cl + 2);
                pq[0] = fma(ry0, c23.x, c23.y - c01.y);
                pq[1] = fma(ry1, c23.y, c45.x - c23.x);
                dep ^= __double2hiint(pq[0]) ^ __double2hiint(pq[1]);
            }
            // j = -1: reaches line 0
            {
                double dl[2], dm[2], qq[2];
                line_fields(S + A2_B0 + (w + 2) * A2_LW, dl, dm, qq, nullptr, nullptr, dep);
                const double2 g25 = lds2(ce0 + 2);
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    const double eq = qq[mm] - pq[mm];
                    pq[mm] = qq[mm];
                    acc[K][0][mm] = fma(-by, eq, fma(-g25.y, dm[mm], fma(-g25.x, dl[mm], acc[K][0][mm])));
                }
            }
        }
        // own lines j = 0 .. 3
#pragma unroll
        for (int y = 0; y < NY; ++y) {
            double dl[2], dm[2], qq[2], pn[2], fn[2];
            line_fields(S + A2_A + (y * 8 + w + 2) * A2_LW, dl, dm, qq, pn, fn, dep);
            const double2 gm = lds2(cm1 + 8 * y), gp = lds2(cp1 + 8 * y);
            double e[2];
#pragma unroll
            for (int mm = 0; mm < 2; ++mm) {
                // x contributions of row r to the output rows r-2, r-1, r, r+1
                e[mm] = pn[mm] - PP[y][mm];
                PP[y][mm] = pn[mm];
                acc[S2][y][mm] = fma(-bx, e[mm], acc[S2][y][mm]);
                acc[S1][y][mm] = fma(gm.y, dm[mm], fma(gm.x, dl[mm], fma(bx7, e[mm], acc[S1][y][mm])));
                acc[K][y][mm] = fma(bx7, e[mm], acc[K][y][mm]);
                acc[SP][y][mm] = -fma(gp.y, dm[mm], fma(gp.x, dl[mm], bx * e[mm]));
            }
            if (centre) {
                const double2 g03 = lds2(ce0 + 8 * y);
                double eq[2];
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    eq[mm] = qq[mm] - pq[mm];
                    pq[mm] = qq[mm];
                    double a = acc[K][y][mm];
                    a = fma(by7, eq[mm], fma(g03.y, dm[mm], fma(g03.x, dl[mm], a)));
                    // f_s of the output cell enters the RK4 combine through the accumulator
                    if (STAGE == 1) a += fn[mm];
                    if (STAGE == 4) a = fma(fn[mm], 1.0 / 3.0, a);
                    acc[K][y][mm] = a;
                    if (y >= 2) acc[K][y - 2][mm] = fma(-by, eq[mm], acc[K][y - 2][mm]);
                }
                if (y >= 1) {
                    const double2 g25 = lds2(ce0 + 8 * (y - 1) + 2);
#pragma unroll
                    for (int mm = 0; mm < 2; ++mm)
                        acc[K][y - 1][mm] = fma(by7, eq[mm], fma(g25.y, dm[mm], fma(g25.x, dl[mm], acc[K][y - 1][mm])));
                }
                if (y + 1 < NY) {
                    const double2 g25 = lds2(ce0 + 8 * (y + 1) + 2);
#pragma unroll
                    for (int mm = 0; mm < 2; ++mm)
                        acc[K][y + 1][mm] = fma(-by, eq[mm], fma(-g25.y, dm[mm], fma(-g25.x, dl[mm], acc[K][y + 1][mm])));
                }
                if (STAGE == 2) {
                    FW[K][y][0] = fn[0];
                    FW[K][y][1] = fn[1];
                }
            }
        }
        if (centre) {
            // j = 4: reaches lines 3 and 2
            {
                double dl[2], dm[2], qq[2];
                line_fields(S + A2_B1 + (w + 2) * A2_LW, dl, dm, qq, nullptr, nullptr, dep);
                const double2 g25 = lds2(ce0 + 8 * (NY - 1) + 2);
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    const double eq = qq[mm] - pq[mm];
                    pq[mm] = qq[mm];
                    acc[K][NY - 1][mm] = fma(by7, eq, fma(g25.y, dm[mm], fma(g25.x, dl[mm], acc[K][NY - 1][mm])));
                    acc[K][NY - 2][mm] = fma(-by, eq, acc[K][NY - 2][mm]);
                }
            }
            // j = 5: Q only, reaches line 3
            {
                const double* Ln = S + A2_C1 + w * A2_LW;
                const double2 c01 = lds2(Ln + cl - 2), c23 = lds2(Ln + cl), c45 = lds2(Ln + cl + 2);
                const double q0 = fma(ry0, c23.x, c23.y - c01.y), q1 = fma(ry1, c23.y, c45.x - c23.x);
                dep ^= __double2hiint(q0) ^ __double2hiint(q1);
                acc[K][NY - 1][0] = fma(-by, q0 - pq[0], acc[K][NY - 1][0]);
                acc[K][NY - 1][1] = fma(-by, q1 - pq[1], acc[K][NY - 1][1]);
            }
        }
        if (OUT) {
            // row i = r - 2 is complete: acc = sc k (+ f_s terms); RK4 stage combine (minimum-traffic
            // form, DESIGN 6.1) with f_n / u of the row from their part
            if (NFU >= 1 && live) mbar_wait(&fu_bar, fu_phase);
            fu_phase ^= 1u;
#pragma unroll
            for (int y = 0; y < NY; ++y) {
                double o[2], un[2] = {0.0, 0.0};
                double2 gF = make_double2(0.0, 0.0);
                if (NFU >= 1) gF = lds2(FU + (y * A2_LT + w) * A2_TM + 2 * lane);
                if (NFU >= 1) dep ^= __double2hiint(gF.x);
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
                    const double kk = acc[S2][y][mm];
                    const double fnm = mm ? gF.y : gF.x;                  // stage 4: u
                    if (STAGE == 0 || STAGE == 1) {
                        o[mm] = kk;                                        // stage 1: f_s + sc k
                    } else if (STAGE == 2) {
                        const double fs = FW[S2][y][mm];                   // f_s of row r-2
                        un[mm] = fma(2.0 / 3.0, kk, (fnm + fs) * (1.0 / 3.0));
                        o[mm] = fnm + kk;
                    } else if (STAGE == 3) {
                        o[mm] = fnm + kk;
                    } else {
                        o[mm] = fnm + kk;                                  // u + (f_s / 3 + sc k)
                    }
                }
                dep ^= __double2hiint(o[0]);
                if (live && act) {
                    const int64_t off = cell0 + (int64_t)i * A.s0 + (int64_t)y * A.s1;
                    *reinterpret_cast<double2*>(A.f_next + off) = make_double2(o[0], o[1]);
                    if (STAGE == 2) *reinterpret_cast<double2*>(A.u_out + off) = make_double2(un[0], un[1]);
                }
                rs[y] = (live && act) ? o[0] + o[1] : 0.0;
            }
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
        double dummy[NY];
        row(I0{}, std::false_type{}, 0, true, false, dummy);
        row(I1{}, std::false_type{}, 1, true, false, dummy);
        row(I2{}, std::false_type{}, 2, true, true, dummy);
        row(I3{}, std::false_type{}, 3, true, rows > 1, dummy);
    }
    for (int q0 = 4; q0 < Q; q0 += 4) {
        double rs[4][NY];
        row(I0{}, std::true_type{}, q0, true, q0 < rows + 2, rs[0]);
        row(I1{}, std::true_type{}, q0 + 1, q0 + 1 < Q, q0 + 1 < rows + 2, rs[1]);
        row(I2{}, std::true_type{}, q0 + 2, q0 + 2 < Q, q0 + 2 < rows + 2, rs[2]);
        row(I3{}, std::true_type{}, q0 + 3, q0 + 3 < Q, q0 + 3 < rows + 2, rs[3]);
        if (A.partials != nullptr) {
            // warp sums of the group's 16 (row, y) values with one transposed butterfly: after the
            // xor-16/8/4/2 stages lane L holds value v = 8 bit4 + 4 bit3 + 2 bit2 + bit1
            // (row = v >> 2, y = v & 3), the xor-1 stage completes it
            const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4, b2 = lane & 2;
            double h8[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const double lo = rs[t >> 2][t & 3], hi = rs[(t + 8) >> 2][t & 3];
                h8[t] = (b16 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b16 ? lo : hi, 16);
            }
            double h4[4];
#pragma unroll
            for (int t = 0; t < 4; ++t)
                h4[t] = (b8 ? h8[t + 4] : h8[t]) + __shfl_xor_sync(0xffffffffu, b8 ? h8[t] : h8[t + 4], 8);
            double h2[2];
#pragma unroll
            for (int t = 0; t < 2; ++t)
                h2[t] = (b4 ? h4[t + 2] : h4[t]) + __shfl_xor_sync(0xffffffffu, b4 ? h4[t] : h4[t + 2], 4);
            double s = (b2 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? h2[0] : h2[1], 2);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            const int vv = (b16 ? 8 : 0) + (b8 ? 4 : 0) + (b4 ? 2 : 0) + (b2 ? 1 : 0);
            const int qq = q0 + (vv >> 2), y = vv & 3;
            if ((lane & 1) == 0 && qq < Q) {
                const int i = wrapa(x0 - 4 + qq, A.nx);
                A.partials[((int64_t)l * A.nmt + mt) * A.nx * A.ny + (int64_t)i * A.ny + (k0 + y)] = s;
            }
        }
    }
    griddep_launch_dependents();
}

// tensor map of one field over the ghosted block of a single-block 2D+2V level, box (vy, vx, y, 1)
static int encode_map_a(const vlasov_level* L, const double* f, unsigned bvy, unsigned bvx, unsigned by,
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
static int launch_acc_t(const StageArgsA& A, const TMapsA& M, unsigned grid, cudaStream_t st) {
    auto kern = k_stage_2d2v_acc<STAGE>;
    static bool configured = false;
    if (!configured) {
        VK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SlotA<STAGE>::smem_bytes()));
        configured = true;
    }
    VK_CUDA(launch_pdl(kern, dim3(grid), dim3(A2_THREADS), SlotA<STAGE>::smem_bytes(), st, A, M));
    return VLASOV_OK;
}

bool stage_2d2v_acc_ok(const vlasov_level* L) {
    // opt-in (VLASOV_C5_ACC=1): measured slower than stage2d_tel.cu on B200 (DESIGN 6.2)
    static const bool on = std::getenv("VLASOV_C5_ACC") != nullptr;
    return on && L->dom[0] >= 4 && L->dom[1] % A2_NY == 0 && L->dom[2] % A2_LT == 0 && L->dom[3] % 2 == 0;
}

int launch_stage_2d2v_acc(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s, double* u,
                          double* f_next, const double* E, double* rho_partials) {
    StageArgsA A;
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
    A.nmt = (A.nvy + A2_TM - 1) / A2_TM;
    if (L->acc_ns == 0) {
        const int64_t tiles = (int64_t)A.nmt * (A.nvx / A2_LT) * (A.ny / A2_NY);
        L->acc_ns = stage_2d2v_choose_strips(tiles, A.nx, A2_RMAX, A2_SMAX, "VLASOV_STRIPS2A", L->acc_xb);
    }
    A.nstrips = L->acc_ns;
    std::copy(L->acc_xb, L->acc_xb + A2_SMAX + 1, A.xb);
    A.hx = L->h[0];
    A.hy = L->h[1];
    A.hvx = L->h[2];
    A.hvy = L->h[3];
    A.vx_lo = L->lower[2];
    A.vy_lo = L->lower[3];
    A.sc = stage == 1 || stage == 2 ? 0.5 * dt : stage == 3 ? dt : stage == 4 ? dt / 6.0 : 1.0;
    A.partials = rho_partials;
    TMapsA M;
    int rc;
    if ((rc = encode_map_a(L, f_s, A2_LW, 8, A2_NY, &M.a)) || (rc = encode_map_a(L, f_s, A2_LW, 8, 1, &M.b)) ||
        (rc = encode_map_a(L, f_s, A2_LW, 4, 1, &M.c)) ||
        (rc = encode_map_a(L, f_n ? f_n : f_s, A2_TM, A2_LT, A2_NY, &M.fn)) ||
        (rc = encode_map_a(L, stage == 4 && u ? u : f_s, A2_TM, A2_LT, A2_NY, &M.fu)))
        return rc;
    const unsigned grid = (unsigned)A.nmt * (A.nvx / A2_LT) * (A.ny / A2_NY) * A.nstrips;
    switch (stage) {
        case 0: return launch_acc_t<0>(A, M, grid, L->stream);
        case 1: return launch_acc_t<1>(A, M, grid, L->stream);
        case 2: return launch_acc_t<2>(A, M, grid, L->stream);
        case 3: return launch_acc_t<3>(A, M, grid, L->stream);
        case 4: return launch_acc_t<4>(A, M, grid, L->stream);
    }
    return fail(VLASOV_EINVAL, "stage must be 0..4");
}

}  // namespace vk
