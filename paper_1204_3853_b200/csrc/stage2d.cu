// 2D+2V fused RK4 stage kernel (BASELINE.json C5): face averages -> fluxes -> divergence -> RK4
// stage combine -> per-(vx line, vy tile) partials of the velocity moment.
//
// PAPER.md: the 1D+1V discretisation generalised dimension by dimension, as the oracle
// (oracle/scheme.py) does: a configuration face along x_d carries one transverse term along v_d
// (dv_d/24); a velocity face along v_d carries one (1/48) product term per configuration dim.
// Divergence of  f_t + div_x(v f) - div_v(E f) = 0  (reading #1).  Periodic x, y; the
// characteristic condition on vx, vy (reading #6) is evaluated in the kernel, so the
// level must be ONE block covering the periodic domain (SELF mode) with nvx % 4 == 0.
//
// Layout: [x][y][vx][vy], vy contiguous, ghost frame 2 (only addressed, never trusted).
// CTA = one y line k, LT = 4 vx lines l0..l0+3 (one consumer warp each), a vy tile of TM = 64
// cells (2 per lane), marching along x over a strip of rows, plus one producer warp.  Per row
// step the producer streams into a 3-slot shared-memory ring with cp.async.bulk (TMA engine,
// completion on mbarriers) every vy line segment (TM + 4 cells) the step needs:
//   A  row r,  y = k,     vx lines l0-2 .. l0+5   (x window, velocity faces of row r)
//   B  row i,  y = k -+ 1, vx lines l0-2 .. l0+5  (y-transverse velocity faces, y faces)
//   C  row i,  y = k -+ 2, vx lines l0 .. l0+3    (y faces)
//   D  row i,  y = k,     vx lines l0 .. l0+3     (y faces)
//   F, U  f_n and u of the output row i = r - 2 (stages 2-4)
// Consumers keep register windows along x (the x faces are computed once per row, the velocity
// faces of rows i-1, i, i+1 are reused for the x-transverse terms) and read everything else from
// shared memory.  Ghost values come from the characteristic condition: a ghost warp writes the
// vy ghost columns into each landed slot (precomputed task descriptors), the consumers derive vx
// ghost lines in registers on a warp-uniform path (CTAs at a vx boundary); E_bc and the profile
// are staged in shared memory at kernel start.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <algorithm>
#include <type_traits>

#include "internal.h"
#include "ptx.cuh"
#include "scheme.cuh"

namespace vk {

constexpr int S2_LT = 4;                  // vx lines (consumer warps) per CTA
constexpr int S2_TM = 64;                 // vy cells per tile (2 per lane)
constexpr int S2_LW = S2_TM + 4;          // doubles per line segment in a slot
#ifndef S2_NSLOT_CFG
#define S2_NSLOT_CFG 4
#endif
constexpr int S2_NSLOT = S2_NSLOT_CFG;
// 1: the velocity ghost frame of f_s is derived in global memory by k_vghost_2d2v before the stage
// (TMA then loads ghost values like interior ones; no ghost warp, branch-free consumers);
// 0: a ghost warp derives them in every landed slot
#ifndef S2_GLOBAL_GHOSTS
#define S2_GLOBAL_GHOSTS 1
#endif
constexpr int S2_GWARP = S2_GLOBAL_GHOSTS ? 0 : 1;
constexpr int S2_NLINE = 8 + 16 + 8 + 4;  // A + B + C + D line segments per slot

struct TMaps2 {                // TMA tensor maps over the ghosted level block [x][y][vx][vy]
    CUtensorMap fs8;           // f_s, box (68 vy, 8 vx): parts A, B
    CUtensorMap fs4;           // f_s, box (68 vy, 4 vx): parts C, D
    CUtensorMap fn4;           // f_n, box (64 vy, 4 vx)
    CUtensorMap u4;            // u,   box (64 vy, 4 vx)
};

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
    int nx, ny, nvx, nvy, nstrips;
    double dt, hx, hy, hvx, hvy, vx_lo, vy_lo;
};

template <int STAGE>
struct Slot2 {
    static constexpr int NFU = STAGE >= 2 ? 1 : 0;           // f_n (stages 2, 3) or u (stage 4)
    static constexpr int SIZE = S2_NLINE * S2_LW + NFU * S2_LT * S2_TM;   // doubles (multiple of 16: 128-B parts)
    static size_t smem_bytes(int qmax) {
        return ((size_t)S2_NSLOT * SIZE + 20 * (size_t)qmax + 32 + 4 * S2_TM) * sizeof(double);  // ring + staging
    }
};

__device__ __forceinline__ int wrapi(int i, int n) {
    i += (i < 0) ? n : 0;
    i -= (i >= n) ? n : 0;
    return i;
}

// S2_PWG 1 (needs the global ghost frame): the producer is a whole warpgroup (one lane issues the
// TMA copies) that hands its registers to the consumer warpgroup with setmaxnreg (launch 256 x 128
// registers; producer 24, consumers 232)
#ifndef S2_PWG
#define S2_PWG 1
#endif
constexpr bool S2_PWG_ON = S2_PWG && S2_GWARP == 0;
constexpr int S2_THREADS = S2_PWG_ON ? 32 * (S2_LT + 4) : 32 * (S2_LT + 1 + S2_GWARP);

template <int STAGE, int RECON>
__global__ void __launch_bounds__(S2_THREADS, 2) k_stage_2d2v(const StageArgs2 A, const __grid_constant__ TMaps2 M) {
    using SL = Slot2<STAGE>;
    constexpr int SIZE = SL::SIZE;
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full_bar[S2_NSLOT];    // TMA landed (producer -> ghost warp)
    __shared__ __align__(8) uint64_t ready_bar[S2_NSLOT];   // vy ghosts derived (ghost warp -> consumers)
    __shared__ __align__(8) uint64_t empty_bar[S2_NSLOT];   // slot consumed (consumers -> producer)
    __shared__ uint32_t s_dep[32 * S2_LT];                   // slot-release dependency sink

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int mt = blockIdx.x, l0 = blockIdx.y * S2_LT;
    const int k = blockIdx.z % A.ny, strip = blockIdx.z / A.ny;
    const int x0 = (int)((int64_t)A.nx * strip / A.nstrips);
    const int x1 = (int)((int64_t)A.nx * (strip + 1) / A.nstrips);
    const int Q = (x1 - x0) + 4;
    const int ncols = min(S2_TM, A.nvy - mt * S2_TM);           // vy cells of this tile
    const int wpad = (ncols + 1) & ~1;
    const int nyg = A.ny + 4;
    const int64_t ecomp = (int64_t)(A.nx + 4) * nyg;

    if (tid == 0) {
        for (int s = 0; s < S2_NSLOT; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&ready_bar[s], 32);
            mbar_init(&empty_bar[s], S2_LT);
        }
        fence_mbar_init();
    }
    // programmatic dependent launch: nothing above read memory earlier kernels write
    griddep_wait();
    // Stage what the ghost values need besides the slots: E_bc (x, y components) of the strip's
    // rows at y = k-2 .. k+2, the unperturbed profile at the vy ghost cells of the CTA's vx lines
    // and at the vx ghost lines (characteristic condition, reading #6).
    double* gE = smem + S2_NSLOT * SIZE;                          // [Q][5][2] E_bc
    double* gEf = gE + 10 * Q;                                    // [Q][5][2] E (the stage's field)
    double* gPv = gEf + 10 * Q;                                   // [8 lines l0-2+L][4]: m = -2, -1, nvy, nvy+1
    double* gPx = gPv + 32;                                       // [4][TM]: vx lines -2, -1, nvx, nvx+1
    for (int t = tid; t < 5 * Q; t += blockDim.x) {
        const int tq = t / 5, dy = t % 5;
        const int xx = wrapi(x0 - 2 + tq, A.nx), yy = wrapi(k - 2 + dy, A.ny);
        gE[2 * t] = __ldg(A.E_bc + (int64_t)(xx + 2) * nyg + (yy + 2));
        gE[2 * t + 1] = __ldg(A.E_bc + ecomp + (int64_t)(xx + 2) * nyg + (yy + 2));
        gEf[2 * t] = __ldg(A.E + (int64_t)(xx + 2) * nyg + (yy + 2));
        gEf[2 * t + 1] = __ldg(A.E + ecomp + (int64_t)(xx + 2) * nyg + (yy + 2));
    }
    if (tid < 32 && A.f0v != nullptr) {
        const int Lg = tid >> 2, which = tid & 3;
        const int ll = min(max(l0 - 2 + Lg, 0), A.nvx - 1);
        const int mm = which < 2 ? which : A.nvy + which;
        gPv[tid] = __ldg(A.f0v + (int64_t)(ll + 2) * (A.nvy + 4) + mm);
    }
    for (int t = tid; t < 4 * S2_TM && A.f0v != nullptr; t += blockDim.x) {
        const int g = t / S2_TM, c = t % S2_TM;
        const int lg = g < 2 ? g - 2 : A.nvx + (g - 2);
        const int m = min(mt * S2_TM + c, A.nvy - 1);
        gPx[t] = __ldg(A.f0v + (int64_t)(lg + 2) * (A.nvy + 4) + (m + 2));
    }
    __syncthreads();

    if (S2_PWG_ON ? warp >= S2_LT : warp == S2_LT) {              // ---------------- producer warp(group)
        // 6-8 tensor copies per row step (coordinates in the ghosted block: +2 per dim; x and y
        // wrapped periodically; out-of-range vx / vy boxes are zero-filled by the TMA unit)
        if (S2_PWG_ON) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(24));
        if (warp == S2_LT && lane == 0) {
            constexpr uint32_t BA = 8 * S2_LW * 8, BC = 4 * S2_LW * 8, BF = 4 * S2_TM * 8;
            int slot = 0;
            uint32_t phase = 0;
            const int cm = mt * S2_TM;                                  // ghosted vy coord of m = mt*TM - 2
            for (int q = 0; q < Q; ++q) {
                if (q >= S2_NSLOT) mbar_wait(&empty_bar[slot], phase ^ 1u);
                const bool out_row = q >= 4;
                const int r = wrapi(x0 - 2 + q, A.nx), i = wrapi(x0 - 4 + q, A.nx);
                double* dst = smem + slot * SIZE;
                uint64_t* fb = &full_bar[slot];
                mbar_arrive_expect_tx(fb, out_row ? 3 * BA + 3 * BC + SL::NFU * BF : BA);
                tma_load_4d(dst, &M.fs8, cm, l0, k + 2, r + 2, fb);                              // A
                if (out_row) {
                    const int km = wrapi(k - 1, A.ny), kp = wrapi(k + 1, A.ny);
                    const int kmm = wrapi(k - 2, A.ny), kpp = wrapi(k + 2, A.ny);
                    tma_load_4d(dst + 8 * S2_LW, &M.fs8, cm, l0, km + 2, i + 2, fb);              // B0
                    tma_load_4d(dst + 16 * S2_LW, &M.fs8, cm, l0, kp + 2, i + 2, fb);             // B1
                    tma_load_4d(dst + 24 * S2_LW, &M.fs4, cm, l0 + 2, kmm + 2, i + 2, fb);        // C0
                    tma_load_4d(dst + 28 * S2_LW, &M.fs4, cm, l0 + 2, kpp + 2, i + 2, fb);        // C1
                    tma_load_4d(dst + 32 * S2_LW, &M.fs4, cm, l0 + 2, k + 2, i + 2, fb);          // D
                    if (SL::NFU >= 1)                                          // F: f_n, or u in stage 4
                        tma_load_4d(dst + S2_NLINE * S2_LW, STAGE == 4 ? &M.u4 : &M.fn4, cm + 2, l0 + 2, k + 2, i + 2, fb);
                }
                if (++slot == S2_NSLOT) { slot = 0; phase ^= 1u; }
            }
        }
        return;
    }

    if (S2_GWARP && warp == S2_LT + 1) {                          // ---------------- ghost warp
        // vy ghost columns of the 24 line segments the consumers read as (m0-2 .. m0+3) triples
        // (A, B lines 2..5; C, D lines 0..3), characteristic condition (reading #6) with E_bc of
        // the segment's (x, y); task descriptors precomputed, <= 2 tasks per lane per slot.
        const bool vlo = (mt == 0), vhi = (mt * S2_TM + ncols == A.nvy);
        int seg[2], side[2], dq[2], dy[2];
        bool valid[2];
        double p0[2], p1[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int t = lane + 32 * j;                          // task: 24 segments x 2 sides
            const int sidx = t >> 1, sd = t & 1;
            int e, ddq, ddy, ll;
            if (sidx < 4) { e = 2 + sidx; ddq = 0; ddy = 2; ll = l0 + sidx; }
            else if (sidx < 8) { e = 10 + (sidx - 4); ddq = 2; ddy = 1; ll = l0 + sidx - 4; }
            else if (sidx < 12) { e = 18 + (sidx - 8); ddq = 2; ddy = 3; ll = l0 + sidx - 8; }
            else if (sidx < 16) { e = 24 + (sidx - 12); ddq = 2; ddy = 0; ll = l0 + sidx - 12; }
            else if (sidx < 20) { e = 28 + (sidx - 16); ddq = 2; ddy = 4; ll = l0 + sidx - 16; }
            else { e = 32 + (sidx - 20); ddq = 2; ddy = 2; ll = l0 + sidx - 20; }
            seg[j] = e; side[j] = sd; dq[j] = ddq; dy[j] = ddy;
            valid[j] = (t < 48) && (ll < A.nvx) && (sd == 0 ? vlo : vhi);
            const int llc = min(ll, A.nvx - 1);
            p0[j] = __ldg(A.f0v + (int64_t)(llc + 2) * (A.nvy + 4) + (sd == 0 ? 0 : A.nvy + 2));
            p1[j] = __ldg(A.f0v + (int64_t)(llc + 2) * (A.nvy + 4) + (sd == 0 ? 1 : A.nvy + 3));
        }
        int slot = 0;
        uint32_t phase = 0;
        for (int q = 0; q < Q; ++q) {
            mbar_wait(&full_bar[slot], phase);
            double* S = smem + slot * SIZE;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (!valid[j] || (dq[j] && q < 4)) continue;
                double* sg = S + seg[j] * S2_LW;
                const double a = -gE[2 * (5 * (q - dq[j]) + dy[j]) + 1];
                if (side[j] == 0) {                               // m = -2, -1 at columns 0, 1
                    const double f0 = sg[2], f1 = sg[3], f2 = sg[4], f3 = sg[5];
                    const bool out = a < 0.0;
                    sg[1] = out ? 4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3 : p1[j];
                    sg[0] = out ? 10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3 : p0[j];
                } else {                                          // m = nvy, nvy+1
                    const int c = ncols + 1;                      // column of m = nvy - 1
                    const double f0 = sg[c], f1 = sg[c - 1], f2 = sg[c - 2], f3 = sg[c - 3];
                    const bool out = a > 0.0;
                    sg[c + 1] = out ? 4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3 : p0[j];
                    sg[c + 2] = out ? 10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3 : p1[j];
                }
            }
            mbar_arrive(&ready_bar[slot]);                        // release: this lane's writes
            if (++slot == S2_NSLOT) { slot = 0; phase ^= 1u; }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    if (S2_PWG_ON) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(232));
    const int w = warp, l = l0 + w;
    const bool lact = l < A.nvx;
    const int lc = lact ? l : A.nvx - 1;
    const int cl = 2 * lane + 2;                                  // slot column of my first cell
    const int m0 = mt * S2_TM + 2 * lane;
    const bool act = lact && (2 * lane < ncols);
    // E of row step tq (row x0 - 2 + tq) at y = k - 2 + dy, staged in shared memory
    auto Efx = [&](int tq, int dy) { return gEf[2 * (5 * tq + dy)]; };
    auto Efy = [&](int tq, int dy) { return gEf[2 * (5 * tq + dy) + 1]; };
    const double vbx = A.vx_lo + ((double)lc + 0.5) * A.hvx;
    const double vbxm = vbx - A.hvx, vbxp = vbx + A.hvx;
    double vby[4];                                                // m0-1 .. m0+2
#pragma unroll
    for (int a = 0; a < 4; ++a) vby[a] = A.vy_lo + ((double)(m0 + a - 1) + 0.5) * A.hvy;
    // face values and fluxes are carried x12 (face12); 1/12 folds into the divergence factors
    const double rdx = 1.0 / (12.0 * A.hx), rdy = 1.0 / (12.0 * A.hy), rdvx = 1.0 / (12.0 * A.hvx),
                 rdvy = 1.0 / (12.0 * A.hvy);
    const double dvx24 = A.hvx * (1.0 / 24.0), dvy24 = A.hvy * (1.0 / 24.0);

    const bool ledge = (l0 == 0) || (l0 + S2_LT >= A.nvx);            // CTA at a vx boundary (uniform)
    // pair (col) of line L of a part; vx ghost lines (warp-uniform) by the characteristic
    // condition from the part's interior lines, a = -E_x of the part's (x, y)
    auto line_pair = [&](const double* part, int L, double a) -> double2 {
        const int lg = l0 - 2 + L;
        if (S2_GWARP && ledge && (lg < 0 || lg >= A.nvx)) {
            const bool lo = lg < 0;
            if (lo ? (a < 0.0) : (a > 0.0)) {
                const int j0 = lo ? 0 : A.nvx - 1, dj = lo ? 1 : -1;
                const double2 f0 = lds2(part + (j0 - l0 + 2) * S2_LW + cl), f1 = lds2(part + (j0 + dj - l0 + 2) * S2_LW + cl);
                const double2 f2 = lds2(part + (j0 + 2 * dj - l0 + 2) * S2_LW + cl);
                const double2 f3 = lds2(part + (j0 + 3 * dj - l0 + 2) * S2_LW + cl);
                if (lo ? (lg == -1) : (lg == A.nvx))
                    return make_double2(4.0 * f0.x - 6.0 * f1.x + 4.0 * f2.x - f3.x, 4.0 * f0.y - 6.0 * f1.y + 4.0 * f2.y - f3.y);
                return make_double2(10.0 * f0.x - 20.0 * f1.x + 15.0 * f2.x - 4.0 * f3.x,
                                    10.0 * f0.y - 20.0 * f1.y + 15.0 * f2.y - 4.0 * f3.y);
            }
            const double* px = gPx + (lo ? lg + 2 : 2 + lg - A.nvx) * S2_TM + 2 * lane;
            return make_double2(px[0], px[1]);
        }
        return lds2(part + L * S2_LW + cl);
    };
    auto Ebx = [&](int tq, int dy) { return gE[2 * (5 * tq + dy)]; };

    double W[4][3][2];        // f rows (mod 4) at vx lines l-1, l, l+1, vy m0, m0+1
    double VX[4][2][2];       // 12 x vx-face averages (rows mod 4) at l-1/2, l+1/2
    double VY[4][3];          // 12 x vy-face averages (rows mod 4) at m0-1/2, m0+1/2, m0+3/2
    double Fxp[2];            // 12 x x-fluxes at i - 1/2
    int slot = 0;
    uint32_t phase = 0;
    // One row step q (row r = x0 - 2 + q, window slot K = q mod 4); OUT rows (q >= 4) produce output
    // row i = r - 2.  `live` == false only in the last group: rows past the strip run without wait,
    // stores or slot release (their arithmetic is discarded).  Straight-line code per K.
    auto row = [&](auto Kc, auto OUTc, int q, bool live, double& rsK) {
        constexpr int K = decltype(Kc)::value;
        constexpr bool OUT = decltype(OUTc)::value;
        constexpr int R0 = (K + 1) & 3, R1 = (K + 2) & 3, R2 = (K + 3) & 3;   // rows r-3, r-2, r-1
        if (live) mbar_wait(S2_GWARP ? &ready_bar[slot] : &full_bar[slot], phase);
        const double* SA = smem + slot * SIZE;
        const double* SB = SA + 8 * S2_LW;
        const double* SC = SB + 16 * S2_LW;
        const double* SD = SC + 8 * S2_LW;
        const double* SF = SA + S2_NLINE * S2_LW;
        // ---- row r: x window, vx faces, vy faces
        const double axr = -Ebx(q, 2);
        const double2 c01 = lds2(SA + (w + 2) * S2_LW + cl - 2), c23 = lds2(SA + (w + 2) * S2_LW + cl),
                      c45 = lds2(SA + (w + 2) * S2_LW + cl + 2);
        const double2 am1 = line_pair(SA, w + 1, axr), ap1 = line_pair(SA, w + 3, axr);
        const double2 am2 = line_pair(SA, w, axr), ap2 = line_pair(SA, w + 4, axr);
        // one word of every shared-memory load of the row (slot-release dependency, below)
        uint32_t dep = __double2hiint(c01.x) ^ __double2hiint(c23.x) ^ __double2hiint(c45.x) ^
                       __double2hiint(am1.x) ^ __double2hiint(ap1.x) ^ __double2hiint(am2.x) ^ __double2hiint(ap2.x);
        W[K][0][0] = am1.x; W[K][0][1] = am1.y;
        W[K][1][0] = c23.x; W[K][1][1] = c23.y;
        W[K][2][0] = ap1.x; W[K][2][1] = ap1.y;
        {
            const double ax = -Efx(q, 2), ay = -Efy(q, 2);
            VX[K][0][0] = face12<RECON>(am2.x, am1.x, c23.x, ap1.x, ax);
            VX[K][0][1] = face12<RECON>(am2.y, am1.y, c23.y, ap1.y, ax);
            VX[K][1][0] = face12<RECON>(am1.x, c23.x, ap1.x, ap2.x, ax);
            VX[K][1][1] = face12<RECON>(am1.y, c23.y, ap1.y, ap2.y, ax);
            VY[K][0] = face12<RECON>(c01.x, c01.y, c23.x, c23.y, ay);
            VY[K][1] = face12<RECON>(c01.y, c23.x, c23.y, c45.x, ay);
            VY[K][2] = face12<RECON>(c23.x, c23.y, c45.x, c45.y, ay);
        }
        if (OUT || K == 3) {
            double XF[3][2];
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
                for (int mm = 0; mm < 2; ++mm)
                    XF[b][mm] = face12<RECON>(W[R0][b][mm], W[R1][b][mm], W[R2][b][mm], W[K][b][mm],
                                              b == 0 ? vbxm : (b == 1 ? vbx : vbxp));
            double Fxn[2];
#pragma unroll
            for (int mm = 0; mm < 2; ++mm) Fxn[mm] = vbx * XF[1][mm] + dvx24 * (XF[2][mm] - XF[0][mm]);
            if (OUT) {
                const int i = wrapi(x0 - 4 + q, A.nx);
                // ---- y faces at (i, k -+ 1/2) for vy m0-1 .. m0+2 (lines k-2 .. k+2)
                double2 t[5][3];
                const double* yl[5] = {SC + w * S2_LW, SB + (w + 2) * S2_LW, SD + w * S2_LW,
                                       SB + (8 + w + 2) * S2_LW, SC + (4 + w) * S2_LW};
#pragma unroll
                for (int d = 0; d < 5; ++d) {
                    t[d][0] = lds2(yl[d] + cl - 2);
                    t[d][1] = lds2(yl[d] + cl);
                    t[d][2] = lds2(yl[d] + cl + 2);
                }
#pragma unroll
                for (int d = 0; d < 5; ++d)
                    dep ^= __double2hiint(t[d][0].x) ^ __double2hiint(t[d][1].x) ^ __double2hiint(t[d][2].x);
                double YL[4], YH[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    double y5[5];
#pragma unroll
                    for (int d = 0; d < 5; ++d)
                        y5[d] = (a == 0) ? t[d][0].y : (a == 1) ? t[d][1].x : (a == 2) ? t[d][1].y : t[d][2].x;
                    YL[a] = face12<RECON>(y5[0], y5[1], y5[2], y5[3], vby[a]);
                    YH[a] = face12<RECON>(y5[1], y5[2], y5[3], y5[4], vby[a]);
                }
                // ---- y-transverse velocity-face averages at (i, k -+ 1)
                double VXk[2][2][2], VYk[2][3];
#pragma unroll
                for (int sg = 0; sg < 2; ++sg) {
                    const double* P = SB + sg * 8 * S2_LW;
                    const double axk = -Ebx(q - 2, sg ? 3 : 1);
                    const double2 bm1 = line_pair(P, w + 1, axk), bp1 = line_pair(P, w + 3, axk);
                    const double2 bm2 = line_pair(P, w, axk), bp2 = line_pair(P, w + 4, axk);
                    dep ^= __double2hiint(bm1.x) ^ __double2hiint(bp1.x) ^ __double2hiint(bm2.x) ^ __double2hiint(bp2.x);
                    const double2 b01 = t[sg ? 3 : 1][0], b23 = t[sg ? 3 : 1][1], b45 = t[sg ? 3 : 1][2];
                    const double ax = -Efx(q - 2, sg ? 3 : 1), ay = -Efy(q - 2, sg ? 3 : 1);
                    VXk[sg][0][0] = face12<RECON>(bm2.x, bm1.x, b23.x, bp1.x, ax);
                    VXk[sg][0][1] = face12<RECON>(bm2.y, bm1.y, b23.y, bp1.y, ax);
                    VXk[sg][1][0] = face12<RECON>(bm1.x, b23.x, bp1.x, bp2.x, ax);
                    VXk[sg][1][1] = face12<RECON>(bm1.y, b23.y, bp1.y, bp2.y, ax);
                    VYk[sg][0] = face12<RECON>(b01.x, b01.y, b23.x, b23.y, ay);
                    VYk[sg][1] = face12<RECON>(b01.y, b23.x, b23.y, b45.x, ay);
                    VYk[sg][2] = face12<RECON>(b23.x, b23.y, b45.x, b45.y, ay);
                }
                const double exi = Efx(q - 2, 2), eyi = Efy(q - 2, 2);
                const double cxi = (Efx(q - 1, 2) - Efx(q - 3, 2)) * (1.0 / 48.0);
                const double cxk = (Efx(q - 2, 3) - Efx(q - 2, 1)) * (1.0 / 48.0);
                const double cyi = (Efy(q - 1, 2) - Efy(q - 3, 2)) * (1.0 / 48.0);
                const double cyk = (Efy(q - 2, 3) - Efy(q - 2, 1)) * (1.0 / 48.0);
                double Fvy[3];
#pragma unroll
                for (int fc = 0; fc < 3; ++fc)
                    Fvy[fc] = eyi * VY[R1][fc] + cyi * (VY[R2][fc] - VY[R0][fc]) + cyk * (VYk[1][fc] - VYk[0][fc]);
                double2 fn = make_double2(0.0, 0.0), uu = make_double2(0.0, 0.0);
                if (STAGE == 2 || STAGE == 3) fn = lds2(SF + w * S2_TM + 2 * lane);
                if (STAGE == 4) uu = lds2(SF + w * S2_TM + 2 * lane);
                dep ^= __double2hiint(fn.x) ^ __double2hiint(uu.x);
                double o[2], un[2];
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
                        un[mm] = (fnm + fs) * (1.0 / 3.0) + (A.dt * (1.0 / 3.0)) * kk;
                        o[mm] = fnm + (0.5 * A.dt) * kk;
                    } else if (STAGE == 3) {
                        o[mm] = fnm + A.dt * kk;
                    } else {
                        o[mm] = um + fs * (1.0 / 3.0) + (A.dt * (1.0 / 6.0)) * kk;
                    }
                }
                if (live && act) {
                    const int64_t off = A.org + (int64_t)i * A.s0 + (int64_t)k * A.s1 + (int64_t)l * A.s2 + m0;
                    *reinterpret_cast<double2*>(A.f_next + off) = make_double2(o[0], o[1]);
                    if (STAGE == 2) *reinterpret_cast<double2*>(A.u_out + off) = make_double2(un[0], un[1]);
                }
                rsK = (live && act) ? (o[0] + o[1]) : 0.0;
            }
            Fxp[0] = Fxn[0];
            Fxp[1] = Fxn[1];
        }
        if (live) {
            // Release the slot.  Shared loads are asynchronous and the compiler may schedule their
            // consumers after the arrive: a volatile store of a value depending on every load of
            // the row precedes it, so in-order issue holds the arrive until they have landed.
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(&s_dep[tid])), "r"(dep) : "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[slot]);
            if (++slot == S2_NSLOT) { slot = 0; phase ^= 1u; }
        }
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    {   // rows q = 0..3 (Q >= 5): windows and velocity faces, x-fluxes at x0 - 1/2 at q = 3
        double dummy;
        row(I0{}, std::false_type{}, 0, true, dummy);
        row(I1{}, std::false_type{}, 1, true, dummy);
        row(I2{}, std::false_type{}, 2, true, dummy);
        row(I3{}, std::false_type{}, 3, true, dummy);
    }
    for (int q0 = 4; q0 < Q; q0 += 4) {
        double rs[4];
        row(I0{}, std::true_type{}, q0, true, rs[0]);
        row(I1{}, std::true_type{}, q0 + 1, q0 + 1 < Q, rs[1]);
        row(I2{}, std::true_type{}, q0 + 2, q0 + 2 < Q, rs[2]);
        row(I3{}, std::true_type{}, q0 + 3, q0 + 3 < Q, rs[3]);
        if (A.partials != nullptr) {
            // warp sums of the group's 4 rows with one transposed butterfly (6 shuffles): lane L
            // ends with row 2 bit4(L) + bit3(L); lanes L % 8 == 0 write it
            const bool b16 = lane & 16, b8 = lane & 8;
            double v0 = b16 ? rs[2] : rs[0], v1 = b16 ? rs[3] : rs[1];
            const double w0 = b16 ? rs[0] : rs[2], w1 = b16 ? rs[1] : rs[3];
            v0 += __shfl_xor_sync(0xffffffffu, w0, 16);
            v1 += __shfl_xor_sync(0xffffffffu, w1, 16);
            double u = b8 ? v1 : v0;
            const double xv = b8 ? v0 : v1;
            u += __shfl_xor_sync(0xffffffffu, xv, 8);
            u += __shfl_xor_sync(0xffffffffu, u, 4);
            u += __shfl_xor_sync(0xffffffffu, u, 2);
            u += __shfl_xor_sync(0xffffffffu, u, 1);
            const int qq = q0 + (b16 ? 2 : 0) + (b8 ? 1 : 0);
            if ((lane & 7) == 0 && lact && qq < Q) {
                const int i = wrapi(x0 - 4 + qq, A.nx);
                A.partials[((int64_t)l * gridDim.x + mt) * A.nx * A.ny + (int64_t)i * A.ny + k] = u;
            }
        }
    }
    griddep_launch_dependents();                 // the march is done: let the next kernel launch
}

// Velocity ghost frame of f (characteristic condition, reading #6, a = -E_bc of the (x, y) column):
// threads [0, nx ny nvx): the vy ghosts m = -2, -1, nvy, nvy+1 of one (x, y, vx) line;
// threads [nx ny nvx, nx ny (nvx + nvy)): the vx ghosts l = -2, -1, nvx, nvx+1 at one (x, y, vy).
// Only the ghosts the stage stencils read are derived (vx ghosts at interior vy and vice versa).
__global__ void k_vghost_2d2v(double* __restrict__ f, int64_t org, int64_t s0, int64_t s1, int64_t s2, int nx, int ny,
                              int nvx, int nvy, const double* __restrict__ E_bc, const double* __restrict__ f0v) {
    griddep_wait();
    griddep_launch_dependents();
    // block = one (x, y) column: threads [0, nvx) the vy ghosts of vx line t (16-B loads of the
    // 4 cells next to each end, one 16-B store per end), threads [nvx, nvx + nvy/2) the vx ghosts
    // at the vy cell pair 2(t - nvx), +1 (16-B loads along vy, coalesced across threads).  Rows
    // are 16-B aligned: org, the strides and nvy are even (level layout, nvy even).
    const int c = blockIdx.x;                                     // i * ny + k
    const int i = c / ny, k = c - (c / ny) * ny;
    const int nyg = ny + 4;
    const int64_t col = (int64_t)(i + 2) * nyg + (k + 2);
    double* base = f + org + (int64_t)i * s0 + (int64_t)k * s1;
    auto ld2 = [](const double* q) { return *reinterpret_cast<const double2*>(q); };
    auto st2 = [](double* q, double a, double b) { *reinterpret_cast<double2*>(q) = make_double2(a, b); };
    auto ex1 = [](double f0, double f1, double f2, double f3) { return 4.0 * f0 - 6.0 * f1 + 4.0 * f2 - f3; };
    auto ex2 = [](double f0, double f1, double f2, double f3) { return 10.0 * f0 - 20.0 * f1 + 15.0 * f2 - 4.0 * f3; };
    for (int t = threadIdx.x; t < nvx + nvy / 2; t += blockDim.x) {
      if (t < nvx) {
        const double a = -__ldg(E_bc + (int64_t)(nx + 4) * nyg + col);
        double* line = base + (int64_t)t * s2;                    // m = 0
        const double2 l01 = ld2(line), l23 = ld2(line + 2);
        const double2 h32 = ld2(line + nvy - 4), h10 = ld2(line + nvy - 2);
        const double* pr = f0v + (int64_t)(t + 2) * (nvy + 4);     // profile at ghosted m index
        const double2 plo = ld2(pr), phi = ld2(pr + nvy + 2);      // m = -2, -1 and nvy, nvy+1
        const bool out_lo = a < 0.0, out_hi = a > 0.0;
        st2(line - 2, out_lo ? ex2(l01.x, l01.y, l23.x, l23.y) : plo.x, out_lo ? ex1(l01.x, l01.y, l23.x, l23.y) : plo.y);
        st2(line + nvy, out_hi ? ex1(h10.y, h10.x, h32.y, h32.x) : phi.x, out_hi ? ex2(h10.y, h10.x, h32.y, h32.x) : phi.y);
      } else {
        const double a = -__ldg(E_bc + col);
        const int m = 2 * (t - nvx);
        double* cm = base + m;                                    // (l = 0, m)
        const double2 f0 = ld2(cm), f1 = ld2(cm + s2), f2 = ld2(cm + 2 * s2), f3 = ld2(cm + 3 * s2);
        double* ce = cm + (int64_t)(nvx - 1) * s2;
        const double2 g0 = ld2(ce), g1 = ld2(ce - s2), g2 = ld2(ce - 2 * s2), g3 = ld2(ce - 3 * s2);
        const int64_t pst = nvy + 4;
        const double* pr = f0v + 2 * pst + (m + 2);                // profile (l = 0, m)
        const double2 pm1 = ld2(pr - pst), pm2 = ld2(pr - 2 * pst);
        const double2 pn = ld2(pr + nvx * pst), pn1 = ld2(pr + (nvx + 1) * pst);
        const bool out_lo = a < 0.0, out_hi = a > 0.0;
        st2(cm - s2, out_lo ? ex1(f0.x, f1.x, f2.x, f3.x) : pm1.x, out_lo ? ex1(f0.y, f1.y, f2.y, f3.y) : pm1.y);
        st2(cm - 2 * s2, out_lo ? ex2(f0.x, f1.x, f2.x, f3.x) : pm2.x, out_lo ? ex2(f0.y, f1.y, f2.y, f3.y) : pm2.y);
        st2(ce + s2, out_hi ? ex1(g0.x, g1.x, g2.x, g3.x) : pn.x, out_hi ? ex1(g0.y, g1.y, g2.y, g3.y) : pn.y);
        st2(ce + 2 * s2, out_hi ? ex2(g0.x, g1.x, g2.x, g3.x) : pn1.x, out_hi ? ex2(g0.y, g1.y, g2.y, g3.y) : pn1.y);
      }
    }
}

// rho[i][k] = 1 - dvx dvy sum_p partials[p][i][k]: block (32 cells, 8 plane groups); group g sums
// the planes g, g + 8, ... of its cell, the 8 group sums are added in group order (deterministic)
__global__ void k_moment_2d2v_finish(const double* __restrict__ partials, int np, int ncfg, double dvv,
                                     double* __restrict__ rho) {
    griddep_wait();
    griddep_launch_dependents();
    __shared__ double sg[8][33];
    const int c = blockIdx.x * 32 + threadIdx.x, g = threadIdx.y;
    double s = 0.0;
    if (c < ncfg)
        for (int p = g; p < np; p += 8) s += partials[(int64_t)p * ncfg + c];
    sg[g][threadIdx.x] = s;
    __syncthreads();
    if (g == 0 && c < ncfg) {
        double t = sg[0][threadIdx.x];
#pragma unroll
        for (int k = 1; k < 8; ++k) t += sg[k][threadIdx.x];
        rho[c] = 1.0 - dvv * t;
    }
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

template <int STAGE, int RECON>
static int launch2_t(const StageArgs2& A, const TMaps2& M, dim3 grid, cudaStream_t st) {
    auto kern = k_stage_2d2v<STAGE, RECON>;
    const int qmax = (A.nx + A.nstrips - 1) / A.nstrips + 4;
    const size_t smem = Slot2<STAGE>::smem_bytes(qmax);
    static bool configured = false;
    if (!configured) {
        VK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    VK_CUDA(launch_pdl(kern, grid, dim3(S2_THREADS), smem, st, A, M));
    return VLASOV_OK;
}

template <int RECON>
static int dispatch2(int stage, const StageArgs2& A, const TMaps2& M, dim3 grid, cudaStream_t st) {
    switch (stage) {
        case 0: return launch2_t<0, RECON>(A, M, grid, st);
        case 1: return launch2_t<1, RECON>(A, M, grid, st);
        case 2: return launch2_t<2, RECON>(A, M, grid, st);
        case 3: return launch2_t<3, RECON>(A, M, grid, st);
        case 4: return launch2_t<4, RECON>(A, M, grid, st);
    }
    return fail(VLASOV_EINVAL, "stage must be 0..4");
}

// tensor map of one field over the ghosted block of a single-block 2D+2V level
static int encode_map(const vlasov_level* L, const double* f, unsigned box_vy, unsigned box_vx, CUtensorMap* out) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
            cudaGetLastError();
            return fail(VLASOV_ECUDA, "cuTensorMapEncodeTiled not available");
        }
        enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const cuuint64_t dims[4] = {(cuuint64_t)L->block_str[0][2], (cuuint64_t)(L->dom[2] + 2 * G),
                                (cuuint64_t)(L->dom[1] + 2 * G), (cuuint64_t)(L->dom[0] + 2 * G)};
    const cuuint64_t strides[3] = {(cuuint64_t)L->block_str[0][2] * 8, (cuuint64_t)L->block_str[0][1] * 8,
                                   (cuuint64_t)L->block_str[0][0] * 8};
    const cuuint32_t box[4] = {box_vy, box_vx, 1, 1}, estr[4] = {1, 1, 1, 1};
    CUresult rc = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)(f + L->block_off[0]), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) return fail(VLASOV_ECUDA, "cuTensorMapEncodeTiled failed");
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
    A.E_bc = E_bc ? E_bc : E;           // staged by the face-form kernel (rhs: its field)
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
    // the row march wraps x once on either side (rows x0-4 .. x1+1): at least 4 x cells
    if (A.nx < 4) return fail(VLASOV_EINVAL, "2D+2V stage: need >= 4 cells along x");
    const int nmt = (A.nvy + S2_TM - 1) / S2_TM, nlg = (A.nvx + S2_LT - 1) / S2_LT;
    A.nstrips = L->strips2;
    A.partials = rho ? L->d_partials : nullptr;
    const dim3 grid(nmt, nlg, A.ny * A.nstrips);
    TMaps2 M;
    int rc;
    if ((rc = encode_map(L, f_s, S2_LW, 8, &M.fs8)) || (rc = encode_map(L, f_s, S2_LW, 4, &M.fs4)) ||
        (rc = encode_map(L, f_n ? f_n : f_s, S2_TM, 4, &M.fn4)) || (rc = encode_map(L, u ? u : f_s, S2_TM, 4, &M.u4)))
        return rc;
    // the velocity ghost frame of f_s from E_bc (vlasov_rhs, stage 0: the frame must be current)
    if (S2_GLOBAL_GHOSTS && E_bc != nullptr && f0v != nullptr) {
        VK_CUDA(launch_pdl(k_vghost_2d2v, dim3((unsigned)(A.nx * A.ny)), dim3((unsigned)std::min(1024, (A.nvx + A.nvy / 2 + 31) / 32 * 32)), 0, L->stream,
                           const_cast<double*>(f_s), A.org, A.s0, A.s1, A.s2, A.nx, A.ny, A.nvx, A.nvy, E_bc, f0v));
    }
    static const bool faces = std::getenv("VLASOV_C5_FACES") != nullptr;   // experiment: face form
    if (recon == VLASOV_CENTERED4 && !faces && stage_2d2v_acc_ok(L)) {
        // CENTERED4: telescoped form with per-output accumulators (stage2d_acc.cu)
        rc = launch_stage_2d2v_acc(L, stage, dt, f_n, f_s, u, f_next, E, rho ? L->d_partials : nullptr);
    } else if (recon == VLASOV_CENTERED4 && !faces && stage_2d2v_tel_ok(L)) {
        // CENTERED4: telescoped form (stage2d_tel.cu); the moment partials have the same layout
        rc = launch_stage_2d2v_tel(L, stage, dt, f_n, f_s, u, f_next, E, rho ? L->d_partials : nullptr);
    } else {
        rc = recon == VLASOV_UPWIND ? dispatch2<VLASOV_UPWIND>(stage, A, M, grid, L->stream)
                                    : dispatch2<VLASOV_CENTERED4>(stage, A, M, grid, L->stream);
    }
    if (rc || !rho) return rc;
    const int ncfg = A.nx * A.ny;
    VK_CUDA(launch_pdl(k_moment_2d2v_finish, dim3((ncfg + 31) / 32), dim3(32, 8), 0, L->stream,
                       (const double*)L->d_partials, A.nvx * nmt, ncfg, A.hvx * A.hvy, rho));
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
