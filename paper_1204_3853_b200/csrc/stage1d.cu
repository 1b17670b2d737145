// 1D+1V fused RK4 stage kernel: (ghost values) -> face averages -> fluxes -> divergence -> RK4
// stage combine -> velocity moment of the new stage state.
//
// PAPER.md: face averages P:322-368, fluxes P:263-282 (+1/48, reading #3), divergence
// P:246-250, RK4 P:389-410 (minimum-traffic rearrangement, see include/vlasov.h), moment
// P:295-297, periodic x and characteristic v-boundary P:222-231 (reading #6).
//
// Design (B200): one CTA owns a v-segment of TV = 2*NT contiguous cells and marches along x
// over `nrows` rows.  A producer warp streams each row segment of f_s (with its 2+2 halo
// columns) and the matching f_n / u rows into an NSLOT-deep shared-memory ring with
// cp.async.bulk (TMA engine), completing on mbarriers; NSLOT is sized so that ~64 KB per CTA
// are in flight.  NT consumer threads own two adjacent v-cells each, keep a 4-row register
// window of f_s, compute every face once per row from registers, and release ring slots via
// "empty" mbarriers.  f_s is read once per tile (+4 halo rows, L2 hits), f_n / u once, f_next / u
// written once: 16/32/24/32 B per cell for stages 1..4 (DESIGN.md roofline).
// SELF mode (single block covering the periodic domain): the producer wraps halo rows
// periodically and the two edge threads of the edge tiles compute the characteristic v-ghosts
// in registers, so no ghost-fill kernel and no ghost-frame traffic are needed.
// Moment: per-(row, tile) warp-shuffle + cross-warp sums -> scratch; the last CTA of a row strip
// (atomic ticket) adds the v-tiles in tile order -> rho = 1 - dv sum (deterministic).
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace vk {

struct StageArgs1 {
    const double* f_s;
    const double* f_n;
    const double* u_in;
    double* u_out;
    double* f_next;
    const double* E;           // level E array, index x + 2
    const double* E_bc;        // SELF: field deciding the characteristic direction
    const double* f0v;         // SELF: unperturbed profile on the ghosted v range
    double* rho;               // nullable: moment of f_next
    double* partials;          // scratch [n_vtiles][dom_x]
    unsigned* tickets;         // scratch [n_strips]
    const Tile1* tiles;
    const Block1* blocks;
    double dt, dx, dv, v_lo;   // v_lo: physical lower velocity of the level domain
    int dom_x, dom_v, n_vtiles, tile_rows;
};

template <int RECON>
__device__ __forceinline__ double face_avg(double fm1, double f0, double fp1, double fp2, double upw) {
    if (RECON == VLASOV_CENTERED4) {
        return (7.0 * (f0 + fp1) - (fm1 + fp2)) * (1.0 / 12.0);
    } else {
        const double L = (-fm1 + 5.0 * f0 + 2.0 * fp1) * (1.0 / 6.0);
        const double R = (2.0 * f0 + 5.0 * fp1 - fp2) * (1.0 / 6.0);
        const double d2l = fm1 - 2.0 * f0 + fp1, d1l = fp1 - fm1;
        const double d2r = f0 - 2.0 * fp1 + fp2, d1r = fp2 - f0;
        const double sl = 1.0e-6 + ((13.0 / 12.0) * d2l * d2l + 0.25 * d1l * d1l);
        const double sr = 1.0e-6 + ((13.0 / 12.0) * d2r * d2r + 0.25 * d1r * d1r);
        // hat w_L = alpha_L/(alpha_L+alpha_R), alpha = 0.5/s^2  ==  s_R^2/(s_L^2 + s_R^2)
        const double ql = sl * sl, qr = sr * sr;
        const double inv = 1.0 / (ql + qr);
        const double wl = qr * inv, wr = ql * inv;
        const double big = fmax(wl, wr), small = fmin(wl, wr);
        return (upw > 0.0) ? (big * L + small * R) : (small * L + big * R);
    }
}

template <int STAGE, int NT>
struct StageGeom {
    static constexpr int TV = 2 * NT;
    static constexpr int SEG = TV + 4;
    static constexpr int SLOT = SEG + (STAGE >= 2 ? TV : 0) + (STAGE == 4 ? TV : 0);
    // ring depth: ~64 KB of row data per CTA, at least 8 and at most 32 slots
    static constexpr int NSLOT_RAW = (64 * 1024) / (SLOT * 8);
    static constexpr int NSLOT = NSLOT_RAW < 8 ? 8 : (NSLOT_RAW > 32 ? 32 : NSLOT_RAW);
};

template <int STAGE, int RECON, int NT, bool SELF>
__global__ void __launch_bounds__(NT + 32) k_stage_1d1v(const StageArgs1 A) {
    using SG = StageGeom<STAGE, NT>;
    constexpr int TV = SG::TV, SEG = SG::SEG, SLOT = SG::SLOT, NSLOT = SG::NSLOT;
    constexpr bool NEED_FN = (STAGE >= 2);
    constexpr bool NEED_U = (STAGE == 4);
    constexpr int NW = NT / 32;

    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full_bar[NSLOT];
    __shared__ __align__(8) uint64_t empty_bar[NSLOT];
    __shared__ unsigned s_ticket;
    double* psum = smem + NSLOT * SLOT;          // [NW][nrows]

    const Tile1 T = A.tiles[blockIdx.x];
    const Block1 B = A.blocks[T.block];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int Q = T.nrows + 4;
    const int wpad = (T.ncols + 1) & ~1;
    double* sE = psum + NW * A.tile_rows;        // E of rows x0-2 .. x0+nrows+1
    double* sEbc = sE + (A.tile_rows + 4);       // E_bc of the same rows (SELF)
    for (int t = tid; t < Q; t += blockDim.x) {
        const int gi = B.lo_x + T.x0 - 2 + t + G;  // index in the ghosted level E array
        sE[t] = __ldg(A.E + gi);
        if (SELF) sEbc[t] = __ldg(A.E_bc + gi);
    }

    if (tid == 0) {
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // row r (block-local interior index, may be -2..nx+1): interior column 0 of that row
    auto rowbase = [&](int r) -> int64_t { return B.off + (int64_t)(r + G) * B.pitch + G; };

    if (warp == NW) {                            // ---------------- producer warp
        if (lane == 0) {
            const uint32_t seg_bytes = (uint32_t)(wpad + 4) * 8u;
            const uint32_t row_bytes = (uint32_t)wpad * 8u;
            for (int q = 0; q < Q; ++q) {
                const int slot = q % NSLOT;
                if (q >= NSLOT) mbar_wait(&empty_bar[slot], ((q / NSLOT) - 1) & 1);
                const int r = T.x0 - 2 + q;
                int rs = r;
                if (SELF) rs = (r < 0) ? r + B.nx : (r >= B.nx ? r - B.nx : r);
                const bool out_row = (q >= 2) && (q < T.nrows + 2);
                uint32_t bytes = seg_bytes;
                if (NEED_FN && out_row) bytes += row_bytes;
                if (NEED_U && out_row) bytes += row_bytes;
                double* dst = smem + slot * SLOT;
                mbar_arrive_expect_tx(&full_bar[slot], bytes);
                bulk_g2s(dst, A.f_s + rowbase(rs) + T.j0 - 2, seg_bytes, &full_bar[slot]);
                if (NEED_FN && out_row) bulk_g2s(dst + SEG, A.f_n + rowbase(r) + T.j0, row_bytes, &full_bar[slot]);
                if (NEED_U && out_row) bulk_g2s(dst + SEG + TV, A.u_in + rowbase(r) + T.j0, row_bytes, &full_bar[slot]);
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int cl = 2 * tid;                      // tile-local column of my first cell
    const bool act0 = cl < T.ncols, act1 = (cl + 1) < T.ncols;
    const int c0 = T.j0 + cl;                    // block-local interior column
    const double vb0 = A.v_lo + ((double)(B.lo_v + c0) + 0.5) * A.dv;   // exact cell averages
    const double vb1 = vb0 + A.dv;
    const double vbm = vb0 - A.dv, vbp = vb1 + A.dv;
    const double dv24 = A.dv * (1.0 / 24.0);
    const double rdx = 1.0 / A.dx, rdv = 1.0 / A.dv;
    const double* E = sE + 2 - T.x0;             // E[i] for block-local row i (x0-2 <= i <= x0+nrows+1)
    // SELF: the thread holding domain cells (0,1) computes the low v-ghosts, the one holding
    // (nv-2, nv-1) the high ones
    const bool lo_edge = SELF && (B.lo_v + c0 == 0);
    const bool hi_edge = SELF && (B.lo_v + c0 + 1 == A.dom_v - 1);
    const double* Ebc = sEbc + 2 - T.x0;

    double W[4][4];                              // f_s rows r-3..r at columns c0-1..c0+2
    double vfm[3], vf0[3], vfp[3];               // v-faces c0-1/2, c0+1/2, c0+3/2 of rows i-1, i, i+1
    double Fxp0 = 0.0, Fxp1 = 0.0;               // x-fluxes at i-1/2
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) W[a][b] = 0.0;
#pragma unroll
    for (int m = 0; m < 3; ++m) { vfm[m] = vf0[m] = vfp[m] = 0.0; }

    for (int q = 0; q < Q; ++q) {
        const int slot = q % NSLOT;
        const int r = T.x0 - 2 + q;
        mbar_wait(&full_bar[slot], (q / NSLOT) & 1);
        const double* seg = smem + slot * SLOT;
        const double2 pa = lds2(seg + cl), pb = lds2(seg + cl + 2), pc = lds2(seg + cl + 4);
        // columns c0-2 .. c0+3
        double v0 = pa.x, v1 = pa.y, v2 = pb.x, v3 = pb.y, v4 = pc.x, v5 = pc.y;
        if (SELF && (lo_edge || hi_edge)) {      // characteristic BC (reading #6), a = -E_bc
            const double a = -Ebc[r];
            if (lo_edge) {
                if (a < 0.0) {
                    v1 = 4.0 * v2 - 6.0 * v3 + 4.0 * v4 - v5;
                    v0 = 10.0 * v2 - 20.0 * v3 + 15.0 * v4 - 4.0 * v5;
                } else {
                    v1 = __ldg(A.f0v + 1);
                    v0 = __ldg(A.f0v + 0);
                }
            }
            if (hi_edge) {
                if (a > 0.0) {
                    v4 = 4.0 * v3 - 6.0 * v2 + 4.0 * v1 - v0;
                    v5 = 10.0 * v3 - 20.0 * v2 + 15.0 * v1 - 4.0 * v0;
                } else {
                    v4 = __ldg(A.f0v + A.dom_v + 2);
                    v5 = __ldg(A.f0v + A.dom_v + 3);
                }
            }
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) { W[0][b] = W[1][b]; W[1][b] = W[2][b]; W[2][b] = W[3][b]; }
        W[3][0] = v1; W[3][1] = v2; W[3][2] = v3; W[3][3] = v4;

        double Fxn0 = 0.0, Fxn1 = 0.0;
        if (q >= 3) {                            // x-face (r-2)+1/2 from rows r-3..r
            const double xm = face_avg<RECON>(W[0][0], W[1][0], W[2][0], W[3][0], vbm);
            const double x0 = face_avg<RECON>(W[0][1], W[1][1], W[2][1], W[3][1], vb0);
            const double x1 = face_avg<RECON>(W[0][2], W[1][2], W[2][2], W[3][2], vb1);
            const double xp = face_avg<RECON>(W[0][3], W[1][3], W[2][3], W[3][3], vbp);
            Fxn0 = vb0 * x0 + dv24 * (x1 - xm);
            Fxn1 = vb1 * x1 + dv24 * (xp - x0);
        }
        if (q >= 4) {                            // output row i = r - 2
            const int i = r - 2;
            const double Ei = E[i], Em = E[i - 1], Ep = E[i + 1];
            const double c48 = (Ep - Em) * (1.0 / 48.0);
            const double Fv0 = Ei * vf0[0] + c48 * (vfp[0] - vfm[0]);
            const double Fv1 = Ei * vf0[1] + c48 * (vfp[1] - vfm[1]);
            const double Fv2 = Ei * vf0[2] + c48 * (vfp[2] - vfm[2]);
            const double k0 = (Fv1 - Fv0) * rdv - (Fxn0 - Fxp0) * rdx;
            const double k1 = (Fv2 - Fv1) * rdv - (Fxn1 - Fxp1) * rdx;
            const double fs0 = W[1][1], fs1 = W[1][2];
            const double* oseg = smem + ((q - 2) % NSLOT) * SLOT;
            double o0, o1;
            if (STAGE == 0) {
                o0 = k0; o1 = k1;
            } else if (STAGE == 1) {
                o0 = fs0 + (0.5 * A.dt) * k0;
                o1 = fs1 + (0.5 * A.dt) * k1;
            } else {
                const double2 fn = lds2(oseg + SEG + cl);
                if (STAGE == 2) {
                    const double u0 = fn.x + (fs0 - fn.x) * (1.0 / 3.0) + (A.dt * (1.0 / 3.0)) * k0;
                    const double u1 = fn.y + (fs1 - fn.y) * (1.0 / 3.0) + (A.dt * (1.0 / 3.0)) * k1;
                    double* up = A.u_out + rowbase(i) + c0;
                    if (act1) *reinterpret_cast<double2*>(up) = make_double2(u0, u1);
                    else if (act0) up[0] = u0;
                    o0 = fn.x + (0.5 * A.dt) * k0;
                    o1 = fn.y + (0.5 * A.dt) * k1;
                } else if (STAGE == 3) {
                    o0 = fn.x + A.dt * k0;
                    o1 = fn.y + A.dt * k1;
                } else {
                    const double2 uu = lds2(oseg + SEG + TV + cl);
                    o0 = uu.x + (fs0 - fn.x) * (1.0 / 3.0) + (A.dt * (1.0 / 6.0)) * k0;
                    o1 = uu.y + (fs1 - fn.y) * (1.0 / 3.0) + (A.dt * (1.0 / 6.0)) * k1;
                }
            }
            double* op = A.f_next + rowbase(i) + c0;
            if (act1) *reinterpret_cast<double2*>(op) = make_double2(o0, o1);
            else if (act0) op[0] = o0;
            if (A.rho != nullptr) {
                double s = (act0 ? o0 : 0.0) + (act1 ? o1 : 0.0);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) psum[warp * T.nrows + (i - T.x0)] = s;
            }
        }
        if (q >= 2) {                            // slot of row r-2 fully consumed
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[(q - 2) % NSLOT]);
        }
        Fxp0 = Fxn0; Fxp1 = Fxn1;
        // v-faces of row r (c0-1/2, c0+1/2, c0+3/2); speed a = -E_r
        const double ar = -E[r];
#pragma unroll
        for (int m = 0; m < 3; ++m) { vfm[m] = vf0[m]; vf0[m] = vfp[m]; }
        vfp[0] = face_avg<RECON>(v0, v1, v2, v3, ar);
        vfp[1] = face_avg<RECON>(v1, v2, v3, v4, ar);
        vfp[2] = face_avg<RECON>(v2, v3, v4, v5, ar);
    }

    if (A.rho != nullptr) {
        named_bar_sync(1, NT);
        for (int rr = tid; rr < T.nrows; rr += NT) {
            double s = psum[rr];
#pragma unroll
            for (int w = 1; w < NW; ++w) s += psum[w * T.nrows + rr];
            A.partials[(int64_t)T.pvt * A.dom_x + B.lo_x + T.x0 + rr] = s;
        }
        // last CTA of this row strip finalises rho in v-tile order (deterministic)
        __threadfence();
        named_bar_sync(1, NT);
        if (tid == 0) s_ticket = atomicAdd(A.tickets + T.strip, 1u);
        named_bar_sync(1, NT);
        if (s_ticket == (unsigned)(A.n_vtiles - 1)) {
            __threadfence();
            for (int rr = tid; rr < T.nrows; rr += NT) {
                const int x = B.lo_x + T.x0 + rr;
                double s = 0.0;
                for (int t = 0; t < A.n_vtiles; ++t) s += __ldcg(A.partials + (int64_t)t * A.dom_x + x);
                A.rho[x] = 1.0 - A.dv * s;
            }
            if (tid == 0) A.tickets[T.strip] = 0u;     // reset for the next launch
        }
    }
}

template <int STAGE, int RECON, int NT, bool SELF>
static int launch_t(const StageArgs1& A, int ntiles, int tile_rows, cudaStream_t st) {
    using SG = StageGeom<STAGE, NT>;
    const size_t smem = (size_t)(SG::NSLOT * SG::SLOT + (NT / 32) * tile_rows + 2 * (tile_rows + 4)) * sizeof(double);
    auto kern = k_stage_1d1v<STAGE, RECON, NT, SELF>;
    static bool configured = false;   // per template instantiation
    if (!configured) {
        VK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    kern<<<ntiles, NT + 32, smem, st>>>(A);
    VK_LAUNCH("k_stage_1d1v");
    return VLASOV_OK;
}

template <int RECON, int NT, bool SELF>
static int dispatch_stage(int stage, const StageArgs1& A, int ntiles, int tile_rows, cudaStream_t st) {
    switch (stage) {
        case 0: return launch_t<0, RECON, NT, SELF>(A, ntiles, tile_rows, st);
        case 1: return launch_t<1, RECON, NT, SELF>(A, ntiles, tile_rows, st);
        case 2: return launch_t<2, RECON, NT, SELF>(A, ntiles, tile_rows, st);
        case 3: return launch_t<3, RECON, NT, SELF>(A, ntiles, tile_rows, st);
        case 4: return launch_t<4, RECON, NT, SELF>(A, ntiles, tile_rows, st);
    }
    return fail(VLASOV_EINVAL, "stage must be 1..4");
}

template <int NT, bool SELF>
static int dispatch_recon(int recon, int stage, const StageArgs1& A, int nt, int rows, cudaStream_t st) {
    return recon == VLASOV_UPWIND ? dispatch_stage<VLASOV_UPWIND, NT, SELF>(stage, A, nt, rows, st)
                                  : dispatch_stage<VLASOV_CENTERED4, NT, SELF>(stage, A, nt, rows, st);
}

// CTAs per SM of the most demanding stage instance (stage 4), for one-wave tiling.
int stage_1d1v_ctas_per_sm(bool wide, int tile_rows) {
    int n = 0;
    cudaError_t e;
    if (wide) {
        using SG = StageGeom<4, 128>;
        const size_t smem = (size_t)(SG::NSLOT * SG::SLOT + 4 * tile_rows + 2 * (tile_rows + 4)) * sizeof(double);
        auto k = k_stage_1d1v<4, VLASOV_CENTERED4, 128, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 128 + 32, smem);
    } else {
        using SG = StageGeom<4, 32>;
        const size_t smem = (size_t)(SG::NSLOT * SG::SLOT + 1 * tile_rows + 2 * (tile_rows + 4)) * sizeof(double);
        auto k = k_stage_1d1v<4, VLASOV_CENTERED4, 32, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 32 + 32, smem);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int launch_stage_1d1v(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s, double* u,
                      double* f_next, const double* E, const double* E_bc, const double* f0v, int recon,
                      double* rho) {
    StageArgs1 A;
    A.f_s = f_s;
    A.f_n = f_n;
    A.u_in = u;
    A.u_out = u;
    A.f_next = f_next;
    A.E = E;
    A.E_bc = E_bc;
    A.f0v = f0v;
    A.rho = rho;
    A.partials = L->d_partials;
    A.tickets = L->d_tickets;
    A.blocks = L->d_blocks1;
    A.dt = dt;
    A.dx = L->h[0];
    A.dv = L->h[1];
    A.v_lo = L->lower[1];
    A.dom_x = L->dom[0];
    A.dom_v = L->dom[1];
    A.n_vtiles = L->n_vtiles;
    A.tile_rows = L->tile_rows;
    const bool self = (E_bc != nullptr && f0v != nullptr);
    const bool wide = !L->h_tiles_wide.empty();
    A.tiles = wide ? L->d_tiles_wide : L->d_tiles_narrow;
    const int nt = (int)(wide ? L->h_tiles_wide.size() : L->h_tiles_narrow.size());
    if (nt == 0) return VLASOV_OK;
    const int rows = L->tile_rows;
    if (wide) {
        return self ? dispatch_recon<128, true>(recon, stage, A, nt, rows, L->stream)
                    : dispatch_recon<128, false>(recon, stage, A, nt, rows, L->stream);
    }
    return self ? dispatch_recon<32, true>(recon, stage, A, nt, rows, L->stream)
                : dispatch_recon<32, false>(recon, stage, A, nt, rows, L->stream);
}

}  // namespace vk
