// 1D+1V fused RK4 stage kernel: face averages -> fluxes -> divergence -> RK4 stage combine ->
// per-(x-row, v-tile) partial sums of the new stage state.
//
// PAPER.md: face averages P:322-368, fluxes P:263-282 (+1/48, reading #3), divergence
// P:246-250, RK4 P:389-410 (minimum-traffic rearrangement, see include/vlasov.h), moment
// P:295-297.
//
// Design (B200): one CTA owns a v-segment of TV = 2*NT contiguous cells and marches along x
// over `nrows` rows.  A producer warp streams each ghosted row segment of f_s (and the matching
// f_n / u rows) into an NSLOT-deep shared-memory ring with cp.async.bulk (TMA engine) completing
// on mbarriers; NT consumer threads own two adjacent v-cells each, keep a 4-row register window
// of f_s, compute every face once per row from registers, and release ring slots through
// "empty" mbarriers.  Every HBM byte of f_s is read once per tile (+4 halo rows, L2 hits),
// f_n / u are read once, f_next / u written once: 16/32/24/32 B per cell for stages 1..4.
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
    double* partials;          // [n_vtiles][dom_x] or null
    const Tile1* tiles;
    const Block1* blocks;
    double dt, dx, dv, v_lo;   // v_lo: physical lower velocity of the level domain
    int dom_x;
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

template <int STAGE, int RECON, int NT, int NSLOT>
__global__ void __launch_bounds__(NT + 32) k_stage_1d1v(const StageArgs1 A) {
    constexpr int TV = 2 * NT;
    constexpr int SEG = TV + 4;
    constexpr bool NEED_FN = (STAGE >= 2);
    constexpr bool NEED_U = (STAGE == 4);
    constexpr int SLOT = SEG + (NEED_FN ? TV : 0) + (NEED_U ? TV : 0);
    constexpr int NW = NT / 32;

    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full_bar[NSLOT];
    __shared__ __align__(8) uint64_t empty_bar[NSLOT];
    double* psum = smem + NSLOT * SLOT;          // [NW][nrows]

    const Tile1 T = A.tiles[blockIdx.x];
    const Block1 B = A.blocks[T.block];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int Q = T.nrows + 4;
    const int wpad = (T.ncols + 1) & ~1;

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
                const bool out_row = (q >= 2) && (q < T.nrows + 2);
                uint32_t bytes = seg_bytes;
                if (NEED_FN && out_row) bytes += row_bytes;
                if (NEED_U && out_row) bytes += row_bytes;
                double* dst = smem + slot * SLOT;
                const int64_t rb = rowbase(r) + T.j0;
                mbar_arrive_expect_tx(&full_bar[slot], bytes);
                bulk_g2s(dst, A.f_s + rb - 2, seg_bytes, &full_bar[slot]);
                if (NEED_FN && out_row) bulk_g2s(dst + SEG, A.f_n + rb, row_bytes, &full_bar[slot]);
                if (NEED_U && out_row) bulk_g2s(dst + SEG + TV, A.u_in + rb, row_bytes, &full_bar[slot]);
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
    const double* E = A.E + B.lo_x + G;          // E[i] for block-local row i (i >= -2)

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
        mbar_wait(&full_bar[slot], (q / NSLOT) & 1);
        const double* seg = smem + slot * SLOT;
        const double2 pa = lds2(seg + cl), pb = lds2(seg + cl + 2), pc = lds2(seg + cl + 4);
        // columns c0-2 .. c0+3
        const double v0 = pa.x, v1 = pa.y, v2 = pb.x, v3 = pb.y, v4 = pc.x, v5 = pc.y;
#pragma unroll
        for (int b = 0; b < 4; ++b) { W[0][b] = W[1][b]; W[1][b] = W[2][b]; W[2][b] = W[3][b]; }
        W[3][0] = v1; W[3][1] = v2; W[3][2] = v3; W[3][3] = v4;
        const int r = T.x0 - 2 + q;

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
            const double Ei = __ldg(E + i), Em = __ldg(E + i - 1), Ep = __ldg(E + i + 1);
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
            if (A.partials != nullptr) {
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
        const double ar = -__ldg(E + r);
#pragma unroll
        for (int m = 0; m < 3; ++m) { vfm[m] = vf0[m]; vf0[m] = vfp[m]; }
        vfp[0] = face_avg<RECON>(v0, v1, v2, v3, ar);
        vfp[1] = face_avg<RECON>(v1, v2, v3, v4, ar);
        vfp[2] = face_avg<RECON>(v2, v3, v4, v5, ar);
    }

    if (A.partials != nullptr && T.pvt >= 0) {
        named_bar_sync(1, NT);
        for (int rr = tid; rr < T.nrows; rr += NT) {
            double s = psum[rr];
#pragma unroll
            for (int w = 1; w < NW; ++w) s += psum[w * T.nrows + rr];
            A.partials[(int64_t)T.pvt * A.dom_x + B.lo_x + T.x0 + rr] = s;
        }
    }
}

template <int STAGE, int RECON, int NT, int NSLOT>
static int launch_t(const StageArgs1& A, int ntiles, int tile_rows, cudaStream_t st) {
    constexpr int TV = 2 * NT;
    constexpr int SEG = TV + 4;
    constexpr int SLOT = SEG + (STAGE >= 2 ? TV : 0) + (STAGE == 4 ? TV : 0);
    const size_t smem = (size_t)(NSLOT * SLOT + (NT / 32) * tile_rows) * sizeof(double);
    auto kern = k_stage_1d1v<STAGE, RECON, NT, NSLOT>;
    static bool configured = false;   // per template instantiation
    if (!configured) {
        VK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    kern<<<ntiles, NT + 32, smem, st>>>(A);
    VK_LAUNCH("k_stage_1d1v");
    return VLASOV_OK;
}

template <int RECON, int NT>
static int dispatch_stage(int stage, const StageArgs1& A, int ntiles, int tile_rows, cudaStream_t st) {
    constexpr int NSLOT = 8;
    switch (stage) {
        case 0: return launch_t<0, RECON, NT, NSLOT>(A, ntiles, tile_rows, st);
        case 1: return launch_t<1, RECON, NT, NSLOT>(A, ntiles, tile_rows, st);
        case 2: return launch_t<2, RECON, NT, NSLOT>(A, ntiles, tile_rows, st);
        case 3: return launch_t<3, RECON, NT, NSLOT>(A, ntiles, tile_rows, st);
        case 4: return launch_t<4, RECON, NT, NSLOT>(A, ntiles, tile_rows, st);
    }
    return fail(VLASOV_EINVAL, "stage must be 1..4");
}

int launch_stage_1d1v(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s,
                      double* u, double* f_next, const double* E, int recon, double* partials) {
    StageArgs1 A;
    A.f_s = f_s;
    A.f_n = f_n;
    A.u_in = u;
    A.u_out = u;
    A.f_next = f_next;
    A.E = E;
    A.partials = partials;
    A.blocks = L->d_blocks1;
    A.dt = dt;
    A.dx = L->h[0];
    A.dv = L->h[1];
    A.v_lo = L->lower[1];
    A.dom_x = L->dom[0];
    const bool wide = !L->h_tiles_wide.empty();
    A.tiles = wide ? L->d_tiles_wide : L->d_tiles_narrow;
    const int nt = (int)(wide ? L->h_tiles_wide.size() : L->h_tiles_narrow.size());
    if (nt == 0) return VLASOV_OK;
    if (wide) {
        return recon == VLASOV_UPWIND ? dispatch_stage<VLASOV_UPWIND, 128>(stage, A, nt, L->tile_rows, L->stream)
                                      : dispatch_stage<VLASOV_CENTERED4, 128>(stage, A, nt, L->tile_rows, L->stream);
    }
    return recon == VLASOV_UPWIND ? dispatch_stage<VLASOV_UPWIND, 32>(stage, A, nt, L->tile_rows, L->stream)
                                  : dispatch_stage<VLASOV_CENTERED4, 32>(stage, A, nt, L->tile_rows, L->stream);
}

}  // namespace vk
