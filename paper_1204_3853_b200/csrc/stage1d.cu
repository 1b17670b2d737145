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

#include <cstdlib>
#include <type_traits>

#include "internal.h"
#include "ptx.cuh"
#include "scheme.cuh"

namespace vk {

// STAGE1D_TRACE (experiments only): per-CTA %globaltimer stamps of the kernel's phases, read back
// with vlasov_debug_stage_trace (not part of the C ABI of include/vlasov.h)
#ifdef STAGE1D_TRACE
__device__ unsigned long long g_trace[2048][10];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TRACE(i) do { if (threadIdx.x == 0 && blockIdx.x < 2048) g_trace[blockIdx.x][i] = gtimer(); } while (0)
#else
#define TRACE(i) do { } while (0)
#endif

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
    double rho_base;           // fused moment: rho = rho_base - dv sum_v f (1 unless a velocity slab)
    int phys_lo, phys_hi;      // SELF: velocity faces with the characteristic BC (else slab faces)
    int dom_x, dom_v, n_vtiles, tile_rows;
    // fused constraint evaluation (vlasov_rk4_stage_vp): E of the stage state from its moment
    const double* rho_in;      // nullable: rho of f_s (dom_x values); then E is computed and written
    const double* gE;          // Green's function of E = -D4 phi(rho) (Poisson plan, dom_x values)
    double* E_out;             // ghosted level E array (owned rows + periodic ghosts)
    int cluster;               // CTAs per cluster of the fused launch (the v-tiles of a strip)
    int g_smem;                // fused field: gX staged in shared memory too
    const double* gX;          // gX[m] = g[(m - GX_PAD) mod n], m in [0, 2n + GX_PAD + GX_TAIL)
    // O(n) field (split of the exact Green's function): E_i = K2 (sum r - r_i)
    //   - Kn (i sum r - sum_k k r_k + n sum_{k>i} r_k) + sum_{|m|<=HM} hs[m + HM] r_{i-m}
    const double* hs;          // nullable: the fast-decaying part h(m), m = -HM .. HM
    double K2, Kn;             // dx / 2, dx / n
    int nstrip1;               // > 0: single block, tiles computed from blockIdx (no table load)
    Block1 blk0;               // that block
    int xshift;                // single block: strips start xshift rows later (periodic wrap; L2 reuse)
    int l2hint;                // L2 eviction priorities per field (single periodic block; see `issue`)
};

// the fused prologue stages the whole (periodically extended) Green's function in shared memory
// for n <= G_SMEM_MAX_N (two CTAs per SM still fit); larger n reads it through L1
constexpr int G_SMEM_MAX_N = 2048;
static bool g_in_smem(int n) { return n <= G_SMEM_MAX_N; }
// shared memory of the fused field prologue: rho [n], row results [PART_MAX >= tile_rows + 4],
// the window of gX the CTA's rows need [<= n + PART_MAX + 32]
constexpr int PART_MAX = 136;
static size_t field_smem_bytes(int n, bool split = false) {
    if (split) return (size_t)(n + PART_MAX + 2 * (n / 32 + 2) + 8) * sizeof(double);
    return (size_t)(n + PART_MAX + (g_in_smem(n) ? n + PART_MAX + 32 : 0)) * sizeof(double);
}
constexpr int EROWS = 8;   // rows of E per warp group in the fused prologue (Toeplitz blocking)
constexpr int HM = 16;     // half-width of the local part of the split Green's function

#ifndef STAGE1D_SEL1
#define STAGE1D_SEL1 1   // experiments: 0 drops stage 1's boundary select (wrong BC, timing only)
#endif
// CPT = 4 cells per consumer thread, TV = 4*NT cells per v-tile.
#ifndef STAGE1D_CPT
#define STAGE1D_CPT 4
#endif
constexpr int CPT = STAGE1D_CPT;
#ifndef STAGE1D_MINB
#define STAGE1D_MINB 2
#endif
#ifndef RING_KB
#define RING_KB 48
#endif
// programmatic dependent launch of the stage kernels: a stage triggers its dependents when its
// march is done, so the next stage's launch and setup overlap this one's tail (C4 graph step
// 179 vs 185 us; triggering at kernel start measured slower, 195 us).  Only constants are read
// before griddep_wait.
#ifndef STAGE1D_PDL
#define STAGE1D_PDL 1
#endif
#ifndef STAGE1D_PDL_EARLY
#define STAGE1D_PDL_EARLY 0
#endif
// 1: a dedicated producer warp issues the TMA ring; 0: thread 0 of the consumers issues it (no
// extra warp: 4 warps x 168 registers lets 3 CTAs share an SM instead of 2)
#ifndef STAGE1D_PRODUCER
#define STAGE1D_PRODUCER 1
#endif
// STAGE1D_PWG 1: for the wide tiles the producer is a whole warpgroup (4 warps, one of which issues
// the ring) that hands its registers to the consumer warpgroup with setmaxnreg (launch: 256 x 128
// registers; producer 24, consumers 232 -- no spills in the row march)
#ifndef STAGE1D_PWG
#define STAGE1D_PWG 1
#endif
template <int NT>
struct Roles {
    static constexpr bool PWG = STAGE1D_PWG && NT == 128;
    static constexpr int PWARPS = PWG ? 4 : STAGE1D_PRODUCER;
    static constexpr int THREADS = NT + 32 * PWARPS;
};
constexpr int PWG_PRODUCER_REGS = 24, PWG_CONSUMER_REGS = 232;
constexpr int NT_WIDE = 128, NT_NARROW = 32;   // consumer threads per CTA

template <int STAGE, int NT>
struct StageGeom {
    static constexpr int TV = CPT * NT;
    static constexpr int SEG = TV + 4;                       // f_s row segment incl. 2+2 halo columns
    static constexpr int NFN = STAGE >= 2 ? 1 : 0;           // f_n row (stages 2, 3) or u row (stage 4)
    static constexpr int SLOT = SEG + NFN * TV;              // doubles per ring slot
    // ring depth: ~RING_KB of row data per CTA, 3..16 slots (a slot is consumed in one row step)
    // ring size per stage (measured on C4: stage 2 best at 48 KB, stages 1, 3 and 4 at 64 KB)
#ifdef RING_KB_ALL
    static constexpr int RKB = RING_KB_ALL;
#else
    static constexpr int RKB = STAGE == 2 ? RING_KB : 64;
#endif
    static constexpr int NSLOT_RAW = (RKB * 1024) / (SLOT * 8);
    static constexpr int NSLOT = NSLOT_RAW < 4 ? 4 : (NSLOT_RAW > 16 ? 16 : NSLOT_RAW);
    static constexpr int NW = NT / 32;
    static size_t smem_bytes(int tile_rows) {
        return (size_t)(NSLOT * SLOT + NW * tile_rows + 2 * (tile_rows + 4) + 2 * CPT * tile_rows) * sizeof(double);
    }
};

// Ring slot of row step q (row r = x0 - 2 + q): [ f_s(r, j0-2 .. j0+TV+1) | f_n(r-2, j0..) or u(r-2, j0..) ];
// the f_n / u row is that of the output row i = r - 2 (q >= 4), so every slot is consumed
// completely in its own row step and released at once.
// GM (ghost mode of f_s): 0 = ghost frame read from memory (any level); 1 = one periodic block,
// x wrapped in-kernel, velocity ghosts derived from E_bc; 2 = one periodic block, velocity ghosts
// carried in memory (written by the stage that produced f_s)
template <int STAGE, int RECON, int NT, int GM>
__global__ void __launch_bounds__(Roles<NT>::THREADS, STAGE1D_MINB) k_stage_1d1v(const StageArgs1 A) {
    constexpr int PWARPS = Roles<NT>::PWARPS;
    constexpr bool PWG = Roles<NT>::PWG;
    using SG = StageGeom<STAGE, NT>;
    constexpr int TV = SG::TV, SEG = SG::SEG, SLOT = SG::SLOT, NSLOT = SG::NSLOT, NW = SG::NW;
    // GM bit 2: the O(n) split field (VLASOV_FIELD=split) instead of the cluster Toeplitz rows --
    // a compile-time variant, so the default kernel carries none of its code or registers
    constexpr bool SPLIT = (GM & 4) != 0;
    constexpr int GMODE = GM & 3;
    constexpr bool SELF = (GMODE != 0);
    constexpr bool NEED_FN = (STAGE == 2 || STAGE == 3);     // stage 4 reads u only (u holds no f_n term)
    constexpr bool NEED_U = (STAGE == 4);

    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full_bar[NSLOT];
    __shared__ __align__(8) uint64_t empty_bar[NSLOT];
    __shared__ __align__(8) uint64_t field_bar;
    __shared__ __align__(8) uint64_t e_bar;      // fused field: all Q rows of E have landed
    __shared__ __align__(8) uint64_t ready_bar[NSLOT];   // stage 1, carried ghosts: slot's ghosts decided
    __shared__ __align__(8) uint64_t e_ready;    // stage 1, carried ghosts: the tile's E rows are in sE
    __shared__ unsigned s_ticket;
    __shared__ double s_f0[4];                   // f0v at v-ghost columns -2, -1, nv, nv + 1 (SELF)
    __shared__ uint32_t s_dep[NT];               // slot-release dependency sink (see the row step)
    double* psum = smem + NSLOT * SLOT;          // [NW][tile_rows]

    TRACE(0);
#if STAGE1D_PDL_EARLY
    // programmatic dependent launch: the next stage may be scheduled as this grid's CTAs retire;
    // everything before griddep_wait() below touches only constants (tiles, f0v, gX)
    griddep_launch_dependents();
#endif
#ifdef STAGE1D_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 2048) { unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); g_trace[blockIdx.x][8] = sm; }
#endif
    Tile1 T;
    Block1 B;
    if (A.nstrip1 > 0) {                         // single block: the tiling of build_tiles_1d
        B = A.blk0;
        const int st = blockIdx.x / A.n_vtiles, vt = blockIdx.x - st * A.n_vtiles;
        T.block = 0;
        T.x0 = (int)((int64_t)B.nx * st / A.nstrip1);
        T.nrows = (int)((int64_t)B.nx * (st + 1) / A.nstrip1) - T.x0;
        T.x0 += A.xshift;                        // rows x0 .. x0+nrows-1 taken mod nx (wr below)
        T.j0 = vt * TV;
        T.ncols = min(TV, B.nv - T.j0);
        T.pvt = vt;
        T.strip = st;
    } else {
        T = A.tiles[blockIdx.x];
        B = A.blocks[T.block];
    }
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int Q = T.nrows + 4;
    const int wpad = (T.ncols + 1) & ~1;
    double* sE = psum + NW * A.tile_rows;        // E of rows x0-2 .. x0+nrows+1
    double* sEbc = sE + (A.tile_rows + 4);       // E_bc of the same rows (SELF)
    const bool field = SELF && (A.rho_in != nullptr);
    // one mbarrier per thread (sequential inits by one thread cost ~35 ns each, ~1 us for a
    // 12-slot ring); every initialising thread fences its own inits
    if (tid < 3 * NSLOT + 3) {
        uint64_t* bar = tid < NSLOT ? &full_bar[tid] : tid < 2 * NSLOT ? &empty_bar[tid - NSLOT]
                      : tid == 2 * NSLOT ? &field_bar : tid == 2 * NSLOT + 1 ? &e_bar
                      : tid == 2 * NSLOT + 2 ? &e_ready : &ready_bar[tid - 2 * NSLOT - 3];
        mbar_init(bar, (tid >= NSLOT && tid < 2 * NSLOT) ? (uint32_t)NW : 1u);
        fence_mbar_init();
    }
    // Stage 1 with carried ghosts (reading #6b): f_n's ghost columns hold the outgoing candidate
    // (stage 4 wrote the cubic extrapolation); the direction is decided with this stage's own
    // field E = E(f_n).  In the edge v-tiles a helper warp of the producer warpgroup keeps the
    // candidate or puts the unperturbed profile into every landed slot, so the consumers of those
    // tiles (which would otherwise set the stage time) do no per-row boundary work.
    constexpr bool SEL1_ANY = STAGE1D_SEL1 && (GMODE == 2 && STAGE == 1);
    constexpr bool SEL1H = SEL1_ANY && PWG;
    const bool sel_lo = SEL1H && A.phys_lo && (B.lo_v + T.j0 == 0);
    const bool sel_hi = SEL1H && A.phys_hi && (B.lo_v + T.j0 + T.ncols == A.dom_v);
    const bool sel_cta = sel_lo || sel_hi;
    // fused field in a cluster (the v-tiles of one row strip): every CTA's barrier is initialised
    // and armed before any CTA pushes E rows into its shared memory
    const bool toep = field && !SPLIT;  // Toeplitz field: rows split over the strip's cluster
    const uint32_t crank = toep ? cluster_ctarank() : 0u, csize = toep ? cluster_nctarank() : 1u;
    __syncthreads();
    // (after the barrier that orders the inits; before this thread's cluster arrive, so no remote
    // push can reach e_bar first)
    if (tid == 0 && csize > 1) mbar_arrive_expect_tx(&e_bar, (uint32_t)Q * 8u);
    // consumers arrive now and wait only before their first remote store; the producer waits at once
    if (toep && csize > 1) {
        if (PWARPS && warp >= NW) cluster_sync_all();
        else cluster_arrive();
    }
    TRACE(1);

    // row r (block-local interior index, may be -2..nx+1): interior column 0 of that row
    auto rowbase = [&](int r) -> int64_t { return B.off + (int64_t)(r + G) * B.pitch + G; };
    // single block: a shifted strip may run past the last row; its rows wrap periodically
    const int wrapn = A.nstrip1 > 0 ? B.nx : 0x40000000;
    auto wr = [&](int r) -> int { return r >= wrapn ? r - wrapn : r; };

    // fused field: rho and the Green's function (twice: periodic extension) staged by the TMA engine
    double* s_edge = sEbc + (A.tile_rows + 4);   // [tile_rows][2 sides][CPT] boundary cells of f_next
    double* f_rho = s_edge + 2 * CPT * A.tile_rows;
    const uint32_t seg_bytes = (uint32_t)(wpad + 4) * 8u;
    const uint32_t row_bytes = (uint32_t)wpad * 8u;
    // TMA loads of row step q into ring slot `sl`
    auto issue = [&](int q, int sl) {
        const int r = T.x0 - 2 + q;
        int rs = r;
        if (SELF) rs = (r < 0) ? r + B.nx : (r >= B.nx ? r - B.nx : r);
        else rs = wr(r);
        const bool out_row = (q >= 4);
        uint32_t bytes = seg_bytes;
        if (NEED_FN && out_row) bytes += row_bytes;
        if (NEED_U && out_row) bytes += row_bytes;
        double* dst = smem + sl * SLOT;
        mbar_arrive_expect_tx(&full_bar[sl], bytes);
        if (A.l2hint) {
            // L2 residency by reuse distance (4 fields of the level size, an L2 of about two): f_n
            // is read by stages 1-3 and overwritten in place by stage 4 -> kept (evict_last, the
            // stage-4 store too); a stage state f_2, f_3, f_4 and u are dead once read -> evict_first;
            // f_next is stored with the default priority (the next stage reads it, strip-shifted).
            bulk_g2s_hint(dst, A.f_s + rowbase(rs) + T.j0 - 2, seg_bytes, &full_bar[sl], STAGE <= 1 ? l2_evict_last() : l2_evict_first());
            if (NEED_FN && out_row)
                bulk_g2s_hint(dst + SEG, A.f_n + rowbase(wr(r - 2)) + T.j0, row_bytes, &full_bar[sl], STAGE == 2 ? l2_evict_last() : l2_evict_first());
            if (NEED_U && out_row) bulk_g2s_hint(dst + SEG, A.u_in + rowbase(wr(r - 2)) + T.j0, row_bytes, &full_bar[sl], l2_evict_first());
            return;
        }
        bulk_g2s(dst, A.f_s + rowbase(rs) + T.j0 - 2, seg_bytes, &full_bar[sl]);
        if (NEED_FN && out_row) bulk_g2s(dst + SEG, A.f_n + rowbase(wr(r - 2)) + T.j0, row_bytes, &full_bar[sl]);
        if (NEED_U && out_row) bulk_g2s(dst + SEG, A.u_in + rowbase(wr(r - 2)) + T.j0, row_bytes, &full_bar[sl]);
    };
    // fused field: this CTA computes rows [tb, te) of the tile's Q rows of E (the strip's v-tiles
    // of a cluster split them); row tb + t is x = gxu0 + t (unwrapped, gxu0 in [0, n)); they read
    // gX[ws, ws + wl) only (see the Toeplitz loop), staged in shared memory at f_g
    const int tb = (int)((int64_t)Q * crank / csize), te = (int)((int64_t)Q * (crank + 1) / csize);
    int gxu0 = B.lo_x + T.x0 - 2 + tb;
    gxu0 += (gxu0 < 0) ? A.dom_x : 0;
    gxu0 -= (gxu0 >= A.dom_x) ? A.dom_x : 0;
    const int ws = (GX_PAD + gxu0 - 14) & ~1;
    const int wl = ((GX_PAD + A.dom_x + gxu0 + (te - tb) + 8 - ws) + 1) & ~1;
    double* f_g = f_rho + A.dom_x + PART_MAX;      // gX[ws ..] staged (A.g_smem)
    // the producing thread: gX (a constant) before the grid dependency wait, rho after it
    auto issue_field_const = [&]() {
        if (field) {
            const uint32_t nb = (uint32_t)A.dom_x * 8u;
            const uint32_t ng = A.g_smem ? (uint32_t)wl * 8u : 0u;
            mbar_arrive_expect_tx(&field_bar, nb + ng);
            if (ng) bulk_g2s(f_g, A.gX + ws, ng, &field_bar);
        }
    };
    auto issue_field = [&]() {
        if (field) bulk_g2s(f_rho, A.rho_in, (uint32_t)A.dom_x * 8u, &field_bar);
    };
    if (PWARPS && warp >= NW) {                  // ---------------- producer warp(group)
        if (PWG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PWG_PRODUCER_REGS));
        if (warp == NW && lane == 0) {
            issue_field_const();
            griddep_wait();                      // f_s, f_n, u, rho of the previous stages
            issue_field();
            int slot = 0;
            uint32_t phase = 0;
            for (int q = 0; q < Q; ++q) {
                if (q >= NSLOT) mbar_wait(&empty_bar[slot], phase ^ 1u);
                issue(q, slot);
                if (++slot == NSLOT) { slot = 0; phase ^= 1u; }
            }
        }
        if (SEL1H && sel_cta && warp == NW + 1 && lane == 0) {
            mbar_wait(&e_ready, 0);
            const double* Er = sE + 2 - T.x0;
            int slot = 0;
            uint32_t phase = 0;
            for (int q = 0; q < Q; ++q) {
                mbar_wait(&full_bar[slot], phase);
                double* seg = smem + slot * SLOT;
                const double a = -Er[T.x0 - 2 + q];
                if (sel_lo && !(a < 0.0)) { seg[0] = s_f0[0]; seg[1] = s_f0[1]; }
                if (sel_hi && !(a > 0.0)) { seg[T.ncols + 2] = s_f0[2]; seg[T.ncols + 3] = s_f0[3]; }
                mbar_arrive(&ready_bar[slot]);
                if (++slot == NSLOT) { slot = 0; phase ^= 1u; }
            }
        }
        return;
    }
    if (PWG) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(PWG_CONSUMER_REGS));
    if (!PWARPS && tid == 0) issue_field_const();
    griddep_wait();                              // E, E_bc, f_s, f_n, u, rho of the previous stages
    for (int t = tid; t < Q; t += NT) {
        const int gi = B.lo_x + wr(T.x0 - 2 + t) + G;  // index in the ghosted level E array
        if (!field) sE[t] = __ldg(A.E + gi);
        if (SELF && A.E_bc && STAGE != 1) sEbc[t] = __ldg(A.E_bc + gi);
    }
    // the unperturbed profile at the velocity ghost columns (read after the setup barrier: a
    // global load there would sit on every CTA's start-up path)
    if (SELF && tid < 4) s_f0[tid] = __ldg(A.f0v + (tid < 2 ? tid : A.dom_v + tid));
    named_bar_sync(1, NT);
    if (!PWARPS && tid == 0) {                   // consumer thread 0 primes the ring
        issue_field();
        for (int q = 0; q < min(Q, NSLOT); ++q) issue(q, q);
    }

    // ---------------------------------------------------------------- consumers
    if (SPLIT && field) {
        // Constraint evaluation of the stage state (Alg.5) in O(n) per CTA: the exact
        // discrete Green's function of E = -D4 phi is a sawtooth plus a part decaying like
        // 0.0718^|m|, so with r = rho - mean
        //   E_i = K2 (sum r - r_i) - Kn (i sum r - sum_k k r_k + n S_i) + sum_{|m|<=HM} h(m) r_{i-m},
        //   S_i = sum_{k>i} r_k.
        // A CTA needs S_i for its Q consecutive rows only: S of its first row i0 is one more block
        // reduction (with sum r and sum k r_k), the others follow from S_{i+1} = S_i - r_{i+1}
        // (periodic rows: + sum r per wrap).  No cluster, no scan; fixed summation orders.
        const int n = A.dom_x;
        const double* s_rho = f_rho;
        double* s_w = f_rho + n + PART_MAX;      // [3 NW] warp partials of sum r, sum k r, S_{i0}
        mbar_wait(&field_bar, 0);
        TRACE(2);
        {   // mean: warp quarters, warp partials in warp order
            const int kb = (int)((int64_t)n * warp / NW), ke = (int)((int64_t)n * (warp + 1) / NW);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int k = kb + lane;
            for (; k + 96 < ke; k += 128) {
                a0 += s_rho[k]; a1 += s_rho[k + 32]; a2 += s_rho[k + 64]; a3 += s_rho[k + 96];
            }
            for (; k < ke; k += 32) a0 += s_rho[k];
            double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) psum[warp] = acc;
        }
        named_bar_sync(1, NT);
        double mean = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) mean += psum[w];
        mean /= (double)n;
        TRACE(3);
        int i0 = B.lo_x + T.x0 - 2;              // periodic row of tile row 0
        i0 += (i0 < 0) ? n : 0;
        i0 -= (i0 >= n) ? n : 0;
        i0 -= (i0 >= n) ? n : 0;
        {   // sum r, sum k r_k, S_{i0}: thread-strided partial sums, shuffle trees, warp order
            double q0 = 0.0, q1 = 0.0, q2 = 0.0;
            for (int k = tid; k < n; k += NT) {
                const double r = s_rho[k] - mean;
                q0 += r;
                q1 = fma((double)k, r, q1);
                q2 += (k > i0) ? r : 0.0;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                q0 += __shfl_xor_sync(0xffffffffu, q0, o);
                q1 += __shfl_xor_sync(0xffffffffu, q1, o);
                q2 += __shfl_xor_sync(0xffffffffu, q2, o);
            }
            if (lane == 0) { s_w[3 * warp] = q0; s_w[3 * warp + 1] = q1; s_w[3 * warp + 2] = q2; }
        }
        named_bar_sync(1, NT);
        double sumr = 0.0, T1 = 0.0, S0 = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) { sumr += s_w[3 * w]; T1 += s_w[3 * w + 1]; S0 += s_w[3 * w + 2]; }
        for (int t = tid; t < Q; t += NT) {
            const int wraps = (i0 + t) / n;                                // periodic wraps (Q may exceed n)
            const int i = i0 + t - wraps * n;                              // row of the periodic domain
            double pa = 0.0, pb = 0.0;           // sum_{s=1..t} r_{i0+s}: two interleaved partial sums
            {
                int k = i0 + 1;
                k -= (k >= n) ? n : 0;
                int sidx = 1;
                for (; sidx + 1 <= t; sidx += 2) {
                    const int k1 = (k + 1 >= n) ? k + 1 - n : k + 1;
                    pa += s_rho[k] - mean;
                    pb += s_rho[k1] - mean;
                    k = (k1 + 1 >= n) ? k1 + 1 - n : k1 + 1;
                }
                if (sidx <= t) pa += s_rho[k] - mean;
            }
            const double sgt = S0 - (pa + pb) + (double)wraps * sumr;      // S_i
            const double ri = s_rho[i] - mean;
            double e0 = A.K2 * (sumr - ri) - A.Kn * ((double)i * sumr - T1 + (double)n * sgt);
            double e1 = 0.0, e2 = 0.0;           // local part: three interleaved partial sums
#pragma unroll
            for (int m = -HM; m <= HM; ++m) {
                int k = i - m;
                k += (k < 0) ? n : 0;
                k -= (k >= n) ? n : 0;
                const double p = __ldg(A.hs + m + HM) * (s_rho[k] - mean);
                if ((m + HM) % 3 == 0) e0 += p; else if ((m + HM) % 3 == 1) e1 += p; else e2 += p;
            }
            const double e = e0 + (e1 + e2);
            sE[t] = e;
            if (T.pvt == 0 && t >= 2 && t < Q - 2) {     // owned rows + periodic ghosts, once per strip
                const int x = B.lo_x + wr(T.x0 - 2 + t);
                A.E_out[x + G] = e;
                if (x < G) A.E_out[x + G + n] = e;
                if (x >= n - G) A.E_out[x + G - n] = e;
            }
        }
        TRACE(4);
        named_bar_sync(1, NT);
    } else if (field) {
        // Constraint evaluation of the stage state (Alg.5) while the producer fills the
        // ring: E_i = sum_k g[(i - k) mod n] (rho_k - mean) for the rows of this tile (projection to
        // mean zero, applied on the fly), from rho and the periodically extended g staged
        // in shared memory by the TMA engine (through L1 for n > G_SMEM_MAX_N).
        const int n = A.dom_x;
        const double* s_rho = f_rho;
        double* s_part = f_rho + n;              // [Q] E of the tile rows
        mbar_wait(&field_bar, 0);
        TRACE(2);
        {   // mean: warp w sums the w-th quarter of rho (lanes strided), warp partials in warp order
            const int kb = (int)((int64_t)n * warp / NW), ke = (int)((int64_t)n * (warp + 1) / NW);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int k = kb + lane;
            for (; k + 96 < ke; k += 128) {
                a0 += s_rho[k]; a1 += s_rho[k + 32]; a2 += s_rho[k + 64]; a3 += s_rho[k + 96];
            }
            for (; k < ke; k += 32) a0 += s_rho[k];
            double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) psum[warp] = acc;
        }
        named_bar_sync(1, NT);
        double mean = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) mean += psum[w];
        mean /= (double)n;
        TRACE(3);
        // Rows [tb, te) of the tile are this CTA's share (the strip's v-tiles of a cluster compute
        // disjoint row ranges); each row is pushed into every CTA's s_part with st.async, which
        // completes on that CTA's e_bar.  Toeplitz blocking: a warp computes EROWS consecutive
        // rows; lane l sums over its own contiguous k-chunk [C l, C l + C) (C odd: conflict-free
        // shared-memory banks) with a sliding window of g, so each g value loaded serves EROWS
        // rows; fixed chunk order and transposed butterflies -> deterministic.
#ifdef STAGE1D_TRACE
        if (tid == 0 && blockIdx.x < 2048) { g_trace[blockIdx.x][9] = te - tb; }
#endif
        const int C = ((n + 31) / 32) | 1;
        const int kc0 = min(n, C * lane), kc1 = min(n, kc0 + C);
        bool waited = false;
        auto erows = [&](const double* gsrc, auto ld) {   // gX[m] = g[(m - GX_PAD) mod n]
        for (int t0 = tb + EROWS * warp; t0 < te; t0 += EROWS * NW) {
            const int gx = gxu0 + (t0 - tb);     // unwrapped (gX is periodic past 2n)
            // row r, step k: g[(gx + r - k) mod n] = gX[GX_PAD + n + gx + r - k];
            // block of 8 steps from kb: H[m] = gX[GX_PAD + n + gx - kb - 7 + m], row r at step u uses H[r - u + 7]
            const double* gq = gsrc + GX_PAD + n + gx - 7 - kc0;
            double acc[EROWS];
#pragma unroll
            for (int r = 0; r < EROWS; ++r) acc[r] = 0.0;
            double H[15];
#pragma unroll
            for (int m = 0; m < 15; ++m) H[m] = ld(gq + m);
            for (int kb = kc0; kb < kc1; kb += 8) {
                double rr[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) rr[u] = (kb + u < kc1) ? s_rho[kb + u] - mean : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int r = 0; r < EROWS; ++r) acc[r] = fma(H[r - u + 7], rr[u], acc[r]);
                gq -= 8;
#pragma unroll
                for (int m = 14; m >= 8; --m) H[m] = H[m - 8];
#pragma unroll
                for (int m = 0; m < 8; ++m) H[m] = ld(gq + m);
            }
            // transposed butterfly: lane ends with row 4 b16 + 2 b8 + b4 (bits of the lane index)
            const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
            double s4[4], s2[2];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const double mine = b16 ? acc[4 + m] : acc[m], oth = b16 ? acc[m] : acc[4 + m];
                s4[m] = mine + __shfl_xor_sync(0xffffffffu, oth, 16);
            }
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const double mine = b8 ? s4[2 + m] : s4[m], oth = b8 ? s4[m] : s4[2 + m];
                s2[m] = mine + __shfl_xor_sync(0xffffffffu, oth, 8);
            }
            double e = (b4 ? s2[1] : s2[0]) + __shfl_xor_sync(0xffffffffu, b4 ? s2[0] : s2[1], 4);
            e += __shfl_xor_sync(0xffffffffu, e, 2);
            e += __shfl_xor_sync(0xffffffffu, e, 1);
            const int t = t0 + (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
            if (csize > 1 && !waited) { cluster_wait(); waited = true; }
            if ((lane & 3) == 0 && t < te) {
                if (csize > 1) {
                    for (uint32_t c = 0; c < csize; ++c)
                        st_async_f64(map_shared_rank(s_part + t, c), e, map_shared_rank(&e_bar, c));
                } else {
                    s_part[t] = e;
                }
                if (t >= 2 && t < Q - 2) {       // owned rows + periodic ghosts
                    const int x = B.lo_x + wr(T.x0 - 2 + t);
                    A.E_out[x + G] = e;
                    if (x < G) A.E_out[x + G + n] = e;
                    if (x >= n - G) A.E_out[x + G - n] = e;
                }
            }
        }
        };
        if (A.g_smem) erows(f_g - ws, [](const double* p) { return *p; });
        else erows(A.gX, [](const double* p) { return __ldg(p); });
        if (csize > 1 && !waited) cluster_wait();   // warps without rows still complete the barrier
        TRACE(4);
        if (csize > 1) mbar_wait(&e_bar, 0);
        else named_bar_sync(1, NT);
        for (int t = tid; t < Q; t += NT) sE[t] = s_part[t];
        named_bar_sync(1, NT);
    } else if (sel_cta) {
        named_bar_sync(1, NT);                   // sE written by every consumer
    }
    if (sel_cta && tid == 0) mbar_arrive(&e_ready);
    TRACE(5);
    const int cl = CPT * tid;                    // tile-local column of my first cell
    const uint64_t pol_st = STAGE == 4 ? l2_evict_last() : l2_evict_first();   // f_{n+1} (stage 4), u (stage 2) stores
    const int c0 = T.j0 + cl;                    // block-local interior column
    const int nact = min(CPT, T.ncols - cl);     // active cells of this thread (may be <= 0)
    // SELF levels have nv % 4 == 0: a thread is either fully active or idle
    const bool act = SELF ? (nact > 0) : (nact == CPT);
    // exact cell-average velocity of column c0 - 1 + n
    const int jb = B.lo_v + c0 - 1;
    auto vbar = [&](int n) -> double { return A.v_lo + ((double)(jb + n) + 0.5) * A.dv; };
    const double vb1 = vbar(1);                  // centered: vbar(n + 1) = vb1 + n dv
    auto vbx = [&](int n) -> double { return RECON == VLASOV_CENTERED4 ? vb1 + (double)(n - 1) * A.dv : vbar(n); };
    const double dv24 = A.dv * (1.0 / 24.0);
    // face values are carried times 12 (face12), fluxes too; 1/12 folds into these factors
    const double rdx12 = 1.0 / (12.0 * A.dx), rdv12 = 1.0 / (12.0 * A.dv);
    const double* E = sE + 2 - T.x0;             // E[i] for block-local row i (x0-2 <= i <= x0+nrows+1)
    const double* Ebc = sEbc + 2 - T.x0;
    // the thread holding domain cells 0..3 / nv-4 .. nv-1 (SELF: level nv % 4 == 0)
    const bool edge_lo = SELF && (B.lo_v + c0 == 0);
    const bool edge_hi = SELF && (B.lo_v + c0 + CPT == A.dom_v);
    // GM 1: input v-ghosts derived in-kernel from E_bc (at stage 1 from its own E = E(f_n), the
    // end-of-step constraint evaluation of Alg.5, reading #6b).  GM 2: read from f_s's
    // ghost columns, written by the stage that produced f_s for its own field -- except that
    // stage 4 writes the outgoing candidate (the cubic extrapolation) and stage 1 decides with its
    // own E: a branch-free select between the carried value and the unperturbed profile (SEL1).
    // Only at physical velocity faces.  SELF: the edge threads stage f_next's boundary cells; its
    // velocity ghost columns are written after the march, off the critical path
    constexpr bool BC_IN = (GMODE == 1);
    constexpr bool SEL1 = SEL1_ANY && !PWG;      // no helper warp: the edge threads select per row
    const bool lo_edge = (BC_IN || SEL1) && edge_lo && A.phys_lo, hi_edge = (BC_IN || SEL1) && edge_hi && A.phys_hi;
    const double* Ebcf = (STAGE == 1) ? E : Ebc;   // the field deciding the direction
    constexpr bool GHOST_OUT = SELF && STAGE >= 1;

    double W[4][CPT + 2];                        // f_s rows (mod 4) at columns c0-1 .. c0+4
    double VF[4][CPT + 1];                       // 12 x v-faces (mod 4) at c0-1/2 .. c0+CPT-1/2
    double Fxp[CPT];                             // 12 x x-fluxes at i-1/2

    int slot = 0;
    uint32_t phase = 0;
    // The slot of row q is released at the end of row q + 1 (see below): pending slot and the
    // dependency word of its fn / u loads
    int pend_slot = 0;
    uint32_t pend_phase = 0, pend_dep = 0;
    // one row step q (row r = x0 - 2 + q, W slot K = q mod 4): OUT rows (q >= 4) produce output
    // row i = r - 2; `live` == false only in the last group (rows past the tile: no wait, no
    // stores, no slot release; their arithmetic is discarded)
    auto row = [&](auto Kc, auto OUTc, int q, bool live, double& rsK) {
        constexpr int K = decltype(Kc)::value;
        constexpr bool OUT = decltype(OUTc)::value;
        const int r = T.x0 - 2 + q;
        if (live) mbar_wait(sel_cta ? &ready_bar[slot] : &full_bar[slot], phase);
#ifdef STAGE1D_TRACE
        if (q == 0) TRACE(6);
#endif
        const double* seg = smem + slot * SLOT;
        double v[CPT + 4];                       // columns c0-2 .. c0+5
#pragma unroll
        for (int m = 0; m < CPT + 4; m += 2) {
            const double2 p = lds2(seg + cl + m);
            v[m] = p.x; v[m + 1] = p.y;
        }
        double fn[CPT], uu[CPT];
        uint32_t fnuu = 0u;                      // dependency word of the fn / u loads
        if (OUT && NEED_FN) {
#pragma unroll
            for (int m = 0; m < CPT; m += 2) { const double2 p = lds2(seg + SEG + cl + m); fn[m] = p.x; fn[m + 1] = p.y; }
        }
        if (OUT && NEED_U) {
#pragma unroll
            for (int m = 0; m < CPT; m += 2) { const double2 p = lds2(seg + SEG + cl + m); uu[m] = p.x; uu[m + 1] = p.y; }
        }
        if (BC_IN && (lo_edge || hi_edge)) {     // characteristic BC (reading #6), a = -E_bc
            const double a = -Ebcf[r];
            if (lo_edge) {
                if (a < 0.0) {
                    v[1] = 4.0 * v[2] - 6.0 * v[3] + 4.0 * v[4] - v[5];
                    v[0] = 10.0 * v[2] - 20.0 * v[3] + 15.0 * v[4] - 4.0 * v[5];
                } else {
                    v[1] = s_f0[1];
                    v[0] = s_f0[0];
                }
            }
            if (hi_edge) {
                constexpr int L = CPT + 1;       // last interior column of the thread
                if (a > 0.0) {
                    v[L + 1] = 4.0 * v[L] - 6.0 * v[L - 1] + 4.0 * v[L - 2] - v[L - 3];
                    v[L + 2] = 10.0 * v[L] - 20.0 * v[L - 1] + 15.0 * v[L - 2] - 4.0 * v[L - 3];
                } else {
                    v[L + 1] = s_f0[2];
                    v[L + 2] = s_f0[3];
                }
            }
        }
        if (SEL1 && (lo_edge || hi_edge)) {      // stage 1, carried ghosts: keep the extrapolation
            const double a = -E[r];              // if outgoing, else the unperturbed profile
                                                 // (edge threads only: the other warps skip it)
            constexpr int L = CPT + 1;
            const bool klo = !lo_edge || (a < 0.0), khi = !hi_edge || (a > 0.0);
            v[1] = klo ? v[1] : s_f0[1];
            v[0] = klo ? v[0] : s_f0[0];
            v[L + 1] = khi ? v[L + 1] : s_f0[2];
            v[L + 2] = khi ? v[L + 2] : s_f0[3];
        }
#pragma unroll
        for (int b = 0; b < CPT + 2; ++b) W[K][b] = v[b + 1];   // register window: row r -> W[K]
        constexpr int R0 = (K + 1) & 3, R1 = (K + 2) & 3, R2 = (K + 3) & 3;   // rows r-3, r-2, r-1
        if (OUT) {
            const int i = r - 2;
            // x-faces at i + 1/2 (rows i-1 .. i+2 = r-3 .. r) for columns c0-1 .. c0+4
            double XF[CPT + 2];
#pragma unroll
            for (int n = 0; n < CPT + 2; ++n) XF[n] = face12<RECON>(W[R0][n], W[R1][n], W[R2][n], W[K][n], vbx(n));
            const double Ei = E[i], Em = E[i - 1], Ep = E[i + 1];
            const double c48 = (Ep - Em) * (1.0 / 48.0);
            // v-fluxes of row i from the v-faces of rows i-1, i, i+1 (= r-3, r-2, r-1)
            double Fv[CPT + 1];
#pragma unroll
            for (int m = 0; m < CPT + 1; ++m) Fv[m] = Ei * VF[R1][m] + c48 * (VF[R2][m] - VF[R0][m]);
            double o[CPT];
#pragma unroll
            for (int n = 0; n < CPT; ++n) {
                const double Fxn = vbx(n + 1) * XF[n + 1] + dv24 * (XF[n + 2] - XF[n]);
                const double dFv = Fv[n + 1] - Fv[n], dFx = Fxn - Fxp[n];
                Fxp[n] = Fxn;
                const double fs = W[R1][n + 1];
                if (STAGE == 0) {
                    o[n] = dFv * rdv12 - dFx * rdx12;
                } else if (STAGE == 1) {
                    o[n] = fma((0.5 * A.dt) * rdv12, dFv, fma(-(0.5 * A.dt) * rdx12, dFx, fs));
                } else if (STAGE == 2) {
                    const double k = dFv * rdv12 - dFx * rdx12;
                    uu[n] = (fn[n] + fs) * (1.0 / 3.0) + (A.dt * (1.0 / 3.0)) * k;
                    o[n] = fn[n] + (0.5 * A.dt) * k;
                } else if (STAGE == 3) {
                    o[n] = fma(A.dt * rdv12, dFv, fma(-A.dt * rdx12, dFx, fn[n]));
                } else {
                    o[n] = fma((A.dt * (1.0 / 6.0)) * rdv12, dFv,
                               fma(-(A.dt * (1.0 / 6.0)) * rdx12, dFx, fma(fs, 1.0 / 3.0, uu[n])));
                }
            }
            if (NEED_FN) fnuu ^= __double2hiint(fn[0]) ^ __double2hiint(fn[2]);
            if (NEED_U) fnuu ^= __double2hiint(uu[0]) ^ __double2hiint(uu[2]);
            const int64_t ib = rowbase(wr(i));
            double* op = A.f_next + ib + c0;
            double* up = A.u_out + ib + c0;
            if (SELF || nact == CPT) {
                if (live && act) {
#pragma unroll
                    for (int m = 0; m < CPT; m += 2) {
                        if (STAGE == 4 && A.l2hint) stg2_hint(op + m, o[m], o[m + 1], pol_st);
                        else *reinterpret_cast<double2*>(op + m) = make_double2(o[m], o[m + 1]);
                        if (STAGE == 2) {
                            if (A.l2hint) stg2_hint(up + m, uu[m], uu[m + 1], pol_st);
                            else *reinterpret_cast<double2*>(up + m) = make_double2(uu[m], uu[m + 1]);
                        }
                    }
                }
            } else if (live) {
#pragma unroll
                for (int m = 0; m < CPT; ++m)
                    if (m < nact) {
                        op[m] = o[m];
                        if (STAGE == 2) up[m] = uu[m];
                    }
            }
            if (GHOST_OUT && live && (edge_lo || edge_hi)) {   // boundary cells of f_next
                double* se = s_edge + (i - T.x0) * 2 * CPT + (edge_lo ? 0 : CPT);
                *reinterpret_cast<double2*>(se) = make_double2(o[0], o[1]);
                *reinterpret_cast<double2*>(se + 2) = make_double2(o[2], o[3]);
                if (edge_lo && edge_hi) {        // nv == 4: one thread holds both boundaries
                    *reinterpret_cast<double2*>(se + CPT) = make_double2(o[0], o[1]);
                    *reinterpret_cast<double2*>(se + CPT + 2) = make_double2(o[2], o[3]);
                }
            }
            double sr = 0.0;
            if (SELF || nact == CPT) {
                sr = (o[0] + o[1]) + (o[2] + o[3]);
            } else {
#pragma unroll
                for (int m = 0; m < CPT; ++m) sr += (m < nact) ? o[m] : 0.0;
            }
            rsK = (live && (act || !SELF)) ? sr : 0.0;
        } else if (K == 3) {                     // x-fluxes at x0 - 1/2 (rows x0-2 .. x0+1)
            double XF[CPT + 2];
#pragma unroll
            for (int n = 0; n < CPT + 2; ++n) XF[n] = face12<RECON>(W[R0][n], W[R1][n], W[R2][n], W[K][n], vbx(n));
#pragma unroll
            for (int n = 0; n < CPT; ++n) Fxp[n] = vbx(n + 1) * XF[n + 1] + dv24 * (XF[n + 2] - XF[n]);
        }
        // v-faces of row r (c0-1/2 .. c0+CPT-1/2); speed a = -E_r; stored in VF[K]
        const double ar = -E[r];
#pragma unroll
        for (int m = 0; m < CPT + 1; ++m) VF[K][m] = face12<RECON>(v[m], v[m + 1], v[m + 2], v[m + 3], ar);
        if (live) {
            // Release the slot of the previous row.  Shared-memory loads are asynchronous and the
            // compiler may schedule their consumers after the arrive, so an integer xor of one
            // word of every load of that row (its window W[R2] = v[1..6], fn / u via pend_dep) is
            // stored (volatile) first: in-order issue holds the arrive until they have landed,
            // which by now costs no stall.  (Row 0 has no previous row.)
            if (OUT || K > 0) {
                const uint32_t dep = pend_dep ^ __double2hiint(W[R2][0]) ^ __double2hiint(W[R2][2]) ^
                                     __double2hiint(W[R2][4]) ^ __double2hiint(W[R2][5]);
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(&s_dep[tid])), "r"(dep) : "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[pend_slot]);
                if (!PWARPS && tid == 0 && q - 1 + NSLOT < Q) {   // refill it once every warp released it
                    mbar_wait(&empty_bar[pend_slot], pend_phase);
                    issue(q - 1 + NSLOT, pend_slot);
                }
            }
            pend_slot = slot;
            pend_phase = phase;
            pend_dep = fnuu;
            if (++slot == NSLOT) { slot = 0; phase ^= 1u; }
        }
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    using NO = std::false_type;
    using YES = std::true_type;
    {   // rows q = 0..3 (Q >= 5): window and v-faces only, x-fluxes at x0 - 1/2 at q = 3
        double dummy;
        row(I0{}, NO{}, 0, true, dummy);
        row(I1{}, NO{}, 1, true, dummy);
        row(I2{}, NO{}, 2, true, dummy);
        row(I3{}, NO{}, 3, true, dummy);
    }
    for (int q0 = 4; q0 < Q; q0 += 4) {
        double rs[4];                            // per-thread moment sums of the group's output rows
        row(I0{}, YES{}, q0, true, rs[0]);
        row(I1{}, YES{}, q0 + 1, q0 + 1 < Q, rs[1]);
        row(I2{}, YES{}, q0 + 2, q0 + 2 < Q, rs[2]);
        row(I3{}, YES{}, q0 + 3, q0 + 3 < Q, rs[3]);
        if (A.rho != nullptr) {
            // warp sums of the 4 rows of the group with one transposed butterfly (6 shuffles
            // instead of 20): lane L ends with row 2*bit4(L) + bit3(L), lanes L % 8 == 0 write it
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
            const int i = T.x0 - 4 + q0 + (b16 ? 2 : 0) + (b8 ? 1 : 0);      // output row of q = q0 + that
            if ((lane & 7) == 0 && i >= T.x0 && i < T.x0 + T.nrows) psum[warp * A.tile_rows + (i - T.x0)] = u;
        }
    }

#if !STAGE1D_PDL_EARLY
    griddep_launch_dependents();                 // the march is done: let the next stage launch
#endif
    if (GHOST_OUT && (T.j0 == 0 || T.j0 + T.ncols == B.nv)) {
        // velocity ghost columns of f_next (characteristic BC, reading #6, for this stage's field:
        // the E_bc of the next stage, reading #6b) from the boundary cells staged during the march
        named_bar_sync(1, NT);
        const bool has_lo = (T.j0 == 0), has_hi = (T.j0 + T.ncols == B.nv);
        for (int idx = tid; idx < 2 * T.nrows; idx += NT) {
            const int rr = idx >> 1, side = idx & 1;
            if (side == 0 ? !has_lo : !has_hi) continue;
            const int i = T.x0 + rr;
            const double* se = s_edge + (rr * 2 + side) * CPT;
            // stage 4: the outgoing candidate for the next stage 1 (SEL1 decides with E(f_n))
            const double a = (STAGE == 4 && GMODE == 2) ? (side == 0 ? -1.0 : 1.0) : -E[i];
            double2 g;
            if (side == 0) {
                g = a < 0.0 ? make_double2(10.0 * se[0] - 20.0 * se[1] + 15.0 * se[2] - 4.0 * se[3],
                                           4.0 * se[0] - 6.0 * se[1] + 4.0 * se[2] - se[3])
                            : make_double2(s_f0[0], s_f0[1]);
                *reinterpret_cast<double2*>(A.f_next + rowbase(wr(i)) - 2) = g;
            } else {
                g = a > 0.0 ? make_double2(4.0 * se[3] - 6.0 * se[2] + 4.0 * se[1] - se[0],
                                           10.0 * se[3] - 20.0 * se[2] + 15.0 * se[1] - 4.0 * se[0])
                            : make_double2(s_f0[2], s_f0[3]);
                *reinterpret_cast<double2*>(A.f_next + rowbase(wr(i)) + B.nv) = g;
            }
        }
    }
    if (A.rho != nullptr) {
        named_bar_sync(1, NT);
        for (int rr = tid; rr < T.nrows; rr += NT) {
            double s = psum[rr];
#pragma unroll
            for (int w = 1; w < NW; ++w) s += psum[w * A.tile_rows + rr];
            A.partials[(int64_t)T.pvt * A.dom_x + B.lo_x + wr(T.x0 + rr)] = s;
        }
        // last CTA of this row strip finalises rho in v-tile order (deterministic)
        __threadfence();
        named_bar_sync(1, NT);
        if (tid == 0) s_ticket = atomicAdd(A.tickets + T.strip, 1u);
        named_bar_sync(1, NT);
        if (s_ticket == (unsigned)(A.n_vtiles - 1)) {
            __threadfence();
            for (int rr = tid; rr < T.nrows; rr += NT) {
                const int x = B.lo_x + wr(T.x0 + rr);
                double s = 0.0;
                for (int t = 0; t < A.n_vtiles; ++t) s += __ldcg(A.partials + (int64_t)t * A.dom_x + x);
                A.rho[x] = A.rho_base - A.dv * s;
            }
            if (tid == 0) A.tickets[T.strip] = 0u;     // reset for the next launch
        }
    }
    TRACE(7);
}

template <int STAGE, int RECON, int NT, int GM>
static int launch_t(const StageArgs1& A, int ntiles, int tile_rows, cudaStream_t st) {
    using SG = StageGeom<STAGE, NT>;
    const size_t smem = SG::smem_bytes(tile_rows) + (A.rho_in ? field_smem_bytes(A.dom_x, A.hs != nullptr) : 0);
    auto kern = k_stage_1d1v<STAGE, RECON, NT, GM>;
    static bool configured = false;   // per template instantiation
    if (!configured) {
        VK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles);
    cfg.blockDim = dim3(Roles<NT>::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    // programmatic dependent launch: this grid may start while the previous kernel on the stream
    // retires; the kernel waits (griddepcontrol.wait) before reading what earlier kernels wrote
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = STAGE1D_PDL;
    ++na;
    if (A.rho_in && A.cluster > 1) {   // the v-tiles of a strip form one cluster (Toeplitz field)
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = (unsigned)A.cluster;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    VK_CUDA(cudaLaunchKernelEx(&cfg, kern, A));
    return VLASOV_OK;
}

template <int RECON, int NT, int GM>
static int dispatch_stage(int stage, const StageArgs1& A, int ntiles, int tile_rows, cudaStream_t st) {
    switch (stage) {
        case 0: return launch_t<0, RECON, NT, GM>(A, ntiles, tile_rows, st);
        case 1: return launch_t<1, RECON, NT, GM>(A, ntiles, tile_rows, st);
        case 2: return launch_t<2, RECON, NT, GM>(A, ntiles, tile_rows, st);
        case 3: return launch_t<3, RECON, NT, GM>(A, ntiles, tile_rows, st);
        case 4: return launch_t<4, RECON, NT, GM>(A, ntiles, tile_rows, st);
    }
    return fail(VLASOV_EINVAL, "stage must be 1..4");
}

template <int NT, int GM>
static int dispatch_recon(int recon, int stage, const StageArgs1& A, int nt, int rows, cudaStream_t st) {
    return recon == VLASOV_UPWIND ? dispatch_stage<VLASOV_UPWIND, NT, GM>(stage, A, nt, rows, st)
                                  : dispatch_stage<VLASOV_CENTERED4, NT, GM>(stage, A, nt, rows, st);
}

// CTAs per SM of the most demanding stage instance (stage 4), for one-wave tiling.
template <int NT>
static int ctas_per_sm_t(int tile_rows) {
    int n = 0;
    using SG = StageGeom<4, NT>;
    auto k = k_stage_1d1v<4, VLASOV_CENTERED4, NT, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, Roles<NT>::THREADS, SG::smem_bytes(tile_rows)) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int stage_1d1v_ctas_per_sm(bool wide, int tile_rows) {
    return wide ? ctas_per_sm_t<NT_WIDE>(tile_rows) : ctas_per_sm_t<NT_NARROW>(tile_rows);
}

int stage_1d1v_tile_width(bool wide) { return CPT * (wide ? NT_WIDE : NT_NARROW); }

// co-resident clusters of `cs` CTAs of the fused stage-4 instance (field smem for n x cells)
int stage_1d1v_max_clusters(bool wide, int tile_rows, int cs, int n) {
    auto q = [&](auto kern, int nt, size_t smem) -> int {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(nt == NT_WIDE ? Roles<NT_WIDE>::THREADS : Roles<NT_NARROW>::THREADS);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int m = 0;
        if (cudaOccupancyMaxActiveClusters(&m, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        return m;
    };
    if (wide)
        return q(k_stage_1d1v<4, VLASOV_CENTERED4, NT_WIDE, 2>, NT_WIDE,
                 StageGeom<4, NT_WIDE>::smem_bytes(tile_rows) + field_smem_bytes(n));
    return q(k_stage_1d1v<4, VLASOV_CENTERED4, NT_NARROW, 2>, NT_NARROW,
             StageGeom<4, NT_NARROW>::smem_bytes(tile_rows) + field_smem_bytes(n));
}

// strip shift of the even stages in quarters of a strip (VLASOV_XSHIFT, experiments; default 2)
// L2 eviction priorities (VLASOV_L2HINT=0 disables; experiments)
static int l2hint_on() {
    static const int q = [] { const char* e = getenv("VLASOV_L2HINT"); return e ? atoi(e) : 1; }();
    return q;
}

// stages whose strips are shifted (bit s = stage s; VLASOV_XSHIFT_MASK for experiments): stages 2-4
// start half a strip later than stage 1, so stage 2 and the next step's stage 1 first read what the
// stage before them wrote last (measured on C4 with the L2 priorities: stages 2, 4 shifted 55.9 G,
// none 56.4 G, stages 2-4 56.8 G)
static int shift_mask() {
    static const int q = [] { const char* e = getenv("VLASOV_XSHIFT_MASK"); return e ? (int)strtol(e, nullptr, 0) : 0x1c; }();
    return q;
}

static int shift_quarters() {
    static const int q = [] { const char* e = getenv("VLASOV_XSHIFT"); return e ? atoi(e) : 2; }();
    return q;
}

int launch_stage_1d1v(vlasov_level* L, int stage, double dt, double* f_n, const double* f_s, double* u,
                      double* f_next, const double* E, const double* E_bc, const double* f0v, int recon,
                      double* rho, const double* rho_in, const double* gE, double* E_out, const double* gX,
                      const double* hs, double K2, double Kn) {
    StageArgs1 A;
    A.hs = rho_in ? hs : nullptr;
    A.K2 = K2;
    A.Kn = Kn;
    A.rho_in = rho_in;
    A.gE = gE;
    A.E_out = E_out;
    A.cluster = rho_in ? L->cluster_size : 1;     // 1 unless chosen at level creation
    A.g_smem = (rho_in && !A.hs && g_in_smem(L->dom[0])) ? 1 : 0;
    A.gX = gX;
    A.nstrip1 = L->single_block ? L->n_strips : 0;
    // L2 reuse between stages: even stages start their strips half a strip later, so each CTA
    // first reads the rows the previous stage wrote last (still in L2)
    A.xshift = (A.nstrip1 > 0 && stage >= 1 && ((shift_mask() >> stage) & 1)) ? L->dom[0] / A.nstrip1 * shift_quarters() / 4 : 0;
    A.l2hint = (A.nstrip1 > 0 && stage >= 1) ? l2hint_on() : 0;
    if (!L->h_blocks1.empty()) A.blk0 = L->h_blocks1[0];
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
    A.rho_base = L->moment_base;
    A.phys_lo = L->vphys[0];
    A.phys_hi = L->vphys[1];
    A.dom_x = L->dom[0];
    A.dom_v = L->dom[1];
    A.n_vtiles = L->n_vtiles;
    A.tile_rows = L->tile_rows;
    const bool self = (f0v != nullptr);     // periodic single block: E_bc (in-kernel input ghosts) or carried ghosts
    const bool wide = !L->h_tiles_wide.empty();
    A.tiles = wide ? L->d_tiles_wide : L->d_tiles_narrow;
    const int nt = (int)(wide ? L->h_tiles_wide.size() : L->h_tiles_narrow.size());
    if (nt == 0) return VLASOV_OK;
    const int rows = L->tile_rows;
    const int gm = (self ? (E_bc ? 1 : 2) : 0) | (A.hs != nullptr ? 4 : 0);
    if (A.hs != nullptr && !self) return fail(VLASOV_EINVAL, "split field needs in-kernel ghosts");
    if (wide) {
        switch (gm) {
            case 6: return dispatch_recon<NT_WIDE, 6>(recon, stage, A, nt, rows, L->stream);
            case 5: return dispatch_recon<NT_WIDE, 5>(recon, stage, A, nt, rows, L->stream);
            case 2: return dispatch_recon<NT_WIDE, 2>(recon, stage, A, nt, rows, L->stream);
            case 1: return dispatch_recon<NT_WIDE, 1>(recon, stage, A, nt, rows, L->stream);
            default: return dispatch_recon<NT_WIDE, 0>(recon, stage, A, nt, rows, L->stream);
        }
    }
    switch (gm) {
        case 6: return dispatch_recon<NT_NARROW, 6>(recon, stage, A, nt, rows, L->stream);
        case 5: return dispatch_recon<NT_NARROW, 5>(recon, stage, A, nt, rows, L->stream);
        case 2: return dispatch_recon<NT_NARROW, 2>(recon, stage, A, nt, rows, L->stream);
        case 1: return dispatch_recon<NT_NARROW, 1>(recon, stage, A, nt, rows, L->stream);
        default: return dispatch_recon<NT_NARROW, 0>(recon, stage, A, nt, rows, L->stream);
    }
}

}  // namespace vk

#ifdef STAGE1D_TRACE
extern "C" int vlasov_debug_stage_trace(unsigned long long* out, int nblocks) {
    return cudaMemcpyFromSymbol(out, vk::g_trace, (size_t)nblocks * 10 * sizeof(unsigned long long)) == cudaSuccess ? 0 : -3;
}
#endif
