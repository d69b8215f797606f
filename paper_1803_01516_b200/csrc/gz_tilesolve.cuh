// gz_tilesolve.cuh -- v4 solver: tile-owned persistent push-relabel (m <= 32).
//
// Same node state and per-chain lane mapping as v3 (gz_warpsolve.cuh: one
// LP-lane warp segment per site chain, column-major [site][LP] arrays), but the
// work is organised around rectangular TILES of sites, each owned by one CTA
// of a persistent cooperative launch (one CTA of 512 threads per SM):
//
//  * global relabel (maxflow.py:138-170): level-synchronous bit-parallel BFS
//    from the sink with TEMPORAL BLOCKING.  A round loads the tile plus a halo
//    of H sites (frontier/visited words into shared memory, the 13 residual
//    arc masks into registers) and advances H BFS levels with CTA barriers
//    only; the interior is valid because information moves at most one site
//    per level.  One team barrier per H levels instead of one per level.
//  * push/relabel pulses (maxflow.py:183-250): synchronous pulses exactly as
//    v3.  Active chains cluster spatially, so pulse work is NOT tile-owned:
//    site groups are interleaved over all warps of the team, and each warp
//    checks its groups' active/inbox words with one load per lane + a ballot,
//    visiting only the chains that have work.
//  * extraction (maxflow.py:267-320): prefix-closure rounds as v2/v3.
//
// The team barrier is a generation-flip counter (one CTA per team adds
// 2^31 - (nb-1), the others 1), so several teams can share a launch.
#pragma once

namespace gz4 {

using namespace gz;
using gz2::Bits2;
using gz2::BW;
using gz3::Arr3;

constexpr unsigned FULL = 0xffffffffu;
constexpr int BLOCK = 512;   // threads per CTA (one CTA per SM)
constexpr int SPT = 4;       // BFS region sites per thread
constexpr int REGMAX = SPT * BLOCK;   // BFS region sites per tile (tile + halo)
constexpr size_t SMEM_BYTES = (size_t)(2 + 13) * REGMAX * sizeof(uint32_t);   // frontier x2 + arc masks

struct Geo {
    int TY, TX, ny, nx, ntiles, H;
};

// Team barrier with a fused 2-bit OR reduction.  Barrier k uses word k % 3 of
// `bar`: each CTA adds, in ONE atomic, its arrival (low 32 bits, generation-flip
// trick: rank 0 adds 2^31 - (nb-1), the others 1, so bit 31 flips exactly when
// the last CTA arrives) plus a count of flag-0 / flag-1 CTAs in bits 32-47 /
// 48-63.  The value a CTA sees when it observes the flip therefore carries the
// team's OR.  After barrier k every CTA has read word (k-1) % 3, so rank 0
// clears it for barrier k+2 (nobody reaches k+2 before rank 0 reaches k+1).
struct Team {
    unsigned long long *bar;   // 3 rotating words of this team
    int nb, rank;
    __device__ __forceinline__ unsigned sync_or(unsigned flags, int &phase, unsigned *s_f3, unsigned *s_r3) const {
        const int k3 = phase % 3;
        const unsigned w = __reduce_or_sync(FULL, flags);
        if ((threadIdx.x & 31) == 0 && w) atomicOr(&s_f3[k3], w);
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned f = s_f3[k3];
            s_f3[(k3 + 1) % 3] = 0u;   // last read two barriers ago
            const unsigned long long inc = (rank == 0 ? 0x80000000ull - (unsigned long long)(nb - 1) : 1ull) |
                                           ((f & 1u) ? 1ull << 32 : 0ull) | ((f & 2u) ? 1ull << 48 : 0ull);
            unsigned long long *word = bar + k3;
            __threadfence();
            const unsigned long long old = atomicAdd(word, inc);
            unsigned long long cur;
            do {
                cur = *(volatile unsigned long long *)word;
            } while (((old ^ cur) & 0x80000000ull) == 0ull);
            if (rank == 0) bar[(k3 + 2) % 3] = 0ull;
            __threadfence();
            s_r3[k3] = ((cur >> 32) & 0xffffull ? 1u : 0u) | ((cur >> 48) ? 2u : 0u);
        }
        __syncthreads();
        const unsigned r = s_r3[k3];
        ++phase;
        return r;
    }
};

struct TileBox {
    int y0, y1, x0, x1;
    __device__ __forceinline__ TileBox(const Prob &p, const Geo &g, int tile) {
        const int ty = tile / g.nx, tx = tile - ty * g.nx;
        y0 = ty * g.TY;
        y1 = min(y0 + g.TY, p.Y);
        x0 = tx * g.TX;
        x1 = min(x0 + g.TX, p.G);
    }
};

// Every site of the tile, in LP-lane warp segments (CPW sites per call).
template <int LP, typename F>
__device__ __forceinline__ void for_tile_groups(const Prob &p, const TileBox &tb, F &&f) {
    constexpr int CPW = 32 / LP;
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int w = tb.x1 - tb.x0;
    for (int r = tb.y0 + warp; r < tb.y1; r += nwarps)
        for (int k = 0; k < w; k += CPW) f(r * p.G + tb.x0 + k, min(CPW, w - k));
}

// ---------------------------------------------------------------------------
// one BFS round on a tile: H levels from depth d.  Returns bit0 = new interior
// nodes, bit1 = a new interior node holds excess.  The region's 13 arc-mask
// words per site live in shared memory (sM, REGMAX stride); they are loaded
// when load_masks is set -- once per sweep when every CTA owns one tile.
template <int LP, bool WIN>
__device__ unsigned bfs_round(const Prob &p, const Arr3 &a, const Bits2 &b, const Geo &g, const TileBox &tb,
                              const uint32_t *Fin, uint32_t *Fout, const uint32_t *Vin, uint32_t *Vout, int d,
                              uint32_t *sF0, uint32_t *sF1, uint32_t *sM, bool load_masks) {
    const int P = p.P, H = g.H;
    const int ry0 = max(tb.y0 - H, 0), ry1 = min(tb.y1 + H, p.Y);
    const int rx0 = max(tb.x0 - H, 0), rx1 = min(tb.x1 + H, p.G);
    const int RW = rx1 - rx0, nreg = (ry1 - ry0) * RW;
    uint32_t V[SPT], EX[SPT], RNG[SPT];
    int C[SPT];
    bool IN_[SPT];
    unsigned NB[SPT];   // neighbour-in-region bits: right, left, down, up
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        const bool ok = i < nreg;
        const int ri = ok ? i / RW : 0, rj = ok ? i - ri * RW : 0;
        const int y = ry0 + ri, x = rx0 + rj;
        const int c = y * p.G + x;
        C[k] = ok ? c : -1;
        IN_[k] = ok && y >= tb.y0 && y < tb.y1 && x >= tb.x0 && x < tb.x1;
        NB[k] = (rj + 1 < RW ? 1u : 0u) | (rj > 0 ? 2u : 0u) | (i + RW < nreg ? 4u : 0u) | (ri > 0 ? 8u : 0u);
        if (load_masks && ok) {
#pragma unroll
            for (int q = 0; q < 13; ++q) sM[q * REGMAX + i] = b.mask[(size_t)q * P + c];
        }
        V[k] = ok ? Vin[c] : 0u;
        EX[k] = IN_[k] ? b.EX[c] : 0u;
        int lo = 0, hi = p.L;
        if (WIN && ok) { lo = p.lo[c]; hi = p.hi[c]; }
        RNG[k] = ok ? BW<1>::range(lo, hi).w[0] : 0u;
        if (ok) sF0[i] = Fin[c];
    }
    __syncthreads();
    unsigned flags = 0;
    uint32_t *cur = sF0, *nxt = sF1;
    for (int lev = 0; lev < H; ++lev) {
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int i = threadIdx.x + k * blockDim.x;
            if (C[k] < 0) continue;
            const uint32_t F = cur[i];
            const uint32_t Fn0 = (NB[k] & 1u) ? cur[i + 1] : 0u;
            const uint32_t Fn1 = (NB[k] & 2u) ? cur[i - 1] : 0u;
            const uint32_t Fn2 = (NB[k] & 4u) ? cur[i + RW] : 0u;
            const uint32_t Fn3 = (NB[k] & 8u) ? cur[i - RW] : 0u;
            if ((F | Fn0 | Fn1 | Fn2 | Fn3) == 0u) {   // no frontier next to this site
                nxt[i] = 0u;
                continue;
            }
            const uint32_t *m = sM + i;
            uint32_t N = (F << 1) | ((F >> 1) & m[A_UP * REGMAX]);
            N |= (Fn0 & m[A_SR * REGMAX]) | ((Fn0 << 1) & m[A_DR * REGMAX]) | ((Fn0 >> 1) & m[A_UR * REGMAX]);
            N |= (Fn1 & m[A_SL * REGMAX]) | ((Fn1 << 1) & m[A_DL * REGMAX]) | ((Fn1 >> 1) & m[A_UL * REGMAX]);
            N |= (Fn2 & m[A_SD * REGMAX]) | ((Fn2 << 1) & m[A_DD * REGMAX]) | ((Fn2 >> 1) & m[A_UD * REGMAX]);
            N |= (Fn3 & m[A_SU * REGMAX]) | ((Fn3 << 1) & m[A_DU * REGMAX]) | ((Fn3 >> 1) & m[A_UU * REGMAX]);
            N &= RNG[k] & ~V[k];
            V[k] |= N;
            nxt[i] = N;
            if (IN_[k] && N) {
                flags |= 1u;
                if (N & EX[k]) flags |= 2u;
                uint32_t x = N;
                const int base = C[k] * LP;
                while (x) {
                    const int bb = __ffs(x) - 1;
                    x &= x - 1;
                    a.h[base + bb] = d + lev + 1;
                }
            }
        }
        __syncthreads();
        uint32_t *t = cur; cur = nxt; nxt = t;
    }
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        if (!IN_[k]) continue;
        const int i = threadIdx.x + k * blockDim.x;
        Fout[C[k]] = cur[i];
        Vout[C[k]] = V[k];
    }
    __syncthreads();   // shared buffers are reused by the next tile
    return flags;
}

// ---------------------------------------------------------------------------
template <int LP, bool WIN>
__global__ void __launch_bounds__(BLOCK, 1) gz_tilesolve_kernel(Prob p, Bits2 b, Arr3 a, Geo g, unsigned long long *bar) {
    __shared__ unsigned s_f3[3], s_r3[3];
    extern __shared__ uint32_t s_dyn[];
    if (threadIdx.x < 3) { s_f3[threadIdx.x] = 0u; s_r3[threadIdx.x] = 0u; }
    __syncthreads();
    int phase = 0;
    uint32_t *sF0 = s_dyn, *sF1 = s_dyn + REGMAX, *sM = s_dyn + 2 * REGMAX;
    const bool resident = g.ntiles <= (int)gridDim.x;   // one tile per CTA: masks stay in smem for the sweep
    const Team tm{bar, (int)gridDim.x, (int)blockIdx.x};
#define TEAM_SYNC() (void)tm.sync_or(0u, phase, s_f3, s_r3)
#define TEAM_OR(f) tm.sync_or((f), phase, s_f3, s_r3)
    unsigned long long t_prev = 0, t_acc[6] = {0, 0, 0, 0, 0, 0};
    const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
    if (timer) t_prev = gz2::gtimer();
    if (timer) p.t_start_ns = t_prev;
#define TICK(slot) do { if (timer) { unsigned long long t_ = gz2::gtimer(); t_acc[slot] += t_ - t_prev; t_prev = t_; } } while (0)
#define FOR_TILES for (int tile = tm.rank; tile < g.ntiles; tile += tm.nb)
    long long flow = 0, offset = 0, presat = 0, pushes = 0, relabels = 0;
    volatile unsigned long long *vctr = p.ctr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    constexpr int CPW = 32 / LP;
    const int ngroups = (p.P + CPW - 1) / CPW;
    const int gnw = tm.nb * nwarps, gwid = tm.rank * nwarps + warp;
    const int giter = (ngroups + gnw - 1) / gnw;
    const int ttid = tm.rank * blockDim.x + threadIdx.x, tstride = tm.nb * blockDim.x;
    long long updates = 0;   // groups processed by pulses (x CPW x L = node updates)

    FOR_TILES {
        const TileBox tb(p, g, tile);
        for_tile_groups<LP>(p, tb, [&](int cb, int ns) { gz3::w_init<LP, WIN>(p, a, b, cb, ns, flow, offset, presat); });
    }
    for (int c = ttid; c < p.P; c += tstride) b.IN[c] = 1u;   // every site starts dirty
    TEAM_SYNC();
    TICK(0);
    int sweeps = 0, levels_total = 0, pulses = 0, parity = 0;
    int converged = 1;
    bool err = false;
    const int bfs_min = p.bfs_cap > 0 ? p.bfs_cap : (1 << 30);
    for (;;) {
        // ---- sweep set-up: bulk coalesced resets, then arc masks of dirty sites only ----
        for (int c = ttid; c < p.P; c += tstride) {
            const int hi = WIN ? p.hi[c] : p.L;
            b.F0[c] = BW<1>::range(hi, p.M).w[0];
            b.V[c] = 0u;
        }
        {
            const int4 hinf4 = make_int4(HINF, HINF, HINF, HINF);
            int4 *h4 = reinterpret_cast<int4 *>(a.h);
            const int n4 = p.P * (LP / 4);
            for (int q = ttid; q < n4; q += tstride) h4[q] = hinf4;
        }
        for (int it0 = 0; it0 < giter; it0 += 32) {
            const int it = it0 + lane;
            const int grp = gwid + it * gnw;
            uint32_t wk = 0u;
            if (it < giter && grp < ngroups) {
                const int c0 = grp * CPW;
                wk = b.IN[c0];
                if (CPW == 2 && c0 + 1 < p.P) wk |= b.IN[c0 + 1];
            }
            uint32_t msk = __ballot_sync(FULL, wk != 0u);
            while (msk) {
                const int k = __ffs(msk) - 1;
                msk &= msk - 1;
                const int c0 = (gwid + (it0 + k) * gnw) * CPW;
                gz3::w_build<LP, WIN, false>(p, a, b, c0, CPW);
                if (lane < CPW && c0 + lane < p.P) b.IN[c0 + lane] = 0u;
            }
        }
        TEAM_SYNC();
        TICK(1);
        // ---- global relabel: temporally blocked BFS ----
        int d = 0;
        bool found = false, exhausted = false;
        uint32_t *Fin = b.F0, *Fout = b.F1, *Vin = b.V, *Vout = b.RL;
        for (;;) {
            unsigned flags = 0;
            FOR_TILES {
                const TileBox tb(p, g, tile);
                flags |= bfs_round<LP, WIN>(p, a, b, g, tb, Fin, Fout, Vin, Vout, d, sF0, sF1, sM, d == 0 || !resident);
            }
            const unsigned gf = TEAM_OR(flags);
            found |= (gf & 2u) != 0;
            uint32_t *t = Fin; Fin = Fout; Fout = t;
            t = Vin; Vin = Vout; Vout = t;
            d += g.H;
            if (!(gf & 1u)) { exhausted = true; break; }
            if (found && d >= bfs_min) break;
            if (d > 4 * (p.P + p.M) + 4 * g.H) { if (threadIdx.x == 0 && tm.rank == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); err = true; break; }
        }
        levels_total += d;
        TICK(2);
        if (err) break;
        if (!found && exhausted) break;
        if (p.capped && sweeps >= p.max_sweeps) { converged = 0; break; }
        FOR_TILES {
            const TileBox tb(p, g, tile);
            for (int r = tb.y0 + warp; r < tb.y1; r += nwarps) {
                const int x = tb.x0 + lane;
                if (x < tb.x1) {
                    const int c = r * p.G + x;
                    b.A[c] = Vin[c] & b.EX[c];
                }
            }
        }
        TEAM_SYNC();
        for (int pulse = 0; pulse < p.K; ++pulse) {
            // Pulses are NOT tile-owned: active chains cluster spatially, so groups are
            // interleaved over every warp of the team (group g -> warp g mod W).  Lane i of
            // a warp checks the i-th of the warp's groups in one load; only groups with
            // active or inbox bits run a pulse.
            const uint32_t *IN_prev = parity ? a.IN0 : a.IN1;
            for (int it0 = 0; it0 < giter; it0 += 32) {
                const int it = it0 + lane;
                const int grp = gwid + it * gnw;
                uint32_t wk = 0u;
                if (it < giter && grp < ngroups) {
                    const int c0 = grp * CPW;
                    wk = b.A[c0] | IN_prev[c0];
                    if (CPW == 2 && c0 + 1 < p.P) wk |= b.A[c0 + 1] | IN_prev[c0 + 1];
                }
                uint32_t msk = __ballot_sync(FULL, wk != 0u);
                updates += __popc(msk);
                while (msk) {
                    const int k = __ffs(msk) - 1;
                    msk &= msk - 1;
                    const int g2 = gwid + (it0 + k) * gnw;
                    gz3::w_pulse<LP, WIN, false>(p, a, b, g2 * CPW, CPW, parity, flow, pushes, relabels, b.IN);
                }
            }
            TEAM_SYNC();
            parity ^= 1;
            ++pulses;
        }
        TICK(3);
        ++sweeps;
        {
            unsigned stop = 0;
            if (threadIdx.x == 0 && tm.rank == 0 && gz2_watchdog_expired(p)) stop = 1;
            if (TEAM_OR(stop)) {
                if (threadIdx.x == 0 && tm.rank == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE);
                break;
            }
        }
        if (sweeps > 1000000) { if (threadIdx.x == 0 && tm.rank == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
    }
    // ---- extraction: prefix closure from the excess nodes ----
#define FOR_TILE_SITES                                                              \
    FOR_TILES                                                                       \
    for (int r = TileBox(p, g, tile).y0 + warp, y1_ = TileBox(p, g, tile).y1; r < y1_; r += nwarps) \
        for (int x = TileBox(p, g, tile).x0 + lane, x1_ = TileBox(p, g, tile).x1; x < x1_; x += 32)
    FOR_TILE_SITES gz3::w_reach_init<WIN>(p, b, r * p.G + x);
    TEAM_SYNC();
    int reach_passes = 0;
    int32_t *Rin = b.R0, *Rout = b.R1;
    for (;;) {
        unsigned ch = 0;
        FOR_TILE_SITES ch |= gz2::bit_reach_iter<WIN, 1>(p, b, r * p.G + x, Rin, Rout) ? 1u : 0u;
        const bool any = TEAM_OR(ch) != 0;
        int32_t *t = Rin; Rin = Rout; Rout = t;
        ++reach_passes;
        if (!any) break;
        if (reach_passes > 4 * (p.P + p.M)) { if (threadIdx.x == 0 && tm.rank == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
    }
    TICK(4);
    long long stranded = 0;
    FOR_TILE_SITES {
        const int c = r * p.G + x;
        const int lo = WIN ? p.lo[c] : 0;
        p.labels[c] = lo + Rin[c];
        stranded += __popc(b.EX[c]);
    }
    TEAM_SYNC();
    long long energy = 0;
    int viol = 0;
    FOR_TILE_SITES gz3::w_energy<LP>(p, a, r * p.G + x, energy, viol);
#undef FOR_TILE_SITES
#undef FOR_TILES
#undef TEAM_SYNC
#undef TEAM_OR
    TICK(5);
#undef TICK
    if (timer)
        for (int q = 0; q < 6; ++q) p.ctr[CTR_T0 + q] = t_acc[q];
    warp_add_u64(&p.ctr[CTR_FLOW], flow);
    warp_add_u64(&p.ctr[CTR_OFFSET], offset);
    warp_add_u64(&p.ctr[CTR_PRESAT], presat);
    warp_add_u64(&p.ctr[CTR_PUSHES], pushes);
    warp_add_u64(&p.ctr[CTR_RELABELS], relabels);
    warp_add_u64(&p.ctr[CTR_ENERGY], energy);
    warp_add_u64(&p.ctr[CTR_STRANDED], stranded);
    if (lane == 0 && updates) atomicAdd(&p.ctr[CTR_UPDATES], (unsigned long long)updates * CPW * p.L);
    if (viol) p.ctr[CTR_HARDVIOL] = 1;
    if (threadIdx.x == 0 && tm.rank == 0) {
        p.ctr[CTR_SWEEPS] = sweeps;
        p.ctr[CTR_BFS_PASSES] = levels_total;
        p.ctr[CTR_REACH_PASSES] = reach_passes;
        p.ctr[CTR_CONVERGED] = converged;
        p.ctr[CTR_PULSES] = pulses;
    }
}

}  // namespace gz4
