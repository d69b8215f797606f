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
//  * extraction (maxflow.py:267-320): prefix-closure rounds (gz_bits.cuh).
//  * chains longer than 32 positions are split into R segments of 32 lanes
//    (gz_chain.cuh); bit words and the BFS are NW = R words per site.
//
// The team barrier is a generation-flip counter (one CTA per team adds
// 2^31 - (nb-1), the others 1), so several teams can share a launch.
#pragma once

namespace gz4 {

using namespace gz;
using gz2::Bits2;
using gz2::BW;
using gz3::Arr3;
using gz3::FULL;

constexpr int BLOCK = 512;   // threads per CTA (one CTA per SM)
constexpr int TAIL_CTAS = 16;        // tail mode: at most this many CTAs had work in the last pulse,
constexpr int TAIL_CTA_GROUPS = 8;   // none of them more than this many groups
// BFS region words per tile (tile + halo, x words per site): 4 per thread with
// one CTA per SM, 3 per thread with two (the shared-memory budget per CTA)
__host__ __device__ constexpr int regmax(int occ) { return (occ == 1 ? 4 : 3) * BLOCK; }
__host__ __device__ constexpr size_t smem_bytes(int occ) { return (size_t)(2 + 13) * regmax(occ) * sizeof(uint32_t); }
// arc masks of the BFS region live in shared memory up to 4 words per site; 8
// words per site (m > 128) read them from global memory
__host__ __device__ constexpr bool smem_masks(int nw) { return nw <= 4; }
// region sites per tile for NW words per site (a multiple of BLOCK)
__host__ __device__ constexpr int region_sites(int nw, int occ) {
    return smem_masks(nw) ? ((regmax(occ) / nw) / BLOCK * BLOCK > 0 ? (regmax(occ) / nw) / BLOCK * BLOCK : BLOCK)
                          : BLOCK;
}

// Tile geometry plus the row band this launch owns.  One problem may be solved
// by several co-resident cooperative launches (row bands): the
// team is all CTAs of all launches (nb, global rank = rank0 + blockIdx.x), and
// each launch works its own tile rows [t0, t1), sites [c0, c1) and pair groups
// [gg0, gg1) (LP = 16).  A single launch is the one-band case (rank0 = 0,
// nb = gridDim.x, the whole grid).
struct Geo {
    int TY, TX, ny, nx, ntiles, H;
    int nb, rank0;         // team size (all bands), first global rank of this launch
    int t0, t1, c0, c1;    // this band's tiles and sites
    int gg0, gg1;          // this band's site-pair groups (LP = 16)
    int sys;               // bands on several GPUs: system-scope fences in the team barrier
    int nbands;            // bands of the team (1: one launch)
    int spin_ms;           // multi-launch team: abort a barrier wait after this long (0: never)
};

// Team barrier with a fused 2-bit OR reduction.  Barrier k uses word k % 3 of
// `bar`: each CTA adds, in ONE atomic, its arrival (low 32 bits, generation-flip
// trick: rank 0 adds 2^31 - (nb-1), the others 1, so bit 31 flips exactly when
// the last CTA arrives) plus a count of flag-0 / flag-1 CTAs in bits 32-47 /
// 48-63.  The value a CTA sees when it observes the flip therefore carries the
// team's OR.  After barrier k every CTA has read word (k-1) % 3, so rank 0
// clears it for barrier k+2 (nobody reaches k+2 before rank 0 reaches k+1).
// Release / acquire half of the team barrier.  fence.acq_rel suffices for the
// pattern (writes -> bar.sync -> fence -> arrive atomic | observe -> fence ->
// bar.sync -> reads) and is cheaper than __threadfence's fence.sc (MEMBAR.SC);
// both also invalidate L1 (CCTL.IVALL), which the plain loads after the barrier rely on.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

struct Team {
    unsigned long long *bar;   // 3 rotating words of this team
    unsigned long long *abort_flag;   // set when a multi-launch team gives up (spin_ns)
    int nb, rank;
    int sys;                   // system-scope fences (team spans GPUs)
    unsigned long long spin_ns;   // > 0: give up a barrier after this long (multi-launch teams)
    // returns the number of CTAs that raised flag 0 (bits 0-15) and flag 1 (16-31)
    __device__ __forceinline__ unsigned sync_count(unsigned flags, int &phase, unsigned *s_f3, unsigned *s_r3) const {
        const int k3 = phase % 3;
        const unsigned w = __reduce_or_sync(FULL, flags);
        if ((threadIdx.x & 31) == 0 && w) atomicOr(&s_f3[k3], w);
        __syncthreads();
        if (nb == 1) {
            // a one-CTA team (batched pair solves): the CTA barrier is the team
            // barrier.  Slot k3-1 was read by every thread before this barrier and
            // is written again only at barrier k3+2, after thread 0 passed k3+1.
            const unsigned f = s_f3[k3];
            if (threadIdx.x == 0) s_f3[(k3 + 2) % 3] = 0u;
            ++phase;
            return (f & 1u) | ((f & 2u) << 15);
        }
        if (threadIdx.x == 0) {
            const unsigned f = s_f3[k3];
            s_f3[(k3 + 1) % 3] = 0u;   // last read two barriers ago
            const unsigned long long inc = (rank == 0 ? 0x80000000ull - (unsigned long long)(nb - 1) : 1ull) |
                                           ((f & 1u) ? 1ull << 32 : 0ull) | ((f & 2u) ? 1ull << 48 : 0ull);
            unsigned long long *word = bar + k3;
            if (sys) __threadfence_system(); else fence_acq_rel_gpu();
            unsigned long long cur = 0ull;
            bool aborted = spin_ns && *(volatile unsigned long long *)abort_flag;
            if (!aborted) {
                // (an aborted team's barriers all return "nothing happened", so every
                // loop of the solve ends and the launch exits)
                const unsigned long long old = sys ? atomicAdd_system(word, inc) : atomicAdd(word, inc);
                unsigned long long t0 = 0ull;
                unsigned spins = 0;
                do {
                    cur = *(volatile unsigned long long *)word;
                    if (spin_ns && ((++spins & 4095u) == 0u)) {
                        // a multi-launch team whose other launches never arrived (not
                        // co-resident): abort instead of hanging the GPU
                        unsigned long long t;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                        if (t0 == 0ull) t0 = t;
                        if (t - t0 > spin_ns || *(volatile unsigned long long *)abort_flag) {
                            atomicExch_system(abort_flag, 1ull);
                            aborted = true;
                            break;
                        }
                    }
                } while (((old ^ cur) & 0x80000000ull) == 0ull);
                if (aborted) cur = 0ull;
                else if (rank == 0) bar[(k3 + 2) % 3] = 0ull;
            }
            if (sys) __threadfence_system(); else fence_acq_rel_gpu();
            s_r3[k3] = (unsigned)(cur >> 32);   // CTAs with flag 0 (low 16) / flag 1 (high 16)
        }
        __syncthreads();
        const unsigned r = s_r3[k3];
        ++phase;
        return r;
    }
    __device__ __forceinline__ unsigned sync_or(unsigned flags, int &phase, unsigned *s_f3, unsigned *s_r3) const {
        const unsigned c = sync_count(flags, phase, s_f3, s_r3);
        return ((c & 0xffffu) ? 1u : 0u) | ((c >> 16) ? 2u : 0u);
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
// nodes, bit1 = a new interior node holds excess.  The region's 13 x NW arc-mask
// words per site live in shared memory; they are loaded when load_masks is set
// -- once per sweep when every CTA owns one tile.  Word w of region site i is
// at [w * RS + i] (RS = region_sites(NW)).
template <int LPT, int NW, bool WIN, int OCC>
__device__ unsigned bfs_round(const Prob &p, const Arr3 &a, const Bits2 &b, const Geo &g, const TileBox &tb,
                              const uint32_t *Fin, uint32_t *Fout, const uint32_t *Vin, uint32_t *Vout, int d,
                              uint32_t *sF0, uint32_t *sF1, uint32_t *sM, bool load_masks, bool &front) {
    constexpr int RS = region_sites(NW, OCC), SPT = RS / BLOCK;
    constexpr bool PACK = LPT == 16;   // 16-lane chains: packed arc masks (gz_bits.cuh mask_word)
    const int P = p.P, H = g.H;
    const int ry0 = max(tb.y0 - H, 0), ry1 = min(tb.y1 + H, p.Y);
    const int rx0 = max(tb.x0 - H, 0), rx1 = min(tb.x1 + H, p.G);
    const int RW = rx1 - rx0, nreg = (ry1 - ry0) * RW;
    BW<NW> V[SPT], EX[SPT], RNG[SPT];
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
        // bits 4+: Manhattan distance to the tile -- the site matters to the tile's
        // level d + H state only through levels < H - distance (see the level loop)
        const int dx_ = max(max(tb.x0 - x, x - (tb.x1 - 1)), 0), dy_ = max(max(tb.y0 - y, y - (tb.y1 - 1)), 0);
        NB[k] = (rj + 1 < RW ? 1u : 0u) | (rj > 0 ? 2u : 0u) | (i + RW < nreg ? 4u : 0u) | (ri > 0 ? 8u : 0u) |
                ((unsigned)(dx_ + dy_) << 4);
        if (smem_masks(NW) && load_masks && ok) {
#pragma unroll
            for (int q = 0; q < (PACK ? 7 : 13 * NW); ++q) sM[q * RS + i] = b.mask[(size_t)q * P + c];
        }
        V[k].zero(); EX[k].zero(); RNG[k].zero();
        if (ok) {
            V[k].load(Vin, P, c);
            if (IN_[k]) EX[k].load(b.EX, P, c);
            int lo = 0, hi = p.L;
            if (WIN) { lo = p.lo[c]; hi = p.hi[c]; }
            RNG[k] = BW<NW>::range(lo, hi);
#pragma unroll
            for (int w = 0; w < NW; ++w) sF0[w * RS + i] = Fin[(size_t)w * P + c];
        }
    }
    __syncthreads();
    unsigned flags = 0;
    uint32_t *cur = sF0, *nxt = sF1;
    for (int lev = 0; lev < H; ++lev) {
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int i = threadIdx.x + k * blockDim.x;
            // a level moves information at most one site (Manhattan), so the tile's
            // state after the round's H levels depends on a site at distance r only
            // through its state after levels < H - r: iteration lev computes the sites
            // with r <= H - 1 - lev (a shrinking diamond-cornered box; the skipped
            // halo sites are never read by a computed one)
            if (C[k] < 0 || (int)(NB[k] >> 4) > H - 1 - lev) continue;
            BW<NW> F, Fn[4];
            uint32_t any = 0u;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const uint32_t *cw = cur + w * RS + i;
                F.w[w] = cw[0];
                Fn[0].w[w] = (NB[k] & 1u) ? cw[1] : 0u;
                Fn[1].w[w] = (NB[k] & 2u) ? cw[-1] : 0u;
                Fn[2].w[w] = (NB[k] & 4u) ? cw[RW] : 0u;
                Fn[3].w[w] = (NB[k] & 8u) ? cw[-RW] : 0u;
                any |= F.w[w] | Fn[0].w[w] | Fn[1].w[w] | Fn[2].w[w] | Fn[3].w[w];
            }
            if (any == 0u) {   // no frontier next to this site
#pragma unroll
                for (int w = 0; w < NW; ++w) nxt[w * RS + i] = 0u;
                continue;
            }
            // mask word (arc q, word w) of this site: shared memory, or global memory (NW = 8)
#define GZ_MASK(q, w) (PACK ? ((sM[((q) >> 1) * RS + i] >> (((q) & 1) * 16)) & 0xffffu) \
                     : smem_masks(NW) ? sM[((q) * NW + (w)) * RS + i] : __ldg(b.mask + ((size_t)(q) * NW + (w)) * P + C[k]))
            BW<NW> M0;
#pragma unroll
            for (int w = 0; w < NW; ++w) M0.w[w] = GZ_MASK(A_UP, w);
            BW<NW> N = F.shl1() | (F.shr1() & M0);
#pragma unroll
            for (int dir = 0; dir < 4; ++dir) {
                if (!Fn[dir].any()) continue;
                BW<NW> ms, md, mu;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    ms.w[w] = GZ_MASK(A_SR + dir, w);
                    md.w[w] = GZ_MASK(A_DR + dir, w);
                    mu.w[w] = GZ_MASK(A_UR + dir, w);
                }
                N = N | (Fn[dir] & ms) | (Fn[dir].shl1() & md) | (Fn[dir].shr1() & mu);
            }
#undef GZ_MASK
            N = gz2::andnot(N & RNG[k], V[k]);
            V[k] = V[k] | N;
#pragma unroll
            for (int w = 0; w < NW; ++w) nxt[w * RS + i] = N.w[w];
            if (IN_[k] && N.any()) {
                flags |= 1u;
                if ((N & EX[k]).any()) flags |= 2u;
                const int base = C[k] * LPT;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    uint32_t x = N.w[w];
                    while (x) {
                        const int bb = __ffs(x) - 1;
                        x &= x - 1;
                        a.h[base + 32 * w + bb] = d + lev + 1;
                    }
                }
            }
        }
        __syncthreads();
        uint32_t *t = cur; cur = nxt; nxt = t;
    }
    bool fr = false;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        if (!IN_[k]) continue;
        const int i = threadIdx.x + k * blockDim.x;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t f = cur[w * RS + i];
            fr |= f != 0u;
            Fout[(size_t)w * P + C[k]] = f;
        }
        V[k].store(Vout, P, C[k]);
    }
    front = __syncthreads_or(fr) != 0;   // also: shared buffers are reused by the next tile
    return flags;
}

// ---------------------------------------------------------------------------
// The solver.  LP = 16: two sites per warp group (m <= 16); LP = 32: one
// (segment, site) per warp group, R segments per chain (m <= 32 R).
// The whole solve of one problem by one team.  cta / ncta: this CTA's index
// in its launch's share of the team and that share's size (a single launch:
// blockIdx.x / gridDim.x; batched pair solves: the CTA's index in its team).
// phase: the team barrier's running count (kept across the problems a
// batched team solves, so its rotating barrier words stay consistent).
// PP / BB / AA: how the descriptors are held -- by reference to the kernel's
// __grid_constant__ parameters (one launch: read in place from the constant
// bank), or by value (batched teams: per-team shifted copies the compiler can
// keep in registers).
template <int LP, int R, bool WIN, int OCC, int RW = 0, class PP = const Prob &, class BB = const Bits2 &,
          class AA = const Arr3 &>
__device__ __forceinline__ void tilesolve_body(PP p, BB b, AA a, const Geo &g, unsigned long long *bar, const int cta,
                                               const int ncta, int &phase) {
    // RW > 0: window-relative 16-lane groups over rows of 32 RW positions (gz_chain.cuh)
    constexpr int NW = RW ? RW : R, LPT = RW ? 32 * RW : LP * R;
    __shared__ unsigned s_f3[3], s_r3[3], s_qn[2];
    __shared__ int s_q[BLOCK];   // per-round pool of active groups (<= 32 per warp)
    __shared__ unsigned s_tn[2];  // tail-mode worklist lengths
    __shared__ unsigned s_wl[2];  // groups this CTA took from the pulse worklist (alternating)
    extern __shared__ uint32_t s_dyn[];
    __syncthreads();   // (a batched team: every thread is done with the last problem's shared state)
    if (threadIdx.x < 3) { s_f3[threadIdx.x] = 0u; s_r3[threadIdx.x] = 0u; }
    if (threadIdx.x < 2) { s_qn[threadIdx.x] = 0u; s_wl[threadIdx.x] = 0u; }
    int qround = 0;
    __syncthreads();
    constexpr int RS = region_sites(NW, OCC);
    uint32_t *sF0 = s_dyn, *sF1 = s_dyn + NW * RS, *sM = s_dyn + 2 * NW * RS;
    const bool resident = g.t1 - g.t0 <= ncta;   // one tile per CTA: masks stay in smem for the sweep
    const Team tm{bar, p.ctr + CTR_ABORT, g.nb, g.rank0 + cta, g.sys,
                  (unsigned long long)g.spin_ms * 1000000ull};
#define TEAM_SYNC() (void)tm.sync_or(0u, phase, s_f3, s_r3)
#define TEAM_OR(f) tm.sync_or((f), phase, s_f3, s_r3)
#define TEAM_COUNT(f) tm.sync_count((f), phase, s_f3, s_r3)
    // phase timers of thread 0 of rank 0, in shared memory (not 16 registers of every
    // thread): [0..5] phase sums, [6] last tick, [7] start (the watchdog's clock)
    __shared__ unsigned long long s_tm[8];
    unsigned long long *const t_acc = s_tm;
    const bool timer = tm.rank == 0 && threadIdx.x == 0;
    if (timer) {
        for (int q = 0; q < 6; ++q) s_tm[q] = 0ull;
        s_tm[6] = s_tm[7] = gz2::gtimer();
    }
#define t_start (s_tm[7])
#define TICK(slot) do { if (timer) { unsigned long long t_ = gz2::gtimer(); t_acc[slot] += t_ - s_tm[6]; s_tm[6] = t_; } } while (0)
#define FOR_TILES for (int tile = g.t0 + cta; tile < g.t1; tile += ncta)
    long long flow = 0;
    unsigned pushes = 0u, relabels = 0u;   // per thread, flushed to the counters every sweep (32 bits suffice)
    volatile unsigned long long *vctr = p.ctr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    constexpr int CPW = 32 / LP;
    const int nwords = NW * p.P;   // one bit word per (segment, site)
    // warp groups: LP = 16 -> pairs of sites; LP = 32 -> (segment, site) words
    const int ngroups = LP == 16 ? (p.P + 1) / 2 : nwords;
    // this band's groups, interleaved over the warps of this launch: local index li
    // -> site pair gg0 + li (LP = 16), or (segment, site) word of the band's sites
    const int bsites = g.c1 - g.c0, bwords = NW * bsites;
    const int nloc = LP == 16 ? g.gg1 - g.gg0 : bwords;
    const int gnw = ncta * nwarps, gwid = cta * nwarps + warp;
    const int giter = (nloc + gnw - 1) / gnw;
    auto band_word = [&](int i) { const int s_ = i / bsites; return s_ * p.P + g.c0 + (i - s_ * bsites); };
    auto grp_of = [&](int li) { return LP == 16 ? g.gg0 + li : band_word(li); };
    const int ttid = cta * (int)blockDim.x + (int)threadIdx.x, tstride = ncta * (int)blockDim.x;
    // tail mode: claim bitmap + two worklists in the (then idle) BFS shared memory
    const int tail_bw = (ngroups + 31) / 32;
    const int tail_cap = min(4096, ((int)(smem_bytes(OCC) / 4) - tail_bw) / 2);
    const bool tail_ok = tail_cap >= 256 && p.tail_mode;
    long long updates = 0;   // groups processed by pulses (x CPW x LP nodes)
    // Pulse worklists (exact solves, one band): the first pulse of a sweep scans
    // every group's active / inbox words; each later pulse consumes the list the
    // previous one filled (the groups it left active and every group it pushed
    // into) instead of scanning all groups.  Four lists rotate through planes
    // that are idle during pulses (F0, F1, V, RL: list k is filled in pulse k-1,
    // consumed in k, its claim bits cleared in k+1, its length reset in k+2);
    // duplicates are dropped by claim bitmaps (two, alternating, in R0).  A list
    // that overflowed falls back to the scan.  Auto (p.worklist < 0): on when a
    // scan takes many rounds per warp (C3q 1.82 -> 1.59 s) and for the
    // concurrent occupancy-2 instance (bench +2.5%); off for lone solves whose
    // scan is one or a few rounds (C1 / C2 lone: the scan is 6-25% faster).
    // With row bands every band keeps its own four lists (in its own sites' part of
    // the planes) and lengths (R1, idle during pulses); pushes route to the band
    // of the target group.  Auto leaves them off for row bands: C3q as two bands
    // on one GPU took 2.61 s with band worklists against 2.09 s scanning (the
    // routing arithmetic per push, round 1); GZ_WORKLIST=1 forces them on.
    const bool wl_on = (p.worklist > 0 || (p.worklist < 0 && g.nbands == 1 && (OCC == 2 || giter >= 16 * 32))) &&
                       !p.capped && p.async_l == 0;
    const int wl_cap = NW * (g.c1 - g.c0);
    const int wl_bw = (ngroups + 31) / 32;
    int *wl_plane[4] = {(int *)b.F0, (int *)b.F1, (int *)b.V, (int *)b.RL};
    const int *wl_list[4] = {wl_plane[0] + (size_t)NW * g.c0, wl_plane[1] + (size_t)NW * g.c0,
                             wl_plane[2] + (size_t)NW * g.c0, wl_plane[3] + (size_t)NW * g.c0};
    uint32_t *wl_bits[2] = {(uint32_t *)b.R0, (uint32_t *)b.R0 + wl_bw};
    unsigned *wl_n = (unsigned *)b.R1 + g.c0;   // this band's 4 list lengths

    // Scan the warps' interleaved groups (group it0+lane of every warp, 32 per
    // round), pool the ones whose word(s) in W1 | W2 are nonzero in shared memory,
    // and deal the pool round-robin to the CTA's warps: the critical path of a
    // phase is the busiest warp, and pooling per CTA flattens the Poisson spread
    // of active groups across warps.  Two pool counters alternate by round.
#define FOR_ACTIVE_GROUPS(W1, W2, CNT, CTAN, FN)                                                         \
    for (int it0 = 0; it0 < giter; it0 += 32, ++qround) {                                        \
        const int it_ = it0 + lane;                                                              \
        const int li_ = gwid + it_ * gnw;                                                        \
        const int grp_ = li_ < nloc ? grp_of(li_) : 0;                                           \
        uint32_t wk_ = 0u;                                                                       \
        if (it_ < giter && li_ < nloc) {                                                         \
            if (LP == 16) {                                                                      \
                for (int w_ = 0; w_ < NW; ++w_) {                                                \
                    const int q_ = w_ * p.P + 2 * grp_;                                          \
                    wk_ |= __ldcg((W1) + q_) | __ldcg((W2) + q_);                                \
                    if (2 * grp_ + 1 < p.P) wk_ |= __ldcg((W1) + q_ + 1) | __ldcg((W2) + q_ + 1); \
                }                                                                                \
            } else {                                                                             \
                wk_ = __ldcg((W1) + grp_) | __ldcg((W2) + grp_);                                 \
            }                                                                                    \
        }                                                                                        \
        const uint32_t msk_ = __ballot_sync(FULL, wk_ != 0u);                                    \
        CNT += __popc(msk_);                                                                     \
        unsigned *qn_ = s_qn + (qround & 1);                                                     \
        int base_ = 0;                                                                           \
        if (lane == 0 && msk_) base_ = (int)atomicAdd(qn_, (unsigned)__popc(msk_));              \
        base_ = __shfl_sync(FULL, base_, 0);                                                     \
        if ((msk_ >> lane) & 1u) s_q[base_ + __popc(msk_ & ((1u << lane) - 1u))] = grp_;         \
        __syncthreads();                                                                         \
        if (threadIdx.x == 0) s_qn[(qround + 1) & 1] = 0u;                                       \
        const int n_ = (int)*qn_;                                                                \
        CTAN += n_;                                                                              \
        for (int q_ = warp; q_ < n_; q_ += nwarps) {                                             \
            const int gg_ = s_q[q_];                                                             \
            const int cb_ = LP == 16 ? 2 * gg_ : gg_ % p.P, sg_ = LP == 16 ? 0 : gg_ / p.P;      \
            FN(cb_, sg_);                                                                        \
        }                                                                                        \
        __syncthreads();                                                                         \
    }

    long long offset = 0, presat = 0;
    FOR_TILES {
        const TileBox tb(p, g, tile);
        for_tile_groups<LP>(p, tb, [&](int cb, int ns) { gz3::w_init<LP, R, WIN, RW>(p, a, cb, ns, flow, offset, presat); });
    }
    // (published now: no live registers for them through the solve)
    warp_add_u64(&p.ctr[CTR_OFFSET], offset, p.sys);
    if (!p.init_only) warp_add_u64(&p.ctr[CTR_PRESAT], presat, p.sys);
    for (int i = ttid; i < bwords; i += tstride) b.IN[band_word(i)] = 1u;   // every site starts dirty
    TEAM_SYNC();
    TICK(0);
    if (p.init_only) return;   // graph export: the state planes now hold the capacities
    int sweeps = 0, levels_total = 0, pulses = 0, parity = 0;
    const uint32_t *v_last = nullptr;   // capped stop: visited words of the final (exhaustive) BFS
    int converged = 1;
    bool err = false;
    int bfs_min = p.bfs_cap > 0 ? p.bfs_cap : (1 << 30);
    for (;;) {
        // ---- sweep set-up: bulk coalesced resets, then arc masks of dirty sites only ----
        // (every inbox is merged by the builds below, so the inbox parity restarts)
        parity = 0;
        if (threadIdx.x == 0 && tm.rank == 0) p.ctr[CTR_TQN] = 0ull;
        for (int i = ttid; i < bwords; i += tstride) {
            const int s = i / bsites, c = g.c0 + (i - s * bsites), w = s * p.P + c;
            const int hi = WIN ? p.hi[c] : p.L;
            b.F0[w] = BW<NW>::range(hi, p.M).w[s];
            b.V[w] = 0u;
        }
        {
            const int4 hinf4 = make_int4(HINF, HINF, HINF, HINF);
            int4 *h4 = reinterpret_cast<int4 *>(a.h);
            const int n4 = g.c1 * (LPT / 4);
            for (int q = g.c0 * (LPT / 4) + ttid; q < n4; q += tstride) h4[q] = hinf4;
        }
        {
            long long dummy = 0;
            int dummy2 = 0;
            auto build = [&](int cb, int sg) {
                gz3::w_build<LP, R, WIN, RW>(p, a, b, cb, CPW, sg);
                if (RW) {   // dirty marks: every bit word of both sites
                    if (lane < CPW && cb + lane < p.P)
                        for (int w = 0; w < NW; ++w) b.IN[w * p.P + cb + lane] = 0u;
                } else {
                    const int w0 = sg * p.P + cb;
                    if (lane < CPW && cb + lane < p.P) b.IN[w0 + lane] = 0u;
                }
            };
            FOR_ACTIVE_GROUPS(b.IN, b.IN, dummy, dummy2, build)
        }
        TEAM_SYNC();
        TICK(1);
        // ---- global relabel: temporally blocked BFS ----
        int d = 0, d_found = 0;
        bool found = false, exhausted = false;
        uint32_t *Fin = b.F0, *Fout = b.F1, *Vin = b.V, *Vout = b.RL;
        // the capped solve's last sweep: its BFS runs to exhaustion, because the
        // capped labeling is read from it (the nodes that cannot reach the sink)
        const bool last = p.capped && sweeps >= p.max_sweeps;
        // per-tile "interior frontier nonempty" flags of the last round (reach arrays
        // are idle during the BFS); a tile whose neighbourhood within H sites had no
        // frontier cannot gain nodes this round and only carries its words forward
        int32_t *tf_in = b.R1, *tf_out = b.R1 + g.ntiles;
        // consecutive inactive rounds per tile: after two, both frontier/visited
        // buffers already hold (no frontier, unchanged visited) and the tile's
        // carry-forward copy is skipped (each tile is handled by one CTA)
        int32_t *tl_idle = 3 * g.ntiles <= 2 * p.P ? b.R1 + 2 * g.ntiles : nullptr;
        const int rty = (g.H + g.TY - 1) / g.TY, rtx = (g.H + g.TX - 1) / g.TX;
        // a tile is active in a round if a tile within H sites had frontier in the
        // last one; the flags of all of this CTA's tiles are gathered at the start of
        // the round by its threads in parallel (independent loads: one round trip
        // instead of up to 9 dependent ones per tile), into s_q (idle during BFS)
        auto tile_act = [&](int tile) {
            const int ty = tile / g.nx, tx = tile - ty * g.nx;
            bool a_ = false;
            for (int dy = -rty; dy <= rty; ++dy)
                for (int dx = -rtx; dx <= rtx; ++dx) {
                    const int yy = ty + dy, xx = tx + dx;
                    if (yy >= 0 && yy < g.ny && xx >= 0 && xx < g.nx) a_ |= __ldcg(tf_in + yy * g.nx + xx) != 0;
                }
            return a_;
        };
        for (;;) {
            unsigned flags = 0;
            if (d > 0) {
                for (int k = threadIdx.x, tile = g.t0 + cta + k * ncta; k < BLOCK && tile < g.t1;
                     k += blockDim.x, tile += (int)blockDim.x * ncta)
                    s_q[k] = tile_act(tile) ? 1 : 0;
                __syncthreads();
            }
            int tk = 0;
            FOR_TILES {
                const TileBox tb(p, g, tile);
                const bool act = d == 0 || (tk < BLOCK ? s_q[tk] != 0 : tile_act(tile));
                ++tk;
                bool front = false;
                const int idle = (d == 0 || !tl_idle) ? 0 : tl_idle[tile];
                if (act) {
                    flags |= bfs_round<LPT, NW, WIN, OCC>(p, a, b, g, tb, Fin, Fout, Vin, Vout, d, sF0, sF1, sM,
                                                         d == 0 || !resident, front);
                } else if (idle < 2) {
                    for (int r = tb.y0 + warp; r < tb.y1; r += nwarps)
                        for (int x = tb.x0 + lane; x < tb.x1; x += 32)
                            for (int w = 0; w < NW; ++w) {
                                const size_t q = (size_t)w * p.P + r * p.G + x;
                                Fout[q] = 0u;
                                Vout[q] = Vin[q];
                            }
                }
                if (threadIdx.x == 0) {
                    tf_out[tile] = front ? 1 : 0;
                    if (tl_idle) tl_idle[tile] = act ? 0 : (idle < 2 ? idle + 1 : 2);
                }
            }
            const unsigned gf = TEAM_OR(flags);
            if (!found && (gf & 2u)) d_found = d + g.H;
            found |= (gf & 2u) != 0;
            uint32_t *t = Fin; Fin = Fout; Fout = t;
            t = Vin; Vin = Vout; Vout = t;
            int32_t *tt = tf_in; tf_in = tf_out; tf_out = tt;
            d += g.H;
            if (!(gf & 1u)) { exhausted = true; break; }
            if (found && d >= bfs_min && !last) break;
            if (d > 4 * (p.P + p.M) + 4 * g.H) { if (threadIdx.x == 0 && tm.rank == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); err = true; break; }
        }
        levels_total += d;
        // adaptive depth (p.bfs_adapt): excess met only beyond the current early-stop
        // depth means the near region is drained -- double the depth
        if (p.bfs_adapt && found && d_found > bfs_min && bfs_min < (1 << 29)) bfs_min *= 2;
        TICK(2);
        if (err) break;
        if (!found && exhausted) break;
        if (last) { converged = 0; v_last = Vin; break; }
        for (int i = ttid; i < bwords; i += tstride) {
            const int w = band_word(i);
            b.A[w] = Vin[w] & b.EX[w];
            if (p.capped) b.RL[w] = 0u;   // (the BFS used RL as a visited buffer)
        }
        if (wl_on) {
            for (int i = tm.rank * blockDim.x + threadIdx.x; i < 2 * wl_bw; i += tm.nb * blockDim.x) wl_bits[0][i] = 0u;
            if (threadIdx.x == 0 && cta == 0)
                for (int i = 0; i < 4; ++i) wl_n[i] = 0u;
        }
        TEAM_SYNC();
        unsigned long long t_pulse = p.trace > 1 ? gz2::gtimer() : 0ull;
        // pulses this sweep: K, or K_tail once the dense opening sweeps are over
        const int kp = (p.k_tail > 0 && sweeps >= p.tail_after) ? p.k_tail : p.K;
        for (int pulse = 0; pulse < kp; ++pulse) {
            // Pulses are NOT tile-owned: active chains cluster spatially, so groups are
            // interleaved over every warp of the team (group g -> warp g mod W).  Lane i of
            // a warp checks the i-th of the warp's groups in one load; only groups with
            // active or inbox bits run a pulse.
            const uint32_t *IN_prev = parity ? a.IN0 : a.IN1;
            auto pulse_fn = [&](int cb, int sg) {
                gz3::w_pulse<LP, R, WIN, false, false, RW>(p, a, b, cb, CPW, sg, parity, flow, pushes, relabels, b.IN);
            };
            long long upd0 = updates;
            int cta_groups = 0;
            if (p.capped) {
                // deterministic (capped, level-2) pulse: push | relabel into h2 | commit,
                // each phase reading state no concurrent phase writes
                int32_t *h2 = a.ein1;   // the second inbox plane is idle in this mode
                auto push_fn = [&](int cb, int sg) {
                    gz3::w_pulse<LP, R, WIN, false, true, RW>(p, a, b, cb, CPW, sg, 0, flow, pushes, relabels, b.IN);
                };
                FOR_ACTIVE_GROUPS(b.A, b.A, updates, cta_groups, push_fn)
                TEAM_SYNC();
                long long dmy = 0;
                int dmy2 = 0;
                auto relabel_fn = [&](int cb, int sg) { gz3::w_relabel<LP, R, WIN, RW>(p, a, b, cb, CPW, sg, h2, relabels); };
                FOR_ACTIVE_GROUPS(b.RL, b.RL, dmy, dmy2, relabel_fn)
                TEAM_SYNC();
                auto commit_fn = [&](int cb, int sg) { gz3::w_commit<LP, R, WIN, RW>(p, a, b, cb, CPW, sg, h2); };
                FOR_ACTIVE_GROUPS(b.RL, a.IN0, dmy, dmy2, commit_fn)
            } else if (p.async_l > 0) {
                // asynchronous pulse: async_l scan-and-process iterations per team
                // barrier; pushes between warps are picked up within the pulse
                auto pulse_async = [&](int cb, int sg) {
                    gz3::w_pulse<LP, R, WIN, true, false, RW>(p, a, b, cb, CPW, sg, 0, flow, pushes, relabels, b.IN);
                };
                for (int ai = 0; ai < p.async_l; ++ai) {
                    FOR_ACTIVE_GROUPS(b.A, a.IN0, updates, cta_groups, pulse_async)
                }
            } else if (wl_on) {
                const int k4 = pulse & 3;
                const gz3::BandRoute rt{wl_plane[(k4 + 1) & 3], (unsigned *)b.R1 + ((k4 + 1) & 3), g.ny, g.nbands,
                                        g.TY, p.G, p.Y, p.P, NW, LP == 16 ? 1 : 0, p.sys};
                const gz3::TailQ nq{nullptr, nullptr, 0, &rt, p.wl_dedupe};
                auto pulse_wl = [&](int cb, int sg) {
                    gz3::w_pulse<LP, R, WIN, false, false, RW>(p, a, b, cb, CPW, sg, parity, flow, pushes, relabels,
                                                               b.IN, &nq);
                };
                const unsigned n_cur = *(volatile unsigned *)(wl_n + k4);
                if (pulse == 0 || n_cur > (unsigned)wl_cap) {
                    FOR_ACTIVE_GROUPS(b.A, IN_prev, updates, cta_groups, pulse_wl)
                } else {
                    const int *lst = wl_list[k4];
                    uint32_t *bits = wl_bits[pulse & 1];
                    unsigned mine = 0;
                    // chunks of `per` consecutive entries per warp: the lanes load and
                    // claim a whole chunk at once (one round trip), then the warp runs
                    // the groups it won; chunks shrink to one entry when the list is
                    // short next to the team's warps (load balance)
                    const int per = min(32, max(1, (int)n_cur / gnw));
                    for (int q0 = gwid * per; q0 < (int)n_cur; q0 += gnw * per) {
                        const int qi = q0 + lane;
                        const bool in = lane < per && qi < (int)n_cur;
                        const int gg = in ? __ldcg(lst + qi) : 0;
                        unsigned old = 1u << (gg & 31);
                        if (in) old = gz_atomic_or(p, &bits[gg >> 5], 1u << (gg & 31));
                        uint32_t won = __ballot_sync(FULL, in && !((old >> (gg & 31)) & 1u));
                        while (won) {   // (a group listed twice in one chunk is won once)
                            const int src = __ffs(won) - 1;
                            won &= won - 1;
                            const int g2 = __shfl_sync(FULL, gg, src);
                            pulse_wl(LP == 16 ? 2 * g2 : g2 % p.P, LP == 16 ? 0 : g2 / p.P);
                            ++mine;
                        }
                    }
                    updates += mine;
                    if (lane == 0 && mine) atomicAdd(&s_wl[pulse & 1], mine);
                    __syncthreads();
                    cta_groups += (int)s_wl[pulse & 1];
                    if (threadIdx.x == 0) s_wl[(pulse + 1) & 1] = 0u;
                }
                // claim bits of the list consumed in the previous pulse
                if (pulse >= 1) {
                    const unsigned n_prev = *(volatile unsigned *)(wl_n + ((k4 + 3) & 3));
                    if (n_prev <= (unsigned)wl_cap) {
                        const int *lq = wl_list[(k4 + 3) & 3];
                        uint32_t *bq = wl_bits[(pulse + 1) & 1];
                        for (int q = ttid; q < (int)n_prev; q += tstride) bq[__ldcg(lq + q) >> 5] = 0u;
                    }
                }
                if (threadIdx.x == 0 && cta == 0) wl_n[(k4 + 2) & 3] = 0u;   // refilled from pulse + 1 on
            } else {
                FOR_ACTIVE_GROUPS(b.A, IN_prev, updates, cta_groups, pulse_fn)
            }
            if (p.trace > 1 && lane == 0 && updates != upd0) atomicAdd(&p.ctr[CTR_TRACE], (unsigned long long)(updates - upd0));
            // an empty pulse (no active or inbox word anywhere) ends the sweep early;
            // a nearly empty one hands the rest of the sweep to CTA 0 (tail mode)
            const unsigned cnt = TEAM_COUNT((cta_groups > 0 ? 1u : 0u) | (cta_groups > TAIL_CTA_GROUPS ? 2u : 0u));
            const bool idle = (cnt & 0xffffu) == 0u;
            if (p.trace > 1 && p.tbuf && threadIdx.x == 0 && tm.rank == 0 && pulses < 4096) {
                const unsigned long long now = gz2::gtimer();
                p.tbuf[2 * pulses] = ((unsigned long long)sweeps << 48) | ((unsigned long long)pulse << 32) |
                                     ((volatile unsigned long long *)p.ctr)[CTR_TRACE];
                p.tbuf[2 * pulses + 1] = now - t_pulse;
                t_pulse = now;
                p.ctr[CTR_TRACE] = 0ull;
            }
            parity ^= 1;
            ++pulses;
            if (idle) break;
            if (tail_ok && p.async_l == 0 && !p.capped && sweeps >= p.tail_after && pulse + 1 < kp &&
                (g.nb == 1 ? cta_groups <= p.tail_groups : ((cnt >> 16) == 0u && (int)(cnt & 0xffffu) <= (p.tail_ctas > 0 ? p.tail_ctas : TAIL_CTAS)))) {
                // ---- tail mode: the few active groups go to CTA 0, which runs the rest of
                // the sweep's pulses on a shared-memory worklist with CTA barriers only ----
                const uint32_t *INn = parity ? a.IN0 : a.IN1;
                unsigned *gq_n = (unsigned *)&p.ctr[CTR_TQN];
                int *gq = (int *)b.F1;   // BFS frontier buffer, idle during pulses
                for (int it0 = 0; it0 < giter; it0 += 32) {
                    const int it_ = it0 + lane, li_ = gwid + it_ * gnw;
                    const int grp_ = li_ < nloc ? grp_of(li_) : 0;
                    uint32_t wk_ = 0u;
                    if (it_ < giter && li_ < nloc) {
                        if (LP == 16) {
                            for (int w_ = 0; w_ < NW; ++w_) {
                                const int q_ = w_ * p.P + 2 * grp_;
                                wk_ |= b.A[q_] | INn[q_];
                                if (2 * grp_ + 1 < p.P) wk_ |= b.A[q_ + 1] | INn[q_ + 1];
                            }
                        } else {
                            wk_ = b.A[grp_] | INn[grp_];
                        }
                    }
                    const uint32_t msk_ = __ballot_sync(FULL, wk_ != 0u);
                    int base_ = 0;
                    if (lane == 0 && msk_) base_ = (int)gz_atomic_add(p, gq_n, (unsigned)__popc(msk_));
                    base_ = __shfl_sync(FULL, base_, 0);
                    if ((msk_ >> lane) & 1u) gq[base_ + __popc(msk_ & ((1u << lane) - 1u))] = grp_;
                }
                TEAM_SYNC();
                if (tm.rank == 0) {
                    uint32_t *bits = s_dyn;                       // claim bitmap over groups
                    int *qa = (int *)(s_dyn + tail_bw), *qb = qa + tail_cap;
                    const int n0 = (int)*(volatile unsigned *)gq_n;
                    if (n0 <= tail_cap) {
                        for (int w = threadIdx.x; w < tail_bw; w += blockDim.x) bits[w] = 0u;
                        for (int q = threadIdx.x; q < n0; q += blockDim.x) qa[q] = gq[q];
                        if (threadIdx.x == 0) { s_tn[0] = (unsigned)n0; s_tn[1] = 0u; }
                        __syncthreads();
                        int cur = 0;
                        for (int tp = pulse + 1; tp < kp; ++tp) {
                            const int n = (int)min(s_tn[cur], (unsigned)tail_cap);
                            if (n == 0) break;
                            int *ql = cur ? qb : qa;
                            const gz3::TailQ tq{cur ? qa : qb, &s_tn[cur ^ 1], tail_cap};
                            for (int q = warp; q < n; q += nwarps) {
                                const int gg = ql[q];
                                unsigned old = 0u;
                                if (lane == 0) old = atomicOr(&bits[gg >> 5], 1u << (gg & 31));
                                old = __shfl_sync(FULL, old, 0);
                                if ((old >> (gg & 31)) & 1u) continue;   // already processed this pulse
                                const int cb = LP == 16 ? 2 * gg : gg % p.P, sg = LP == 16 ? 0 : gg / p.P;
                                gz3::w_pulse<LP, R, WIN, false, false, RW>(p, a, b, cb, CPW, sg, parity, flow, pushes, relabels, b.IN, &tq);
                                ++updates;
                            }
                            __syncthreads();
                            for (int q = threadIdx.x; q < n; q += blockDim.x) bits[ql[q] >> 5] = 0u;
                            const bool ovf = s_tn[cur ^ 1] > (unsigned)tail_cap;
                            __syncthreads();
                            if (threadIdx.x == 0) s_tn[cur] = 0u;
                            if (p.trace > 1 && p.tbuf && threadIdx.x == 0 && pulses < 4096) {   // tail pulses: pulse + 1000
                                const unsigned long long now = gz2::gtimer();
                                p.tbuf[2 * pulses] = ((unsigned long long)sweeps << 48) |
                                                     ((unsigned long long)(1000 + tp) << 32) | (unsigned long long)n;
                                p.tbuf[2 * pulses + 1] = now - t_pulse;
                                t_pulse = now;
                            }
                            parity ^= 1;
                            ++pulses;
                            cur ^= 1;
                            __syncthreads();
                            if (ovf) break;   // worklist overflow: the A / inbox words hold the rest
                        }
                    }
                }
                TEAM_SYNC();
                break;
            }
        }
        TICK(3);
        ++sweeps;
        warp_add_u64(&p.ctr[CTR_PUSHES], pushes, p.sys);
        warp_add_u64(&p.ctr[CTR_RELABELS], relabels, p.sys);
        pushes = relabels = 0u;
        if (p.trace && threadIdx.x == 0 && tm.rank == 0)
            printf("gz_trace sweep %d levels %d pulses %d t %.3f ms bfs %.3f pulses %.3f\n", sweeps, d, pulses,
                   (gz2::gtimer() - t_start) * 1e-6, t_acc[2] * 1e-6, t_acc[3] * 1e-6);
        {
            unsigned stop = 0;
            if (threadIdx.x == 0 && tm.rank == 0 && p.watchdog_ns && gz2::gtimer() - t_start > p.watchdog_ns) stop = 1;
            if (TEAM_OR(stop)) {
                if (threadIdx.x == 0 && tm.rank == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE);
                break;
            }
        }
        if (sweeps > 1000000) { if (threadIdx.x == 0 && tm.rank == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
    }
#undef FOR_ACTIVE_GROUPS
    // ---- extraction: prefix closure from the excess nodes ----
#define FOR_TILE_SITES                                                              \
    FOR_TILES                                                                       \
    for (int r = TileBox(p, g, tile).y0 + warp, y1_ = TileBox(p, g, tile).y1; r < y1_; r += nwarps) \
        for (int x = TileBox(p, g, tile).x0 + lane, x1_ = TileBox(p, g, tile).x1; x < x1_; x += 32)
    // A capped stop reads the labeling off the last BFS instead: every node that
    // cannot reach the sink in the residual network goes to the source side (a
    // valid cut for any preflow; its cost is the sink inflow plus the excess
    // still able to reach the sink, and it becomes a minimum cut as the capped
    // preflow converges).  Reaching the sink is closed upward along a chain
    // (uncuttable chain arcs down), so the source side is a prefix.
    const bool capped_stop = v_last != nullptr;
    if (!capped_stop) FOR_TILE_SITES gz3::w_reach_init<NW, WIN, LPT == 16>(p, b, r * p.G + x);
    TEAM_SYNC();
    int reach_passes = 0;
    // In place (Gauss-Seidel): R only grows and every value a pass reads is a
    // lower bound of the fixpoint, so a read of a neighbour already updated in
    // this pass is as valid as the old one and converges in fewer passes; a
    // pass that changes nothing read only settled values, i.e. the fixpoint.
    int32_t *const Rin = b.R0;
    for (; !capped_stop;) {
        unsigned ch = 0;
        FOR_TILE_SITES ch |= gz2::bit_reach_iter<WIN, NW, LPT == 16>(p, b, r * p.G + x, Rin) ? 1u : 0u;
        const bool any = TEAM_OR(ch) != 0;
        ++reach_passes;
        if (!any) break;
        if (reach_passes > 4 * (p.P + p.M)) { if (threadIdx.x == 0 && tm.rank == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
    }
    TICK(4);
    long long stranded = 0;
    FOR_TILE_SITES {
        const int c = r * p.G + x;
        const int lo = WIN ? p.lo[c] : 0;
        if (capped_stop) {
            const int hi = WIN ? p.hi[c] : p.L;
            BW<NW> v;
            v.load(v_last, p.P, c);
            v = v & BW<NW>::range(lo, hi);
            int reach = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) reach += __popc(v.w[w]);
            p.labels[c] = hi - reach;
        } else {
            p.labels[c] = lo + Rin[c];
        }
        for (int w = 0; w < NW; ++w) stranded += __popc(b.EX[(size_t)w * p.P + c]);
    }
    TEAM_SYNC();
    long long energy = 0;
    int viol = 0;
    FOR_TILE_SITES gz3::w_energy<LPT>(p, a, r * p.G + x, energy, viol);
#undef FOR_TILE_SITES
#undef FOR_TILES
#undef TEAM_SYNC
#undef TEAM_OR
#undef TEAM_COUNT
    TICK(5);
#undef TICK
#undef t_start
    if (timer)
        for (int q = 0; q < 6; ++q) p.ctr[CTR_T0 + q] = t_acc[q];
    warp_add_u64(&p.ctr[CTR_FLOW], flow, p.sys);
    warp_add_u64(&p.ctr[CTR_PUSHES], pushes, p.sys);
    warp_add_u64(&p.ctr[CTR_RELABELS], relabels, p.sys);
    warp_add_u64(&p.ctr[CTR_ENERGY], energy, p.sys);
    warp_add_u64(&p.ctr[CTR_STRANDED], stranded, p.sys);
    if (lane == 0 && updates) gz_atomic_add(p, &p.ctr[CTR_UPDATES], (unsigned long long)updates * CPW * (LP < p.L ? LP : p.L));
    if (viol) p.ctr[CTR_HARDVIOL] = 1;
    if (threadIdx.x == 0 && tm.rank == 0) {
        p.ctr[CTR_SWEEPS] = sweeps;
        p.ctr[CTR_BFS_PASSES] = levels_total;
        p.ctr[CTR_REACH_PASSES] = reach_passes;
        p.ctr[CTR_CONVERGED] = converged;
        p.ctr[CTR_PULSES] = pulses;
    }
}

template <int LP, int R, bool WIN, int OCC, int RW = 0>
// (__grid_constant__: the body reads the parameters in place, from the constant bank)
__global__ void __launch_bounds__(BLOCK, OCC) gz_tilesolve_kernel(const __grid_constant__ Prob p,
                                                                  const __grid_constant__ Bits2 b,
                                                                  const __grid_constant__ Arr3 a,
                                                                  const __grid_constant__ Geo g,
                                                                  unsigned long long *bar) {
    int phase = 0;
    tilesolve_body<LP, R, WIN, OCC, RW>(p, b, a, g, bar, (int)blockIdx.x, (int)gridDim.x, phase);
}

// ---------------------------------------------------------------------------
// Batched pair solves (gz_solve_pairs, BASELINE config 4): ONE launch of
// nteams x T CTAs; team k (CTAs kT .. kT+T-1) owns workspace slice k and takes
// pairs from a global queue until the batch is done.  Per pair the team
// computes the data term (energy.py:83-114 / k_sad) straight into its volume
// plane, clears its bit planes and counters, runs the whole solve, and copies
// its counters to the pair's stats row.  Small teams waste no time on
// cross-SM barriers (T = 1: the CTA barrier is the team barrier) and keep many
// pairs in flight; one launch avoids the per-stream concurrency limit of
// separate cooperative launches (CUDA_DEVICE_MAX_CONNECTIONS).
//
// Tail launch: small teams are the most efficient per CTA, but once the queue
// runs dry a team that finishes early idles until the slowest pair in flight
// is done.  The last pairs therefore go to a SECOND launch of bigger teams
// (T2 CTAs), issued on another stream as soon as the first launch's queue is
// empty (the first launch raises a host-visible flag; the host then launches):
// its CTAs take the SM slots the first launch's CTAs free as they exit.  It
// cannot deadlock -- the first launch is fully resident by then and never
// waits on the second -- and a tail team works in the workspace slice of a
// finished small team (released once all its CTAs are done, `free`).
struct PairBatch {
    const uint8_t *left, *right;   // batch x (img_h, img_w, ch) uint8
    int img_w, ch;
    size_t img_bytes;
    gz_cuboid cb;
    int batch, T;                   // this launch hands out pairs [lo, batch)
    size_t ws_stride;               // bytes between two teams' workspace slices
    size_t bits_bytes;              // bytes of the bit planes to clear per pair
    int32_t *labels_out;            // batch x P
    unsigned long long *stats;      // batch x CTR_COUNT counters
    unsigned *queue;                // next pair to hand out (relative to lo)
    int lo;
    int tail;                       // 0: first launch (slice = team); 1: tail launch (slices from `free`)
    unsigned *drained;              // host-mapped: set when the first launch's queue runs dry (or nullptr)
    unsigned *done;                 // first launch: per team, CTAs done
    int *free_slices;               // released slices, in release order (-1: not yet)
    unsigned *free_n;               // [0] released, [1] taken
    int *pub;                       // tail launch: per team, 1 + its slice
};

template <typename T>
__device__ __forceinline__ T *shifted(T *q, size_t off) { return q ? (T *)((uint8_t *)q + off) : q; }

template <int LP, int R, int OCC>
__global__ void __launch_bounds__(BLOCK, OCC) gz_pairs_kernel(const __grid_constant__ Prob p0,
                                                              const __grid_constant__ Bits2 b0,
                                                              const __grid_constant__ Arr3 a0,
                                                              const __grid_constant__ Geo g, PairBatch pb) {
    const int T = pb.T, team = (int)blockIdx.x / T, cta = (int)blockIdx.x % T;
    size_t off = (size_t)team * pb.ws_stride;
    if (pb.tail) {
        // a tail team takes the next released slice (CTA 0) and clears its
        // barrier words and pair slot before the team's first barrier
        __shared__ int s_slice;
        if (threadIdx.x == 0) {
            int sl;
            if (cta == 0) {
                const unsigned k = atomicAdd(pb.free_n + 1, 1u);
                while ((sl = *(volatile int *)&pb.free_slices[k]) < 0) __nanosleep(1000);
                __threadfence();
                unsigned long long *c = (unsigned long long *)((uint8_t *)p0.ctr + (size_t)sl * pb.ws_stride);
                for (int i = 0; i < CTR_COUNT; ++i) ((volatile unsigned long long *)c)[i] = 0ull;
                __threadfence();
                *(volatile int *)&pb.pub[team] = sl + 1;
            } else {
                while ((sl = *(volatile int *)&pb.pub[team]) == 0) __nanosleep(1000);
                sl -= 1;
                __threadfence();
            }
            s_slice = sl;
        }
        __syncthreads();
        off = (size_t)s_slice * pb.ws_stride;
    }
    Prob p = p0;
    p.vol = shifted(p.vol, off); p.cu = shifted(p.cu, off); p.ph = shifted(p.ph, off); p.pv = shifted(p.pv, off);
    p.dar = shifted(p.dar, off); p.dbr = shifted(p.dbr, off); p.dad = shifted(p.dad, off); p.dbd = shifted(p.dbd, off);
    p.e = shifted(p.e, off); p.ein = shifted(p.ein, off); p.h = shifted(p.h, off); p.h2 = shifted(p.h2, off);
    p.reach = shifted(p.reach, off); p.reach2 = shifted(p.reach2, off); p.ctr = shifted(p.ctr, off);
    Bits2 b = b0;
    b.mask = shifted(b.mask, off); b.V = shifted(b.V, off); b.F0 = shifted(b.F0, off); b.F1 = shifted(b.F1, off);
    b.A = shifted(b.A, off); b.IN = shifted(b.IN, off); b.EX = shifted(b.EX, off); b.RL = shifted(b.RL, off);
    b.R0 = shifted(b.R0, off); b.R1 = shifted(b.R1, off);
    Arr3 a = a0;
    a.vol = shifted(a.vol, off); a.cu = shifted(a.cu, off); a.ph = shifted(a.ph, off); a.pv = shifted(a.pv, off);
    a.dar = shifted(a.dar, off); a.dbr = shifted(a.dbr, off); a.dad = shifted(a.dad, off); a.dbd = shifted(a.dbd, off);
    a.e = shifted(a.e, off); a.ein0 = shifted(a.ein0, off); a.ein1 = shifted(a.ein1, off); a.h = shifted(a.h, off);
    a.IN0 = shifted(a.IN0, off); a.IN1 = shifted(a.IN1, off);
    unsigned long long *bar = p.ctr + CTR_BAR0;
    uint32_t *bits = b.mask;   // the bit planes are one contiguous run starting at the masks
    const Team tm{bar, p.ctr + CTR_ABORT, T, cta, 0, 0ull};
    __shared__ unsigned s_t3[3], s_u3[3];
    __shared__ int s_pair;
    __shared__ unsigned long long s_tdraw;
    // timeline words after the two queue counters: u64 [1] queue dry, [2] tail launch start
    if (pb.tail && blockIdx.x == 0 && threadIdx.x == 0) *(unsigned long long *)(pb.queue + 3) = gz2::gtimer();
    if (threadIdx.x < 3) { s_t3[threadIdx.x] = 0u; s_u3[threadIdx.x] = 0u; }
    __syncthreads();
    int phase = 0;
    const int P = p.P, ttid = cta * (int)blockDim.x + (int)threadIdx.x, tstride = T * (int)blockDim.x;
    for (;;) {
        // ---- next pair: CTA 0 of the team draws it, the team barrier publishes it ----
        if (cta == 0 && threadIdx.x == 0) {
            const int k = pb.lo + (int)atomicAdd(pb.queue, 1u);
            s_tdraw = gz2::gtimer();
            if (k == pb.batch && !pb.tail) *(unsigned long long *)(pb.queue + 2) = s_tdraw;   // queue dry (timeline)
            if (T == 1) s_pair = k;
            else *(volatile int *)&p.ctr[CTR_PAIR] = k;
            if (k >= pb.batch && pb.drained && !*(volatile unsigned *)pb.drained) {
                *(volatile unsigned *)pb.drained = 1u;   // the host may launch the tail now
                __threadfence_system();
            }
        }
        (void)tm.sync_or(0u, phase, s_t3, s_u3);
        const int pair = T == 1 ? s_pair : *(volatile int *)&p.ctr[CTR_PAIR];
        if (pair >= pb.batch) break;
        // ---- clear the team's bit planes and counters, data term into the volume plane ----
        {
            uint4 *z = reinterpret_cast<uint4 *>(bits);
            const size_t n16 = pb.bits_bytes / 16;
            for (size_t i = ttid; i < n16; i += tstride) z[i] = make_uint4(0u, 0u, 0u, 0u);
            if (cta == 0 && threadIdx.x < CTR_COUNT && threadIdx.x != CTR_PAIR &&
                (threadIdx.x < CTR_BAR0 || threadIdx.x > CTR_BAR0 + 2))
                p.ctr[threadIdx.x] = 0ull;
            const uint8_t *lp = pb.left + (size_t)pair * pb.img_bytes, *rp = pb.right + (size_t)pair * pb.img_bytes;
            const gz_cuboid &cb = pb.cb;
            for (int c = ttid; c < P; c += tstride) {
                const int yi = c / cb.g_extent, gi = c - yi * cb.g_extent, gg = cb.g_min + gi;
                const size_t row = (size_t)(cb.y_min + yi) * pb.img_w * pb.ch;
                constexpr int LPT = LP * R;
                for (int kk = 0; kk < LPT; ++kk) {
                    int acc = 0;
                    if (kk < cb.m) {   // geometry.py:325-335 site_columns, energy.py:96-113
                        const int d = cb.d_min + kk;
                        int xr = gg + d, xl = (cb.width - 1) + gg - d;
                        xr = xr < 0 ? 0 : (xr > cb.width - 1 ? cb.width - 1 : xr);
                        xl = xl < 0 ? 0 : (xl > cb.width - 1 ? cb.width - 1 : xl);
                        for (int q = 0; q < pb.ch; ++q)
                            acc += abs((int)lp[row + (size_t)xl * pb.ch + q] - (int)rp[row + (size_t)xr * pb.ch + q]);
                    }
                    a.vol[(size_t)c * LPT + kk] = acc;
                }
            }
        }
        __threadfence();
        (void)tm.sync_or(0u, phase, s_t3, s_u3);
        unsigned long long t0 = gz2::gtimer();
        Prob q = p;
        q.labels = pb.labels_out + (size_t)pair * P;
        tilesolve_body<LP, R, false, OCC, 0, Prob, Bits2, Arr3>(q, b, a, g, bar, cta, T, phase);
        __threadfence();
        (void)tm.sync_or(0u, phase, s_t3, s_u3);
        if (cta == 0 && threadIdx.x < CTR_COUNT) {
            unsigned long long v = ((volatile unsigned long long *)p.ctr)[threadIdx.x];
            if (threadIdx.x == CTR_NS) v = gz2::gtimer() - t0;
            if (threadIdx.x == CTR_TDRAW) v = s_tdraw;
            if (threadIdx.x == CTR_TEND) v = gz2::gtimer();
            pb.stats[(size_t)pair * CTR_COUNT + threadIdx.x] = v;
        }
    }
    // first launch with a tail launch behind it: the last of the team's CTAs to
    // finish releases the slice (no CTA of the team touches it afterwards)
    if (!pb.tail && pb.free_slices && threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&pb.done[team], 1u) == (unsigned)(T - 1)) {
            const unsigned k = atomicAdd(pb.free_n, 1u);
            *(volatile int *)&pb.free_slices[k] = team;
        }
    }
}

}  // namespace gz4
