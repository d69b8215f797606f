// gz_bitsolve.cuh -- v2 solver: bit-parallel chains.
//
// Every site's chain positions 1..m are packed into NW = ceil(m/32) 32-bit
// words (bit t-1 <-> position t; position m is always the sink).  Per sweep:
//
//   1. mask build      one pass: for every real node, which of its 13
//                      non-infinite arcs have residual > 0 (chain-up, and
//                      same-level / inhibit-down / reverse-diagonal-up to each
//                      of the 4 neighbours) -> 13 bit-words per column.
//   2. global relabel  level-synchronous BFS from the sink (maxflow.py:138-158)
//                      on the bit-words: one level of a whole column is ~30
//                      AND/OR/shift ops against the neighbours' frontier
//                      words.  Exact distances; it stops early once it has
//                      gone `bfs_min` levels deep and met an active node
//                      (unvisited nodes are parked at HINF, dormant), and it
//                      runs to exhaustion before the solver may conclude.
//   3. K pulses        push / relabel only on nodes flagged in per-column
//                      active-bit words; lateral pushes set inbox bits.
//
// Extraction (maxflow.py:267-320) is a prefix-closure on the same masks.
#pragma once

namespace gz2 {

using namespace gz;

__device__ __forceinline__ unsigned long long gtimer();

}  // namespace gz2

// device watchdog: true once the solve has run longer than p.watchdog_ns
__device__ __forceinline__ bool gz2_watchdog_expired(const gz::Prob &p) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return p.watchdog_ns && t - p.t_start_ns > p.watchdog_ns;
}

namespace gz2 {

struct Bits2 {
    uint32_t *mask;   // [13][NW][P] indexed like gz::Arc: 0 chain-up, 1..4 same-level R L D U,
                      // 5..8 diagonal-up (reverse inhibit) R L D U, 9..12 inhibit diagonal-down R L D U
    uint32_t *V, *F0, *F1, *A, *IN, *EX, *RL;   // [NW][P]
    int32_t *R0, *R1;                            // reach prefix length [P]
    int NW;
};

template <int NW>
struct BW {
    uint32_t w[NW];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = 0u;
    }
    __device__ __forceinline__ bool any() const {
        uint32_t a = 0;
#pragma unroll
        for (int i = 0; i < NW; ++i) a |= w[i];
        return a != 0u;
    }
    __device__ __forceinline__ void load(const uint32_t *base, int P, int c) {
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = base[(size_t)i * P + c];
    }
    __device__ __forceinline__ void store(uint32_t *base, int P, int c) const {
#pragma unroll
        for (int i = 0; i < NW; ++i) base[(size_t)i * P + c] = w[i];
    }
    // toward higher positions (bit b -> b+1)
    __device__ __forceinline__ BW shl1() const {
        BW r;
#pragma unroll
        for (int i = NW - 1; i >= 0; --i) r.w[i] = (w[i] << 1) | (i > 0 ? (w[i - 1] >> 31) : 0u);
        return r;
    }
    // toward lower positions (bit b -> b-1)
    __device__ __forceinline__ BW shr1() const {
        BW r;
#pragma unroll
        for (int i = 0; i < NW; ++i) r.w[i] = (w[i] >> 1) | (i + 1 < NW ? (w[i + 1] << 31) : 0u);
        return r;
    }
    __device__ __forceinline__ int top() const {   // highest set bit index or -1
#pragma unroll
        for (int i = NW - 1; i >= 0; --i)
            if (w[i]) return 32 * i + 31 - __clz(w[i]);
        return -1;
    }
    __device__ __forceinline__ bool test(int b) const { return (w[b >> 5] >> (b & 31)) & 1u; }
    __device__ __forceinline__ void set(int b) { w[b >> 5] |= 1u << (b & 31); }
    __device__ __forceinline__ void clr(int b) { w[b >> 5] &= ~(1u << (b & 31)); }
    // bits [lo, hi) set
    __device__ __forceinline__ static BW range(int lo, int hi) {
        BW r;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            int a = lo - 32 * i, b = hi - 32 * i;
            a = a < 0 ? 0 : (a > 32 ? 32 : a);
            b = b < 0 ? 0 : (b > 32 ? 32 : b);
            uint32_t mb = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
            uint32_t ma = a >= 32 ? 0xffffffffu : ((1u << a) - 1u);
            r.w[i] = mb & ~ma;
        }
        return r;
    }
};

template <int NW>
__device__ __forceinline__ BW<NW> operator&(BW<NW> a, const BW<NW> &b) {
#pragma unroll
    for (int i = 0; i < NW; ++i) a.w[i] &= b.w[i];
    return a;
}
template <int NW>
__device__ __forceinline__ BW<NW> operator|(BW<NW> a, const BW<NW> &b) {
#pragma unroll
    for (int i = 0; i < NW; ++i) a.w[i] |= b.w[i];
    return a;
}
template <int NW>
__device__ __forceinline__ BW<NW> andnot(BW<NW> a, const BW<NW> &b) {
#pragma unroll
    for (int i = 0; i < NW; ++i) a.w[i] &= ~b.w[i];
    return a;
}

// ---------------------------------------------------------------------------
// 1. mask build (+ excess bits); also resets the BFS state of the column.
template <bool WIN, int NW>
__device__ void bit_build(const Prob &p, const Bits2 &b, int c) {
    Col<WIN> k;
    k.load(p, c);
    const int P = p.P;
    BW<NW> M[13], ex;
#pragma unroll
    for (int q = 0; q < 13; ++q) M[q].zero();
    ex.zero();
    for (int t = k.lo + 1; t <= k.hi; ++t) {
        const int bit = t - 1;
        if (p.e[t * P + c] > 0) ex.set(bit);
#pragma unroll
        for (int j = 0; j < 13; ++j) {
            int v, kind;
            int r = arc_resid<WIN>(p, k, j, t, v, kind);
            if (kind != K_SRC && r > 0) M[j].set(bit);
        }
        p.h[t * P + c] = HINF;
    }
#pragma unroll
    for (int q = 0; q < 13; ++q) M[q].store(b.mask + (size_t)q * NW * P, P, c);
    ex.store(b.EX, P, c);
    BW<NW> z;
    z.zero();
    z.store(b.V, P, c);
    z.store(b.A, P, c);
    // level 0 frontier: the sink positions (t > hi)
    BW<NW>::range(k.hi, p.M).store(b.F0, P, c);
}

// 2. one BFS level: frontier `Fin` -> `Fout` (nodes at distance d+1).
// Returns (new nodes?, new nodes with excess?) packed in bits 0/1.
template <bool WIN, int NW>
__device__ int bit_bfs_level(const Prob &p, const Bits2 &b, int c, const uint32_t *Fin, uint32_t *Fout, int d) {
    const int P = p.P;
    BW<NW> F;
    F.load(Fin, P, c);
    const int y = c / p.G, g = c - y * p.G;
    const bool has[4] = {g + 1 < p.G, g > 0, y + 1 < p.Y, y > 0};
    const int nc[4] = {c + 1, c - 1, c + p.G, c - p.G};
    BW<NW> Fn[4];
    bool any = F.any();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (has[i]) { Fn[i].load(Fin, P, nc[i]); any |= Fn[i].any(); }
        else Fn[i].zero();
    }
    BW<NW> N;
    N.zero();
    if (any) {
        const uint32_t *m = b.mask;
        BW<NW> cu;
        cu.load(m, P, c);
        N = F.shl1() | (F.shr1() & cu);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!Fn[i].any()) continue;
            BW<NW> s, dd, uu;
            s.load(m + (size_t)(A_SR + i) * NW * P, P, c);
            dd.load(m + (size_t)(A_DR + i) * NW * P, P, c);
            uu.load(m + (size_t)(A_UR + i) * NW * P, P, c);
            N = N | (Fn[i] & s) | (Fn[i].shl1() & dd) | (Fn[i].shr1() & uu);
        }
        int lo = 0, hi = p.L;
        if (WIN) { lo = p.lo[c]; hi = p.hi[c]; }
        BW<NW> V;
        V.load(b.V, P, c);
        N = andnot(N & BW<NW>::range(lo, hi), V);
        if (N.any()) {
            (V | N).store(b.V, P, c);
#pragma unroll
            for (int i = 0; i < NW; ++i) {
                uint32_t x = N.w[i];
                while (x) {
                    int bb = __ffs(x) - 1;
                    x &= x - 1;
                    p.h[(32 * i + bb + 1) * P + c] = d + 1;
                }
            }
        }
    }
    N.store(Fout, P, c);
    int ret = N.any() ? 1 : 0;
    if (ret) {
        BW<NW> ex;
        ex.load(b.EX, P, c);
        if ((N & ex).any()) ret |= 2;
    }
    return ret;
}

// active bits = visited & excess; returns the count
template <int NW>
__device__ int bit_activate(const Prob &p, const Bits2 &b, int c) {
    BW<NW> V, ex;
    V.load(b.V, p.P, c);
    ex.load(b.EX, p.P, c);
    BW<NW> A = V & ex;
    A.store(b.A, p.P, c);
    int n = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) n += __popc(A.w[i]);
    return n;
}

// 3a. push pulse on the active nodes of column c (chain pushes Gauss-Seidel upward)
template <bool WIN, int NW>
__device__ void bit_push(const Prob &p, const Bits2 &b, int c, long long &flow, long long &pushes) {
    const int P = p.P;
    BW<NW> A;
    A.load(b.A, P, c);
    if (!A.any()) return;
    Col<WIN> k;
    k.load(p, c);
    BW<NW> newA;
    newA.zero();
#pragma unroll
    for (int wi = 0; wi < NW; ++wi) {
        uint32_t bits = A.w[wi];
        while (bits) {
            const int bb = __ffs(bits) - 1;
            bits &= bits - 1;
            const int t = 32 * wi + bb + 1;
            const int u = t * P + c;
            int ex = p.e[u];
            const int hu = p.h[u];
            if (ex <= 0 || hu >= HINF) continue;
#pragma unroll
            for (int j = 0; j < A_COUNT; ++j) {
                if (ex <= 0) break;
                int v, kind;
                int r = arc_resid<WIN>(p, k, j, t, v, kind);
                if (kind == K_SRC || r <= 0) continue;
                int hv = kind == K_SNK ? 0 : p.h[v];
                if (hu != hv + 1) continue;
                int d = imin(ex, r);
                arc_push<WIN>(p, k, j, t, d);
                ex -= d;
                ++pushes;
                if (kind == K_SNK) {
                    flow += d;
                } else if (j == A_UP) {
                    p.e[v] += d;   // next position of this chain: processed later in this pass
                    if (bb + 1 < 32) bits |= 1u << (bb + 1);
                    else if (wi + 1 < NW) A.w[wi + 1] |= 1u;
                } else if (j == A_DN) {
                    p.e[v] += d;
                    newA.set(t - 2);
                } else {
                    atomicAdd(&p.ein[v], d);
                    const int nb = v / P - 1;   // target position - 1
                    atomicOr(&b.IN[(size_t)(nb >> 5) * P + (v % P)], 1u << (nb & 31));
                }
            }
            p.e[u] = ex;
            if (ex > 0) newA.set(t - 1);
        }
    }
    newA.store(b.A, P, c);
}

// 3b. merge inboxes, relabel active nodes without an admissible arc.
// DET: heights go to h2 and are committed by bit_commit (snapshot semantics).
template <bool WIN, int NW, bool DET>
__device__ void bit_relabel(const Prob &p, const Bits2 &b, int c, long long &relabels) {
    const int P = p.P;
    BW<NW> A, IN;
    A.load(b.A, P, c);
    IN.load(b.IN, P, c);
    if (!A.any() && !IN.any()) return;
    if (IN.any()) {
#pragma unroll
        for (int wi = 0; wi < NW; ++wi) {
            uint32_t x = IN.w[wi];
            while (x) {
                const int bb = __ffs(x) - 1;
                x &= x - 1;
                const int u = (32 * wi + bb + 1) * P + c;
                const int add = p.ein[u];
                p.ein[u] = 0;
                const int ex = p.e[u] + add;
                p.e[u] = ex;
                if (ex > 0 && p.h[u] < HINF) A.w[wi] |= 1u << bb;
            }
        }
        BW<NW> z;
        z.zero();
        z.store(b.IN, P, c);
    }
    Col<WIN> k;
    k.load(p, c);
    BW<NW> RLm;
    RLm.zero();
#pragma unroll
    for (int wi = 0; wi < NW; ++wi) {
        uint32_t bits = A.w[wi];
        while (bits) {
            const int bb = __ffs(bits) - 1;
            bits &= bits - 1;
            const int t = 32 * wi + bb + 1;
            const int u = t * P + c;
            const int hu = p.h[u];
            int best = HINF;
            bool adm = false;
#pragma unroll
            for (int j = 0; j < A_COUNT; ++j) {
                int v, kind;
                int r = arc_resid<WIN>(p, k, j, t, v, kind);
                if (kind == K_SRC || r <= 0) continue;
                int hv = kind == K_SNK ? 0 : p.h[v];
                if (hu == hv + 1) { adm = true; break; }
                best = imin(best, hv + 1);
            }
            if (adm) continue;
            ++relabels;
            if (DET) { p.h2[u] = best; RLm.w[wi] |= 1u << bb; }
            else p.h[u] = best;
            if (best >= HINF) A.w[wi] &= ~(1u << bb);
        }
    }
    A.store(b.A, P, c);
    if (DET) RLm.store(b.RL, P, c);
}

template <int NW>
__device__ void bit_commit(const Prob &p, const Bits2 &b, int c) {
    const int P = p.P;
    BW<NW> RLm;
    RLm.load(b.RL, P, c);
    if (!RLm.any()) return;
#pragma unroll
    for (int wi = 0; wi < NW; ++wi) {
        uint32_t x = RLm.w[wi];
        while (x) {
            const int bb = __ffs(x) - 1;
            x &= x - 1;
            const int u = (32 * wi + bb + 1) * P + c;
            p.h[u] = p.h2[u];
        }
    }
    BW<NW> z;
    z.zero();
    z.store(b.RL, P, c);
}

// ---------------------------------------------------------------------------
// extraction on the final masks: reach prefix r (positions lo+1 .. lo+r).
template <bool WIN, int NW>
__device__ int bit_close_up(const Bits2 &b, int P, int c, int lo, int hi, int r) {
    if (r <= 0) return 0;
    BW<NW> cu;
    cu.load(b.mask, P, c);
    while (lo + r < hi && cu.test(lo + r - 1)) ++r;
    return r;
}

template <bool WIN, int NW>
__device__ void bit_reach_init(const Prob &p, const Bits2 &b, int c) {
    const int P = p.P;
    int lo = 0, hi = p.L;
    if (WIN) { lo = p.lo[c]; hi = p.hi[c]; }
    BW<NW> ex;
    ex.zero();
    for (int t = lo + 1; t <= hi; ++t)
        if (p.e[t * P + c] > 0) ex.set(t - 1);
    const int top = ex.top();
    const int r = top < 0 ? 0 : top + 1 - lo;
    b.R0[c] = bit_close_up<WIN, NW>(b, P, c, lo, hi, r);
}

template <bool WIN, int NW>
__device__ bool bit_reach_iter(const Prob &p, const Bits2 &b, int c, const int32_t *Rin, int32_t *Rout) {
    const int P = p.P;
    const int y = c / p.G, g = c - y * p.G;
    const bool has[4] = {g + 1 < p.G, g > 0, y + 1 < p.Y, y > 0};
    const int nc[4] = {c + 1, c - 1, c + p.G, c - p.G};
    int lo = 0, hi = p.L;
    if (WIN) { lo = p.lo[c]; hi = p.hi[c]; }
    const int r0 = Rin[c];
    int r = r0;
    BW<NW> T;
    T.zero();
    bool anyn = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (!has[i]) continue;
        const int rn = Rin[nc[i]];
        if (rn <= 0) continue;
        const int lon = WIN ? p.lo[nc[i]] : 0;
        BW<NW> Rn = BW<NW>::range(lon, lon + rn);
        const int j = i ^ 1;   // direction from the neighbour back to c
        BW<NW> s, dd, uu;
        s.load(b.mask + (size_t)(A_SR + j) * NW * P, P, nc[i]);
        dd.load(b.mask + (size_t)(A_DR + j) * NW * P, P, nc[i]);
        uu.load(b.mask + (size_t)(A_UR + j) * NW * P, P, nc[i]);
        T = T | (Rn & s) | (Rn & dd).shr1() | (Rn & uu).shl1();
        anyn = true;
    }
    if (anyn) {
        T = T & BW<NW>::range(lo, hi);
        const int top = T.top();
        if (top >= 0 && top + 1 - lo > r) r = bit_close_up<WIN, NW>(b, P, c, lo, hi, top + 1 - lo);
    }
    Rout[c] = r;
    return r != r0;
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Grid-wide OR of per-thread flag bits, one grid barrier: warp reduce ->
// shared atomic -> one global atomic per block; the result is read by one
// thread per block and broadcast through shared memory.  Both the global and
// the shared slot rotate over three entries: a slot is only reset two calls
// after its last reader passed a barrier (otherwise a fast thread 0 could
// clear the broadcast before a slow warp read it, splitting the grid's
// control flow across a grid barrier).
__device__ __forceinline__ unsigned grid_or(cg::grid_group &grid, unsigned flags, unsigned long long *slots, int &rot,
                                            unsigned *s_acc3) {
    unsigned *s_acc = s_acc3 + rot;
    if (threadIdx.x == 0) *s_acc = 0u;
    __syncthreads();
    const unsigned w = __reduce_or_sync(0xffffffffu, flags);
    if ((threadIdx.x & 31) == 0 && w) atomicOr(s_acc, w);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (*s_acc) atomicOr(&slots[rot], (unsigned long long)*s_acc);
        if (blockIdx.x == 0) slots[(rot + 1) % 3] = 0ull;
    }
    grid.sync();
    if (threadIdx.x == 0) *s_acc = (unsigned)((volatile unsigned long long *)slots)[rot];
    __syncthreads();
    const unsigned r = *s_acc;
    rot = (rot + 1) % 3;
    return r;
}

template <bool WIN, int NW, bool DET>
__global__ void __launch_bounds__(256) gz_bitsolve_kernel(Prob p, Bits2 b) {
    __shared__ unsigned s_acc[3];
    unsigned long long t_prev = 0, t_acc[6] = {0, 0, 0, 0, 0, 0};
    const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
    if (timer) t_prev = gtimer();
    if (timer) p.t_start_ns = t_prev;
#define TICK(slot) do { if (timer) { unsigned long long t_ = gtimer(); t_acc[slot] += t_ - t_prev; t_prev = t_; } } while (0)
    cg::grid_group grid = cg::this_grid();
    const int stride = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int niter = (p.P + stride - 1) / stride;
    long long flow = 0, offset = 0, presat = 0, pushes = 0, relabels = 0;
    volatile unsigned long long *vctr = p.ctr;
#define FOR_COLS for (int it_ = 0, c = tid; it_ < niter; ++it_, c += stride) if (c < p.P)

    FOR_COLS phase_init_a<WIN>(p, c);
    grid.sync();
    FOR_COLS phase_init_b<WIN>(p, c, flow, offset, presat);
    grid.sync();
    TICK(0);

    int sweeps = 0, levels_total = 0, pulses = 0, rot = 0;
    int converged = 1;
    const int bfs_min = p.bfs_cap > 0 ? p.bfs_cap : (1 << 30);
    for (;;) {
        FOR_COLS bit_build<WIN, NW>(p, b, c);
        grid.sync();
        TICK(1);
        // ---- BFS from the sink ----
        int d = 0;
        bool found = false, exhausted = false, err = false;
        uint32_t *Fin = b.F0, *Fout = b.F1;
        for (;;) {
            unsigned flags = 0;
            FOR_COLS flags |= (unsigned)bit_bfs_level<WIN, NW>(p, b, c, Fin, Fout, d);
            const unsigned g = grid_or(grid, flags, p.ctr + CTR_FLAG0, rot, s_acc);
            const bool nn = (g & 1u) != 0;
            found |= (g & 2u) != 0;
            uint32_t *tmp = Fin; Fin = Fout; Fout = tmp;
            ++d;
            if (!nn) { exhausted = true; break; }
            if (found && d >= bfs_min) break;
            if (d > 4 * (p.P + p.M)) { if (tid == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); err = true; break; }
        }
        levels_total += d;
        TICK(2);
        if (err) break;
        if (!found) {
            if (exhausted) break;   // no node with excess can reach the sink: maximum preflow
        }
        if (p.capped && sweeps >= p.max_sweeps) { converged = 0; break; }
        FOR_COLS bit_activate<NW>(p, b, c);
        grid.sync();
        for (int pulse = 0; pulse < p.K; ++pulse) {
            FOR_COLS bit_push<WIN, NW>(p, b, c, flow, pushes);
            grid.sync();
            FOR_COLS bit_relabel<WIN, NW, DET>(p, b, c, relabels);
            grid.sync();
            if (DET) {
                FOR_COLS bit_commit<NW>(p, b, c);
                grid.sync();
            }
            ++pulses;
        }
        TICK(3);
        ++sweeps;
        // watchdog: one thread decides, the decision is broadcast through the grid barrier
        {
            unsigned stop = 0;
            if (tid == 0 && gz2_watchdog_expired(p)) stop = 1;
            if (gz2::grid_or(grid, stop, p.ctr + CTR_FLAG0, rot, s_acc)) {
                if (tid == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE);
                break;
            }
        }
        if (sweeps > 1000000) { if (tid == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
    }

    // ---- extraction ----
    FOR_COLS bit_reach_init<WIN, NW>(p, b, c);
    grid.sync();
    int reach_passes = 0;
    int32_t *Rin = b.R0, *Rout = b.R1;
    for (;;) {
        unsigned ch = 0;
        FOR_COLS ch |= bit_reach_iter<WIN, NW>(p, b, c, Rin, Rout) ? 1u : 0u;
        const bool any = grid_or(grid, ch, p.ctr + CTR_FLAG0, rot, s_acc) != 0;
        int32_t *tmp = Rin; Rin = Rout; Rout = tmp;
        ++reach_passes;
        if (!any) break;
        if (reach_passes > 4 * (p.P + p.M)) { if (tid == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
    }
    TICK(4);
    long long stranded = 0;
    FOR_COLS {
        int lo = WIN ? p.lo[c] : 0, hi = WIN ? p.hi[c] : p.L;
        p.labels[c] = lo + Rin[c];
        for (int t = lo + 1; t <= hi; ++t) stranded += p.e[t * p.P + c] > 0;
    }
    grid.sync();
    long long energy = 0;
    int viol = 0;
    FOR_COLS phase_energy_col(p, c, energy, viol);
#undef FOR_COLS
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
    if (viol) p.ctr[CTR_HARDVIOL] = 1;
    if (tid == 0) {
        p.ctr[CTR_SWEEPS] = sweeps;
        p.ctr[CTR_BFS_PASSES] = levels_total;
        p.ctr[CTR_REACH_PASSES] = reach_passes;
        p.ctr[CTR_CONVERGED] = converged;
        p.ctr[CTR_PULSES] = pulses;
    }
}

}  // namespace gz2
