// gz_chain.cuh -- per-chain warp machinery of the v4 solver (gz_tilesolve.cuh).
//
// Node arrays are column-major, [site][LPT] with LPT = 16 (m <= 16) or 32*R
// (R = 1, 2, 4 segments of 32 chain positions), so a warp segment of LP lanes
// holds LP consecutive chain positions of one site and every per-node load is
// coalesced.  Lane j of segment s <-> chain position t = s*LP + j + 1.
//   vol[c][k]   data cost of label k              (k < m)
//   cu [c][t-1] residual of chain arc t -> t+1     (arc 0 from the source is
//               saturated at init and never stored)
//   ph/pv/dar/dbr/dad/dbd [c][t-1]  lateral pair state at level t (gz_graph.cuh)
//   e, h, ein0/ein1 [c][t-1]
// Bit arrays (masks, excess, active, inbox, BFS frontier/visited) hold one
// 32-bit word per (segment, site) at word index s*P + c; bit j <-> position
// s*32 + j + 1 (LP = 16: one word per site, bits 0..15).
//
// A pulse is ONE team-synchronised phase per chain segment:
//   merge last pulse's inbox -> upward chain wave (segmented min-plus scan:
//   x_{t+1} = min(cu_t, e_t + x_t) over admissible chain arcs, the exact
//   Gauss-Seidel result of pushing bottom-up) -> lateral and downward pushes
//   of the remaining excess on admissible arcs -> relabel of nodes that could
//   not push (in place).  A node pushes with its phase-start height and only
//   relabels if it made no push, so two nodes can never push along one arc
//   pair in opposite directions; lateral pushes land in the other inbox
//   buffer (no reader this pulse).  The chain arc between two segments is
//   treated like a lateral arc: the wave leaving the top of segment s and a
//   downward push out of the bottom of segment s+1 travel through the inbox.
#pragma once

namespace gz3 {

using namespace gz;
using gz2::BW;
using gz2::Bits2;

struct Arr3 {
    int32_t *vol, *cu, *ph, *pv, *dar, *dbr, *dad, *dbd, *e, *ein0, *ein1, *h;
    uint32_t *IN0, *IN1;   // inbox bits per (segment, site) word, double-buffered
};

constexpr unsigned FULL = 0xffffffffu;

template <int LP>
__device__ __forceinline__ int from_above(int v) { return __shfl_down_sync(FULL, v, 1, LP); }   // lane j+1
template <int LP>
__device__ __forceinline__ int from_below(int v) { return __shfl_up_sync(FULL, v, 1, LP); }     // lane j-1

// c / G for 0 <= c < P (< 2^26): float reciprocal estimate, corrected by one step
__device__ __forceinline__ int div_g(const Prob &p, int c) {
    int y = __float2int_rz((float)c * p.inv_g);
    if (y * p.G > c) --y;
    else if ((y + 1) * p.G <= c) ++y;
    return y;
}

// Per-lane context: node (t, c) plus neighbour sites.
// RW > 0: window-relative lanes.  Lane j of a 16-lane segment handles position
// lo + 1 + j of its site (windows of width <= 15), over the unchanged absolute
// memory layout (rows of 32 RW positions, RW absolute bit words per site).
template <int LP, int R, bool WIN, int RW = 0>
struct Lane {
    static constexpr int LPT = RW ? 32 * RW : LP * R;   // memory row length (positions)
    static constexpr int NWB = RW ? RW : R;             // bit words per site
    int c, s, j, t, lo, hi, y, g, I, wi;
    bool valid, real;
    int nc[4], nlo[4], nhi[4];
    bool has[4];
    // sites c_base .. c_base + nsites - 1 (nsites <= 32 / LP), segment seg
    __device__ __forceinline__ void init(const Prob &p, int c_base, int nsites, int seg = 0) {
        const int lane = threadIdx.x & 31;
        c = c_base + lane / LP;
        j = lane % LP;
        s = seg;
        t = s * LP + j + 1;
        valid = lane / LP < nsites && c < p.P;
        const int cc = valid ? c : 0;
        y = div_g(p, cc);
        g = cc - y * p.G;
        has[0] = valid && g + 1 < p.G; nc[0] = cc + 1;
        has[1] = valid && g > 0;       nc[1] = cc - 1;
        has[2] = valid && y + 1 < p.Y; nc[2] = cc + p.G;
        has[3] = valid && y > 0;       nc[3] = cc - p.G;
        if (WIN) {
            lo = valid ? p.lo[cc] : 0;
            hi = valid ? p.hi[cc] : 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) { nlo[i] = has[i] ? p.lo[nc[i]] : 0; nhi[i] = has[i] ? p.hi[nc[i]] : 0; }
        } else {
            lo = 0; hi = p.L;
#pragma unroll
            for (int i = 0; i < 4; ++i) { nlo[i] = 0; nhi[i] = p.L; }
        }
        if (RW) {
            t = lo + 1 + j;
            if (t > LPT) { valid = false; t = LPT; }   // beyond the row: never real, never loaded
        }
        real = valid && t > lo && t <= hi;
        I = (valid ? cc : 0) * LPT + t - 1;
        wi = s * p.P + cc;
    }
    __device__ __forceinline__ int kown(int tt) const { return tt <= lo ? K_SRC : (tt > hi ? K_SNK : K_REAL); }
    __device__ __forceinline__ int knb(int i, int tt) const { return tt <= nlo[i] ? K_SRC : (tt > nhi[i] ? K_SNK : K_REAL); }
    __device__ __forceinline__ int nidx(int i) const { return nc[i] * LPT + t - 1; }
    // segment boundary lanes whose t+1 / t-1 neighbour lives in another segment
    __device__ __forceinline__ bool top_edge() const { return !RW && R > 1 && j == LP - 1 && s + 1 < R && valid; }
    __device__ __forceinline__ bool bot_edge() const {
        return RW ? (j == 0 && t > 1 && valid) : (R > 1 && j == 0 && s > 0 && valid);
    }
    // bit word / bit of this lane's position in the site's absolute bit words
    __device__ __forceinline__ int bword(const Prob &p) const { return RW ? ((t - 1) >> 5) * p.P + c : wi; }
    __device__ __forceinline__ int bbit() const { return RW ? ((t - 1) & 31) : j; }
};

// a segment ballot (bit j = lane j) as the site's absolute bit words (RW mode:
// shifted by lo); returns word w of it
template <int RW>
__device__ __forceinline__ uint32_t abs_word(uint32_t rel, int lo, int w) {
    if (!RW) return rel;
    const unsigned long long a = (unsigned long long)rel << lo;
    return (uint32_t)(a >> (32 * w));
}

// global load of solver state; CG = bypass L1 (the asynchronous pulses: other
// SMs and this warp's own atomics update the state between two reads)
template <bool CG>
__device__ __forceinline__ int ldx(const int32_t *p) { return CG ? __ldcg(p) : *p; }

// value at position t+1 / t-1 of the same array: shuffle inside the segment,
// load across a segment boundary (every lane executes the shuffle)
template <bool CG = false, int LP, int R, bool WIN, int RW>
__device__ __forceinline__ int up_of(const Lane<LP, R, WIN, RW> &L, int v, const int32_t *arr, int idx, bool ok = true) {
    int r = from_above<LP>(v);
    if (ok && L.top_edge()) r = ldx<CG>(arr + idx + 1);
    return r;
}
template <bool CG = false, int LP, int R, bool WIN, int RW>
__device__ __forceinline__ int dn_of(const Lane<LP, R, WIN, RW> &L, int v, const int32_t *arr, int idx) {
    int r = from_below<LP>(v);
    if (L.bot_edge()) r = ldx<CG>(arr + idx - 1);
    return r;
}

// Worklist of the groups a pulse leaves active and every group it pushes into:
// shared memory in the single-CTA tail mode, global memory for the team's
// pulse worklists (gz_tilesolve.cuh).
// Team worklists are split by row band: band j's list lives at list + nw c0(j)
// (in its own band's memory) and its length at cnt[c0(j)].
struct BandRoute {
    int *list;
    unsigned *cnt;
    int ny, nbands, TY, G, Y, P, nw, lp16, sys;
    __device__ __forceinline__ int c0(int j) const { return min(ny * j / nbands * TY, Y) * G; }
    __device__ __forceinline__ int band_of(int grp) const {
        const int site = lp16 ? min(2 * grp + 1, P - 1) : grp % P;   // a pair goes where its upper site is
        const int ty = (site / G) / TY;
        return ((ty + 1) * nbands + ny - 1) / ny - 1;
    }
};

struct TailQ {
    int *q;
    unsigned *n;
    int cap;
    const BandRoute *rt = nullptr;   // team worklist: route to the target group's band
    // push-time dedupe (team worklists): a push whose inbox word was already
    // nonzero this pulse skips the list -- the first push into that word listed
    // the group (inbox words are zero at pulse start: the owner clears them when
    // it is processed, and every group with inbox bits is listed or scanned)
    int dedupe = 0;
    __device__ __forceinline__ void push(int grp) const {
        if (rt && rt->nbands == 1) {   // one band: list and length at the plane bases
            const unsigned k = atomicAdd(rt->cnt, 1u);
            if ((int)k < rt->nw * rt->P) rt->list[k] = grp;
            return;
        }
        if (rt) {
            const int j = rt->band_of(grp), c0 = rt->c0(j), c1 = rt->c0(j + 1);
            const unsigned k = rt->sys ? atomicAdd_system(rt->cnt + c0, 1u) : atomicAdd(rt->cnt + c0, 1u);
            if ((int)k < rt->nw * (c1 - c0)) rt->list[(size_t)rt->nw * c0 + k] = grp;
            return;
        }
        const unsigned k = atomicAdd(n, 1u);
        if ((int)k < cap) q[k] = grp;
    }
    // Warp-aggregated append (one band or the shared-memory tail list): every
    // lane of the warp calls it with its number of entries; ONE atomic per warp
    // reserves them all.  Returns this lane's first slot.
    __device__ __forceinline__ bool aggregated() const { return !rt || rt->nbands == 1; }
    __device__ __forceinline__ int reserve_warp(int cnt) const {
        const int lane = threadIdx.x & 31;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        unsigned base = 0u;
        if (lane == 0 && total) base = atomicAdd(rt ? rt->cnt : n, (unsigned)total);
        base = __shfl_sync(0xffffffffu, base, 0);
        return (int)base + incl - cnt;
    }
    __device__ __forceinline__ void store(int k, int grp) const {
        if (rt) {
            if (k < rt->nw * rt->P) rt->list[k] = grp;
        } else if (k < cap) {
            q[k] = grp;
        }
    }
};

// Residuals of the 14 arcs of a lane's node, target heights and kinds.
// All shuffles are executed by every lane (uniform control flow).
template <int LP, int R, bool WIN, bool CG = false, int RW = 0>
struct Arcs {
    // (the 14 residuals are not kept: `pos` has their signs, and an arc's residual
    // is recomputed from the raw words when it is pushed along -- fewer live
    // registers through the pulse, whose 64-register batched instance spills)
    unsigned pos;   // bit j: arc j has residual > 0
    unsigned snk;   // bit j: arc j leads into the sink (arcs into the source have r = 0)
    unsigned adm;   // bit j: arc j admissible (residual > 0 and h(u) = h(target) + 1)
    int best;       // relabel height: 1 + the lowest target height over residual arcs (HINF if none)
    // raw words (for write-back)
    int w_cu, w_ph, w_pv, w_dar, w_dbr, w_dad, w_dbd;   // own-stored at I
    int w_phL, w_pvU, w_darL, w_dbrL, w_dadU, w_dbdU;   // neighbour-stored at the same position
    int w_dbr_up, w_darL_up, w_dbd_up, w_dadU_up;       // same arrays at position t+1
    int h_u;

    // target heights are folded into adm / best as soon as they are known (fewer
    // live registers in w_pulse)
    __device__ __forceinline__ void finish(const int (&r)[A_COUNT], const int (&hv)[A_COUNT]) {
        adm = 0u;
        pos = 0u;
        best = HINF;
#pragma unroll
        for (int jj = 0; jj < A_COUNT; ++jj)
            if (r[jj] > 0) {
                pos |= 1u << jj;
                const int c = hv[jj] + 1;
                best = min(best, c);
                if (h_u == c) adm |= 1u << jj;
            }
    }

    // residual of arc jj, valid when its `pos` bit is set (the conditions that zero
    // an arc -- missing neighbour, source-side target -- clear that bit)
    __device__ __forceinline__ int res(const Prob &p, int jj) const {
        const int P2 = 2 * p.pen, cap = p.hard ? p.hcap : p.inh;
        switch (jj) {
        case A_UP: return w_cu;
        case A_DN: return HINF;
        case A_SR: return w_ph;
        case A_SL: return P2 - w_phL;
        case A_SD: return w_pv;
        case A_SU: return P2 - w_pvU;
        case A_UR: return w_dbr_up;
        case A_UL: return w_darL_up;
        case A_UD: return w_dbd_up;
        case A_UU: return w_dadU_up;
        case A_DR: return cap - w_dar;
        case A_DL: return cap - w_dbrL;
        case A_DD: return cap - w_dad;
        default: return cap - w_dbdU;   // A_DU
        }
    }

    __device__ __forceinline__ void load(const Prob &p, const Arr3 &a, const Lane<LP, R, WIN, RW> &L) {
        int hv[A_COUNT], r[A_COUNT];
        const int I = L.I;
        const bool v = L.valid;
        w_cu = v ? ldx<CG>(a.cu + I) : 0;
        w_ph = v ? ldx<CG>(a.ph + I) : 0;
        w_pv = v ? ldx<CG>(a.pv + I) : 0;
        w_dar = v ? ldx<CG>(a.dar + I) : 0;
        w_dbr = v ? ldx<CG>(a.dbr + I) : 0;
        w_dad = v ? ldx<CG>(a.dad + I) : 0;
        w_dbd = v ? ldx<CG>(a.dbd + I) : 0;
        const int iL = L.nidx(1), iU = L.nidx(3);
        w_phL = L.has[1] ? ldx<CG>(a.ph + iL) : 0;
        w_darL = L.has[1] ? ldx<CG>(a.dar + iL) : 0;
        w_dbrL = L.has[1] ? ldx<CG>(a.dbr + iL) : 0;
        w_pvU = L.has[3] ? ldx<CG>(a.pv + iU) : 0;
        w_dadU = L.has[3] ? ldx<CG>(a.dad + iU) : 0;
        w_dbdU = L.has[3] ? ldx<CG>(a.dbd + iU) : 0;
        int hn[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) hn[i] = L.has[i] ? ldx<CG>(a.h + L.nidx(i)) : HINF;
        h_u = v ? ldx<CG>(a.h + I) : HINF;
        // position t+1 / t-1 values
        w_dbr_up = up_of<CG>(L, w_dbr, a.dbr, I);
        w_darL_up = up_of<CG>(L, w_darL, a.dar, iL, L.has[1]);
        w_dbd_up = up_of<CG>(L, w_dbd, a.dbd, I);
        w_dadU_up = up_of<CG>(L, w_dadU, a.dad, iU, L.has[3]);
        const int h_above = up_of<CG>(L, h_u, a.h, I), h_below = dn_of<CG>(L, h_u, a.h, I);
        int hn_above[4], hn_below[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int ni = L.has[i] ? L.nidx(i) : 0;
            hn_above[i] = from_above<LP>(hn[i]);
            hn_below[i] = from_below<LP>(hn[i]);
            if (L.top_edge() && L.has[i]) hn_above[i] = ldx<CG>(a.h + ni + 1);
            if (L.bot_edge() && L.has[i]) hn_below[i] = ldx<CG>(a.h + ni - 1);
        }

        const int t = L.t, P2 = 2 * p.pen, cap = p.hard ? p.hcap : p.inh;
        const bool top_ok = t < p.L;   // a position t+1 <= L exists (diagonals up)
        if (!WIN) {
            // full windows: for a real node (1 <= t <= L) the only terminal targets are
            // the sink above t = L (chain up) and the source below t = 1 (chain down and
            // inhibit diagonals down); every lateral target is a real node
            const bool bot = t == 1, top = t == p.L;
            snk = top ? 1u << A_UP : 0u;
            r[A_UP] = w_cu; hv[A_UP] = top ? 0 : h_above;
            r[A_DN] = bot ? 0 : HINF; hv[A_DN] = h_below;
            r[A_SR] = L.has[0] ? w_ph : 0; hv[A_SR] = hn[0];
            r[A_SL] = L.has[1] ? P2 - w_phL : 0; hv[A_SL] = hn[1];
            r[A_SD] = L.has[2] ? w_pv : 0; hv[A_SD] = hn[2];
            r[A_SU] = L.has[3] ? P2 - w_pvU : 0; hv[A_SU] = hn[3];
            r[A_UR] = (L.has[0] && top_ok) ? w_dbr_up : 0; hv[A_UR] = hn_above[0];
            r[A_UL] = (L.has[1] && top_ok) ? w_darL_up : 0; hv[A_UL] = hn_above[1];
            r[A_UD] = (L.has[2] && top_ok) ? w_dbd_up : 0; hv[A_UD] = hn_above[2];
            r[A_UU] = (L.has[3] && top_ok) ? w_dadU_up : 0; hv[A_UU] = hn_above[3];
            r[A_DR] = (L.has[0] && !bot) ? cap - w_dar : 0; hv[A_DR] = hn_below[0];
            r[A_DL] = (L.has[1] && !bot) ? cap - w_dbrL : 0; hv[A_DL] = hn_below[1];
            r[A_DD] = (L.has[2] && !bot) ? cap - w_dad : 0; hv[A_DD] = hn_below[2];
            r[A_DU] = (L.has[3] && !bot) ? cap - w_dbdU : 0; hv[A_DU] = hn_below[3];
            finish(r, hv);
            return;
        }
        snk = 0u;
#define SETA(J, RR, KIND, HV) do { const int k_ = (KIND); if (k_ == K_SNK) snk |= 1u << (J); r[J] = k_ == K_SRC ? 0 : (RR); hv[J] = k_ == K_SNK ? 0 : (HV); } while (0)
        SETA(A_UP, w_cu, L.kown(t + 1), h_above);
        SETA(A_DN, HINF, L.kown(t - 1), h_below);
        SETA(A_SR, L.has[0] ? w_ph : 0, L.has[0] ? L.knb(0, t) : K_SRC, hn[0]);
        SETA(A_SL, L.has[1] ? P2 - w_phL : 0, L.has[1] ? L.knb(1, t) : K_SRC, hn[1]);
        SETA(A_SD, L.has[2] ? w_pv : 0, L.has[2] ? L.knb(2, t) : K_SRC, hn[2]);
        SETA(A_SU, L.has[3] ? P2 - w_pvU : 0, L.has[3] ? L.knb(3, t) : K_SRC, hn[3]);
        SETA(A_UR, (L.has[0] && top_ok) ? w_dbr_up : 0, (L.has[0] && top_ok) ? L.knb(0, t + 1) : K_SRC, hn_above[0]);
        SETA(A_UL, (L.has[1] && top_ok) ? w_darL_up : 0, (L.has[1] && top_ok) ? L.knb(1, t + 1) : K_SRC, hn_above[1]);
        SETA(A_UD, (L.has[2] && top_ok) ? w_dbd_up : 0, (L.has[2] && top_ok) ? L.knb(2, t + 1) : K_SRC, hn_above[2]);
        SETA(A_UU, (L.has[3] && top_ok) ? w_dadU_up : 0, (L.has[3] && top_ok) ? L.knb(3, t + 1) : K_SRC, hn_above[3]);
        SETA(A_DR, L.has[0] ? cap - w_dar : 0, L.has[0] ? L.knb(0, t - 1) : K_SRC, hn_below[0]);
        SETA(A_DL, L.has[1] ? cap - w_dbrL : 0, L.has[1] ? L.knb(1, t - 1) : K_SRC, hn_below[1]);
        SETA(A_DD, L.has[2] ? cap - w_dad : 0, L.has[2] ? L.knb(2, t - 1) : K_SRC, hn_below[2]);
        SETA(A_DU, L.has[3] ? cap - w_dbdU : 0, L.has[3] ? L.knb(3, t - 1) : K_SRC, hn_below[3]);
#undef SETA
        finish(r, hv);
    }
};

// site and position of a lateral arc's target
template <int LP, int R, bool WIN, int RW>
__device__ __forceinline__ void lateral_target(const Lane<LP, R, WIN, RW> &L, int jarc, int &site, int &pos) {
    const int i = (jarc - A_SR) & 3;
    site = L.nc[i];
    pos = jarc <= A_SU ? L.t : (jarc <= A_UU ? L.t + 1 : L.t - 1);
}

// inclusive scan of f_j(x) = min(A_j, B_j + x) over the segment; returns F_j(x0)
template <int LP>
__device__ __forceinline__ int chain_wave(int A, int B, int j, int x0 = 0) {
#pragma unroll
    for (int o = 1; o < LP; o <<= 1) {
        const int A2 = __shfl_up_sync(FULL, A, o, LP), B2 = __shfl_up_sync(FULL, B, o, LP);
        if (j >= o) {   // compose: f_this o f_below
            A = min(A, B + A2);
            B = B + B2;
        }
    }
    return min(A, B + x0);
}

template <int LP>
__device__ __forceinline__ uint32_t seg_ballot(bool pred) {
    const uint32_t b = __ballot_sync(FULL, pred);
    if (LP == 32) return b;
    return (b >> ((threadIdx.x & 31) & ~(LP - 1))) & (LP >= 32 ? 0xffffffffu : ((1u << (LP & 31)) - 1u));
}

// ---------------------------------------------------------------------------
// init of one warp group (LP = 16: two sites; LP = 32: one site, all R
// segments in order): residuals from the volume, source saturation, greedy
// upward chain wave (carried across segments), constant offset.
template <int LP, int R, bool WIN, int RW = 0>
__device__ void w_init(const Prob &p, const Arr3 &a, int c_base, int nsites, long long &flow, long long &offset,
                       long long &presat) {
    int carry = 0;   // wave flow entering the bottom of the next segment
#pragma unroll 1
    for (int s = 0; s < R; ++s) {
        Lane<LP, R, WIN, RW> L;
        L.init(p, c_base, nsites, s);
        const int I = L.I;
        if (RW) {
            // window-relative lanes cover only the window: initialise the whole row
            // and fold the terminal arcs of every position into the offset here
            constexpr int LPT = Lane<LP, R, WIN, RW>::LPT;
            const int lane = threadIdx.x & 31, cs = c_base + lane / LP;
            if (lane / LP < nsites && cs < p.P) {
                for (int k = L.j; k < LPT; k += LP) {
                    const int idx = cs * LPT + k;
                    a.cu[idx] = (k + 1 < p.M) ? a.vol[idx + 1] : 0;
                    a.ph[idx] = p.pen; a.pv[idx] = p.pen;
                    a.dar[idx] = 0; a.dbr[idx] = 0; a.dad[idx] = 0; a.dbd[idx] = 0;
                    a.ein0[idx] = 0; a.ein1[idx] = 0;
                    a.h[idx] = HINF;
                    a.e[idx] = 0;
                }
                const long long icap_off = p.hard ? UNCUTTABLE : (long long)p.inh;
                if (L.j == 0 && L.lo == L.hi) offset += a.vol[cs * LPT + L.lo];
                for (int t = L.j + 1; t <= p.L; t += LP)
                    for (int i = 0; i < 4; i += 2) {   // forward neighbours right (0), down (2)
                        if (!L.has[i]) continue;
                        const int ka = L.kown(t), kb = L.knb(i, t);
                        if ((ka == K_SRC && kb == K_SNK) || (ka == K_SNK && kb == K_SRC)) offset += p.pen;
                        if (L.kown(t) == K_SRC && L.knb(i, t - 1) == K_SNK) offset += icap_off;
                        if (L.knb(i, t) == K_SRC && L.kown(t - 1) == K_SNK) offset += icap_off;
                    }
            }
            __syncwarp();
        }
        const int volj = (L.valid && L.t - 1 < p.M) ? a.vol[I] : 0;
        const int vol_above = up_of(L, volj, a.vol, I);
        if (!RW && L.valid) {
            a.cu[I] = (L.t < p.M) ? vol_above : 0;
            a.ph[I] = p.pen; a.pv[I] = p.pen;
            a.dar[I] = 0; a.dbr[I] = 0; a.dad[I] = 0; a.dbd[I] = 0;
            a.ein0[I] = 0; a.ein1[I] = 0;
            a.h[I] = HINF;
        }
        long long e = 0;
        // chain arc lo: source -> position lo+1 carries vol[lo]
        const int vol_lo_src = L.valid ? a.vol[L.c * Lane<LP, R, WIN, RW>::LPT + L.lo] : 0;
        if (L.real && L.t == L.lo + 1) e += vol_lo_src;
        if (WIN && L.valid) {
            const long long icap_off = p.hard ? UNCUTTABLE : (long long)p.inh;
            const int icap = p.hard ? p.hcap : p.inh;
            if (!RW && L.t == 1 && L.lo == L.hi) offset += vol_lo_src;
            if (!RW && L.t <= p.L) {
                const int t = L.t;
                for (int i = 0; i < 4; i += 2) {   // forward neighbours right (0), down (2)
                    if (!L.has[i]) continue;
                    const int ka = L.kown(t), kb = L.knb(i, t);
                    if ((ka == K_SRC && kb == K_SNK) || (ka == K_SNK && kb == K_SRC)) offset += p.pen;
                    if (L.kown(t) == K_SRC && L.knb(i, t - 1) == K_SNK) offset += icap_off;
                    if (L.knb(i, t) == K_SRC && L.kown(t - 1) == K_SNK) offset += icap_off;
                }
            }
            if (L.real) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (!L.has[i]) continue;
                    if (L.knb(i, L.t) == K_SRC) e += p.pen;
                    if (L.t + 1 <= p.L && L.knb(i, L.t + 1) == K_SRC) e += icap;
                }
            }
        }
        // greedy upward wave (no heights yet): every chain arc out of a real node is usable
        int ex = (int)e;
        if (!p.no_wave) {
            const bool up_ok = L.real;
            const int cuw = (L.valid && L.t < p.M) ? vol_above : 0;
            const int cin = (L.j == 0 && L.real) ? carry : 0;   // carry enters at the segment's first lane
            const int x_out = chain_wave<LP>(up_ok ? cuw : 0, up_ok ? ex + cin : 0, L.j);
            const int x_below = from_below<LP>(x_out);
            const int x_in = L.j > 0 ? x_below : cin;
            if (L.real) {
                ex = ex + x_in - x_out;
                a.cu[I] = cuw - x_out;
                if (L.kown(L.t + 1) == K_SNK) { flow += x_out; presat += x_out; }
            }
            carry = __shfl_sync(FULL, (L.real && L.kown(L.t + 1) == K_REAL) ? x_out : 0, LP - 1, LP);
        }
        if (L.valid) a.e[I] = L.real ? ex : 0;
    }
}

// ---------------------------------------------------------------------------
// mask build of one (segment, site) group: pending inbox merge, 13 arc-mask
// words, excess word, BFS reset words.
template <int LP, int R, bool WIN, int RW = 0>
__device__ void w_build(const Prob &p, const Arr3 &a, const Bits2 &b, int c_base, int nsites, int seg) {
    Lane<LP, R, WIN, RW> L;
    L.init(p, c_base, nsites, seg);
    const int I = L.I, P = p.P;
    // every global load of the group is issued before the first store (one
    // round trip): inbox words and values, excess, then the arc state
    const uint32_t in0 = L.valid ? a.IN0[L.wi] : 0u, in1 = L.valid ? a.IN1[L.wi] : 0u;
    int e = L.valid ? a.e[I] : 0;
    const int x0 = L.valid ? a.ein0[I] : 0, x1 = L.valid ? a.ein1[I] : 0;
    Arcs<LP, R, WIN, false, RW> A;
    A.load(p, a, L);
    // merge both inbox buffers (pushes since the last merge).  Values are merged
    // whether or not their inbox bit is set: an asynchronous pulse can consume a
    // bit before the value it announces lands (gz_tilesolve.cuh, async pulses),
    // and the pusher always marks this site dirty, so it is merged here.
    (void)in0; (void)in1;
    if (x0) { e += x0; a.ein0[I] = 0; }
    if (x1) { e += x1; a.ein1[I] = 0; }
    if (L.valid && (x0 | x1)) a.e[I] = e;
    uint32_t m[13];
#pragma unroll
    for (int q = 0; q < 13; ++q) m[q] = seg_ballot<LP>(L.real && ((A.pos >> q) & 1u));
    const uint32_t ex = seg_ballot<LP>(L.real && e > 0);
    if (RW && L.valid && L.j == 0) {
        // window-relative ballots -> the site's absolute words
#pragma unroll
        for (int w = 0; w < RW; ++w) {
            const int wi = w * P + L.c;
#pragma unroll
            for (int q = 0; q < 13; ++q) b.mask[((size_t)q * RW + w) * P + L.c] = abs_word<RW>(m[q], L.lo, w);
            b.EX[wi] = abs_word<RW>(ex, L.lo, w);
            b.V[wi] = 0u;
            b.A[wi] = 0u;
            a.IN0[wi] = 0u;
            a.IN1[wi] = 0u;
            b.F0[wi] = BW<RW ? RW : 1>::range(L.hi, p.M).w[w];
        }
    } else if (!RW && L.valid && L.j == 0) {
#pragma unroll
        if (LP == 16 && R == 1) {   // packed 16-bit masks (gz_bits.cuh mask_word)
#pragma unroll
            for (int q = 0; q < 13; q += 2) b.mask[(size_t)(q >> 1) * P + L.c] = m[q] | (q + 1 < 13 ? m[q + 1] << 16 : 0u);
        } else {
#pragma unroll
            for (int q = 0; q < 13; ++q) b.mask[((size_t)q * R + L.s) * P + L.c] = m[q];
        }
        b.EX[L.wi] = ex;
        b.V[L.wi] = 0u;
        b.A[L.wi] = 0u;
        a.IN0[L.wi] = 0u;
        a.IN1[L.wi] = 0u;
        b.F0[L.wi] = BW<R>::range(L.hi, p.M).w[L.s];
    }
}

// ---------------------------------------------------------------------------
// one pulse on a warp group of chains
template <int LP, int R, bool WIN, bool ASYNC = false, bool DETPUSH = false, int RW = 0>
__device__ void w_pulse(const Prob &p, const Arr3 &a, const Bits2 &b, int c_base, int nsites, int seg, int parity,
                        long long &flow, unsigned &pushes, unsigned &relabels, uint32_t *dirty,
                        const TailQ *tq = nullptr) {
    Lane<LP, R, WIN, RW> L;
    L.init(p, c_base, nsites, seg);
    const int I = L.I, P = p.P;
    constexpr int LPT = Lane<LP, R, WIN, RW>::LPT;
    // worklist fields read once (the queue lives in local / shared memory and the
    // list stores below could alias it, so the compiler would reload them per use)
    const bool dedupe = tq && tq->dedupe;
    // synchronous pulses double-buffer the inbox by parity; asynchronous ones use
    // one buffer consumed atomically
    uint32_t *IN_prev = (ASYNC || parity) ? a.IN0 : a.IN1;
    uint32_t *IN_cur = (ASYNC || DETPUSH || !parity) ? a.IN0 : a.IN1;
    int32_t *ein_prev = (ASYNC || parity) ? a.ein0 : a.ein1;
    int32_t *ein_cur = (ASYNC || DETPUSH || !parity) ? a.ein0 : a.ein1;
    constexpr int NWB = Lane<LP, R, WIN, RW>::NWB;
    int e, xin;
    Arcs<LP, R, WIN, ASYNC, RW> A;
    if (DETPUSH) {
        // deterministic push phase: inboxes are merged by the commit phase
        e = L.valid ? a.e[I] : 0;
        xin = 0;
        A.load(p, a, L);
    } else if (ASYNC) {
        uint32_t inb = 0u;
        if (L.valid && L.j == 0) {
            if (RW) for (int w = 0; w < NWB; ++w) inb |= atomicExch(&IN_prev[w * P + L.c], 0u);
            else inb = atomicExch(&IN_prev[L.wi], 0u);
        }
        e = L.valid ? __ldcg(a.e + I) : 0;
        xin = L.valid ? atomicExch(&ein_prev[I], 0) : 0;
        A.load(p, a, L);
        (void)__shfl_sync(FULL, inb, (threadIdx.x & 31) & ~(LP - 1));
        e += xin;
    } else {
        // all loads before the first store: one round trip per group (ein_prev has
        // no writer during this pulse, so reading it unconditionally is safe)
        const uint32_t inw = L.valid ? IN_prev[L.bword(p)] : 0u;
        e = L.valid ? a.e[I] : 0;
        xin = L.valid ? ein_prev[I] : 0;
        A.load(p, a, L);
        if ((inw >> L.bbit()) & 1u) { e += xin; ein_prev[I] = 0; }
        if (RW) {
            if (L.valid && L.j == 0)
                for (int w = 0; w < NWB; ++w) IN_prev[w * P + L.c] = 0u;
        } else if (L.valid && L.j == 0 && inw) {
            IN_prev[L.wi] = 0u;
        }
    }
    const int hu = A.h_u;
    const bool live = L.real && hu < HINF;
    // upward chain wave through admissible chain arcs
    const bool adm_up = live && ((A.adm >> A_UP) & 1u);
    const int x_out = chain_wave<LP>(adm_up ? A.w_cu : 0, adm_up ? max(e, 0) : 0, L.j);
    const int x_below = from_below<LP>(x_out);   // every lane shuffles (full mask)
    const int x_in = L.j > 0 ? x_below : 0;
    int cu_new = A.w_cu;
    bool pushed = false;
    if (L.real) {
        e += x_in - x_out;
        if (x_out > 0) {
            cu_new -= x_out;
            pushed = true;
            ++pushes;
            if ((A.snk >> A_UP) & 1u) {
                flow += x_out;
            } else if (L.top_edge()) {   // into the next segment's first node
                gz_atomic_add(p, &ein_cur[I + 1], x_out);
                const uint32_t o_ = gz_atomic_or(p, &IN_cur[L.wi + P], 1u);
                if (tq && !(o_ && tq->dedupe)) tq->push(L.wi + P);
            }
        }
    }
    // Lateral and downward pushes of the remaining excess along admissible arcs,
    // in arc order.  Each push updates its arc pair's state at once (only this
    // node pushes along that pair this pulse) and lands in the target's inbox;
    // every inbox add and inbox-bit OR is issued before any result is used (one
    // memory round trip for all of them), and the target groups that go on the
    // worklist are appended after the write-back with one warp-aggregated atomic
    // (TailQ::reserve_warp).  Asynchronous pulses apply pair-state deltas
    // atomically (concurrent opposite pushes stay within capacity because each is
    // bounded by its own stale-low read).
    uint32_t lmask = 0u;   // bit jj: lateral push along arc jj into a real node
    uint32_t dup = 0u;     // bit jj: its inbox word was already set this pulse
    int dn = 0;            // chain-down push
    {
        int rem = (live && e > 0) ? e : 0;
        const int iL = L.nidx(1), iU = L.nidx(3);
#define GZ_PAIR(arr, idx, word, delta) do { if (ASYNC) atomicAdd(&a.arr[idx], (delta)); else a.arr[idx] = (word) + (delta); } while (0)
#pragma unroll
        for (int jj = A_SR; jj <= A_DN; ++jj) {
            const int d = ((A.adm >> jj) & 1u) ? min(rem, A.res(p, jj)) : 0;
            rem -= d;
            if (d <= 0) continue;
            pushed = true;
            ++pushes;
            switch (jj) {
            case A_SR: GZ_PAIR(ph, I, A.w_ph, -d); break;
            case A_SD: GZ_PAIR(pv, I, A.w_pv, -d); break;
            case A_DR: GZ_PAIR(dar, I, A.w_dar, d); break;
            case A_DD: GZ_PAIR(dad, I, A.w_dad, d); break;
            case A_SL: GZ_PAIR(ph, iL, A.w_phL, d); break;
            case A_DL: GZ_PAIR(dbr, iL, A.w_dbrL, d); break;
            case A_SU: GZ_PAIR(pv, iU, A.w_pvU, d); break;
            case A_DU: GZ_PAIR(dbd, iU, A.w_dbdU, d); break;
            case A_UR: GZ_PAIR(dbr, I + 1, A.w_dbr_up, -d); break;
            case A_UD: GZ_PAIR(dbd, I + 1, A.w_dbd_up, -d); break;
            case A_UL: GZ_PAIR(dar, iL + 1, A.w_darL_up, -d); break;
            case A_UU: GZ_PAIR(dad, iU + 1, A.w_dadU_up, -d); break;
            default: break;
            }
            if (jj == A_DN) { dn = d; continue; }
            if ((A.snk >> jj) & 1u) { flow += d; continue; }
            int site, pos;
            lateral_target(L, jj, site, pos);
            gz_atomic_add(p, &ein_cur[site * LPT + pos - 1], d);
            uint32_t *inw = &IN_cur[((pos - 1) >> 5) * P + site];
            const uint32_t bit = 1u << ((pos - 1) & 31);
            if (dedupe) dup |= (gz_atomic_or(p, inw, bit) != 0u ? 1u : 0u) << jj;
            else gz_atomic_or(p, inw, bit);   // (result unused: a fire-and-forget reduction)
            lmask |= 1u << jj;
        }
#undef GZ_PAIR
        if (live && e > 0) e = rem;
    }
    // chain-down pushes arrive at lane j-1 (adds to its excess and to its chain-up
    // residual); out of a segment's first lane they cross into the segment below
    const int dn_recv = from_above<LP>(dn);
    const int dn_in = (L.real && L.j + 1 < LP) ? dn_recv : 0;
    if (L.real) {
        e += dn_in;
        cu_new += dn_in;
    }
    if (!RW && dn > 0 && L.bot_edge()) {
        gz_atomic_add(p, &a.cu[I - 1], dn);   // (the segment below applies its own cu change atomically too)
        gz_atomic_add(p, &ein_cur[I - 1], dn);
        const uint32_t o_ = gz_atomic_or(p, &IN_cur[L.wi - P], 1u << (LP - 1));
        if (tq && !(o_ && tq->dedupe)) tq->push(L.wi - P);
    }
    // relabel a live node that could not push (deterministic mode: a later phase)
    int hnew = hu;
    if (!DETPUSH && live && !pushed && e > 0) {
        hnew = A.best;
        ++relabels;
    }
    // write back the node's own excess, chain residual and height
    if (L.real) {
        a.e[I] = e;
        if (cu_new != A.w_cu) {
            if (ASYNC) atomicAdd(&a.cu[I], cu_new - A.w_cu);   // (a segment above can change it too)
            else a.cu[I] = cu_new;
        }
        if (hnew != hu) a.h[I] = hnew;
    }
    const uint32_t newA = seg_ballot<LP>(L.real && e > 0 && hnew < HINF && (!DETPUSH || pushed));
    uint32_t rl = 0u;
    if (DETPUSH) rl = seg_ballot<LP>(live && !pushed && e > 0);   // relabel candidates for the relabel phase
    if (L.valid && L.j == 0) {
        if (RW) {
            for (int w = 0; w < NWB; ++w) {
                b.A[w * P + L.c] = abs_word<RW>(newA, L.lo, w);
                if (DETPUSH) b.RL[w * P + L.c] = abs_word<RW>(rl, L.lo, w);
            }
        } else {
            b.A[L.wi] = newA;
            if (DETPUSH) b.RL[L.wi] = rl;
        }
    }
    if (tq) {
        // worklist: the groups pushed into (a push into an inbox word already set
        // this pulse is skipped with dedupe: that word's first push listed the
        // group) and this group if it stays active
        uint32_t want = 0u;
#pragma unroll
        for (int jj = A_SR; jj < A_DN; ++jj)
            if (((lmask >> jj) & 1u) && !(((dup >> jj) & 1u) && dedupe)) want |= 1u << jj;
        const bool self = __any_sync(FULL, newA != 0u) && (threadIdx.x & 31) == 0;
        auto gid = [&](int jj) {
            int site, pos;
            lateral_target(L, jj, site, pos);
            return LP == 16 ? site >> 1 : ((pos - 1) / LP) * P + site;
        };
        if (tq->aggregated()) {
            int *const lst = tq->rt ? tq->rt->list : tq->q;
            unsigned *const cnt = tq->rt ? tq->rt->cnt : tq->n;
            const int cap = tq->rt ? tq->rt->nw * tq->rt->P : tq->cap;
            // warp-aggregated append: lane prefix of the entry counts, ONE atomic
            const int lane = threadIdx.x & 31, mine = __popc(want) + (self ? 1 : 0);
            int incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += v;
            }
            const int total = __shfl_sync(FULL, incl, 31);
            unsigned base = 0u;
            if (lane == 0 && total) base = atomicAdd(cnt, (unsigned)total);
            int k = (int)__shfl_sync(FULL, base, 0) + incl - mine;
#pragma unroll
            for (int jj = A_SR; jj < A_DN; ++jj)
                if ((want >> jj) & 1u) {
                    if (k < cap) lst[k] = gid(jj);
                    ++k;
                }
            if (self && k < cap) lst[k] = LP == 16 ? c_base >> 1 : L.wi;
        } else {
#pragma unroll
            for (int jj = A_SR; jj < A_DN; ++jj)
                if ((want >> jj) & 1u) tq->push(gid(jj));
            if (self) tq->push(LP == 16 ? c_base >> 1 : L.wi);
        }
    }
    // a push changes this site's residuals and the pair state / excess of its
    // neighbours: all their segments need their arc masks rebuilt next sweep
    const uint32_t pm = seg_ballot<LP>(pushed);
    if (pm && L.valid && L.j == 0) {
#pragma unroll
        for (int q = 0; q < NWB; ++q) {
            dirty[q * P + L.c] = 1u;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (L.has[i]) dirty[q * P + L.nc[i]] = 1u;
        }
    }
}

// Deterministic relabel phase (capped solves): relabel candidates of the push
// phase take one above their lowest residual neighbour; the state is settled
// (no pushes run in this phase) and heights are written to h2 (commit phase).
template <int LP, int R, bool WIN, int RW = 0>
__device__ void w_relabel(const Prob &p, const Arr3 &a, const Bits2 &b, int c_base, int nsites, int seg,
                          int32_t *h2, unsigned &relabels) {
    Lane<LP, R, WIN, RW> L;
    L.init(p, c_base, nsites, seg);
    const uint32_t rl = L.valid ? b.RL[L.bword(p)] : 0u;
    Arcs<LP, R, WIN, false, RW> A;
    A.load(p, a, L);
    if (L.valid && ((rl >> L.bbit()) & 1u)) {
        h2[L.I] = A.best;
        ++relabels;
    }
}

// Deterministic commit phase: relabeled heights take effect, inboxes merge, and
// the active bits of the touched nodes are recomputed.
template <int LP, int R, bool WIN, int RW = 0>
__device__ void w_commit(const Prob &p, const Arr3 &a, const Bits2 &b, int c_base, int nsites, int seg, int32_t *h2) {
    Lane<LP, R, WIN, RW> L;
    L.init(p, c_base, nsites, seg);
    const int I = L.I;
    const uint32_t rl = L.valid ? b.RL[L.bword(p)] : 0u, inb = L.valid ? a.IN0[L.bword(p)] : 0u;
    const bool r_ = (rl >> L.bbit()) & 1u, i_ = (inb >> L.bbit()) & 1u;
    int h = L.valid ? a.h[I] : HINF, e = L.valid ? a.e[I] : 0;
    if (r_) { h = h2[I]; a.h[I] = h; h2[I] = 0; }
    if (i_) { e += a.ein0[I]; a.ein0[I] = 0; a.e[I] = e; }
    const uint32_t touched = seg_ballot<LP>(r_ || i_);
    const uint32_t act = seg_ballot<LP>((r_ || i_) && L.real && e > 0 && h < HINF);
    if (L.valid && L.j == 0) {
        if (RW) {
            for (int w = 0; w < RW; ++w) {
                const int wi = w * p.P + L.c;
                b.A[wi] = (b.A[wi] & ~abs_word<RW>(touched, L.lo, w)) | abs_word<RW>(act, L.lo, w);
                b.RL[wi] = 0u;
                a.IN0[wi] = 0u;
            }
        } else {
            b.A[L.wi] = (b.A[L.wi] & ~touched) | act;
            b.RL[L.wi] = 0u;
            a.IN0[L.wi] = 0u;
        }
    }
}

// extraction seeds: highest position holding excess (last mask build's words)
template <int R, bool WIN, bool PACK = false>
__device__ void w_reach_init(const Prob &p, const Bits2 &b, int c) {
    int lo = 0, hi = p.L;
    if (WIN) { lo = p.lo[c]; hi = p.hi[c]; }
    BW<R> ex;
    ex.load(b.EX, p.P, c);
    const int top = ex.top();
    const int r = top >= 0 ? top + 1 - lo : 0;
    b.R0[c] = gz2::bit_close_up<WIN, R, PACK>(b, p.P, c, lo, hi, r);
}

template <int LPT>
__device__ void w_energy(const Prob &p, const Arr3 &a, int c, long long &energy, int &viol) {
    const int y = c / p.G, g = c - y * p.G;
    const int lab = p.labels[c];
    energy += a.vol[c * LPT + lab];
    for (int i = 0; i < 2; ++i) {
        const bool has = i == 0 ? g + 1 < p.G : y + 1 < p.Y;
        if (!has) continue;
        const int o = p.labels[i == 0 ? c + 1 : c + p.G];
        const int dl = lab > o ? lab - o : o - lab;
        if (p.hard && dl > 1) viol = 1;
        energy += (long long)p.pen * dl + (long long)p.inh * (dl > 1 ? dl - 1 : 0);
    }
}

}  // namespace gz3
