// gz_warpsolve.cuh -- v3 solver: one warp segment per site chain (m <= 32).
//
// Node arrays are column-major, [site][LP] with LP = 16 (m <= 16) or 32, so
// the LP lanes of a warp segment hold the chain positions of one site and
// every per-node load is coalesced.  Lane j <-> chain position t = j + 1.
//   vol[c][k]   data cost of label k              (k < m)
//   cu [c][j]   residual of chain arc t -> t+1     (arc t; arc 0 from the
//               source is saturated at init and never stored)
//   ph/pv/dar/dbr/dad/dbd [c][j]  lateral pair state at level t (see gz_graph.cuh)
//   e, h, ein0/ein1 [c][j]
//
// A pulse is ONE grid-synchronised phase per chain segment:
//   merge last pulse's inbox -> upward chain wave (segmented min-plus scan:
//   x_{t+1} = min(cu_t, e_t + x_t) over admissible chain arcs, the exact
//   Gauss-Seidel result of pushing bottom-up) -> lateral and downward pushes
//   of the remaining excess on admissible arcs -> relabel of nodes that could
//   not push (in place).  A node pushes with its phase-start height and only
//   relabels if it made no push, so two nodes can never push along one arc
//   pair in opposite directions; lateral pushes land in the other inbox
//   buffer (no reader this pulse).
// The BFS / extraction machinery is the bit-parallel one of gz_bitsolve.cuh.
#pragma once

namespace gz3 {

using namespace gz;
using gz2::BW;
using gz2::Bits2;

struct Arr3 {
    int32_t *vol, *cu, *ph, *pv, *dar, *dbr, *dad, *dbd, *e, *ein0, *ein1, *h;
    uint32_t *IN0, *IN1;   // inbox bits per site, double-buffered
};

constexpr unsigned FULL = 0xffffffffu;

template <int LP>
__device__ __forceinline__ int from_above(int v) { return __shfl_down_sync(FULL, v, 1, LP); }   // lane j+1
template <int LP>
__device__ __forceinline__ int from_below(int v) { return __shfl_up_sync(FULL, v, 1, LP); }     // lane j-1

// Per-lane context: node (t, c) plus neighbour sites.
template <int LP, bool WIN>
struct Lane {
    int c, j, t, lo, hi, y, g, I;
    bool valid, real;
    int nc[4], nlo[4], nhi[4];
    bool has[4];
    // sites c_base .. c_base + nsites - 1 (nsites <= 32 / LP), one per LP-lane segment
    __device__ __forceinline__ void init(const Prob &p, int c_base, int nsites) {
        const int lane = threadIdx.x & 31;
        c = c_base + lane / LP;
        j = lane % LP;
        t = j + 1;
        valid = lane / LP < nsites && c < p.P;
        const int cc = valid ? c : 0;
        y = cc / p.G;
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
        real = valid && t > lo && t <= hi;
        I = cc * LP + j;
    }
    __device__ __forceinline__ int kown(int tt) const { return tt <= lo ? K_SRC : (tt > hi ? K_SNK : K_REAL); }
    __device__ __forceinline__ int knb(int i, int tt) const { return tt <= nlo[i] ? K_SRC : (tt > nhi[i] ? K_SNK : K_REAL); }
    __device__ __forceinline__ int nidx(int i) const { return nc[i] * LP + j; }
};

// Residuals of the 14 arcs of a lane's node, target heights and kinds.
// All shuffles are executed by every lane (uniform control flow).
template <int LP, bool WIN>
struct Arcs {
    int r[A_COUNT], hv[A_COUNT], kd[A_COUNT];
    // raw words (for write-back)
    int w_cu, w_ph, w_pv, w_dar, w_dbr, w_dad, w_dbd;   // own-stored at I
    int w_phL, w_pvU, w_darL, w_dbrL, w_dadU, w_dbdU;   // neighbour-stored at the same lane
    int w_dbr_up, w_darL_up, w_dbd_up, w_dadU_up;       // same arrays at lane j+1
    int h_u;

    __device__ __forceinline__ void load(const Prob &p, const Arr3 &a, const Lane<LP, WIN> &L) {
        const int I = L.I;
        const bool v = L.valid;
        w_cu = v ? a.cu[I] : 0;
        w_ph = v ? a.ph[I] : 0;
        w_pv = v ? a.pv[I] : 0;
        w_dar = v ? a.dar[I] : 0;
        w_dbr = v ? a.dbr[I] : 0;
        w_dad = v ? a.dad[I] : 0;
        w_dbd = v ? a.dbd[I] : 0;
        const int iL = L.nidx(1), iU = L.nidx(3);
        w_phL = L.has[1] ? a.ph[iL] : 0;
        w_darL = L.has[1] ? a.dar[iL] : 0;
        w_dbrL = L.has[1] ? a.dbr[iL] : 0;
        w_pvU = L.has[3] ? a.pv[iU] : 0;
        w_dadU = L.has[3] ? a.dad[iU] : 0;
        w_dbdU = L.has[3] ? a.dbd[iU] : 0;
        int hn[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) hn[i] = L.has[i] ? a.h[L.nidx(i)] : HINF;
        h_u = v ? a.h[I] : HINF;
        // lane j+1 values
        w_dbr_up = from_above<LP>(w_dbr);
        w_darL_up = from_above<LP>(w_darL);
        w_dbd_up = from_above<LP>(w_dbd);
        w_dadU_up = from_above<LP>(w_dadU);
        const int h_above = from_above<LP>(h_u), h_below = from_below<LP>(h_u);
        int hn_above[4], hn_below[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { hn_above[i] = from_above<LP>(hn[i]); hn_below[i] = from_below<LP>(hn[i]); }

        const int t = L.t, P2 = 2 * p.pen, cap = p.hard ? p.hcap : p.inh;
        const bool top_ok = t < p.L;   // a position t+1 <= L exists (diagonals up)
#define SETA(J, R, KIND, HV) do { kd[J] = (KIND); r[J] = (KIND) == K_SRC ? 0 : (R); hv[J] = (KIND) == K_SNK ? 0 : (HV); } while (0)
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
    }
};

// flat index and site of an arc's target (only for lateral arcs)
template <int LP, bool WIN>
__device__ __forceinline__ void lateral_target(const Lane<LP, WIN> &L, int jarc, int &site, int &pos) {
    const int i = (jarc - A_SR) & 3;
    site = L.nc[i];
    pos = jarc <= A_SU ? L.t : (jarc <= A_UU ? L.t + 1 : L.t - 1);
}

// inclusive segmented scan of f_j(x) = min(A_j, B_j + x); returns F_j(0)
template <int LP>
__device__ __forceinline__ int chain_wave(int A, int B, int j) {
#pragma unroll
    for (int o = 1; o < LP; o <<= 1) {
        const int A2 = __shfl_up_sync(FULL, A, o, LP), B2 = __shfl_up_sync(FULL, B, o, LP);
        if (j >= o) {   // compose: f_this o f_below
            A = min(A, B + A2);
            B = B + B2;
        }
    }
    return min(A, B);
}

template <int LP>
__device__ __forceinline__ uint32_t seg_ballot(bool pred) {
    const uint32_t b = __ballot_sync(FULL, pred);
    if (LP == 32) return b;
    return (b >> ((threadIdx.x & 31) & ~(LP - 1))) & (LP >= 32 ? 0xffffffffu : ((1u << (LP & 31)) - 1u));
}

// ---------------------------------------------------------------------------
// init: residuals from the volume, source saturation, chain wave, offset
template <int LP, bool WIN>
__device__ void w_init(const Prob &p, const Arr3 &a, const Bits2 &b, int c_base, int nsites, long long &flow,
                       long long &offset, long long &presat) {
    Lane<LP, WIN> L;
    L.init(p, c_base, nsites);
    const int I = L.I;
    const int volj = (L.valid && L.j < p.M) ? a.vol[I] : 0;
    const int vol_above = from_above<LP>(volj);
    if (L.valid) {
        a.cu[I] = (L.j + 1 < p.M) ? vol_above : 0;
        a.ph[I] = p.pen; a.pv[I] = p.pen;
        a.dar[I] = 0; a.dbr[I] = 0; a.dad[I] = 0; a.dbd[I] = 0;
        a.ein0[I] = 0; a.ein1[I] = 0;
        a.h[I] = HINF;
    }
    long long e = 0;
    // chain arc lo: source -> position lo+1 carries vol[lo] (lane lo holds vol[lo])
    const int vol_lo_src = __shfl_sync(FULL, volj, ((threadIdx.x & 31) & ~(LP - 1)) + (L.lo < LP ? L.lo : 0));
    if (L.real && L.t == L.lo + 1) e += vol_lo_src;
    if (WIN && L.valid) {
        const long long icap_off = p.hard ? UNCUTTABLE : (long long)p.inh;
        const int icap = p.hard ? p.hcap : p.inh;
        if (L.j == 0 && L.lo == L.hi) offset += vol_lo_src;
        if (L.t <= p.L) {
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
    // greedy upward wave (no heights yet): every chain arc into a non-source position is usable
    int ex = (int)e;
    int x_out = 0;
    if (!p.no_wave) {
        const bool up_ok = L.real;   // arc t -> t+1 from a real node (target real or sink)
        const int cuw = (L.valid && L.j + 1 < p.M) ? vol_above : 0;
        x_out = chain_wave<LP>(up_ok ? cuw : 0, up_ok ? ex : 0, L.j);
        const int x_below = from_below<LP>(x_out);   // every lane shuffles (full mask)
        const int x_in = L.j > 0 ? x_below : 0;
        const int x_in_use = L.real ? x_in : 0;
        if (L.real) {
            ex = ex + x_in_use - x_out;
            a.cu[I] = cuw - x_out;
            if (L.kown(L.t + 1) == K_SNK) { flow += x_out; presat += x_out; }
        }
    } else {
        (void)from_below<LP>(0);
    }
    if (L.valid) a.e[I] = L.real ? ex : 0;
    (void)b;
}

// ---------------------------------------------------------------------------
// mask build (ballots) + pending inbox merge + BFS reset
template <int LP, bool WIN, bool RESET_H = true>
__device__ void w_build(const Prob &p, const Arr3 &a, const Bits2 &b, int c_base, int nsites) {
    Lane<LP, WIN> L;
    L.init(p, c_base, nsites);
    const int I = L.I, P = p.P;
    // every global load of the group is issued before the first store (one
    // round trip): inbox words and values, excess, then the arc state
    const uint32_t in0 = L.valid ? a.IN0[L.c] : 0u, in1 = L.valid ? a.IN1[L.c] : 0u;
    int e = L.valid ? a.e[I] : 0;
    const int x0 = L.valid ? a.ein0[I] : 0, x1 = L.valid ? a.ein1[I] : 0;
    Arcs<LP, WIN> R;
    R.load(p, a, L);
    // merge both inbox buffers (the last pulse's lateral pushes)
    if ((in0 >> L.j) & 1u) { e += x0; a.ein0[I] = 0; }
    if ((in1 >> L.j) & 1u) { e += x1; a.ein1[I] = 0; }
    if (L.valid && ((in0 | in1) >> L.j) & 1u) a.e[I] = e;
    uint32_t m[13];
#pragma unroll
    for (int q = 0; q < 13; ++q) m[q] = seg_ballot<LP>(L.real && R.r[q] > 0);
    const uint32_t ex = seg_ballot<LP>(L.real && e > 0);
    if (RESET_H && L.valid) a.h[I] = HINF;
    if (L.valid && L.j == 0) {
#pragma unroll
        for (int q = 0; q < 13; ++q) b.mask[(size_t)q * P + L.c] = m[q];
        b.EX[L.c] = ex;
        b.V[L.c] = 0u;
        b.A[L.c] = 0u;
        a.IN0[L.c] = 0u;
        a.IN1[L.c] = 0u;
        b.F0[L.c] = BW<1>::range(L.hi, p.M).w[0];
    }
}

// one BFS level (bit-parallel, thread per site), heights column-major
template <int LP, bool WIN>
__device__ int w_bfs_level(const Prob &p, const Arr3 &a, const Bits2 &b, int c, const uint32_t *Fin, uint32_t *Fout, int d) {
    const int P = p.P;
    const uint32_t F = Fin[c];
    const int y = c / p.G, g = c - y * p.G;
    const bool has[4] = {g + 1 < p.G, g > 0, y + 1 < p.Y, y > 0};
    const int nc[4] = {c + 1, c - 1, c + p.G, c - p.G};
    uint32_t Fn[4];
    uint32_t any = F;
#pragma unroll
    for (int i = 0; i < 4; ++i) { Fn[i] = has[i] ? Fin[nc[i]] : 0u; any |= Fn[i]; }
    uint32_t N = 0u;
    if (any) {
        const uint32_t *m = b.mask;
        N = (F << 1) | ((F >> 1) & m[c]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!Fn[i]) continue;
            N |= (Fn[i] & m[(size_t)(A_SR + i) * P + c]) | ((Fn[i] << 1) & m[(size_t)(A_DR + i) * P + c]) |
                 ((Fn[i] >> 1) & m[(size_t)(A_UR + i) * P + c]);
        }
        int lo = 0, hi = p.L;
        if (WIN) { lo = p.lo[c]; hi = p.hi[c]; }
        const uint32_t V = b.V[c];
        N &= BW<1>::range(lo, hi).w[0] & ~V;
        if (N) {
            b.V[c] = V | N;
            uint32_t x = N;
            while (x) {
                const int bb = __ffs(x) - 1;
                x &= x - 1;
                a.h[c * LP + bb] = d + 1;
            }
        }
    }
    Fout[c] = N;
    int ret = N ? 1 : 0;
    if (N & b.EX[c]) ret |= 2;
    return ret;
}

// ---------------------------------------------------------------------------
// one pulse on a warp group of chains
template <int LP, bool WIN, bool CHECK_IDLE = true>
__device__ void w_pulse(const Prob &p, const Arr3 &a, const Bits2 &b, int c_base, int nsites, int parity,
                        long long &flow, long long &pushes, long long &relabels, uint32_t *dirty = nullptr) {
    Lane<LP, WIN> L;
    L.init(p, c_base, nsites);
    const int I = L.I;
    uint32_t *IN_prev = parity ? a.IN0 : a.IN1;
    uint32_t *IN_cur = parity ? a.IN1 : a.IN0;
    int32_t *ein_prev = parity ? a.ein0 : a.ein1;
    int32_t *ein_cur = parity ? a.ein1 : a.ein0;
    const uint32_t act = L.valid ? b.A[L.c] : 0u, inb = L.valid ? IN_prev[L.c] : 0u;
    if (CHECK_IDLE && !__any_sync(FULL, (act | inb) != 0u)) return;
    // all loads before the first store: one round trip per group (ein_prev has
    // no writer during this pulse, so reading it unconditionally is safe)
    int e = L.valid ? a.e[I] : 0;
    const int xin = L.valid ? ein_prev[I] : 0;
    Arcs<LP, WIN> R;
    R.load(p, a, L);
    if ((inb >> L.j) & 1u) { e += xin; ein_prev[I] = 0; }
    if (L.valid && L.j == 0 && inb) IN_prev[L.c] = 0u;
    const int hu = R.h_u;
    const bool live = L.real && hu < HINF;
    // upward chain wave through admissible chain arcs
    const bool adm_up = live && R.r[A_UP] > 0 && R.kd[A_UP] != K_SRC && hu == R.hv[A_UP] + 1;
    const int x_out = chain_wave<LP>(adm_up ? R.r[A_UP] : 0, adm_up ? max(e, 0) : 0, L.j);
    const int x_below = from_below<LP>(x_out);   // every lane shuffles (full mask)
    const int x_in = L.j > 0 ? x_below : 0;
    int cu_new = R.w_cu;
    bool pushed = false;
    if (L.real) {
        e += x_in - x_out;
        if (x_out > 0) {
            cu_new -= x_out;
            pushed = true;
            ++pushes;
            if (R.kd[A_UP] == K_SNK) flow += x_out;
        }
    }
    // lateral and downward pushes of the remaining excess
    int dn = 0;
    int ph_d = 0, pv_d = 0, dar_d = 0, dad_d = 0;
    int phL_d = 0, pvU_d = 0, dbrL_d = 0, dbdU_d = 0, dbr_up_d = 0, darL_up_d = 0, dbd_up_d = 0, dadU_up_d = 0;
    if (live && e > 0) {
#pragma unroll
        for (int jj = A_SR; jj <= A_DN; ++jj) {
            if (e <= 0) break;
            if (R.kd[jj] == K_SRC || R.r[jj] <= 0 || hu != R.hv[jj] + 1) continue;
            const int d = min(e, R.r[jj]);
            e -= d;
            pushed = true;
            ++pushes;
            switch (jj) {
            case A_SR: ph_d -= d; break;
            case A_SL: phL_d += d; break;
            case A_SD: pv_d -= d; break;
            case A_SU: pvU_d += d; break;
            case A_UR: dbr_up_d -= d; break;
            case A_UL: darL_up_d -= d; break;
            case A_UD: dbd_up_d -= d; break;
            case A_UU: dadU_up_d -= d; break;
            case A_DR: dar_d += d; break;
            case A_DL: dbrL_d += d; break;
            case A_DD: dad_d += d; break;
            case A_DU: dbdU_d += d; break;
            case A_DN: dn += d; break;
            }
            if (jj == A_DN) continue;
            if (R.kd[jj] == K_SNK) { flow += d; continue; }
            int site, pos;
            lateral_target<LP, WIN>(L, jj, site, pos);
            atomicAdd(&ein_cur[site * LP + pos - 1], d);
            atomicOr(&IN_cur[site], 1u << (pos - 1));
        }
    }
    // chain-down pushes arrive at lane j-1 (adds to its excess and to its chain-up residual)
    const int dn_recv = from_above<LP>(dn);
    const int dn_in = (L.real && L.j + 1 < LP) ? dn_recv : 0;
    if (L.real) {
        e += dn_in;
        cu_new += dn_in;
    }
    // relabel a live node that could not push
    int hnew = hu;
    if (live && !pushed && e > 0) {
        int best = HINF;
#pragma unroll
        for (int jj = 0; jj < A_COUNT; ++jj)
            if (R.kd[jj] != K_SRC && R.r[jj] > 0) best = min(best, R.hv[jj] + 1);
        hnew = best;
        ++relabels;
    }
    // write back
    if (L.real) {
        a.e[I] = e;
        if (cu_new != R.w_cu) a.cu[I] = cu_new;
        if (hnew != hu) a.h[I] = hnew;
        if (ph_d) a.ph[I] = R.w_ph + ph_d;
        if (pv_d) a.pv[I] = R.w_pv + pv_d;
        if (dar_d) a.dar[I] = R.w_dar + dar_d;
        if (dad_d) a.dad[I] = R.w_dad + dad_d;
        if (phL_d) a.ph[L.nidx(1)] = R.w_phL + phL_d;
        if (dbrL_d) a.dbr[L.nidx(1)] = R.w_dbrL + dbrL_d;
        if (pvU_d) a.pv[L.nidx(3)] = R.w_pvU + pvU_d;
        if (dbdU_d) a.dbd[L.nidx(3)] = R.w_dbdU + dbdU_d;
        if (dbr_up_d) a.dbr[I + 1] = R.w_dbr_up + dbr_up_d;
        if (dbd_up_d) a.dbd[I + 1] = R.w_dbd_up + dbd_up_d;
        if (darL_up_d) a.dar[L.nidx(1) + 1] = R.w_darL_up + darL_up_d;
        if (dadU_up_d) a.dad[L.nidx(3) + 1] = R.w_dadU_up + dadU_up_d;
    }
    const uint32_t newA = seg_ballot<LP>(L.real && e > 0 && hnew < HINF);
    if (L.valid && L.j == 0) b.A[L.c] = newA;
    if (dirty) {
        // a push changes this site's residuals and the pair state / excess of its
        // neighbours: all of them need their arc masks rebuilt next sweep
        const uint32_t pm = seg_ballot<LP>(pushed);
        if (pm && L.valid && L.j == 0) {
            dirty[L.c] = 1u;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (L.has[i]) dirty[L.nc[i]] = 1u;
        }
    }
}

// extraction seeds from the last mask build's excess bits
template <bool WIN>
__device__ void w_reach_init(const Prob &p, const Bits2 &b, int c) {
    int lo = 0, hi = p.L;
    if (WIN) { lo = p.lo[c]; hi = p.hi[c]; }
    const uint32_t ex = b.EX[c];
    const int r = ex ? (31 - __clz(ex)) + 1 - lo : 0;
    b.R0[c] = gz2::bit_close_up<WIN, 1>(b, p.P, c, lo, hi, r);
}

template <int LP>
__device__ void w_energy(const Prob &p, const Arr3 &a, int c, long long &energy, int &viol) {
    const int y = c / p.G, g = c - y * p.G;
    const int lab = p.labels[c];
    energy += a.vol[c * LP + lab];
    for (int i = 0; i < 2; ++i) {
        const bool has = i == 0 ? g + 1 < p.G : y + 1 < p.Y;
        if (!has) continue;
        const int o = p.labels[i == 0 ? c + 1 : c + p.G];
        const int dl = lab > o ? lab - o : o - lab;
        if (p.hard && dl > 1) viol = 1;
        energy += (long long)p.pen * dl + (long long)p.inh * (dl > 1 ? dl - 1 : 0);
    }
}

// ---------------------------------------------------------------------------
template <int LP, bool WIN>
__global__ void __launch_bounds__(256) gz_warpsolve_kernel(Prob p, Bits2 b, Arr3 a) {
    __shared__ unsigned s_acc[3];
    cg::grid_group grid = cg::this_grid();
    unsigned long long t_prev = 0, t_acc[6] = {0, 0, 0, 0, 0, 0};
    const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
    if (timer) t_prev = gz2::gtimer();
    if (timer) p.t_start_ns = t_prev;
#define TICK(slot) do { if (timer) { unsigned long long t_ = gz2::gtimer(); t_acc[slot] += t_ - t_prev; t_prev = t_; } } while (0)
    unsigned prog_ = 0;
#define PROG() do { if (p.progress && threadIdx.x == 0) { p.progress[blockIdx.x] = ++prog_; __threadfence_system(); } } while (0)
    const int stride = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int niter = (p.P + stride - 1) / stride;
    constexpr int CPW = 32 / LP;
    const int ngroups = (p.P + CPW - 1) / CPW;
    const int nwarps = stride / 32, wid = tid / 32;
    const int giter = (ngroups + nwarps - 1) / nwarps;
    long long flow = 0, offset = 0, presat = 0, pushes = 0, relabels = 0;
    volatile unsigned long long *vctr = p.ctr;
#define FOR_COLS for (int it_ = 0, c = tid; it_ < niter; ++it_, c += stride) if (c < p.P)
#define FOR_GROUPS for (int it_ = 0, grp = wid; it_ < giter; ++it_, grp += nwarps) if (grp < ngroups)

    PROG();
    FOR_GROUPS w_init<LP, WIN>(p, a, b, grp * CPW, CPW, flow, offset, presat);
    PROG();
    grid.sync();
    TICK(0);
    int sweeps = 0, levels_total = 0, pulses = 0, rot = 0, parity = 0;
    int converged = 1;
    bool err = false;
    const int bfs_min = p.bfs_cap > 0 ? p.bfs_cap : (1 << 30);
    for (;;) {
        FOR_GROUPS w_build<LP, WIN>(p, a, b, grp * CPW, CPW);
        PROG();
        grid.sync();
        TICK(1);
        int d = 0;
        bool found = false, exhausted = false;
        uint32_t *Fin = b.F0, *Fout = b.F1;
        for (;;) {
            unsigned flags = 0;
            FOR_COLS flags |= (unsigned)w_bfs_level<LP, WIN>(p, a, b, c, Fin, Fout, d);
            PROG();
            const unsigned gf = gz2::grid_or(grid, flags, p.ctr + CTR_FLAG0, rot, s_acc);
            found |= (gf & 2u) != 0;
            uint32_t *tmp = Fin; Fin = Fout; Fout = tmp;
            ++d;
            if (!(gf & 1u)) { exhausted = true; break; }
            if (found && d >= bfs_min) break;
            if (d > 4 * (p.P + p.M)) { if (tid == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); err = true; break; }
        }
        levels_total += d;
        TICK(2);
        if (err) break;
        if (!found && exhausted) break;
        if (p.capped && sweeps >= p.max_sweeps) { converged = 0; break; }
        FOR_COLS b.A[c] = b.V[c] & b.EX[c];
        grid.sync();
        for (int pulse = 0; pulse < p.K; ++pulse) {
            FOR_GROUPS w_pulse<LP, WIN>(p, a, b, grp * CPW, CPW, parity, flow, pushes, relabels);
            PROG();
            grid.sync();
            parity ^= 1;
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
    // extraction
    FOR_COLS w_reach_init<WIN>(p, b, c);
    grid.sync();
    int reach_passes = 0;
    int32_t *Rin = b.R0, *Rout = b.R1;
    for (;;) {
        unsigned ch = 0;
        FOR_COLS ch |= gz2::bit_reach_iter<WIN, 1>(p, b, c, Rin, Rout) ? 1u : 0u;
        PROG();
        const bool any = gz2::grid_or(grid, ch, p.ctr + CTR_FLAG0, rot, s_acc) != 0;
        int32_t *tmp = Rin; Rin = Rout; Rout = tmp;
        ++reach_passes;
        if (!any) break;
        if (reach_passes > 4 * (p.P + p.M)) { if (tid == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
    }
    TICK(4);
    long long stranded = 0;
    FOR_COLS {
        const int lo = WIN ? p.lo[c] : 0;
        p.labels[c] = lo + Rin[c];
        stranded += __popc(b.EX[c]);
    }
    grid.sync();
    long long energy = 0;
    int viol = 0;
    FOR_COLS w_energy<LP>(p, a, c, energy, viol);
#undef FOR_COLS
#undef FOR_GROUPS
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

}  // namespace gz3
