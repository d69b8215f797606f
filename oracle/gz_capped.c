/* gz_capped.c -- CPU restatement of the device's deterministic CAPPED schedule
 * (level-2 fine solves), so capped labelings can be pinned bit
 * for bit.
 *
 * TEST INFRASTRUCTURE ONLY (tests/test_gpu_level2.py).  The reference's own
 * capped schedule is a sequential FIFO sorted by block (maxflow.py:198-249),
 * which a GPU cannot replay; the device runs its own schedule, restated here
 * from paper_1803_01516_b200/csrc (gz_chain.cuh w_init / w_build / w_pulse
 * with DETPUSH, w_relabel, w_commit; gz_tilesolve.cuh sweep loop and BFS).
 * Every step is a function of the state at the start of its phase, so the
 * order in which the device's warps visit chains does not matter and this
 * sequential loop reproduces it exactly:
 *
 *   init   residuals from the data term (chain arc t -> t+1 = vol[t], penalty
 *          pairs at 2 x penalty / 2, inhibit flows 0); source arcs (chain arc
 *          lo, penalty / inhibit arcs out of source positions) saturated into
 *          the excess; a greedy bottom-up chain wave (maxflow.py:287-304 stands
 *          in for the paper's wave front fetch).
 *   sweep  exact BFS distance to the sink over residual arcs (maxflow.py:138-158)
 *          in rounds of H levels (H = the device's blocking depth,
 *          gz_stats.bfs_h), stopping after the first round that ends at depth
 *          >= bfs_min having met a node with excess, or when a round finds
 *          nothing new; unvisited nodes park at HINF.  Then K pulses:
 *            push     every live node with excess: a bottom-up chain wave over
 *                     admissible chain arcs, then its remaining excess along
 *                     admissible arcs in the fixed arc order (lateral pushes
 *                     land in the target's inbox, chain-down pushes go to the
 *                     node below at once);
 *            relabel  nodes that kept excess without pushing: one above their
 *                     lowest residual neighbour, into a second height buffer;
 *            commit   heights take effect, inboxes merge.
 *          A pulse in which no node had work ends the sweep.
 *   stop   converged when a BFS reaches no excess; capped after max_sweeps
 *          sweeps, after one more BFS run to exhaustion.
 *   read   converged: labels = lo + the prefix of each chain reachable in the
 *          residual network from the nodes holding excess (maxflow.py:267-320);
 *          capped: every node that cannot reach the sink is on the source side
 *          (labels = hi - the nodes the last BFS reached).
 *
 * Full-chain segments only: the caller ensures every chain is one warp segment
 * on the device (m <= 16, or windows <= 15 positions wide with m <= 64: the
 * window-relative 16-lane instance), which is the case for level-2 fine
 * solves.  Soft inhibit only.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;
#define HINF 0x3fffffff

enum { K_SRC = 0, K_REAL = 1, K_SNK = 2 };
enum { A_UP = 0, A_SR, A_SL, A_SD, A_SU, A_UR, A_UL, A_UD, A_UU, A_DR, A_DL, A_DD, A_DU, A_DN, A_COUNT };

typedef struct {
    int Y, G, M, L, P;
    i64 pen, inh;
    const int32_t *lo, *hi;   /* per site */
    i64 *cu, *ph, *pv, *dar, *dbr, *dad, *dbd, *e, *ein;
    int32_t *h, *h2;
} St;

#define IX(c, t) ((i64)(c) * S->L + (t) - 1)

static int kind(const St *S, int c, int t) { return t <= S->lo[c] ? K_SRC : (t > S->hi[c] ? K_SNK : K_REAL); }

static int nbr(const St *S, int c, int i) {   /* right, left, down, up; -1 if none */
    const int y = c / S->G, g = c % S->G;
    if (i == 0) return g + 1 < S->G ? c + 1 : -1;
    if (i == 1) return g > 0 ? c - 1 : -1;
    if (i == 2) return y + 1 < S->Y ? c + S->G : -1;
    return y > 0 ? c - S->G : -1;
}

/* residual, target site / position and kind of arc jj out of real node (c, t)
 * (gz_chain.cuh Arcs::load, windowed form) */
static i64 arc(const St *S, int c, int t, int jj, int *tc, int *tt, int *tk) {
    int n = -1;
    i64 r = 0;
    *tc = c; *tt = t;
    switch (jj) {
    case A_UP: *tt = t + 1; r = S->cu[IX(c, t)]; break;
    case A_DN: *tt = t - 1; r = HINF; break;
    case A_SR: n = nbr(S, c, 0); if (n >= 0) r = S->ph[IX(c, t)]; break;
    case A_SL: n = nbr(S, c, 1); if (n >= 0) r = 2 * S->pen - S->ph[IX(n, t)]; break;
    case A_SD: n = nbr(S, c, 2); if (n >= 0) r = S->pv[IX(c, t)]; break;
    case A_SU: n = nbr(S, c, 3); if (n >= 0) r = 2 * S->pen - S->pv[IX(n, t)]; break;
    case A_UR: n = nbr(S, c, 0); *tt = t + 1; if (n >= 0 && t < S->L) r = S->dbr[IX(c, t + 1)]; break;
    case A_UL: n = nbr(S, c, 1); *tt = t + 1; if (n >= 0 && t < S->L) r = S->dar[IX(n, t + 1)]; break;
    case A_UD: n = nbr(S, c, 2); *tt = t + 1; if (n >= 0 && t < S->L) r = S->dbd[IX(c, t + 1)]; break;
    case A_UU: n = nbr(S, c, 3); *tt = t + 1; if (n >= 0 && t < S->L) r = S->dad[IX(n, t + 1)]; break;
    case A_DR: n = nbr(S, c, 0); *tt = t - 1; if (n >= 0) r = S->inh - S->dar[IX(c, t)]; break;
    case A_DL: n = nbr(S, c, 1); *tt = t - 1; if (n >= 0) r = S->inh - S->dbr[IX(n, t)]; break;
    case A_DD: n = nbr(S, c, 2); *tt = t - 1; if (n >= 0) r = S->inh - S->dad[IX(c, t)]; break;
    case A_DU: n = nbr(S, c, 3); *tt = t - 1; if (n >= 0) r = S->inh - S->dbd[IX(n, t)]; break;
    }
    if (jj != A_UP && jj != A_DN) {
        if (n < 0 || (jj >= A_UR && jj <= A_UU && t >= S->L)) { *tk = K_SRC; return 0; }
        *tc = n;
    }
    *tk = kind(S, *tc, *tt);
    return *tk == K_SRC ? 0 : r;
}

static int height_of(const St *S, int tc, int tt, int tk) { return tk == K_SNK ? 0 : S->h[IX(tc, tt)]; }

/* apply a push of d along arc jj of (c, t) to the pair state (gz_chain.cuh write-back) */
static void apply(St *S, int c, int t, int jj, i64 d) {
    switch (jj) {
    case A_SR: S->ph[IX(c, t)] -= d; break;
    case A_SD: S->pv[IX(c, t)] -= d; break;
    case A_DR: S->dar[IX(c, t)] += d; break;
    case A_DD: S->dad[IX(c, t)] += d; break;
    case A_SL: S->ph[IX(nbr(S, c, 1), t)] += d; break;
    case A_SU: S->pv[IX(nbr(S, c, 3), t)] += d; break;
    case A_DL: S->dbr[IX(nbr(S, c, 1), t)] += d; break;
    case A_DU: S->dbd[IX(nbr(S, c, 3), t)] += d; break;
    case A_UR: S->dbr[IX(c, t + 1)] -= d; break;
    case A_UD: S->dbd[IX(c, t + 1)] -= d; break;
    case A_UL: S->dar[IX(nbr(S, c, 1), t + 1)] -= d; break;
    case A_UU: S->dad[IX(nbr(S, c, 3), t + 1)] -= d; break;
    }
}

/* BFS from the sink (gz_tilesolve.cuh bfs_round semantics); returns found, sets *exhausted */
static int bfs(St *S, int H, int bfs_min, int *exhausted, const uint8_t *ex, uint8_t *vis, int *lev_of,
               i64 *q, i64 *nq) {
    const i64 N = (i64)S->P * S->L;
    for (i64 i = 0; i < N; ++i) { S->h[i] = HINF; vis[i] = 0; }
    /* level 1: real nodes with a residual arc into a sink position */
    i64 nf = 0;
    for (int c = 0; c < S->P; ++c)
        for (int t = S->lo[c] + 1; t <= S->hi[c]; ++t)
            for (int jj = 0; jj < A_COUNT; ++jj) {
                int tc, tt, tk;
                const i64 r = arc(S, c, t, jj, &tc, &tt, &tk);
                if (r > 0 && tk == K_SNK) { vis[IX(c, t)] = 1; q[nf++] = IX(c, t); break; }
            }
    int d = 0, found = 0, lev = 1;
    *exhausted = 0;
    for (;;) {
        /* one round: levels d+1 .. d+H */
        int any = 0;
        for (int k = 0; k < H; ++k, ++lev) {
            if (lev == 1) {   /* the level-1 set was built above */
                for (i64 i = 0; i < nf; ++i) { S->h[q[i]] = 1; any = 1; found |= ex[q[i]]; }
                continue;
            }
            i64 nn = 0;
            for (i64 i = 0; i < nf; ++i) {   /* nodes with a residual arc into the last level */
                const int c = (int)(q[i] / S->L), t = (int)(q[i] % S->L) + 1;
                for (int i2 = -1; i2 < 4; ++i2) {   /* the site itself, then its neighbours */
                    const int cc = i2 < 0 ? c : nbr(S, c, i2);
                    if (cc < 0) continue;
                    for (int tt = t - 1; tt <= t + 1; ++tt) {
                        if (tt <= S->lo[cc] || tt > S->hi[cc] || vis[IX(cc, tt)]) continue;
                        for (int jj = 0; jj < A_COUNT; ++jj) {
                            int xc, xt, xk;
                            const i64 r = arc(S, cc, tt, jj, &xc, &xt, &xk);
                            if (r > 0 && xk == K_REAL && xc == c && xt == t) {
                                vis[IX(cc, tt)] = 1;
                                nq[nn++] = IX(cc, tt);
                                break;
                            }
                        }
                    }
                }
            }
            for (i64 i = 0; i < nn; ++i) { S->h[nq[i]] = lev; any = 1; found |= ex[nq[i]]; q[i] = nq[i]; }
            nf = nn;
        }
        d += H;
        if (!any) { *exhausted = 1; break; }
        if (found && d >= bfs_min) break;
        if (d > 4 * (S->P + S->M) + 4 * H) break;
    }
    (void)lev_of;
    return found;
}

/* Returns 0; labels (P), report: [0] flow, [1] sweeps, [2] pulses, [3] converged */
int gzo_capped(const int32_t *vol, int rows, int cols, int m, int32_t penalty, int32_t inhibit, const int32_t *lo,
               const int32_t *hi, int K, int max_sweeps, int bfs_min, int H, int wave, int32_t *labels, i64 *report) {
    St s_, *S = &s_;
    S->Y = rows; S->G = cols; S->M = m; S->L = m - 1; S->P = rows * cols;
    S->pen = penalty; S->inh = inhibit; S->lo = lo; S->hi = hi;
    const i64 N = (i64)S->P * S->L;
    i64 *buf = (i64 *)calloc((size_t)N * 9, sizeof(i64));
    S->cu = buf; S->ph = buf + N; S->pv = buf + 2 * N; S->dar = buf + 3 * N; S->dbr = buf + 4 * N;
    S->dad = buf + 5 * N; S->dbd = buf + 6 * N; S->e = buf + 7 * N; S->ein = buf + 8 * N;
    S->h = (int32_t *)malloc((size_t)N * 4); S->h2 = (int32_t *)malloc((size_t)N * 4);
    uint8_t *ex = (uint8_t *)calloc((size_t)N, 1), *vis = (uint8_t *)calloc((size_t)N, 1);
    uint8_t *rl = (uint8_t *)calloc((size_t)N, 1), *inb = (uint8_t *)calloc((size_t)N, 1);
    i64 *q = (i64 *)malloc((size_t)(N + 1) * 8), *nq = (i64 *)malloc((size_t)(N + 1) * 8);
    i64 flow = 0;
    /* ---- init (w_init) ---- */
    for (int c = 0; c < S->P; ++c) {
        const int32_t *v = vol + (i64)c * m;
        for (int t = 1; t <= S->L; ++t) {
            S->cu[IX(c, t)] = t < m ? v[t] : 0;
            S->ph[IX(c, t)] = S->pen; S->pv[IX(c, t)] = S->pen;
        }
        for (int t = lo[c] + 1; t <= hi[c]; ++t) {
            i64 e = t == lo[c] + 1 ? v[lo[c]] : 0;
            for (int i = 0; i < 4; ++i) {
                const int n = nbr(S, c, i);
                if (n < 0) continue;
                if (kind(S, n, t) == K_SRC) e += S->pen;
                if (t + 1 <= S->L && kind(S, n, t + 1) == K_SRC) e += S->inh;
            }
            S->e[IX(c, t)] = e;
        }
        if (wave) {   /* greedy bottom-up wave over the whole chain */
            i64 x = 0;
            for (int t = lo[c] + 1; t <= hi[c]; ++t) {
                const i64 cu = S->cu[IX(c, t)], xo = cu < S->e[IX(c, t)] + x ? cu : S->e[IX(c, t)] + x;
                S->e[IX(c, t)] += x - xo;
                S->cu[IX(c, t)] = cu - xo;
                if (kind(S, c, t + 1) == K_SNK) flow += xo;
                x = xo;
            }
        }
    }
    int sweeps = 0, pulses = 0, converged = 1;
    for (;;) {
        for (i64 i = 0; i < N; ++i) ex[i] = 0;
        for (int c = 0; c < S->P; ++c)
            for (int t = lo[c] + 1; t <= hi[c]; ++t) ex[IX(c, t)] = S->e[IX(c, t)] > 0;
        int exhausted = 0;
        const int last = sweeps >= max_sweeps;   /* the last BFS runs to exhaustion (read-out) */
        const int found = bfs(S, H, last ? 0x7fffffff : bfs_min, &exhausted, ex, vis, NULL, q, nq);
        if (!found && exhausted) break;
        if (last) { converged = 0; break; }
        for (int pulse = 0; pulse < K; ++pulse) {
            int work = 0;
            memset(rl, 0, (size_t)N);
            memset(inb, 0, (size_t)N);
            /* ---- push phase (w_pulse, DETPUSH), chain by chain ---- */
            for (int c = 0; c < S->P; ++c) {
                const int l0 = lo[c], h0 = hi[c];
                if (h0 <= l0) continue;
                int any = 0;
                for (int t = l0 + 1; t <= h0; ++t) any |= S->e[IX(c, t)] > 0 && S->h[IX(c, t)] < HINF;
                if (!any) continue;
                work = 1;
                /* chain-start snapshot: excess, heights, the wave */
                i64 e0[64], xo[64], dn[64];
                int pushed[64];
                for (int t = l0 + 1; t <= h0; ++t) e0[t] = S->e[IX(c, t)];
                i64 x = 0;
                for (int t = l0 + 1; t <= h0; ++t) {
                    const int hu = S->h[IX(c, t)];
                    const int live = hu < HINF;
                    int tc, tt, tk;
                    const i64 r = arc(S, c, t, A_UP, &tc, &tt, &tk);
                    const int adm = live && r > 0 && hu == height_of(S, tc, tt, tk) + 1;
                    const i64 A = adm ? r : 0, B = adm ? (e0[t] > 0 ? e0[t] : 0) : 0;
                    const i64 out = A < B + x ? A : B + x;
                    xo[t] = out;
                    x = out;
                }
                for (int t = l0 + 1; t <= h0; ++t) {
                    const i64 xin = t > l0 + 1 ? xo[t - 1] : 0;
                    i64 e = e0[t] + xin - xo[t];
                    pushed[t] = 0;
                    dn[t] = 0;
                    if (xo[t] > 0) {
                        S->cu[IX(c, t)] -= xo[t];
                        pushed[t] = 1;
                        if (kind(S, c, t + 1) == K_SNK) flow += xo[t];
                    }
                    const int hu = S->h[IX(c, t)];
                    const int live = hu < HINF;
                    i64 rem = (live && e > 0) ? e : 0;
                    for (int jj = A_SR; jj <= A_DN; ++jj) {
                        int tc, tt, tk;
                        const i64 r = arc(S, c, t, jj, &tc, &tt, &tk);
                        if (!(r > 0 && hu == height_of(S, tc, tt, tk) + 1)) continue;
                        const i64 d = rem < r ? rem : r;
                        if (d <= 0) continue;
                        rem -= d;
                        pushed[t] = 1;
                        if (jj == A_DN) { dn[t] = d; continue; }
                        apply(S, c, t, jj, d);
                        if (tk == K_SNK) flow += d;
                        else { S->ein[IX(tc, tt)] += d; inb[IX(tc, tt)] = 1; }
                    }
                    if (live && e > 0) e = rem;
                    S->e[IX(c, t)] = e;
                }
                /* chain-down pushes reach the node below within the pulse */
                for (int t = l0 + 1; t <= h0; ++t)
                    if (t + 1 <= h0 && dn[t + 1] > 0) {
                        S->e[IX(c, t)] += dn[t + 1];
                        S->cu[IX(c, t)] += dn[t + 1];
                    }
                for (int t = l0 + 1; t <= h0; ++t)
                    rl[IX(c, t)] = S->h[IX(c, t)] < HINF && !pushed[t] && S->e[IX(c, t)] > 0;
            }
            /* ---- relabel phase (w_relabel): settled residuals, committed heights ---- */
            for (int c = 0; c < S->P; ++c)
                for (int t = lo[c] + 1; t <= hi[c]; ++t) {
                    if (!rl[IX(c, t)]) continue;
                    int best = HINF;
                    for (int jj = 0; jj < A_COUNT; ++jj) {
                        int tc, tt, tk;
                        const i64 r = arc(S, c, t, jj, &tc, &tt, &tk);
                        if (r > 0) {
                            const int hv = height_of(S, tc, tt, tk) + 1;
                            if (hv < best) best = hv;
                        }
                    }
                    S->h2[IX(c, t)] = best;
                }
            /* ---- commit phase (w_commit) ---- */
            for (i64 i = 0; i < N; ++i) {
                if (rl[i]) S->h[i] = S->h2[i];
                if (inb[i]) { S->e[i] += S->ein[i]; S->ein[i] = 0; }
            }
            ++pulses;
            if (!work) break;
        }
        ++sweeps;
        if (sweeps > 1000000) break;
    }
    /* ---- read-out ---- */
    if (!converged) {
        /* capped stop: the source side is every node that cannot reach the sink
           (vis = the last, exhaustive BFS) -- a prefix of each chain */
        for (int c = 0; c < S->P; ++c) {
            int reach = 0;
            for (int t = lo[c] + 1; t <= hi[c]; ++t) reach += vis[IX(c, t)];
            labels[c] = hi[c] - reach;
        }
        report[0] = flow; report[1] = sweeps; report[2] = pulses; report[3] = converged;
        free(buf); free(S->h); free(S->h2); free(ex); free(vis); free(rl); free(inb); free(q); free(nq);
        return 0;
    }
    /* converged: residual reach from the excess nodes (w_reach_init / bit_reach_iter) */
    memset(vis, 0, (size_t)N);
    i64 qt = 0;
    for (int c = 0; c < S->P; ++c)
        for (int t = lo[c] + 1; t <= hi[c]; ++t)
            if (S->e[IX(c, t)] > 0) { vis[IX(c, t)] = 1; q[qt++] = IX(c, t); }
    for (i64 qh = 0; qh < qt; ++qh) {
        const int c = (int)(q[qh] / S->L), t = (int)(q[qh] % S->L) + 1;
        for (int jj = 0; jj < A_COUNT; ++jj) {
            int tc, tt, tk;
            const i64 r = arc(S, c, t, jj, &tc, &tt, &tk);
            if (r > 0 && tk == K_REAL && !vis[IX(tc, tt)]) { vis[IX(tc, tt)] = 1; q[qt++] = IX(tc, tt); }
        }
    }
    for (int c = 0; c < S->P; ++c) {
        int k = 0;
        while (lo[c] + 1 + k <= hi[c] && vis[IX(c, lo[c] + 1 + k)]) ++k;
        labels[c] = lo[c] + k;
    }
    report[0] = flow; report[1] = sweeps; report[2] = pulses; report[3] = converged;
    free(buf); free(S->h); free(S->h2); free(ex); free(vis); free(rl); free(inb); free(q); free(nq);
    return 0;
}
