/* gz_certify.c -- CPU optimality certificate for device solves of configs the
 * reference cannot build (C3 1920x1080x128, C5 3840x2160x256: its int32 CSR
 * cannot hold their 3.6 G / 29.5 G arcs, flownet.py:204-207).
 *
 * TEST INFRASTRUCTURE ONLY (tests/test_gpu_big.py).  SURVEY.md §8(c): the
 * device's final state must be a feasible PREFLOW of the reference's network
 * (flownet.py:102-181 _emit semantics for full windows: chain arcs with
 * capacity vol[t] and uncuttable reverse, penalty pairs both ways, inhibit
 * diagonals forward), whose value equals the cut cost of the returned
 * labeling (energy.py:129-155 total_energy; const_offset is 0 for full
 * windows).  A preflow's sink inflow bounds every cut from below, so a cut of
 * the same cost is a minimum cut (weak duality).  The labeling must further
 * be the MINIMAL source side the reference reads (maxflow.py:267-284,
 * 307-320): the nodes reachable in the residual network from the source and
 * from every node holding excess (for a maximum preflow that set is the
 * minimal source side of the minimum cut).
 *
 * State planes (gz_export_state, include/gazecut_b200.h), int32 [P][L],
 * P = rows * cols sites (row-major), L = m - 1 positions, column t-1 holds
 * position t:
 *   cu   residual of chain arc t -> t+1 (capacity vol[t]; t = L: into the sink)
 *   ph   residual of (c,t) -> (c+1,t); reverse residual 2*penalty - ph
 *   pv   residual of (c,t) -> (c+G,t)
 *   dar  flow (c,t) -> (c+1,t-1)     dbr  flow (c+1,t) -> (c,t-1)
 *   dad  flow (c,t) -> (c+G,t-1)     dbd  flow (c+G,t) -> (c,t-1)
 *        (capacity inhibit, reverse capacity 0; t = 1 would enter the source
 *         and must carry nothing)
 *   e    excess
 * vol: int32 (rows, cols, m), the data term.
 *
 * Returns 0 when every check passes, else the number of the first failed
 * check (details in report[]):
 *   1 capacity bounds   2 conservation (in - out == excess)   3 flow value
 *   4 cut cost          5 minimal source side                 6 out of memory
 * report (int64[8]): [0] flow into the sink, [1] labeling energy, [2] nodes
 * reached by the source-side search, [3] first failing node (or -1),
 * [4] sites whose label disagrees with the search, [5] nodes with excess.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

static i64 pair_cost(i64 a, i64 b, i64 pen, i64 inh) {
    const i64 d = a > b ? a - b : b - a;
    return pen * d + inh * (d > 1 ? d - 1 : 0);   /* energy.py:60-67 */
}

int gzc_certify(int rows, int cols, int m, const int32_t *vol, int32_t penalty, int32_t inhibit,
                const int32_t *cu, const int32_t *ph, const int32_t *pv, const int32_t *dar, const int32_t *dbr,
                const int32_t *dad, const int32_t *dbd, const int32_t *e, const int32_t *labels, i64 device_flow,
                i64 *report) {
    const i64 G = cols, P = (i64)rows * cols, L = m - 1, N = P * L;
    const i64 pen = penalty, inh = inhibit;
    for (int k = 0; k < 8; ++k) report[k] = 0;
    report[3] = -1;
#define AT(c, t) ((c) * L + (t) - 1)
    /* 1. capacity bounds */
    for (i64 c = 0; c < P; ++c) {
        const i64 g = c % G, y = c / G;
        for (i64 t = 1; t <= L; ++t) {
            const i64 i = AT(c, t);
            int ok = cu[i] >= 0 && e[i] >= 0;
            if (g + 1 < G) ok = ok && ph[i] >= 0 && ph[i] <= 2 * pen && dar[i] >= 0 && dar[i] <= inh &&
                                dbr[i] >= 0 && dbr[i] <= inh && (t > 1 || (dar[i] == 0 && dbr[i] == 0));
            if (y + 1 < rows) ok = ok && pv[i] >= 0 && pv[i] <= 2 * pen && dad[i] >= 0 && dad[i] <= inh &&
                                   dbd[i] >= 0 && dbd[i] <= inh && (t > 1 || (dad[i] == 0 && dbd[i] == 0));
            if (!ok) { report[3] = i; return 1; }
        }
    }
    /* 2. conservation: in - out == excess at every node; 3. sink inflow */
    i64 *net = (i64 *)calloc((size_t)N, sizeof(i64));
    if (!net) return 6;
    i64 sink_in = 0;
    for (i64 c = 0; c < P; ++c) {
        const i64 g = c % G, y = c / G;
        const int32_t *v = vol + c * m;
        net[AT(c, 1)] += v[0];                       /* saturated source arc (label 0) */
        for (i64 t = 1; t <= L; ++t) {
            const i64 i = AT(c, t);
            const i64 f = (i64)v[t] - cu[i];         /* chain arc t -> t+1 (label t) */
            net[i] -= f;
            if (t < L) net[AT(c, t + 1)] += f; else sink_in += f;
            if (g + 1 < G) {
                const i64 cn = c + 1, fs = pen - ph[i];
                net[i] -= fs; net[AT(cn, t)] += fs;
                if (t > 1) {
                    net[i] -= dar[i]; net[AT(cn, t - 1)] += dar[i];
                    net[AT(cn, t)] -= dbr[i]; net[AT(c, t - 1)] += dbr[i];
                }
            }
            if (y + 1 < rows) {
                const i64 cn = c + G, fs = pen - pv[i];
                net[i] -= fs; net[AT(cn, t)] += fs;
                if (t > 1) {
                    net[i] -= dad[i]; net[AT(cn, t - 1)] += dad[i];
                    net[AT(cn, t)] -= dbd[i]; net[AT(c, t - 1)] += dbd[i];
                }
            }
        }
    }
    i64 nex = 0;
    for (i64 i = 0; i < N; ++i) {
        if (net[i] != e[i]) { report[3] = i; free(net); return 2; }
        nex += e[i] > 0;
    }
    free(net);
    report[0] = sink_in;
    report[5] = nex;
    if (sink_in != device_flow) return 3;
    /* 4. cut cost of the labeling */
    i64 en = 0;
    for (i64 c = 0; c < P; ++c) {
        const i64 g = c % G, y = c / G, a = labels[c];
        if (a < 0 || a >= m) { report[3] = c; return 4; }
        en += vol[c * m + a];
        if (g + 1 < G) en += pair_cost(a, labels[c + 1], pen, inh);
        if (y + 1 < rows) en += pair_cost(a, labels[c + G], pen, inh);
    }
    report[1] = en;
    if (en != sink_in) return 4;
    /* 5. residual reach from the excess nodes (the saturated source adds none) */
    uint8_t *seen = (uint8_t *)calloc((size_t)N, 1);
    int64_t *q = (int64_t *)malloc((size_t)(nex > 0 ? N : 1) * sizeof(int64_t));
    if (!seen || !q) { free(seen); free(q); return 6; }
    i64 qh = 0, qt = 0;
    for (i64 i = 0; i < N; ++i)
        if (e[i] > 0) { seen[i] = 1; q[qt++] = i; }
    int hit_sink = 0;
#define VISIT(j) do { const i64 j_ = (j); if (!seen[j_]) { seen[j_] = 1; q[qt++] = j_; } } while (0)
    while (qh < qt) {
        const i64 i = q[qh++], c = i / L, t = i % L + 1, g = c % G, y = c / G;
        if (cu[i] > 0) { if (t < L) VISIT(i + 1); else hit_sink = 1; }   /* chain up */
        if (t > 1) VISIT(i - 1);                                          /* chain down: uncuttable */
        if (g + 1 < G) {                                                  /* to the right neighbour */
            if (ph[i] > 0) VISIT(AT(c + 1, t));
            if (t > 1 && inh - dar[i] > 0) VISIT(AT(c + 1, t - 1));
            if (t < L && dbr[AT(c, t + 1)] > 0) VISIT(AT(c + 1, t + 1));   /* reverse of (c+1,t+1)->(c,t) */
        }
        if (g > 0) {                                                      /* to the left neighbour */
            const i64 cl = c - 1, il = AT(cl, t);
            if (2 * pen - ph[il] > 0) VISIT(il);
            if (t > 1 && inh - dbr[il] > 0) VISIT(AT(cl, t - 1));        /* (c,t) -> (c-1,t-1) */
            if (t < L && dar[AT(cl, t + 1)] > 0) VISIT(AT(cl, t + 1));   /* reverse of (c-1,t+1)->(c,t) */
        }
        if (y + 1 < rows) {
            if (pv[i] > 0) VISIT(AT(c + G, t));
            if (t > 1 && inh - dad[i] > 0) VISIT(AT(c + G, t - 1));
            if (t < L && dbd[AT(c, t + 1)] > 0) VISIT(AT(c + G, t + 1));
        }
        if (y > 0) {
            const i64 cu_ = c - G, iu = AT(cu_, t);
            if (2 * pen - pv[iu] > 0) VISIT(iu);
            if (t > 1 && inh - dbd[iu] > 0) VISIT(AT(cu_, t - 1));
            if (t < L && dad[AT(cu_, t + 1)] > 0) VISIT(AT(cu_, t + 1));
        }
    }
#undef VISIT
    report[2] = qt;
    i64 bad = 0, first = -1;
    for (i64 c = 0; c < P; ++c) {
        i64 k = 0;
        while (k < L && seen[c * L + k]) ++k;       /* reach is prefix-closed (chain down is uncuttable) */
        int mism = k != labels[c];
        for (i64 t = k; t < L && !mism; ++t) mism = seen[c * L + t];
        if (mism) { ++bad; if (first < 0) first = c; }
    }
    free(seen);
    free(q);
    report[4] = bad;
    if (hit_sink || bad) { report[3] = hit_sink ? -2 : first; return 5; }
    return 0;
#undef AT
}
