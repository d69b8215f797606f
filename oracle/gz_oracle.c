/*
 * gz_oracle.c -- CPU restatement of the reference `gazecut` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the shipped package links or calls
 * this file: it is the parity checker used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg.
 *
 * Parity pinned against the reference's golden vectors and against outputs of
 * the reference itself (tests/golden/, produced by oracle/make_golden.py from
 * /root/reference/pkg/src/gazecut), see tests/test_oracle.py.
 *
 * Every routine cites the reference function it restates (paths relative to
 * /root/reference/pkg/src/gazecut/).  Integer widths follow the reference:
 * capacities/residuals/excess int64, arc ids int32, heights int32.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GZO_UNCUTTABLE ((int64_t)1 << 56) /* energy.py:34 */
#define GZO_BIG ((int64_t)1 << 62)        /* maxflow.py:31 */
#define GZO_SRC ((int64_t)-1)             /* flownet.py:37 */
#define GZO_SNK ((int64_t)-2)             /* flownet.py:38 */

static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* ------------------------------------------------------------------------ */
/* energy.py:83-114 sad_volume with geometry.py:325-335 site_columns.         */
/* left/right: (h, w, channels) uint8 row-major.  width = the image width the */
/* cuboid was built for (clamp range).  vol: (y_extent, g_extent, m) int64.   */
void gzo_sad_volume(const uint8_t *left, const uint8_t *right, int h, int w, int channels,
                    int width, int g_min, int g_extent, int y_min, int y_extent, int d_min, int m,
                    int64_t *vol)
{
    (void)h;
    for (int y = 0; y < y_extent; ++y) {
        const uint8_t *lrow = left + (size_t)(y_min + y) * w * channels;
        const uint8_t *rrow = right + (size_t)(y_min + y) * w * channels;
        for (int gi = 0; gi < g_extent; ++gi) {
            int64_t g = (int64_t)g_min + gi;
            int64_t *out = vol + ((size_t)y * g_extent + gi) * m;
            for (int k = 0; k < m; ++k) {
                int64_t d = (int64_t)d_min + k;
                int64_t xr = clampi(g + d, 0, width - 1);
                int64_t xl = clampi((int64_t)(width - 1) + g - d, 0, width - 1);
                int64_t acc = 0;
                for (int c = 0; c < channels; ++c) {
                    int a = lrow[xl * channels + c], b = rrow[xr * channels + c];
                    acc += a > b ? a - b : b - a;
                }
                out[k] = acc;
            }
        }
    }
}

/* energy.py:129-155 total_energy (caller validated shapes/ranges). */
int64_t gzo_total_energy(const int32_t *lab, const int64_t *vol, int rows, int cols, int m,
                         int64_t penalty, int64_t inhibit, int hard)
{
    int64_t data = 0, smooth = 0;
    for (int y = 0; y < rows; ++y)
        for (int g = 0; g < cols; ++g)
            data += vol[((size_t)y * cols + g) * m + lab[y * cols + g]];
    for (int dir = 0; dir < 2; ++dir) {
        for (int y = 0; y < rows - (dir == 1); ++y) {
            for (int g = 0; g < cols - (dir == 0); ++g) {
                int64_t a = lab[y * cols + g];
                int64_t b = dir == 0 ? lab[y * cols + g + 1] : lab[(y + 1) * cols + g];
                int64_t dl = a > b ? a - b : b - a;
                if (hard && dl > 1) return GZO_UNCUTTABLE;
                smooth += penalty * dl + inhibit * (dl > 1 ? dl - 1 : 0);
            }
        }
    }
    return data + smooth;
}

/* ------------------------------------------------------------------------ */
/* flownet.py:41-89 FlowNetwork, CSR form.                                    */
typedef struct {
    int64_t n_nodes, source, sink, n_arcs, const_offset;
    int64_t rows, cols, m, n_chain; /* rows == 0: generic network */
    int64_t *first_out;             /* n+1 */
    int32_t *head, *rev;            /* n_arcs */
    int64_t *cap, *resid;           /* n_arcs */
    int32_t *lo, *hi;               /* sites */
    int64_t *node_base;             /* sites+1 */
    int32_t *chain_arcs;            /* n_chain */
    int64_t *chain_base;            /* sites+1 */
} gzo_net;

void gzo_free(gzo_net *net)
{
    if (!net) return;
    free(net->first_out); free(net->head); free(net->rev); free(net->cap); free(net->resid);
    free(net->lo); free(net->hi); free(net->node_base); free(net->chain_arcs); free(net->chain_base);
    free(net);
}

/* flownet.py:92-99 _chain_node */
static inline int64_t chain_node(int64_t base, int64_t l0, int64_t h0, int64_t t)
{
    if (t <= l0) return GZO_SRC;
    if (t > h0) return GZO_SNK;
    return base + (t - l0 - 1);
}

typedef struct { int64_t *pu, *pv, *pc, *prc, *chain_pairs; int fill; } emit_buf;

/* flownet.py:102-181 _emit: same fixed enumeration order (site row-major;  */
/* chain arcs by label; per forward neighbour same-level then diagonals).    */
static void emit(const int64_t *vol, int64_t rows, int64_t cols, int64_t m, const int32_t *lo,
                 const int32_t *hi, int64_t penalty, int64_t inhibit_cap, const int64_t *node_base,
                 emit_buf *eb, int64_t *n_out, int64_t *nchain_out, int64_t *offset_out)
{
    int64_t n = 0, nchain = 0, offset = 0;
#define EMIT(A, B, C, RC)                                                                          \
    do {                                                                                           \
        if (eb->fill) { eb->pu[n] = (A); eb->pv[n] = (B); eb->pc[n] = (C); eb->prc[n] = (RC); }    \
        ++n;                                                                                       \
    } while (0)
    for (int64_t y = 0; y < rows; ++y) {
        for (int64_t g = 0; g < cols; ++g) {
            int64_t s = y * cols + g, l0 = lo[s], h0 = hi[s], base = node_base[s];
            for (int64_t lab = l0; lab <= h0; ++lab) {
                int64_t a = chain_node(base, l0, h0, lab), b = chain_node(base, l0, h0, lab + 1);
                int64_t c = vol[s * m + lab];
                if (a == GZO_SRC && b == GZO_SNK) {
                    offset += c;
                } else {
                    if (eb->fill) eb->chain_pairs[nchain] = n;
                    EMIT(a, b, c, GZO_UNCUTTABLE);
                    ++nchain;
                }
            }
            for (int nb = 0; nb < 2; ++nb) {
                int64_t yn = nb == 0 ? y : y + 1, gn = nb == 0 ? g + 1 : g;
                if (yn >= rows || gn >= cols) continue;
                int64_t sn = yn * cols + gn, ln = lo[sn], hn = hi[sn], basen = node_base[sn];
                for (int64_t t = 1; t < m; ++t) {
                    int64_t a = chain_node(base, l0, h0, t), b = chain_node(basen, ln, hn, t);
                    if (a != b) {
                        if (a == GZO_SNK || b == GZO_SRC) { int64_t tmp = a; a = b; b = tmp; }
                        if (a == GZO_SRC && b == GZO_SNK) offset += penalty;
                        else EMIT(a, b, penalty, penalty);
                    }
                    for (int dir = 0; dir < 2; ++dir) {
                        if (dir == 0) { a = chain_node(base, l0, h0, t); b = chain_node(basen, ln, hn, t - 1); }
                        else { a = chain_node(basen, ln, hn, t); b = chain_node(base, l0, h0, t - 1); }
                        if (a == GZO_SNK || b == GZO_SRC || a == b) continue;
                        if (a == GZO_SRC && b == GZO_SNK) offset += inhibit_cap;
                        else EMIT(a, b, inhibit_cap, 0);
                    }
                }
            }
        }
    }
#undef EMIT
    *n_out = n; *nchain_out = nchain; *offset_out = offset;
}

/* flownet.py:184-222 _pairs_to_csr.  Returns pair_arc (malloc'd). */
static int32_t *pairs_to_csr(gzo_net *net, int64_t npairs, int64_t *pu, int64_t *pv, const int64_t *pc,
                             const int64_t *prc)
{
    int64_t n = net->n_nodes;
    int64_t *deg = calloc((size_t)n, sizeof(int64_t));
    for (int64_t i = 0; i < npairs; ++i) {
        int64_t u = pu[i], v = pv[i];
        if (u < 0) u = u == GZO_SRC ? net->source : net->sink;
        if (v < 0) v = v == GZO_SRC ? net->source : net->sink;
        pu[i] = u; pv[i] = v;
        deg[u]++; deg[v]++;
    }
    net->first_out = malloc((size_t)(n + 1) * sizeof(int64_t));
    net->first_out[0] = 0;
    for (int64_t u = 0; u < n; ++u) net->first_out[u + 1] = net->first_out[u] + deg[u];
    int64_t *cursor = deg; /* reuse */
    for (int64_t u = 0; u < n; ++u) cursor[u] = net->first_out[u];
    net->n_arcs = 2 * npairs;
    size_t na = (size_t)(net->n_arcs ? net->n_arcs : 1);
    net->head = malloc(na * sizeof(int32_t));
    net->rev = malloc(na * sizeof(int32_t));
    net->cap = malloc(na * sizeof(int64_t));
    net->resid = malloc(na * sizeof(int64_t));
    int32_t *pair_arc = malloc((size_t)(npairs ? npairs : 1) * sizeof(int32_t));
    for (int64_t i = 0; i < npairs; ++i) {
        int64_t u = pu[i], v = pv[i];
        int64_t au = cursor[u]++, av = cursor[v]++;
        net->head[au] = (int32_t)v; net->head[av] = (int32_t)u;
        net->cap[au] = pc[i]; net->cap[av] = prc[i];
        net->rev[au] = (int32_t)av; net->rev[av] = (int32_t)au;
        pair_arc[i] = (int32_t)au;
    }
    memcpy(net->resid, net->cap, na * sizeof(int64_t));
    free(deg);
    return pair_arc;
}

/* flownet.py:233-296 build_network.  lo/hi NULL = full windows           */
/* (flownet.py:225-230).  Returns NULL on bad windows (caller raises).    */
gzo_net *gzo_build_network(const int64_t *vol, int64_t rows, int64_t cols, int64_t m, int64_t penalty,
                           int64_t inhibit_cap, const int32_t *lo_in, const int32_t *hi_in)
{
    int64_t sites = rows * cols;
    gzo_net *net = calloc(1, sizeof(gzo_net));
    net->rows = rows; net->cols = cols; net->m = m;
    net->lo = malloc((size_t)(sites ? sites : 1) * sizeof(int32_t));
    net->hi = malloc((size_t)(sites ? sites : 1) * sizeof(int32_t));
    for (int64_t s = 0; s < sites; ++s) {
        net->lo[s] = lo_in ? lo_in[s] : 0;
        net->hi[s] = hi_in ? hi_in[s] : (int32_t)(m - 1);
        if (net->lo[s] < 0 || net->hi[s] >= m || net->lo[s] > net->hi[s]) { gzo_free(net); return NULL; }
    }
    net->node_base = malloc((size_t)(sites + 1) * sizeof(int64_t));
    net->node_base[0] = 0;
    for (int64_t s = 0; s < sites; ++s) net->node_base[s + 1] = net->node_base[s] + (net->hi[s] - net->lo[s]);
    int64_t n_int = net->node_base[sites];
    net->n_nodes = n_int + 2; net->source = n_int; net->sink = n_int + 1;

    emit_buf eb = {0};
    int64_t npairs, nchain, offset;
    emit(vol, rows, cols, m, net->lo, net->hi, penalty, inhibit_cap, net->node_base, &eb, &npairs, &nchain, &offset);
    size_t np1 = (size_t)(npairs ? npairs : 1);
    eb.pu = malloc(np1 * 8); eb.pv = malloc(np1 * 8); eb.pc = malloc(np1 * 8); eb.prc = malloc(np1 * 8);
    eb.chain_pairs = malloc((size_t)(nchain ? nchain : 1) * 8);
    eb.fill = 1;
    emit(vol, rows, cols, m, net->lo, net->hi, penalty, inhibit_cap, net->node_base, &eb, &npairs, &nchain, &offset);
    int32_t *pair_arc = pairs_to_csr(net, npairs, eb.pu, eb.pv, eb.pc, eb.prc);
    net->n_chain = nchain;
    net->chain_arcs = malloc((size_t)(nchain ? nchain : 1) * sizeof(int32_t));
    for (int64_t i = 0; i < nchain; ++i) net->chain_arcs[i] = pair_arc[eb.chain_pairs[i]];
    net->chain_base = malloc((size_t)(sites + 1) * sizeof(int64_t));
    net->chain_base[0] = 0;
    for (int64_t s = 0; s < sites; ++s) {
        int64_t wdt = net->hi[s] - net->lo[s];
        net->chain_base[s + 1] = net->chain_base[s] + (wdt > 0 ? wdt + 1 : 0);
    }
    net->const_offset = offset;
    free(eb.pu); free(eb.pv); free(eb.pc); free(eb.prc); free(eb.chain_pairs); free(pair_arc);
    return net;
}

/* flownet.py:325-353 network_from_arcs (caller validated ranges). */
gzo_net *gzo_network_from_arcs(int64_t n_nodes, int64_t source, int64_t sink, int64_t npairs,
                               const int64_t *pu_in, const int64_t *pv_in, const int64_t *pc,
                               const int64_t *prc)
{
    gzo_net *net = calloc(1, sizeof(gzo_net));
    net->n_nodes = n_nodes; net->source = source; net->sink = sink;
    size_t np1 = (size_t)(npairs ? npairs : 1);
    int64_t *pu = malloc(np1 * 8), *pv = malloc(np1 * 8);
    memcpy(pu, pu_in, (size_t)npairs * 8); memcpy(pv, pv_in, (size_t)npairs * 8);
    free(pairs_to_csr(net, npairs, pu, pv, pc, prc));
    free(pu); free(pv);
    return net;
}

void gzo_reset(gzo_net *net) { memcpy(net->resid, net->cap, (size_t)net->n_arcs * sizeof(int64_t)); }

/* flownet.py:356-382 node_blocks / _fill_blocks */
void gzo_node_blocks(const gzo_net *net, int64_t block, int32_t *out)
{
    int64_t gb = (net->cols + block - 1) / block, mb = (net->m + block - 1) / block;
    memset(out, 0, (size_t)net->n_nodes * sizeof(int32_t));
    for (int64_t y = 0; y < net->rows; ++y)
        for (int64_t g = 0; g < net->cols; ++g) {
            int64_t s = y * net->cols + g;
            int64_t yb = (y / block) * gb * mb + (g / block) * mb;
            for (int64_t j = 0; j < net->node_base[s + 1] - net->node_base[s]; ++j) {
                int64_t t = net->lo[s] + 1 + j;
                out[net->node_base[s] + j] = (int32_t)(yb + t / block);
            }
        }
}

/* ------------------------------------------------------------------------ */
/* maxflow.py:59-131 _dinic */
int64_t gzo_maxflow_dinic(gzo_net *net)
{
    int64_t n = net->n_nodes, source = net->source, sink = net->sink;
    const int64_t *first_out = net->first_out; const int32_t *head = net->head, *rev = net->rev;
    int64_t *resid = net->resid;
    int32_t *level = malloc((size_t)n * 4), *queue = malloc((size_t)n * 4), *nodes = malloc((size_t)(n + 1) * 4);
    int64_t *cur = malloc((size_t)n * 8), *path = malloc((size_t)(n + 1) * 8);
    int64_t total = 0;
    for (;;) {
        for (int64_t i = 0; i < n; ++i) level[i] = -1;
        level[source] = 0; queue[0] = (int32_t)source;
        int64_t qh = 0, qt = 1;
        while (qh < qt) {
            int64_t u = queue[qh++];
            for (int64_t a = first_out[u]; a < first_out[u + 1]; ++a)
                if (resid[a] > 0) { int64_t v = head[a]; if (level[v] < 0) { level[v] = level[u] + 1; queue[qt++] = (int32_t)v; } }
        }
        if (level[sink] < 0) break;
        for (int64_t u = 0; u < n; ++u) cur[u] = first_out[u];
        int64_t top = 0; nodes[0] = (int32_t)source;
        int64_t u = source;
        for (;;) {
            if (u == sink) {
                int64_t bott = GZO_BIG;
                for (int64_t i = 0; i < top; ++i) if (resid[path[i]] < bott) bott = resid[path[i]];
                for (int64_t i = 0; i < top; ++i) { int64_t a = path[i]; resid[a] -= bott; resid[rev[a]] += bott; }
                total += bott;
                int64_t newtop = top;
                for (int64_t i = 0; i < top; ++i) if (resid[path[i]] == 0) { newtop = i; break; }
                top = newtop; u = nodes[top];
                continue;
            }
            int advanced = 0;
            while (cur[u] < first_out[u + 1]) {
                int64_t a = cur[u], v = head[a];
                if (resid[a] > 0 && level[v] == level[u] + 1) {
                    path[top] = a; nodes[top + 1] = (int32_t)v; ++top; u = v; advanced = 1; break;
                }
                cur[u]++;
            }
            if (advanced) continue;
            level[u] = -1;
            if (u == source) break;
            --top; u = nodes[top]; cur[u]++;
        }
    }
    free(level); free(queue); free(nodes); free(cur); free(path);
    return total;
}

/* maxflow.py:138-170 _global_relabel */
static void global_relabel(const gzo_net *net, int32_t *h, int32_t *queue)
{
    int64_t n = net->n_nodes, source = net->source, sink = net->sink;
    int32_t hmax = (int32_t)(2 * n);
    for (int64_t u = 0; u < n; ++u) h[u] = hmax;
    h[sink] = 0; queue[0] = (int32_t)sink;
    int64_t qh = 0, qt = 1;
    while (qh < qt) {
        int64_t w = queue[qh++];
        for (int64_t a = net->first_out[w]; a < net->first_out[w + 1]; ++a) {
            int64_t v = net->head[a];
            if (v != source && h[v] == hmax && net->resid[net->rev[a]] > 0) { h[v] = h[w] + 1; queue[qt++] = (int32_t)v; }
        }
    }
    h[source] = (int32_t)n; queue[0] = (int32_t)source; qh = 0; qt = 1;
    while (qh < qt) {
        int64_t w = queue[qh++];
        for (int64_t a = net->first_out[w]; a < net->first_out[w + 1]; ++a) {
            int64_t v = net->head[a];
            if (v != sink && h[v] == hmax && net->resid[net->rev[a]] > 0) { h[v] = h[w] + 1; queue[qt++] = (int32_t)v; }
        }
    }
}

/* maxflow.py:173-180 _saturate_source */
static void saturate_source(gzo_net *net, int64_t *excess)
{
    for (int64_t a = net->first_out[net->source]; a < net->first_out[net->source + 1]; ++a) {
        int64_t f = net->resid[a];
        if (f > 0) { net->resid[a] = 0; net->resid[net->rev[a]] += f; excess[net->head[a]] += f; }
    }
}

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return x < y ? -1 : (x > y);
}

/* maxflow.py:183-250 _discharge_rounds (order_key NULL = plain FIFO). */
static int64_t discharge_rounds(gzo_net *net, int32_t *h, int64_t *excess, int64_t *cur, int32_t *queue,
                                int32_t *nextq, uint8_t *in_queue, int64_t nq, int rounds,
                                const int32_t *order_key, int64_t *keys, int64_t *pushes_out,
                                int64_t *relabels_out)
{
    int64_t n = net->n_nodes, source = net->source, sink = net->sink;
    const int64_t *first_out = net->first_out; const int32_t *head = net->head, *rev = net->rev;
    int64_t *resid = net->resid;
    int32_t hmax = (int32_t)(2 * n);
    int64_t pushes = 0, relabels = 0;
    for (int r = 0; r < rounds; ++r) {
        if (nq == 0) break;
        if (order_key) {
            /* key = order_key[q]*n + q is unique, so any sort reproduces argsort */
            for (int64_t i = 0; i < nq; ++i) keys[i] = (int64_t)order_key[queue[i]] * n + queue[i];
            qsort(keys, (size_t)nq, sizeof(int64_t), cmp_i64);
            for (int64_t i = 0; i < nq; ++i) queue[i] = (int32_t)(keys[i] % n);
        }
        int64_t nn = 0;
        for (int64_t qi = 0; qi < nq; ++qi) {
            int64_t u = queue[qi];
            in_queue[u] = 0;
            if (excess[u] <= 0 || h[u] >= hmax) continue;
            while (excess[u] > 0 && h[u] < hmax) {
                if (cur[u] >= first_out[u + 1]) {
                    int32_t newh = hmax;
                    for (int64_t a = first_out[u]; a < first_out[u + 1]; ++a)
                        if (resid[a] > 0 && h[head[a]] + 1 < newh) newh = h[head[a]] + 1;
                    h[u] = newh; cur[u] = first_out[u]; ++relabels;
                    if (newh >= hmax) break;
                    continue;
                }
                int64_t a = cur[u], v = head[a];
                if (resid[a] > 0 && h[u] == h[v] + 1) {
                    int64_t f = excess[u] < resid[a] ? excess[u] : resid[a];
                    resid[a] -= f; resid[rev[a]] += f; excess[u] -= f; excess[v] += f; ++pushes;
                    if (v != source && v != sink && in_queue[v] == 0 && h[v] < hmax) {
                        nextq[nn++] = (int32_t)v; in_queue[v] = 1;
                    }
                } else {
                    cur[u]++;
                }
            }
            if (excess[u] > 0 && h[u] < hmax && in_queue[u] == 0) { nextq[nn++] = (int32_t)u; in_queue[u] = 1; }
        }
        memcpy(queue, nextq, (size_t)nn * sizeof(int32_t));
        nq = nn;
    }
    *pushes_out += pushes; *relabels_out += relabels;
    return nq;
}

/* maxflow.py:253-264 _collect_active */
static int64_t collect_active(const gzo_net *net, const int64_t *excess, const int32_t *h, int32_t *queue,
                              uint8_t *in_queue)
{
    int64_t n = net->n_nodes, nq = 0;
    int32_t hmax = (int32_t)(2 * n);
    memset(in_queue, 0, (size_t)n);
    for (int64_t u = 0; u < n; ++u)
        if (u != net->source && u != net->sink && excess[u] > 0 && h[u] < hmax) { queue[nq++] = (int32_t)u; in_queue[u] = 1; }
    return nq;
}

/* maxflow.py:287-304 _chain_presaturate */
int64_t gzo_chain_presaturate(gzo_net *net)
{
    if (net->rows == 0) return 0;
    int64_t total = 0, nsites = net->rows * net->cols;
    for (int64_t s = 0; s < nsites; ++s) {
        int64_t a0 = net->chain_base[s], a1 = net->chain_base[s + 1];
        if (a1 <= a0) continue;
        int64_t f = GZO_BIG;
        for (int64_t i = a0; i < a1; ++i) if (net->resid[net->chain_arcs[i]] < f) f = net->resid[net->chain_arcs[i]];
        if (f > 0) {
            for (int64_t i = a0; i < a1; ++i) { int32_t a = net->chain_arcs[i]; net->resid[a] -= f; net->resid[net->rev[a]] += f; }
            total += f;
        }
    }
    return total;
}

typedef struct {
    int64_t flow, presaturated, pushes, relabels, stranded;
    int32_t sweeps, converged;
} gzo_pr_stats;

/* maxflow.py:403-478 maxflow_push_relabel (max_sweeps < 0: uncapped;   */
/* block <= 0: unordered FIFO).                                          */
int gzo_maxflow_push_relabel(gzo_net *net, int rounds_per_sweep, int max_sweeps, int block, int presaturate,
                             gzo_pr_stats *st)
{
    if (rounds_per_sweep < 1) return -1;
    int64_t n = net->n_nodes;
    int64_t base_flow = presaturate ? gzo_chain_presaturate(net) : 0;
    int32_t *order_key = NULL;
    int64_t *keys = NULL;
    if (block > 0) {
        if (net->rows == 0) return -2;
        order_key = malloc((size_t)n * 4);
        gzo_node_blocks(net, block, order_key);
        keys = malloc((size_t)n * 8);
    }
    int32_t *h = calloc((size_t)n, 4), *queue = malloc((size_t)n * 4), *nextq = malloc((size_t)n * 4);
    int64_t *excess = calloc((size_t)n, 8), *cur = calloc((size_t)n, 8);
    uint8_t *in_queue = calloc((size_t)n, 1);
    saturate_source(net, excess);
    int32_t sweeps = 0, converged = 1;
    int64_t pushes = 0, relabels = 0;
    for (;;) {
        global_relabel(net, h, queue);
        int64_t nq = collect_active(net, excess, h, queue, in_queue);
        if (nq == 0) break;
        if (max_sweeps >= 0 && sweeps >= max_sweeps) { converged = 0; break; }
        for (int64_t u = 0; u < n; ++u) cur[u] = net->first_out[u];
        discharge_rounds(net, h, excess, cur, queue, nextq, in_queue, nq, rounds_per_sweep, order_key, keys,
                         &pushes, &relabels);
        ++sweeps;
    }
    st->flow = base_flow + excess[net->sink];
    st->presaturated = base_flow;
    st->pushes = pushes; st->relabels = relabels;
    st->sweeps = sweeps; st->converged = converged;
    int64_t stranded = 0;
    for (int64_t u = 0; u < n; ++u) if (excess[u] > 0 && u != net->source && u != net->sink) ++stranded;
    st->stranded = stranded;
    free(order_key); free(keys); free(h); free(queue); free(nextq); free(excess); free(cur); free(in_queue);
    return 0;
}

/* maxflow.py:267-284 _bfs_source_side */
void gzo_source_side(const gzo_net *net, uint8_t *side)
{
    int64_t n = net->n_nodes;
    int32_t *queue = malloc((size_t)n * 4);
    memset(side, 0, (size_t)n);
    side[net->source] = 1; queue[0] = (int32_t)net->source;
    int64_t qh = 0, qt = 1;
    while (qh < qt) {
        int64_t u = queue[qh++];
        for (int64_t a = net->first_out[u]; a < net->first_out[u + 1]; ++a)
            if (net->resid[a] > 0) { int64_t v = net->head[a]; if (!side[v]) { side[v] = 1; queue[qt++] = (int32_t)v; } }
    }
    free(queue);
}

/* maxflow.py:307-320 _extract_labels; returns the chains-cut-twice count. */
int64_t gzo_extract_labels(const gzo_net *net, const uint8_t *side, int32_t *labels)
{
    int64_t bad = 0, nsites = net->rows * net->cols;
    for (int64_t s = 0; s < nsites; ++s) {
        int64_t count = 0; int prev = 1;
        for (int64_t i = net->node_base[s]; i < net->node_base[s + 1]; ++i) {
            if (side[i]) { if (!prev) ++bad; ++count; }
            prev = side[i];
        }
        labels[s] = (int32_t)(net->lo[s] + count);
    }
    return bad;
}

/* maxflow.py:323-334 _conservation_violations */
int64_t gzo_conservation_violations(const gzo_net *net)
{
    int64_t bad = 0;
    for (int64_t u = 0; u < net->n_nodes; ++u) {
        if (u == net->source || u == net->sink) continue;
        int64_t s = 0;
        for (int64_t a = net->first_out[u]; a < net->first_out[u + 1]; ++a) s += net->cap[a] - net->resid[a];
        if (s != 0) ++bad;
    }
    return bad;
}
