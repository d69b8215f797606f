// gz_csr.cuh -- explicit-network side of the C ABI.  Included at the end of
// gz_solver.cu (same translation unit: Workspace, carve, solve_planar).
//
//  * gz_export_arcs   the implicit device graph as arc pairs in the
//                     reference's emission order (flownet.py:102-181 _emit),
//                     capacities read from the solver's initialised state
//                     planes (the device graph itself, not a host model).  The
//                     Python side turns the pairs into CSR exactly as
//                     flownet.py:184-222 _pairs_to_csr does.
//  * gz_export_state  one state plane of the last solve in a workspace
//                     (residuals, pair flows, excess, heights) as int32
//                     (sites, m-1): the input of the optimality certificate
//                     (oracle/gz_certify.c).
//  * gz_maxflow_csr   push-relabel with global relabeling on an explicit CSR
//                     network (flownet.py:325-353 network_from_arcs networks,
//                     materialised grid networks): maxflow.py:403-478 with the
//                     reference's height convention (sink distance, n + source
//                     distance, 2n parked), phases 1 and 2, so the residual
//                     left behind is a maximum FLOW (no excess) like the
//                     reference's.  Synchronous pulses on a cooperative grid.
//  * gz_chain_presaturate_csr, gz_conservation_violations_csr
//                     maxflow.py:287-304 and 323-334 on the same CSR arrays.

#include <cub/device/device_scan.cuh>

namespace {

// ---------------------------------------------------------------------------
// implicit graph -> arc pairs

struct ExportArgs {
    const int32_t *vol, *cu, *ph, *pv, *dar, *dbr, *dad, *dbd;   // [site][LPT] device state
    const int32_t *lo, *hi;                                      // windows or null (full)
    const long long *node_base;                                  // [P + 1]
    long long *cnt;                                              // [P + 1] pairs per site
    const long long *offs;                                       // [P + 1] exclusive scan of cnt
    long long *pu, *pv_, *pc, *prc;                              // [npairs] (fill pass)
    unsigned long long *offset_acc;                              // folded source->sink capacity
    int rows, cols, m, LPT, pen, icap_dev, hard;
    long long src, snk;
};

__device__ __forceinline__ long long x_node(const ExportArgs &x, int s, int lo, int hi, int t) {
    if (t <= lo) return x.src;   // flownet.py:92-99 _chain_node
    if (t > hi) return x.snk;
    return x.node_base[s] + (t - lo - 1);
}

// One thread per site, the emission order of flownet.py:115-180: chain arcs by
// label, then per forward neighbour (right, down) and level t: the same-level
// pair, then both inhibit diagonals.
// MODE 0: capacities of the initialised graph (cap, rcap); MODE 1: residuals of
// the state a solve left (resid forward, resid reverse).  Arcs out of the
// source are saturated at initialisation and a solve never pushes into source
// positions (gz_chain.cuh), so in MODE 1 they read (0, cap + rcap).
template <bool FILL, int MODE = 0>
__global__ void k_export_arcs(ExportArgs x) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int P = x.rows * x.cols;
    if (s >= P) return;
    const int y = s / x.cols, g = s - y * x.cols;
    const int l0 = x.lo ? x.lo[s] : 0, h0 = x.hi ? x.hi[s] : x.m - 1;
    const size_t row = (size_t)s * x.LPT;
    long long n = 0, k = FILL ? x.offs[s] : 0;
    unsigned long long off = 0;
    const unsigned long long UNC = (unsigned long long)gz::UNCUTTABLE;
    auto emit = [&](long long a, long long b, long long c, long long rc) {
        if (MODE == 1 && a == x.src) { rc += c; c = 0; }
        if (FILL) {
            x.pu[k] = a; x.pv_[k] = b; x.pc[k] = c; x.prc[k] = rc;
            ++k;
        }
        ++n;
    };
    for (int lab = l0; lab <= h0; ++lab) {
        const long long a = x_node(x, s, l0, h0, lab), b = x_node(x, s, l0, h0, lab + 1);
        // chain arc lab -> lab+1: the device keeps it as the chain residual of
        // position lab (cu, initialised to the data cost vol[lab]); the arc out of
        // position 0 has no residual slot and is read from the data-term plane
        const long long cap = lab == 0 ? x.vol[row] : x.cu[row + lab - 1];
        if (a == x.src && b == x.snk) off += (unsigned long long)cap;
        else if (MODE == 0 || a == x.src) emit(a, b, cap, (long long)UNC);
        else emit(a, b, cap, (long long)UNC + (x.vol[row + lab] - cap));   // cu = residual; flow = vol - cu
    }
    for (int nb = 0; nb < 2; ++nb) {
        const int yn = nb == 0 ? y : y + 1, gn = nb == 0 ? g + 1 : g;
        if (yn >= x.rows || gn >= x.cols) continue;
        const int sn = yn * x.cols + gn;
        const int ln = x.lo ? x.lo[sn] : 0, hn = x.hi ? x.hi[sn] : x.m - 1;
        const int32_t *pair = nb == 0 ? x.ph : x.pv;       // same-level residual s -> sn
        const int32_t *dfw = nb == 0 ? x.dar : x.dad;      // flow (s,t) -> (sn,t-1)
        const int32_t *dbk = nb == 0 ? x.dbr : x.dbd;      // flow (sn,t) -> (s,t-1)
        for (int t = 1; t < x.m; ++t) {
            const size_t I = row + t - 1;
            long long a = x_node(x, s, l0, h0, t), b = x_node(x, sn, ln, hn, t);
            if (a != b) {
                const long long r = pair[I], r2 = 2LL * x.pen - r;   // residuals s->sn, sn->s
                long long c = r, rc = r2;
                if (a == x.snk || b == x.src) { long long q = a; a = b; b = q; c = r2; rc = r; }
                if (a == x.src && b == x.snk) off += (unsigned long long)c;
                else emit(a, b, c, rc);
            }
            for (int dir = 0; dir < 2; ++dir) {
                const long long u = dir == 0 ? x_node(x, s, l0, h0, t) : x_node(x, sn, ln, hn, t);
                const long long v = dir == 0 ? x_node(x, sn, ln, hn, t - 1) : x_node(x, s, l0, h0, t - 1);
                if (u == x.snk || v == x.src || u == v) continue;
                const long long f = (dir == 0 ? dfw : dbk)[I];
                // inhibit capacity: the device's finite stand-in (hard mode) maps back
                // to the reference's UNCUTTABLE (gz_graph.cuh)
                const long long c = x.hard ? (long long)UNC - f : (long long)x.icap_dev - f;
                if (u == x.src && v == x.snk) off += (unsigned long long)c;
                else emit(u, v, c, f);
            }
        }
    }
    if (!FILL) {
        x.cnt[s] = n;
        if (off) atomicAdd(x.offset_acc, off);
    }
}

__global__ void k_window_widths(const int32_t *lo, const int32_t *hi, int P, int m, long long *w) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s > P) return;
    w[s] = s == P ? 0 : (long long)((hi ? hi[s] : m - 1) - (lo ? lo[s] : 0));
}

// exclusive scan of n int64 values in place (cub), temp storage from the stream's pool
int scan_exclusive(long long *d, long long n, cudaStream_t s) {
    size_t tmp = 0;
    if (cub::DeviceScan::ExclusiveSum(nullptr, tmp, d, d, (int)n, s) != cudaSuccess) return GZ_ERR_CUDA;
    void *t = nullptr;
    CK(cudaMallocAsync(&t, tmp ? tmp : 16, s));
    const cudaError_t e = cub::DeviceScan::ExclusiveSum(t, tmp, d, d, (int)n, s);
    cudaFreeAsync(t, s);
    return e == cudaSuccess ? GZ_OK : GZ_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// one state plane of a finished solve -> int32 (sites, m - 1)

__global__ void k_export_plane(const int32_t *a, const int32_t *b, const int32_t *c, int P, int LPT, int L,
                               int32_t *out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)P * L) return;
    const long long s = i / L, t = i - s * L;
    const size_t I = (size_t)s * LPT + t;
    int32_t v = a[I];
    if (b) v += b[I] + c[I];   // excess: merged value plus both inbox buffers
    out[i] = v;
}

// ---------------------------------------------------------------------------
// generic CSR push-relabel (maxflow.py:403-478), cooperative grid

struct CsrArgs {
    long long n, source, sink;
    const long long *first_out;
    const int32_t *head, *rev;
    const long long *cap;
    long long *resid, *excess, *ein;
    int *h, *pushed;
    unsigned char *side;
    unsigned long long *ctr;   // 0 changed flags x3, 3 active x3, 6 pushes, 7 relabels, 8 sweeps,
                               // 9 converged, 10 stranded, 11 pulses
    int rounds, max_sweeps;    // max_sweeps < 0: uncapped
};

constexpr int CSR_CTR = 16;

__device__ __forceinline__ bool grid_any(cg::grid_group &grid, unsigned long long *slots, int &rot, bool mine) {
    // rotating slots: slot rot is read after the barrier; slot rot+1 is cleared
    // for the next call (every thread has passed its last read of it)
    if (mine) slots[rot] = 1ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) slots[(rot + 1) % 3] = 0ull;
    grid.sync();
    const bool r = ((volatile unsigned long long *)slots)[rot] != 0ull;
    rot = (rot + 1) % 3;
    return r;
}

__global__ void __launch_bounds__(256) k_csr_solve(CsrArgs a) {
    cg::grid_group grid = cg::this_grid();
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long n = a.n, hmax = 2 * n;
    int rot = 0;
    long long pushes = 0, relabels = 0;
    // excess of the flow already in the network (a presaturated chain, or the
    // preflow a grid solve left behind): minus the net outflow cap - resid
    for (long long v = tid; v < n; v += stride) {
        long long out = 0;
        for (long long q = a.first_out[v]; q < a.first_out[v + 1]; ++q) out += a.cap[q] - a.resid[q];
        a.excess[v] = -out;
    }
    grid.sync();
    // maxflow.py:173-180 _saturate_source
    for (long long q = a.first_out[a.source] + tid; q < a.first_out[a.source + 1]; q += stride) {
        const long long f = a.resid[q];
        if (f > 0) {
            a.resid[q] = 0;
            atomicAdd((unsigned long long *)&a.resid[a.rev[q]], (unsigned long long)f);
            atomicAdd((unsigned long long *)&a.excess[a.head[q]], (unsigned long long)f);
        }
    }
    grid.sync();
    int sweeps = 0, pulses = 0, converged = 1;
    for (;;) {
        // ---- maxflow.py:138-170 _global_relabel, level-synchronous ----
        for (long long v = tid; v < n; v += stride) a.h[v] = v == a.sink ? 0 : (int)hmax;
        grid.sync();
        for (int side = 0; side < 2; ++side) {
            const long long root = side == 0 ? a.sink : a.source, skip = side == 0 ? a.source : a.sink;
            if (side == 1) {
                if (tid == 0) a.h[a.source] = (int)n;
                grid.sync();
            }
            for (long long d = side == 0 ? 0 : n;; ++d) {
                bool ch = false;
                for (long long w = tid; w < n; w += stride) {
                    if (a.h[w] != d) continue;
                    for (long long q = a.first_out[w]; q < a.first_out[w + 1]; ++q) {
                        const long long v = a.head[q];
                        if (v != skip && a.h[v] == hmax && a.resid[a.rev[q]] > 0) {
                            a.h[v] = (int)(d + 1);
                            ch = true;
                        }
                    }
                }
                (void)root;
                if (!grid_any(grid, a.ctr, rot, ch)) break;
            }
        }
        // ---- maxflow.py:253-264 _collect_active ----
        bool act = false;
        for (long long v = tid; v < n; v += stride)
            act |= v != a.source && v != a.sink && a.excess[v] > 0 && a.h[v] < hmax;
        if (!grid_any(grid, a.ctr, rot, act)) break;
        if (a.max_sweeps >= 0 && sweeps >= a.max_sweeps) { converged = 0; break; }
        // ---- rounds synchronous pulses (maxflow.py:183-250 restated for a grid):
        // push from the pulse-start heights, then merge the inboxes and relabel
        // the nodes whose admissible arcs ran out; heights only rise, so a
        // relabel that reads a neighbour being relabeled stays a valid labeling
        for (int k = 0; k < a.rounds; ++k) {
            bool any = false;
            for (long long v = tid; v < n; v += stride) {
                a.pushed[v] = 0;
                if (v == a.source || v == a.sink) continue;
                long long e = a.excess[v];
                const int hv = a.h[v];
                if (e <= 0 || hv >= hmax) continue;
                any = true;
                for (long long q = a.first_out[v]; q < a.first_out[v + 1] && e > 0; ++q) {
                    const long long r = a.resid[q];
                    const long long w = a.head[q];
                    if (r > 0 && hv == a.h[w] + 1) {
                        const long long f = e < r ? e : r;
                        atomicAdd((unsigned long long *)&a.resid[q], (unsigned long long)(-f));
                        atomicAdd((unsigned long long *)&a.resid[a.rev[q]], (unsigned long long)f);
                        atomicAdd((unsigned long long *)&a.ein[w], (unsigned long long)f);
                        e -= f;
                        ++pushes;
                    }
                }
                a.excess[v] = e;
                a.pushed[v] = e > 0 ? 2 : 1;   // 2: admissible arcs exhausted with excess left
            }
            grid.sync();
            for (long long v = tid; v < n; v += stride) {
                const long long x = a.ein[v];
                if (x) { a.excess[v] += x; a.ein[v] = 0; }
                if (a.pushed[v] == 2) {
                    long long best = hmax;
                    for (long long q = a.first_out[v]; q < a.first_out[v + 1]; ++q)
                        if (a.resid[q] > 0 && a.h[a.head[q]] + 1 < best) best = a.h[a.head[q]] + 1;
                    a.h[v] = (int)best;
                    ++relabels;
                }
            }
            ++pulses;
            if (!grid_any(grid, a.ctr, rot, any)) break;
        }
        ++sweeps;
        if (sweeps > 100000000) break;
    }
    // ---- maxflow.py:267-284 _bfs_source_side ----
    if (a.side) {
        for (long long v = tid; v < n; v += stride) a.side[v] = v == a.source ? 1 : 0;
        grid.sync();
        for (;;) {
            bool ch = false;
            for (long long u = tid; u < n; u += stride) {
                if (!a.side[u]) continue;
                for (long long q = a.first_out[u]; q < a.first_out[u + 1]; ++q)
                    if (a.resid[q] > 0 && !a.side[a.head[q]]) {
                        a.side[a.head[q]] = 1;
                        ch = true;
                    }
            }
            if (!grid_any(grid, a.ctr, rot, ch)) break;
        }
    }
    long long stranded = 0;
    for (long long v = tid; v < n; v += stride) stranded += v != a.source && v != a.sink && a.excess[v] > 0;
    warp_add_u64(&a.ctr[6], pushes);
    warp_add_u64(&a.ctr[7], relabels);
    warp_add_u64(&a.ctr[10], stranded);
    if (tid == 0) {
        a.ctr[8] = sweeps;
        a.ctr[9] = converged;
        a.ctr[11] = pulses;
    }
}

// maxflow.py:267-284 _bfs_source_side on its own (no solve): level-synchronous
__global__ void __launch_bounds__(256) k_csr_side(long long n, long long source, const long long *first_out,
                                                  const int32_t *head, const long long *resid, unsigned char *side,
                                                  unsigned long long *slots) {
    cg::grid_group grid = cg::this_grid();
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    int rot = 0;
    for (long long v = tid; v < n; v += stride) side[v] = v == source ? 1 : 0;
    grid.sync();
    for (;;) {
        bool ch = false;
        for (long long u = tid; u < n; u += stride) {
            if (!side[u]) continue;
            for (long long q = first_out[u]; q < first_out[u + 1]; ++q)
                if (resid[q] > 0 && !side[head[q]]) {
                    side[head[q]] = 1;
                    ch = true;
                }
        }
        if (!grid_any(grid, slots, rot, ch)) break;
    }
}

// maxflow.py:287-304: per chain, push the chain's smallest residual through it
__global__ void k_chain_presaturate(const int32_t *rev, long long *resid, const int32_t *chain_arcs,
                                    const long long *chain_base, long long nsites, unsigned long long *total) {
    const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long sent = 0;
    if (s < nsites) {
        const long long a0 = chain_base[s], a1 = chain_base[s + 1];
        if (a1 > a0) {
            long long f = 1LL << 62;
            for (long long i = a0; i < a1; ++i) f = resid[chain_arcs[i]] < f ? resid[chain_arcs[i]] : f;
            if (f > 0) {
                for (long long i = a0; i < a1; ++i) {
                    const int q = chain_arcs[i];
                    resid[q] -= f;
                    atomicAdd((unsigned long long *)&resid[rev[q]], (unsigned long long)f);
                }
                sent = (unsigned long long)f;
            }
        }
    }
    warp_add_u64(total, (long long)sent);
}

// maxflow.py:323-334
__global__ void k_conservation(const long long *first_out, const long long *cap, const long long *resid, long long n,
                               long long source, long long sink, unsigned long long *bad) {
    const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long b = 0;
    if (u < n && u != source && u != sink) {
        long long net = 0;
        for (long long q = first_out[u]; q < first_out[u + 1]; ++q) net += cap[q] - resid[q];
        b = net != 0;
    }
    warp_add_u64(bad, b);
}

}  // namespace

extern "C" {

int gz_export_arcs(const int32_t *vol, int32_t rows, int32_t cols, int32_t m, const gz_energy *energy,
                   const int32_t *lo, const int32_t *hi, int32_t residual, int64_t *pair_u, int64_t *pair_v,
                   int64_t *pair_cap, int64_t *pair_rcap, int64_t capacity, int64_t *info, void *workspace,
                   size_t workspace_bytes, void *stream) {
    if ((!vol && !residual) || !energy || !info || rows < 1 || cols < 1 || m < 1 || (!lo) != (!hi)) return GZ_ERR_ARG;
    if (energy->penalty < 0 || energy->inhibit < 0) return GZ_ERR_ARG;
    if (!index_fits(rows, cols, m) || lanes_for(m) == 0) return m > 256 ? GZ_ERR_ARG : GZ_ERR_OVERFLOW;
    if (workspace_bytes < ws_bytes(rows, cols, m)) return GZ_ERR_WORKSPACE;
    int rc = check_sm100();
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    Workspace w = carve(workspace, rows, cols, m);
    const int P = rows * cols, lp = lanes_for(m);
    const long long nel = (long long)P * lp;
    if (!residual) {
        k_to_colmajor<<<(unsigned)((nel + 255) / 256), 256, 0, s>>>(vol, P, m, lp, w.vol);
        CK(cudaGetLastError());
    }
    // the solver's own initialisation, stopped before the first sweep, without
    // the presaturating chain wave: the state planes then hold the capacities
    // (residual mode: the state the last solve in this workspace left)
    long long dev_offset = 0;
    int hcap = HARD_CAP_DEFAULT;
    if (m > 1 && !residual) {
        CK(cudaMemsetAsync(w.ctr, 0, 24, s));
        k_source_caps<<<(P + 255) / 256, 256, 0, s>>>(vol, rows, cols, m, lo, hi, *energy, w.ctr);
        unsigned long long census[3];
        CK(cudaMemcpyAsync(census, w.ctr, 24, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (energy->hard_inhibit) {
            unsigned long long hc = 1ull << 16;
            while (hc <= census[0]) hc <<= 1;
            if (census[0] >= 0x7fffffffull || (census[1] + 1) * hc + census[0] >= 0x7fffffffull) return GZ_ERR_OVERFLOW;
            hcap = (int)hc;
        } else if (census[0] >= 0x7fffffffull) {
            return GZ_ERR_OVERFLOW;
        }
        gz_sched sc = {12, 0, 0, GZ_SCHED_NO_WAVE | GZ_SCHED_INIT_ONLY};
        gz_stats st;
        rc = solve_planar(w, rows, cols, m, energy, &sc, lo, hi, nullptr, &st, s, hcap, -1);
        if (rc) return rc;
        dev_offset = st.const_offset;
    }
    long long *nb = nullptr, *cnt = nullptr;
    unsigned long long *acc = nullptr;
    CK(cudaMallocAsync((void **)&nb, (size_t)(P + 1) * 8, s));
    CK(cudaMallocAsync((void **)&cnt, (size_t)(P + 1) * 8, s));
    CK(cudaMallocAsync((void **)&acc, 8, s));
    CK(cudaMemsetAsync(acc, 0, 8, s));
    k_window_widths<<<(P + 256) / 256, 256, 0, s>>>(lo, hi, P, m, nb);
    rc = scan_exclusive(nb, P + 1, s);
    long long n_int = 0;
    CK(cudaMemcpyAsync(&n_int, nb + P, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ExportArgs x;
    x.vol = w.vol; x.cu = w.cu; x.ph = w.ph; x.pv = w.pv; x.dar = w.dar; x.dbr = w.dbr; x.dad = w.dad; x.dbd = w.dbd;
    x.lo = lo; x.hi = hi; x.node_base = nb; x.cnt = cnt; x.offs = cnt; x.offset_acc = acc;
    x.pu = (long long *)pair_u; x.pv_ = (long long *)pair_v; x.pc = (long long *)pair_cap; x.prc = (long long *)pair_rcap;
    x.rows = rows; x.cols = cols; x.m = m; x.LPT = lp; x.pen = energy->penalty;
    x.icap_dev = energy->hard_inhibit ? hcap : energy->inhibit;
    x.hard = energy->hard_inhibit ? 1 : 0;
    x.src = n_int; x.snk = n_int + 1;
    CK(cudaMemsetAsync(cnt + P, 0, 8, s));
    if (rc == GZ_OK) {
        if (residual) k_export_arcs<false, 1><<<(P + 127) / 128, 128, 0, s>>>(x);
        else k_export_arcs<false, 0><<<(P + 127) / 128, 128, 0, s>>>(x);
        CK(cudaGetLastError());
        rc = scan_exclusive(cnt, P + 1, s);
    }
    long long npairs = 0;
    unsigned long long folded = 0;
    if (rc == GZ_OK) {
        CK(cudaMemcpyAsync(&npairs, cnt + P, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&folded, acc, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (pair_u && pair_v && pair_cap && pair_rcap && capacity >= npairs) {
            if (residual) k_export_arcs<true, 1><<<(P + 127) / 128, 128, 0, s>>>(x);
            else k_export_arcs<true, 0><<<(P + 127) / 128, 128, 0, s>>>(x);
            CK(cudaGetLastError());
        }
    }
    cudaFreeAsync(nb, s);
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(acc, s);
    CK(cudaStreamSynchronize(s));
    if (rc) return rc;
    info[0] = npairs;
    info[1] = (int64_t)folded;   // the export's own fold (flownet.py:124-125, 153-154, 172-173; int64 wrap)
    info[2] = n_int + 2;
    info[3] = m > 1 && !residual ? dev_offset : (int64_t)folded;   // the solver initialisation's constant offset
    return GZ_OK;
}

int gz_export_state(const void *workspace, int32_t rows, int32_t cols, int32_t m, int32_t plane, int32_t *out,
                    void *stream) {
    if (!workspace || !out || rows < 1 || cols < 1 || m < 2 || plane < 0 || plane > GZ_PLANE_HEIGHT)
        return GZ_ERR_ARG;
    if (lanes_for(m) == 0 || !index_fits(rows, cols, m)) return GZ_ERR_ARG;
    Workspace w = carve((void *)workspace, rows, cols, m);
    const int32_t *src[] = {w.cu, w.ph, w.pv, w.dar, w.dbr, w.dad, w.dbd, w.e, w.h};
    const int P = rows * cols, L = m - 1;
    const long long n = (long long)P * L;
    const bool ex = plane == GZ_PLANE_EXCESS;
    k_export_plane<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        src[plane], ex ? w.ein : nullptr, ex ? w.h2 : nullptr, P, lanes_for(m), L, out);
    CK(cudaGetLastError());
    return GZ_OK;
}

size_t gz_csr_workspace_bytes(int64_t n_nodes) {
    if (n_nodes < 2) return 0;
    return align_up((size_t)n_nodes * 8) * 2 + align_up((size_t)n_nodes * 4) * 2 + align_up(CSR_CTR * 8) + 256;
}

int gz_maxflow_csr(int64_t n_nodes, int64_t source, int64_t sink, const int64_t *first_out, const int32_t *head,
                   const int32_t *rev, const int64_t *cap, int64_t *resid, int32_t rounds_per_sweep, int32_t max_sweeps,
                   uint8_t *side_out, int64_t *excess_out, gz_csr_stats *stats_out, void *workspace,
                   size_t workspace_bytes, void *stream) {
    if (n_nodes < 2 || source < 0 || sink < 0 || source >= n_nodes || sink >= n_nodes || source == sink ||
        !first_out || !head || !rev || !cap || !resid || rounds_per_sweep < 1)
        return GZ_ERR_ARG;
    if (n_nodes >= (1LL << 30)) return GZ_ERR_OVERFLOW;   // heights are int32 (2n must fit)
    if (!workspace || workspace_bytes < gz_csr_workspace_bytes(n_nodes)) return GZ_ERR_WORKSPACE;
    int rc = check_sm100();
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t *b = (uint8_t *)(((uintptr_t)workspace + 255) & ~(uintptr_t)255);
    CsrArgs a;
    a.n = n_nodes; a.source = source; a.sink = sink;
    a.first_out = (const long long *)first_out; a.head = head; a.rev = rev; a.cap = (const long long *)cap;
    a.resid = (long long *)resid;
    a.excess = (long long *)b; b += align_up((size_t)n_nodes * 8);
    a.ein = (long long *)b; b += align_up((size_t)n_nodes * 8);
    a.h = (int *)b; b += align_up((size_t)n_nodes * 4);
    a.pushed = (int *)b; b += align_up((size_t)n_nodes * 4);
    a.ctr = (unsigned long long *)b;
    a.side = side_out;
    a.rounds = rounds_per_sweep;
    a.max_sweeps = max_sweeps;
    CK(cudaMemsetAsync(a.ein, 0, (size_t)n_nodes * 8, s));
    CK(cudaMemsetAsync(a.ctr, 0, CSR_CTR * 8, s));
    int grid = 0;
    rc = coop_grid((const void *)k_csr_solve, 256, &grid);
    if (rc) return rc;
    const long long need = (n_nodes + 255) / 256;
    if (grid > need) grid = (int)need;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
    void *args[] = {&a};
    CK(cudaLaunchCooperativeKernel((const void *)k_csr_solve, dim3(grid), dim3(256), args, 0, s));
    CK(cudaEventRecord(e1, s));
    unsigned long long h[CSR_CTR];
    CK(cudaMemcpyAsync(h, a.ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
    long long flow = 0;
    CK(cudaMemcpyAsync(&flow, a.excess + sink, 8, cudaMemcpyDeviceToHost, s));
    if (excess_out) CK(cudaMemcpyAsync(excess_out, a.excess, (size_t)n_nodes * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (stats_out) {
        stats_out->flow = flow;
        stats_out->pushes = (int64_t)h[6];
        stats_out->relabels = (int64_t)h[7];
        stats_out->sweeps = (int32_t)h[8];
        stats_out->converged = (int32_t)h[9];
        stats_out->stranded_excess_nodes = (int64_t)h[10];
        stats_out->pulses = (int32_t)h[11];
        stats_out->ms_total = ms;
    }
    return GZ_OK;
}

int gz_source_side_csr(int64_t n_nodes, int64_t source, const int64_t *first_out, const int32_t *head,
                       const int64_t *resid, uint8_t *side_out, void *stream) {
    if (n_nodes < 1 || source < 0 || source >= n_nodes || !first_out || !head || !resid || !side_out)
        return GZ_ERR_ARG;
    int rc = check_sm100();
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *slots = nullptr;
    CK(cudaMallocAsync((void **)&slots, 3 * 8, s));
    CK(cudaMemsetAsync(slots, 0, 3 * 8, s));
    int grid = 0;
    rc = coop_grid((const void *)k_csr_side, 256, &grid);
    if (rc) return rc;
    const long long need = (n_nodes + 255) / 256;
    if (grid > need) grid = (int)need;
    long long n = n_nodes, src = source;
    const long long *fo = (const long long *)first_out, *rs = (const long long *)resid;
    unsigned char *sd = side_out;
    void *args[] = {&n, &src, &fo, (void *)&head, &rs, &sd, &slots};
    CK(cudaLaunchCooperativeKernel((const void *)k_csr_side, dim3(grid), dim3(256), args, 0, s));
    cudaFreeAsync(slots, s);
    CK(cudaStreamSynchronize(s));
    return GZ_OK;
}

int gz_chain_presaturate_csr(const int32_t *rev, int64_t *resid, const int32_t *chain_arcs, const int64_t *chain_base,
                             int64_t nsites, int64_t *sent_out, void *stream) {
    if (!rev || !resid || !chain_arcs || !chain_base || nsites < 0 || !sent_out) return GZ_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(sent_out, 0, 8, s));
    if (nsites == 0) return GZ_OK;
    k_chain_presaturate<<<(unsigned)((nsites + 255) / 256), 256, 0, s>>>(rev, (long long *)resid, chain_arcs,
                                                                        (const long long *)chain_base, nsites,
                                                                        (unsigned long long *)sent_out);
    CK(cudaGetLastError());
    return GZ_OK;
}

int gz_conservation_violations_csr(const int64_t *first_out, const int64_t *cap, const int64_t *resid, int64_t n_nodes,
                                   int64_t source, int64_t sink, int64_t *bad_out, void *stream) {
    if (!first_out || !cap || !resid || n_nodes < 0 || !bad_out) return GZ_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(bad_out, 0, 8, s));
    if (n_nodes == 0) return GZ_OK;
    k_conservation<<<(unsigned)((n_nodes + 255) / 256), 256, 0, s>>>((const long long *)first_out,
                                                                    (const long long *)cap, (const long long *)resid,
                                                                    n_nodes, source, sink,
                                                                    (unsigned long long *)bad_out);
    CK(cudaGetLastError());
    return GZ_OK;
}

}  // extern "C"
