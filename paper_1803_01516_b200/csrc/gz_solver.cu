// gz_solver.cu -- B200 (sm_100a) push-relabel max-flow / min-cut on the
// implicit gaze-line graph, plus the data term, energy and hierarchy helpers,
// exported through the C ABI declared in include/gazecut_b200.h.
//
// Reference path (paths under /root/reference/pkg/src/gazecut/):
//   sad_volume          energy.py:83-114      -> k_sad_planar / gz_sad_volume
//   build_network       flownet.py:233-296    -> phase_init (implicit graph, no CSR)
//   maxflow_push_relabel maxflow.py:403-478   -> gz_solve_kernel (persistent, cooperative)
//   _global_relabel     maxflow.py:138-170    -> phase_bfs_* (exact BFS distance to the sink)
//   _discharge_rounds   maxflow.py:183-250    -> phase_push / phase_relabel (synchronous pulses)
//   _bfs_source_side    maxflow.py:267-284    -> phase_reach_* (prefix reach per chain)
//   _extract_labels     maxflow.py:307-320    -> labels = lo + reach
//   total_energy        energy.py:129-155     -> phase_energy (identity check, maxflow.py:501-505)
//   coarsen / thin_skin hierarchy.py:39-73    -> k_coarsen / k_thin_skin
//
// The solver runs phase 1 of push-relabel only (no excess is returned to the
// source).  The minimal source side of the minimum cut -- the set the
// reference reads its labeling from -- is recovered exactly as the nodes
// reachable in the residual graph from {source} U {nodes holding excess}; see
// DESIGN.md section 3 for the argument and tests/test_gpu_parity.py for the
// bit-exact checks against the oracle.
#include <ctime>
#include <unistd.h>

#include <chrono>
#include <mutex>
#include <thread>
#include <vector>

#include "gz_common.cuh"

namespace cg = cooperative_groups;
using namespace gz;

namespace {

__device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }

// Per-column view: own window and the four neighbours (right, left, down, up).
template <bool WIN>
struct Col {
    int c, y, g, lo, hi;
    int nc[4], nlo[4], nhi[4];
    bool has[4];

    __device__ __forceinline__ void load(const Prob &p, int c_) {
        c = c_;
        y = c / p.G;
        g = c - y * p.G;
        has[0] = g + 1 < p.G; nc[0] = c + 1;
        has[1] = g > 0;       nc[1] = c - 1;
        has[2] = y + 1 < p.Y; nc[2] = c + p.G;
        has[3] = y > 0;       nc[3] = c - p.G;
        if (WIN) {
            lo = p.lo[c]; hi = p.hi[c];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                nlo[i] = has[i] ? p.lo[nc[i]] : 0;
                nhi[i] = has[i] ? p.hi[nc[i]] : 0;
            }
        } else {
            lo = 0; hi = p.L;
#pragma unroll
            for (int i = 0; i < 4; ++i) { nlo[i] = 0; nhi[i] = p.L; }
        }
    }
    __device__ __forceinline__ int kind_own(int t) const { return t <= lo ? K_SRC : (t > hi ? K_SNK : K_REAL); }
    __device__ __forceinline__ int kind_nb(int i, int t) const {
        return t <= nlo[i] ? K_SRC : (t > nhi[i] ? K_SNK : K_REAL);
    }
};

// Arc j out of real node (t, col): returns the residual (0 when the arc does
// not exist), the target flat index (valid when kind == K_REAL), target kind.
template <bool WIN>
__device__ __forceinline__ int arc_resid(const Prob &p, const Col<WIN> &k, int j, int t, int &v, int &kind) {
    const int P = p.P, c = k.c, L = p.L;
    const int cap_i = p.hard ? p.hcap : p.inh;
    kind = K_SRC;
    v = 0;
    switch (j) {
    case A_UP:
        kind = k.kind_own(t + 1); v = (t + 1) * P + c;
        return p.cu[t * P + c];
    case A_DN:
        kind = k.kind_own(t - 1); v = (t - 1) * P + c;
        return HINF;
    case A_SR:
        if (!k.has[0]) return 0;
        kind = k.kind_nb(0, t); v = t * P + k.nc[0];
        return p.ph[t * P + c];
    case A_SL:
        if (!k.has[1]) return 0;
        kind = k.kind_nb(1, t); v = t * P + k.nc[1];
        return 2 * p.pen - p.ph[t * P + k.nc[1]];
    case A_SD:
        if (!k.has[2]) return 0;
        kind = k.kind_nb(2, t); v = t * P + k.nc[2];
        return p.pv[t * P + c];
    case A_SU:
        if (!k.has[3]) return 0;
        kind = k.kind_nb(3, t); v = t * P + k.nc[3];
        return 2 * p.pen - p.pv[t * P + k.nc[3]];
    case A_UR:
        if (!k.has[0] || t >= L) return 0;
        kind = k.kind_nb(0, t + 1); v = (t + 1) * P + k.nc[0];
        return p.dbr[(t + 1) * P + c];
    case A_UL:
        if (!k.has[1] || t >= L) return 0;
        kind = k.kind_nb(1, t + 1); v = (t + 1) * P + k.nc[1];
        return p.dar[(t + 1) * P + k.nc[1]];
    case A_UD:
        if (!k.has[2] || t >= L) return 0;
        kind = k.kind_nb(2, t + 1); v = (t + 1) * P + k.nc[2];
        return p.dbd[(t + 1) * P + c];
    case A_UU:
        if (!k.has[3] || t >= L) return 0;
        kind = k.kind_nb(3, t + 1); v = (t + 1) * P + k.nc[3];
        return p.dad[(t + 1) * P + k.nc[3]];
    case A_DR:
        if (!k.has[0]) return 0;
        kind = k.kind_nb(0, t - 1); v = (t - 1) * P + k.nc[0];
        return cap_i - p.dar[t * P + c];
    case A_DL:
        if (!k.has[1]) return 0;
        kind = k.kind_nb(1, t - 1); v = (t - 1) * P + k.nc[1];
        return cap_i - p.dbr[t * P + k.nc[1]];
    case A_DD:
        if (!k.has[2]) return 0;
        kind = k.kind_nb(2, t - 1); v = (t - 1) * P + k.nc[2];
        return cap_i - p.dad[t * P + c];
    case A_DU:
        if (!k.has[3]) return 0;
        kind = k.kind_nb(3, t - 1); v = (t - 1) * P + k.nc[3];
        return cap_i - p.dbd[t * P + k.nc[3]];
    }
    return 0;
}

// Push d units along arc j out of (t, col): update the stored residual/flow.
template <bool WIN>
__device__ __forceinline__ void arc_push(const Prob &p, const Col<WIN> &k, int j, int t, int d) {
    const int P = p.P, c = k.c;
    switch (j) {
    case A_UP: p.cu[t * P + c] -= d; break;
    case A_DN: p.cu[(t - 1) * P + c] += d; break;
    case A_SR: p.ph[t * P + c] -= d; break;
    case A_SL: p.ph[t * P + k.nc[1]] += d; break;
    case A_SD: p.pv[t * P + c] -= d; break;
    case A_SU: p.pv[t * P + k.nc[3]] += d; break;
    case A_UR: p.dbr[(t + 1) * P + c] -= d; break;
    case A_UL: p.dar[(t + 1) * P + k.nc[1]] -= d; break;
    case A_UD: p.dbd[(t + 1) * P + c] -= d; break;
    case A_UU: p.dad[(t + 1) * P + k.nc[3]] -= d; break;
    case A_DR: p.dar[t * P + c] += d; break;
    case A_DL: p.dbr[t * P + k.nc[1]] += d; break;
    case A_DD: p.dad[t * P + c] += d; break;
    case A_DU: p.dbd[t * P + k.nc[3]] += d; break;
    }
}

// ---------------------------------------------------------------------------
// initialisation: residuals from the volume, source saturation, chain wave,
// constant offset (flownet.py:115-181 folded into an implicit graph;
// maxflow.py:173-180 _saturate_source; maxflow.py:287-304 _chain_presaturate
// generalised to a greedy upward wave along each chain).

template <bool WIN>
__device__ void phase_init_a(const Prob &p, int c) {
    const int P = p.P;
    for (int k = 0; k < p.M; ++k) {
        p.cu[k * P + c] = p.vol[k * P + c];
        p.ph[k * P + c] = p.pen;
        p.pv[k * P + c] = p.pen;
        p.dar[k * P + c] = 0; p.dbr[k * P + c] = 0; p.dad[k * P + c] = 0; p.dbd[k * P + c] = 0;
        p.e[k * P + c] = 0; p.ein[k * P + c] = 0;
    }
}

template <bool WIN>
__device__ void phase_init_b(const Prob &p, int c, long long &flow, long long &offset, long long &presat) {
    Col<WIN> k;
    k.load(p, c);
    const int P = p.P, L = p.L;
    const long long icap_off = p.hard ? UNCUTTABLE : (long long)p.inh;
    const int icap = p.hard ? p.hcap : p.inh;
    if (WIN) {
        // constant offset: source->sink arcs (flownet.py:124-125, 153-154, 172-173)
        if (k.lo == k.hi) offset += p.vol[k.lo * P + c];
        for (int i = 0; i < 4; i += 2) {   // forward neighbours: right (0), down (2)
            if (!k.has[i]) continue;
            for (int t = 1; t <= L; ++t) {
                int a = k.kind_own(t), b = k.kind_nb(i, t);
                if ((a == K_SRC && b == K_SNK) || (a == K_SNK && b == K_SRC)) offset += p.pen;
                // diagonal dir 0: (c,t)->(n,t-1); dir 1: (n,t)->(c,t-1)
                int a0 = k.kind_own(t), b0 = k.kind_nb(i, t - 1);
                if (a0 == K_SRC && b0 == K_SNK) offset += icap_off;
                int a1 = k.kind_nb(i, t), b1 = k.kind_own(t - 1);
                if (a1 == K_SRC && b1 == K_SNK) offset += icap_off;
            }
        }
        // saturate arcs leaving source positions into this column's real nodes
        for (int t = k.lo + 1; t <= k.hi; ++t) {
            long long add = 0;
            if (t == k.lo + 1) add += p.vol[k.lo * P + c];           // chain arc lo
            for (int i = 0; i < 4; ++i) {
                if (!k.has[i]) continue;
                if (k.kind_nb(i, t) == K_SRC) add += p.pen;           // same level
                if (t + 1 <= L && k.kind_nb(i, t + 1) == K_SRC) add += icap;  // inhibit diagonal down into (c,t)
            }
            p.e[t * P + c] = (int)add;
        }
    } else {
        p.e[1 * P + c] = p.vol[c];   // chain arc 0 from the source
    }
    // greedy wave up the chain: push as much as each chain arc admits
    if (p.no_wave) return;
    long long carry = 0;
    for (int t = k.lo + 1; t <= k.hi; ++t) {
        int x = p.e[t * P + c] + (int)carry;
        int r = p.cu[t * P + c];
        int d = imin(x, r);
        p.cu[t * P + c] = r - d;
        p.e[t * P + c] = x - d;
        carry = d;
    }
    flow += carry;
    presat += carry;
}

// ---------------------------------------------------------------------------
// synchronous push pulse: every active node pushes on admissible arcs using the
// height field as it stands (heights do not change during this phase, so no
// two pushes on one arc pair can meet).  Own-column chain pushes feed the next
// position immediately (Gauss-Seidel along the chain); lateral pushes land in
// the neighbour's inbox `ein`, merged by the relabel phase.
template <bool WIN>
__device__ void phase_push(const Prob &p, int c, long long &flow, long long &pushes) {
    Col<WIN> k;
    k.load(p, c);
    const int P = p.P;
    for (int t = k.lo + 1; t <= k.hi; ++t) {
        const int u = t * P + c;
        int ex = p.e[u];
        if (ex <= 0) continue;
        const int hu = p.h[u];
        if (hu >= HINF) continue;
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
            if (kind == K_SNK) flow += d;
            else if (j == A_UP || j == A_DN) p.e[v] += d;
            else atomicAdd(&p.ein[v], d);
        }
        p.e[u] = ex;
    }
}

// relabel phase: merge the inbox, then every active node with no admissible
// arc moves to one above its lowest residual neighbour (maxflow.py:217-228).
// Reads h, writes h2 (snapshot semantics).
template <bool WIN>
__device__ void phase_relabel(const Prob &p, int c, long long &relabels) {
    Col<WIN> k;
    k.load(p, c);
    const int P = p.P;
    for (int t = k.lo + 1; t <= k.hi; ++t) {
        const int u = t * P + c;
        int ex = p.e[u] + p.ein[u];
        p.ein[u] = 0;
        p.e[u] = ex;
        const int hu = p.h[u];
        int hn = hu;
        if (ex > 0 && hu < HINF) {
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
            if (!adm) { hn = best; ++relabels; }
        }
        p.h2[u] = hn;
    }
}

// ---------------------------------------------------------------------------
// global relabel: exact BFS distance to the sink over residual arcs
// (maxflow.py:138-158).  Jacobi over lateral arcs (reads h, writes h2), then
// the column is closed under its own chain arcs in registers-order sweeps.
template <bool WIN>
__device__ void phase_bfs_reset(const Prob &p, int c) {
    for (int t = 1; t <= p.L; ++t) p.h[t * p.P + c] = HINF;
}

template <bool WIN>
__device__ bool phase_bfs_iter(const Prob &p, int c) {
    Col<WIN> k;
    k.load(p, c);
    const int P = p.P;
    bool changed = false;
    for (int t = k.lo + 1; t <= k.hi; ++t) {
        const int u = t * P + c;
        int best = p.h[u];
#pragma unroll
        for (int j = 0; j < A_DN; ++j) {    // all but chain-down (handled by the sweep)
            int v, kind;
            int r = arc_resid<WIN>(p, k, j, t, v, kind);
            if (kind == K_SRC || r <= 0) continue;
            int hv = kind == K_SNK ? 0 : p.h[v];
            best = imin(best, hv + 1);
        }
        p.h2[u] = best;
    }
    // close the column under its chain arcs: down (t+1 -> t via cu[t] > 0) and
    // up (t-1 reaches t's height + 1 through the infinite reverse arc)
    for (int pass = 0; pass < 2; ++pass) {
        int above = HINF;   // height of position t+1 (sink: 0)
        for (int t = k.hi; t > k.lo; --t) {
            const int u = t * P + c;
            int hv = (t == k.hi) ? 0 : above;
            int cur = p.h2[u];
            if (p.cu[u] > 0 && hv + 1 < cur) { cur = hv + 1; p.h2[u] = cur; }
            above = cur;
        }
        int below = HINF;
        for (int t = k.lo + 1; t <= k.hi; ++t) {
            const int u = t * P + c;
            int cur = p.h2[u];
            if (below < HINF && below + 1 < cur) { cur = below + 1; p.h2[u] = cur; }
            below = cur;
        }
    }
    for (int t = k.lo + 1; t <= k.hi; ++t) {
        const int u = t * P + c;
        if (p.h2[u] != p.h[u]) { changed = true; break; }
    }
    return changed;
}

// ---------------------------------------------------------------------------
// extraction: the source side is downward closed along every chain (reverse
// chain arcs are uncuttable), so it is one prefix length per site.  Seeds are
// the nodes holding excess; closure over residual arcs to a fixpoint
// (maxflow.py:267-284, 307-320).
template <bool WIN>
__device__ int column_close_up(const Prob &p, const Col<WIN> &k, int r) {
    // reached real positions lo+1 .. lo+r; position q reaches q+1 if cu[q] > 0
    const int P = p.P;
    while (r > 0 && k.lo + r < k.hi && p.cu[(k.lo + r) * P + k.c] > 0) ++r;
    return r;
}

template <bool WIN>
__device__ void phase_reach_init(const Prob &p, int c) {
    Col<WIN> k;
    k.load(p, c);
    int r = 0;
    for (int t = k.hi; t > k.lo; --t)
        if (p.e[t * p.P + c] > 0) { r = t - k.lo; break; }
    p.reach[c] = column_close_up<WIN>(p, k, r);
}

// Highest position of column c reached from the reached prefix of neighbour i.
template <bool WIN>
__device__ __forceinline__ int reach_from_nb(const Prob &p, const Col<WIN> &k, int i, int rn, int best_pos) {
    // neighbour i's reached real positions: nlo+1 .. nlo+rn.  Arcs from (n, q)
    // into column c: same level (c,q), inhibit-down (c,q-1), reverse-diagonal up (c,q+1).
    const int P = p.P, c = k.c, n = k.nc[i], L = p.L;
    const int cap_i = p.hard ? p.hcap : p.inh;
    const int top = k.nlo[i] + rn;
    for (int q = top; q > k.nlo[i]; --q) {
        if (q + 1 <= best_pos) break;   // nothing from here down can improve
        // diagonal up: (n,q) -> (c,q+1) is the reverse of (c,q+1)->(n,q)
        if (q + 1 <= L && q + 1 > best_pos && k.kind_own(q + 1) == K_REAL) {
            int r = 0;
            switch (i) {
            case 0: r = p.dar[(q + 1) * P + c]; break;   // (c,q+1)->(c+1,q) flow = dar[q+1][c]
            case 1: r = p.dbr[(q + 1) * P + n]; break;   // (c,q+1)->(c-1,q): pair (n,c) dir 1
            case 2: r = p.dad[(q + 1) * P + c]; break;
            case 3: r = p.dbd[(q + 1) * P + n]; break;
            }
            if (r > 0) best_pos = q + 1;
        }
        // same level: (n,q) -> (c,q)
        if (q > best_pos && k.kind_own(q) == K_REAL) {
            int r = 0;
            switch (i) {
            case 0: r = 2 * p.pen - p.ph[q * P + c]; break;   // (c+1,q)->(c,q)
            case 1: r = p.ph[q * P + n]; break;               // (c-1,q)->(c,q)
            case 2: r = 2 * p.pen - p.pv[q * P + c]; break;
            case 3: r = p.pv[q * P + n]; break;
            }
            if (r > 0) best_pos = q;
        }
        // inhibit diagonal down: (n,q) -> (c,q-1)
        if (q - 1 > best_pos && k.kind_own(q - 1) == K_REAL) {
            int r = 0;
            switch (i) {
            case 0: r = cap_i - p.dbr[q * P + c]; break;   // (c+1,q)->(c,q-1): pair (c,c+1) dir 1
            case 1: r = cap_i - p.dar[q * P + n]; break;   // (c-1,q)->(c,q-1): pair (n,c) dir 0
            case 2: r = cap_i - p.dbd[q * P + c]; break;
            case 3: r = cap_i - p.dad[q * P + n]; break;
            }
            if (r > 0) best_pos = q - 1;
        }
    }
    return best_pos;
}

template <bool WIN>
__device__ bool phase_reach_iter(const Prob &p, int c) {
    Col<WIN> k;
    k.load(p, c);
    const int r0 = p.reach[c];
    int best_pos = k.lo + r0;   // highest reached position (lo = none)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (!k.has[i]) continue;
        int rn = p.reach[k.nc[i]];
        if (rn > 0) best_pos = reach_from_nb<WIN>(p, k, i, rn, best_pos);
    }
    int r = column_close_up<WIN>(p, k, best_pos - k.lo);
    p.reach2[c] = r;
    return r != r0;
}

// energy.py:129-155 on the labeling (labels are cuboid-local)
__device__ void phase_energy_col(const Prob &p, int c, long long &energy, int &viol) {
    const int y = c / p.G, g = c - y * p.G;
    const int a = p.labels[c];
    energy += p.vol[a * p.P + c];
    for (int i = 0; i < 2; ++i) {
        bool has = i == 0 ? g + 1 < p.G : y + 1 < p.Y;
        if (!has) continue;
        int b = p.labels[i == 0 ? c + 1 : c + p.G];
        int dl = a > b ? a - b : b - a;
        if (p.hard && dl > 1) viol = 1;
        energy += (long long)p.pen * dl + (long long)p.inh * (dl > 1 ? dl - 1 : 0);
    }
}


// ---------------------------------------------------------------------------
// The whole solve in one cooperative launch: no host round trips.
template <bool WIN>
__global__ void __launch_bounds__(256) gz_solve_kernel(Prob p) {
    cg::grid_group grid = cg::this_grid();
    const int stride = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int ncols_iter = (p.P + stride - 1) / stride;   // uniform trip count (warp-shuffle safety)
    long long flow = 0, offset = 0, presat = 0, pushes = 0, relabels = 0;
    volatile unsigned long long *vctr = p.ctr;

    for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride)
        if (c < p.P) phase_init_a<WIN>(p, c);
    grid.sync();
    for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride)
        if (c < p.P) phase_init_b<WIN>(p, c, flow, offset, presat);
    grid.sync();

    int sweeps = 0, bfs_passes = 0, pulses = 0, flag_rot = 0, act_rot = 0;
    int converged = 1;
    const int bfs_guard = 4 * (p.P + p.M) + 64;
    for (;;) {
        // ---- global relabel (exact unless bfs_cap > 0) ----
        for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride)
            if (c < p.P) phase_bfs_reset<WIN>(p, c);
        grid.sync();
        int iters = 0;
        bool exact = true;
        for (;;) {
            bool ch = false;
            for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride)
                if (c < p.P) ch |= phase_bfs_iter<WIN>(p, c);
            if (tid == 0) vctr[CTR_FLAG0 + (flag_rot + 1) % 3] = 0;
            if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) vctr[CTR_FLAG0 + flag_rot] = 1;
            grid.sync();
            bool any = vctr[CTR_FLAG0 + flag_rot] != 0;
            flag_rot = (flag_rot + 1) % 3;
            int32_t *tmp = p.h; p.h = p.h2; p.h2 = tmp;
            ++iters;
            if (!any) break;
            if (p.bfs_cap > 0 && iters >= p.bfs_cap) { exact = false; break; }
            if (iters > bfs_guard) { if (tid == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
        }
        bfs_passes += iters;
        // ---- active nodes? ----
        {
            int cnt = 0;
            for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride) {
                if (c >= p.P) continue;
                int lo = WIN ? p.lo[c] : 0, hi = WIN ? p.hi[c] : p.L;
                for (int t = lo + 1; t <= hi; ++t) {
                    int u = t * p.P + c;
                    cnt += (p.e[u] > 0 && p.h[u] < HINF);
                }
            }
            if (tid == 0) vctr[CTR_ACT0 + (act_rot + 1) % 3] = 0;
            warp_add_u64((unsigned long long *)&p.ctr[CTR_ACT0 + act_rot], cnt);
            grid.sync();
            unsigned long long act = vctr[CTR_ACT0 + act_rot];
            act_rot = (act_rot + 1) % 3;
            if (act == 0) {
                if (exact) break;
                // a truncated relabel found nothing: rerun it exactly before concluding
                p.bfs_cap = 0;
                continue;
            }
        }
        if (p.capped && sweeps >= p.max_sweeps) { converged = 0; break; }
        if (vctr[CTR_STATUS] != 0) break;
        // ---- K synchronous push/relabel pulses ----
        for (int pulse = 0; pulse < p.K; ++pulse) {
            for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride)
                if (c < p.P) phase_push<WIN>(p, c, flow, pushes);
            grid.sync();
            for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride)
                if (c < p.P) phase_relabel<WIN>(p, c, relabels);
            grid.sync();
            int32_t *tmp = p.h; p.h = p.h2; p.h2 = tmp;
            ++pulses;
        }
        ++sweeps;
        if (sweeps > 1000000) { if (tid == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
    }

    // ---- extraction: reach closure from the excess nodes ----
    for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride)
        if (c < p.P) phase_reach_init<WIN>(p, c);
    grid.sync();
    int reach_passes = 0;
    const int reach_guard = 4 * (p.P + p.M) + 64;
    for (;;) {
        bool ch = false;
        for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride)
            if (c < p.P) ch |= phase_reach_iter<WIN>(p, c);
        if (tid == 0) vctr[CTR_FLAG0 + (flag_rot + 1) % 3] = 0;
        if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) vctr[CTR_FLAG0 + flag_rot] = 1;
        grid.sync();
        bool any = vctr[CTR_FLAG0 + flag_rot] != 0;
        flag_rot = (flag_rot + 1) % 3;
        int32_t *tmp = p.reach; p.reach = p.reach2; p.reach2 = tmp;
        ++reach_passes;
        if (!any) break;
        if (reach_passes > reach_guard) { if (tid == 0) vctr[CTR_STATUS] = (unsigned long long)(-GZ_ERR_NOCONVERGE); break; }
    }
    // labels, stranded excess
    long long stranded = 0;
    for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride) {
        if (c >= p.P) continue;
        int lo = WIN ? p.lo[c] : 0, hi = WIN ? p.hi[c] : p.L;
        p.labels[c] = lo + p.reach[c];
        for (int t = lo + 1; t <= hi; ++t) stranded += p.e[t * p.P + c] > 0;
    }
    grid.sync();
    long long energy = 0;
    int viol = 0;
    for (int it = 0, c = tid; it < ncols_iter; ++it, c += stride)
        if (c < p.P) phase_energy_col(p, c, energy, viol);
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
        p.ctr[CTR_BFS_PASSES] = bfs_passes;
        p.ctr[CTR_REACH_PASSES] = reach_passes;
        p.ctr[CTR_CONVERGED] = converged;
        p.ctr[CTR_PULSES] = pulses;
    }
}

}  // namespace


namespace {

// ---------------------------------------------------------------------------
// data term (energy.py:83-114, geometry.py:325-335): one thread per site,
// labels looped; output planar [k][y][g] (solver layout) or (y, g, k).
// LAYOUT 0: (y, g, k) reference order; 1: planar [k][site]; 2: column-major [site][LP]
template <int LAYOUT>
__global__ void k_sad(const uint8_t *__restrict__ left, const uint8_t *__restrict__ right, int img_w, int ch,
                      gz_cuboid cb, int32_t *__restrict__ vol, int LP = 16) {
    const int P = cb.y_extent * cb.g_extent;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P) return;
    const int yi = c / cb.g_extent, gi = c - yi * cb.g_extent;
    const int g = cb.g_min + gi;
    const size_t row = (size_t)(cb.y_min + yi) * img_w * ch;
    const uint8_t *lr = left + row, *rr = right + row;
    for (int kk = 0; kk < cb.m; ++kk) {
        const int d = cb.d_min + kk;
        int xr = g + d, xl = (cb.width - 1) + g - d;
        xr = xr < 0 ? 0 : (xr > cb.width - 1 ? cb.width - 1 : xr);
        xl = xl < 0 ? 0 : (xl > cb.width - 1 ? cb.width - 1 : xl);
        int acc = 0;
        for (int q = 0; q < ch; ++q) acc += abs((int)lr[xl * ch + q] - (int)rr[xr * ch + q]);
        if (LAYOUT == 1) vol[(size_t)kk * P + c] = acc;
        else if (LAYOUT == 2) vol[(size_t)c * LP + kk] = acc;
        else vol[(size_t)c * cb.m + kk] = acc;
    }
    if (LAYOUT == 2)
        for (int kk = cb.m; kk < LP; ++kk) vol[(size_t)c * LP + kk] = 0;
}

// (rows, cols, m) -> column-major [site][LP], zero padded
__global__ void k_to_colmajor(const int32_t *__restrict__ src, int P, int M, int LP, int32_t *__restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)P * LP) return;
    const int c = (int)(i / LP), k = (int)(i % LP);
    dst[i] = k < M ? src[(size_t)c * M + k] : 0;
}

// Source-capacity census (windows or hard mode): out[0] += finite capacity of
// arcs leaving source positions into real nodes, out[1] += number of such
// arcs that are uncuttable (hard inhibit diagonals).  vol: (rows, cols, m).
__global__ void k_source_caps(const int32_t *__restrict__ vol, int rows, int cols, int m, const int32_t *lo,
                              const int32_t *hi, gz_energy en, unsigned long long *out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int P = rows * cols;
    unsigned long long fin = 0, inf = 0;
    if (c < P) {
        const int y = c / cols, g = c - y * cols;
        const int l0 = lo ? lo[c] : 0, h0 = hi ? hi[c] : m - 1;
        if (h0 > l0) fin += (unsigned long long)vol[(size_t)c * m + l0];   // chain arc lo
        const int nc[4] = {c + 1, c - 1, c + cols, c - cols};
        const bool has[4] = {g + 1 < cols, g > 0, y + 1 < rows, y > 0};
        for (int i = 0; i < 4; ++i) {
            if (!has[i]) continue;
            const int ln = lo ? lo[nc[i]] : 0;
            for (int t = l0 + 1; t <= h0; ++t) {
                if (t <= ln) fin += (unsigned long long)en.penalty;                // same level from a source position
                if (t + 1 <= m - 1 && t + 1 <= ln) {                                // inhibit diagonal (n,t+1)->(c,t)
                    if (en.hard_inhibit) ++inf;
                    else fin += (unsigned long long)en.inhibit;
                }
            }
        }
    }
    warp_add_u64(&out[0], (long long)fin);
    warp_add_u64(&out[1], (long long)inf);
    if (c < P && lo) atomicMax(&out[2], (unsigned long long)(hi[c] - lo[c]));   // widest window
}

__global__ void k_fill_i32(int32_t *dst, int n, int32_t v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = v;
}

// (rows, cols, m) -> planar [k][rows*cols]
__global__ void k_to_planar(const int32_t *__restrict__ src, int P, int M, int32_t *__restrict__ dst) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P) return;
    for (int k = 0; k < M; ++k) dst[(size_t)k * P + c] = src[(size_t)c * M + k];
}

__global__ void k_total_energy(const int32_t *__restrict__ lab, const int32_t *__restrict__ vol, int rows, int cols,
                               int m, gz_energy en, unsigned long long *out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int P = rows * cols;
    long long acc = 0;
    int viol = 0;
    if (c < P) {
        const int y = c / cols, g = c - y * cols;
        const int a = lab[c];
        acc += vol[(size_t)c * m + a];
        for (int i = 0; i < 2; ++i) {
            bool has = i == 0 ? g + 1 < cols : y + 1 < rows;
            if (!has) continue;
            int b = lab[i == 0 ? c + 1 : c + cols];
            int dl = a > b ? a - b : b - a;
            if (en.hard_inhibit && dl > 1) viol = 1;
            acc += (long long)en.penalty * dl + (long long)en.inhibit * (dl > 1 ? dl - 1 : 0);
        }
    }
    warp_add_u64(&out[0], acc);
    if (viol) out[1] = 1;
}

// hierarchy.py:39-57: coarse[Y][X][Z] = sum of the (zero padded) b^3 cube
__global__ void k_coarsen(const int32_t *__restrict__ vol, int rows, int cols, int m, int b, int32_t *__restrict__ out) {
    const int rb = (rows + b - 1) / b, cb = (cols + b - 1) / b, mb = (m + b - 1) / b;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)rb * cb * mb) return;
    const int z = (int)(idx % mb);
    const int x = (int)((idx / mb) % cb);
    const int yb = (int)(idx / ((long long)mb * cb));
    long long acc = 0;
    for (int dy = 0; dy < b; ++dy) {
        int y = yb * b + dy;
        if (y >= rows) break;
        for (int dx = 0; dx < b; ++dx) {
            int g = x * b + dx;
            if (g >= cols) break;
            const int32_t *src = vol + ((size_t)y * cols + g) * m;
            for (int dz = 0; dz < b; ++dz) {
                int k = z * b + dz;
                if (k >= m) break;
                acc += src[k];
            }
        }
    }
    out[idx] = (int32_t)acc;
}

// hierarchy.py:60-73
__global__ void k_thin_skin(const int32_t *__restrict__ coarse, int crows, int ccols, int rows, int cols, int m,
                            int b, int radius, int32_t *__restrict__ lo, int32_t *__restrict__ hi) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= rows * cols) return;
    const int y = c / cols, g = c - y * cols;
    const int D = coarse[(y / b) * ccols + (g / b)];
    long long l = (long long)b * (D - radius), h = (long long)b * (D + radius + 1) - 1;
    lo[c] = (int32_t)(l < 0 ? 0 : l);
    hi[c] = (int32_t)(h > m - 1 ? m - 1 : h);
    (void)crows;
}

// ---------------------------------------------------------------------------
// host side

struct Workspace {
    int32_t *vol, *cu, *ph, *pv, *dar, *dbr, *dad, *dbd, *e, *ein, *h, *h2;
    int32_t *reach, *reach2, *labels;
    unsigned long long *ctr;
    gz2::Bits2 bits;
    uint32_t *IN0, *IN1;
    uint32_t *bits_base;
    size_t bits_bytes;
};

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// words per column of the bit-parallel solver (positions 1..m), rounded to a template instance
int words_for(int m) {
    const int w = (m + 31) / 32;
    return w <= 1 ? 1 : w <= 2 ? 2 : w <= 4 ? 4 : w <= 8 ? 8 : 0;
}

size_t bit_bytes(int rows, int cols, int m) {
    const size_t P = (size_t)rows * cols;
    const int NW = words_for(m) ? words_for(m) : 1;
    // + R0 (P ints) and R1 (2P ints: also the BFS per-tile flag pair, ntiles <= P)
    return align_up((size_t)(13 + 9) * NW * P * 4) + align_up(P * 4) + align_up(2 * P * 4);
}

// positions per site row of the v4 solver's node arrays (16, or 32 x segments; 0: m too large)
int lanes_for(int m) { return m <= 16 ? 16 : (m <= 256 ? 32 * words_for(m) : 0); }

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t err__ = (x);                                                               \
        if (err__ != cudaSuccess) {                                                            \
            fprintf(stderr, "gazecut_b200: %s failed: %s\n", #x, cudaGetErrorString(err__));   \
            return GZ_ERR_CUDA;                                                                \
        }                                                                                      \
    } while (0)

// The kernels index node state with int32 (site * LPT + position for the v4
// [site][LPT] planes, position * P + site for the v1 planar layout).  Problems
// whose planes would exceed 2^31 - 1 elements are refused with GZ_ERR_OVERFLOW
// instead of wrapping (C5, 3840 x 2160 x 256, is 2.12e9: inside, with ~1% to
// spare; 4096 x 2160 x 256 is outside).
bool index_fits(int rows, int cols, int m) {
    const unsigned long long P = (unsigned long long)rows * (unsigned long long)cols;
    const unsigned long long per = lanes_for(m) ? (unsigned long long)lanes_for(m) : (unsigned long long)m + 1;
    return P * per <= 0x7fffffffull;
}

// Streams and the pinned counter buffer of the concurrent-solve entry points
// (gz_solve_pairs, gz_solve_volume_batch), one set per device.  A call holds
// its device's lock for its whole duration: calls on one device from several
// host threads are serialised, calls on different devices run concurrently.
struct DevicePool {
    std::mutex mu;
    static constexpr int MAX_STREAMS = 128;   // concurrent pair solves (the hardware runs up to 128 kernels at once)
    cudaStream_t streams[MAX_STREAMS] = {};
    bool have_streams = false;
    unsigned long long *pinned = nullptr;
    size_t pinned_n = 0;
    int streams_ready() {
        if (have_streams) return GZ_OK;
        for (int k = 0; k < MAX_STREAMS; ++k) CK(cudaStreamCreateWithFlags(&streams[k], cudaStreamNonBlocking));
        have_streams = true;
        return GZ_OK;
    }
    unsigned *flag_host = nullptr, *flag_dev = nullptr;   // host-mapped word (batched tail launch)
    int flag_ready() {
        if (flag_host) return GZ_OK;
        CK(cudaHostAlloc((void **)&flag_host, 256, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer((void **)&flag_dev, flag_host, 0));
        return GZ_OK;
    }
    void *scratch = nullptr;   // per-call device scratch of gz_solve_pairs (grow-only)
    size_t scratch_n = 0;
    int scratch_ready(size_t n) {
        if (scratch_n >= n) return GZ_OK;
        if (scratch) cudaFree(scratch);
        scratch = nullptr;
        scratch_n = 0;
        CK(cudaMalloc(&scratch, n));
        scratch_n = n;
        return GZ_OK;
    }
    int pinned_ready(size_t n) {
        if (pinned_n >= n) return GZ_OK;
        if (pinned) cudaFreeHost(pinned);
        pinned = nullptr;
        pinned_n = 0;
        CK(cudaHostAlloc((void **)&pinned, n * 8, cudaHostAllocDefault));
        pinned_n = n;
        return GZ_OK;
    }
};
constexpr int MAX_DEVICES = 64;

DevicePool *device_pool() {
    static DevicePool pools[MAX_DEVICES];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAX_DEVICES) return nullptr;
    return &pools[dev];
}

size_t ws_bytes(int rows, int cols, int m) {
    const int mp = m > lanes_for(m) ? m : lanes_for(m);
    const size_t P = (size_t)rows * cols, plane = align_up((size_t)mp * P * 4), col = align_up(P * 4);
    return 12 * plane + 3 * col + align_up(gz::CTR_COUNT * 8) + bit_bytes(rows, cols, m) + 256;
}

Workspace carve(void *ws, int rows, int cols, int m) {
    const int mp = m > lanes_for(m) ? m : lanes_for(m);
    const size_t P = (size_t)rows * cols, plane = align_up((size_t)mp * P * 4), col = align_up(P * 4);
    uint8_t *b = (uint8_t *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    Workspace w;
    int32_t **planes[12] = {&w.vol, &w.cu, &w.ph, &w.pv, &w.dar, &w.dbr, &w.dad, &w.dbd, &w.e, &w.ein, &w.h, &w.h2};
    for (int i = 0; i < 12; ++i) { *planes[i] = (int32_t *)b; b += plane; }
    w.reach = (int32_t *)b; b += col;
    w.reach2 = (int32_t *)b; b += col;
    w.labels = (int32_t *)b; b += col;
    w.ctr = (unsigned long long *)b; b += align_up(gz::CTR_COUNT * 8);
    const int NW = words_for(m) ? words_for(m) : 1;
    w.bits_base = (uint32_t *)b;
    w.bits_bytes = bit_bytes(rows, cols, m);
    uint32_t *u = (uint32_t *)b;
    const size_t word_plane = (size_t)NW * P;
    w.bits.NW = NW;
    w.bits.mask = u; u += 13 * word_plane;
    uint32_t **arr[9] = {&w.bits.V, &w.bits.F0, &w.bits.F1, &w.bits.A, &w.bits.IN, &w.bits.EX, &w.bits.RL,
                         &w.IN0, &w.IN1};
    for (int i = 0; i < 9; ++i) { *arr[i] = u; u += word_plane; }
    uint8_t *rb = (uint8_t *)(((uintptr_t)u + 255) & ~(uintptr_t)255);
    w.bits.R0 = (int32_t *)rb; rb += col;
    w.bits.R1 = (int32_t *)rb;
    return w;
}


int coop_grid(const void *kernel, int threads, int *grid_out, size_t dyn_smem = 0) {
    int dev = 0, sms = 0, occ = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, dyn_smem));
    if (occ < 1) return GZ_ERR_CUDA;
    *grid_out = sms * occ;
    return GZ_OK;
}

// 1: v1 column relaxation (m > 256, or forced with GZ_SCHED_V1 for
// comparison), 4: tile-owned warp-per-chain-segment solver with temporally
// blocked BFS (m <= 256; exact and capped level-2; the default).
int choose_solver(int m, const gz_sched *sc) {
    const int flags = sc ? sc->flags : 0;
    if ((flags & GZ_SCHED_V1) || words_for(m) == 0) return 1;
    return 4;
}

// Tile geometry of the v4 solver for a team of nb CTAs, BFS blocking depth H.
gz4::Geo tile_geo_h(int rows, int cols, int nb, int nw, int occ, int H) {
    const int regmax = gz4::region_sites(nw, occ);
    gz4::Geo g;
    g.H = H;
    g.TX = 32;
    // the smallest region (one tile row plus halo) must fit the BFS register tiles
    while (g.H > 1 && (1 + 2 * g.H) * (g.TX + 2 * g.H) > regmax) --g.H;
    if (g.H < 1) g.H = 1;
    g.nx = (cols + g.TX - 1) / g.TX;
    int tile_rows = nb / g.nx;
    if (tile_rows < 1) tile_rows = 1;
    g.TY = (rows + tile_rows - 1) / tile_rows;
    const int rw = cols < g.TX + 2 * g.H ? cols : g.TX + 2 * g.H;
    while (g.TY > 1 && (rows < g.TY + 2 * g.H ? rows : g.TY + 2 * g.H) * rw > regmax) --g.TY;
    g.ny = (rows + g.TY - 1) / g.TY;
    g.ntiles = g.nx * g.ny;
    return g;
}

// H = 8 when every CTA owns one tile (its arc masks stay in shared memory for
// the whole sweep, so deep blocking saves team barriers).  When CTAs cycle
// through several tiles the masks are reloaded every round and the halo of a
// deep round dwarfs its tile: H = 3 (NW >= 2) / 4 (NW = 1) measured best
// (C3 21.4 -> 10.4 s, C3q 2.41 -> 1.73 s, C2 68 -> 57 ms, bench C1 472 -> 486
// pairs/s; tools/sweep_cfg.py, round 1).  GZ_BFS_H overrides.
gz4::Geo tile_geo(int rows, int cols, int nb, int nw, int occ) {
    const char *hs = getenv("GZ_BFS_H");
    gz4::Geo g = tile_geo_h(rows, cols, nb, nw, occ, hs ? atoi(hs) : 8);
    if (!hs && g.ntiles > nb) g = tile_geo_h(rows, cols, nb, nw, occ, nw >= 2 ? 3 : 4);
    // one band: the whole grid (row bands override these, solve_launch)
    g.nb = nb; g.rank0 = 0;
    g.t0 = 0; g.t1 = g.ntiles;
    g.c0 = 0; g.c1 = rows * cols;
    g.gg0 = 0; g.gg1 = (rows * cols + 1) / 2;
    g.sys = 0; g.spin_ms = 0; g.nbands = 1;
    return g;
}

// Row-band plan of one problem: band k is a cooperative launch
// of grid[k] CTAs on dev[k] / stream[k]; all launches form one team.  Band k owns
// tile rows [ny k / n, ny (k+1) / n) of the team's tile geometry.
constexpr int MAX_BANDS = 64;
struct BandPlan {
    int n = 0;
    int dev[MAX_BANDS], grid[MAX_BANDS];
    cudaStream_t stream[MAX_BANDS];
    int home = 0;       // device of the caller's stream
    int multi_dev = 0;  // bands on more than one device: system-scope fences
    int spin_ms = 30000;
    gz4::Geo geo;       // team geometry (nb = sum of grid)
};

// Band k's share of the team geometry.
gz4::Geo band_geo(const gz4::Geo &g, int rows, int cols, int n, int k, int rank0, int multi_dev, int spin_ms) {
    gz4::Geo b = g;
    const int ty0 = (int)((long long)g.ny * k / n), ty1 = (int)((long long)g.ny * (k + 1) / n);
    const int P = rows * cols;
    b.t0 = ty0 * g.nx; b.t1 = ty1 * g.nx;
    b.c0 = (ty0 * g.TY < rows ? ty0 * g.TY : rows) * cols;
    b.c1 = (ty1 * g.TY < rows ? ty1 * g.TY : rows) * cols;
    b.gg0 = b.c0 / 2;                                   // a pair straddling a band edge goes to the lower band
    b.gg1 = k + 1 == n ? (P + 1) / 2 : b.c1 / 2;
    b.rank0 = rank0;
    b.sys = multi_dev;
    b.spin_ms = n > 1 ? spin_ms : 0;
    b.nbands = n;
    return b;
}

// Solve one problem whose volume is already in w.vol (layout of the chosen solver).
// A launched, not yet collected solve.
struct Pending {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    unsigned long long *h_ctr = nullptr;   // counters copied back (pinned for asynchronous use)
    int hard = 0, hcap = 0;
    volatile unsigned *progress = nullptr;
    int grid = 0;
    int bfs_h = 0;   // BFS levels per blocked round (the capped schedule depends on it)
    unsigned long long *tbuf = nullptr;
};

// Enqueue one solve of the problem whose volume is already in w.vol (layout of
// the chosen solver) on stream s, using 1/conc of the SMs.  Counters go to
// h_ctr, labels to labels_out; collect with solve_finish after the stream.
// Solver parameters of one problem (the schedule knobs and their tuning
// overrides) and its state pointers into workspace w.
void setup_prob(Prob &p, const Workspace &w, int rows, int cols, int m, const gz_energy *en, const gz_sched *sc,
                const int32_t *lo, const int32_t *hi, int hcap) {
    memset(&p, 0, sizeof(p));
    p.Y = rows; p.G = cols; p.M = m; p.L = m - 1; p.P = rows * cols;
    p.inv_g = 1.0f / (float)cols;
    p.pen = en->penalty; p.inh = en->inhibit; p.hard = en->hard_inhibit ? 1 : 0;
    p.hcap = hcap;
    p.K = sc && sc->rounds_per_sweep > 0 ? sc->rounds_per_sweep : 12;
    p.bfs_cap = sc ? sc->bfs_cap : 0;
    p.max_sweeps = sc ? sc->max_sweeps : 0;
    p.no_wave = sc ? (sc->flags & GZ_SCHED_NO_WAVE) : 0;
    p.capped = sc ? ((sc->flags & GZ_SCHED_CAPPED) != 0) : 0;
    p.init_only = sc ? ((sc->flags & GZ_SCHED_INIT_ONLY) != 0) : 0;
    {
        const char *wd = getenv("GZ_WATCHDOG_MS");
        // default: 20 s plus 1 s per 2 M graph nodes (C3, 261 M nodes: ~150 s)
        const double def_ms = 20000.0 + (double)rows * cols * (m - 1) / 2000.0;
        p.watchdog_ns = (unsigned long long)(wd ? atof(wd) : def_ms) * 1000000ull;
    }
    p.trace = getenv("GZ_TRACE") ? atoi(getenv("GZ_TRACE")) : 0;
    p.lo = lo; p.hi = hi;
    p.vol = w.vol; p.cu = w.cu; p.ph = w.ph; p.pv = w.pv; p.dar = w.dar; p.dbr = w.dbr; p.dad = w.dad; p.dbd = w.dbd;
    p.e = w.e; p.ein = w.ein; p.h = w.h; p.h2 = w.h2; p.reach = w.reach; p.reach2 = w.reach2; p.labels = w.labels;
    p.ctr = w.ctr;
    const int which = choose_solver(m, sc);
    const bool v1 = which == 1;
    // Exact v4 solves stop a relabel early once it is max(24, m) levels deep and has
    // met excess, and double that depth whenever a relabel meets excess only beyond
    // it (the near region is drained).  A fixed depth either wastes levels (C1/C2)
    // or starves far excess (960x540x128: 2m+16 levels -> 1600 sweeps); adaptive:
    // C1 ~420 -> ~490 pairs/s, C2 88 -> 58 ms, C3 30 -> 12 s (tools/bench_tune.py,
    // tools/sweep_cfg.py)
    if (!v1 && p.bfs_cap == 0) p.bfs_cap = which == 4 ? (m > 24 ? m : 24) : 64;
    p.bfs_adapt = (which == 4 && !p.capped) ? 1 : 0;
    if (const char *ba = getenv("GZ_BFS_ADAPT")) p.bfs_adapt = atoi(ba);
    // exact v4 solves (canonical cut: the schedule only affects speed) use their own
    // tuned pulses per sweep instead of the reference's rounds_per_sweep
    if (which == 4 && !p.capped) p.K = m - 12 > 8 ? m - 12 : 8;
    if (which == 4 && !p.capped) {   // tuning overrides (GZ_K pulses per sweep, GZ_BFS_CAP)
        if (const char *k = getenv("GZ_K")) p.K = atoi(k) > 0 ? atoi(k) : p.K;
        if (const char *bc = getenv("GZ_BFS_CAP")) p.bfs_cap = atoi(bc);
    }
    // capped (level-2) solves run rounds_per_sweep pulses per sweep (the reference's
    // parameter, maxflow.py:403-409; 12 by default) and read the labeling off the
    // sink side of the capped preflow (gz_tilesolve.cuh), a speed / quality trade:
    // 24-label ladder L2 b=3, 8 sweeps: K = 12 -> 4.9 ms, energy 791805 (reference
    // L2b3 790883, L1b3 790627 in 5.0 ms); K = 24 -> 7.0 ms, 790728
    // (tools/l2_speed.py, profiles/r2_runs/l2_speed.txt)
    if (p.capped)
        if (const char *ck = getenv("GZ_CAPPED_K")) p.K = atoi(ck) > 0 ? atoi(ck) : p.K;   // tuning override
    if (which == 4 && !p.capped) {   // tail sweeps: few active chains, pulses are cheap next to a global relabel
        const char *kt = getenv("GZ_KTAIL"), *ta = getenv("GZ_TAIL_AFTER");
        // measured (tools/bench_tune.py with adaptive relabels): 64 pulses from the fifth sweep on
        p.k_tail = kt ? atoi(kt) : (p.K > 64 ? p.K : 64);
        p.tail_after = ta ? atoi(ta) : 4;
        const char *tmode = getenv("GZ_TAIL_MODE");
        p.tail_mode = tmode ? atoi(tmode) : 1;
        const char *tc = getenv("GZ_TAIL_CTAS");
        p.tail_ctas = tc ? atoi(tc) : 16;
        const char *al = getenv("GZ_ASYNC_L");
        p.async_l = al ? atoi(al) : 0;
        const char *wl = getenv("GZ_WORKLIST");
        p.worklist = wl ? atoi(wl) : -1;   // -1: auto (gz_tilesolve.cuh)
        const char *wd = getenv("GZ_WL_DEDUPE");
        p.wl_dedupe = wd ? atoi(wd) : 1;   // measured: bench pulses -10%, C3q 1.76 -> 1.60 s
    }
    if (!v1 && p.bfs_cap < 0) p.bfs_cap = 0;            // exhaustive BFS every sweep
    // one-CTA teams (batched pairs): the shared-memory tail mode takes over a sweep
    // once its active groups fit the shared-memory worklist (GZ_TAIL_GROUPS)
    p.tail_groups = getenv("GZ_TAIL_GROUPS") ? atoi(getenv("GZ_TAIL_GROUPS")) : 8;
}

int solve_launch(const Workspace &w, int rows, int cols, int m, const gz_energy *en, const gz_sched *sc,
                 const int32_t *lo, const int32_t *hi, int32_t *labels_out, cudaStream_t s, int hcap, int conc,
                 unsigned long long *h_ctr, Pending *pd, int max_width = -1, const BandPlan *bp = nullptr) {
    Prob p;
    setup_prob(p, w, rows, cols, m, en, sc, lo, hi, hcap);
    static unsigned long long *tbuf = nullptr;
    if (p.trace > 1) {
        if (!tbuf) CK(cudaMalloc((void **)&tbuf, 8192 * 8));
        CK(cudaMemsetAsync(tbuf, 0, 8192 * 8, s));
        p.tbuf = tbuf;
    }
    CK(cudaMemsetAsync(w.ctr, 0, gz::CTR_COUNT * 8, s));
    CK(cudaEventCreate(&pd->e0));
    CK(cudaEventCreate(&pd->e1));
    pd->h_ctr = h_ctr;
    pd->hard = p.hard;
    pd->hcap = p.hcap;
    CK(cudaEventRecord(pd->e0, s));
    const bool win = lo != nullptr;
    const int NW = words_for(m);
    const int which = choose_solver(m, sc);
    const bool v1 = which == 1;
    const void *kern = nullptr;
    const int LPn = lanes_for(m);
    // two CTAs per SM (64 registers, smaller BFS regions) for the m <= 16 instance
    // (spills cost ~12% on a lone solve; with concurrent pair solves the doubled
    // warp count wins ~12%: bench A/B, round 1)
    int occ4 = 1;
    if (LPn == 16) {
        const char *oc = getenv("GZ_OCC");
        occ4 = oc ? (atoi(oc) == 2 ? 2 : 1) : (conc >= 2 ? 2 : 1);
    }
    if (which == 4) {
        kern = LPn == 16 ? gz4::kernel_for(16, 1, win, occ4, 0) : gz4::kernel_for(32, LPn / 32, win, 1, 0);
        // windowed solves whose windows are at most 15 positions wide (the level-1/2
        // fine solves): window-relative 16-lane groups over the absolute rows
        if (win && max_width >= 0 && max_width <= 15 && (LPn == 32 || LPn == 64) && !getenv("GZ_NO_REL"))
            kern = gz4::kernel_for(16, 1, true, 1, LPn / 32);
    } else {
        kern = win ? (const void *)gz_solve_kernel<true> : (const void *)gz_solve_kernel<false>;
    }
    if (!kern) return GZ_ERR_ARG;
    if (!v1) CK(cudaMemsetAsync(w.bits_base, 0, w.bits_bytes, s));
    const int threads = which == 4 ? gz4::BLOCK : 256;
    const size_t dyn_smem = which == 4 ? gz4::smem_bytes(occ4) : 0;
    if (which == 4) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem));
    int grid = 0;
    int rc = coop_grid(kern, threads, &grid, dyn_smem);
    if (rc) return rc;
    if (conc > 1) grid = grid / conc > 0 ? grid / conc : 1;
    if (conc == 1)   // tuning override: CTAs of a lone solve
        if (const char *lg = getenv("GZ_LONE_GRID")) grid = atoi(lg) > 0 && atoi(lg) < grid ? atoi(lg) : grid;
    const int need = (p.P + 255) / 256;
    if (grid > need) grid = need < 1 ? 1 : need;
    gz4::Geo geo{};
    unsigned long long *bar = w.ctr + gz::CTR_BAR0;
    if (which == 4) geo = tile_geo(rows, cols, grid, words_for(m), occ4);
    if (getenv("GZ_DEBUG_PROGRESS")) {
        static unsigned *prog = nullptr;
        if (!prog) CK(cudaHostAlloc((void **)&prog, 65536 * sizeof(unsigned), cudaHostAllocMapped));
        memset(prog, 0, 65536 * sizeof(unsigned));
        unsigned *dprog = nullptr;
        CK(cudaHostGetDevicePointer((void **)&dprog, prog, 0));
        p.progress = dprog;
    }
    gz2::Bits2 bb = w.bits;
    gz3::Arr3 a3{w.vol, w.cu, w.ph, w.pv, w.dar, w.dbr, w.dad, w.dbd, w.e, w.ein, w.h2, w.h, w.IN0, w.IN1};
    void *args1[] = {&p};
    void *args4[] = {&p, &bb, &a3, &geo, &bar};
    if (which == 4 && bp) {
        // row bands: one cooperative launch per band, forked from and joined to s
        p.sys = bp->multi_dev;
        if (occ4 != 1 || bp->geo.ny < bp->n) return GZ_ERR_ARG;
        cudaEvent_t fork;
        CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        CK(cudaEventRecord(fork, s));
        cudaEvent_t joins[MAX_BANDS];
        int rank0 = 0;
        for (int k = 0; k < bp->n; ++k) {
            CK(cudaSetDevice(bp->dev[k]));
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem));
            CK(cudaStreamWaitEvent(bp->stream[k], fork, 0));
            gz4::Geo gk = band_geo(bp->geo, rows, cols, bp->n, k, rank0, bp->multi_dev, bp->spin_ms);
            void *argsk[] = {&p, &bb, &a3, &gk, &bar};
            CK(cudaLaunchCooperativeKernel(kern, dim3(bp->grid[k]), dim3(threads), argsk, dyn_smem, bp->stream[k]));
            CK(cudaEventCreateWithFlags(&joins[k], cudaEventDisableTiming));
            CK(cudaEventRecord(joins[k], bp->stream[k]));
            rank0 += bp->grid[k];
        }
        CK(cudaSetDevice(bp->home));
        for (int k = 0; k < bp->n; ++k) CK(cudaStreamWaitEvent(s, joins[k], 0));
        for (int k = 0; k < bp->n; ++k) cudaEventDestroy(joins[k]);
        cudaEventDestroy(fork);
        grid = rank0;
    } else if (which == 4) {
        if (geo.ntiles < grid) grid = geo.ntiles;   // every CTA owns at least one tile
        geo = tile_geo(rows, cols, grid, words_for(m), occ4);
        CK(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(threads), args4, dyn_smem, s));
    } else {
        CK(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(256), args1, 0, s));
    }
    CK(cudaEventRecord(pd->e1, s));
    pd->progress = p.progress;
    pd->tbuf = p.tbuf;
    pd->grid = grid;
    pd->bfs_h = which == 4 ? (bp ? bp->geo.H : geo.H) : 1;
    CK(cudaMemcpyAsync(h_ctr, w.ctr, gz::CTR_COUNT * 8, cudaMemcpyDeviceToHost, s));
    if (labels_out && labels_out != w.labels)
        CK(cudaMemcpyAsync(labels_out, w.labels, (size_t)p.P * 4, cudaMemcpyDeviceToDevice, s));
    return GZ_OK;
}

// Solver counters of one finished solve -> gz_stats (GZ_OK or its status).
int stats_from_ctr(const unsigned long long *h_ctr, int hard, int hcap, float ms, int bfs_h, gz_stats *st) {
    if (h_ctr[CTR_ABORT]) return GZ_ERR_BANDS;
    if (h_ctr[CTR_STATUS]) return -(int)h_ctr[CTR_STATUS];
    if (st) {
        memset(st, 0, sizeof(*st));
        st->flow = (int64_t)h_ctr[CTR_FLOW];
        if (hard) {   // rescale uncuttable multiples to the reference's 2^56 (see gz_graph.cuh)
            const int64_t k = st->flow / hcap, f = st->flow % hcap;
            st->flow = k * (int64_t)gz::UNCUTTABLE + f;
        }
        st->const_offset = (int64_t)h_ctr[CTR_OFFSET];
        st->presaturated = (int64_t)h_ctr[CTR_PRESAT];
        st->pushes = (int64_t)h_ctr[CTR_PUSHES];
        st->relabels = (int64_t)h_ctr[CTR_RELABELS];
        st->labeling_energy = h_ctr[CTR_HARDVIOL] ? (int64_t)gz::UNCUTTABLE : (int64_t)h_ctr[CTR_ENERGY];
        st->node_updates = (int64_t)h_ctr[CTR_UPDATES];
        st->converged = (int32_t)h_ctr[CTR_CONVERGED];
        st->energy = st->converged ? st->flow + st->const_offset : st->labeling_energy;
        st->sweeps = (int32_t)h_ctr[CTR_SWEEPS];
        // maxflow.py:466-470 counts nodes still holding excess when the solve stops.
        // The reference drains excess back to the source (phase 2), so a converged
        // solve leaves none: every node with excess in a preflow has a residual
        // path back to the source, so it stays active until drained.  This solver
        // stops after phase 1 and its leftover excess is
        // exactly what phase 2 would return; the converged count is therefore 0,
        // like the reference's.  Capped solves report the nodes holding excess
        // at the stop (the level-2 state the labeling is read from).
        st->excess_nodes = (int32_t)h_ctr[CTR_STRANDED];
        st->stranded_excess_nodes = st->converged ? 0 : st->excess_nodes;
        st->bfs_passes = (int32_t)h_ctr[CTR_BFS_PASSES];
        st->reach_passes = (int32_t)h_ctr[CTR_REACH_PASSES];
        st->pulses = (int32_t)h_ctr[CTR_PULSES];
        st->bfs_h = bfs_h;
        st->ms_total = ms;
        for (int q = 0; q < 6; ++q) st->ms_phase[q] = (float)(h_ctr[CTR_T0 + q] * 1e-6);
    }
    return GZ_OK;
}

// Collect a solve once its stream has completed.
int solve_finish(Pending &pd, gz_stats *st) {
    if (pd.tbuf) {   // debug: dump the per-pulse trace
        static unsigned long long h[8192];
        CK(cudaMemcpy(h, pd.tbuf, sizeof(h), cudaMemcpyDeviceToHost));
        for (int i = 0; i < 4096 && h[2 * i + 1]; ++i)
            fprintf(stderr, "gz_pulse sweep %llu pulse %llu groups %llu dt_us %.2f\n", h[2 * i] >> 48,
                    (h[2 * i] >> 32) & 0xffff, h[2 * i] & 0xffffffffull, h[2 * i + 1] * 1e-3);
    }
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, pd.e0, pd.e1));
    cudaEventDestroy(pd.e0);
    cudaEventDestroy(pd.e1);
    return stats_from_ctr(pd.h_ctr, pd.hard, pd.hcap, ms, pd.bfs_h, st);
}

// Synchronous solve (one problem, all SMs).
int solve_planar(const Workspace &w, int rows, int cols, int m, const gz_energy *en, const gz_sched *sc,
                 const int32_t *lo, const int32_t *hi, int32_t *labels_out, gz_stats *st, cudaStream_t s,
                 int hcap = HARD_CAP_DEFAULT, int max_width = -1) {
    unsigned long long h_ctr[gz::CTR_COUNT];
    Pending pd;
    int rc = solve_launch(w, rows, cols, m, en, sc, lo, hi, labels_out, s, hcap, 1, h_ctr, &pd, max_width);
    if (rc) return rc;
    if (pd.progress) {   // debug: poll instead of blocking, report where blocks stall
        const double limit = atof(getenv("GZ_DEBUG_PROGRESS"));
        const double t0 = (double)clock() / CLOCKS_PER_SEC;
        while (cudaEventQuery(pd.e1) == cudaErrorNotReady) {
            if ((double)clock() / CLOCKS_PER_SEC - t0 > limit) {
                fprintf(stderr, "gazecut_b200: solve still running after %.1fs; per-block phase counters:\n", limit);
                for (int i = 0; i < pd.grid; ++i) fprintf(stderr, "%u%c", pd.progress[i], (i % 32 == 31) ? '\n' : ' ');
                fprintf(stderr, "\n");
                fflush(stderr);
                _exit(3);
            }
        }
    }
    CK(cudaStreamSynchronize(s));
    return solve_finish(pd, st);
}

// CTAs per team of the batched pair solves: 2 measured best (C1, 1184 pairs:
// T = 1 / 2 / 4 -> 556 / 623 / 612 pairs/s; the round-1 one-launch-per-pair path
// with 32 hardware queues: 529).  GZ_PAIR_TEAM overrides (0: the round-1 path).
int pair_team() {
    const char *tm = getenv("GZ_PAIR_TEAM");
    return tm ? atoi(tm) : 2;
}

// Teams a batched pair solve runs side by side (one workspace slice each).
int pair_teams(int m) {
    const int T = pair_team();
    if (lanes_for(m) != 16 || T <= 0) {
        const char *cs = getenv("GZ_PAIR_CONC");
        return cs ? atoi(cs) : 8;
    }
    int occ = 2;
    if (const char *oc = getenv("GZ_OCC")) occ = atoi(oc) == 1 ? 1 : 2;
    const void *kern = gz4::pairs_kernel_lp16(occ);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gz4::smem_bytes(occ)) !=
        cudaSuccess)
        return 0;
    int grid = 0;
    if (coop_grid(kern, gz4::BLOCK, &grid, gz4::smem_bytes(occ))) return 0;
    return grid / T;
}

// Batched teams (gz4::gz_pairs_kernel): the whole batch in ONE launch of
// nteams x T CTAs, team k on workspace slice k, pairs handed out by a device
// queue.  One-CTA teams (T = 1, the default) synchronise with CTA barriers
// only and keep up to 2 x 148 pairs in flight.
// The launch plan of a batched solve: teams of T CTAs in one cooperative launch
// (as many as fit the SMs and the workspace), then -- for batches of at least
// four pairs per team -- a tail launch of T2-CTA teams for the last `tail`
// pairs (gz_tilesolve.cuh PairBatch; 1184 C1 pairs: ~1575 -> ~1500 ms per
// batch, profiles/r2_runs/tail_launch.txt).
struct PairsPlan {
    int occ, T, nteams, T2, nt2, tail;
    const void *kern;
    size_t dyn;
};

int plan_pairs(int rows, int cols, int m, int batch, size_t workspace_bytes, int T, PairsPlan &pl) {
    const size_t one = ws_bytes(rows, cols, m);
    pl.T = T;
    pl.occ = 2;
    if (const char *oc = getenv("GZ_OCC")) pl.occ = atoi(oc) == 1 ? 1 : 2;
    pl.kern = gz4::pairs_kernel_lp16(pl.occ);
    pl.dyn = gz4::smem_bytes(pl.occ);
    CK(cudaFuncSetAttribute(pl.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.dyn));
    int grid = 0;
    int rc = coop_grid(pl.kern, gz4::BLOCK, &grid, pl.dyn);
    if (rc) return rc;
    int nteams = grid / T;
    if ((size_t)nteams * one > workspace_bytes) nteams = (int)(workspace_bytes / one);
    if (nteams > batch) nteams = batch;
    if (const char *e = getenv("GZ_PAIR_TEAMS"))   // (tests: fewer teams than pairs on small batches)
        if (atoi(e) > 0 && atoi(e) < nteams) nteams = atoi(e);
    if (nteams < 1) return GZ_ERR_WORKSPACE;
    pl.nteams = nteams;
    int T2 = 8, tail = batch >= 4 * nteams ? batch / 12 : 0;
    if (const char *e = getenv("GZ_PAIR_TEAM2")) T2 = atoi(e);
    if (const char *e = getenv("GZ_PAIR_TAIL")) tail = atoi(e);
    const int nt2 = T2 > T ? nteams * T / T2 : 0;   // T2 > T: never more tail teams than slices
    if (nt2 < 1 || tail < 0) tail = 0;
    if (tail > batch - nteams) tail = batch - nteams > 0 ? batch - nteams : 0;
    pl.T2 = T2;
    pl.nt2 = nt2;
    pl.tail = tail;
    return GZ_OK;
}

int solve_pairs_batched(const uint8_t *left, const uint8_t *right, int batch, int img_h, int img_w, int channels,
                        const gz_cuboid *cb, const gz_energy *energy, const gz_sched *sched, int32_t *labels_out,
                        gz_stats *stats_out, void *workspace, size_t workspace_bytes, cudaStream_t s, int T) {
    const auto h_t0 = std::chrono::steady_clock::now();   // (GZ_PAIR_TIMELINE: host phases)
    auto h_us = [&]() { return (long long)std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - h_t0).count(); };
    long long h_launch = 0, h_tail = 0, h_sync = 0;
    const int rows = cb->y_extent, cols = cb->g_extent, m = cb->m, P = rows * cols;
    const size_t one = ws_bytes(rows, cols, m);
    PairsPlan pl;
    int rc = plan_pairs(rows, cols, m, batch, workspace_bytes, T, pl);
    if (rc) return rc;
    const int occ = pl.occ, nteams = pl.nteams, T2 = pl.T2, nt2 = pl.nt2, tail = pl.tail;
    const void *kern = pl.kern;
    const size_t dyn = pl.dyn;
    int grid = 0;
    Workspace w = carve(workspace, rows, cols, m);
    Prob p;
    gz_sched sc = sched ? *sched : gz_sched{12, 0, 0, 0};
    setup_prob(p, w, rows, cols, m, energy, &sc, nullptr, nullptr, 1 << 30);
    p.tbuf = nullptr;
    p.trace = 0;
    p.labels = nullptr;   // per pair (PairBatch.labels_out)
    if (!getenv("GZ_TAIL_GROUPS")) p.tail_groups = 8;
    // batched teams: no push-time worklist dedupe -- the inbox OR then needs no
    // result (a fire-and-forget reduction) and the consumer's claim bitmap drops
    // the duplicates (1184 C1 pairs: 704 / 710 -> 722 / 728 pairs/s, paired runs)
    if (!getenv("GZ_WL_DEDUPE")) p.wl_dedupe = 0;
    gz4::Geo geo = tile_geo(rows, cols, T, words_for(m), occ);
    gz2::Bits2 bb = w.bits;
    gz3::Arr3 a3{w.vol, w.cu, w.ph, w.pv, w.dar, w.dbr, w.dad, w.dbd, w.e, w.ein, w.h2, w.h, w.IN0, w.IN1};
    gz4::PairBatch pb;
    pb.left = left; pb.right = right; pb.img_w = img_w; pb.ch = channels;
    pb.img_bytes = (size_t)img_h * img_w * channels;
    pb.cb = *cb;
    pb.batch = batch; pb.T = T;
    pb.ws_stride = one;
    pb.bits_bytes = w.bits_bytes;
    pb.labels_out = labels_out;
    DevicePool *pool = device_pool();
    if (!pool) return GZ_ERR_CUDA;
    std::lock_guard<std::mutex> lock(pool->mu);
    unsigned long long *dbuf = nullptr;
    const size_t sbytes = (size_t)batch * gz::CTR_COUNT * 8;
    // tail launch (gz_tilesolve.cuh PairBatch): the last `tail` pairs go to a
    // second launch of T2-CTA teams, issued once the first launch's queue is dry
    const int grid1 = nteams * T, batch1 = batch - tail;
    const size_t tbytes = align_up((size_t)nteams * 4) * 2 + align_up((size_t)(nt2 > 0 ? nt2 : 1) * 4) + 256;
    // per-call device scratch (stats rows, queue, team words) from the pool: a
    // cudaMallocAsync / cudaFreeAsync pair per call let the stream-ordered pool
    // trim at the closing synchronize, which stalled the call 0.2-0.9 s now and
    // then after the kernels were done (tools/pair_timeline.py)
    if ((rc = pool->scratch_ready(sbytes + 256 + tbytes))) return rc;
    dbuf = (unsigned long long *)pool->scratch;
    pb.stats = dbuf;
    pb.queue = (unsigned *)((uint8_t *)dbuf + sbytes);
    uint8_t *tb = (uint8_t *)dbuf + sbytes + 256;
    pb.done = (unsigned *)tb;
    pb.free_slices = tail ? (int *)(tb + align_up((size_t)nteams * 4)) : nullptr;
    pb.pub = (int *)(tb + 2 * align_up((size_t)nteams * 4));
    pb.free_n = (unsigned *)(tb + 2 * align_up((size_t)nteams * 4) + align_up((size_t)(nt2 > 0 ? nt2 : 1) * 4));
    CK(cudaMemsetAsync(pb.queue, 0, 256 + tbytes, s));
    if (tail) CK(cudaMemsetAsync(pb.free_slices, 0xff, (size_t)nteams * 4, s));
    pb.lo = 0;
    pb.batch = batch1;
    pb.tail = 0;
    pb.drained = nullptr;
    // team barrier words and counters of every slice start clear
    for (int k = 0; k < nteams; ++k) {
        Workspace wk = carve((uint8_t *)workspace + (size_t)k * one, rows, cols, m);
        CK(cudaMemsetAsync(wk.ctr, 0, gz::CTR_COUNT * 8, s));
    }
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (tail) {
        if ((rc = pool->flag_ready()) || (rc = pool->streams_ready())) return rc;
        *(volatile unsigned *)pool->flag_host = 0u;
        pb.drained = pool->flag_dev;
        s2 = pool->streams[0] == s ? pool->streams[1] : pool->streams[0];
        CK(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming));
        CK(cudaEventRecord(ev0, s));   // the tail launch follows this call's memsets
        CK(cudaStreamWaitEvent(s2, ev0, 0));
    }
    void *args[] = {&p, &bb, &a3, &geo, &pb};
    grid = grid1;
    const char *tl_path = getenv("GZ_PAIR_TIMELINE");   // debug: per-pair draw / end times, host phases
    cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
    if (tl_path)
        for (auto &e : tev) CK(cudaEventCreate(&e));
    if (tl_path) CK(cudaEventRecord(tev[0], s));
    CK(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(gz4::BLOCK), args, dyn, s));
    if (tl_path) CK(cudaEventRecord(tev[1], s));
    h_launch = h_us();
    gz4::Geo geo2 = geo;
    if (tail) {
        gz4::PairBatch pb2 = pb;
        pb2.T = T2;
        pb2.lo = batch1;
        pb2.batch = batch;
        pb2.queue = pb.queue + 1;
        pb2.tail = 1;
        pb2.drained = nullptr;
        geo2 = tile_geo(rows, cols, T2, words_for(m), occ);
        // wait until the first launch's queue is dry (or the launch is over),
        // then launch the tail teams behind it on a second stream
        while (!*(volatile unsigned *)pool->flag_host) {
            const cudaError_t q = cudaStreamQuery(s);
            if (q == cudaSuccess) break;
            if (q != cudaErrorNotReady) return GZ_ERR_CUDA;
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
        void *args2[] = {&p, &bb, &a3, &geo2, &pb2};
        CK(cudaLaunchKernel(kern, dim3(nt2 * T2), dim3(gz4::BLOCK), args2, dyn, s2));
        if (tl_path) CK(cudaEventRecord(tev[2], s2));
        h_tail = h_us();
        CK(cudaEventRecord(ev1, s2));
        CK(cudaStreamWaitEvent(s, ev1, 0));
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
    }
    if ((rc = pool->pinned_ready((size_t)batch * gz::CTR_COUNT))) return rc;
    CK(cudaMemcpyAsync(pool->pinned, dbuf, sbytes, cudaMemcpyDeviceToHost, s));
    unsigned long long tl[3] = {0ull, 0ull, 0ull};
    if (tl_path) CK(cudaMemcpyAsync(tl, pb.queue, sizeof(tl), cudaMemcpyDeviceToHost, s));
    if (tl_path) CK(cudaEventRecord(tev[3], s));
    const long long h_copy = h_us();
    CK(cudaStreamSynchronize(s));
    h_sync = h_us();
    if (tl_path) {
        if (FILE *fp = fopen(tl_path, "a")) {
            float k1 = 0.f, k2 = 0.f, k3 = 0.f;
            cudaEventElapsedTime(&k1, tev[0], tev[1]);
            if (tail) cudaEventElapsedTime(&k2, tev[0], tev[2]);
            cudaEventElapsedTime(&k3, tev[0], tev[3]);
            fprintf(fp, "batch %d batch1 %d T %d T2 %d teams %d tail_teams %d dry %llu tail_start %llu h_launch_us %lld h_tail_us %lld h_copy_us %lld h_sync_us %lld ev_k1_us %d ev_k2_us %d ev_end_us %d\n",
                    batch, batch1, T, T2, nteams, nt2, tl[1], tl[2], h_launch, h_tail, h_copy, h_sync, (int)(k1 * 1e3f),
                    (int)(k2 * 1e3f), (int)(k3 * 1e3f));
            for (int b = 0; b < batch; ++b) {
                const unsigned long long *h = pool->pinned + (size_t)b * gz::CTR_COUNT;
                fprintf(fp, "pair %d %llu %llu\n", b, h[CTR_TDRAW], h[CTR_TEND]);
            }
            fclose(fp);
        }
        for (auto &e : tev) cudaEventDestroy(e);
    }
    for (int b = 0; b < batch && rc == GZ_OK; ++b) {
        const unsigned long long *h = pool->pinned + (size_t)b * gz::CTR_COUNT;
        rc = stats_from_ctr(h, energy->hard_inhibit ? 1 : 0, 1 << 30, (float)(h[CTR_NS] * 1e-6), b < batch1 ? geo.H : geo2.H,
                            stats_out ? stats_out + b : nullptr);
    }
    if (rc) return rc;
    if (stats_out)
        for (int b = 0; b < batch; ++b)
            if (stats_out[b].energy != stats_out[b].labeling_energy) return GZ_ERR_CONSISTENCY;
    return GZ_OK;
}

}  // namespace

const void *gz4::kernel_for(int LP, int R, bool win, int occ, int rw) {
    if (LP == 16) return kernels_lp16(win, occ, rw);
    if (LP == 32 && R <= 2) return kernels_lp32(R, win);
    if (LP == 32) return kernels_lp32w(R, win);
    return nullptr;
}

namespace {

int check_sm100() {
    int dev = 0, major = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    return major == 10 ? GZ_OK : GZ_ERR_NOGPU;
}

}  // namespace

// ===========================================================================
// C ABI
extern "C" {

size_t gz_workspace_bytes(int32_t rows, int32_t cols, int32_t m) {
    if (rows < 1 || cols < 1 || m < 1 || !index_fits(rows, cols, m)) return 0;
    return ws_bytes(rows, cols, m);
}

int gz_sad_volume(const uint8_t *left, const uint8_t *right, int32_t img_h, int32_t img_w, int32_t channels,
                  const gz_cuboid *cb, int32_t *vol_out, void *stream) {
    if (!cb || !left || !right || !vol_out || channels < 1) return GZ_ERR_ARG;
    if (cb->y_min < 0 || cb->y_min + cb->y_extent > img_h || cb->g_extent < 1 || cb->m < 1) return GZ_ERR_ARG;
    // columns are clamped to [0, width-1] and rows are img_w pixels apart: a
    // cuboid wider than the image would read past the rows (the reference raises
    // IndexError there, geometry.py:325-335)
    if (cb->width < 1 || cb->width > img_w) return GZ_ERR_ARG;
    const int P = cb->y_extent * cb->g_extent;
    k_sad<0><<<(P + 127) / 128, 128, 0, (cudaStream_t)stream>>>(left, right, img_w, channels, *cb, vol_out);
    CK(cudaGetLastError());
    return GZ_OK;
}

int gz_solve_volume(const int32_t *vol, int32_t rows, int32_t cols, int32_t m, const gz_energy *energy,
                    const gz_sched *sched, const int32_t *lo, const int32_t *hi, int32_t *labels_out,
                    gz_stats *stats_out, void *workspace, size_t workspace_bytes, void *stream) {
    if (!vol || !energy || rows < 1 || cols < 1 || m < 1 || (!lo) != (!hi)) return GZ_ERR_ARG;
    if (energy->penalty < 0 || energy->inhibit < 0) return GZ_ERR_ARG;
    if (!index_fits(rows, cols, m)) return GZ_ERR_OVERFLOW;
    if (workspace_bytes < ws_bytes(rows, cols, m)) return GZ_ERR_WORKSPACE;
    int rc = check_sm100();
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    Workspace w = carve(workspace, rows, cols, m);
    const int P = rows * cols;
    if (choose_solver(m, sched) == 4) {
        const int lp = lanes_for(m);
        const long long n = (long long)P * lp;
        k_to_colmajor<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(vol, P, m, lp, w.vol);
    } else {
        k_to_planar<<<(P + 255) / 256, 256, 0, s>>>(vol, P, m, w.vol);
    }
    CK(cudaGetLastError());
    if (m == 1) {
        // single label: everything folds into the offset (flownet.py:305-322)
        CK(cudaMemsetAsync(labels_out ? labels_out : w.labels, 0, (size_t)P * 4, s));
        unsigned long long *d = w.ctr;
        CK(cudaMemsetAsync(d, 0, 16, s));
        gz_energy en = *energy;
        k_total_energy<<<(P + 255) / 256, 256, 0, s>>>(labels_out ? labels_out : w.labels, vol, rows, cols, 1, en, d);
        unsigned long long hv[2];
        CK(cudaMemcpyAsync(hv, d, 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (stats_out) {
            memset(stats_out, 0, sizeof(*stats_out));
            stats_out->const_offset = (int64_t)hv[0];
            stats_out->energy = stats_out->labeling_energy = (int64_t)hv[0];
            stats_out->converged = 1;
        }
        return GZ_OK;
    }
    // int32 device state: the total source capacity bounds every excess,
    // residual and flow value, so it must fit (and picks the hard stand-in)
    CK(cudaMemsetAsync(w.ctr, 0, 24, s));
    k_source_caps<<<(P + 255) / 256, 256, 0, s>>>(vol, rows, cols, m, lo, hi, *energy, w.ctr);
    CK(cudaGetLastError());
    unsigned long long census[3];
    CK(cudaMemcpyAsync(census, w.ctr, 24, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const unsigned long long lim = 0x7fffffffull;
    int hcap = HARD_CAP_DEFAULT;
    if (energy->hard_inhibit) {
        unsigned long long hc = 1ull << 16;
        while (hc <= census[0]) hc <<= 1;
        if (census[0] >= lim || (census[1] + 1) * hc + census[0] >= lim) return GZ_ERR_OVERFLOW;
        hcap = (int)hc;
    } else if (census[0] >= lim) {
        return GZ_ERR_OVERFLOW;
    }
    return solve_planar(w, rows, cols, m, energy, sched, lo, hi, labels_out, stats_out, s, hcap,
                        lo ? (int)census[2] : -1);
}

int gz_solve_pairs(const uint8_t *left, const uint8_t *right, int32_t batch, int32_t img_h, int32_t img_w,
                   int32_t channels, const gz_cuboid *cb, const gz_energy *energy, const gz_sched *sched,
                   int32_t *labels_out, gz_stats *stats_out, void *workspace, size_t workspace_bytes,
                   void *stream) {
    if (!cb || !energy || batch < 1 || channels < 1 || cb->m < 2) return GZ_ERR_ARG;
    if (cb->y_min < 0 || cb->y_min + cb->y_extent > img_h || cb->width > img_w || cb->width < 1) return GZ_ERR_ARG;
    if (cb->g_extent < 1 || cb->y_extent < 1) return GZ_ERR_ARG;
    const int rows = cb->y_extent, cols = cb->g_extent, m = cb->m, P = rows * cols;
    if (!index_fits(rows, cols, m)) return GZ_ERR_OVERFLOW;
    const size_t one = ws_bytes(rows, cols, m);
    if (workspace_bytes < one) return GZ_ERR_WORKSPACE;
    int rc = check_sm100();
    if (rc) return rc;
    // SAD costs are <= 255*channels, which bounds the total source capacity
    const unsigned long long fin = (unsigned long long)P * 255ull * (unsigned long long)channels;
    if (fin >= (energy->hard_inhibit ? (1ull << 29) : 0x7fffffffull)) return GZ_ERR_OVERFLOW;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t img = (size_t)img_h * img_w * channels;
    const int which = choose_solver(m, sched);
    // 16-lane chains (m <= 16, BASELINE config 4): one launch of one-CTA teams
    // (GZ_PAIR_TEAM = CTAs per team; 0 = one cooperative launch per pair on
    // its own stream, the round-1 path)
    {
        const int T = pair_team();
        if (which == 4 && lanes_for(m) == 16 && T > 0 && !(sched && (sched->flags & (GZ_SCHED_CAPPED | GZ_SCHED_INIT_ONLY))))
            return solve_pairs_batched(left, right, batch, img_h, img_w, channels, cb, energy, sched, labels_out,
                                       stats_out, workspace, workspace_bytes, (cudaStream_t)stream, T);
    }
    // Concurrent solves: up to `conc` pairs run at once, each a cooperative launch
    // over 1/conc of the SMs on its own stream with its own workspace slice.
    int conc = 8;   // measured: 1 -> 250, 4 -> 366, 8 -> ~400 pairs/s (C1, 64 pairs per call)
    if (const char *cs = getenv("GZ_PAIR_CONC")) conc = atoi(cs);
    if (conc > DevicePool::MAX_STREAMS) conc = DevicePool::MAX_STREAMS;
    if ((size_t)conc * one > workspace_bytes) conc = (int)(workspace_bytes / one);
    if (conc > batch) conc = batch;
    if (which != 4 || conc < 1) conc = 1;
    DevicePool *pool = device_pool();
    if (!pool) return GZ_ERR_CUDA;
    std::lock_guard<std::mutex> lock(pool->mu);
    if (conc > 1 && (rc = pool->streams_ready())) return rc;
    if ((rc = pool->pinned_ready((size_t)batch * gz::CTR_COUNT))) return rc;
    cudaStream_t *streams = pool->streams;
    unsigned long long *pinned = pool->pinned;
    cudaEvent_t fork = nullptr;
    if (conc > 1) {
        CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        CK(cudaEventRecord(fork, s));
        for (int k = 0; k < conc; ++k) CK(cudaStreamWaitEvent(streams[k], fork, 0));
    }
    Pending *pend = new Pending[batch];
    auto enqueue = [&](int b, int k) -> int {   // data term + solve of pair b on slot k
        cudaStream_t sk = conc > 1 ? streams[k] : s;
        Workspace w = carve((uint8_t *)workspace + (size_t)k * one, rows, cols, m);
        if (which == 4)
            k_sad<2><<<(P + 127) / 128, 128, 0, sk>>>(left + b * img, right + b * img, img_w, channels, *cb, w.vol,
                                                      lanes_for(m));
        else
            k_sad<1><<<(P + 127) / 128, 128, 0, sk>>>(left + b * img, right + b * img, img_w, channels, *cb, w.vol);
        if (cudaGetLastError() != cudaSuccess) return GZ_ERR_CUDA;
        return solve_launch(w, rows, cols, m, energy, sched, nullptr, nullptr, labels_out + (size_t)b * P, sk, 1 << 30,
                            conc, pinned + (size_t)b * gz::CTR_COUNT, &pend[b]);
    };
    const char *dy = getenv("GZ_PAIR_DYNAMIC");
    if (conc > 1 && (!dy || atoi(dy))) {
        // Dynamic dispatch: every slot holds at most two pairs (one running, one
        // queued behind it); the host hands the next pair to the first slot whose
        // oldest pair has finished.  Pair solve times vary by 2x, so a static
        // round-robin of 8 pairs per slot left the step waiting on the slowest
        // slot (step 149 ms against 124 ms of mean slot work, round 1).
        std::vector<std::vector<int>> q(conc);
        int next = 0;
        for (int d = 0; d < 2; ++d)
            for (int k = 0; k < conc && next < batch && rc == GZ_OK; ++k) {
                rc = enqueue(next, k);
                q[k].push_back(next++);
            }
        while (rc == GZ_OK) {
            bool any = false;
            for (int k = 0; k < conc && rc == GZ_OK; ++k) {
                if (q[k].empty()) continue;
                any = true;
                const cudaError_t e = cudaEventQuery(pend[q[k].front()].e1);
                if (e == cudaErrorNotReady) continue;
                if (e != cudaSuccess) { rc = GZ_ERR_CUDA; break; }
                q[k].erase(q[k].begin());
                if (next < batch) {
                    rc = enqueue(next, k);
                    q[k].push_back(next++);
                }
            }
            if (!any) break;
        }
    } else {
        for (int b = 0; b < batch && rc == GZ_OK; ++b) {
            rc = enqueue(b, b % conc);
            if (rc) break;
            if (conc == 1) {   // one at a time: collect now (keeps the pinned slot reuse trivial)
                if (cudaStreamSynchronize(s) != cudaSuccess) { rc = GZ_ERR_CUDA; break; }
                rc = solve_finish(pend[b], stats_out ? stats_out + b : nullptr);
                pend[b].e0 = nullptr;
            }
        }
    }
    if (conc > 1) {
        for (int k = 0; k < conc; ++k) {
            cudaEvent_t join;
            cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
            cudaEventRecord(join, streams[k]);
            cudaStreamWaitEvent(s, join, 0);
            cudaEventDestroy(join);
        }
        cudaEventDestroy(fork);
        if (cudaStreamSynchronize(s) != cudaSuccess && rc == GZ_OK) rc = GZ_ERR_CUDA;
        for (int b = 0; b < batch; ++b) {
            if (!pend[b].e0) continue;
            const int r = solve_finish(pend[b], stats_out ? stats_out + b : nullptr);
            if (rc == GZ_OK) rc = r;
        }
    }
    delete[] pend;
    if (rc) return rc;
    if (stats_out)
        for (int b = 0; b < batch; ++b)
            if (stats_out[b].energy != stats_out[b].labeling_energy) return GZ_ERR_CONSISTENCY;
    return GZ_OK;
}

int gz_solve_pairs_host(const uint8_t *left_host, const uint8_t *right_host, int32_t batch, int32_t img_h,
                        int32_t img_w, int32_t channels, const gz_cuboid *cb, const gz_energy *energy,
                        const gz_sched *sched, int32_t *labels_host, gz_stats *stats_host, void *workspace,
                        size_t workspace_bytes, void *stream) {
    if (!cb || batch < 1) return GZ_ERR_ARG;
    const int P = cb->y_extent * cb->g_extent;
    const size_t img = (size_t)img_h * img_w * channels * batch;
    const size_t one = ws_bytes(cb->y_extent, cb->g_extent, cb->m);
    const size_t io = 2 * align_up(img) + align_up((size_t)batch * P * 4) + 256;
    if (workspace_bytes < one + io) return GZ_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    // device copies of the inputs / labels at the start, solver workspace after
    uint8_t *base = (uint8_t *)(((uintptr_t)workspace + 255) & ~(uintptr_t)255);
    uint8_t *dl = base, *dr = dl + align_up(img);
    int32_t *dlab = (int32_t *)(dr + align_up(img));
    uint8_t *wsp = (uint8_t *)dlab + align_up((size_t)batch * P * 4);
    const size_t ws_left = workspace_bytes - (size_t)(wsp - (uint8_t *)workspace);
    CK(cudaMemcpyAsync(dl, left_host, img, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dr, right_host, img, cudaMemcpyHostToDevice, s));
    int rc = gz_solve_pairs(dl, dr, batch, img_h, img_w, channels, cb, energy, sched, dlab, stats_host, wsp, ws_left, s);
    if (rc) return rc;
    CK(cudaMemcpyAsync(labels_host, dlab, (size_t)batch * P * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return GZ_OK;
}

int gz_total_energy(const int32_t *labels, const int32_t *vol, int32_t rows, int32_t cols, int32_t m,
                    const gz_energy *energy, int64_t *energy_out, void *stream) {
    if (!labels || !vol || !energy || !energy_out || rows < 1 || cols < 1 || m < 1) return GZ_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    // energy_out must hold 2 int64: [0] energy, [1] hard-inhibit violation flag
    CK(cudaMemsetAsync(energy_out, 0, 16, s));
    const int P = rows * cols;
    k_total_energy<<<(P + 255) / 256, 256, 0, s>>>(labels, vol, rows, cols, m, *energy,
                                                   (unsigned long long *)energy_out);
    CK(cudaGetLastError());
    return GZ_OK;
}

int gz_coarsen(const int32_t *vol, int32_t rows, int32_t cols, int32_t m, int32_t block, int32_t *coarse_out,
               void *stream) {
    if (!vol || !coarse_out || block < 1 || rows < 1 || cols < 1 || m < 1) return GZ_ERR_ARG;
    const long long n = (long long)((rows + block - 1) / block) * ((cols + block - 1) / block) * ((m + block - 1) / block);
    k_coarsen<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(vol, rows, cols, m, block, coarse_out);
    CK(cudaGetLastError());
    return GZ_OK;
}

int gz_thin_skin(const int32_t *coarse_labels, int32_t crows, int32_t ccols, int32_t rows, int32_t cols, int32_t m,
                 int32_t block, int32_t radius, int32_t *lo_out, int32_t *hi_out, void *stream) {
    if (!coarse_labels || !lo_out || !hi_out || block < 1 || radius < 0 || rows < 1 || cols < 1 || m < 1)
        return GZ_ERR_ARG;
    // the coarse grid must cover the fine one (k_thin_skin reads coarse[(y/b, g/b)])
    if ((long long)crows * block < rows || (long long)ccols * block < cols) return GZ_ERR_ARG;
    const int P = rows * cols;
    k_thin_skin<<<(P + 255) / 256, 256, 0, (cudaStream_t)stream>>>(coarse_labels, crows, ccols, rows, cols, m, block,
                                                                  radius, lo_out, hi_out);
    CK(cudaGetLastError());
    return GZ_OK;
}

int gz_pairs_launches(int32_t rows, int32_t cols, int32_t m, int32_t batch, size_t workspace_bytes) {
    if (rows < 1 || cols < 1 || m < 2 || batch < 1 || !index_fits(rows, cols, m)) return GZ_ERR_ARG;
    int rc = check_sm100();
    if (rc) return rc;
    const int T = pair_team();
    if (choose_solver(m, nullptr) != 4 || lanes_for(m) != 16 || T < 1) return -1;
    PairsPlan pl;
    if ((rc = plan_pairs(rows, cols, m, batch, workspace_bytes, T, pl))) return rc;
    return pl.tail ? 2 : 1;
}

size_t gz_pairs_workspace_bytes(int32_t rows, int32_t cols, int32_t m, int32_t batch) {
    if (rows < 1 || cols < 1 || m < 2 || batch < 1 || !index_fits(rows, cols, m)) return 0;
    int k = pair_teams(m);
    if (k < 1) return 0;
    if (k > batch) k = batch;
    return (size_t)k * ws_bytes(rows, cols, m);
}

const char *gz_status_string(int status) {
    switch (status) {
    case GZ_OK: return "ok";
    case GZ_ERR_ARG: return "invalid argument";
    case GZ_ERR_CUDA: return "CUDA runtime error";
    case GZ_ERR_WORKSPACE: return "workspace too small";
    case GZ_ERR_CONSISTENCY: return "cut cost != labeling energy";
    case GZ_ERR_OVERFLOW: return "capacities exceed the int32 device state";
    case GZ_ERR_NOCONVERGE: return "iteration guard tripped";
    case GZ_ERR_NOGPU: return "no sm_100 GPU";
    case GZ_ERR_BANDS: return "row-band launches were not co-resident (team barrier timed out)";
    }
    return "unknown status";
}

const char *gz_build_info(void) { return "gazecut_b200 v4 sm_100a tile-owned persistent push-relabel (temporally blocked BFS)"; }

}  // extern "C"

#include "gz_bands.cuh"
#include "gz_eval.cuh"
#include "gz_csr.cuh"
