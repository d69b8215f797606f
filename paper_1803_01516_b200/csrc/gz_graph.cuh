// gz_graph.cuh -- implicit Ishikawa layered graph on the (level, row, gaze) grid.
//
// The reference builds an explicit CSR network (flownet.py:102-222).  Here the
// graph is never materialised: node (t, c) for chain position t = 1..M-1 of site
// c = y*G + g lives at flat index t*P + c (P = Y*G, "plane-major"), and the
// 14 arcs of a node are enumerated by index arithmetic.  Residual state:
//
//   cu [k][c]  forward residual of chain arc k (position k -> k+1), k = 0..M-1.
//              The reverse chain arc is UNCUTTABLE (flownet.py:131) and never
//              saturates, so it is not stored.
//   ph [t][c]  residual of the same-level arc (y,g,t)->(y,g+1,t); the reverse
//              residual is 2*penalty - ph (capacity penalty each way,
//              flownet.py:147-161).
//   pv [t][c]  same for (y,g,t)->(y+1,g,t).
//   dar[t][c]  flow on the inhibit diagonal (y,g,t)->(y,g+1,t-1)   (flownet.py:163-180,
//   dbr[t][c]  flow on (y,g+1,t)->(y,g,t-1)                         direction 0 / 1,
//   dad[t][c]  flow on (y,g,t)->(y+1,g,t-1)                         forward capacity
//   dbd[t][c]  flow on (y+1,g,t)->(y,g,t-1)                         inhibit, reverse 0)
//
// Label windows (flownet.py:17-21, 92-99): position t of site c is the source
// if t <= lo[c], the sink if t > hi[c], a real node otherwise.  Arcs into
// sink positions are exits to the sink; arcs into source positions are never
// used (the solver stops after phase 1); arcs out of source
// positions are saturated at initialisation; source->sink arcs fold into the
// constant offset exactly as flownet.py:124-125,153-154,172-173 do.
#pragma once
#include <cstdint>

namespace gz {

constexpr int32_t HINF = 0x3fffffff;        // "cannot reach the sink"
// Hard inhibit: UNCUTTABLE diagonals get a finite stand-in capacity p.hcap, a
// power of two above the total finite source capacity of the problem (chosen
// on the host by a device pre-pass).  A minimum cut that crosses k uncuttable
// arcs then has value k*hcap + f with f < hcap on the device and is reported
// as k*2^56 + f, the reference's value.  If (k_max+1)*hcap would not fit the
// int32 state the solve returns GZ_ERR_OVERFLOW instead of a wrong answer.
constexpr int32_t HARD_CAP_DEFAULT = 1 << 27;
constexpr long long UNCUTTABLE = 1LL << 56; // energy.py:34

// arc slots of a node, in push order
enum Arc : int {
    A_UP = 0,      // chain (t -> t+1)
    A_SR, A_SL, A_SD, A_SU,   // same level  right/left/down/up
    A_UR, A_UL, A_UD, A_UU,   // diagonal up (t -> t+1) = reverse of neighbour's inhibit diagonal
    A_DR, A_DL, A_DD, A_DU,   // diagonal down (t -> t-1) = inhibit diagonal
    A_DN,          // chain (t -> t-1), infinite
    A_COUNT
};

enum Kind : int { K_SRC = 0, K_REAL = 1, K_SNK = 2 };

struct Prob {
    int Y, G, M, L;      // L = M-1 chain positions carry nodes
    int P;               // Y*G
    float inv_g;         // 1 / G (fast site-row division, gz_chain.cuh:div_g)
    int pen, inh, hard;
    int hcap;            // stand-in capacity of uncuttable inhibit arcs (hard mode)
    int K;               // pulses per sweep
    int k_tail, tail_after;   // v4: pulses per sweep from sweep `tail_after` on (0 = K)
    int tail_mode;            // v4: hand nearly empty pulse phases to one CTA
    int tail_ctas;            // v4: tail mode once at most this many CTAs had work (GZ_TAIL_CTAS)
    int async_l;              // v4: > 0 = asynchronous pulses, this many iterations per team barrier
    int wl_dedupe;            // v4 exact: push-time dedupe of worklist entries (GZ_WL_DEDUPE)
    int worklist;             // v4 exact: later pulses of a sweep consume a global worklist (1 on, 0 off, -1 auto)
    int bfs_adapt;            // v4: double the BFS early-stop depth when excess lies only beyond it
    int bfs_cap;         // lateral relaxations per non-final global relabel (0 = exact)
    int max_sweeps;      // honoured when capped
    int capped;
    unsigned long long watchdog_ns, t_start_ns;   // 0 = no watchdog; start stamped on device
    volatile unsigned *progress;                  // debug: per-block phase counter (mapped host memory) or null
    int trace;                                    // debug: 1 per-sweep device printf, 2 per-pulse trace (env GZ_TRACE)
    unsigned long long *tbuf;                     // debug: per-pulse (sweep|pulse|groups, ns) records
    int no_wave;         // skip the initial chain wave
    const int32_t *lo, *hi;   // windowed only
    int32_t *vol, *cu, *ph, *pv, *dar, *dbr, *dad, *dbd;
    int32_t *e, *ein, *h, *h2;
    int32_t *reach, *reach2, *labels;
    unsigned long long *ctr;  // counters, see CTR_*
    int sys;                  // row bands spanning GPUs: system-scope global atomics (gz_atomic_*)
    int init_only;            // stop after the initialisation (graph export, gz_export_arcs)
    int tail_groups;          // one-CTA teams: enter the shared-memory tail mode at <= this many active groups
};

// Global-memory atomics of the v4 solver that can land in another GPU's band
// (inboxes, chain residuals, counters): system scope when the team spans GPUs,
// so peer-memory atomics are formally atomic against the owner GPU's own.
// One uniform branch otherwise.
template <typename T>
__device__ __forceinline__ T gz_atomic_add(const Prob &p, T *a, T v) {
    return p.sys ? atomicAdd_system(a, v) : atomicAdd(a, v);
}
template <typename T>
__device__ __forceinline__ T gz_atomic_or(const Prob &p, T *a, T v) {
    return p.sys ? atomicOr_system(a, v) : atomicOr(a, v);
}

enum Ctr : int {
    CTR_FLOW = 0, CTR_OFFSET, CTR_PRESAT, CTR_PUSHES, CTR_RELABELS, CTR_ENERGY, CTR_HARDVIOL,
    CTR_SWEEPS, CTR_BFS_PASSES, CTR_REACH_PASSES, CTR_STATUS, CTR_CONVERGED, CTR_STRANDED, CTR_PULSES,
    CTR_TDRAW = 14,     // batched pair solves: %globaltimer when the pair was drawn (stats rows only)
    CTR_TEND = 15,      // batched pair solves: %globaltimer when it finished (stats rows only)
    CTR_FLAG0 = 16,     // 3 rotating "changed" flags
    CTR_ACT0 = 20,      // 3 rotating active counters
    CTR_T0 = 24,        // 6 phase timers (ns): init, mask build, bfs, pulses, reach, tail
    CTR_TRACE = 35,     // debug trace accumulator (GZ_TRACE=2)
    CTR_TQN = 36,       // tail-mode global worklist length
    CTR_ABORT = 37,     // multi-launch (row-band) team gave up waiting at a barrier
    CTR_NS = 38,        // batched pair solves: device time of the pair (ns, %globaltimer)
    CTR_PAIR = 39,      // batched pair solves: the pair a team is working on
    CTR_UPDATES = 30,   // node updates performed by pulses (v4)
    CTR_BAR0 = 32,      // 3 rotating team-barrier words (v4)
    CTR_COUNT = 40
};

__host__ __device__ inline size_t plane_elems(int M, int P) { return (size_t)M * (size_t)P; }

}  // namespace gz
