/*
 * gazecut_b200.h -- C ABI of the B200-native gaze-line stereo graph-cut path.
 *
 * Drop-in boundary for the reference package `gazecut` (arXiv 1803.01516).
 * The reference has no FFI: its boundary is the Python API exported by
 * pkg/src/gazecut/__init__.py:11-97.  Each entry point below replaces the
 * reference function named beside it; the Python mirror in
 * paper_1803_01516_b200/ binds them with ctypes.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers unless the name ends in _host.
 *  - Calls are ordered on the given stream (a cudaStream_t passed as void*;
 *    NULL = legacy default stream).  Functions that fill a gz_stats block
 *    synchronise the stream before returning.
 *  - Return value: GZ_OK (0) or a negative gz_status.
 *  - Volumes cross the ABI as int32 in the reference's (rows, cols, m)
 *    order (energy.py:83-114 returns int64; the Python mirror range-checks
 *    and narrows on upload).
 *  - Labelings are int32 (rows, cols), cuboid-local label indices, exactly
 *    as maxflow.py:362-373 extract_labeling returns them.
 */
#ifndef GAZECUT_B200_H
#define GAZECUT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum gz_status {
    GZ_OK = 0,
    GZ_ERR_ARG = -1,          /* ValueError in the reference (bad shape / window / params) */
    GZ_ERR_CUDA = -2,         /* a CUDA runtime call failed */
    GZ_ERR_WORKSPACE = -3,    /* workspace smaller than gz_workspace_bytes() */
    GZ_ERR_CONSISTENCY = -4,  /* InternalConsistencyError (maxflow.py:51-52): cut cost != labeling energy */
    GZ_ERR_OVERFLOW = -5,     /* capacities too large for the int32 device state */
    GZ_ERR_NOCONVERGE = -6,   /* internal iteration guard tripped (never expected) */
    GZ_ERR_NOGPU = -7,        /* no sm_100 device */
    GZ_ERR_BANDS = -8         /* row-band launches were not co-resident (team barrier timed out) */
};

/* geometry.py:61-138 CuboidSpec (the fields the data term needs) */
typedef struct {
    int32_t width, height;     /* image size the cuboid was built for */
    int32_t g_min, g_extent;
    int32_t y_min, y_extent;
    int32_t d_min, m;          /* first depth number, number of labels */
} gz_cuboid;

/* geometry.py:61-138 CuboidSpec offsets for the ground-truth transform
 * (imaging.py:155-201); rows/cols = y_extent/g_extent, m = d_extent. */
typedef struct {
    int32_t g_min, y_min, d_min, rows, cols, m;
    int32_t offset1, offset2, offset3, lw_offset, rw_offset, h_offset;
} gz_gaze;

/* energy.py:37-50 EnergyParams */
typedef struct {
    int32_t penalty, inhibit, hard_inhibit;
} gz_energy;

/* Solver schedule.  maxflow.py:403-409 maxflow_push_relabel arguments plus
 * the device schedule knobs.  Zero-initialised = the defaults. */
typedef struct {
    int32_t rounds_per_sweep;  /* synchronous push/relabel pulses per sweep (default 12) */
    int32_t max_sweeps;        /* sweep cap, honoured only with GZ_SCHED_CAPPED (level-2 mode) */
    int32_t bfs_cap;           /* BFS depth before a global relabel may stop at the first active node
                                  (0 = library default, < 0 = exhaustive every sweep) */
    int32_t flags;             /* GZ_SCHED_NO_WAVE: skip the chain wave (maxflow.py:422 presaturate=False);
                                  GZ_SCHED_CAPPED: stop after max_sweeps sweeps (maxflow.py:447-449) */
} gz_sched;

#define GZ_SCHED_NO_WAVE 1
#define GZ_SCHED_CAPPED 2
#define GZ_SCHED_V1 4      /* force the v1 (column-relaxation) solver; debugging/comparison */
#define GZ_SCHED_V2 8      /* retired v2 solver (deleted in round 2); accepted and ignored (v4 runs) */
#define GZ_SCHED_V3 16     /* retired v3 solver; accepted and ignored (v4 runs) */
#define GZ_SCHED_INIT_ONLY 32  /* stop after the solver's initialisation (graph export, gz_export_arcs) */

/* maxflow.py:460-471 + 506-509 stats keys, plus device timings. */
typedef struct {
    int64_t flow, energy, const_offset, nodes, arcs, presaturated, pushes, relabels;
    int64_t labeling_energy;       /* energy.py:129-155 recomputed on device */
    int64_t node_updates;          /* node updates done by push/relabel pulses (v4; roofline units) */
    int32_t sweeps, converged, stranded_excess_nodes, bfs_passes, reach_passes, pulses;
    int32_t bfs_h;                 /* BFS levels per temporally blocked round (v4): the capped level-2
                                      schedule's early-stop granularity (oracle/gz_oracle.c restates it) */
    int32_t excess_nodes;          /* nodes holding excess when the solve stopped (phase-1 leftover that
                                      the reference's phase 2 would return to the source) */
    float ms_total;                /* device time of the solve (CUDA events) */
    float ms_phase[6];             /* in-kernel phase times: init, mask build, global relabel, pulses,
                                      extraction, energy/labels (v2 solver; 0 for v1) */
} gz_stats;

/* Device bytes the caller must provide as workspace for one problem of the
 * given site grid and label count (batch problems: multiply). */
size_t gz_workspace_bytes(int32_t rows, int32_t cols, int32_t m);

/* energy.py:83-114 sad_volume.  left/right: uint8 (height, width, channels)
 * row-major; vol_out: int32 (y_extent, g_extent, m). */
int gz_sad_volume(const uint8_t *left, const uint8_t *right, int32_t img_h, int32_t img_w,
                  int32_t channels, const gz_cuboid *cuboid, int32_t *vol_out, void *stream);

/* maxflow.py:481-510 solve_exact (lo == hi == NULL) and
 * hierarchy.py:76-89 _solve_restricted_exact (per-site windows lo/hi, int32
 * rows*cols, 0 <= lo <= hi < m).  vol: int32 (rows, cols, m).
 * labels_out: int32 (rows, cols).  The source side (maxflow.py:355-359) is
 * the prefix lo+1 .. label of every chain, so it is derived from the labels. */
int gz_solve_volume(const int32_t *vol, int32_t rows, int32_t cols, int32_t m, const gz_energy *energy,
                    const gz_sched *sched, const int32_t *lo, const int32_t *hi, int32_t *labels_out,
                    gz_stats *stats_out, void *workspace, size_t workspace_bytes,
                    void *stream);

/* Fused path: sad_volume + solve_exact for `batch` stereo pairs laid out
 * back to back (left/right: batch x height x width x channels uint8).
 * labels_out: batch x (y_extent, g_extent) int32; stats_out: batch entries
 * (host memory).  workspace: k * gz_workspace_bytes(y_extent, g_extent, m)
 * runs up to k pair solves at once.  m <= 16 (BASELINE config 4): ONE launch
 * of teams of GZ_PAIR_TEAM (2) CTAs, team k on workspace slice k, pairs handed
 * out by a device queue (gz4::gz_pairs_kernel; size the workspace with
 * gz_pairs_workspace_bytes); for batches of at least four pairs per team the
 * last twelfth of the pairs go to a second launch of 8-CTA teams on another
 * stream, issued when the first launch's queue runs dry (GZ_PAIR_TAIL /
 * GZ_PAIR_TEAM2 override; gz_pairs_launches).  Otherwise up to GZ_PAIR_CONC (8) cooperative
 * launches over 1/k of the SMs each, one stream per slice.  At least one
 * slice is required.  Calls on one device are serialised (a per-device lock
 * guards the stream pool and the pinned counter buffer). */
int gz_solve_pairs(const uint8_t *left, const uint8_t *right, int32_t batch, int32_t img_h, int32_t img_w,
                   int32_t channels, const gz_cuboid *cuboid, const gz_energy *energy, const gz_sched *sched,
                   int32_t *labels_out, gz_stats *stats_out, void *workspace, size_t workspace_bytes,
                   void *stream);

/* Workspace for gz_solve_pairs to keep as many pairs of `batch` in flight as
 * the device runs at once (m <= 16: one workspace slice per team of the
 * batched launch, GZ_PAIR_TEAM CTAs per team; otherwise GZ_PAIR_CONC slices).
 * Queries the current device; 0 on error. */
size_t gz_pairs_workspace_bytes(int32_t rows, int32_t cols, int32_t m, int32_t batch);

/* Kernel launches gz_solve_pairs makes for `batch` pairs of this shape with a
 * workspace of workspace_bytes on the current device: 1 or 2 (the batched
 * launch, plus its tail launch), or -1 when the batch takes the per-pair
 * launch path (m > 16).  Negative gz_status on error. */
int gz_pairs_launches(int32_t rows, int32_t cols, int32_t m, int32_t batch, size_t workspace_bytes);

/* Same as gz_solve_pairs with HOST buffers (pinned or pageable): copies in,
 * solves, copies labels out.  The reference-facing end-to-end call. */
int gz_solve_pairs_host(const uint8_t *left_host, const uint8_t *right_host, int32_t batch, int32_t img_h,
                        int32_t img_w, int32_t channels, const gz_cuboid *cuboid, const gz_energy *energy,
                        const gz_sched *sched, int32_t *labels_host, gz_stats *stats_host, void *workspace,
                        size_t workspace_bytes, void *stream);

/* Row-band solve of ONE volume too large for one GPU (SURVEY.md §8(e),
 * BASELINE config 5).  Same semantics as gz_solve_volume (replaces
 * maxflow.py:481-510 solve_exact / maxflow.py:403-478 for exact solves; the
 * cut is canonical, so the result is bit-identical to the one-launch solve),
 * but the site rows are split into nbands bands: band k's rows of every state
 * plane live in the HBM of devices[k] (one virtual range, CUDA VMM) and band k
 * runs as a cooperative launch on devices[k].  All launches form one team;
 * arcs across a band edge are read and written in place over NVLink (peer
 * loads, stores, atomics).  devices may repeat: bands on one GPU split its SMs.
 * HOST buffers: vol_host (rows, cols, m) int32, lo_host/hi_host (rows, cols)
 * int32 or both NULL, labels_host (rows, cols) int32 out, stats_out host.
 * Exact solves only (GZ_SCHED_CAPPED is rejected); m <= 256.
 * Env GZ_BAND_SPIN_MS: a band that waits this long at a team barrier aborts
 * the solve with GZ_ERR_BANDS instead of hanging (30000). */
int gz_solve_volume_banded(const int32_t *vol_host, int32_t rows, int32_t cols, int32_t m,
                           const gz_energy *energy, const gz_sched *sched, const int32_t *lo_host,
                           const int32_t *hi_host, int32_t nbands, const int32_t *devices,
                           int32_t *labels_host, gz_stats *stats_out);

/* imaging.py:155-201 ground_truth_to_depth on device.  gt: (img_h, img_w)
 * uint8 disparity * scale, 0 = none.  depth_out (rows, cols) int32 cuboid-local
 * depth numbers (nearest surface wins), valid_out uint8, counts_out 4 int64:
 * out_of_range, off_grid, kept pixels, valid sites (collisions = kept - valid).
 * Device pointers, stream-ordered. */
int gz_ground_truth_to_depth(const uint8_t *gt, int32_t img_h, int32_t img_w, int32_t scale, const gz_gaze *gaze,
                             int32_t *depth_out, uint8_t *valid_out, int64_t *counts_out, void *stream);

/* evalreport.py:47-61 error_count for `batch` labelings (batch x rows x cols
 * int32) against one ground truth.  out: batch x (tail + 3) int64 = total
 * error, evaluated sites, histogram[0..tail] (|diff| >= tail pooled).
 * Device pointers, stream-ordered. */
int gz_error_count(const int32_t *labels, int32_t batch, const int32_t *depth, const uint8_t *valid, int32_t rows,
                   int32_t cols, int32_t tail, int64_t *out, void *stream);

/* imaging.py:211-246 write_disparity_image's raster: labels (rows, cols) int32
 * -> image_out (img_h, img_w) uint8, site pixel x = g + d painted with
 * dis * scale (nearer wins, uncovered pixels 0).  scratch: img_h * img_w int32.
 * The caller checks scale * max disparity <= 255.  Device pointers. */
int gz_render_disparity(const int32_t *labels, const gz_gaze *gaze, int32_t img_w, int32_t img_h, int32_t scale,
                        int32_t *scratch, uint8_t *image_out, void *stream);

/* The solves of evalreport.py:88-126 sweep_penalty: one volume (rows, cols, m)
 * int32 on the device, n energy parameter sets, exact solves (up to 8 in
 * flight, each on 1/8 of the SMs).  labels_out: n x rows x cols int32 (device),
 * stats_out: n entries (host).  workspace: k x gz_workspace_bytes(rows, cols, m)
 * runs k solves at once. */
int gz_solve_volume_batch(const int32_t *vol, int32_t rows, int32_t cols, int32_t m, const gz_energy *energies,
                          int32_t n, const gz_sched *sched, int32_t *labels_out, gz_stats *stats_out,
                          void *workspace, size_t workspace_bytes, void *stream);

/* energy.py:129-155 total_energy on device.  energy_out (device) must hold TWO
 * int64: [0] the energy, [1] a hard-inhibit violation flag (1 when a hard
 * inhibit is violated; the reference then reports UNCUTTABLE, energy.py:149-150). */
int gz_total_energy(const int32_t *labels, const int32_t *vol, int32_t rows, int32_t cols, int32_t m,
                    const gz_energy *energy, int64_t *energy_out, void *stream);

/* hierarchy.py:39-57 coarsen: vol (rows, cols, m) -> coarse (ceil(rows/b), ceil(cols/b), ceil(m/b)). */
int gz_coarsen(const int32_t *vol, int32_t rows, int32_t cols, int32_t m, int32_t block, int32_t *coarse_out,
               void *stream);

/* hierarchy.py:60-73 thin_skin: coarse labeling (crows, ccols) -> lo/hi (rows, cols). */
int gz_thin_skin(const int32_t *coarse_labels, int32_t crows, int32_t ccols, int32_t rows, int32_t cols,
                 int32_t m, int32_t block, int32_t radius, int32_t *lo_out, int32_t *hi_out, void *stream);

/* Runtime knobs (environment, read per solve; defaults are the measured best):
 *   GZ_PAIR_CONC     concurrent pair solves in gz_solve_pairs (8)
 *   GZ_PAIR_DYNAMIC  0: static round-robin of pairs over the concurrent slots instead of
 *                    handing the next pair to the first slot that finishes (1)
 *   GZ_OCC           2: occupancy-2 instance for m <= 16 (default when concurrent)
 *   GZ_BFS_H         BFS levels per temporally blocked round (8)
 *   GZ_KTAIL, GZ_TAIL_AFTER   pulses per sweep from sweep GZ_TAIL_AFTER on (max(K, 96), 4)
 *   GZ_TAIL_MODE     0 disables the single-CTA tail mode (1)
 *   GZ_ASYNC_L       > 0: asynchronous pulses, iterations per team barrier (0)
 *   GZ_WORKLIST      pulse worklists instead of per-pulse scans: 1 on, 0 off (auto: on for
 *                    concurrent solves and for scans of >= 16 rounds per warp)
 *   GZ_WL_DEDUPE     0: keep every push in the pulse worklist (1: a push into an inbox word
 *                    already set this pulse is not listed again)
 *   GZ_BAND_SPIN_MS  row bands: abort a team barrier wait after this long (30000)
 *   GZ_WATCHDOG_MS   device watchdog (20 s + 1 s per 2 M nodes)
 *   GZ_TRACE         1: per-sweep device trace, 2: per-pulse trace to stderr
 */

/* ---- explicit networks (debug export, certificates, generic graphs) ---- */

/* flownet.py:102-181 _emit / flownet.py:233-296 build_network, read back from
 * the DEVICE graph: runs the solver's own initialisation (no presaturating
 * wave) and enumerates the implicit graph's arc pairs in the reference's
 * emission order, capacities taken from the initialised state planes.
 * pair_u/v/cap/rcap: device int64[capacity] (tail, head, capacity, reverse
 * capacity; node ids as flownet.py numbers them, source = n-2, sink = n-1), or
 * all NULL to count only.  info (host int64[4]): [0] pairs, [1] the constant
 * offset folded by the export, [2] nodes, [3] the constant offset of the
 * device initialisation (the two must agree).  m <= 256.
 * residual = 1: no initialisation; the pairs carry the forward and reverse
 * RESIDUALS of the state the last solve in `workspace` left (vol unused; the
 * same windows): the preflow in the reference's arc order, for
 * maxflow.py-style inspection of a solved grid network. */
int gz_export_arcs(const int32_t *vol, int32_t rows, int32_t cols, int32_t m, const gz_energy *energy,
                   const int32_t *lo, const int32_t *hi, int32_t residual, int64_t *pair_u, int64_t *pair_v,
                   int64_t *pair_cap, int64_t *pair_rcap, int64_t capacity, int64_t *info, void *workspace,
                   size_t workspace_bytes, void *stream);

/* One state plane of the last v4 solve run in `workspace` (m <= 256), as
 * int32 (rows*cols, m-1), position t at column t-1: the certificate input
 * (oracle/gz_certify.c).  Device pointers, stream-ordered. */
enum gz_plane {
    GZ_PLANE_CHAIN = 0,        /* residual of chain arc t -> t+1 (capacity vol[t]) */
    GZ_PLANE_SAME_RIGHT = 1,   /* residual of (y,g,t) -> (y,g+1,t); reverse = 2*penalty - r */
    GZ_PLANE_SAME_DOWN = 2,    /* residual of (y,g,t) -> (y+1,g,t) */
    GZ_PLANE_DIAG_RIGHT = 3,   /* flow on (y,g,t) -> (y,g+1,t-1) (capacity inhibit) */
    GZ_PLANE_DIAG_LEFT = 4,    /* flow on (y,g+1,t) -> (y,g,t-1), stored at (y,g) */
    GZ_PLANE_DIAG_DOWN = 5,    /* flow on (y,g,t) -> (y+1,g,t-1) */
    GZ_PLANE_DIAG_UP = 6,      /* flow on (y+1,g,t) -> (y,g,t-1), stored at (y,g) */
    GZ_PLANE_EXCESS = 7,       /* excess (inboxes merged) */
    GZ_PLANE_HEIGHT = 8        /* height of the last relabel */
};
int gz_export_state(const void *workspace, int32_t rows, int32_t cols, int32_t m, int32_t plane, int32_t *out,
                    void *stream);

/* maxflow.py:403-478 result counters of gz_maxflow_csr. */
typedef struct {
    int64_t flow, pushes, relabels, stranded_excess_nodes;
    int32_t sweeps, converged, pulses;
    float ms_total;
} gz_csr_stats;

/* Device workspace for gz_maxflow_csr on n_nodes nodes. */
size_t gz_csr_workspace_bytes(int64_t n_nodes);

/* maxflow.py:403-478 maxflow_push_relabel on an explicit CSR network
 * (flownet.py:41-89 FlowNetwork arrays; flownet.py:325-353 network_from_arcs):
 * source saturation, global relabeling (sink distance, n + source distance,
 * 2n parked: maxflow.py:138-170) and rounds_per_sweep synchronous pulses per
 * sweep until no active node remains (or max_sweeps >= 0 sweeps ran).  The
 * run starts from the flow already in `resid` (excess = -(net outflow of
 * cap - resid): a presaturated or partially solved network).  Both
 * phases run, so `resid` (device int64, updated in place) ends as a maximum
 * flow with no excess left, like the reference's.  side_out (device uint8[n],
 * or NULL): maxflow.py:267-284 source side.  excess_out (device int64[n] or
 * NULL).  Device pointers except stats_out (host). */
int gz_maxflow_csr(int64_t n_nodes, int64_t source, int64_t sink, const int64_t *first_out, const int32_t *head,
                   const int32_t *rev, const int64_t *cap, int64_t *resid, int32_t rounds_per_sweep, int32_t max_sweeps,
                   uint8_t *side_out, int64_t *excess_out, gz_csr_stats *stats_out, void *workspace,
                   size_t workspace_bytes, void *stream);

/* maxflow.py:267-284 _bfs_source_side / maxflow.py:355-359 source_side on
 * CSR arrays: side_out (device uint8[n]) = reachable from the source over
 * resid > 0.  Synchronous. */
int gz_source_side_csr(int64_t n_nodes, int64_t source, const int64_t *first_out, const int32_t *head,
                       const int64_t *resid, uint8_t *side_out, void *stream);

/* maxflow.py:287-304 _chain_presaturate on CSR arrays (device; sent_out is a
 * device int64). */
int gz_chain_presaturate_csr(const int32_t *rev, int64_t *resid, const int32_t *chain_arcs, const int64_t *chain_base,
                             int64_t nsites, int64_t *sent_out, void *stream);

/* maxflow.py:323-334 _conservation_violations on CSR arrays (device; bad_out
 * is a device int64). */
int gz_conservation_violations_csr(const int64_t *first_out, const int64_t *cap, const int64_t *resid, int64_t n_nodes,
                                   int64_t source, int64_t sink, int64_t *bad_out, void *stream);

/* Human-readable status. */
const char *gz_status_string(int status);

/* Library/kernel build identification (for provenance). */
const char *gz_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* GAZECUT_B200_H */
