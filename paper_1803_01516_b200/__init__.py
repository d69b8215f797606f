"""B200-native gaze-line stereo graph cuts (arXiv 1803.01516).

Drop-in for the hot path of the reference package ``gazecut``
(pkg/src/gazecut/__init__.py:11-97): stereo pair in, per-site depth labels,
flow and energy out.  The data term, graph initialisation, push-relabel
max-flow, min-cut read-out, energy check and hierarchy helpers run as
hand-written sm_100a CUDA kernels in ``libgazecut_b200.so`` behind a C ABI
(include/gazecut_b200.h).  There is no CPU fallback.

Accuracy accounting (ground truth -> depth numbers, error counts, penalty
sweeps) also runs on the device, and so do explicit networks: the reference's
CSR arrays exported from the device graph, generic ``network_from_arcs``
networks and the CSR solver behind ``maxflow_reference``.
"""

from .energy import UNCUTTABLE, EnergyParams, pairwise_term, sad_volume, sad_volume_device, total_energy
from .flownet import (
    FlowNetwork,
    build_network,
    dump_network,
    node_blocks,
    pairs_to_csr,
    expected_arc_count,
    expected_node_count,
    full_windows,
    network_from_arcs,
)
from .geometry import (
    CuboidSpec,
    GazeDepthCoord,
    WhsCoord,
    cross_from_pixels,
    cuboid_from_disparity_range,
    cuboid_with_offsets,
    disparity_from_whs,
    pixels_from_gaze_depth,
    whs_from_disparity,
)
from .evalreport import (
    HISTOGRAM_TAIL,
    ErrorReport,
    MethodRow,
    SweepRecord,
    best_penalty,
    compare_methods,
    error_count,
    error_count_device,
    error_from_histogram,
    sweep_penalty,
    write_compare_csv,
    write_sweep_csv,
)
from .hierarchy import coarsen, solve_level1, solve_level2, thin_skin
from .maxflow import (
    CutResult,
    InternalConsistencyError,
    chain_presaturate,
    conservation_violations,
    extract_labeling,
    maxflow_push_relabel,
    maxflow_reference,
    solve_exact,
    solve_exact_bands,
    source_side,
)
from .imaging import (
    FileFormatError,
    GroundTruthDepth,
    disparity_of_labeling,
    ground_truth_to_depth,
    load_pgm,
    load_ppm,
    read_labeling,
    render_disparity_device,
    write_disparity_image,
    write_labeling,
    write_pgm,
    write_ppm,
)
from .pairs import PairSolver, solve_pairs
from .synthetic import SyntheticScene, make_scene

__version__ = "0.1.0"

__all__ = [
    "HISTOGRAM_TAIL", "ErrorReport", "MethodRow", "compare_methods", "write_compare_csv", "write_sweep_csv", "SweepRecord", "GroundTruthDepth", "best_penalty", "error_count",
    "error_count_device", "error_from_histogram", "ground_truth_to_depth", "sweep_penalty",
    "FileFormatError", "disparity_of_labeling", "load_pgm", "load_ppm", "read_labeling",
    "render_disparity_device", "write_disparity_image", "write_labeling", "write_pgm", "write_ppm",
    "CuboidSpec", "CutResult", "EnergyParams", "FlowNetwork", "GazeDepthCoord", "InternalConsistencyError",
    "PairSolver", "SyntheticScene", "UNCUTTABLE", "WhsCoord", "build_network", "coarsen",
    "cross_from_pixels", "cuboid_from_disparity_range", "cuboid_with_offsets", "disparity_from_whs",
    "expected_arc_count", "expected_node_count", "extract_labeling", "full_windows", "make_scene",
    "maxflow_push_relabel", "maxflow_reference", "network_from_arcs", "pairwise_term",
    "pixels_from_gaze_depth", "sad_volume", "sad_volume_device", "solve_exact", "solve_level1",
    "solve_level2", "solve_exact_bands", "solve_pairs", "source_side", "thin_skin", "total_energy", "whs_from_disparity",
    "chain_presaturate", "conservation_violations", "dump_network", "node_blocks", "pairs_to_csr",
    "__version__",
]
