"""Thin command line front end: ``solve`` (cli.py:179-249 cmd_solve).

    python -m paper_1803_01516_b200 solve --left L.ppm --right R.ppm --out PREFIX \\
        [--gt GT.pgm] [--dis-min A --dis-max B] [--level 0|1|2] ...

Same arguments, output files (PREFIX.pgm disparity image, PREFIX.labels.txt,
PREFIX.stats.txt, each with the run configuration in header comments) and
exit codes as the reference's ``gazecut solve`` (cli.py:48-50, 479-492):
0 success, 2 bad usage or parameters, 3 unreadable or malformed input files,
4 failed internal consistency check.  The data term, the solve, the
disparity raster and the error count run on the device.  The reference's
other subcommands (sweep, compare, convert-gt, selftest) are host-side
experiment drivers outside the B200 hot path."""

from __future__ import annotations

import argparse
import sys

import numpy as np

from . import __version__
from .energy import EnergyParams, sad_volume
from .evalreport import error_count
from .geometry import cuboid_from_disparity_range, cuboid_with_offsets
from .hierarchy import DEFAULT_L2_SWEEPS, solve_level1, solve_level2
from .imaging import FileFormatError, ground_truth_to_depth, load_pgm, load_ppm, write_disparity_image, write_labeling
from .maxflow import InternalConsistencyError, solve_exact

EXIT_USAGE = 2
EXIT_IO = 3
EXIT_CHECK = 4


def _disparity_range(args, gt_img):
    """cli.py:109-123: explicit --dis-min/--dis-max, else from the ground truth."""
    dis_min, dis_max = args.dis_min, args.dis_max
    if dis_min is None or dis_max is None:
        if gt_img is None:
            raise ValueError("--dis-min/--dis-max required when no --gt is given")
        vals = gt_img[gt_img > 0].astype(np.int64)
        if vals.size == 0:
            raise ValueError("ground truth image has no labelled pixels")
        scale = args.gt_scale
        if dis_min is None:
            dis_min = int((2 * vals.min() + scale) // (2 * scale))
        if dis_max is None:
            dis_max = int((2 * vals.max() + scale) // (2 * scale))
    return dis_min, dis_max


def _setup(args):
    """cli.py:151-166: images, cuboid, data volume, optional ground truth."""
    left, right = load_ppm(args.left), load_ppm(args.right)
    if left.shape != right.shape:
        raise ValueError(f"image shapes differ: {left.shape} vs {right.shape}")
    gt_img = load_pgm(args.gt) if args.gt else None
    if gt_img is not None and gt_img.shape != left.shape[:2]:
        raise ValueError(f"ground truth shape {gt_img.shape} != image shape {left.shape[:2]}")
    height, width = left.shape[:2]
    dis_min, dis_max = _disparity_range(args, gt_img)
    cuboid = cuboid_from_disparity_range(width, height, dis_min, dis_max, margin=args.margin,
                                         num_labels=args.labels, g_extent=args.g_extent)
    if args.offsets:
        try:
            o1, o2, o3 = (int(p) for p in args.offsets.split(","))
        except ValueError:
            raise ValueError(f"bad --offsets {args.offsets!r}, want O1,O2,O3")
        cuboid = cuboid_with_offsets(cuboid, o1, o2, o3, width, height)
    volume = sad_volume(left, right, cuboid)
    gt = ground_truth_to_depth(gt_img, args.gt_scale, cuboid) if gt_img is not None else None
    return left, cuboid, volume, gt, (dis_min, dis_max)


def cmd_solve(args) -> int:
    """cli.py:179-249."""
    if args.threads < 1:
        raise ValueError("--threads must be >= 1")
    left, cuboid, volume, gt, (dis_min, dis_max) = _setup(args)
    params = EnergyParams(penalty=args.penalty, inhibit=args.inhibit, hard_inhibit=args.hard_inhibit)
    if args.level == 0:
        result = solve_exact(volume, params, solver=args.solver)
    elif args.level == 1:
        result = solve_level1(volume, params, args.block, skin_radius=args.skin_radius, solver=args.solver)
    else:
        result = solve_level2(volume, params, args.block, skin_radius=args.skin_radius, max_sweeps=args.max_sweeps)
    height, width = left.shape[:2]
    config = [f"gazecut {args.command}"] + [f"{k} {v}" for k, v in (
        ("left", args.left), ("right", args.right), ("dis_range", f"{dis_min} {dis_max}"),
        ("labels", cuboid.num_labels), ("penalty", params.penalty), ("inhibit", params.inhibit),
        ("hard_inhibit", int(params.hard_inhibit)), ("level", args.level), ("block", args.block),
        ("skin_radius", args.skin_radius), ("solver", args.solver), ("threads", args.threads))]
    out = args.out
    scale_used = write_disparity_image(result.labeling, cuboid, f"{out}.pgm", width, height, scale=args.scale,
                                       comments=config)
    write_labeling(f"{out}.labels.txt", result.labeling, comments=config)
    stats_lines = [f"energy={result.energy}", f"flow={result.flow}", f"nodes={result.stats.get('nodes', 0)}",
                   f"arcs={result.stats.get('arcs', 0)}", f"converged={int(result.stats.get('converged', True))}",
                   f"disparity_scale={scale_used}"]
    if gt is not None:
        report = error_count(result.labeling, gt)
        stats_lines += [f"error={report.total_error}", f"evaluated={report.evaluated}",
                        f"exact_fraction={report.exact_fraction:.6f}", f"gt_out_of_range={gt.out_of_range}",
                        f"gt_off_grid={gt.off_grid}", f"gt_collisions={gt.collisions}"]
        print(f"error {report.total_error} over {report.evaluated} sites ({report.exact_fraction:.1%} exact)")
    if args.timings:
        stats_lines.append(f"wall_s={result.stats.get('wall_s', 0.0):.3f}")
        print(f"wall {result.stats.get('wall_s', 0.0):.3f}s")
    with open(f"{out}.stats.txt", "w") as f:
        for line in config:
            f.write(f"# {line}\n")
        f.write("\n".join(stats_lines) + "\n")
    print(f"energy {result.energy} (flow {result.flow})")
    if not result.stats.get("converged", True):
        print(f"note: sweep cap hit after {result.stats.get('sweeps')} sweeps")
    print(f"wrote {out}.pgm, {out}.labels.txt, {out}.stats.txt")
    return 0


def build_parser() -> argparse.ArgumentParser:
    """cli.py:403-476 (the solve subcommand)."""
    parser = argparse.ArgumentParser(prog="gazecut", description="Stereo depth estimation by exact graph cuts over "
                                     "gaze-line / depth-number space (B200).")
    parser.add_argument("--version", action="version", version=f"gazecut {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("solve", help="estimate depth for one stereo pair")
    p.add_argument("--left", required=True, help="left image (ppm)")
    p.add_argument("--right", required=True, help="right image (ppm)")
    p.add_argument("--gt", help="ground-truth disparity image (pgm), registered to the right view")
    p.add_argument("--gt-scale", type=int, default=8, help="ground-truth pixel value per disparity step (default 8)")
    p.add_argument("--dis-min", type=int, help="smallest disparity searched")
    p.add_argument("--dis-max", type=int, help="largest disparity searched")
    p.add_argument("--labels", type=int, help="number of depth labels (default: cover the disparity range)")
    p.add_argument("--margin", type=int, default=0, help="spare depth labels on each side of the covered range")
    p.add_argument("--g-extent", type=int, help="number of gaze lines (default: width - dis_min - 2)")
    p.add_argument("--offsets", metavar="O1,O2,O3", help="override the gaze/row/depth coordinate offsets")
    p.add_argument("--penalty", type=int, default=14, help="cost per unit label step")
    p.add_argument("--inhibit", type=int, default=1023, help="extra cost per unit beyond the first label step")
    p.add_argument("--hard-inhibit", action="store_true", help="forbid neighbour label jumps larger than one")
    p.add_argument("--out", required=True, help="output path prefix")
    p.add_argument("--level", type=int, default=0, choices=(0, 1, 2),
                   help="0 exact, 1 hierarchical exact, 2 hierarchical capped")
    p.add_argument("--block", type=int, default=2, help="hierarchy block size")
    p.add_argument("--skin-radius", type=int, default=1, help="label window radius around the coarse surface")
    p.add_argument("--max-sweeps", type=int, default=DEFAULT_L2_SWEEPS, help="level-2 sweep cap")
    p.add_argument("--solver", default="push-relabel", choices=("push-relabel", "dinic"))
    p.add_argument("--scale", type=int, help="disparity image scale (default: widest that cannot clip)")
    p.add_argument("--threads", type=int, default=1, help="recorded in provenance (the device runs the solve)")
    p.add_argument("--timings", action="store_true", help="report wall-clock times")
    p.set_defaults(func=cmd_solve)
    return parser


def main(argv=None) -> int:
    """cli.py:479-492: exceptions -> exit codes 3 / 4 / 2."""
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (OSError, FileFormatError) as exc:
        print(f"gazecut: {exc}", file=sys.stderr)
        return EXIT_IO
    except InternalConsistencyError as exc:
        print(f"gazecut: consistency check failed: {exc}", file=sys.stderr)
        return EXIT_CHECK
    except ValueError as exc:
        print(f"gazecut: {exc}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
