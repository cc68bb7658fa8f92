"""`run` / `sweep` front end on the GPU path.

    python -m paper_2202_06111_b200 run   [--config FILE] [--key value ...] [--output-dir D]
    python -m paper_2202_06111_b200 sweep [--N 0,1,3,full] [--mode ...] [--workers ...] ...

The same flags, configuration keys and exit codes as the reference's
`cisgraph run` / `cisgraph sweep` (cg/cli.py:42-228): 0 success, 1 invalid
configuration (the message names the key), 2 runtime failure, 3 the run
ended with an empty covering.  A sweep runs the cartesian product of the
comma-listed plan keys (mode, N -- where `full` means full subdivision --,
workers, batch_size), one output directory per point, and gathers their
metrics into sweep.tsv.  Every run goes through engine.run, i.e. the
device-resident loop.  The reference's `hull` / `compare` subcommands are
shapely post-processing outside this package's path.
"""

from __future__ import annotations

import argparse
import itertools
import sys
from pathlib import Path

from .config import ConfigError, parse_config_text, render_config, resolve_config
from .engine import METRICS_COLUMNS, run, write_run_outputs

EXIT_OK, EXIT_CONFIG, EXIT_RUNTIME, EXIT_EMPTY = 0, 1, 2, 3

# flag -> (config key, help); plan keys take comma lists in sweeps
SCALAR_FLAGS = {
    "--model": ("model", "model name"),
    "--iterations": ("iterations", "maximum iteration count"),
    "--delta": ("delta", "boundary-test enlargement factor"),
    "--samples-per-dim": ("samples_per_dim", "image sample points per state dimension"),
    "--bloat": ("bloat", "image enclosure inflation factor"),
    "--input-grid": ("input_grid", "input grid points per input dimension"),
    "--min-diameter": ("min_diameter", "stop when the covering diameter falls below this"),
}
PLAN_FLAGS = {
    "--mode": ("mode", "full or adaptive"),
    "--N": ("N", "neighbourhood size ('full' = full subdivision in sweeps)"),
    "--workers": ("workers", "BuildPlan.workers"),
    "--batch-size": ("batch_size", "BuildPlan.batch_size"),
}
SWITCHES = {
    "--include-face-points": ("include_face_points", "probe edge midpoints too"),
    "--strict-largest-scc": ("strict_largest_scc", "keep the largest SCC's closure only"),
}


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2202_06111_b200",
                                 description="GIS outer approximations of largest control "
                                             "invariant sets on the GPU")
    sub = ap.add_subparsers(dest="command", required=True)
    for name, listy in (("run", False), ("sweep", True)):
        p = sub.add_parser(name)
        p.add_argument("--config", help="flat key = value configuration file")
        for flag, (key, text) in SCALAR_FLAGS.items():
            p.add_argument(flag, dest=key, help=text)
        for flag, (key, text) in PLAN_FLAGS.items():
            p.add_argument(flag, dest=key, help=text + (" (comma list)" if listy else ""),
                           type=(lambda v: v.split(",")) if listy else str)
        for flag, (key, text) in SWITCHES.items():
            p.add_argument(flag, dest=key, action="store_const", const="true", help=text)
        p.add_argument("--set", dest="extra", action="append", default=[], metavar="KEY=VALUE",
                       help="override any configuration key")
        p.add_argument("--output-dir", default="cisgraph-out")
        p.add_argument("--export-edges", action="store_true",
                       help="also write the last graph's edge list")
    return ap


def _overrides(args, keys) -> dict:
    out = {k: getattr(args, k) for k in keys if getattr(args, k) is not None}
    for item in args.extra:
        key, sep, value = item.partition("=")
        if not sep:
            raise ConfigError(item, "expected KEY=VALUE in --set")
        out[key.strip()] = value.strip()
    return out


def _one(file_values: dict, overrides: dict, outdir: Path, export_edges: bool) -> int:
    resolved = resolve_config(file_values, overrides, keep_final_graph=export_edges)
    result = run(resolved.run_config)
    write_run_outputs(result, outdir, export_edges=export_edges)
    (outdir / "effective.cfg").write_text(render_config(resolved.effective))
    print(f"wrote {outdir}: cells={len(result.covering)} termination={result.termination}")
    if result.empty:
        print("no invariant set at this resolution", file=sys.stderr)
        return EXIT_EMPTY
    return EXIT_OK


def _sweep(args, file_values: dict) -> int:
    scalars = [k for k, _ in SCALAR_FLAGS.values()] + [k for k, _ in SWITCHES.values()]
    base = _overrides(args, scalars)
    axes = {}
    for key, _ in PLAN_FLAGS.values():
        vals = getattr(args, key)
        if vals is None:
            continue
        if len(vals) == 1:
            base[key] = vals[0]
        else:
            axes[key] = vals
    root = Path(args.output_dir)
    table = ["point\t" + "\t".join(METRICS_COLUMNS)]
    names = sorted(axes)
    points = []
    for combo in itertools.product(*(axes[k] for k in names)):
        point = dict(zip(names, combo))
        ov = dict(base)
        for key, value in point.items():
            if key == "N":  # N=full means a full-subdivision run
                if value == "full":
                    ov["mode"] = "full"
                else:
                    ov.setdefault("mode", "adaptive")
                    ov["N"] = value
            else:
                ov[key] = value
        label = "__".join(f"{k}_{v}" for k, v in point.items()) or "base"
        resolve_config(file_values, ov)  # every point's configuration checked up front
        points.append((label, ov))
    root.mkdir(parents=True, exist_ok=True)
    for label, ov in points:
        _one(file_values, ov, root / label, args.export_edges)
        rows = (root / label / "metrics.tsv").read_text().splitlines()[1:]
        table += [f"{label}\t{r}" for r in rows]
    (root / "sweep.tsv").write_text("\n".join(table) + "\n")
    print(f"sweep table written to {root / 'sweep.tsv'}")
    return EXIT_OK


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        file_values = parse_config_text(Path(args.config).read_text()) if args.config else {}
        if args.command == "sweep":
            return _sweep(args, file_values)
        keys = ([k for k, _ in SCALAR_FLAGS.values()] + [k for k, _ in PLAN_FLAGS.values()]
                + [k for k, _ in SWITCHES.values()])
        return _one(file_values, _overrides(args, keys), Path(args.output_dir),
                    args.export_edges)
    except ConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except Exception as exc:  # a runtime failure, distinct from a bad configuration
        print(f"error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return EXIT_RUNTIME
