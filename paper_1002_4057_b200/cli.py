"""Command-line entry point: the `tileinv` CLI the
reference declares (`pyproject.toml:12-13`) and specifies (SPEC.md module
`cli`: cmd_invert, cmd_bench, cmd_dag, cmd_table) but does not ship, driving
the B200 path.

    python -m paper_1002_4057_b200 invert --n 4096 --b 256 [--placement out] [--loops UDU] [--no-pipeline]
    python -m paper_1002_4057_b200 bench  --n 4096 8192 --b 256 --workers 1 [--placement in out] [--both-pipelining]
    python -m paper_1002_4057_b200 dag    --t 4 --step 3 [--placement out] --out step3.dot
    python -m paper_1002_4057_b200 table  --t-min 2 --t-max 8

Exit codes (SPEC.md `cli` invariants): 0 success, 2 validation error,
3 numerical failure (non-SPD / singular tile, residual above tolerance),
4 I/O error, 1 device error (no B200 / CUDA failure: there is no CPU path).
`--workers` is validated as the reference does; the device executor always
uses every SM.
"""

from __future__ import annotations

import argparse
import statistics
import sys
import time

import numpy as np

EXIT_OK, EXIT_VALIDATION, EXIT_NUMERICAL, EXIT_IO = 0, 2, 3, 4


def _spd(n: int, seed: int) -> np.ndarray:
    """SURVEY.md §8(d) input recipe: A = G G^T / n + I, G iid N(0,1), mirrored lower."""
    g = np.random.default_rng(seed).standard_normal((n, n))
    a = g @ g.T / n + np.eye(n)
    return np.tril(a) + np.tril(a, -1).T


def _sizes(args) -> tuple[int, int]:
    if args.t is not None:
        if args.b is None:
            raise ValueError("--t needs --b")
        return args.b * args.t, args.b
    if args.n is None or args.b is None:
        raise ValueError("give --n and --b (or --b and --t)")
    return args.n, args.b


def _config(args, pipelined=None):
    from .taskgen import Placement, VariantConfig

    return VariantConfig(Placement(args.placement), args.loops,
                         (not args.no_pipeline) if pipelined is None else pipelined, args.workers)


def _read_input(path: str) -> np.ndarray:
    a = np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2)
    return a


def cmd_invert(args) -> int:
    """SPEC.md cmd_invert: run the configured variant, print residual
    max|A A^-1 - I|, elapsed time and Gflop/s = n^3 / (time 1e9); nonzero exit
    if the residual exceeds 1e-9 n."""
    from . import inversion
    from .scheduler import ExecutionError

    if args.input:
        a = _read_input(args.input)
        n, b = a.shape[0], args.b if args.b is not None else a.shape[0]
    else:
        n, b = _sizes(args)
        a = _spd(n, args.seed)
    cfg = _config(args)
    t0 = time.perf_counter()
    try:
        x = inversion.invert(a, b, cfg)
    except ExecutionError as e:
        print(f"inversion failed: {e}", file=sys.stderr)
        return EXIT_NUMERICAL
    dt = time.perf_counter() - t0
    res = float(np.abs(a @ x - np.eye(n)).max())
    print(f"n={n} b={b} t={n // b} placement={cfg.placement.value} loops={cfg.loops} "
          f"pipelined={cfg.pipelined} residual={res:.3e} time_s={dt:.4f} gflops={n ** 3 / dt / 1e9:.2f}")
    if args.out:
        np.save(args.out, x)
    return EXIT_OK if res <= 1e-9 * n else EXIT_NUMERICAL


def cmd_bench(args) -> int:
    """SPEC.md cmd_bench: for each (n, workers, variant) the median of 3 timed
    runs (after one untimed run), CSV `variant,n,b,workers,loops,pipelined,time_s,gflops`.
    The timed call is the whole public path (from_dense -> execute -> to_dense)."""
    from . import inversion
    from .taskgen import Placement, VariantConfig

    pipes = (True, False) if args.both_pipelining else (not args.no_pipeline,)
    rows = ["variant,n,b,workers,loops,pipelined,time_s,gflops"]
    print(rows[0], flush=True)
    for n in args.n:
        if n % args.b:
            raise ValueError(f"matrix order {n} not divisible by tile order {args.b}")
        a = _spd(n, args.seed)
        for w in args.workers:
            for pl in args.placement_list:
                for pipe in pipes:
                    cfg = VariantConfig(Placement(pl), args.loops, pipe, w)
                    inversion.invert(a, args.b, cfg)  # untimed
                    ts = []
                    for _ in range(3):
                        t0 = time.perf_counter()
                        inversion.invert(a, args.b, cfg)
                        ts.append(time.perf_counter() - t0)
                    med = statistics.median(ts)
                    row = (f"{pl},{n},{args.b},{w},{args.loops},{str(pipe).lower()},{med:.6f},"
                           f"{n ** 3 / med / 1e9:.2f}")
                    rows.append(row)
                    print(row, flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write("\n".join(rows) + "\n")
    return EXIT_OK


def cmd_dag(args) -> int:
    """SPEC.md cmd_dag: DOT of the selected step / full pipeline at tile count t,
    and its PathReport."""
    from . import dag_analysis as D
    from .scheduler import build_dag
    from .taskgen import Placement, gen_inversion, gen_step1, gen_step2, gen_step3

    pl = Placement(args.placement)
    d = args.direction
    if args.step == 1:
        s = gen_step1(args.t, d or "U")
    elif args.step == 2:
        s = gen_step2(args.t, d or "D", pl)
    elif args.step == 3:
        s = gen_step3(args.t, d or "U", pl)
    else:
        s = gen_inversion(args.t, _config(args))
    dag = build_dag(s)
    dot = D.export_dot(dag, include_copies=not args.no_copies)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(dot)
    else:
        sys.stdout.write(dot)
    print(D.critical_path(dag), file=sys.stderr if not args.out else sys.stdout)
    return EXIT_OK


def cmd_table(args) -> int:
    """SPEC.md cmd_table: Table 1 formulas vs measured critical paths as CSV;
    nonzero exit on any mismatch."""
    from . import dag_analysis as D

    if not (2 <= args.t_min <= args.t_max <= 12):
        raise ValueError("t range must lie within 2..12")
    rows = D.formula_table(range(args.t_min, args.t_max + 1))
    sys.stdout.write(D.formula_csv(rows))
    bad = [r for r in rows if not r.match]
    return EXIT_OK if not bad or args.allow_mismatch else EXIT_NUMERICAL


def _parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="tileinv", description="B200 tile inversion of SPD matrices")
    sub = p.add_subparsers(dest="cmd", required=True)

    def variant(q, multi_placement=False):
        if multi_placement:
            q.add_argument("--placement", dest="placement_list", nargs="+", choices=["in", "out"], default=["in"])
        else:
            q.add_argument("--placement", choices=["in", "out"], default="in")
        q.add_argument("--loops", default="UDU")
        q.add_argument("--no-pipeline", action="store_true")
        q.add_argument("--seed", type=int, default=0)

    q = sub.add_parser("invert", help="invert one generated (or CSV) SPD matrix and check the residual")
    q.add_argument("--n", type=int)
    q.add_argument("--b", type=int, default=None)
    q.add_argument("--t", type=int)
    q.add_argument("--workers", type=int, default=1)
    q.add_argument("--input")
    q.add_argument("--out")
    variant(q)
    q = sub.add_parser("bench", help="median-of-3 timings as CSV")
    q.add_argument("--n", type=int, nargs="+", required=True)
    q.add_argument("--b", type=int, required=True)
    q.add_argument("--workers", type=int, nargs="+", default=[1])
    q.add_argument("--both-pipelining", action="store_true", help="time pipelined and barriered")
    q.add_argument("--out")
    variant(q, multi_placement=True)
    q = sub.add_parser("dag", help="DOT export and critical path of a step or the full pipeline")
    q.add_argument("--t", type=int, required=True)
    q.add_argument("--step", type=int, choices=[0, 1, 2, 3], default=0, help="0: full inversion")
    q.add_argument("--direction", choices=["U", "D"])
    q.add_argument("--workers", type=int, default=1)
    q.add_argument("--no-copies", action="store_true")
    q.add_argument("--out")
    variant(q)
    q = sub.add_parser("table", help="Table 1 formulas vs measured critical paths")
    q.add_argument("--t-min", type=int, default=2)
    q.add_argument("--t-max", type=int, default=8)
    q.add_argument("--allow-mismatch", action="store_true",
                   help="exit 0 even though the pipelined rows do not follow the paper's formulas")
    return p


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        if hasattr(args, "workers") and isinstance(args.workers, int) and args.workers < 1:
            raise ValueError(f"workers must be >= 1, got {args.workers}")
        return {"invert": cmd_invert, "bench": cmd_bench, "dag": cmd_dag, "table": cmd_table}[args.cmd](args)
    except OSError as e:
        print(f"I/O error: {e}", file=sys.stderr)
        return EXIT_IO
    except RuntimeError as e:  # _native.NativeError: no device, CUDA failure (no CPU fallback)
        print(f"device error: {e}", file=sys.stderr)
        return 1
    except ValueError as e:  # InvalidSizeError, bad loops / placement, divisibility
        print(f"invalid arguments: {e}", file=sys.stderr)
        return EXIT_VALIDATION


if __name__ == "__main__":
    sys.exit(main())
