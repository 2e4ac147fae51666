"""GPU command line for the solve path: `solve` and `bench` with the reference CLI's arguments,
printout, RunRecord JSON/CSV schema and exit codes (reference pkg/src/spaimg/cli.py:18-52,
:215-266, :326-377, :416-447); the hot path runs through this package on cuda:0.

    python -m paper_2206_05543_b200.cli solve --example 3 --N 64 --cycle v --nu1 1 --nu2 1 --smoother m7
    python -m paper_2206_05543_b200.cli bench --examples 1,3 --Ns 64,128 --cycles v1+1 --out runs.csv

Exit codes: 0 success, 1 numerical failure (not converged), 2 usage error.  The LFA / table /
verify subcommands are analysis, not part of the hot path: use the reference CLI for them.
"""

import argparse
import csv
import json
import sys
from dataclasses import asdict, dataclass

from . import multigrid, problems
from .stencils import NAMED_SMOOTHER_IDS, named

SCHEMA_VERSION = 1
BENCH_COLUMNS = ["example", "dim", "N", "smoother", "omega", "cycle", "nu1", "nu2", "iters", "rho_hat", "error_inf",
                 "wall_time_s", "seed"]


@dataclass
class RunRecord:
    command: str
    params: dict
    outputs: dict
    schema_version: int = SCHEMA_VERSION

    def flat(self) -> dict:
        return {**self.params, **self.outputs}


def _write_records(records, out, fmt):
    if out is None:
        return
    if fmt == "json":
        payload = [asdict(r) for r in records]
        with open(out, "w") as fh:
            json.dump(payload[0] if len(payload) == 1 else payload, fh, indent=2)
            fh.write("\n")
    else:
        rows = [r.flat() for r in records]
        names = list(dict.fromkeys(k for row in rows for k in row))
        with open(out, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=names)
            w.writeheader()
            w.writerows(rows)


def _fmt(x, digits=6):
    return "-" if x is None else f"{x:.{digits}g}"


def _run_solve(example_k, N, cycle, nu1, nu2, smoother_id, omega, seed, tol=1e-10, max_iters=100):
    import torch
    prob = problems.example(example_k)
    sm = named(smoother_id)
    if sm.dim != prob.dim:
        raise ValueError(f"smoother {smoother_id} is {sm.dim}D but example {example_k} is {prob.dim}D")
    cfg = multigrid.MgConfig(smoother=sm, cycle=cycle, nu1=nu1, nu2=nu2, omega=omega, tol=tol, max_iters=max_iters,
                             rng_seed=seed)
    b = problems.assemble_rhs(prob, N)
    u, report = multigrid.solve(multigrid.Grid(N, torch.as_tensor(b.values).cuda()), cfg)
    if prob.u_exact is not None:
        report.error_inf = problems.error_inf(u, prob)
    return prob, cfg, report


def cmd_solve(args, parser) -> int:
    try:
        prob, cfg, report = _run_solve(args.example, args.N, args.cycle, args.nu1, args.nu2, args.smoother, args.omega,
                                       args.seed, tol=args.tol, max_iters=args.max_iters)
    except ValueError as exc:
        parser.error(str(exc))
    omega_used = cfg.resolve_smoother()[1]
    print(f"example {args.example} ({prob.name}), N={args.N}, {cfg.cycle}({cfg.nu1}+{cfg.nu2}), "
          f"smoother {args.smoother}, omega {_fmt(omega_used)}, seed {args.seed}, device cuda")
    print(f"iterations    {report.iterations}  ({'converged' if report.converged else 'NOT CONVERGED'})")
    print(f"rho_hat       {_fmt(report.rho_hat)}")
    if report.error_inf is not None:
        print(f"error_inf     {_fmt(report.error_inf)}")
    print(f"wall_time_s   {_fmt(report.wall_time, 4)}")
    print("residual_history " + " ".join(f"{r:.4e}" for r in report.residual_norms))
    rec = RunRecord(
        command="solve",
        params={"example": args.example, "dim": prob.dim, "N": args.N, "smoother": args.smoother, "omega": omega_used,
                "cycle": cfg.cycle, "nu1": cfg.nu1, "nu2": cfg.nu2, "seed": args.seed, "tol": args.tol},
        outputs={"iters": report.iterations, "rho_hat": report.rho_hat, "error_inf": report.error_inf,
                 "wall_time_s": report.wall_time, "converged": report.converged,
                 "residual_norms": report.residual_norms})
    _write_records([rec], args.out, args.format)
    return 0 if report.converged else 1


def _parse_cycles(spec, parser):
    out = []
    for item in spec.split(","):
        s = item.strip().lower().replace("(", "").replace(")", "")
        try:
            kind = s[0]
            nu1, nu2 = s[1:].split("+")
            if kind not in "vw":
                raise ValueError
            out.append((kind.upper(), int(nu1), int(nu2)))
        except (ValueError, IndexError):
            parser.error(f"bad cycle spec {item!r}; expected like w1+0 or v1+1")
    return out


def cmd_bench(args, parser) -> int:
    examples = [int(e) for e in args.examples.split(",")]
    Ns = [int(n) for n in args.Ns.split(",")]
    cycles = _parse_cycles(args.cycles, parser)
    smoothers = args.smoothers.split(",") if args.smoothers else None
    rows, failures = [], 0
    for ex in examples:
        dim = problems.example(ex).dim
        ids = smoothers or (("jacobi2d", "m5", "m9") if dim == 2 else ("jacobi3d", "m7"))
        for N in Ns:
            for cyc, nu1, nu2 in cycles:
                for sid in ids:
                    row = {"example": ex, "dim": dim, "N": N, "smoother": sid, "cycle": cyc, "nu1": nu1, "nu2": nu2,
                           "seed": args.seed}
                    try:
                        _, cfg, report = _run_solve(ex, N, cyc, nu1, nu2, sid, args.omega, args.seed,
                                                    max_iters=args.max_iters)
                        row.update(omega=cfg.resolve_smoother()[1], iters=report.iterations, rho_hat=report.rho_hat,
                                   error_inf=report.error_inf, wall_time_s=report.wall_time)
                        if not report.converged:
                            failures += 1
                    except ValueError as exc:
                        row.update(omega=None, iters=None, rho_hat=None, error_inf=None, wall_time_s=None)
                        print(f"skipped {row}: {exc}", file=sys.stderr)
                        failures += 1
                    rows.append({k: row.get(k) for k in BENCH_COLUMNS})
    print(" ".join(BENCH_COLUMNS))
    for row in rows:
        print(" ".join("-" if row[k] is None else (f"{row[k]:.4g}" if isinstance(row[k], float) else str(row[k]))
                       for k in BENCH_COLUMNS))
    if args.out:
        if args.format == "json":
            records = [RunRecord("bench", params={k: row[k] for k in BENCH_COLUMNS[:8]},
                                 outputs={k: row[k] for k in BENCH_COLUMNS[8:]}) for row in rows]
            _write_records(records, args.out, "json")
        else:
            with open(args.out, "w", newline="") as fh:
                w = csv.DictWriter(fh, fieldnames=BENCH_COLUMNS)
                w.writeheader()
                w.writerows(rows)
    return 1 if failures else 0


def _add_output_args(p):
    p.add_argument("--out", help="write the run record(s) to this path")
    p.add_argument("--format", choices=("csv", "json"), default="csv", help="output file format (default csv)")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="spaimg-cuda", description="B200 SPAI multigrid solves")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("solve", help="run a multigrid solve on a benchmark problem")
    p.add_argument("--example", type=int, choices=(1, 2, 3), required=True)
    p.add_argument("--N", type=int, required=True)
    p.add_argument("--cycle", choices=("v", "w", "V", "W"), default="w")
    p.add_argument("--nu1", type=int, default=1)
    p.add_argument("--nu2", type=int, default=0)
    p.add_argument("--smoother", choices=NAMED_SMOOTHER_IDS, required=True)
    p.add_argument("--omega", type=float, help="override the analytic optimum")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--tol", type=float, default=1e-10)
    p.add_argument("--max-iters", type=int, default=100)
    _add_output_args(p)
    p.set_defaults(func=cmd_solve)
    p = sub.add_parser("bench", help="sweep solves over examples/N/smoothers/cycles")
    p.add_argument("--examples", default="1")
    p.add_argument("--Ns", default="64,128,256")
    p.add_argument("--smoothers", help="comma list; defaults to all for the dimension")
    p.add_argument("--cycles", default="w1+0,v1+1")
    p.add_argument("--omega", type=float)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--max-iters", type=int, default=100)
    _add_output_args(p)
    p.set_defaults(func=cmd_bench)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    return args.func(args, parser)


if __name__ == "__main__":
    sys.exit(main())
