"""`python -m paper_1502_03543_b200 check|bench` -- the reference CLI's
verification and benchmark subcommands (cli.py:144-217) on the GPU path.
See harness.py; the solve/gen front end is out of scope."""

import argparse
import sys

from . import harness as H


def _parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_1502_03543_b200",
                                description="B200 PDAS harnesses (check, bench)")
    sub = p.add_subparsers(dest="subcommand", required=True)
    c = sub.add_parser("check", help="verification sweep over seeded instances")
    c.add_argument("--seeds", default="1..20", help="N or A..B")
    c.add_argument("--m", type=int, default=None)
    c.add_argument("--n", type=int, default=None)
    c.add_argument("--z-tol", type=float, default=1e-9)
    c.add_argument("--equiv-tol", type=float, default=1e-8)
    b = sub.add_parser("bench", help="time backends over an instance grid")
    b.add_argument("--grid", required=True, help="MxN[,MxN...]")
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--max-iter", type=int, default=20)
    return p


def main(argv=None) -> int:
    from .errors import AdascaleError

    args = _parser().parse_args(argv)
    try:
        if args.subcommand == "check":
            return H.run_check(H.parse_seed_range(args.seeds), args.m, args.n, args.z_tol,
                               args.equiv_tol)
        H.run_bench(H.parse_grid(args.grid), args.seed, args.max_iter)
        return H.EXIT_OK
    except (AdascaleError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return H.EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
