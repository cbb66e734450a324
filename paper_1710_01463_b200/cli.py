"""`factorize` command-line drop-in (rlftn cli.cpp:180-244) on the B200 engine.

    python -m paper_1710_01463_b200.cli factorize --in M.bin --rank K
        [--method tsvd|rsvd] [--oversample L] [--power Q] [--seed S] [--out DIR]
    python -m paper_1710_01463_b200.cli --version

Same outputs as the reference: DIR/spectrum.csv (values with %.17g),
DIR/left.bin and DIR/right.bin (RLFMAT01), DIR/summary.json, and the
three-line stdout summary; rank clipped to min(m, n); the rsvd seed is
derive_seed(S, rsvd_stream) (cli.cpp:197); output directory precedence
RLFTN_OUT, then --out, then "factors".  Exit codes: 0 ok, 1 runtime error
("error: ..." or, with --error-json, a JSON object), 2 usage error.
Real and complex matrices (the reference's std::visit over AnyMatrix,
cli.cpp:185-240): a complex file runs the complex instantiation and writes
complex factors, "complex": true in summary.json.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

VERSION = "0.1.0"


class UsageError(Exception):
    pass


def fmt(v: float, prec: int = 17) -> str:
    return "%.*g" % (prec, v)


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise UsageError(message)


def _resolve_out(value, given, fallback):
    env = os.environ.get("RLFTN_OUT")
    if env:
        return env
    return value if given else fallback


def cmd_factorize(o) -> int:
    from . import RsvdParams, reconstruction_error, rsvd, tsvd
    from .matrix_io import load_matrix, save_matrix_binary
    from .rng import derive_seed, seed_tag

    if o.rank < 1:
        raise UsageError("--rank must be at least 1")
    if o.power < 0:
        raise UsageError("--power must be nonnegative")
    if o.method not in ("tsvd", "rsvd"):
        raise UsageError("--method must be tsvd or rsvd")
    a = load_matrix(o.inp)
    cplx = bool(np.iscomplexobj(a))
    out_dir = _resolve_out(o.out, o.out is not None, "factors")
    os.makedirs(out_dir, exist_ok=True)
    m, n = a.shape
    rank = min(o.rank, min(m, n))
    if o.method == "rsvd":
        f = rsvd(a, RsvdParams(rank, o.oversample, o.power,
                               derive_seed(o.seed, seed_tag.rsvd_stream)))
    else:
        f = tsvd(a, rank)
    fro = reconstruction_error(a, f)
    sig = np.asarray(f.sigma)
    with open(os.path.join(out_dir, "spectrum.csv"), "w") as fh:
        fh.write(",".join(fmt(x) for x in sig) + "\n")
    save_matrix_binary(os.path.join(out_dir, "left.bin"), np.asarray(f.left))
    save_matrix_binary(os.path.join(out_dir, "right.bin"), np.asarray(f.right_adj))
    j = {"rows": m, "cols": n, "complex": cplx, "requested_rank": o.rank, "rank": f.rank(),
         "method": o.method, "discarded_weight": f.discarded_weight,
         "discarded_exact": f.discarded_exact, "frobenius_error": fro,
         "files": {"spectrum": "spectrum.csv", "left": "left.bin", "right": "right.bin"}}
    if o.method == "rsvd":
        j.update({"oversample": o.oversample, "power": o.power, "seed": o.seed})
    with open(os.path.join(out_dir, "summary.json"), "w") as fh:
        fh.write(json.dumps(j, indent=2, sort_keys=True) + "\n")
    print(f"{o.method} rank {f.rank()} of {m}x{n}: discarded weight = "
          f"{fmt(f.discarded_weight, 6)}, frobenius error = {fmt(fro, 6)}")
    head = " ".join(fmt(x, 6) for x in sig[:8])
    print("spectrum:" + (" " + head if head else "") + (" ..." if len(sig) > 8 else ""))
    print("wrote " + os.path.join(out_dir, "summary.json"))
    return 0


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    error_json = "--error-json" in argv
    if error_json:
        argv.remove("--error-json")
    try:
        if argv and argv[0] == "--version":
            print("rlftn-b200 " + VERSION)
            return 0
        p = _Parser(prog="rlftn-b200", add_help=True)
        sub = p.add_subparsers(dest="cmd")
        f = sub.add_parser("factorize")
        f.error = p.error
        f.add_argument("--in", dest="inp", required=True)
        f.add_argument("--rank", type=int, required=True)
        f.add_argument("--method", default="tsvd")
        f.add_argument("--oversample", type=int, default=0)
        f.add_argument("--power", type=int, default=4)
        f.add_argument("--seed", type=int, default=1)
        f.add_argument("--out", default=None)
        o = p.parse_args(argv)
        if o.cmd is None:
            raise UsageError("a subcommand is required")
        return cmd_factorize(o)
    except UsageError as e:
        print("usage error: " + str(e), file=sys.stderr)
        return 2
    except Exception as e:  # runtime failures (I/O, engine), like the reference's exit 1
        if error_json:
            print(json.dumps({"exit": 1, "error": str(e)}))
        else:
            print("error: " + str(e), file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
