"""`python -m paper_1808_01995_b200.verify adjoint|gradient|bench [...]`: the reference's
verification recipes (proj/include/sf/verify.hpp; the `sf verify|bench` CLI it specifies at
SPEC.md:570 but never shipped) run on the GPU operators.  One JSON object on stdout."""
import argparse
import json
import sys


def main(argv=None):
    from . import _sfb_host as H
    ap = argparse.ArgumentParser(prog="paper_1808_01995_b200.verify")
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("adjoint", help="<F q, d> vs <q, F^T d> (proj/src/verify.cpp:201-253)")
    a.add_argument("--ndim", type=int, default=2)
    a.add_argument("--n", type=int, default=64)
    a.add_argument("--order", type=int, default=8)
    a.add_argument("--tn", type=float, default=300.0)
    g = sub.add_parser("gradient", help="Taylor remainders of the FWI objective (:255-331)")
    g.add_argument("--nx", type=int, default=81)
    g.add_argument("--nz", type=int, default=61)
    g.add_argument("--order", type=int, default=8)
    g.add_argument("--tn", type=float, default=450.0)
    b = sub.add_parser("bench", help="operator metrics + n^3 vs (2n)^3 wall ratio (:338-393)")
    b.add_argument("--n", type=int, default=128)
    b.add_argument("--steps", type=int, default=200)
    b.add_argument("--order", type=int, default=8)
    args = ap.parse_args(argv)
    if args.cmd == "adjoint":
        c = H.AdjointConfig()
        c.ndim, c.n, c.space_order, c.tn = args.ndim, args.n, args.order, args.tn
        r = H.adjoint_test(c)
        out = {"forward_dot": r.forward_dot, "adjoint_dot": r.adjoint_dot, "rel_err": r.rel_err,
               "pass": r.rel_err <= 1e-4}
    elif args.cmd == "gradient":
        c = H.GradientConfig()
        c.nx, c.nz, c.space_order, c.tn = args.nx, args.nz, args.order, args.tn
        r = H.gradient_test(c)
        out = {"phi0": r.phi0, "dphi": r.dphi, "steps": r.steps, "eps0": r.eps0, "eps1": r.eps1,
               "eps1_fitted": r.eps1_fitted, "slope0": r.fit0.slope,
               "slope1": r.fit1.slope if r.fit1_valid else None}
    else:
        c = H.BenchConfig()
        c.n, c.steps, c.wall_order = args.n, args.steps, args.order
        r = H.bench(c)
        out = {"orders": r.orders, "flops_per_point": r.flops, "oi": r.oi, "wall_small_s": r.wall_small,
               "wall_big_s": r.wall_big, "wall_ratio": r.wall_ratio}
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main())
