"""Command line: ``python -m paper_1310_5541_b200 {backends,track,pseudo}``.

``backends`` times the device likelihood operator on the reference CLI's
micro-benchmark workloads (cli.py:191-213); ``track`` runs a GPU tracking
sweep and writes the reference's summary CSV (cli.py:123-138, reports.py).
Exit codes follow the reference: 0 ok, 2 invalid configuration.
"""

import argparse
import sys


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1310_5541_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("backends", help="likelihood operator micro-benchmark")
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--seed", type=int, default=0)
    t = sub.add_parser("track", help="GPU tracking sweep -> summary CSV")
    t.add_argument("--variants", default="SIR,pcSIR-1x1-CoM,pcSIR-2x2-CoM")
    t.add_argument("--n", default="1000,10000,100000", help="strictly increasing particle counts")
    t.add_argument("--reps", type=int, default=3)
    t.add_argument("--frames", type=int, default=20)
    t.add_argument("--size", type=int, default=128)
    t.add_argument("--sigma-xi", type=float, default=10.0)
    t.add_argument("--seed", type=int, default=0)
    t.add_argument("--out", default="gpu_tracking_summary.csv")
    q = sub.add_parser("pseudo", help="GPU pseudo-tracking convergence study -> summary CSV")
    q.add_argument("--variants", default="SIR,pcSIR-1x1-CoM,pcSIR-2x2-CoM")
    q.add_argument("--n", default="100,1000,10000")
    q.add_argument("--reps", type=int, default=100)
    q.add_argument("--prior", default="uniform3x3")
    q.add_argument("--seed", type=int, default=0)
    q.add_argument("--out", default="gpu_pseudo_summary.csv")
    args = ap.parse_args(argv)

    from . import experiments as ex
    if args.cmd == "backends":
        print("available backends: cuda")
        ex.likelihood_benchmark(args.repeats, args.seed)
        return 0
    from .imaging import PsfParams
    from .synthesis import SceneConfig
    if args.cmd == "pseudo":
        try:
            records = ex.run_pseudo_tracking(args.variants.split(","),
                                             [int(x) for x in args.n.split(",") if x], args.reps,
                                             prior=args.prior, seed=args.seed)
        except (ex.ConfigError, ValueError) as e:
            print(f"error: {e}", file=sys.stderr)
            return 2
        rows = ex.summarize(records)
        for r in rows:
            print(f"{r.variant:>16s} N={r.n_particles:>8d} rms error={r.rmse_mean:.4f} "
                  f"evals={r.lik_evals_mean:.0f}")
        print(f"wrote {ex.write_summary_csv(rows, args.out)}")
        return 0
    try:
        ns = [int(x) for x in args.n.split(",") if x]
        scene = SceneConfig(PsfParams(1.5, 10.0), frames=args.frames, width=args.size,
                            height=args.size)
        records = ex.run_tracking_experiment(args.variants.split(","), ns, args.reps, scene=scene,
                                             sigma_xi=args.sigma_xi, seed=args.seed)
    except (ex.ConfigError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    rows = ex.summarize(records)
    for r in rows:
        print(f"{r.variant:>16s} N={r.n_particles:>8d} rmse={r.rmse_mean:.3f} "
              f"t={r.time_mean_s * 1e3:.2f} ms evals={r.lik_evals_mean:.0f} "
              f"speedup={r.speedup_vs_sir:.2f}")
    print(f"wrote {ex.write_summary_csv(rows, args.out)}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
