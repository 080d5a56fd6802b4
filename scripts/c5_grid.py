"""Config 5 end to end through the reference's own API: `lpdsvm.grid_search` (factor
built once per γ, every (fold, pair) problem warm-started along the ascending C list,
modelsel.cpp:170-230) from one build of the reference's `_core`:

  integration/_build  — compute_G, the held-out scoring and the warm-start sweeps on the
                        B200 (resident G), everything else the reference's host code
  oracle/_ref         — the reference as is (CPU, all host threads)

  python scripts/c5_grid.py <module_dir> <out.json> [--n N --budget B ...]

Prints / writes one JSON object: wall seconds, the grid's errors and solve counts.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("module_dir")
    ap.add_argument("out")
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--d", type=int, default=54)
    ap.add_argument("--budget", type=int, default=2048)
    ap.add_argument("--folds", type=int, default=3)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--tau", type=float, default=1e-12)
    ap.add_argument("--gamma-mults", default="0.5,1,2", help="γ = mult/d, comma separated")
    ap.add_argument("--Cs", default="0.25,1,4")
    args = ap.parse_args()

    mdir = args.module_dir if os.path.isabs(args.module_dir) else os.path.join(ROOT, args.module_dir)
    sys.path.insert(0, mdir)
    if os.path.isdir(os.path.join(mdir, "lpdsvm")):
        import lpdsvm
    else:
        import _core as lpdsvm
    from integration_train import libsvm_text
    from paper_2207_01016_b200 import synthetic

    X, y = synthetic.blobs(args.n, args.d, seed=2)
    data = lpdsvm.parse_dataset(libsvm_text(X, y))
    g0 = 1.0 / args.d
    # log2 γ around γ* (PAPER.md:828-832 style grid)
    gammas = [float(m) * g0 for m in args.gamma_mults.split(",")]
    Cs = [float(c) for c in args.Cs.split(",")]
    threads = args.threads or os.cpu_count()
    t0 = time.perf_counter()
    rep = lpdsvm.grid_search(data, gammas=gammas, Cs=Cs, budget=args.budget, folds=args.folds,
                             threads=threads, tau=args.tau)
    wall = time.perf_counter() - t0
    out = {"build": args.module_dir, "n": args.n, "d": args.d, "budget": args.budget, "folds": args.folds,
           "gammas": gammas, "Cs": Cs, "threads": threads, "grid_wall_seconds": wall,
           "best_gamma": rep["best_gamma"], "best_C": rep["best_C"], "best_error": rep["best_error"],
           "binary_solves": rep["binary_solves"], "warm_started_solves": rep["warm_started_solves"],
           "entries": [{"gamma": e["gamma"], "C": e["C"], "mean_error": e["mean_error"], "epochs": e["epochs"],
                        "seconds": e["seconds"]} for e in rep["entries"]]}
    with open(args.out, "w") as f:
        json.dump(out, f)
    print(json.dumps({k: out[k] for k in ("build", "grid_wall_seconds", "best_gamma", "best_C", "best_error",
                                          "binary_solves", "warm_started_solves")}))


if __name__ == "__main__":
    main()
