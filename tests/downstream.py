"""Downstream parity of the B200 factor (north star: "the trained α, w and test
accuracy must match the reference within a stated tolerance"; SURVEY.md §8(c)
criterion 3). TEST INFRASTRUCTURE: the reference's own code is the checker.

For one configuration:
  1. landmarks by the reference's select_landmarks (factor.cpp:27-31, seed 1), and L,
     G_ref by the reference's build_factor_with_landmarks (factor.cpp:112-143) built
     unmodified in oracle/_ref;
  2. G_gpu = the same rows through the C ABI (lpd_set_basis_dense + lpd_compute_g_dense)
     with the same landmarks and L — the product path;
  3. the reference's stage-2 solver, unchanged (make_binary_problem + solve_binary,
     dcd.cpp:60-89, 212-259), run on G_ref and on G_gpu with identical options;
  4. test decisions: reference = G_ref(test)·w_ref (its compute_G on the test rows);
     B200 = Z(test)·β with β = L·w_gpu (multiclass.cpp:126) as the projection operand
     of the factor kernel (K5) — the device prediction path;
  5. the solver's own noise floor: the reference solve on G_ref with another epoch-order
     seed (SolveOptions::seed, dcd.hpp:34), i.e. what the solver itself does not pin.

Metrics: |ΔD(α)| (absolute and relative), ‖Δw‖/‖w‖, max|Δα|/C, test error in
percentage points, agreement of test predictions, and the same numbers for the
seed-noise floor. The DCD dual Q = GGᵀ has rank b_eff < n, so α is not unique —
w and D(α) are (SPEC.md:315-318 judges solutions by dual objective and predictions).

  python tests/downstream.py c1 [out.json]     (needs a B200 and oracle/_ref)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2207_01016_b200 import synthetic  # noqa: E402

# name: (n_train, n_test, d, B, gamma, C, tau, data seed)
CASES = {
    # BASELINE.json config 1 exactly
    "c1": (20_000, 10_000, 50, 1_000, 0.02, 1.0, 1e-12, 1),
    # covtype-shaped (C2 d, B, γ = 1/d) at n = 200k rows
    "c2_200k": (200_000, 20_000, 54, 4_096, 1.0 / 54, 1.0, 1e-12, 2),
}


def run(name: str, ctx=None, eps: float = 1e-3, threads: int = 0) -> dict:
    import paper_2207_01016_b200 as P

    n, n_test, d, B, gamma, C, tau, seed = CASES[name]
    threads = threads or os.cpu_count() or 1
    X, y = synthetic.blobs(n + n_test, d, seed=seed)
    Xt, yt = X[n:], y[n:]
    X, y = X[:n], y[:n]
    ids = O.ref_select_landmarks(n, B, 1)
    csr_lm = O.dense_to_csr(X[ids])
    t0 = time.perf_counter()
    f = O.ref_factor_with_landmarks(O.dense_to_csr(X), csr_lm, gamma, tau, 4096, threads)
    ref_factor_s = time.perf_counter() - t0
    L, G_ref = f["L"], f["G"]
    own = ctx is None
    ctx = P.Context(1) if own else ctx
    try:
        ctx.set_basis_dense(X[ids], L, gamma)
        t0 = time.perf_counter()
        G_gpu = ctx.compute_g_dense(X)
        gpu_factor_s = time.perf_counter() - t0
        g_row_err = float(np.max(np.linalg.norm(G_gpu - G_ref, axis=1) / np.linalg.norm(G_ref, axis=1)))

        t0 = time.perf_counter()
        ref = O.ref_solve_binary(G_ref, y, C=C, eps=eps)
        ref_solve_s = time.perf_counter() - t0
        gpu = O.ref_solve_binary(G_gpu, y, C=C, eps=eps)
        floor = O.ref_solve_binary(G_ref, y, C=C, eps=eps, seed=2)

        # test decisions: reference path on the host, B200 path = K5 with β = L·w
        Gt_ref = O.ref_compute_g(O.dense_to_csr(Xt), csr_lm, L, gamma, 4096, threads)
        dec_ref = Gt_ref @ ref["w"]
        dec_floor = Gt_ref @ floor["w"]
        ctx.set_basis_dense(X[ids], np.ascontiguousarray((L @ gpu["w"])[:, None]), gamma)
        dec_gpu = ctx.compute_g_dense(Xt)[:, 0]
    finally:
        if own:
            ctx.close()

    def cmp(a, b, da, db):
        pa, pb = np.where(da > 0, 1.0, -1.0), np.where(db > 0, 1.0, -1.0)
        return {
            "dual_objective_abs_diff": abs(a["dual_objective"] - b["dual_objective"]),
            "dual_objective_rel_diff": abs(a["dual_objective"] - b["dual_objective"]) / abs(b["dual_objective"]),
            "w_rel_diff": float(np.linalg.norm(a["w"] - b["w"]) / np.linalg.norm(b["w"])),
            "alpha_max_abs_diff_over_C": float(np.max(np.abs(a["alpha"] - b["alpha"])) / C),
            "alpha_frac_diff_gt_1e-2C": float(np.mean(np.abs(a["alpha"] - b["alpha"]) > 1e-2 * C)),
            "test_error_pp_diff": 100.0 * abs(float(np.mean(pa != yt)) - float(np.mean(pb != yt))),
            "test_pred_agreement": float(np.mean(pa == pb)),
            "test_decision_max_abs_diff": float(np.max(np.abs(da - db))),
        }

    return {
        "case": name, "n": n, "n_test": n_test, "d": d, "B": B, "b_eff": int(f["b_eff"]), "gamma": gamma,
        "C": C, "tau": tau, "eps": eps, "threads": threads,
        "G_max_row_rel_err": g_row_err,
        "reference": {"dual_objective": ref["dual_objective"], "epochs": ref["epochs"],
                      "converged": ref["converged"], "test_error": float(np.mean(np.where(dec_ref > 0, 1.0, -1.0) != yt)),
                      "support_vectors": int(np.sum(ref["alpha"] > 0))},
        "b200": {"dual_objective": gpu["dual_objective"], "epochs": gpu["epochs"], "converged": gpu["converged"],
                 "test_error": float(np.mean(np.where(dec_gpu > 0, 1.0, -1.0) != yt)),
                 "support_vectors": int(np.sum(gpu["alpha"] > 0))},
        "b200_vs_reference": cmp(gpu, ref, dec_gpu, dec_ref),
        "solver_seed_floor": cmp(floor, ref, dec_floor, dec_ref),
        "seconds": {"reference_factor": ref_factor_s, "b200_factor_call": gpu_factor_s,
                    "reference_solve": ref_solve_s},
    }


if __name__ == "__main__":
    out = run(sys.argv[1] if len(sys.argv) > 1 else "c1")
    s = json.dumps(out, indent=1)
    print(s)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as fh:
            fh.write(s + "\n")
