"""Per-point decision values through the reference's own Python API, from one build of
its `_core` module (tests/test_integration.py runs both builds in separate processes).

  python tests/integration_dv.py <module_dir> train <workdir> [--classes C --sparse-extra]
      trains a model with the build (the unmodified reference, oracle/_ref), saves it to
      <workdir>/model.txt and the test points to <workdir>/test.libsvm
  python tests/integration_dv.py <module_dir> dv <workdir> <out.npy>
      load_model + load_dataset + Model.decision_values (module.cpp:157-171 ->
      lpdsvm::decision_values, multiclass.cpp:137-151) and, for the B200 build, the
      adapter's device-call counter
"""
import ctypes
import glob
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _import(mdir):
    mdir = mdir if os.path.isabs(mdir) else os.path.join(ROOT, mdir)
    sys.path.insert(0, mdir)
    if os.path.isdir(os.path.join(mdir, "lpdsvm")):
        import lpdsvm
    else:
        import _core as lpdsvm
    return lpdsvm


def main():
    mdir, mode, work = sys.argv[1], sys.argv[2], sys.argv[3]
    lpdsvm = _import(mdir)
    if mode == "train":
        sys.path.insert(0, ROOT)
        from integration_train import libsvm_text
        from paper_2207_01016_b200 import synthetic

        classes = int(sys.argv[sys.argv.index("--classes") + 1]) if "--classes" in sys.argv else 2
        n, n_test, d = 3000, 400, 24
        if classes == 2:
            X, y = synthetic.blobs(n + n_test, d, seed=5)
        else:
            X, y = synthetic.imagenet_like(n + n_test, d, classes, seed=5)
            X = (X / 4.0).astype(np.float32).astype(np.float64)
        # sparse rows: explicit zeros are dropped by the parser, so every point has its own
        # support; with --sparse-extra the test points also carry features (d .. d+5) no
        # training point or landmark has (squared_distance's one-sided merge terms)
        X[np.abs(X) < 0.3] = 0.0
        Xt = X[n:].copy()
        if "--sparse-extra" in sys.argv:
            Xt = np.concatenate([Xt, np.round(np.linspace(-1, 1, 6 * n_test).reshape(n_test, 6), 3)], axis=1)
        train = lpdsvm.parse_dataset(libsvm_text(X[:n], y[:n]))
        model, _ = lpdsvm.train(train, budget=300, C=1.0, gamma=0.05, threads=4, tau=1e-10)
        model.save(os.path.join(work, "model.txt"))
        with open(os.path.join(work, "test.libsvm"), "w") as fh:
            fh.write(libsvm_text(Xt, y[n:]))
        return
    out = sys.argv[4]
    model = lpdsvm.load_model(os.path.join(work, "model.txt"))
    test = lpdsvm.load_dataset(os.path.join(work, "test.libsvm"))
    dv = model.decision_values(test)
    np.save(out, dv)
    calls = -1
    so = glob.glob(os.path.join(os.path.dirname(lpdsvm.__file__), "_core*.so"))[0]
    lib = ctypes.CDLL(so)
    if hasattr(lib, "lpd_adapter_dv_calls"):
        lib.lpd_adapter_dv_calls.restype = ctypes.c_longlong
        calls = int(lib.lpd_adapter_dv_calls())
    with open(out + ".json", "w") as fh:
        json.dump({"dv_calls": calls, "n": len(test), "pairs": int(model.num_pairs)}, fh)


if __name__ == "__main__":
    main()
