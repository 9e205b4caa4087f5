"""Diagnose a CV golden case fit by fit: replay each fold's (warm-started)
path on the device and in the oracle, report the first fit whose support,
iterations or weights differ.

    python tools/cv_diag.py cvL_train_warm_miss [--compact 1]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)

import golden_io  # noqa: E402
import oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--compact", default="1")
    ap.add_argument("--exact", default="")
    a = ap.parse_args()
    os.environ["GI_CV_COMPACT"] = a.compact
    if a.exact:
        os.environ["GI_XTR_EXACT"] = a.exact
    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200 import model_select as ms
    from paper_1608_01398_b200.iht import last_native_fit_info

    case = golden_io.load("large")[a.case]
    n, p = case["n"], case["p"]
    m = gi.PackedGenotypeMatrix.synthetic(n, p, case["seed"], missing_rate=case["missing"])
    data = np.array(m.data)
    ref = oracle.OraclePacked.from_bed(data, n)
    y = case["y"]
    labels = case["labels"]
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
    for f in range(case["q"]):
        test = np.flatnonzero(labels == f)
        train = np.flatnonzero(labels != f)
        v_tr, v_te = ms._fold_views(view, train, test, case["std_mode"], a.compact == "1")
        g_tr = ref.subset_rows(train)
        if case["std_mode"] == "global":
            g_tr = g_tr.with_stats(ref.u, ref.v)
        o_tr = oracle.OracleView(g_tr, oracle.intercept(train.size))
        warm_d = warm_o = None
        for k in case["path"]:
            cfg = gi.IhtConfig(k=int(k))
            got = gi.fit(v_tr, y[train], cfg, warm=warm_d if case["warm"] else None)
            info = last_native_fit_info()
            want = oracle.fit(o_tr, y[train], int(k), warm=warm_o if case["warm"] else None)
            warm_d, warm_o = got.model, (want.support, want.weights, want.covar)
            same_sup = np.array_equal(got.model.support, want.support)
            rel = float(np.max(np.abs(got.model.weights - want.weights) / np.abs(want.weights))) \
                if same_sup and want.weights.size else float("nan")
            flag = "" if same_sup and got.iterations == want.iterations and rel < 1e-6 else "  <-- DIFF"
            print(f"fold {f} k={k}: iters {got.iterations}/{want.iterations} reason "
                  f"{got.reason}/{want.reason} support_equal={same_sup} beta_rel={rel:.2e} "
                  f"kernel={info and info['xtr_kernel']}{flag}", flush=True)
            if flag:
                print("   got ", got.model.support.tolist(), got.loss_trace.tolist())
                print("   want", want.support.tolist(), want.loss_trace.tolist())


if __name__ == "__main__":
    main()
