"""Full-size parity of config 4 (n = 20k, p = 500k, 5-fold CV over k = 1..20,
cold starts, train standardisation): the device cv_iht (lock-step group,
held-out scoring in the fits) against the oracle's cv -- the reference's
per-fold re-pack and loop -- on the same bytes and phenotype.  Compares
k_best, the whole (budget, fold) MSE grid and the final refit model.

    python tools/parity_c4_full.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
import paper_1608_01398_b200 as gi  # noqa: E402
from paper_1608_01398_b200.model_select import LAST_BATCH  # noqa: E402
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_c4_full.json"
    n, p, seed, pheno_seed = 20_000, 500_000, 1608, 1398
    path = np.arange(1, 21)
    m = gi.PackedGenotypeMatrix.synthetic(n, p, seed)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
    y, truth = simulate_phenotype(view, SimulationSpec(k_true=10, seed=pheno_seed))
    plan = gi.CvPlan.build(n, 5, path, seed=2016)
    gi.cv_iht(view, y, plan, gi.IhtConfig(k=20))  # warm-up
    t0 = time.perf_counter()
    rep = gi.cv_iht(view, y, plan, gi.IhtConfig(k=20))
    t_dev = time.perf_counter() - t0
    batch = dict(LAST_BATCH)
    oracle.set_threads(os.cpu_count() or 1)
    ref = oracle.OraclePacked.from_bed(oracle.synth_bed(seed, n, 0, p, missing=0.0), n)
    t0 = time.perf_counter()
    want = oracle.cv(oracle.OracleView(ref, oracle.intercept(n)), y, 5, path, 2016,
                     labels=plan.fold_labels)
    t_cpu = time.perf_counter() - t0
    f_sup, f_w, f_cov = want.final
    mse_rel = float(np.max(np.abs(rep.mse - want.mse) / np.abs(want.mse)))
    same_sup = bool(np.array_equal(rep.final_model.support, f_sup))
    w_rel = float(np.max(np.abs(rep.final_model.weights - f_w) / np.abs(f_w))) if same_sup else None
    rec = {"workload": "BASELINE config 4: n=20000 x p=500000, 5-fold CV over k=1..20, cold, train",
           "checker": "oracle cv (the reference's per-fold re-pack and loop, pinned to its golden "
                      "vectors) on the CPU twin of the device generator's bytes",
           "k_best": [int(rep.k_best), int(want.k_best)],
           "k_best_equal": int(rep.k_best) == int(want.k_best),
           "mse_grid_max_rel": mse_rel,
           "final_support_equal": same_sup,
           "final_weights_max_rel": w_rel,
           "device_cv_s": t_dev, "oracle_cv_s": t_cpu, "oracle_threads": os.cpu_count(),
           "xtr_batching": batch,
           "ok": int(rep.k_best) == int(want.k_best) and same_sup and mse_rel <= 1e-6}
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec), flush=True)
    return 0 if rec["ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
