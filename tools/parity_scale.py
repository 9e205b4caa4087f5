"""Full-size parity: device IHT fit vs the CPU oracle (reference algorithm) on
identical bytes and response.

    python tools/parity_scale.py --n 100000 --p 1000000 --k 20     # BASELINE config 3
    python tools/parity_scale.py --n 500000 --p 50000 --k 100 --missing 0.02

The matrix is generated on the device, downloaded verbatim, and the oracle
(C restatement of genoiht's kernels + numpy restatement of its solver, pinned
bit-exact to the reference in tests/test_oracle.py) fits the same y.
Writes a JSON record (support/iterations equality, max relative differences).
"""
import argparse
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
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return float("inf")
    scale = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--p", type=int, default=1_000_000)
    ap.add_argument("--k", type=int, default=20)
    ap.add_argument("--k-true", type=int, default=0)
    ap.add_argument("--missing", type=float, default=0.0)
    ap.add_argument("--seed", type=int, default=1608)
    ap.add_argument("--pheno-seed", type=int, default=1398)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    k_true = a.k_true or a.k

    t0 = time.time()
    m = gi.PackedGenotypeMatrix.synthetic(a.n, a.p, a.seed, missing_rate=a.missing)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=a.n))
    y, truth = simulate_phenotype(view, SimulationSpec(k_true=k_true, seed=a.pheno_seed))
    t1 = time.time()
    got = gi.fit(view, y, gi.IhtConfig(k=a.k))
    t2 = time.time()
    data = np.asarray(m.data)  # verbatim BED bytes, p x ceil(n/4) (no second copy)
    ref = oracle.OraclePacked.from_bed(data, a.n)
    assert np.array_equal(ref.u, m.u) and np.array_equal(ref.v, m.v), "stats differ"
    oracle.set_threads(os.cpu_count() or 1)
    t3 = time.time()
    want = oracle.fit(oracle.OracleView(ref, oracle.intercept(a.n)), y, a.k)
    t4 = time.time()
    rec = {
        "n": a.n, "p": a.p, "k": a.k, "k_true": k_true, "missing": a.missing,
        "xtr_format": "base-3" if m.xtr_base3 else "2-bit",
        "seed": a.seed, "pheno_seed": a.pheno_seed,
        "support_equal": bool(np.array_equal(got.model.support, want.support)),
        "iterations_gpu": got.iterations, "iterations_oracle": want.iterations,
        "reason_gpu": got.reason, "reason_oracle": want.reason,
        "stats_bit_identical": True,
        "beta_max_rel_diff": rel(got.model.weights, want.weights),
        "covar_max_rel_diff": rel(got.model.covar, want.covar),
        "loss_trace_max_rel_diff": rel(got.loss_trace, want.loss_trace),
        "support_gpu": got.model.support.tolist(),
        "planted_support_recovered": int(np.intersect1d(got.model.support, truth.support).size),
        "gpu_fit_seconds": t2 - t1, "oracle_fit_seconds": t4 - t3,
        "oracle_threads": os.cpu_count(), "setup_seconds": t1 - t0,
    }
    rec["parity"] = bool(rec["support_equal"] and got.iterations == want.iterations
                         and rec["beta_max_rel_diff"] <= 1e-6
                         and rec["loss_trace_max_rel_diff"] <= 1e-6)
    line = json.dumps(rec)
    print(line, flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(line + "\n")
    sys.exit(0 if rec["parity"] else 1)


if __name__ == "__main__":
    main()
