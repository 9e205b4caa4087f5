"""Per-fit comparison of a warm-started CV fold chain (device vs the oracle)
for one stress_cv seed: support, iterations, reason, beta and loss trace."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
import paper_1608_01398_b200 as gi  # noqa: E402
from paper_1608_01398_b200 import model_select as ms  # noqa: E402


def main(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(150, 1500)); p = int(rng.integers(50, 3000))
    miss = float(rng.choice([0.0, 0.02]))
    codes = oracle.random_codes(n, p, seed=seed, missing_rate=miss)
    q = int(rng.integers(3, 6)); path = np.arange(1, int(rng.integers(3, 11)))
    std_mode = str(rng.choice(["train", "global"])); warm = bool(rng.random() < 0.3)
    covar = rng.standard_normal((n, 2)) if rng.random() < 0.3 else None
    support = np.sort(rng.choice(p, min(p, int(rng.integers(1, 6))), replace=False))
    ref_p = oracle.OraclePacked.from_codes(codes)
    y = ref_p.ax_columns(support, rng.standard_normal(support.size)) + \
        rng.normal(0, float(rng.choice([0.1, 0.5])), n)
    block = gi.CovariateBlock.build(covar, n=n)
    m = gi.PackedGenotypeMatrix.from_codes(codes)
    view = gi.StandardizedView(m, block)
    plan = gi.CvPlan.build(n, q, path, seed=seed)
    labels = plan.fold_labels
    for f in range(q):
        tr = np.flatnonzero(labels != f)
        v_train, _ = ms._fold_views(view, tr, np.flatnonzero(labels == f), std_mode)
        o_p = oracle.OraclePacked.from_codes(codes[tr])
        if std_mode == "global":
            o_p = o_p.with_stats(ref_p.u, ref_p.v)
        o_view = oracle.OracleView(o_p, block.values[tr])
        wd = wo = None
        for k in path:
            got = gi.fit(v_train, y[tr], gi.IhtConfig(k=int(k)), warm=wd)
            want = oracle.fit(o_view, y[tr], int(k), warm=wo)
            same = np.array_equal(got.model.support, want.support)
            b = np.max(np.abs(got.model.weights - want.weights) / np.maximum(np.abs(want.weights), 1e-300)) if same and want.weights.size else -1
            lt = np.max(np.abs(got.loss_trace[:min(len(got.loss_trace), len(want.loss_trace))] - want.loss_trace[:min(len(got.loss_trace), len(want.loss_trace))]) / np.abs(want.loss_trace[:min(len(got.loss_trace), len(want.loss_trace))]))
            print(f"loss {lt:.2e}", end=" ")
            print(f"fold {f} k={k}: support {'=' if same else '!='} it {got.iterations}/{want.iterations} "
                  f"reason {got.reason}/{want.reason} beta {b:.2e} bt {got.backtracks}")
            if os.environ.get("TRACE") and f == 0 and k == 2:
                print("  dev loss", got.loss_trace[:6])
                print("  ora loss", want.loss_trace[:6])
                print("  warm dev", wd.support, wd.weights, wd.covar)
                print("  warm ora", wo)
            wd, wo = got.model, (want.support, want.weights, want.covar)
    return 0


if __name__ == "__main__" and len(sys.argv) == 2:
    main(int(sys.argv[1]))


def first_step(seed, fold=0, k_prev=1, k=2):
    """The first iteration of the warm-started fit: device step-level API vs
    the oracle's step (restriction gradient, covariate gradient, mu, result)."""
    from paper_1608_01398_b200 import iht as giht
    rng = np.random.default_rng(seed)
    n = int(rng.integers(150, 1500)); p = int(rng.integers(50, 3000))
    miss = float(rng.choice([0.0, 0.02]))
    codes = oracle.random_codes(n, p, seed=seed, missing_rate=miss)
    q = int(rng.integers(3, 6)); path = np.arange(1, int(rng.integers(3, 11)))
    std_mode = str(rng.choice(["train", "global"])); rng.random()
    covar = rng.standard_normal((n, 2)) if rng.random() < 0.3 else None
    support = np.sort(rng.choice(p, min(p, int(rng.integers(1, 6))), replace=False))
    ref_p = oracle.OraclePacked.from_codes(codes)
    y = ref_p.ax_columns(support, rng.standard_normal(support.size)) + \
        rng.normal(0, float(rng.choice([0.1, 0.5])), n)
    block = gi.CovariateBlock.build(covar, n=n)
    view = gi.StandardizedView(gi.PackedGenotypeMatrix.from_codes(codes), block)
    plan = gi.CvPlan.build(n, q, path, seed=seed)
    tr = np.flatnonzero(plan.fold_labels != fold)
    v_train, _ = ms._fold_views(view, tr, np.flatnonzero(plan.fold_labels == fold), std_mode)
    o_view = oracle.OracleView(oracle.OraclePacked.from_codes(codes[tr]), block.values[tr])
    want0 = oracle.fit(o_view, y[tr], k_prev)
    warm_o = (want0.support, want0.weights, want0.covar)
    st_o = oracle.start(o_view, y[tr], k, warm_o)
    warm_d = gi.SparseModel.from_parts(want0.support, want0.weights, want0.covar, k_prev, p)
    cfg = gi.IhtConfig(k=k)
    st_d = giht.initial_state(v_train, y[tr], cfg, warm_d)
    print("loss", st_d.loss, st_o.loss)
    print("g on support dev", st_d.grad_gen[st_d.support], "ora", st_o.g[st_o.support])
    print("g_cov dev", st_d.grad_cov, "ora", st_o.g_cov)
    gi_ = np.argsort(-np.abs(st_o.g))[:5]
    print("top |g| ora", gi_, st_o.g[gi_], "dev", st_d.grad_gen[gi_])
    st_o2 = oracle.step(st_o, o_view, y[tr], k)
    st_d2 = giht.iht_step(st_d, v_train, y[tr], cfg)
    print("mu dev", st_d2.mu, "ora", st_o2.mu, "bt", st_d2.backtracks, st_o2.backtracks)
    print("support dev", st_d2.support, "ora", st_o2.support, "loss", st_d2.loss, st_o2.loss)


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "step":
    first_step(int(sys.argv[1]))


def native_first(seed, fold=0, k_prev=1, k=2):
    """The native fit of (fold, k) warm-started from the oracle's k_prev fit,
    with GI_TRACE_FIT=2 per-iteration lines, beside the oracle's first mu."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(150, 1500)); p = int(rng.integers(50, 3000))
    miss = float(rng.choice([0.0, 0.02]))
    codes = oracle.random_codes(n, p, seed=seed, missing_rate=miss)
    q = int(rng.integers(3, 6)); path = np.arange(1, int(rng.integers(3, 11)))
    std_mode = str(rng.choice(["train", "global"])); rng.random()
    covar = rng.standard_normal((n, 2)) if rng.random() < 0.3 else None
    support = np.sort(rng.choice(p, min(p, int(rng.integers(1, 6))), replace=False))
    ref_p = oracle.OraclePacked.from_codes(codes)
    y = ref_p.ax_columns(support, rng.standard_normal(support.size)) + \
        rng.normal(0, float(rng.choice([0.1, 0.5])), n)
    block = gi.CovariateBlock.build(covar, n=n)
    view = gi.StandardizedView(gi.PackedGenotypeMatrix.from_codes(codes), block)
    plan = gi.CvPlan.build(n, q, path, seed=seed)
    tr = np.flatnonzero(plan.fold_labels != fold)
    v_train, _ = ms._fold_views(view, tr, np.flatnonzero(plan.fold_labels == fold), std_mode)
    o_view = oracle.OracleView(oracle.OraclePacked.from_codes(codes[tr]), block.values[tr])
    want0 = oracle.fit(o_view, y[tr], k_prev)
    st_o = oracle.start(o_view, y[tr], k, (want0.support, want0.weights, want0.covar))
    idx, cols = oracle._restriction(st_o, o_view)
    print("oracle: restriction", idx, "g", st_o.g[idx], "g_cov", st_o.g_cov,
          "mu %.17g" % oracle._mu(st_o, o_view, idx, cols), flush=True)
    warm_d = gi.SparseModel.from_parts(want0.support, want0.weights, want0.covar, k_prev, p)
    res = gi.fit(v_train, y[tr], gi.IhtConfig(k=k), warm=warm_d)
    from paper_1608_01398_b200.iht import last_native_fit_info
    print("native", last_native_fit_info(), res.iterations, flush=True)


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "native":
    native_first(int(sys.argv[1]))
