"""Where a config-4 CV's time goes: per-job fit / predict intervals, fold setup,
final fit and refit (host timestamps), lock-step sweep counts.

    python tools/cv_timeline.py [--n 20000 --p 500000]
"""
import argparse
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--p", type=int, default=500000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--switch", type=float, default=0.0, help="sys.setswitchinterval (s)")
    ap.add_argument("--gc-off", action="store_true", help="gc.disable() around the runs")
    a = ap.parse_args()
    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200 import model_select as ms
    from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

    m = gi.PackedGenotypeMatrix.synthetic(a.n, a.p, 1608)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=a.n))
    y, _ = simulate_phenotype(view, SimulationSpec(k_true=10, seed=1398))
    plan = gi.CvPlan.build(a.n, 5, np.arange(1, 21), seed=2016)
    events = []
    lock = threading.Lock()
    orig_fit, orig_pred, orig_views = ms.fit, ms.predict, ms._fold_views
    orig_refit = ms.refit_least_squares

    def wrap(name, fn):
        def inner(*args, **kw):
            t0 = time.perf_counter()
            out = fn(*args, **kw)
            with lock:
                events.append((name, threading.get_ident(), t0, time.perf_counter()))
            return out
        return inner

    from paper_1608_01398_b200 import _native
    L = _native.lib()
    for fn in ("gi_fit_batched", "gi_fit"):
        setattr(L, fn, wrap("native", getattr(L, fn)))
    if a.switch > 0:
        sys.setswitchinterval(a.switch)
    if a.gc_off:
        import gc
        gc.disable()
    orig_run = ms._run_concurrently

    def run_concurrently(jobs, workers):
        t_sub = time.perf_counter()

        def tagged(job):
            def inner():
                with lock:
                    events.append(("job", threading.get_ident(), time.perf_counter(), t_sub))
                return job()
            return inner
        return orig_run([tagged(j) for j in jobs], workers)

    ms._run_concurrently = run_concurrently
    ms.fit_many = wrap("fit_many", ms.fit_many)
    ms.fit = wrap("fit", orig_fit)
    ms.predict = wrap("predict", orig_pred)
    ms._fold_views = wrap("fold_views", orig_views)
    ms.refit_least_squares = wrap("refit", orig_refit)
    for rep in range(a.reps):
        events.clear()
        t0 = time.perf_counter()
        gi.cv_iht(view, y, plan, gi.IhtConfig(k=20))
        total = time.perf_counter() - t0
        by = {}
        for name, _, s, e in events:
            by.setdefault(name, []).append((s - t0, e - t0))
        print(f"rep {rep}: cv {1e3 * total:.1f} ms, batch {ms.LAST_BATCH}")
        for name, iv in by.items():
            d = [e - s for s, e in iv]
            print(f"  {name:10s} n={len(iv):3d} first start {1e3 * min(s for s, _ in iv):7.1f} "
                  f"last end {1e3 * max(e for _, e in iv):7.1f} ms, mean {1e3 * np.mean(d):6.2f} "
                  f"max {1e3 * max(d):6.2f} ms")
        fits = sorted(iv for iv in by.get("fit", []))
        if fits:
            # fits still running at each millisecond: how full the group stays
            horizon = int(1e3 * max(e for _, e in fits)) + 1
            live = [sum(1 for s, e in fits if s * 1e3 <= t < e * 1e3) for t in range(horizon)]
            print("  live fits per 10 ms:", [max(live[i:i + 10]) for i in range(0, horizon, 10)])
        jobs = sorted(s for s, _ in by.get("job", []))
        if jobs:
            print("  job dequeue ms (sorted, every 4th of the first 40):",
                  [round(1e3 * j, 1) for j in jobs[:40:4]])
        nat = sorted(by.get("native", []))
        if fits and len(nat) == len(fits):
            pre = [ns - fs for (fs, _), (ns, _) in zip(fits, nat)]
            post = [fe - ne for (_, fe), (_, ne) in zip(fits, nat)]
            print(f"  python before native: mean {1e3 * np.mean(pre):.2f} max {1e3 * max(pre):.2f} ms;"
                  f" after: mean {1e3 * np.mean(post):.2f} max {1e3 * max(post):.2f} ms")


if __name__ == "__main__":
    main()
