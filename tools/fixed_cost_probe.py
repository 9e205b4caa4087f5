"""Per-fit wall time of the native loop at the small / shard shapes (median of
many fits), optionally A/B over an environment switch: GI_AB="NAME=a,b".

    python tools/fixed_cost_probe.py
"""
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = {"c1": (1000, 10000, 10), "c2k30": (5000, 100000, 30),
          "shard8": (100000, 125000, 20)}


def one(shape):
    sys.path.insert(0, ROOT)
    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

    n, p, k = SHAPES[shape]
    m = gi.PackedGenotypeMatrix.synthetic(n, p, 1608)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
    y, _ = simulate_phenotype(view, SimulationSpec(k_true=k, seed=1398))
    cfg = gi.IhtConfig(k=k)
    gi.fit(view, y, cfg)
    ts, it = [], 0
    for _ in range(30 if n < 50000 else 10):
        t0 = time.perf_counter()
        r = gi.fit(view, y, cfg, _resident=True)
        ts.append(time.perf_counter() - t0)
        it = r.iterations
    med = statistics.median(ts)
    print(f"{shape} {os.environ.get('GI_AB_TAG', '')}: {1e3 * med:.3f} ms per fit, "
          f"{it} iterations, {it / med:.0f} it/s, support {r.model.support[:5].tolist()}...",
          flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        one(sys.argv[1])
    else:
        ab = os.environ.get("GI_AB", "")
        name, vals = (ab.split("=", 1)[0], ab.split("=", 1)[1].split(",")) if ab else ("", [""])
        for shape in SHAPES:
            for val in vals:
                env = dict(os.environ, GI_AB_TAG=f"{name}={val}" if name else "")
                if name:
                    env[name] = val
                subprocess.run([sys.executable, __file__, shape], env=env, check=True)
