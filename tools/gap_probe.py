"""Host-gap probe of the native loop at one GPU's shard of config 3 on 8 GPUs
(n = 100k, p = 125k): fit time vs time spent waiting in cudaStreamSynchronize."""
import os
import time

os.environ["GI_TRACE_FIT"] = "1"
import paper_1608_01398_b200 as gi  # noqa: E402
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype  # noqa: E402

m = gi.PackedGenotypeMatrix.synthetic(100000, 125000, 1608)
view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=100000))
y, _ = simulate_phenotype(view, SimulationSpec(k_true=20, seed=1398))
cfg = gi.IhtConfig(k=20)
gi.fit(view, y, cfg)
for _ in range(3):
    t0 = time.perf_counter()
    r = gi.fit(view, y, cfg, _resident=True)
    print(f"fit {1e3 * (time.perf_counter() - t0):.3f} ms, {r.iterations} iterations", flush=True)
