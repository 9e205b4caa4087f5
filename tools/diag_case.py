"""Replay one stress_parity case step by step on the device (Python loop over
the device primitives) and in the oracle; report the first divergence and the
top-k boundary margin |v_(k)| - |v_(k+1)| of the candidate at each step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import stress_parity as sp  # noqa: E402
import oracle  # noqa: E402
import paper_1608_01398_b200 as gi  # noqa: E402

seed = int(sys.argv[1])
view, ref_view, y, k, warm, warm_model, desc = sp.build(seed)
print(desc)
cfg = gi.IhtConfig(k=k)
st = oracle.start(ref_view, y, k, warm)
dst = gi.initial_state(view, y, cfg, warm=warm_model)
for it in range(60):
    g_ref, g_dev = st.g.copy(), np.asarray(dst.gradient[: view.p])
    gerr = np.max(np.abs(g_dev - g_ref)) / max(np.sqrt(np.mean(g_ref ** 2)), 1e-300)
    beta0 = st.beta.copy()
    oracle.step(st, ref_view, y, k)
    gi.iht_step(dst, view, y, cfg)
    mu = st.mu
    vals = np.sort(np.abs(beta0 - mu * g_ref))[::-1]
    gap = (vals[k - 1] - vals[k]) / vals[k - 1] if k < vals.size and vals[k - 1] > 0 else np.inf
    print(f"   top-k boundary gap (relative) {gap:.2e}")
    sup_ref = np.flatnonzero(st.beta)
    sup_dev = np.asarray(dst.support)
    print(f"it {it:2d}: g err {gerr:.1e} rms, mu {mu:.6g}, backtracks {st.backtracks}, "
          f"support equal {np.array_equal(np.sort(sup_ref), np.sort(sup_dev))}, loss "
          f"{st.loss:.12g} vs {dst.loss:.12g}")
    if not np.array_equal(np.sort(sup_ref), np.sort(sup_dev)):
        print("  oracle support", sup_ref, "\n  device support", sup_dev)
        break
    if st.step_inf < cfg.tol or st.collapsed:
        break
