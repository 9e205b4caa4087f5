"""Time the X^T r kernels on the device (CUDA events around the C-ABI calls'
device work is not separable here, so this times gi_aty / gi_aty_batched end
to end with the residual upload -- use ncu for kernel-only numbers).

    python tools/xtr_mma_bench.py --n 500000 --p 100000 --missing 0.02
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=500_000)
    ap.add_argument("--p", type=int, default=100_000)
    ap.add_argument("--missing", type=float, default=0.02)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import paper_1608_01398_b200 as gi

    m = gi.PackedGenotypeMatrix.synthetic(a.n, a.p, 1608, missing_rate=a.missing)
    rng = np.random.default_rng(1)
    R = rng.standard_normal((a.batch, a.n))
    nb = (a.n + 3) // 4
    for mode in ("fast", "mma"):
        if a.batch == 1:
            fn = lambda: m.aty_genetic(R[0], mode=mode)  # noqa: E731
        else:
            fn = lambda: m.aty_batched(R, mode=mode)  # noqa: E731
        fn()
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            out = fn()
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"{mode:5s} n={a.n} p={a.p} miss={a.missing} B={a.batch}: {1e3 * t:.2f} ms per call "
              f"(incl. H2D of R, D2H of G), {a.batch * a.p * nb / t / 1e9:.0f} RHS-packed-GB/s",
              flush=True)
        if mode == "fast":
            ref = out
        else:
            g1 = np.atleast_2d(ref)
            g2 = np.atleast_2d(out)
            rms = np.sqrt(np.mean(g1 ** 2))
            print(f"      max |mma - fast| = {np.max(np.abs(g2 - g1)) / rms:.3g} rms(g)")


if __name__ == "__main__":
    main()
