"""Latency model of the stream primitives the native loop uses (tiny copies, launches, syncs)."""
import time

import torch

x = torch.zeros(64, dtype=torch.float64, device="cuda")
h = torch.empty(64, dtype=torch.float64).pin_memory()
s = torch.cuda.current_stream()


def bench(label, fn, reps=2000):
    for _ in range(50):
        fn()
    s.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    dt = (time.perf_counter() - t0) / reps * 1e6
    print(f"{label:48s} {dt:7.1f} us", flush=True)


bench("sync only", lambda: s.synchronize())
bench("1 kernel + sync", lambda: (x.add_(1), s.synchronize()))
bench("5 kernels + sync", lambda: ([x.add_(1) for _ in range(5)], s.synchronize()))
bench("10 kernels + sync", lambda: ([x.add_(1) for _ in range(10)], s.synchronize()))
bench("1 D2H 64B + sync", lambda: (h[:8].copy_(x[:8], non_blocking=True), s.synchronize()))
bench("3 D2H 64B + sync", lambda: ([h[:8].copy_(x[:8], non_blocking=True) for _ in range(3)],
                                   s.synchronize()))
bench("1 H2D 64B + sync", lambda: (x[:8].copy_(h[:8], non_blocking=True), s.synchronize()))
bench("4 H2D 64B + sync", lambda: ([x[:8].copy_(h[:8], non_blocking=True) for _ in range(4)],
                                   s.synchronize()))
bench("H2D, kernel, D2H + sync", lambda: (x[:8].copy_(h[:8], non_blocking=True), x.add_(1),
                                          h[:8].copy_(x[:8], non_blocking=True), s.synchronize()))
bench("10 H2D + 5 kernels + 5 D2H + sync",
      lambda: ([x[:8].copy_(h[:8], non_blocking=True) for _ in range(10)],
               [x.add_(1) for _ in range(5)],
               [h[:8].copy_(x[:8], non_blocking=True) for _ in range(5)], s.synchronize()))
