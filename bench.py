#!/usr/bin/env python
"""Benchmark: IHT iterations/s and X^T r packed-genotype GB/s on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on):
synthetic genotypes n = 100,000 x p = 1,000,000 (25 GB packed, generated on
the device; law of the reference's random_packed_matrix), intercept covariate,
planted phenotype k_true = 20 (seed 1398), IhtConfig(k=20) with the reference
defaults.  One step = one cold-start IHT fit to convergence; the metric is
iterations per second.  The 25 GB matrix is far larger than the 126 MB L2, so
every X^T r streams from HBM (no flush needed).

  value   device-resident: matrix, response and covariates already in HBM;
          the native loop (gi_fit, or gi_fit_sharded under torchrun) runs each
          fit; CUDA events around the timed fits, host syncs included.
  e2e     public API: fit(view, y, IhtConfig(k=20)) with y in pinned host
          memory; the response upload and the FitResult download are inside
          the timed region.
  roofline  the X^T r kernel (aty_fast_kernel): algorithmic bytes per launch
          (p*ceil(n/4) + 8n + 24p) over its average
          CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the reference's own CPU path on the host: genoiht 0.1.0 itself
          (installed unmodified into baseline/_ref; its numba kernels on all
          host threads) fitting the first ~0.4 GB of SNPs of the same matrix
          with the same response law; per-iteration time is scaled by p / p_slice
          (the reference spends >97% of a config-3 iteration in work linear in
          p).  The oracle port stands in when baseline/_ref
          is absent (kind "port").
  parity  the timed fit against the oracle fit on the same bytes (support,
          iterations, reason equal; beta / loss relative differences), N=1.

--impl reference runs only that CPU path (rank 0): one slice fit per step,
ms_per_step = the wall time a step took, value scaled to the full matrix
("extrapolated" states the factor).

Multi-GPU: `bench.py --gpus N` launches N ranks itself through
torch.distributed.run when WORLD_SIZE is unset (or run it under torchrun):
one process per GPU, the SNPs sharded over the ranks, NCCL for the n-vector
all-reduces and the top-k candidate all-gathers; the fit size stays fixed
(strong scaling).  The timed loop runs uninstrumented; X^T r launch times
come from a separate instrumented pass.
"""

from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IHT iterations/sec (X^T r packed-genotype GB/s vs HBM peak)"
FALLBACK_HBM_GBS = 6650.0
SPEC_HBM_GBS = 8000.0  # B200 datasheet HBM3e bandwidth ("~8 TB/s", BASELINE.json)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--samples", dest="n", type=int, default=100_000)
    ap.add_argument("--snps", dest="p", type=int, default=1_000_000)
    ap.add_argument("--k", type=int, default=20)
    ap.add_argument("--missing", type=float, default=0.0)
    ap.add_argument("--seed", type=int, default=1608)
    ap.add_argument("--pheno-seed", type=int, default=1398)
    ap.add_argument("--cpu-slice", type=int, default=0,
                    help="SNPs in the CPU sample (0 = auto, ~0.4 GB of packed genotypes)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-parity", dest="parity", action="store_false",
                    help="skip the parity leg (oracle fit on the same bytes, N=1 only)")
    ap.add_argument("--workload", default="c3", choices=["c3", "c2path", "c4cv", "c5"],
                    help="c3 (default, the metric's config), c2path (BASELINE config 2: "
                         "k=10..50 model-size path at n=5k x p=100k), c4cv (config 4: "
                         "5-fold CV over k=1..20 at n=20k x p=500k), c5 (config 5: "
                         "n=p=500k, 2%% missing, k=100; 62.5 GB)")
    a = ap.parse_args()
    if a.workload == "c5":  # same measurement as c3 on the UK-Biobank-scale shape
        a.n, a.p, a.k, a.missing = 500_000, 500_000, 100, 0.02
    return a


def config_of(a, world):
    which = "5" if a.workload == "c5" else "3"
    return {"workload": f"BASELINE config {which}: synthetic BED n={a.n} x p={a.p} "
                        f"({a.p * ((a.n + 3) // 4) / 1e9:.1f} GB packed), k={a.k}, "
                        f"k_true={a.k}, intercept covariate, missing={a.missing}",
            "n": a.n, "p": a.p, "k": a.k, "step": "one cold-start IHT fit to convergence",
            "parallelism": (f"snp-shard{world}" if world > 1 or
                            os.environ.get("GI_FORCE_SHARDED") == "1" else "single-gpu"),
            "l2": "inputs (packed X) >> 126 MB L2; no flush needed"}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def smem_roofline(n, p, ms, sm_mhz, sms, missing, miss_group_frac=None, base3=False):
    """Secondary roofline of aty_fast_kernel: its shared-memory traffic against
    the SM crossbar (128 B/clk/SM, B300_MICROARCH.md "LDS/STS") at the SM clock
    sampled during the run.  LSU shared-memory traffic per byte of the tiled
    matrix: 1 B read back from the TMA-staged block by the consumer warp and
    4 B of lookup-table read, plus one 128 KiB table build per (work item,
    sample tile).  The TMA bulk copies fill shared memory through the async
    copy path, not the LSU crossbar: this count matches ncu's
    shared-memory LSU wavefronts of the kernel (1.04e9 modelled vs 1.078e9
    measured at config 3, profiles/r01_summary.md).  Groups with a missing
    genotype add a second 4 B lookup per byte: counted when the fraction of
    such groups is known (`miss_group_frac`)."""
    if not ms or not sm_mhz:
        return None
    # base-3 copy (missing-free matrices): 640-sample tiles of the same 4 KiB blocks
    T = (n + 639) // 640 if base3 else (n + 511) // 512
    G = (p + 31) // 32
    per_wave = sms * 112  # kMaxGroups groups per work item (aty.cu)
    items = min(sms * ((G + per_wave - 1) // per_wave), G)
    per_byte = 5.0 + 4.0 * (miss_group_frac or 0.0)
    smem_bytes = int(per_byte * G * T * 4096) + items * T * 131072
    achieved = smem_bytes / (ms / 1e3) / 1e9
    peak = 128 * sms * sm_mhz * 1e6 / 1e9
    return {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "bytes_per_launch": smem_bytes,
            "peak_basis": f"128 B/clk/SM x {sms} SMs x {sm_mhz:.0f} MHz (median sampled SM clock)",
            "missing_group_fraction": miss_group_frac,
            "note": ("lower bound: groups with missing genotypes not counted"
                     if missing and miss_group_frac is None else None)}


def traffic_from_profile(n, p, fmt, missing=0.0):
    """DRAM bytes per aty_fast_kernel launch from the committed ncu capture of
    this shape and format (profiles/aty_fast_traffic*.json), else None."""
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "aty_fast_traffic*.json"))):
        try:
            with open(path) as fh:
                rec = json.load(fh)
            if rec.get("n") == n and rec.get("p") == p and rec.get("format", "2-bit") == fmt \
                    and float(rec.get("missing", 0.0)) == float(missing):
                return float(rec["dram_bytes_per_launch"])
        except Exception:
            continue
    return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx = float(s[1])
                for name, flag in zip(names, s[3:7]):
                    if flag.strip().lower() == "active":
                        reasons.add(name)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU leg
def load_genoiht():
    """The UNMODIFIED reference package, installed into baseline/_ref by
    `pip install --no-index --no-deps --target baseline/_ref <reference pkg>`
    (git-ignored; travels to the GPU box with the snapshot).  None when absent."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "genoiht")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/genoiht_numba_cache")
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    try:
        import genoiht
    except Exception as exc:  # numba missing or broken: fall back to the port
        print(f"bench: reference package not importable ({exc}); timing the oracle port",
              file=sys.stderr)
        return None
    return genoiht


def slice_snps(n):
    """SNPs of the CPU sample: ~0.4 GB of packed genotypes, so one reference
    X^T r sweep takes ~0.1-0.3 s and a whole fit a few seconds."""
    nb = (n + 3) // 4
    return max(2000, int(0.4e9 // nb))


def reference_slice_fits(n, p, p_slice, seed, missing, k, pheno_seed, reps):
    """The reference's own CPU implementation of the path, timed: cold-start
    IHT fits through genoiht's public API (genoiht.fit, reference iht.py:326 ->
    _aty_kernel geno_matrix.py:142) on the first p_slice SNPs of the
    workload's matrix (same bytes: the CPU twin of the device generator),
    with all host threads.  The matrix is built with the SURVEY.md section
    8(c) adapter (variant-major bytes + genoiht's own _packed_stats; data_t is
    never read at these support sizes).  Falls back to the oracle port when
    baseline/_ref is absent.  Returns a dict with per-fit seconds and
    iterations, the thread count and the kind ("reference" | "port")."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # the CPU twin of the synthetic-BED generator (same bytes)

    threads = os.cpu_count() or 1
    data = oracle.synth_bed(seed, n, 0, p_slice, missing=missing)
    genoiht = load_genoiht()
    kk = min(k, p_slice)
    if genoiht is not None:
        from genoiht import geno_matrix as ref_gm

        threads = genoiht.set_worker_threads(threads)
        u, v = ref_gm._packed_stats(data, n)
        mat = genoiht.PackedGenotypeMatrix(n=n, p=p_slice, data=data,
                                           data_t=np.zeros((n, 0), np.uint8), u=u, v=v)
        view = genoiht.StandardizedView(mat, genoiht.CovariateBlock.build(None, n=n))
        y, _ = genoiht.simulate_phenotype(view, genoiht.SimulationSpec(k_true=kk, seed=pheno_seed))

        def one():
            return genoiht.fit(view, y, genoiht.IhtConfig(k=kk)).iterations
        kind = "reference"
        what = "genoiht 0.1.0 (baseline/_ref, numba) fit()"
    else:
        oracle.set_threads(threads)
        mat = oracle.OraclePacked.from_bed(data, n)
        view = oracle.OracleView(mat, oracle.intercept(n))
        rng = np.random.default_rng(pheno_seed)
        causal = np.sort(rng.choice(p_slice, size=kk, replace=False)).astype(np.int64)
        eff = rng.normal(0.0, np.sqrt(0.01), size=kk)
        y = mat.ax_columns(causal, eff) + rng.normal(0.0, np.sqrt(0.01), size=n)

        def one():
            return oracle.fit(view, y, kk).iterations
        kind = "port"
        what = "oracle port (C restatement of genoiht's kernels + its solver) fit"
    secs, iters = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        iters.append(one())
        secs.append(time.perf_counter() - t0)
    return {"secs": secs, "iters": iters, "threads": threads, "kind": kind, "what": what,
            "k": kk}


def slice_rate(rec, p, p_slice, skip=0):
    """it/s of the full-p workload from the slice fits: the reference spends
    >97% of a config-3 iteration in work linear in p (X^T r, top-k, axpy;
    SURVEY.md section 0), so per-iteration time is scaled by p / p_slice."""
    secs, iters = rec["secs"][skip:], rec["iters"][skip:]
    t_it = sum(secs) / max(sum(iters), 1)
    return 1.0 / (t_it * p / p_slice), t_it


def secondary_shape(workload):
    """(n, p, k_true, path) of the config-2 / config-4 workloads."""
    if workload == "c2path":
        return 5000, 100_000, 20, np.arange(10, 51)
    return 20_000, 500_000, 10, np.arange(1, 21)


def reference_secondary(a):
    """Reference arm of --workload c2path / c4cv, on the host only: the same
    bytes (CPU twin of the device generator) and the same phenotype draws
    (simulate.py's rng sequence, X_S b through the oracle's bit-exact ax)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    n, p, k_true, path = secondary_shape(a.workload)
    threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    ref = oracle.OraclePacked.from_bed(oracle.synth_bed(a.seed, n, 0, p, missing=a.missing), n)
    rng = np.random.default_rng(a.pheno_seed)  # simulate_phenotype (simulate.py:68-83)
    causal = np.sort(rng.choice(p, size=k_true, replace=False)).astype(np.int64)
    effects = rng.normal(0.0, np.sqrt(0.01), size=k_true)
    y = ref.ax_columns(causal, effects) + rng.normal(0.0, np.sqrt(0.01), size=n)
    view = oracle.OracleView(ref, oracle.intercept(n))
    line = {"impl": "reference", "metric": METRIC, "unit": "it/s", "n_gpus": a.gpus,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "steps": a.steps, "warmup": a.warmup}
    if a.workload == "c2path":
        line["config"] = {"workload": f"BASELINE config 2: n={n} x p={p}, model-size path "
                                      f"k=10..50 (41 cold fits), k_true={k_true}",
                          "step": "all 41 fits of the path"}
        times, iters = [], 0
        for step in range(a.warmup + a.steps):
            t0 = time.perf_counter()
            fits = [oracle.fit(view, y, int(k)) for k in path]
            if step >= a.warmup:
                times.append(time.perf_counter() - t0)
                iters = sum(f.iterations for f in fits)
        t = statistics.median(times)
        line.update(value=iters / t, ms_per_step=1e3 * t,
                    cpu_baseline={"value": iters / t, "unit": "it/s", "cores": threads,
                                  "kind": "port", "sample": "the full 41-fit path on the oracle"})
    else:
        line["config"] = {"workload": f"BASELINE config 4: n={n} x p={p}, 5-fold CV over "
                                      f"k=1..20 + final fit and refit, k_true={k_true}, "
                                      f"fold seed 2016", "step": "one cv_iht call"}
        labels = oracle.folds(n, 5, 2016)
        train, test = np.flatnonzero(labels != 0), np.flatnonzero(labels == 0)
        t0 = time.perf_counter()
        g_train = ref.subset_rows(train)
        ref.subset_rows(test)
        t_repack = time.perf_counter() - t0
        t0 = time.perf_counter()
        fold_fit = oracle.fit(oracle.OracleView(g_train, oracle.intercept(train.size)),
                              y[train], k_true)
        t_fit = time.perf_counter() - t0
        t_cv = 5 * t_repack + 101 * t_fit
        line.update(value=None, cv_seconds=t_cv, ms_per_step=1e3 * t_cv,
                    cpu_baseline={"value": 1.0 / t_cv, "unit": "cv/s", "cores": threads,
                                  "kind": "port",
                                  "sample": f"one fold re-pack ({t_repack:.1f} s, x5) + one fit "
                                            f"at k={k_true} ({fold_fit.iterations} iterations, "
                                            f"{t_fit:.2f} s, x101 fits), extrapolated"})
    v = line["value"] if line["value"] is not None else 1.0 / line["cv_seconds"]
    line["e2e"] = {"value": v, "unit": line["unit"] if line["value"] is not None else "cv/s",
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if a.workload in ("c2path", "c4cv"):
        reference_secondary(a)
        return
    p_slice = min(a.p, a.cpu_slice or slice_snps(a.n))
    rec = reference_slice_fits(a.n, a.p, p_slice, a.seed, a.missing, a.k, a.pheno_seed,
                               a.warmup + a.steps)
    value, t_it = slice_rate(rec, a.p, p_slice, skip=a.warmup)
    timed = rec["secs"][a.warmup:]
    nb = (a.n + 3) // 4
    sample = (f"{rec['what']} with k={rec['k']} on the first {p_slice} of the workload's "
              f"{a.p} SNPs at n={a.n} ({p_slice * nb / 1e9:.2f} GB packed, same bytes), "
              f"{rec['threads']} host threads; one fit per step; per-iteration time scaled "
              f"by p / p_slice = {a.p / p_slice:.1f} to the full matrix")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "it/s",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            # the wall time a step actually took (one slice fit)
            "ms_per_step": 1e3 * statistics.mean(timed),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(a, a.gpus),  # the workload our arm runs at this N
            "host": "reference CPU path on the box's host cores (no GPU)",
            "extrapolated": {"from_p": p_slice, "to_p": a.p, "factor": a.p / p_slice,
                             "seconds_per_iteration_slice": t_it,
                             "iterations_per_step": rec["iters"][a.warmup:]},
            "cpu_baseline": {"value": value, "unit": "it/s", "cores": rec["threads"],
                             "kind": rec["kind"], "sample": sample},
            "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def secondary(a):
    """Model-size path (config 2) or cross-validation (config 4), 1 GPU.

    One step = the whole path / the whole CV; value = IHT iterations per second
    over it (all fits run concurrently on the device, one stream each).  The
    CPU baseline runs the oracle (reference algorithm) on the same bytes: the
    full path for config 2 (and checks supports/iterations), a bounded sample
    of fits for config 4."""
    import torch

    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200 import model_select as ms_mod
    from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    n, p, k_true, path = secondary_shape(a.workload)
    m = gi.PackedGenotypeMatrix.synthetic(n, p, a.seed, missing_rate=a.missing)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
    y, _ = simulate_phenotype(view, SimulationSpec(k_true=k_true, seed=a.pheno_seed))
    stream = torch.cuda.current_stream()

    def run():
        ms_mod.LAST_BATCH.clear()
        if a.workload == "c2path":
            res = gi.fit_path(view, y, path)
            return sum(r.iterations for r in res), res
        plan = gi.CvPlan.build(n, 5, path, seed=2016)
        rep = gi.cv_iht(view, y, plan, gi.IhtConfig(k=int(path.max())))
        return None, rep

    for _ in range(a.warmup):
        run()
    iters_per_step = None
    with ClockSampler(0) as clocks:
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            iters_per_step, out = run()
        torch.cuda.synchronize()  # every fit stream has drained before e1
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    line = {"metric": METRIC, "unit": "it/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64 (fp32 lookup tables)", "data": "synthetic",
            "clocks": clocks.summary()}
    data = np.array(m.data)
    ref = oracle.OraclePacked.from_bed(data, n)
    oracle.set_threads(os.cpu_count() or 1)
    rview = oracle.OracleView(ref, oracle.intercept(n))
    if a.workload == "c2path":
        line["config"] = {"workload": f"BASELINE config 2: n={n} x p={p}, model-size path "
                                      f"k=10..50 (41 cold fits), k_true={k_true}",
                          "step": "all 41 fits of the path"}
        line["value"] = iters_per_step / (ms / 1e3)
        line["fits_per_s"] = path.size / (ms / 1e3)
        if ms_mod.LAST_BATCH:
            line["xtr_batching"] = dict(ms_mod.LAST_BATCH)
        t0 = time.perf_counter()
        want = [oracle.fit(rview, y, int(k)) for k in path]
        t_cpu = time.perf_counter() - t0
        cpu_iters = sum(w.iterations for w in want)
        line["cpu_baseline"] = {"value": cpu_iters / t_cpu, "unit": "it/s",
                                "cores": os.cpu_count(), "kind": "port",
                                "sample": "the full 41-fit path on the oracle (C restatement "
                                          "of genoiht's kernels + its solver)",
                                "seconds": t_cpu}
        line["parity"] = {
            "supports_equal": all(np.array_equal(g.model.support, w.support)
                                  for g, w in zip(out, want)),
            "iterations_equal": all(g.iterations == w.iterations for g, w in zip(out, want)),
            "max_beta_rel_diff": max(float(np.max(np.abs(g.model.weights - w.weights)
                                                  / np.abs(w.weights))) if w.weights.size else 0.0
                                     for g, w in zip(out, want))}
    else:
        rep = out
        line["config"] = {"workload": f"BASELINE config 4: n={n} x p={p}, 5-fold CV over "
                                      f"k=1..20 + final fit and refit, k_true={k_true}, "
                                      f"fold seed 2016", "step": "one cv_iht call",
                          "folds": ("row masks over the resident matrix, every (fold, budget) "
                                    "fit in one lock-step group: their X^T r sweeps batched "
                                    "as a multi-RHS X^T R on the tensor cores"
                                    if ms_mod.LAST_BATCH else
                                    "compact device copies of the training rows"
                                    if ms_mod._compact_folds(m, 5) else
                                    "row masks over the resident matrix")}
        if ms_mod.LAST_BATCH:
            line["xtr_batching"] = dict(ms_mod.LAST_BATCH)
        line["value"] = None
        line["cv_seconds"] = ms / 1e3
        line["k_best"] = int(rep.k_best)
        # bounded CPU sample: one fold's re-pack (the reference re-packs the
        # training and test rows of every fold) and one fit at k = k_best
        labels = gi.make_folds(n, 5, 2016)
        train, test = np.flatnonzero(labels != 0), np.flatnonzero(labels == 0)
        t0 = time.perf_counter()
        g_train = ref.subset_rows(train)
        ref.subset_rows(test)
        t_repack = time.perf_counter() - t0
        t0 = time.perf_counter()
        fold_fit = oracle.fit(oracle.OracleView(g_train, oracle.intercept(train.size)), y[train],
                              int(rep.k_best))
        t_fit = time.perf_counter() - t0
        t_cv = 5 * t_repack + 101 * t_fit
        line["cpu_baseline"] = {"value": 1.0 / t_cv, "unit": "cv/s",
                                "cores": os.cpu_count(), "kind": "port",
                                "sample": f"oracle: one fold re-pack ({t_repack:.1f} s, x5) + one "
                                          f"fit at k={rep.k_best} ({fold_fit.iterations} "
                                          f"iterations, {t_fit:.2f} s, x101 fits); "
                                          f"extrapolated CV = {t_cv:.0f} s"}
        line["cv_per_s"] = 1.0 / (ms / 1e3)
        if a.parity:
            line["parity"] = cv_fold_parity(gi, ms_mod, view, y, path, g_train, train, test)
    print(json.dumps(line), flush=True)


def cv_fold_parity(gi, ms_mod, view, y, path, g_train, train, test):
    """Config-4 parity record at full size: fold 0's whole budget path.  The
    device fits run as cv_iht runs them (row masks over the resident matrix,
    all budgets in one lock-step group with tensor-core X^T R sweeps); the
    oracle fits the re-packed training rows as the reference does
    (model_select.py:82-139).  Support, iterations, beta and the held-out MSE
    per budget.  (The full 5-fold oracle CV takes ~4 min on 16 cores; the
    golden CV runs of tests/golden hold the complete k_best / MSE grid check.)"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    t0 = time.perf_counter()
    v_tr, v_te = ms_mod._fold_views(view, train, test, "train", False)
    jobs = []
    with ms_mod.BatchGroup(view.genotypes) as group:
        jobs = [lambda k=int(k): gi.fit(v_tr, y[train], gi.IhtConfig(k=k), _batch=group)
                for k in path]
        got = [r for r, _ in ms_mod._run_concurrently(jobs, len(jobs))]
    t_dev = time.perf_counter() - t0
    o_tr = oracle.OracleView(g_train, oracle.intercept(train.size))
    g_test = view.genotypes  # (device) test rows predicted with the training stats
    t0 = time.perf_counter()
    want = [oracle.fit(o_tr, y[train], int(k)) for k in path]
    t_cpu = time.perf_counter() - t0
    sup_eq = [bool(np.array_equal(g.model.support, w.support)) for g, w in zip(got, want)]
    it_eq = [g.iterations == w.iterations for g, w in zip(got, want)]
    beta = max((rel_diff(g.model.weights, w.weights) for g, w in zip(got, want)
                if np.array_equal(g.model.support, w.support)), default=0.0)
    mse_rel = 0.0
    for g, w in zip(got, want):
        e_g = y[test] - gi.predict(v_te, g.model)
        e_w = y[test] - gi.predict(v_te, gi.SparseModel.from_parts(w.support, w.weights, w.covar,
                                                                   g.model.k, g.model.p))
        mse_rel = max(mse_rel, abs(float(e_g @ e_g) - float(e_w @ e_w)) / float(e_w @ e_w))
    del g_test
    return {"checker": "oracle fits of fold 0's training rows (re-packed, train stats) over "
                       "the whole path, against the device fits as cv_iht runs them",
            "fold": 0, "budgets": [int(k) for k in path],
            "supports_equal": all(sup_eq), "iterations_equal": all(it_eq),
            "beta_max_rel": beta, "heldout_mse_max_rel": mse_rel,
            "device_s": t_dev, "oracle_s": t_cpu,
            "ok": bool(all(sup_eq) and all(it_eq) and beta <= 1e-6 and mse_rel <= 1e-6)}


def spawn_ranks(a):
    """`bench.py --gpus N` without a torchrun environment: launch the N ranks
    ourselves (one process per GPU, NCCL) through torch.distributed.run on
    127.0.0.1, with the same arguments; rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench: launching {a.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def rel_diff(a, b):
    """max |a - b| / |b| over the entries (inf on a shape mismatch)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return float("inf")
    if not a.size:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def parity_leg(matrix, y, k, got):
    """The fit the timed loop ran, checked against the oracle (the reference
    algorithm restated on the host and pinned to golden vectors the reference
    produced, tests/test_oracle.py) on the same bytes and response: support,
    iteration count and reason equal; beta, b_cov and the loss trace within
    1e-6 relative (north star)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    t0 = time.perf_counter()
    data = np.asarray(matrix.data)  # the verbatim BED bytes, read back from the device
    ref = oracle.OraclePacked.from_bed(data, matrix.n)
    stats_equal = bool(np.array_equal(ref.u, matrix.u) and np.array_equal(ref.v, matrix.v))
    oracle.set_threads(os.cpu_count() or 1)
    t1 = time.perf_counter()
    want = oracle.fit(oracle.OracleView(ref, oracle.intercept(matrix.n)), y, k)
    t2 = time.perf_counter()
    out = {"checker": "oracle (C + numpy restatement of genoiht, pinned to its golden vectors)",
           "support_equal": bool(np.array_equal(got.model.support, want.support)),
           "iterations_equal": got.iterations == want.iterations,
           "reason_equal": got.reason == want.reason,
           "stats_bit_identical": stats_equal,
           "beta_max_rel": rel_diff(got.model.weights, want.weights),
           "covar_max_rel": rel_diff(got.model.covar, want.covar),
           "loss_max_rel": rel_diff(got.loss_trace, want.loss_trace),
           "iterations": [got.iterations, want.iterations],
           "oracle_fit_s": t2 - t1, "readback_and_stats_s": t1 - t0}
    out["ok"] = bool(out["support_equal"] and out["iterations_equal"] and out["reason_equal"]
                     and out["beta_max_rel"] <= 1e-6 and out["loss_max_rel"] <= 1e-6)
    del data
    return out


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.impl == "reference":
        reference_arm(a)
        return
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a))
    if os.environ.get("GI_BENCH_PROBE_RANKS") == "1":  # tests: the rank launch alone
        line = json.dumps({"probe_rank": int(os.environ.get("RANK", "0")), "world": world,
                           "master_addr": os.environ.get("MASTER_ADDR")}) + "\n"
        os.write(1, line.encode())  # one write: the ranks share the pipe
        return
    if a.workload not in ("c3", "c5"):
        secondary(a)
        return
    import torch

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # GI_DIST_BACKEND=gloo lets several ranks share one GPU (host-staged
    # collectives; used to test the sharded path where only one GPU exists)
    backend = os.environ.get("GI_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200 import dist as gdist
    from paper_1608_01398_b200 import iht as giht
    from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

    # GI_FORCE_SHARDED=1 runs the sharded path (its communicator and exchange
    # steps) also at world size 1, e.g. to exercise NCCL on a single GPU
    sharded = world > 1 or os.environ.get("GI_FORCE_SHARDED") == "1"
    if sharded:
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            torch.distributed.init_process_group(backend)
        comm = gdist.TorchComm()
        geno = gdist.ShardedGenotypes.synthetic(a.n, a.p, a.seed, comm, device=local,
                                                missing_rate=a.missing)
    else:
        comm = gdist.LocalComm()
        geno = gi.PackedGenotypeMatrix.synthetic(a.n, a.p, a.seed, missing_rate=a.missing,
                                                 device=local)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    cov = gi.CovariateBlock.build(None, n=a.n)
    view = gi.StandardizedView(geno, cov)
    y, truth = simulate_phenotype(view, SimulationSpec(k_true=a.k, seed=a.pheno_seed))
    cfg = gi.IhtConfig(k=a.k)
    stream = torch.cuda.current_stream()

    def run_fit():
        return gi.fit(view, y, cfg, _resident=True)

    gi.fit(view, y, cfg)  # primes the native loop's resident inputs (sharded or not)
    nccl_info = None
    if sharded:
        nc = geno.native_comm()
        nccl_info = {"backend": nc.kind, "nranks": comm.world}
        if rank == 0:
            print(f"bench: native communicator {nc.kind}, nranks={comm.world}", file=sys.stderr,
                  flush=True)

    # ---- device-resident fits (value): the timed loop is not instrumented
    for _ in range(a.warmup):
        run_fit()
    with ClockSampler(local) as clocks:
        iters = 0
        last = None
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            last = run_fit()
            iters += last.iterations
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        ms = comm.allreduce_max(ms)
    value = iters / (ms / 1e3)

    # ---- instrumented pass (not timed): X^T r launch durations by CUDA events
    # on the fit's stream, and the kernel launches per fit (identical fits, so
    # the timed loop launched steps x this many)
    counters = {}
    n_prof = max(1, min(a.steps, 4))
    giht.profile_native(counters, time_xtr=True)
    for _ in range(n_prof):
        run_fit()
    giht.profile_native(None)
    aty_avg = counters["aty_ms"] / max(counters["aty_launches"], 1)
    launches = int(round(counters["kernel_launches"] / n_prof * a.steps))
    if world > 1:
        aty_avg = comm.allreduce_max(aty_avg)  # the slowest shard's sweep

    # ---- end to end through the public API (host y in, FitResult out)
    y_pin = torch.as_tensor(y).pin_memory().numpy()
    gi.fit(view, y_pin, cfg)
    barrier()
    torch.cuda.synchronize()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_iters = 0
    d2h = 0
    for _ in range(a.steps):
        res = gi.fit(view, y_pin, cfg)
        e2e_iters += res.iterations
        d2h += res.model.support.nbytes + res.model.weights.nbytes + res.model.covar.nbytes \
            + res.loss_trace.nbytes
    f1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = f0.elapsed_time(f1)
    if world > 1:
        e2e_ms = comm.allreduce_max(e2e_ms)
    e2e_value = e2e_iters / (e2e_ms / 1e3)

    if rank != 0:
        if sharded:
            torch.distributed.destroy_process_group()
        return

    clk = clocks.summary()
    # groups of 32 SNPs holding a missing genotype take the second lookup
    miss_frac = 0.0
    if a.missing > 0:
        local_m = geno.local if sharded else geno
        mc = local_m.missing_counts
        pad = (-mc.size) % 32
        miss_frac = float(np.mean(np.concatenate([mc, np.zeros(pad, mc.dtype)])
                                  .reshape(-1, 32).sum(axis=1) > 0)) if mc.size else 0.0
    # ---- roofline of the X^T r kernel
    n, p_local = a.n, (geno.local.p if sharded else a.p)
    nb = (n + 3) // 4
    # X^T r streams the base-3 copy (1.6 bits per genotype) when the matrix has
    # no missing genotypes, else the 2-bit BED tiles: algorithmic bytes are
    # those of the format it reads (packed X + r + u, v, s1/cnt + g)
    geno_l = geno.local if sharded else geno
    base3 = geno_l.xtr_base3
    # with missing genotypes the base-3 sweep comes with the missing-genotype
    # list (2 B per missing genotype + 8 B per 4 KiB block; csrc/missing.cu)
    mlist = base3 and geno_l.xtr_missing_list
    fmt = "base-3+missing-list" if mlist else ("base-3" if base3 else "2-bit")
    list_bytes = 0
    if mlist:
        list_bytes = 2 * int(np.sum(geno_l.missing_counts, dtype=np.int64)) + \
            8 * (((n + 511) // 512) * ((p_local + 31) // 32) + 1)
    x_bytes = (p_local * ((n + 4) // 5) + list_bytes) if base3 else p_local * nb
    alg_bytes = x_bytes + 8 * n + 24 * p_local
    achieved = alg_bytes / (aty_avg / 1e3) / 1e9
    peak, peak_kind = measured_peak()
    traffic = traffic_from_profile(n, p_local, fmt, a.missing)

    parity = None
    if world == 1 and not sharded and a.parity:
        parity = parity_leg(geno, y, a.k, last)

    cpu = None
    if world == 1 and not a.no_cpu:
        p_slice = min(a.p, a.cpu_slice or slice_snps(a.n))
        rec = reference_slice_fits(n, a.p, p_slice, a.seed, a.missing, a.k, a.pheno_seed, 3)
        cpu_value, t_it = slice_rate(rec, a.p, p_slice, skip=1)  # the first fit JITs
        cpu = {"value": cpu_value, "unit": "it/s", "cores": rec["threads"], "kind": rec["kind"],
               "sample": f"{rec['what']} with k={rec['k']} on the first {p_slice} SNPs at "
                         f"n={n} ({p_slice * nb / 1e9:.2f} GB, same bytes), 2 timed fits "
                         f"after one warm-up, per-iteration time scaled by p / p_slice = "
                         f"{a.p / p_slice:.1f}",
               "seconds_per_iteration_slice": t_it}

    h2d = 8 * n + 8 * n * cov.c  # response + covariate block uploaded per fit
    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (fp32 lookup tables)",
        "data": "synthetic (device generator, law of genoiht random_packed_matrix)",
        "config": config_of(a, world),
        "iterations_per_fit": last.iterations if last else None,
        # planted causal SNPs found by the last fit (effects ~ N(0, 0.01): the
        # smallest are below the noise, so not every one is recoverable)
        "planted_recovered": (f"{np.intersect1d(last.model.support, truth.support).size}"
                              f"/{truth.support.size}") if last is not None else None,
        # BED-equivalent: 2-bit packed genotype bytes per second per GPU (above
        # the HBM bandwidth when the kernel streams the 1.6-bit base-3 copy)
        "xtr_packed_gbs": p_local * nb / (aty_avg / 1e3) / 1e9,
        "xtr_packed_gbs_all_gpus": a.p * nb / (aty_avg / 1e3) / 1e9,
        "xtr_ms": aty_avg,
        "xtr_format": ("base-3 device copy, 5 genotypes per byte (missing as dose 0) + "
                       f"missing-genotype list ({list_bytes / 1e9:.2f} GB)" if mlist else
                       "base-3 device copy, 5 genotypes per byte (no missing genotypes)"
                       if base3 else "2-bit BED tiles"),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     # against the B200 datasheet's ~8 TB/s as well (north star)
                     "spec_peak": SPEC_HBM_GBS, "frac_of_spec": achieved / SPEC_HBM_GBS,
                     "kernel": ("missum_kernel + aty_fast_kernel (one X^T r)" if mlist
                                else "aty_fast_kernel"), "bytes_per_launch": alg_bytes,
                     "timing": f"CUDA events around each launch on the fit stream, "
                               f"separate instrumented pass of {n_prof} fits",
                     "smem": smem_roofline(n, p_local, aty_avg, clk.get("sm_mhz"),
                                           torch.cuda.get_device_properties(local)
                                           .multi_processor_count, a.missing,
                                           0.0 if mlist else miss_frac, base3)},
        "parity": parity,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "it/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h // max(a.steps, 1)},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if nccl_info is not None:
        line["comm"] = nccl_info
    print(json.dumps(line), flush=True)
    if sharded:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
