"""bench.py's reference arm on the host (no GPU): the JSON line the driver
reads, and the torchrun contract -- under N ranks rank 0 alone runs and prints,
the other ranks exit 0 without work."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["--impl", "reference", "--samples", "400", "--snps", "3000", "--cpu-slice", "1000",
         "--steps", "2", "--warmup", "1"]


def _oracle_built():
    return os.path.exists(os.path.join(ROOT, "oracle", "build", "libgenoiht_oracle.so"))


pytestmark = pytest.mark.skipif(not _oracle_built(), reason="oracle C library not built")


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    return env


def _lines(out):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_reference_arm_line():
    res = subprocess.run([sys.executable, "bench.py", *SMALL], cwd=ROOT, env=_env(),
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    (line,) = _lines(res.stdout)
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["value"] > 0 and line["unit"] == "it/s" and line["higher_is_better"] is True
    assert line["steps"] == 2 and line["warmup"] == 1 and line["n_gpus"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "it/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert "workload" in line["config"]


def test_reference_arm_under_torchrun_prints_once():
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", "29731", "bench.py", "--gpus", "2", *SMALL],
                         cwd=ROOT, env=_env(), capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    (line,) = _lines(res.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 2


def test_gpus_flag_launches_the_ranks_itself():
    """`python bench.py --gpus N` (the driver's form, no torchrun environment)
    must start N ranks itself -- one process per GPU on 127.0.0.1 -- rather
    than silently measuring one GPU.  GI_BENCH_PROBE_RANKS makes each rank
    report its place in the world and exit before touching a GPU."""
    env = _env()
    env["GI_BENCH_PROBE_RANKS"] = "1"
    for key in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(key, None)
    res = subprocess.run([sys.executable, "bench.py", "--gpus", "3", "--steps", "1",
                          "--warmup", "3"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0, res.stderr
    probes = sorted(_lines(res.stdout), key=lambda d: d["probe_rank"])
    assert [d["probe_rank"] for d in probes] == [0, 1, 2]
    assert all(d["world"] == 3 and d["master_addr"] == "127.0.0.1" for d in probes)
